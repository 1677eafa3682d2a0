import sys, numpy as np, torch
sys.path.insert(0, '.')
import tfn_scenes as ts, paper_2005_08165_b200 as tfn
r = ts.render(ts.config1_scene(), ts.K_VGA, 480, 640)
x = r.depth.cuda()
for mode in ("mean", "median"):
    a = tfn.Estimator(ts.K_VGA, "sobel", mode, kernel="strip").estimate(x).cpu().numpy()
    b = tfn.Estimator(ts.K_VGA, "sobel", mode, kernel="pixel").estimate(x).cpu().numpy()
    d = a.view(np.uint32) != b.view(np.uint32)
    idx = np.argwhere(d.any(1))
    print(mode, "mismatch px", len(idx))
    for (bb, v, u) in idx[:8]:
        print(v, u, a[bb, :, v, u], b[bb, :, v, u], [hex(q) for q in a[bb, :, v, u].view(np.uint32)], [hex(q) for q in b[bb, :, v, u].view(np.uint32)])
