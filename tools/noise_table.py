#!/usr/bin/env python
"""Table VII-style accuracy under depth noise
on the seeded synthetic scenes — NOT the paper's datasets, so the numbers are this workload's,
not a reproduction of the paper's table.  GPU path + a8 stats kernel; prints a markdown table
of e_A (AAE, degrees) and PGP_10 for every filter x Phi at the S:374 noise presets.

    python tools/noise_table.py [--frames 64]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_08165_b200 as tfn  # noqa: E402
import tfn_scenes as ts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    sc = ts.random_scenes(a.frames, ts.K_VGA, 480, 640, seed=a.seed)
    r = ts.render(sc, ts.K_VGA, 480, 640, device="cuda")
    levels = [("clean", 0.0)] + list(ts.NOISE_PRESETS.items())
    rows = []
    for f in ("fd", "sobel", "scharr", "prewitt"):
        for m in ("mean", "median"):
            est = tfn.Estimator(ts.K_VGA, f, m)
            cells = []
            for name, rel in levels:
                z = ts.add_gaussian_noise(r.depth, rel, seed=a.seed + 1)
                acc = tfn.stats(est.estimate(z), r.gt).cpu().tolist()
                cells.append((acc[0] / 1e6 / acc[1], acc[2] / acc[1]))
            rows.append((f"{f.upper() if f == 'fd' else f.capitalize()}-{m.capitalize()}", cells))
    hdr = " | ".join(f"{n} ({100 * rel:.1f} %) e_A / PGP10" if rel else "clean e_A / PGP10" for n, rel in levels)
    print(f"| SNE | {hdr} |")
    print("|---|" + "---|" * len(levels))
    for name, cells in rows:
        print(f"| {name} | " + " | ".join(f"{e:.3f}° / {p:.4f}" for e, p in cells) + " |")
    print(f"\n{a.frames} frames 480x640 (seeded plane + sphere scenes, seed {a.seed}); sigma = preset x mean valid depth")


if __name__ == "__main__":
    main()
