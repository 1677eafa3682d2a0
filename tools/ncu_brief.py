"""One-screen summary of an ncu --set full report: time, DRAM, issue, occupancy, stall reasons,
pipes, instruction count per pixel (if px given).  python tools/ncu_brief.py rep.ncu-rep [pixels]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
px = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))

    def g(k, default=float("nan")):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return default
    print(d.get("Kernel Name", "")[:100])
    un = dict(zip(h, units))
    print(f"duration {d.get('gpu__time_duration.sum')} {un.get('gpu__time_duration.sum')}  "
          f"dram read {d.get('dram__bytes_read.sum')} {un.get('dram__bytes_read.sum')}  "
          f"write {d.get('dram__bytes_write.sum')} {un.get('dram__bytes_write.sum')}  "
          f"dram {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of peak")
    inst = g("smsp__inst_executed.sum")
    print(f"warp-inst {inst:.4g}" + (f"  thread-inst/px {inst * 32 / px:.1f}" if px else "") +
          f"  issue-active {g('sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%"
          f"  warps/SM {g('sm__warps_active.avg.per_cycle_active'):.1f}  regs {g('launch__registers_per_thread'):.0f}")
    print(f"pipes: fma {g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"fmaheavy {g('sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"alu {g('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"xu {g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"lsu {g('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):.1f}%  "
          f"local ld/st {g('sass__inst_executed_local_loads'):.3g}/{g('sass__inst_executed_local_stores'):.3g}")
    st = sorted(((g(k, 0), k) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")), reverse=True)
    print("stalls/issue: " + "  ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {val:.2f}" for val, k in st[:9]))
