"""Read `ncu --csv --metrics smsp__inst_executed.sum,gpu__time_duration.sum,...` from stdin and
print thread-instructions per pixel of a config-2 launch (1024 x 480x640 px) — tools/ab_inst.sh."""
import csv
import sys

rows = list(csv.reader(l for l in sys.stdin if l.startswith('"')))
h = [r for r in rows if "Metric Name" in r][0]
m = {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows if r is not h and len(r) == len(h)}
px = 1024 * 480 * 640
inst = float(m["smsp__inst_executed.sum"].replace(",", ""))
print(sys.argv[1], "inst/px %.1f" % (inst * 32 / px), "ms", m["gpu__time_duration.sum"],
      "regs", m.get("launch__registers_per_thread"))
