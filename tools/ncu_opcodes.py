"""Executed thread-instructions per pixel by opcode from an ncu report's source page
(--import-source on).  python tools/ncu_opcodes.py rep.ncu-rep pixels [top]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, px = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
ops = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iE or not r[iE]:
        continue
    e = int(r[iE])
    tot += e
    op = re.sub(r"^\s*(@!?U?P\w+\s+)?", "", r[iS]).split(" ")[0]
    if op.startswith("IMAD.MOV") or op == "MOV":
        op = "MOV(+IMAD.MOV)"
    ops[op.split(".")[0] if not op.startswith("MOV") else op] += e
print(f"thread-instructions/px {tot * 32 / px:.1f}")
for k, v in ops.most_common(top):
    print(f"  {k:16s} {v * 32 / px:7.2f}")
