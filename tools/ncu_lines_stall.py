"""Per-CUDA-source-line warp stall samples from an ncu report (cuda,sass source view).

    python tools/ncu_lines_stall.py REP.ncu-rep [TOP]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
rows = {}
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    key = (f, int(r[0]))
    d = rows.setdefault(key, [0, r[1]])
    d[0] += s
tot = sum(v[0] for v in rows.values()) or 1
for (f, ln), (s, src) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s / tot * 100:6.2f}%  {f}:{ln:<5d} {src.strip()[:110]}")
