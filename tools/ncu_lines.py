"""Per-source-line stall samples / instructions of one kernel from an ncu report (cuda,sass view).
usage: python tools/ncu_lines.py REP KERNEL_SUBSTR [TOP]"""
import csv, io, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fpath = fn = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        fn = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or kern not in (fn or ""):
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        n = int(d.get("Instructions Executed") or 0)
    except ValueError:
        continue
    key = (fpath, r[0])
    a = agg[key]
    a[0] += s; a[1] += n; a[3] = r[1][:70]
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            try: a[2][k[6:]] += int(d.get(k) or 0)
            except ValueError: pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (s, n, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{ln:>5} {s/tot*100:5.1f}% inst {n:>11d}  {src:70s} | " + " ".join(f"{k}={v}" for k, v in st.most_common(3)))
