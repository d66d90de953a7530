"""Per-CUDA-source-line warp-stall samples from an ncu report (cuda,sass source view).
usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
si = h.index("Warp Stall Sampling (All Samples)")
agg = {}; src = {}; tot = 0
for r in rows[hdr_i + 1:]:
    if len(r) <= si or not r[0].strip().isdigit():
        continue
    ln = int(r[0]); src.setdefault(ln, r[1])
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    agg[ln] = agg.get(ln, 0) + v; tot += v
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100*v/max(tot,1):5.1f}%  L{ln:4d}  {src[ln].strip()[:110]}")
