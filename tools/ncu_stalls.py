"""Stall-reason totals and the top SASS lines per reason from an ncu report.
usage: python tools/ncu_stalls.py REPORT [reason ...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]; body = [r for r in rows[hi + 1:] if len(r) == len(h)]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
def f(x):
    try: return float(x or 0)
    except ValueError: return 0.0
tot = {c: sum(f(r[h.index(c)]) for r in body) for c in cols}
T = sum(tot.values())
print("totals:", ", ".join(f"{c[6:]}={100*v/T:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
for c in sys.argv[2:]:
    ci = h.index("stall_" + c)
    top = sorted(body, key=lambda r: -f(r[ci]))[:8]
    print(f"-- {c}")
    for r in top:
        print(f"  {100*f(r[ci])/T:5.2f}%  {r[0]}  {r[1][:90]}")
