"""Per-region (split at barriers / mbarrier waits) instruction and stall-sample
totals of one kernel from an ncu report: python tools/sass_regions.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
si, ws, ie = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
    "Instructions Executed")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
sidx = [hdr.index(h) for h in stalls]
f = lambda v: float(v or 0)  # noqa: E731
tot_i = sum(f(r[ie]) for r in data)
tot_s = sum(f(r[ws]) for r in data)
print(f"total inst {tot_i:.0f}, samples {tot_s:.0f}")
start, acc = 0, []
cur = [0.0, 0.0, {}]
for n, r in enumerate(data):
    if "BAR.SYNC" in r[si] or "SYNCS.PHASECHK" in r[si]:
        acc.append((start, n, cur))
        cur, start = [0.0, 0.0, {}], n
    cur[0] += f(r[ie])
    cur[1] += f(r[ws])
    for h, i in zip(stalls, sidx):
        cur[2][h] = cur[2].get(h, 0.0) + f(r[i])
acc.append((start, len(data), cur))
for a, b, (i, s, st) in acc:
    if i < 0.005 * tot_i and s < 0.01 * tot_s:
        continue
    tops = sorted(((v, k[6:]) for k, v in st.items()), reverse=True)[:3]
    print(f"[{a:5d},{b:5d}) inst {i:10.0f} ({100*i/tot_i:4.1f}%) samples {100*s/tot_s:4.1f}%  "
          + " ".join(f"{k}={v:.0f}" for v, k in tops) + f"  | {data[a][si].strip()[:40]}")
if top:
    for n in sorted(range(len(data)), key=lambda n: -f(data[n][ie]))[:top]:
        print(n, data[n][ie], data[n][si].strip()[:80])
