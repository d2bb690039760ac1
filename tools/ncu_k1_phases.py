"""K1 instruction counts per phase (source-line ranges of flatten16.cu) from an ncu report's CSV source page."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
cur = None; out = []; hdr = None
for r in rows:
    if not r: continue
    if r[0] in ("File Path", "File Name"): cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No": hdr = r; ie = r.index("Instructions Executed"); continue
    if hdr and r[0].isdigit() and len(r) > ie:
        try: out.append((cur, int(r[0]), int(r[ie]), r[1]))
        except ValueError: pass
byf = collections.Counter()
for f, l, n, s in out: byf[f] += n
print(dict(byf))
srcf = sys.argv[2] if len(sys.argv) > 2 else "paper_2402_17985_b200/csrc/flatten16.cu"
marks = [(i + 1, t.strip()) for i, t in enumerate(open(srcf).read().splitlines())
         if t.strip().startswith("// ----") or "k_flatten16(const" in t]
print(marks)
cnt = {l: n for f, l, n, s in out if f == 'flatten16.cu'}
bounds = [l for l, _ in marks] + [10**9]
for i, (l, s) in enumerate(marks):
    print(f"{s[:60]:60s} {sum(n for ll, n in cnt.items() if bounds[i] <= ll < bounds[i+1])}")
print("before kernel (helpers/lambdas):", sum(n for ll, n in cnt.items() if ll < bounds[0]))
