"""Summarise an ncu report: time, instructions, and the hottest source lines / SASS regions."""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:70])
    for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__registers_per_thread"):
        print("  ", k, d.get(k))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ie = h.index("Instructions Executed"); ist = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) > ie and r[0].isdigit():
        try:
            data.append((int(r[ie]), int(r[ist]), int(r[0]), r[1][:90]))
        except ValueError:
            pass
print("total inst", sum(d[0] for d in data), "stall samples", sum(d[1] for d in data))
for d in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(d)
