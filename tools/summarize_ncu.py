"""Summarise ncu output from gpurun_out/ into tracked files under profiles/.

  python tools/summarize_ncu.py <tag> [--launches gpurun_out/launches.csv]
         [--rep name=gpurun_out/x.ncu-rep ...] [--bench gpurun_out/bench_*.json ...]

Writes profiles/<tag>_launches.csv (kernel, duration ns), profiles/<tag>_<name>.txt
(the --page details text plus the key raw counters) and merges the per-launch
DRAM traffic into profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_utcmma.sum",
    "smsp__sass_inst_executed_op_tma_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
]
UNIT_TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--bench", action="append", default=[])
    ap.add_argument("--config", default="w4a4_4096")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[h]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        with open(os.path.join(prof, f"{a.tag}_launches.csv"), "w") as f:
            f.write("kernel,duration,unit\n")
            for r in rows[h + 1:]:
                f.write(f"\"{r[ki][:120]}\",{r[vi]},{r[ui]}\n")
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for spec in a.rep:
        name, rep = spec.split("=", 1)
        details = ncu("-i", rep, "--page", "details")
        ms = raw_metrics(rep)
        with open(os.path.join(prof, f"{a.tag}_{name}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none capture: {os.path.basename(rep)}\n")
            f.write("# key raw counters (per launch)\n")
            for d in ms:
                for k in KEYS:
                    if k in d:
                        f.write(f"{k} = {d[k][0]} {d[k][1]}\n")
            f.write("\n# --page details\n")
            f.write(details)
        d = ms[0]
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[k]
            tot += float(v.replace(",", "")) * UNIT_TO_BYTES.get(u, 1)
        traffic.setdefault(a.config, {})[f"{name}_dram_bytes"] = tot
        traffic[a.config][f"{name}_source"] = f"profiles/{a.tag}_{name}.txt"
    if a.rep:
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    if a.bench:
        with open(os.path.join(prof, f"{a.tag}_bench.jsonl"), "w") as f:
            for b in a.bench:
                for line in open(b):
                    line = line.strip()
                    if line.startswith("{"):
                        f.write(line + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
