#!/usr/bin/env python3
"""Benchmark of the flattened W4A4 / W8A8 linear layer on B200.

Workload (BASELINE.json configs[1]): a FlattenQuant-flattened W4A4 linear layer
4096x4096 at M=2048 tokens (INT4 weights packed, unpacked to int8 in shared
memory before the tcgen05 kind::i8 MMA), synthetic activations with injected
outlier channels from the reference generator (seed 42), rounded to bf16 once.
One step = flatten + quantize (K1) + INT8 tensor-core GEMM with fused dequant
epilogue to fp16 (K4) over one batch; inputs resident in HBM, L2 flushed
(256 MiB write) between timed steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N>1 (torchrun): the layer is N-sharded over ranks (global s_w), each rank runs
its column shard, outputs are all-gathered with NCCL; scaling "strong".
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "flattened W8A8/W4A4 linear TOPS (flatten+quant+GEMM) vs INT8 peak; tokens/s"
CONFIGS = {
    # name: (K, N, M, bits)
    "w4a4_4096": (4096, 4096, 2048, 4),        # BASELINE configs[1] (headline)
    "w8a8_4096_m256": (4096, 4096, 256, 8),    # configs[0]
    "llama13b_up": (5120, 13824, 2048, 4),     # configs[3]
    "sweep_8192": (8192, 8192, 8192, 8),       # configs[4] largest point
}
SPEC_INT8_TOPS = 4500.0


def peaks():
    """(HBM GB/s, bf16 TFLOP/s, source, INT8 MMA TOPS, source)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        hbm, bf16, src = float(p["hbm_gbs"]), float(p["bf16_tflops"]), "MEASURED_PEAKS.json"
    except Exception:
        hbm, bf16, src = 6650.0, 1590.0, "fallback (B200_PROFILING.md)"
    try:  # MEASURED_PEAKS.json has no INT8 figure: our tcgen05 kind::i8 microbenchmark
        with open(os.path.join(ROOT, "profiles", "measured_int8_peak.json")) as f:
            i8, i8src = float(json.load(f)["int8_mma_tops"]), "measured (tools/mma_peak.cu)"
    except Exception:
        i8, i8src = 2.0 * bf16, f"2 x bf16 ({src})"
    return hbm, bf16, src, i8, i8src


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for line in (getattr(self, "out", "") or "").splitlines():
            f = [c.strip() for c in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"], f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


from paper_2402_17985_b200.shard import gather_columns, shard_bounds  # noqa: E402


def cpu_reference_sample(k, n, bits, rows, threads, steps=1, warmup=0, recipe_layer=None):
    """Times the UNMODIFIED reference fq::run_layer (oracle/_ref), row-parallel
    over `threads` host threads, on a bounded row sample of the workload."""
    from oracle import Ref

    ref = Ref()
    w, calib, x, _ = ref.synthetic_layer(0, in_channels=k, out_channels=n, rows=32, samples=4)
    if recipe_layer is None:
        rl = ref.quantize_layer(w, calib, mode=1 if bits == 8 else 2,
                                gamma=1.86 if bits == 8 else 1e6)
    else:
        rl = ref.layer_from(recipe_layer)
    xs = np.ascontiguousarray(np.tile(x, (-(-rows // x.shape[0]), 1))[:rows])
    for _ in range(warmup):
        rl.run_layer(xs, nthreads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        rl.run_layer(xs, nthreads=threads)
        ts.append(time.perf_counter() - t0)
    kp = rl.info.Kp
    t = float(np.mean(ts))
    return {"rows": rows, "seconds": t, "tops": 2.0 * rows * n * kp / t / 1e12,
            "tokens_per_s": rows / t, "kp": kp}


def run_reference_arm(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    k, n, m, bits = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    res = cpu_reference_sample(k, n, bits, rows=args.cpu_rows or m, threads=threads,
                               steps=args.steps, warmup=max(0, min(args.warmup, 1)))
    line = {
        "impl": "reference", "metric": METRIC, "value": res["tops"], "unit": "TOPS",
        "tokens_per_s": res["tokens_per_s"], "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["seconds"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (int64 GEMM)", "data": "synthetic",
        "config": {"workload": args.config, "K": k, "N": n, "M": m, "bits": bits,
                   "Kp": res["kp"], "parallelism": "host threads"},
        "cpu_baseline": {"value": res["tops"], "unit": "TOPS", "cores": threads,
                         "kind": "reference",
                         "sample": f"{res['rows']} rows of the M={m} workload per step, "
                                   f"fq::run_layer row-parallel ({threads} threads), "
                                   "recipe from fq::quantize_layer"},
        "e2e": {"value": res["tops"], "unit": "TOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="w4a4_4096", choices=sorted(CONFIGS))
    ap.add_argument("--a-format", default="auto", choices=["auto", "i8", "i4"])
    ap.add_argument("--b-format", default="auto", choices=["auto", "i8", "i4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0, help="CPU sample rows (0: the full M)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2402_17985_b200 as fq

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if world > 1:
            dist.barrier()

    k, n, m, bits = CONFIGS[args.config]
    a_fmt = {"i8": fq.I8, "i4": fq.I4}.get(args.a_format, fq.I8)
    b_fmt = {"i8": fq.I8, "i4": fq.I4}.get(args.b_format, fq.I4 if bits == 4 else fq.I8)
    if bits == 8:
        a_fmt = b_fmt = fq.I8

    # Synthetic layer (reference generator, seed 42) -> recipe (host plan) ->
    # device weight tail (K3). Setup, untimed.
    w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    cfg = fq.quantize_layer(w, calib, bits)
    b0, b1 = shard_bounds(n, world, rank)
    layer = fq.Layer(cfg, device=local_rank, a_format=a_fmt, b_format=b_fmt, n_begin=b0,
                     n=b1 - b0)
    kp = layer.kp
    xt = torch.from_numpy(x).to(torch.bfloat16).to(f"cuda:{local_rank}")
    ldq = kp // 2 if a_fmt == fq.I4 else kp
    q = torch.empty((m, ldq), dtype=torch.int8, device=xt.device)
    y = torch.empty((m, b1 - b0), dtype=torch.float16, device=xt.device)
    rowsum = torch.empty(m, dtype=torch.int32, device=xt.device)  # K1 -> K4 (biased int4 weights)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=xt.device)
    cur = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731 (capture-aware)

    def k1():
        fq.check(fq.lib().fqg_layer_quantize_acts_ex(layer._h, xt.data_ptr(), fq.BF16, m,
                                                     q.data_ptr(), rowsum.data_ptr(), None, cur()))

    def k4():
        fq.check(fq.lib().fqg_layer_gemm_ex(layer._h, q.data_ptr(), rowsum.data_ptr(), m,
                                            y.data_ptr(), fq.F16, y.stride(0), None, fq.NONE,
                                            cur()))

    def gather():
        if world > 1:
            gather_columns(y, n)  # NCCL all-gather of the column shards -> [M, N]

    for _ in range(args.warmup):
        k1()
        k4()
        gather()
    torch.cuda.synchronize()
    barrier()
    # K1 and K4 are replayed from CUDA graphs (captured once after warm-up), so
    # the timed region measures the device, not the Python/ctypes launch path.
    # g_step holds K1 -> K4 as one graph: K4 is a programmatic dependent launch
    # (its prologue overlaps K1's tail); g_k1 / g_k4 time the kernels apart.
    g_k1, g_k4, g_step = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_k1):
        k1()
    with torch.cuda.graph(g_k4):
        k4()
    with torch.cuda.graph(g_step):
        k1()
        k4()
    for _ in range(2):
        g_k1.replay()
        g_k4.replay()
        g_step.replay()
    torch.cuda.synchronize()

    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [(E(), E(), E(), E()) for _ in range(args.steps)]
    evs_step = [(E(), E()) for _ in range(args.steps)]
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 255)
            evs_step[i][0].record()
            g_step.replay()
            evs_step[i][1].record()
            gather()
        torch.cuda.synchronize()
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 255)  # evict L2 between timed steps (not timed)
            e0, e1, e2, e3 = evs[i]
            e0.record()
            g_k1.replay()
            e1.record()
            g_k4.replay()
            e2.record()
            gather()
            e3.record()
        torch.cuda.synchronize()
        barrier()
    launches_per_step = 2 + (1 if m <= 512 else 0)  # + split-K reduce for small M
    t_k1 = sum(a.elapsed_time(b) for a, b, _, _ in evs) / args.steps
    t_k4 = sum(b.elapsed_time(c) for _, b, c, _ in evs) / args.steps
    # no collective at N = 1 (the empty e2 -> e3 pair only measures event overhead)
    t_ag = sum(c.elapsed_time(d) for _, _, c, d in evs) / args.steps if world > 1 else 0.0
    t_k1k4 = sum(a.elapsed_time(b) for a, b in evs_step) / args.steps  # one graph, PDL
    t_step = t_k1k4 + t_ag
    if world > 1:
        tt = torch.tensor([t_step, t_k1, t_k4, t_ag, t_k1k4], dtype=torch.float64,
                          device=xt.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_k1, t_k4, t_ag, t_k1k4 = tt.tolist()

    # ---- e2e: the reference-facing drop-in call with HOST f64 buffers ----
    xh = torch.from_numpy(x).to(torch.bfloat16).double().pin_memory().numpy()
    yh = torch.empty((m, b1 - b0), dtype=torch.float64).pin_memory().numpy()
    for _ in range(2):  # warm: the pool grows to the full-size buffers, streams exist
        fq.check(fq.lib().fqg_layer_run_host(layer._h, xh.ctypes.data, m, yh.ctypes.data,
                                             ctypes.byref(ctypes.c_int64())))
    te = []
    sat = ctypes.c_int64()
    for _ in range(args.e2e_steps):
        barrier()
        t0 = time.perf_counter()
        fq.check(fq.lib().fqg_layer_run_host(layer._h, xh.ctypes.data, m, yh.ctypes.data,
                                             ctypes.byref(sat)))
        te.append(time.perf_counter() - t0)
    t_e2e = float(np.mean(te))
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device=xt.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = tt.item()

    ops = 2.0 * m * n * kp  # whole layer (all ranks), reference bitops K' (pipeline.cpp:211)
    tops = ops / (t_step * 1e-3) / 1e12
    hbm_gbs, bf16_tf, peak_src, int8_peak, i8_src = peaks()
    gemm_ops_rank = 2.0 * m * (b1 - b0) * kp
    gemm_tops = gemm_ops_rank / (t_k4 * 1e-3) / 1e12
    k1_bytes = m * k * 2 + m * ldq + kp * 4 + k * 12
    k1_gbs = k1_bytes / (t_k1 * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config, {})
            traffic = tr.get("gemm_dram_bytes")
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": tops, "unit": "TOPS",
        "tokens_per_s": m / (t_step * 1e-3),
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int8 MMA / int32 accumulate (4-bit values)" if bits == 4 else
                 "int8 MMA / int32 accumulate",
        "data": "synthetic (fq::make_synthetic_layer generator, seed 42, 1% outlier channels x "
                "U[20,100]); activations rounded to bf16",
        "config": {"workload": args.config, "K": k, "N": n, "M": m, "bits": bits, "Kp": kp,
                   "flatten_ratio_x": cfg.plan_x.flatten_ratio(),
                   "a_format": "i4 packed" if a_fmt == fq.I4 else "i8",
                   "b_format": "i4 packed" if b_fmt == fq.I4 else "i8",
                   "out_dtype": "fp16", "parallelism": f"N-shard x{world}" if world > 1 else "1 GPU",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "breakdown_ms": {"flatten_quant_K1": t_k1, "gemm_K4": t_k4, "all_gather": t_ag,
                         "K1_K4_graph": t_k1k4},
        "roofline": {"bound": "tensor", "achieved": gemm_tops, "peak": int8_peak,
                     "unit": "TFLOP/s", "frac": gemm_tops / int8_peak, "traffic": traffic,
                     "kernel": "k_gemm_i8_pair (tcgen05.mma.cta_group::2.kind::i8, 256x512 tiles)",
                     "peak_basis": f"tcgen05 kind::i8 MMA peak, {i8_src}; frac vs spec 4.5 "
                                   f"POPS: {gemm_tops / SPEC_INT8_TOPS:.3f}; vs 2 x bf16 "
                                   f"measured ({peak_src}): {gemm_tops / (2 * bf16_tf):.3f}",
                     "effective_tops_on_K": 2.0 * m * (b1 - b0) * k / (t_k4 * 1e-3) / 1e12},
        "roofline_k1": {"bound": "hbm", "achieved": k1_gbs, "peak": hbm_gbs, "unit": "GB/s",
                        "frac": k1_gbs / hbm_gbs, "bytes_per_launch": k1_bytes},
        "e2e": {"value": ops / t_e2e / 1e12, "unit": "TOPS",
                "tokens_per_s": m / t_e2e,
                "h2d_bytes_per_step": m * k * 8, "d2h_bytes_per_step": m * (b1 - b0) * 8 + 8,
                "api": "fqg_layer_run_host (drop-in fq::run_layer, f64 host buffers, pinned)"},
        "gpu_launches": launches_per_step * args.steps,  # the headline (one-graph) loop;
        # the per-kernel loop launches the same number again
        "launch": "one CUDA graph per step (K1, then K4 as a programmatic dependent launch); "
                  "K1 and K4 also timed apart from their own graphs for the rooflines",
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rec = __import__("oracle").Layer(
            bits=bits, s=cfg.smooth_scales, t_x=cfg.plan_x.threshold, e_x=cfg.plan_x.extensions,
            t_w=cfg.plan_w.threshold, e_w=cfg.plan_w.extensions, wq=layer.weight_q(),
            s_w=layer.w_scale, act_scale=cfg.act_scale)
        res = cpu_reference_sample(k, n, bits, rows=args.cpu_rows or m, threads=threads,
                                   recipe_layer=rec)
        line["cpu_baseline"] = {
            "value": res["tops"], "unit": "TOPS", "cores": threads, "kind": "reference",
            "tokens_per_s": res["tokens_per_s"],
            "sample": f"{res['rows']} rows of the same layer/recipe, unmodified fq::run_layer "
                      f"(oracle/_ref) row-parallel on {threads} host threads, "
                      f"{res['seconds']:.2f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
