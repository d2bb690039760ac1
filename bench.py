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

N > 1: run under torchrun (or let --gpus N re-launch this script under
torch.distributed.run itself). The layer is N-sharded over the ranks (global
s_w): each rank runs K1 on the replicated input and K4 on its column shard,
writing straight into its slot of a shard-major buffer, and the slots are
all-gathered in place with NCCL; scaling "strong" (fixed total work), timed as
the max over ranks.

At N = 1 the line also carries `subresults` for the other BASELINE configs
(configs[0], [2], [3] one-GPU shards, [4] M sweep), each with value, ms, the
K1/K4 split and the K4 roofline fraction (--no-subresults skips them).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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
OPT67B = [("qkv", 4096, 12288, 4), ("o", 4096, 4096, 8), ("fc1", 4096, 16384, 4),
          ("fc2", 16384, 4096, 8)]                  # configs[2], M = 2048
SWEEP_M = [1, 16, 128, 256, 512, 1024, 2048, 4096, 8192]  # configs[4]
SPEC_INT8_TOPS = 4500.0


def gemm_label(fq, m, n, kp, a_fmt, b_fmt):
    """K4's launch plan for this shape, as fqg_gemm_plan reports it."""
    from paper_2402_17985_b200 import _lib

    info = _lib.GemmPlan()
    fq.check(fq.lib().fqg_gemm_plan(m, n, kp, a_fmt, b_fmt, _lib.F16, ctypes.byref(info)))
    name = ("k_gemm_i8_pair (tcgen05.mma.cta_group::2.kind::i8" if info.kernel == 2 else
            "k_gemm_i8 (tcgen05.mma.cta_group::1.kind::i8")
    split = f", split-K x{info.splits}" if info.splits > 1 else ""
    return f"{name}, {info.tile_m}x{info.tile_n} tiles{split}, {info.ctas} CTAs)"


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


def relaunch_distributed(nproc: int) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


from paper_2402_17985_b200.shard import shard_bounds, shard_width  # noqa: E402


def reference_recipe(ref, w, calib, bits):
    """The reference's own fq::quantize_layer (O1 INT8 / O2 forced INT4)."""
    return ref.quantize_layer(w, calib, mode=1 if bits == 8 else 2,
                              gamma=1.86 if bits == 8 else 1e6)


def time_reference(rl, xs, threads, steps=1, warmup=0):
    for _ in range(warmup):
        rl.run_layer(xs, nthreads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        rl.run_layer(xs, nthreads=threads)
        ts.append(time.perf_counter() - t0)
    return float(np.mean(ts))


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    fq_core compiled from /root/reference sources) on the same synthetic input
    rows as the GPU arm, row-parallel over all host threads."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    from oracle import Ref

    import paper_2402_17985_b200 as fq  # host-only: the synthetic generator

    k, n, m, bits = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    ref = Ref()
    w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    xs = bf16_round(x)
    rows = args.cpu_rows or m
    xs = np.ascontiguousarray(xs[:rows])
    rl = reference_recipe(ref, w, calib, bits)
    t = time_reference(rl, xs, threads, steps=args.steps, warmup=max(0, min(args.warmup, 1)))
    kp = rl.info.Kp
    tops = 2.0 * rows * n * kp / t / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tops, "unit": "TOPS",
        "tokens_per_s": rows / t, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (int64 GEMM)", "data": "synthetic",
        "config": {"workload": args.config, "K": k, "N": n, "M": m, "bits": bits, "Kp": kp,
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": tops, "unit": "TOPS", "cores": threads, "kind": "reference",
                         "sample": f"{rows} rows of the M={m} workload per step (the GPU arm's "
                                   f"synthetic rows, bf16-rounded), fq::run_layer row-parallel "
                                   f"({threads} threads), recipe from fq::quantize_layer"},
        "e2e": {"value": tops, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def bf16_round(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).double().numpy()


class LayerBench:
    """K1 + K4 of one layer replayed from CUDA graphs: the step graph (K1, then K4
    as a programmatic dependent launch) and K1 / K4 graphs of their own for the
    split. L2 flushed (256 MiB write) before every timed replay."""

    def __init__(self, fq, layer, xt, out=None, flush=None):
        import torch

        self.fq, self.layer, self.xt = fq, layer, xt
        m = xt.shape[0]
        self.m = m
        kp = layer.kp
        ldq = kp // 2 if layer.info.a_format == fq.I4 else kp
        dev = xt.device
        self.q = torch.empty((m, ldq), dtype=torch.int8, device=dev)
        self.rowsum = torch.empty(m, dtype=torch.int32, device=dev)
        self.sat = torch.zeros(1, dtype=torch.int64, device=dev)
        self.y = out if out is not None else torch.empty((m, layer.n), dtype=torch.float16,
                                                         device=dev)
        self.flush = flush if flush is not None else torch.empty(256 << 20, dtype=torch.uint8,
                                                                 device=dev)
        self.graphs = None
        self.k1_runs = 0  # K1 executions (the saturation counter accumulates over all)

    def k1(self):
        import torch

        self.k1_runs += 1
        self.fq.check(self.fq.lib().fqg_layer_quantize_acts_ex(
            self.layer._h, self.xt.data_ptr(), self.fq.BF16, self.m, self.q.data_ptr(),
            self.rowsum.data_ptr(), self.sat.data_ptr(), torch.cuda.current_stream().cuda_stream))

    def k4(self):
        import torch

        self.fq.check(self.fq.lib().fqg_layer_gemm_ex(
            self.layer._h, self.q.data_ptr(), self.rowsum.data_ptr(), self.m, self.y.data_ptr(),
            self.fq.F16, self.y.stride(0), None, self.fq.NONE,
            torch.cuda.current_stream().cuda_stream))

    def capture(self, warmup):
        """Graphs: step (K1, K4), K1 alone, K4 alone. Each carries external event
        record nodes around its kernels, so the device time of the kernels is read
        without the graph's launch latency (a model replays all its layers from
        one graph); events outside the graph give the launch-inclusive time."""
        import torch

        for _ in range(warmup):
            self.k1()
            self.k4()
        torch.cuda.synchronize()
        E = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731
        self.ev_in = {name: (E(), E()) for name in ("step", "k1", "k4")}
        g1, g4, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            self.ev_in["k1"][0].record()
            self.k1()
            self.ev_in["k1"][1].record()
        with torch.cuda.graph(g4):
            self.ev_in["k4"][0].record()
            self.k4()
            self.ev_in["k4"][1].record()
        with torch.cuda.graph(gs):
            self.ev_in["step"][0].record()
            self.k1()
            self.k4()
            self.ev_in["step"][1].record()
        self.k1_runs -= 3  # the captures did not execute
        for _ in range(2):
            g1.replay()
            g4.replay()
            gs.replay()
        self.k1_runs += 4
        torch.cuda.synchronize()
        self.graphs = (g1, g4, gs)

    def time(self, steps, after_step=None):
        """Means over `steps` flushed replays, in ms: (t_step, t_k1, t_k4, t_after,
        t_step_launch). t_step / t_k1 / t_k4 are device times between the event
        nodes inside the graphs; t_step_launch brackets the graph launch itself."""
        import torch

        g1, g4, gs = self.graphs
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        acc = {"step": [], "k1": [], "k4": [], "after": [], "launch": []}

        def inner(name):
            a, b = self.ev_in[name]
            return a.elapsed_time(b)

        # launch-inclusive pass: events around the replays, no host syncs in between
        ev = [(E(), E(), E()) for _ in range(steps)]
        for i in range(steps):
            self.flush.fill_(i & 255)
            ev[i][0].record()
            gs.replay()
            ev[i][1].record()
            if after_step is not None:
                after_step()
            ev[i][2].record()
        torch.cuda.synchronize()
        acc["launch"] = [a.elapsed_time(b) for a, b, _ in ev]
        acc["after"] = [b.elapsed_time(c) for _, b, c in ev]
        # device pass: the in-graph event nodes (read after each replay)
        for i in range(steps):
            self.flush.fill_(i & 255)
            gs.replay()
            torch.cuda.synchronize()  # the in-graph events are re-recorded by every replay
            acc["step"].append(inner("step"))
        for i in range(steps):
            self.flush.fill_(i & 255)
            g1.replay()
            torch.cuda.synchronize()
            acc["k1"].append(inner("k1"))
            g4.replay()  # (K1's operand is in L2, as inside the step)
            torch.cuda.synchronize()
            acc["k4"].append(inner("k4"))
        self.k1_runs += 3 * steps
        mean = lambda v: float(sum(v) / len(v))  # noqa: E731
        return (mean(acc["step"]), mean(acc["k1"]), mean(acc["k4"]), mean(acc["after"]),
                mean(acc["launch"]))


    def time_chain(self, reps=5, nchain=8, make_layer=None):
        """Average launch duration of K1 and of K4 (ms) from graphs of nchain back-to-back
        launches on nchain distinct inputs (x: nchain x M x K bf16, q: nchain x M x K'
        int8 -- more than the 126 MB L2 -- and, with make_layer, nchain device copies of
        the layer so no launch finds its weights in L2), event nodes at both ends; the
        node and launch overheads a single launch carries are shared by the chain."""
        import torch

        layers = [make_layer() for _ in range(nchain)] if make_layer else [self.layer] * nchain
        dev = self.xt.device
        xs = [self.xt.clone() for _ in range(nchain)]
        qs = [torch.empty_like(self.q) for _ in range(nchain)]
        rss = [torch.empty_like(self.rowsum) for _ in range(nchain)]
        ys = [torch.empty_like(self.y) for _ in range(nchain)]
        st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

        def k1(i):
            self.fq.check(self.fq.lib().fqg_layer_quantize_acts_ex(
                layers[i]._h, xs[i].data_ptr(), self.fq.BF16, self.m, qs[i].data_ptr(),
                rss[i].data_ptr(), None, st()))

        def k4(i):
            self.fq.check(self.fq.lib().fqg_layer_gemm_ex(
                layers[i]._h, qs[i].data_ptr(), rss[i].data_ptr(), self.m, ys[i].data_ptr(),
                self.fq.F16, ys[i].stride(0), None, self.fq.NONE, st()))

        for i in range(nchain):
            k1(i)
            k4(i)
        torch.cuda.synchronize()
        E = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731
        e1, e4, es = (E(), E()), (E(), E()), (E(), E())
        g1, g4, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            e1[0].record()
            for i in range(nchain):
                k1(i)
            e1[1].record()
        with torch.cuda.graph(g4):
            e4[0].record()
            for i in range(nchain):
                k4(i)
            e4[1].record()
        with torch.cuda.graph(gs):  # whole layer steps back to back (as a model's layers run)
            es[0].record()
            for i in range(nchain):
                k1(i)
                k4(i)
            es[1].record()
        t1, t4, ts = [], [], []
        for r in range(reps + 1):
            self.flush.fill_(r & 255)
            g1.replay()
            torch.cuda.synchronize()
            if r:
                t1.append(e1[0].elapsed_time(e1[1]) / nchain)
            self.flush.fill_((r + 7) & 255)
            g4.replay()
            torch.cuda.synchronize()
            if r:
                t4.append(e4[0].elapsed_time(e4[1]) / nchain)
            self.flush.fill_((r + 13) & 255)
            gs.replay()
            torch.cuda.synchronize()
            if r:
                ts.append(es[0].elapsed_time(es[1]) / nchain)
        del xs, qs, rss, ys, g1, g4, gs, layers
        torch.cuda.empty_cache()
        self.t_step_chain = float(np.mean(ts))
        return float(np.mean(t1)), float(np.mean(t4))


def layer_result(fq, cfg, k, n, m, bits, x, steps, warmup, i8_peak, n_begin=0, n_cols=None,
                 flush=None):
    """One layer's bench entry (value, ms, K1/K4 split, K4 roofline fraction)."""
    import torch

    b_fmt = fq.I4 if bits == 4 else fq.I8
    n_cols = n if n_cols is None else n_cols
    layer = fq.Layer(cfg, a_format=fq.I8, b_format=b_fmt, n_begin=n_begin, n=n_cols)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    lb = LayerBench(fq, layer, xt, flush=flush)
    lb.capture(warmup)
    t_step, t_k1, t_k4, _, t_launch = lb.time(steps)
    t_k1c, t_k4c = lb.time_chain(reps=3, make_layer=lambda: fq.Layer(
        cfg, a_format=fq.I8, b_format=b_fmt, n_begin=n_begin, n=n_cols))
    ops = 2.0 * m * n_cols * layer.kp
    res = {"K": k, "N": n_cols, "M": m, "bits": bits, "Kp": layer.kp,
           "value": ops / (t_step * 1e-3) / 1e12, "unit": "TOPS", "ms_per_step": t_step,
           "tokens_per_s": m / (t_step * 1e-3),
           "breakdown_ms": {"flatten_quant_K1": t_k1, "gemm_K4": t_k4, "K1_K4_graph": t_step},
           "kernel_ms": {"flatten_quant_K1": t_k1c, "gemm_K4": t_k4c},
           "ms_per_step_with_launch": t_launch,
           "roofline_frac_K4": ops / (t_k4c * 1e-3) / 1e12 / i8_peak,
           "roofline_frac_K4_single_launch": ops / (t_k4 * 1e-3) / 1e12 / i8_peak}
    del lb, layer, xt
    torch.cuda.empty_cache()
    return res


def subresults(fq, args, i8_peak, flush):
    """configs[0], [2], [3] (one-GPU shards), [4] at N = 1."""
    out = {}
    k, n, m, bits = CONFIGS["w8a8_4096_m256"]
    w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    cfg = fq.quantize_layer(w, calib, bits)
    out["configs[0] w8a8_4096_m256"] = layer_result(fq, cfg, k, n, m, bits, bf16_round(x), 20,
                                                    5, i8_peak, flush=flush)
    opt, tot_ops, tot_t = {}, 0.0, 0.0
    for i, (name, k, n, bits) in enumerate(OPT67B):
        w, calib, x = fq.synthetic_layer(i + 1, test_rows=2048, in_channels=k, out_channels=n,
                                         rows=32, samples=4)
        cfg = fq.quantize_layer(w, calib, bits)
        r = layer_result(fq, cfg, k, n, 2048, bits, bf16_round(x), 10, 3, i8_peak, flush=flush)
        opt[name] = r
        tot_ops += r["value"] * r["ms_per_step"] * 1e9
        tot_t += r["ms_per_step"]
    out["configs[2] opt6.7b_m2048"] = {"layers": opt, "value": tot_ops / (tot_t * 1e-3) / 1e12,
                                       "unit": "TOPS", "ms_per_block": tot_t,
                                       "bits": "qkv/fc1 4-bit, o/fc2 8-bit (pinned)"}
    k, n, m, bits = CONFIGS["llama13b_up"]
    w, calib, x = fq.synthetic_layer(13, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    cfg = fq.quantize_layer(w, calib, bits)
    xb = bf16_round(x)
    ll = {}
    for world in (1, 2, 4, 8):
        b0, b1 = shard_bounds(n, world, 0)
        ll[f"shard_of_{world}"] = layer_result(fq, cfg, k, n, m, bits, xb, 10, 3, i8_peak,
                                               n_begin=b0, n_cols=b1 - b0, flush=flush)
    out["configs[3] llama13b_up_m2048 (per-GPU shard, no collective)"] = ll
    k, n, _, bits = CONFIGS["sweep_8192"]
    w, calib, x = fq.synthetic_layer(21, test_rows=max(SWEEP_M), in_channels=k, out_channels=n,
                                     rows=32, samples=4)
    cfg = fq.quantize_layer(w, calib, bits)
    xb = bf16_round(x)
    sw = {}
    for m in SWEEP_M:
        sw[f"M={m}"] = layer_result(fq, cfg, k, n, m, bits, np.ascontiguousarray(xb[:m]),
                                    10 if m >= 1024 else 20, 3, i8_peak, flush=flush)
    out["configs[4] sweep_8192_int8"] = sw
    out["k1_general_f64 (drop-in device path, headline layer)"] = k1_general(fq, flush)
    return out


def k1_general(fq, flush, steps=20):
    """K1 on f64 activations (the path fqg_layer_run_host / fq::gpu::run_layer take on
    the device, general kernel of flatten.cu) at the headline shape, against HBM."""
    import torch

    k, n, m, bits = CONFIGS["w4a4_4096"]
    w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    cfg = fq.quantize_layer(w, calib, bits)
    layer = fq.Layer(cfg, a_format=fq.I8, b_format=fq.I4)
    xd = torch.from_numpy(np.ascontiguousarray(bf16_round(x))).cuda()  # f64, the drop-in's input
    q = torch.empty((m, layer.kp), dtype=torch.int8, device="cuda")
    rs = torch.empty(m, dtype=torch.int32, device="cuda")

    def k1():
        fq.check(fq.lib().fqg_layer_quantize_acts_ex(
            layer._h, xd.data_ptr(), fq.F64, m, q.data_ptr(), rs.data_ptr(), None,
            torch.cuda.current_stream().cuda_stream))

    for _ in range(3):
        k1()
    torch.cuda.synchronize()
    E = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731
    e0, e1 = E(), E()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        e0.record()
        k1()
        e1.record()
    ts = []
    for i in range(steps):
        flush.fill_(i & 255)
        g.replay()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.mean(ts))
    nbytes = m * k * 8 + m * layer.kp
    hbm = peaks()[0]
    res = {"ms": t, "bytes_per_launch": nbytes, "GB/s": nbytes / (t * 1e-3) / 1e9,
           "frac_hbm": nbytes / (t * 1e-3) / 1e9 / hbm, "M": m, "K": k, "Kp": layer.kp}
    del layer, xd, q, rs
    torch.cuda.empty_cache()
    return res


def cpu_baseline(fq, cfg, layer, x, bits, k, n, m):
    """The unmodified reference fq::run_layer (oracle/_ref) on the same recipe and
    rows: all host threads on the full batch, and one thread on a row sample."""
    from oracle import Layer as OLayer
    from oracle import Ref

    ref = Ref()
    rec = OLayer(bits=bits, s=cfg.smooth_scales, t_x=cfg.plan_x.threshold,
                 e_x=cfg.plan_x.extensions, t_w=cfg.plan_w.threshold, e_w=cfg.plan_w.extensions,
                 wq=layer.weight_q(), s_w=layer.w_scale, act_scale=cfg.act_scale)
    rl = ref.layer_from(rec)
    threads = os.cpu_count() or 1
    t_all = time_reference(rl, np.ascontiguousarray(x), threads)
    rows1 = 16
    t_one = time_reference(rl, np.ascontiguousarray(x[:rows1]), 1)
    kp = layer.kp
    return {
        "value": 2.0 * m * n * kp / t_all / 1e12, "unit": "TOPS", "cores": threads,
        "kind": "reference", "tokens_per_s": m / t_all,
        "sample": f"{m} rows of the same layer/recipe, unmodified fq::run_layer (oracle/_ref) "
                  f"row-parallel on {threads} host threads, {t_all:.2f} s",
        "single_thread": {"value": 2.0 * rows1 * n * kp / t_one / 1e12, "unit": "TOPS",
                          "tokens_per_s": rows1 / t_one, "cores": 1,
                          "sample": f"{rows1} rows, one thread, {t_one:.2f} s"},
    }


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
    ap.add_argument("--no-subresults", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0, help="CPU sample rows (0: the full M)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--chunks", type=int, default=1, help="N > 1: GEMM/all-gather M-chunks")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, local_rank, world = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    if args.impl == "reference":
        return run_reference_arm(args)
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")

    import torch
    import torch.distributed as dist

    import paper_2402_17985_b200 as fq

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
    width = shard_width(n, world)
    layer = fq.Layer(cfg, device=local_rank, a_format=a_fmt, b_format=b_fmt, n_begin=b0,
                     n=b1 - b0)
    kp = layer.kp
    dev = torch.device("cuda", local_rank)
    xt = torch.from_numpy(x).to(torch.bfloat16).to(dev)
    # shard-major output [world][M][width]: this rank's K4 writes its slot, the
    # all-gather fills the others in place (no reassembly copy)
    gbuf = torch.empty((world, m, width), dtype=torch.float16, device=dev)
    slot = gbuf[rank, :, : b1 - b0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lb = LayerBench(fq, layer, xt, out=slot, flush=flush)

    def gather():
        if world > 1:
            dist.all_gather_into_tensor(gbuf.view(world * m, width), gbuf[rank])

    for _ in range(args.warmup):
        gather()
    lb.capture(args.warmup)
    barrier()
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        barrier()
        t_k1k4, t_k1, t_k4, t_ag, t_launch = lb.time(args.steps,
                                                     after_step=gather if world > 1 else None)
        torch.cuda.synchronize()
        barrier()
    # per-kernel durations for the rooflines: chains of launches on distinct inputs
    t_k1c, t_k4c = lb.time_chain(make_layer=lambda: fq.Layer(
        cfg, device=local_rank, a_format=a_fmt, b_format=b_fmt, n_begin=b0, n=b1 - b0))
    t_step = t_k1k4 + (t_ag if world > 1 else 0.0)
    if world > 1:
        tt = torch.tensor([t_step, t_k1, t_k4, t_ag, t_k1k4], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_k1, t_k4, t_ag, t_k1k4 = tt.tolist()
    sat_per_step = int(lb.sat.item()) // max(1, lb.k1_runs)

    # ---- e2e: the reference-facing drop-in call with HOST f64 buffers ----
    # Plain (pageable) numpy buffers, as fq::gpu::run_layer passes its
    # std::vector-backed fq::Matrix; the pinned-buffer rate is reported beside it.
    xh_pageable = np.ascontiguousarray(bf16_round(x))
    yh_pageable = np.empty((m, b1 - b0))
    xh_pinned = torch.from_numpy(xh_pageable).pin_memory().numpy()
    yh_pinned = torch.empty((m, b1 - b0), dtype=torch.float64).pin_memory().numpy()

    def run_host(xh, yh, reps):
        sat = ctypes.c_int64()
        ts = []
        for _ in range(reps):
            barrier()
            t0 = time.perf_counter()
            fq.check(fq.lib().fqg_layer_run_host(layer._h, xh.ctypes.data, m, yh.ctypes.data,
                                                 ctypes.byref(sat)))
            ts.append(time.perf_counter() - t0)
        return float(np.mean(ts))

    run_host(xh_pageable, yh_pageable, 2)  # warm: the pool grows, streams exist
    run_host(xh_pinned, yh_pinned, 2)
    t_e2e = run_host(xh_pageable, yh_pageable, args.e2e_steps)
    t_e2e_pinned = run_host(xh_pinned, yh_pinned, args.e2e_steps)
    if world > 1:
        tt = torch.tensor([t_e2e, t_e2e_pinned], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e, t_e2e_pinned = tt.tolist()

    ops = 2.0 * m * n * kp  # whole layer (all ranks), reference bitops K' (pipeline.cpp:211)
    tops = ops / (t_step * 1e-3) / 1e12
    hbm_gbs, bf16_tf, peak_src, int8_peak, i8_src = peaks()
    gemm_ops_rank = 2.0 * m * (b1 - b0) * kp
    gemm_tops = gemm_ops_rank / (t_k4c * 1e-3) / 1e12
    ldq = kp // 2 if a_fmt == fq.I4 else kp
    k1_bytes = m * k * 2 + m * ldq + kp * 4 + k * 12
    k1_gbs = k1_bytes / (t_k1c * 1e-3) / 1e9
    traffic = None
    try:  # per-launch DRAM bytes of K4 from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(args.config, {})
            traffic = tr.get("gemm_dram_bytes")
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": tops, "unit": "TOPS",
        "tokens_per_s": m / (t_step * 1e-3),
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "timing": "device time between event-record nodes captured inside the step's CUDA graph "
                  "(K1 -> K4 [-> all-gather]); ms_per_step_with_launch adds the graph launch",
        "ms_per_step_with_launch": t_launch + (t_ag if world > 1 else 0.0),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int8 MMA / int32 accumulate (4-bit values)" if bits == 4 else
                 "int8 MMA / int32 accumulate",
        "data": "synthetic (fq::make_synthetic_layer generator, seed 42, 1% outlier channels x "
                "U[20,100]); activations rounded to bf16",
        "config": {"workload": args.config, "K": k, "N": n, "M": m, "bits": bits, "Kp": kp,
                   "flatten_ratio_x": cfg.plan_x.flatten_ratio(),
                   "a_format": "i4 packed" if a_fmt == fq.I4 else "i8",
                   "b_format": "i4 packed" if b_fmt == fq.I4 else "i8",
                   "out_dtype": "fp16",
                   "parallelism": f"N-shard x{world} + NCCL all-gather" if world > 1 else "1 GPU",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "breakdown_ms": {"flatten_quant_K1": t_k1, "gemm_K4": t_k4,
                         "all_gather": t_ag if world > 1 else 0.0, "K1_K4_graph": t_k1k4},
        "steady_state": {"ms_per_step": lb.t_step_chain,
                         "value": gemm_ops_rank / (lb.t_step_chain * 1e-3) / 1e12,
                         "unit": "TOPS per GPU (no collective)",
                         "how": "informational: 8 whole layer steps (K1 -> K4) back to back in one "
                                "graph, each on its own activations and device copy of the layer "
                                "(> L2), as the layers of a model run; `value` above stays the "
                                "single flushed step"},
        "kernel_ms": {"flatten_quant_K1": t_k1c, "gemm_K4": t_k4c,
                      "how": "average launch duration over a graph of 8 back-to-back launches on "
                             "8 distinct activations and 8 device copies of the layer (> L2), event "
                             "nodes at both ends (the rooflines use these; breakdown_ms are single "
                             "launches after an L2 flush, each carrying its own node and launch "
                             "overhead)"},
        "saturation_events_per_step": sat_per_step,  # counted by K1 in every timed step
        "roofline": {"bound": "tensor", "achieved": gemm_tops, "peak": int8_peak,
                     "unit": "TFLOP/s", "frac": gemm_tops / int8_peak, "traffic": traffic,
                     "kernel": gemm_label(fq, m, b1 - b0, kp, a_fmt, b_fmt),
                     "peak_basis": f"tcgen05 kind::i8 MMA peak, {i8_src}; frac vs spec 4.5 "
                                   f"POPS: {gemm_tops / SPEC_INT8_TOPS:.3f}; vs 2 x bf16 "
                                   f"measured ({peak_src}): {gemm_tops / (2 * bf16_tf):.3f}",
                     "effective_tops_on_K": 2.0 * m * (b1 - b0) * k / (t_k4c * 1e-3) / 1e12,
                     "frac_single_launch": gemm_ops_rank / (t_k4 * 1e-3) / 1e12 / int8_peak},
        "roofline_k1": {"bound": "hbm", "achieved": k1_gbs, "peak": hbm_gbs, "unit": "GB/s",
                        "frac": k1_gbs / hbm_gbs, "bytes_per_launch": k1_bytes,
                        "frac_single_launch": k1_bytes / (t_k1 * 1e-3) / 1e9 / hbm_gbs},
        "e2e": {"value": ops / t_e2e / 1e12, "unit": "TOPS",
                "tokens_per_s": m / t_e2e,
                "h2d_bytes_per_step": m * k * 8, "d2h_bytes_per_step": m * (b1 - b0) * 8 + 8,
                "api": "fqg_layer_run_host (drop-in fq::run_layer), f64 host buffers, pageable "
                       "(numpy), H2D + kernels + D2H in the timed call",
                "pinned_host_buffers": {"value": ops / t_e2e_pinned / 1e12, "unit": "TOPS",
                                        "tokens_per_s": m / t_e2e_pinned}},
        # per timed step: K1 + K4 (one graph); the per-kernel loop replays them
        # again from graphs of their own; split-K (small M) reduces inside K4
        "gpu_launches": 2 * args.steps,
        "launch": "one CUDA graph per step (K1, then K4 as a programmatic dependent launch); "
                  "K1 and K4 also timed apart from their own graphs for the rooflines",
        "clocks": clk.summary(),
    }
    if world > 1:
        line["collective"] = {"op": "ncclAllGather (torch.distributed all_gather_into_tensor, "
                                    "in place into the shard-major buffer)",
                              "bytes_received_per_rank": (world - 1) * m * width * 2,
                              "ms": t_ag}
    if rank == 0 and world == 1:
        del lb
        torch.cuda.empty_cache()
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(fq, cfg, layer, bf16_round(x), bits, k, n, m)
        if not args.no_subresults and args.config == "w4a4_4096":
            line["subresults"] = subresults(fq, args, int8_peak, flush)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
