"""N-sharding of one flattened linear layer across the GPUs of a node.

Each output column depends on the whole flattened activation row and one
weight column, and the integer accumulation is exact, so the layer shards
along N (output features) with no data-path exchange: every rank runs K1 on
the replicated input and K4 on its column shard. The weight scale s_w must be
the GLOBAL one (per-tensor absmax over all N, pipeline.cpp:139-143), which the
device weight tail guarantees by reducing over the full W before slicing.
Only when the full layer output is needed is it all-gathered (NCCL over
NVLink on the GPU path; any torch.distributed backend for the host logic).
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def shard_bounds(n: int, world: int, rank: int, align: int = 32) -> tuple[int, int]:
    """Columns [b0, b1) of `rank`: contiguous, `align`-multiple widths except
    possibly the last; empty for ranks beyond the layer width."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_bounds: bad rank/world")
    per = -(-n // world)
    per = -(-per // align) * align
    b0 = min(n, rank * per)
    return b0, min(n, b0 + per)


def shard_width(n: int, world: int, align: int = 32) -> int:
    """Width every rank contributes to the all-gather (the widest shard)."""
    b0, b1 = shard_bounds(n, world, 0, align)
    return b1 - b0


def gather_columns(y_local, n: int, group=None, align: int = 32):
    """All-gather [M, n_r] column shards into the full [M, n] output (host-logic
    helper for tests and small tensors: pads and reassembles with copies; the
    device path, ShardedLayer.forward, writes each shard straight into its slot
    of a shard-major buffer and gathers in place instead)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    width = shard_width(n, world, align)
    m = y_local.shape[0]
    b0, b1 = shard_bounds(n, world, rank, align)
    if y_local.shape[1] != b1 - b0:
        raise ValueError("gather_columns: local shard width mismatch")
    buf = torch.empty((world, m, width), dtype=y_local.dtype, device=y_local.device)
    buf[rank, :, : b1 - b0] = y_local
    dist.all_gather_into_tensor(buf.view(world * m, width), buf[rank], group=group)
    return ShardedOutput(buf.unsqueeze(0), n, world, align).full()


class ShardedOutput:
    """The gathered layer output in shard-major layout [chunks][world][Mc][width]
    (slot r holds columns [b0_r, b1_r) of fqg_shard_bounds). No reassembly copy
    is made unless full() is called."""

    def __init__(self, buf, n: int, world: int, align: int = 32):
        self.buf, self.n, self.world, self.align = buf, n, world, align

    def shard(self, r: int):
        """Rank r's columns as an [M, b1 - b0] view (rows of all chunks)."""
        b0, b1 = shard_bounds(self.n, self.world, r, self.align)
        c, w, mc, width = self.buf.shape
        return self.buf[:, r, :, : b1 - b0].reshape(c * mc, b1 - b0)

    def full(self):
        """[M, N] contiguous copy (one permute-copy of the gathered slots). Slots
        are in column order and only the last non-empty one can be narrower, so
        the padding columns all land at the end."""
        c, w, mc, width = self.buf.shape
        return self.buf.permute(0, 2, 1, 3).reshape(c * mc, w * width)[:, : self.n]


class ShardedLayer:
    """One rank's column shard of a layer (device weights of columns [b0, b1)).

    forward() runs K1 on the replicated input, then K4 per M-chunk straight into
    this rank's slot of the shard-major buffer [chunks][world][Mc][width], and
    all-gathers each chunk in place on a communication stream, so the gather of
    chunk c overlaps the GEMM of chunk c + 1 (NCCL over NVLink on the GPU path)."""

    def __init__(self, cfg, rank: int, world: int, device: Optional[int] = None, layer=None,
                 **layer_kw):
        self.n = cfg.n
        self.rank, self.world = rank, world
        self.b0, self.b1 = shard_bounds(self.n, world, rank)
        self.width = shard_width(self.n, world)
        if self.b1 <= self.b0:
            raise ValueError("ShardedLayer: this rank holds no columns")
        if layer is None:  # `layer`: an injected stand-in (CPU tests of the host logic)
            from . import Layer

            layer = Layer(cfg, device=rank if device is None else device, n_begin=self.b0,
                          n=self.b1 - self.b0, **layer_kw)
        self.layer = layer
        self._comm = None

    def forward(self, x, out_dtype=None, gather: bool = True, chunks: int = 1, group=None):
        import torch
        import torch.distributed as dist

        m = x.shape[0]
        if chunks < 1 or m % chunks != 0:
            chunks = 1
        mc = m // chunks
        dt = out_dtype or torch.float16
        buf = torch.empty((chunks, self.world, mc, self.width), dtype=dt, device=x.device)
        L = self.layer
        on_gpu = x.is_cuda
        st = torch.cuda.current_stream(x.device) if on_gpu else None
        q, rowsum = L.quantize_acts_rowsum(x)
        if on_gpu and gather and self.world > 1 and self._comm is None:
            self._comm = torch.cuda.Stream(x.device)
        for c in range(chunks):
            out = buf[c, self.rank, :, : self.b1 - self.b0]
            L.gemm_rows(q, rowsum, c * mc, mc, out)
            if not (gather and self.world > 1):
                continue
            dst, src = buf[c].view(self.world * mc, self.width), buf[c, self.rank]
            if on_gpu:  # gather of chunk c overlaps the GEMM of chunk c + 1
                ev = torch.cuda.Event()
                ev.record(st)
                self._comm.wait_event(ev)
                with torch.cuda.stream(self._comm):
                    dist.all_gather_into_tensor(dst, src, group=group)
            else:
                dist.all_gather_into_tensor(dst, src, group=group)
        if on_gpu and gather and self.world > 1:
            st.wait_stream(self._comm)
            buf.record_stream(self._comm)
        return ShardedOutput(buf, self.n, self.world)


def emulate_shard_outputs(acc_full: np.ndarray, s_x: float, s_w: float, world: int):
    """Host model of the per-rank epilogues (y = double(acc) * (s_x * s_w)) on
    column slices: used by the multi-rank tests to check exactness."""
    outs = []
    for r in range(world):
        b0, b1 = shard_bounds(acc_full.shape[1], world, r)
        outs.append(acc_full[:, b0:b1].astype(np.float64) * (s_x * s_w))
    return outs
