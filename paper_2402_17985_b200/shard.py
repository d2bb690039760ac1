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
    """All-gather [M, n_r] column shards into the full [M, n] output.

    all_gather_into_tensor needs equal contributions, so each rank pads its
    shard to the common width; the result is reassembled column-block by
    column-block (the collective returns [world, M, width])."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    width = shard_width(n, world, align)
    m = y_local.shape[0]
    b0, b1 = shard_bounds(n, world, rank, align)
    if y_local.shape[1] != b1 - b0:
        raise ValueError("gather_columns: local shard width mismatch")
    send = y_local
    if y_local.shape[1] != width:
        send = torch.zeros((m, width), dtype=y_local.dtype, device=y_local.device)
        send[:, : b1 - b0] = y_local
    flat = torch.empty((world * m, width), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(flat, send.contiguous(), group=group)
    out = flat.view(world, m, width)
    parts = []
    for r in range(world):
        c0, c1 = shard_bounds(n, world, r, align)
        if c1 > c0:
            parts.append(out[r, :, : c1 - c0])
    return torch.cat(parts, dim=1)


class ShardedLayer:
    """One rank's column shard of a layer (device weights of columns [b0, b1))."""

    def __init__(self, cfg, rank: int, world: int, device: Optional[int] = None, **layer_kw):
        from . import Layer

        self.n = cfg.n
        self.rank, self.world = rank, world
        self.b0, self.b1 = shard_bounds(self.n, world, rank)
        if self.b1 <= self.b0:
            raise ValueError("ShardedLayer: this rank holds no columns")
        self.layer = Layer(cfg, device=rank if device is None else device, n_begin=self.b0,
                           n=self.b1 - self.b0, **layer_kw)

    def forward(self, x, gather: bool = True, **kw):
        y = self.layer.forward(x, **kw)
        return gather_columns(y, self.n) if gather else y


def emulate_shard_outputs(acc_full: np.ndarray, s_x: float, s_w: float, world: int):
    """Host model of the per-rank epilogues (y = double(acc) * (s_x * s_w)) on
    column slices: used by the multi-rank tests to check exactness."""
    outs = []
    for r in range(world):
        b0, b1 = shard_bounds(acc_full.shape[1], world, r)
        outs.append(acc_full[:, b0:b1].astype(np.float64) * (s_x * s_w))
    return outs
