"""N>1 host logic on CPU: world_size-2 `gloo` process groups running the
column-shard + all-gather path of paper_2402_17985_b200.shard: gather_columns,
and ShardedLayer.forward (shard-major buffer, per-chunk in-place all-gather)
with the device layer replaced by an oracle-backed stand-in that computes the
rank's columns from its slice of weight_q (global s_w). A 2-GPU NCCL variant
runs the real device layers when two GPUs are present."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_17985_b200.shard import gather_columns, shard_bounds, shard_width


def test_shard_bounds_partition():
    for n in (1, 31, 32, 100, 640, 1728, 4096, 13824):
        for world in (1, 2, 3, 4, 8):
            cols = []
            for r in range(world):
                b0, b1 = shard_bounds(n, world, r)
                assert b0 <= b1 and (b1 - b0) <= shard_width(n, world)
                if r < world - 1 and b1 < n:
                    assert (b1 - b0) % 32 == 0
                cols.extend(range(b0, b1))
            assert cols == list(range(n))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import Port

        import paper_2402_17985_b200 as fq

        p = Port()
        k, n, m = 192, 200, 24  # uneven last shard (200 = 128 + 72 at world 2)
        w, calib, x = fq.synthetic_layer(3, test_rows=m, in_channels=k, out_channels=n, rows=16,
                                         samples=3)
        L = p.quantize_layer(w, calib, 8)  # global s_w over all N
        y_ref, _, qx, _ = p.run_layer(L, x, debug=True)
        b0, b1 = shard_bounds(n, world, rank)
        acc = p.int_matmul_raw(qx, np.ascontiguousarray(L.wq[:, b0:b1]))
        y_local = torch.from_numpy(acc.astype(np.float64) * (L.act_scale * L.s_w))
        y = gather_columns(y_local, n)
        ok = bool(torch.equal(y, torch.from_numpy(y_ref)))
        # a per-shard (local absmax) weight scale would NOT be exact:
        wl = np.abs(L.wq[:, b0:b1]).max()
        q.put((rank, ok, int(wl)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1))


def test_two_rank_shard_and_gather_is_exact():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok, _ in res:
        assert ok is True, f"rank {rank}: {ok}"


class _OracleShard:
    """Stand-in for a device Layer of columns [b0, b1): K1 = oracle quantize_acts,
    K4 = exact integer product on the slice, epilogue y = double(acc) * (s_x * s_w)."""

    def __init__(self, port, L, b0, b1):
        self.port, self.L, self.b0, self.b1 = port, L, b0, b1

    def quantize_acts_rowsum(self, x):
        qx, _ = self.port.quantize_acts(self.L, x.numpy())
        return qx, None

    def gemm_rows(self, q, rowsum, r0, rows, out):
        from oracle import Port

        acc = Port.exact_acc(q[r0:r0 + rows], np.ascontiguousarray(self.L.wq[:, self.b0:self.b1]))
        out.copy_(torch.from_numpy(acc.astype(np.float64) * (self.L.act_scale * self.L.s_w)))
        return out


def _worker_sharded(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import Port

        import paper_2402_17985_b200 as fq
        from paper_2402_17985_b200.shard import ShardedLayer

        p = Port()
        k, n, m = 160, 200, 32
        w, calib, x = fq.synthetic_layer(5, test_rows=m, in_channels=k, out_channels=n, rows=16,
                                         samples=3)
        L = p.quantize_layer(w, calib, 4)
        y_ref, _ = p.run_layer(L, x)
        cfg = fq.quantize_layer(w, calib, 4)
        b0, b1 = shard_bounds(n, world, rank)
        oks = []
        for chunks in (1, 2, 4):
            sl = ShardedLayer(cfg, rank, world, layer=_OracleShard(p, L, b0, b1))
            out = sl.forward(torch.from_numpy(x), out_dtype=torch.float64, chunks=chunks)
            oks.append(bool(np.array_equal(out.full().numpy(), y_ref)))
            oks.append(bool(np.array_equal(out.shard(rank).numpy(), y_ref[:, b0:b1])))
        q.put((rank, all(oks), 0))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), -1))


def _spawn(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    return res


def test_two_rank_sharded_layer_host_logic():
    for rank, ok, _ in _spawn(_worker_sharded):
        assert ok is True, f"rank {rank}: {ok}"


def _worker_nccl(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
        import paper_2402_17985_b200 as fq
        from paper_2402_17985_b200.shard import ShardedLayer

        k, n, m = 1024, 3000, 512
        w, calib, x = fq.synthetic_layer(9, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                         samples=4)
        cfg = fq.quantize_layer(w, calib, 4)
        xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
        full = fq.Layer(cfg, device=rank, b_format=fq.I4).forward(xt, out_dtype=torch.float16)
        sl = ShardedLayer(cfg, rank, world, b_format=fq.I4)
        ok = True
        for chunks in (1, 4):
            y = sl.forward(xt, out_dtype=torch.float16, chunks=chunks).full()
            ok = ok and bool(torch.equal(y, full))
        q.put((rank, ok, 0))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), -1))


@pytest.mark.gpu
def test_two_gpu_nccl_sharded_layer():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    for rank, ok, _ in _spawn(_worker_nccl):
        assert ok is True, f"rank {rank}: {ok}"
