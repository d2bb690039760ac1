"""N>1 host logic on CPU: world_size-2 `gloo` process group running the
column-shard + all-gather path of paper_2402_17985_b200.shard with per-rank
outputs computed by the oracle on the rank's slice of weight_q (global s_w)."""
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
