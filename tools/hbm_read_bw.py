"""Read-only HBM bandwidth ceilings for the decode-size weight stream (torch reductions, D2D copy)."""
import torch

n = 8192 * 14848
b = torch.randint(-127, 128, (n,), dtype=torch.int8, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = torch.empty_like(b)


def t(f, reps=10):
    ts = []
    for i in range(reps + 2):
        fl.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts[2:])[len(ts[2:]) // 2]


for name, f, nbytes in [
    ("sum int32 view", lambda: b.view(torch.int32).sum(), n),
    ("amax int64 view", lambda: b.view(torch.int64).amax(), n),
    ("d2d copy (read+write)", lambda: out.copy_(b), 2 * n),
]:
    ms = t(f)
    print(f"{name:24s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:8.0f} GB/s")
