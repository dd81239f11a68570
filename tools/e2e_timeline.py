"""GPU timeline (CUPTI) of host-path matvec calls: pinned tensor in/out vs numpy in/out, cfg2."""
import os, sys, time
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty, precompute_spectral  # noqa

op = precompute_spectral(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
n = op.dim
u_host = pin(dense_rhs(n, seed=1)[:, None])
out = pinned_empty(u_host.shape, u_host.dtype)
u_np = dense_rhs(n, seed=1)
for name, call in (("pinned", lambda: matvec(op, u_host, out=out)), ("numpy", lambda: matvec(op, u_np))):
    for _ in range(20):
        call()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter(); call(); ts.append((time.perf_counter() - t0) * 1e6)
    print(f"{name}: per-call us min {min(ts):.0f} median {np.median(ts):.0f} max {max(ts):.0f}")
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(6):
            call()
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    prev = None
    for e in ev[:24]:
        gap = 0 if prev is None else e.time_range.start - prev
        print(f"  {e.time_range.start - t0:9.1f} +{e.time_range.elapsed_us():7.1f}  gap {gap:7.1f}  {e.name[:50]}")
        prev = e.time_range.end
