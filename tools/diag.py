"""Diagnostics on the GPU box: per-phase GMRES timings and matvec timings (cfg2)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="all")
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--nb", type=int, default=128)
ap.add_argument("--mv", type=int, default=20)
args = ap.parse_args()

ny = nx = args.n
nb = args.nb
sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(ny, nx, nb, seed=0)))
op = BorderedOperator.from_system(sys_)
torch.cuda.synchronize()
dim = ny * nx * nb
u = torch.from_numpy(dense_rhs(dim, seed=1)[:, None]).cuda()
if args.mode in ("all", "mv"):
    for _ in range(3):
        matvec(op.spectral, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(args.mv):
        matvec(op.spectral, u)
    e1.record()
    torch.cuda.synchronize()
    print(f"matvec {e0.elapsed_time(e1) / args.mv * 1e3:.1f} us", flush=True)
if args.mode in ("all", "kernel"):
    spec = op.spectral
    hi = torch.randn((spec.bins, nb, 1), dtype=torch.complex128, device="cuda")
    ho = torch.empty_like(hi)
    for _ in range(3):
        spec.spectral_apply(hi, ho)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(args.mv):
        spec.spectral_apply(hi, ho)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / args.mv * 1e-3
    byt = spec.bins * nb * nb * 16 + 2 * spec.bins * nb * 16
    ref = torch.einsum("kmj,kj->km", spec.diag_blocks, hi[:, :, 0])
    err = (torch.linalg.norm(ref - ho[:, :, 0]) / torch.linalg.norm(ref)).item()
    print(f"binprod {t * 1e6:.1f} us  {byt / t / 1e9:.0f} GB/s  rel err vs torch {err:.2e}", flush=True)
if args.mode in ("all", "gmres"):
    b = torch.from_numpy(unit_feed_rhs(ny, nx, nb)[:, None]).cuda()
    pk = build_pk(sys_)
    for tag, p in (("none", None), ("pk", pk), ("none", None), ("pk", pk)):
        t0 = time.perf_counter()
        x, rep = solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(tag, rep.iterations, f"wall {dt * 1e3:.2f} ms", json.dumps({k: round(v * 1e3, 3) for k, v in rep.phase_timings.items()}), flush=True)
