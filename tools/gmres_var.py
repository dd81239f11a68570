"""Repeat cfg2 GMRES solves in one process and report device matvec time per solve (variance probe)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized  # noqa
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec  # noqa

sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(30, 30, 128, 0)))
op = BorderedOperator.from_system(sys_)
b = torch.from_numpy(unit_feed_rhs(30, 30, 128)[:, None]).cuda()
u = torch.from_numpy(dense_rhs(sys_.dim, seed=1)[:, None]).cuda()
pk = build_pk(sys_)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    for tag, p in (("none", None), ("pk", pk)):
        t0 = time.perf_counter()
        x, r = solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=50))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        print(rep, tag, f"{dt:.2f} ms  matvec {r.phase_timings['matvec_total'] * 1e3:.2f}  orth {r.phase_timings['orthogonalization'] * 1e3:.2f}", flush=True)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        matvec(op.spectral, u)
    e1.record()
    torch.cuda.synchronize()
    print(rep, "matvec", f"{e0.elapsed_time(e1) / 50 * 1e3:.1f} us", flush=True)
