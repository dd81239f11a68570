"""Secondary BASELINE configurations on one B200 (cfg1, cfg3, cfg4 c128/c64, cfg5)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator, unit_feed_rhs  # noqa
from paper_2506_20350_b200.solvers import (BorderedOperator, GmresConfig, build_pk, schur_solve,  # noqa
                                            solve_multi_rhs_sequential, solve_multi_rhs_vectorized)
from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, precompute_spectral  # noqa


def med_time(fn, warm=2, reps=5):
    """median of `reps` CUDA-event-timed calls after `warm` untimed ones (transient slow windows)."""
    for _ in range(warm):
        fn()
    ts, out = [], None
    for _ in range(reps):
        t, out = ev_time(fn)
        ts.append(t)
    return float(np.median(ts)), out


def ev_time(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


res = {}
which = sys.argv[1:] or ["cfg1", "cfg4", "cfg5", "cfg3"]
if "cfg1" in which:
    sys_ = system_from_generator(generator_from_stacked(seeded_stacked4(4, 4, 32, 0)))
    op = BorderedOperator.from_system(sys_)
    u = torch.from_numpy(dense_rhs(sys_.dim, seed=1)[:, None]).cuda()
    for _ in range(10): matvec(op.spectral, u)
    ms, _ = ev_time(lambda: matvec(op.spectral, u), 200)
    b = torch.from_numpy(unit_feed_rhs(4, 4, 32)[:, None]).cuda()
    g = {}
    for tag, p in (("none", None), ("pk", build_pk(sys_))):
        solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=30))
        t, (x, rep) = med_time(lambda: solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-8, restart=30)))
        g[tag] = {"iterations": rep.iterations, "ms": t}
    res["cfg1"] = {"matvec_us": ms * 1e3, "gmres": g}
    print(json.dumps(res["cfg1"]), flush=True)
if "cfg4" in which:
    gen = generator_from_stacked(seeded_stacked4(64, 64, 128, 0))
    sys_ = system_from_generator(gen)
    u = torch.from_numpy(dense_rhs(sys_.dim, seed=1)[:, None]).cuda()
    b = torch.from_numpy(unit_feed_rhs(64, 64, 128)[:, None]).cuda()
    for dt in (torch.complex128, torch.complex64):
        op = BorderedOperator.from_system(sys_, dtype=dt)
        for _ in range(5): matvec(op.spectral, u)
        ms, _ = ev_time(lambda: matvec(op.spectral, u), 50)
        g = {}
        for tag, p in (("none", None), ("pk", build_pk(sys_))):
            solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-6, restart=50))
            t, (x, rep) = med_time(lambda: solve_multi_rhs_vectorized(op, p, b, GmresConfig(tol=1e-6, restart=50)))
            g[tag] = {"iterations": rep.iterations, "ms": t, "final_residual": rep.final_residual}
        es = 16 if dt == torch.complex128 else 8
        byt = op.spectral.bins * 128 * 128 * es + 2 * sys_.dim * 16
        res[f"cfg4_{str(dt)[6:]}"] = {"matvec_us": ms * 1e3, "GBps": byt / (ms * 1e-3) / 1e9, "gmres": g}
        print(json.dumps(res[f"cfg4_{str(dt)[6:]}"]), flush=True)
        del op
if "cfg5" in which:
    gen = generator_from_stacked(seeded_stacked4(16, 16, 64, 0))
    sys_ = system_from_generator(gen)
    y = torch.from_numpy(dense_rhs(gen.dim, 4, seed=1)).cuda()
    schur_solve(sys_, y, "rybicki")
    t, (x, rep) = ev_time(lambda: schur_solve(sys_, y, "rybicki"))
    flops = 0
    s = 1024
    for m in range(1, 16):
        flops += 8 * s**3 * (m + m + (m if m < 15 else 0) * 4) + 8 * s * s * 4 * 2 * m
    res["cfg5"] = {"rybicki_ms": t, "timings": rep.phase_timings, "approx_gemm_tflop": flops / 1e12,
                   "tflops": flops / (t * 1e-3) / 1e12}
    print(json.dumps(res["cfg5"]), flush=True)
if "cfg3" in which:
    gen = generator_from_stacked(seeded_stacked4(30, 30, 256, 0))
    sys_ = system_from_generator(gen)
    op = BorderedOperator.from_system(sys_)
    W = 900
    B = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).cuda()
    matvec(op.spectral, B)
    ms, _ = ev_time(lambda: matvec(op.spectral, B), 3)
    fl = 8 * op.spectral.bins * 256 * 256 * W
    out = {"multirhs_matvec_ms": ms, "tflops_gemm_equiv": fl / (ms * 1e-3) / 1e12}
    for tag, p in (("pk", build_pk(sys_)), ("none", None)):
        solve_multi_rhs_sequential(op, p, B, GmresConfig(tol=1e-6))  # warm: PK fold, workspaces
        t, (x, reps) = ev_time(lambda: solve_multi_rhs_sequential(op, p, B, GmresConfig(tol=1e-6)))
        its = [r.iterations for r in reps]
        out[tag] = {"solve_ms": t, "it_min": min(its), "it_max": max(its), "it_cols_0_1_449_899": [its[i] for i in (0, 1, 449, 899)]}
        print(tag, json.dumps(out[tag]), flush=True)
    res["cfg3"] = out
    print(json.dumps(out), flush=True)
json.dump(res, open(os.path.join("gpurun_out", "configs.json"), "w"), indent=1)
