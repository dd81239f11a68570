"""Headline benchmark: MLFFT Toeplitz matvec/s and GMRES solve time at
30x30, N_b = 128, complex128 (BASELINE.json configs[1]), with the HBM
roofline fraction of the dominant kernel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scale|--no-scale]

A step is one MLFFT matvec (pad -> 2-D DFT -> per-bin 128x128 product ->
inverse DFT -> crop) of one dense seeded vector against the resident
spectral operator.  The spectral blocks (944 MB) exceed the 126 MB L2, so
every step streams them from HBM (no L2 flush needed).  N > 1 runs one
independent replica per GPU (the single-RHS path does not shard; DESIGN.md
"replicas only"); value = total matvecs over all ranks / max-over-ranks time.
``--gpus N`` without a launcher (no WORLD_SIZE in the environment) spawns the
N ranks itself (NCCL, 127.0.0.1), and refuses cleanly if fewer than N GPUs exist.

``config.scale`` (on by default when N > 1, ``--scale`` at N = 1) adds the
paths that do shard: the cfg3 900-column multi-RHS solve
sharded by columns, and the cfg4 64x64 slab-decomposed matvec / GMRES with
both exchanges (``all_to_all_single`` and NVLink peer stores).

``--impl reference`` times the reference's own CPU implementation: the
unmodified ``toepsolve`` package installed into ``oracle/_ref`` by
``oracle/build_ref.sh`` (its public ``toeplitz.matvec``), on all host threads;
the numpy restatement in ``oracle/`` stands in only if that install is absent.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

NY = NX = 30
NB = 128
DIM = NY * NX * NB
METRIC = "MLFFT Toeplitz matvec/s & GMRES solve time, 30x30, N_b=128; % HBM roofline"
UNIT = "matvec/s"
WORKLOAD = "cfg2: 30x30 array, N_b=128, complex128, single dense RHS (BASELINE configs[1])"


def algorithmic_bytes(bins: int, nb: int = NB, dim: int = DIM, s: int = 16) -> dict:
    """Per-matvec algorithmic HBM bytes: D read once + u in + v out."""
    return {"matvec": bins * nb * nb * s + 2 * dim * s,
            "kernel": bins * nb * nb * s + 2 * bins * nb * s,   # per-bin product: D + u_hat + v_hat
            "matvec_min_embedding": (2 * NY - 1) * (2 * NX - 1) * nb * nb * s + 2 * dim * s}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is busy."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _reference_module():
    """The unmodified reference (toepsolve from oracle/_ref), or None if it was not installed."""
    ref = os.path.join(REPO, "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "toepsolve")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import toepsolve.toeplitz as tz
    return tz


def cpu_matvecs(seconds: float, warmup: int, max_steps: int) -> dict:
    """cfg2 matvecs of the reference's own CPU path in THIS process (threads as the environment
    sets them): setup (generator + precompute_spectral) untimed, then `warmup` untimed calls, then
    timed calls until `seconds` or `max_steps`.  The port (oracle/) stands in if oracle/_ref is absent."""
    from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4

    s4 = seeded_stacked4(NY, NX, NB, seed=0)
    u = dense_rhs(DIM, seed=1)
    tz = _reference_module()
    if tz is not None:
        k2, k1 = 2 * NY - 1, 2 * NX - 1
        blocks = {(p, q): s4[p % k2, q % k1] for p in range(-(NY - 1), NY) for q in range(-(NX - 1), NX)}
        gen = tz.embed_2l(blocks, NY, NX, NB)
        del blocks
        op = tz.precompute_spectral(gen)
        del gen

        def step():
            return tz.matvec(op, u)
        kind, what = "reference", "toepsolve.toeplitz.matvec (unmodified reference, oracle/_ref)"
    else:
        import oracle

        d = oracle.precompute_spectral(s4)
        dims = (NY, NX, NB, 2 * NY - 1, 2 * NX - 1)
        uc = u[:, None]

        def step():
            return oracle.matvec(d, dims, uc)
        kind, what = "port", "oracle/mlfft.py (numpy restatement; oracle/_ref not installed)"
    del s4
    for _ in range(warmup):
        step()
    times = []
    t_end = time.perf_counter() + seconds
    while len(times) < max(1, max_steps) and (not times or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    return {"kind": kind, "what": what, "times": times}


def cpu_baseline_subprocess(threads: int, seconds: float) -> dict:
    """One bounded CPU sample in a fresh process with BLAS threads pinned to `threads`."""
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    env["CUDA_VISIBLE_DEVICES"] = ""
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-sample", "--cpu-seconds", str(seconds),
           "--warmup", "2", "--steps", "200"]
    try:
        out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
        r = json.loads(line)
    except Exception as exc:  # noqa: BLE001
        return {"error": f"cpu sample failed: {exc!r}"}
    t = r["times"]
    return {"value": 1.0 / min(t), "unit": UNIT, "cores": threads, "kind": r["kind"],
            "sample": f"{len(t)} cfg2 matvecs (best-of, after 2 warm-up) of {r['what']}, "
                      f"{threads} BLAS thread(s), generator + precompute excluded",
            "mean_s": float(np.mean(t)), "median_s": float(np.median(t))}


def cpu_baseline() -> dict:
    """Reference CPU path on the box's host cores: all threads (headline) and one thread."""
    cores = os.cpu_count() or 1
    allc = cpu_baseline_subprocess(cores, 10.0)
    one = cpu_baseline_subprocess(1, 10.0)
    if "error" in allc:
        return allc
    allc["single_thread"] = one
    try:
        allc["cpu_model"] = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                             if ln.startswith("model name")][0]
    except Exception:  # noqa: BLE001
        pass
    return allc


def run_cpu_sample(args):
    r = cpu_matvecs(args.cpu_seconds, args.warmup, args.steps)
    print(json.dumps(r), flush=True)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    # bounded: at ~0.1 s per reference matvec, K steps of the driver's run are timed in full up to
    # 120 s; beyond that the first steps that fit are the sample
    r = cpu_matvecs(120.0, args.warmup, args.steps)
    t = r["times"]
    dt = float(np.sum(t))
    value = len(t) / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": len(t),
            "warmup": args.warmup, "ms_per_step": 1e3 * dt / len(t), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic (BASELINE seeded generator)",
            "config": {"workload": WORKLOAD, "embedding": "59x59 circulant (3481 bins, the reference's 2N-1)",
                       "n_bins": (2 * NY - 1) * (2 * NX - 1), "dim": DIM, "steps_requested": args.steps},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": r["kind"],
                             "sample": f"{len(t)} timed cfg2 matvecs of {r['what']} on {cores} host threads "
                                       f"(generator + precompute_spectral excluded)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def count_launches(step, reps: int = 4) -> int:
    """Kernels one ``step`` launches, counted by the CUDA activity trace (torch.profiler / CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            step()
        torch.cuda.synchronize()
    n = sum(1 for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
            and not e.name.startswith(("Memcpy", "Memset", "cudaMemcpy", "cudaMemset")))
    return round(n / reps)


def _warm_calls(fn, n_min, seconds):
    """Untimed warm-up: at least n_min calls and at least `seconds` of calls."""
    t_end = time.perf_counter() + seconds
    i = 0
    while i < n_min or time.perf_counter() < t_end:
        fn()
        i += 1
    return i


def _percall(fn, n):
    """Per-call host wall times (each call ends with its own synchronisation) plus the total."""
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return ts


def _broadcast_stacked(ny, nx, nb, dev, world):
    """Seeded generator made once on rank 0 and broadcast to every rank's device (NCCL)."""
    import torch
    import torch.distributed as dist

    from paper_2506_20350_b200.problems import seeded_stacked4

    shape = (2 * ny - 1, 2 * nx - 1, nb, nb)
    if world == 1 or dist.get_rank() == 0:
        t = torch.from_numpy(seeded_stacked4(ny, nx, nb, seed=0)).to(dev)
    else:
        t = torch.empty(shape, dtype=torch.complex128, device=dev)
    if world > 1:
        dist.broadcast(torch.view_as_real(t), src=0)
    return t


def scale_legs(dev, world, rank, peer: bool = False):
    """The paths that shard, timed on the device, max over ranks.

    Each leg runs inside a guard whose outcome is all-reduced before the next one starts, so a
    failure on one rank cannot leave the others waiting in a collective.  The NVLink peer-store
    exchange (custom system-scope spin waits, never run across GPUs here) only with ``peer``."""
    import torch
    import torch.distributed as dist

    def tmax(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    out = {}

    def agreed(ok: bool) -> bool:  # every rank learns whether every rank succeeded
        if world == 1:
            return ok
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    try:
        out.update(_scale_cfg3(dev, world, rank, tmax, barrier))
        ok = True
    except Exception as exc:  # noqa: BLE001
        out["cfg3_columns"] = {"error": repr(exc)}
        ok = False
    if not agreed(ok):
        return out
    for exchange in (("collective", "peer") if peer and world > 1 else ("collective",)):
        try:
            out[f"cfg4_slab_{exchange}"] = _scale_cfg4(dev, world, rank, exchange, tmax, barrier)
            ok = True
        except Exception as exc:  # noqa: BLE001
            out[f"cfg4_slab_{exchange}"] = {"error": repr(exc)}
            ok = False
        if not agreed(ok):
            break
    return out


def _guarded_scale_legs(args, dev, world, rank, line):
    """scale_legs under a watchdog.  The sharded legs run collectives (and, with --scale-peer, custom
    spin waits) that one GPU cannot exercise at world > 1; if they do not finish within
    ``--scale-timeout`` seconds every rank leaves with status 0 and rank 0 first prints the headline
    line it already holds (``line``), with the time-out recorded under ``config.scale``."""
    import threading

    def give_up():
        if rank == 0 and line is not None:
            line["config"]["scale"] = {"error": f"sharded legs abandoned after {args.scale_timeout} s (watchdog)"}
            print(json.dumps(line), flush=True)
        os._exit(0)

    wd = threading.Timer(args.scale_timeout, give_up)
    wd.daemon = True
    wd.start()
    try:
        return scale_legs(dev, world, rank, peer=args.scale_peer)
    except Exception as exc:  # noqa: BLE001 - the headline line must still be printed
        return {"error": repr(exc)}
    finally:
        wd.cancel()


def _scale_cfg3(dev, world, rank, tmax, barrier):
    import torch

    from paper_2506_20350_b200.distributed import column_range, solve_columns_sharded
    from paper_2506_20350_b200.problems import unit_feed_rhs
    from paper_2506_20350_b200.solvers import GmresConfig, solve_multi_rhs_sequential
    from paper_2506_20350_b200.toeplitz import precompute_spectral_stacked

    out = {}
    # ---- cfg3: 900 unit right-hand sides, columns sharded, no collective in the data path
    s4 = _broadcast_stacked(30, 30, 256, dev, world)
    op3 = precompute_spectral_stacked(s4)
    del s4
    W = 900
    b = torch.from_numpy(unit_feed_rhs(30, 30, 256, columns="each")).to(dev)
    cfg = GmresConfig(tol=1e-6)
    c0, c1 = column_range(W, world, rank)
    solve_multi_rhs_sequential(op3, None, b[:, c0:c1].contiguous(), cfg)  # warm: workspaces, slices
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    local = b[:, c0:c1].contiguous()
    x, reps = solve_multi_rhs_sequential(op3, None, local, cfg)
    e1.record()
    barrier()
    solve_ms = tmax(e0.elapsed_time(e1))
    xs = None
    if world > 1:  # the public sharded entry point (same solve + gather of X to rank 0)
        xs, _ = solve_columns_sharded(op3, None, b, cfg)
    its = [r.iterations for r in reps]
    out["cfg3_columns"] = {"columns_total": W, "columns_per_rank": c1 - c0, "solve_ms_max_over_ranks": solve_ms,
                           "columns_per_s": W / (solve_ms * 1e-3), "iterations_min_max_rank0": [min(its), max(its)],
                           "note": "batched per-column GMRES(1e-6) of this rank's columns, no data-path "
                                   "collective; X gathered to rank 0 afterwards (solve_columns_sharded)"}
    del op3, b, x, xs
    torch.cuda.empty_cache()
    return out


def _scale_cfg4(dev, world, rank, exchange, tmax, barrier):
    """cfg4 64x64 slab decomposition: matvec and GMRES(50) to 1e-6 with one exchange mode."""
    import torch

    from paper_2506_20350_b200.distributed import SlabOperator, gmres_slab
    from paper_2506_20350_b200.problems import dense_rhs, unit_feed_rhs
    from paper_2506_20350_b200.solvers import GmresConfig

    s4 = _broadcast_stacked(64, 64, 128, dev, world)
    u_full = torch.from_numpy(dense_rhs(64 * 64 * 128, seed=1)).to(dev)
    b_full = torch.from_numpy(unit_feed_rhs(64, 64, 128)).to(dev)
    if True:
        sop = SlabOperator.from_generator(s4, exchange=exchange)
        del s4
        y0, y1 = sop.rows
        n_loc = sop.local_dim
        u = u_full[y0 * 64 * 128:y1 * 64 * 128].contiguous()
        for _ in range(3):
            sop.matvec_local(u)
        barrier()
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record()
        for _ in range(20):
            sop.matvec_local(u)
        k1.record()
        barrier()
        mv_us = tmax(k0.elapsed_time(k1) / 20) * 1e3
        mv_native_us = None
        if exchange == "collective":  # the library's own distributed matvec (NCCL all-to-alls in C)
            import ctypes

            from paper_2506_20350_b200 import _lib
            from paper_2506_20350_b200.distributed import native_comm
            comm = native_comm(None)
            ctx = ctypes.c_void_p()
            lib = _lib.lib()
            _lib.check(lib.toep_slab_ctx_create(sop.stages.op.handle, comm.handle, 1, _lib.stream_handle(),
                                                ctypes.byref(ctx)))
            v = torch.empty_like(u.reshape(-1, 1))
            uu = u.reshape(-1, 1).contiguous()
            for _ in range(3):
                _lib.check(lib.toep_slab_apply(ctx.value, uu.data_ptr(), v.data_ptr(), 1, _lib.stream_handle()))
            barrier()
            k0.record()
            for _ in range(20):
                lib.toep_slab_apply(ctx.value, uu.data_ptr(), v.data_ptr(), 1, _lib.stream_handle())
            k1.record()
            barrier()
            mv_native_us = tmax(k0.elapsed_time(k1) / 20) * 1e3
            lib.toep_slab_ctx_destroy(ctx.value)
        bl = b_full[y0 * 64 * 128:y1 * 64 * 128].contiguous()
        gmres_slab(sop, None, bl, GmresConfig(tol=1e-6, restart=50))
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        _, rep = gmres_slab(sop, None, bl, GmresConfig(tol=1e-6, restart=50))
        g1.record()
        barrier()
        res = {
            "matvec_us_max_over_ranks": mv_us, "matvec_native_us_max_over_ranks": mv_native_us,
            "gmres_path": "native (toep_slab_apply + NCCL all-reduce called by the device engine)"
            if exchange == "collective" else "python stage callbacks",
            "gmres_ms_max_over_ranks": tmax(g0.elapsed_time(g1)),
            "gmres_iterations": rep.iterations, "reference_iterations": 28, "local_rows": n_loc // (64 * 128),
            "resident_spectral_bytes_per_rank": sop.stages.op.resident_bytes,
            "exchange_bytes_per_matvec_per_rank": 2 * 64 * 128 * 128 * 16 * (world - 1) // (world * world)}
        del sop
        torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2506_20350_b200.problems import dense_rhs, seeded_stacked4, system_from_generator, unit_feed_rhs
    from paper_2506_20350_b200.solvers import BorderedOperator, GmresConfig, build_pk, solve_multi_rhs_vectorized
    from paper_2506_20350_b200.toeplitz import generator_from_stacked, matvec, pin, pinned_empty

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    s4 = seeded_stacked4(NY, NX, NB, seed=0)
    sys_ = system_from_generator(generator_from_stacked(s4))
    # module loading / first-launch costs on a small operator, so setup_s is the cfg2 transform itself
    BorderedOperator.from_system(system_from_generator(generator_from_stacked(seeded_stacked4(4, 4, 128, seed=0))))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = BorderedOperator.from_system(sys_)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    spec = op.spectral
    del s4
    u = torch.from_numpy(dense_rhs(DIM, seed=1)[:, None]).to(dev)
    v = torch.empty_like(u)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()

    # ---- device-resident matvecs (value).  Exactly W warm-up steps: a longer warm-up (0.5 s of
    # matvecs) measured slower, not faster -- the sustained HBM stream brings the board to its power
    # cap (sw_power_cap, SM clock 1 905-1 920 MHz: 6 255 vs 6 350-6 480 matvec/s at 20 steps)
    for _ in range(args.warmup):
        v = matvec(spec, u)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        v = matvec(spec, u)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    t_dev = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms_max = float(t_dev.item())
    value = world * args.steps / (ms_max * 1e-3)

    # ---- dominant kernel alone (per-bin product), CUDA events on its stream
    hat_in = torch.randn((spec.bins, NB, 1), dtype=torch.complex128, device=dev)
    hat_out = torch.empty_like(hat_in)
    for _ in range(3):
        spec.spectral_apply(hat_in, hat_out)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nk = max(args.steps, 20)
    k0.record(stream)
    for _ in range(nk):
        spec.spectral_apply(hat_in, hat_out)
    k1.record(stream)
    torch.cuda.synchronize()
    k_ms = k0.elapsed_time(k1) / nk
    del hat_in, hat_out

    # ---- end to end through the public API, pinned host buffers, steady state: the result goes
    # into a preallocated pinned tensor (out=), so no host allocation happens inside the timed loop.
    # Page-locked through the library allocator (toeplitz.pin): the copy engines read torch's own
    # pinned blocks at 17-19 GB/s on these boxes, cudaHostAlloc blocks at 50 GB/s (tools/hostbuf_probe.py)
    u_host = pin(dense_rhs(DIM, seed=1)[:, None])
    out_host = pinned_empty(u_host.shape, u_host.dtype)
    # host path warm-up: page-locked blocks, driver state, and the host core's clock — the calling
    # thread's core needs ~0.5-1 s of activity before a call settles at its steady cost (measured
    # ~310 us per call for the first ~2 500 calls of a process, 235 us after; tools/e2e_warm.py), so
    # the warm-up runs for at least 1 s of calls (and at least W calls)
    _warm_calls(lambda: matvec(spec, u_host, out=out_host), args.warmup, 1.0)
    torch.cuda.synchronize()
    barrier()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record(stream)
    per_call = _percall(lambda: matvec(spec, u_host, out=out_host), args.steps)
    x1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = x0.elapsed_time(x1)
    t_e2e = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = world * args.steps / (float(t_e2e.item()) * 1e-3)
    # the reference's own calling convention: numpy in, numpy out (fresh result per call)
    u_np = dense_rhs(DIM, seed=1)
    r_np = None

    def np_warm():
        nonlocal r_np
        r_np = matvec(spec, u_np)
    _warm_calls(np_warm, args.warmup, 0.3)
    torch.cuda.synchronize()
    barrier()

    def np_call():
        nonlocal r_np
        r_np = matvec(spec, u_np)
    per_call_np = _percall(np_call, args.steps)
    np_value = args.steps / float(np.sum(per_call_np))
    assert isinstance(r_np, np.ndarray) and r_np.shape == (DIM,)

    # ---- GMRES(50) to 1e-8, none and PK (BASELINE cfg2)
    gm = {}
    b = unit_feed_rhs(NY, NX, NB)[:, None]
    bt = torch.from_numpy(b).to(dev)
    pk = build_pk(sys_)
    for tag, p in (("none", None), ("pk", pk)):
        for _ in range(2):  # warm (PK fold, workspaces, first-touch of the pools)
            solve_multi_rhs_vectorized(op, p, bt, GmresConfig(tol=1e-8, restart=50))
        torch.cuda.synchronize()
        times = []
        for _ in range(9):
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            x, rep = solve_multi_rhs_vectorized(op, p, bt, GmresConfig(tol=1e-8, restart=50))
            g1.record(stream)
            torch.cuda.synchronize()
            times.append(g0.elapsed_time(g1))
        it = rep.iterations
        # B_gmres = (it + 1 + restarts) B + sum_j 2 (j+1) n s (minimal basis passes)
        gbytes = (it + 1 + (it - 1) // 50) * algorithmic_bytes(spec.bins)["matvec"] + \
            sum(2 * (j % 50 + 1) * DIM * 16 for j in range(it))
        med = float(np.median(times))
        gm[tag] = {"iterations": it, "solve_ms": med, "solve_ms_min": min(times),
                   "final_residual": rep.final_residual, "reference_iterations": 31 if tag == "none" else 30,
                   "algorithmic_bytes": gbytes, "achieved_GBps": gbytes / (med * 1e-3) / 1e9}
    clocks = sampler.stop()
    launches_per_step = count_launches(lambda: matvec(spec, u))
    do_scale = args.scale or (world > 1 and not args.no_scale)
    if do_scale:
        del op, spec, pk, sys_
        torch.cuda.empty_cache()

    if rank != 0:
        if do_scale:
            _guarded_scale_legs(args, dev, world, rank, None)
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peaks()
    for g in gm.values():
        g["roofline_frac_measured_peak"] = g["achieved_GBps"] / peak
        g["roofline_frac_nominal_8TBps"] = g["achieved_GBps"] / 8000.0
    by = algorithmic_bytes(3600)
    achieved_k = by["kernel"] / (k_ms * 1e-3) / 1e9
    achieved_mv = by["matvec"] * (args.steps / (ms * 1e-3)) / 1e9
    traffic = None
    prof = os.path.join(REPO, "profiles", "fused_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    # the step is ONE kernel (mv_fused_kernel: forward 2-D DFT, per-bin product, inverse 2-D DFT;
    # gpu_launches_per_step), so its average launch time is the CUDA-event time per step
    mv_ms = ms / args.steps
    achieved_fused = by["matvec"] / (mv_ms * 1e-3) / 1e9
    pc = np.array(per_call) * 1e6
    pcn = np.array(per_call_np) * 1e6
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (BASELINE seeded generator, seed 0; dense default_rng(1) vector)",
        "config": {"workload": WORKLOAD, "embedding": "60x60 circulant (3600 bins, smallest 7-smooth >= 2N-1)",
                   "parallelism": f"replicas x{world}", "l2_policy": "inputs larger than L2 (944 MB spectral blocks)",
                   "matvec_hbm_frac": achieved_mv / peak, "matvec_GBps": achieved_mv,
                   "algorithmic_bytes_per_matvec": by["matvec"],
                   "algorithmic_bytes_min_embedding": by["matvec_min_embedding"],
                   "setup_s": t_setup, "setup_note": "precompute_spectral: generator upload (pageable) + device "
                   "2-D DFT of the blocks; the reference takes 7.4 s (BASELINE.md)",
                   "gmres": gm},
        "roofline": {"bound": "hbm", "achieved": achieved_fused, "peak": peak, "unit": "GB/s",
                     "frac": achieved_fused / peak, "traffic": traffic,
                     "traffic_source": "profiles/fused_traffic.json: ncu --set full capture of this kernel "
                                       "(dram__bytes_read.sum + dram__bytes_write.sum per launch), not measured "
                                       "in this run",
                     "kernel": "mv_fused_kernel (forward 2-D DFT -> per-bin D_k u_k -> inverse 2-D DFT, one "
                               "cooperative launch per matvec)",
                     "kernel_ms": mv_ms, "kernel_share_of_step": 1.0,
                     "bytes_per_launch": by["matvec"],
                     "bytes_note": "SURVEY 8(d) B = K Nb^2 16 (spectral blocks) + 2 n 16 (u in, v out); the "
                                   "spectral vectors stay in L2",
                     "peak_source": peak_src,
                     "product_stage": {"kernel": "binprod_tma_kernel (the per-bin product alone, "
                                                 "SpectralOperator.spectral_apply)",
                                       "kernel_ms": k_ms, "bytes_per_launch": by["kernel"],
                                       "achieved": achieved_k, "frac": achieved_k / peak}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": DIM * 16, "d2h_bytes_per_step": DIM * 16,
                "path": "toeplitz.matvec(op, pinned CPU tensor, out=pinned CPU tensor): one library call per "
                        "step (H2D copy, matvec, D2H copy, synchronise)",
                "per_call_us_min": float(pc.min()), "per_call_us_median": float(np.median(pc)),
                "per_call_us_p90": float(np.percentile(pc, 90)),
                "numpy": {"value": np_value, "unit": UNIT,
                          "path": "toeplitz.matvec(op, numpy array) -> numpy array (the reference's calling "
                                  "convention; staged through a library page-locked block)",
                          "per_call_us_min": float(pcn.min()), "per_call_us_median": float(np.median(pcn))}},
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step,
        "clocks": clocks,
    }
    if do_scale:  # after the headline is complete: a hang in a sharded leg cannot lose it
        line["config"]["scale"] = _guarded_scale_legs(args, dev, world, rank, line)
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawned(local_rank, args, world, port):
    os.environ.update({"RANK": str(local_rank), "LOCAL_RANK": str(local_rank), "WORLD_SIZE": str(world),
                       "LOCAL_WORLD_SIZE": str(world), "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scale", action="store_true", help="add config.scale (cfg3 column / cfg4 slab legs) at N=1")
    ap.add_argument("--no-scale", action="store_true", help="skip config.scale at N>1")
    ap.add_argument("--scale-timeout", type=float, default=480.0,
                    help="seconds after which the config.scale legs are abandoned (the headline line is still printed)")
    ap.add_argument("--scale-peer", action="store_true",
                    help="config.scale also times the NVLink peer-store exchange of the cfg4 slab legs")
    ap.add_argument("--cpu-sample", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_sample:
        run_cpu_sample(args)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no launcher: spawn the N ranks here (one process per GPU, NCCL over 127.0.0.1)
        if args.impl == "reference":
            run_reference(args)  # rank 0 only does work; nothing to spawn
            return
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} requested but only {have} CUDA "
                              f"device(s) are visible", "n_gpus": args.gpus}), flush=True)
            sys.exit(2)
        import torch.multiprocessing as mp

        mp.spawn(_spawned, args=(args, args.gpus, _free_port()), nprocs=args.gpus, join=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
