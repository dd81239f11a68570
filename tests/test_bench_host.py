"""Host-side logic of bench.py that needs no GPU: the watchdog around the sharded ``config.scale`` legs."""
import json
import os
import subprocess
import sys
import types

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code: str, timeout: float = 60.0):
    return subprocess.run([sys.executable, "-c", code], cwd=REPO, capture_output=True, text=True, timeout=timeout)


def test_scale_watchdog_prints_the_headline_and_exits_zero():
    # a sharded leg that never returns: rank 0 must still print the line it holds, with the
    # time-out recorded under config.scale, and leave with status 0
    code = (
        "import time, types, bench\n"
        "bench.scale_legs = lambda *a, **k: time.sleep(120)\n"
        "args = types.SimpleNamespace(scale_timeout=0.5, scale_peer=False)\n"
        "line = {'metric': 'm', 'value': 1.0, 'config': {}}\n"
        "bench._guarded_scale_legs(args, None, 2, 0, line)\n"
        "print('not reached')\n"
    )
    r = _run(code)
    assert r.returncode == 0, r.stderr
    out = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(out) == 1
    line = json.loads(out[0])
    assert line["value"] == 1.0 and "abandoned" in line["config"]["scale"]["error"]


def test_scale_watchdog_other_ranks_exit_silently():
    code = (
        "import time, types, bench\n"
        "bench.scale_legs = lambda *a, **k: time.sleep(120)\n"
        "args = types.SimpleNamespace(scale_timeout=0.5, scale_peer=False)\n"
        "bench._guarded_scale_legs(args, None, 2, 1, None)\n"
    )
    r = _run(code)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_scale_legs_result_and_error_pass_through():
    sys.path.insert(0, REPO)
    import bench

    args = types.SimpleNamespace(scale_timeout=30.0, scale_peer=True)
    seen = {}

    def legs(dev, world, rank, peer=False):
        seen.update(dev=dev, world=world, rank=rank, peer=peer)
        return {"cfg3_columns": {"solve_ms_max_over_ranks": 1.0}}

    old = bench.scale_legs
    try:
        bench.scale_legs = legs
        assert bench._guarded_scale_legs(args, "cuda:0", 4, 2, None) == {"cfg3_columns": {"solve_ms_max_over_ranks": 1.0}}
        assert seen == {"dev": "cuda:0", "world": 4, "rank": 2, "peer": True}

        def boom(*a, **k):
            raise RuntimeError("nccl went away")

        bench.scale_legs = boom
        assert "nccl went away" in bench._guarded_scale_legs(args, "cuda:0", 4, 0, {"config": {}})["error"]
    finally:
        bench.scale_legs = old
