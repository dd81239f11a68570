"""Host placement probe for the e2e (pinned host in / host out) path: NUMA nodes, the GPU's node,
and the 1.84 MB H2D / D2H copy time with the pinned buffers first-touched from each node's CPUs."""
import os
import subprocess
import sys
import time

import torch


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception as exc:  # noqa: BLE001
        return repr(exc)


print("cpus:", os.cpu_count(), "affinity:", len(os.sched_getaffinity(0)))
print(sh("lscpu | grep -i -E 'numa|model name|socket'"))
bdf = sh("nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader").splitlines()[0].lower()
bdf = bdf[4:] if bdf.count(":") == 2 and len(bdf.split(":")[0]) == 8 else bdf
print("gpu bdf:", bdf, "numa_node:", sh(f"cat /sys/bus/pci/devices/{bdf}/numa_node"),
      "local_cpulist:", sh(f"cat /sys/bus/pci/devices/{bdf}/local_cpulist"))
print(sh("nvidia-smi topo -m | head -5"))
print(sh("cat /sys/bus/pci/devices/%s/current_link_speed /sys/bus/pci/devices/%s/current_link_width" % (bdf, bdf)))

nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit())


def cpulist(node):
    txt = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    out = []
    for part in txt.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


n = 115200
dev = torch.device("cuda:0")
ud = torch.empty((n, 1), dtype=torch.complex128, device=dev)
full = os.sched_getaffinity(0)
for node in nodes:
    cpus = set(cpulist(node)) & full
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    # distinct sizes per node: the caching host allocator must not hand back another node's block
    extra = 4096 * (node + 1)
    uh = torch.empty((n + extra, 1), dtype=torch.complex128).pin_memory()[:n]
    uh.zero_()
    oh = torch.empty((n + 2 * extra, 1), dtype=torch.complex128).pin_memory()[:n]
    oh.zero_()
    for name, fn in (("h2d", lambda: ud.copy_(uh, non_blocking=True)), ("d2h", lambda: oh.copy_(ud, non_blocking=True))):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(200):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 200 * 1e3
        print(f"node {node} ({len(cpus)} cpus) {name}: {us:.1f} us/copy ({n * 16 / us / 1e3:.1f} GB/s), "
              f"wall {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
    del uh, oh
os.sched_setaffinity(0, full)
sys.stdout.flush()
