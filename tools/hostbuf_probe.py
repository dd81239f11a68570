"""H2D / D2H time of a 1.84 MB (cfg2 vector) copy from pinned host buffers allocated different ways:
torch pin_memory (caching host allocator), cudaHostAlloc, and 2 MB-aligned anonymous mmap with
MADV_HUGEPAGE + cudaHostRegister.  Probes whether the host->device direction is limited by the
IOMMU / page size of the pinned buffer rather than by PCIe."""
import ctypes
import ctypes.util
import mmap
import time

import torch

libc = ctypes.CDLL(ctypes.util.find_library("c"), use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = ctypes.CDLL("libcudart.so.12") if False else None


def sh(path):
    try:
        return open(path).read().strip()
    except OSError as exc:
        return repr(exc)


print("THP enabled:", sh("/sys/kernel/mm/transparent_hugepage/enabled"))
print("THP defrag:", sh("/sys/kernel/mm/transparent_hugepage/defrag"))
print("hugepages:", sh("/proc/sys/vm/nr_hugepages"))
print("iommu groups:", len(__import__("os").listdir("/sys/kernel/iommu_groups")) if __import__("os").path.isdir(
    "/sys/kernel/iommu_groups") else "none")

n = 115200
nbytes = n * 16
dev = torch.device("cuda:0")
ud = torch.empty((n,), dtype=torch.complex128, device=dev)
rt = torch.cuda.cudart()
HUGE = 2 << 20
MADV_HUGEPAGE = 14


def mmap_buf(huge: bool):
    size = 4 * HUGE
    p = libc.mmap(None, size, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    base = (p + HUGE - 1) // HUGE * HUGE
    if huge:
        libc.madvise(ctypes.c_void_p(base), 2 * HUGE, MADV_HUGEPAGE)
    buf = (ctypes.c_char * (2 * HUGE)).from_address(base)
    ctypes.memset(base, 0, 2 * HUGE)
    rc = rt.cudaHostRegister(base, 2 * HUGE, 0)
    t = torch.frombuffer(buf, dtype=torch.complex128, count=n)
    return t, rc, base


def hostalloc():
    # cudaHostAlloc through the CUDA runtime bundled with torch
    lib = ctypes.CDLL(None)
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    ptr = ctypes.c_void_p()
    rc = lib.cudaHostAlloc(ctypes.byref(ptr), ctypes.c_size_t(nbytes), 0)
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    return torch.frombuffer(buf, dtype=torch.complex128, count=n), rc, ptr.value


def smaps_kernelpagesize(addr):
    try:
        cur = None
        for line in open("/proc/self/smaps"):
            if "-" in line.split()[0] and len(line.split()) >= 5:
                a, b = (int(x, 16) for x in line.split()[0].split("-"))
                cur = a <= addr < b
            elif cur and line.startswith(("AnonHugePages", "KernelPageSize")):
                print("   ", line.strip())
    except OSError:
        pass


def timeit(name, h):
    for direction, fn in (("h2d", lambda: ud.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(ud, non_blocking=True))):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(300):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 300 * 1e3
        print(f"{name:28s} {direction}: {us:6.1f} us ({nbytes / us / 1e3:5.1f} GB/s)")


for i in range(3):
    t = torch.empty((n,), dtype=torch.complex128).pin_memory()
    t.zero_()
    timeit(f"torch pin_memory #{i} @{t.data_ptr() % HUGE:#x}", t)
    smaps_kernelpagesize(t.data_ptr())
for i in range(2):
    t, rc, base = hostalloc()
    timeit(f"cudaHostAlloc #{i} rc={rc} @{base % HUGE:#x}", t)
    smaps_kernelpagesize(base)
for huge in (False, True, True):
    t, rc, base = mmap_buf(huge)
    timeit(f"mmap huge={huge} register rc={rc}", t)
    smaps_kernelpagesize(base)
