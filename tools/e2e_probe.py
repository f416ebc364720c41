"""e2e breakdown on configs[2]: the same 256-query call with outputs left in
HBM, copied to pinned host memory, or not written at all."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P

g = P.generate_rmat(22, 16, 3)
src = P.sample_sources(np.diff(g.out_offsets()), 256, 3).astype(np.uint32)
n, k = g.n(), len(src)
L = P.load_library()
dres = torch.empty((k, n), dtype=torch.float64, device="cuda")
drsd = torch.empty_like(dres)
hres = torch.empty((k, n), dtype=torch.float64).pin_memory()
hrsd = torch.empty_like(hres).pin_memory()


def call(rp, dp, flags):
    q = (P._abi.QStats * k)()
    c = P._abi.CStats()
    P._abi._check(L.pprg_power_push(g.handle, src.ctypes.data, k, 0.2, 1e-8, 8, -1, rp, dp, flags,
                                    q, ctypes.byref(c), None))
    return c


for name, args in (("none", (None, None, 0)), ("device", (dres.data_ptr(), drsd.data_ptr(), 1)),
                   ("host", (hres.data_ptr(), hrsd.data_ptr(), 0)),
                   ("host-reserve-only", (hres.data_ptr(), None, 0))):
    call(*args)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = call(*args)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:18s} {min(ts)*1e3:8.1f} ms  device_ms {c.device_ms:8.1f}  final {c.final_ms:6.1f}"
          f"  sweep {c.sweep_ms:7.1f}  q/s {k/min(ts):6.1f}", flush=True)

# does a concurrent D2H on another stream slow a device-output call?
big = torch.empty(2 * 64 * n, dtype=torch.float64, device="cuda")
hbig = torch.empty_like(big, device="cpu").pin_memory()
side = torch.cuda.Stream()
sub = src[:64]


def call64():
    q = (P._abi.QStats * 64)()
    c = P._abi.CStats()
    P._abi._check(L.pprg_power_push(g.handle, sub.ctypes.data, 64, 0.2, 1e-8, 8, -1,
                                    dres.data_ptr(), drsd.data_ptr(), 1, q, ctypes.byref(c), None))


call64()
for with_copy in (False, True, False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if with_copy:
        with torch.cuda.stream(side):
            hbig.copy_(big, non_blocking=True)
    call64()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"64-query call, concurrent 2.45 GB D2H={with_copy}: call {1e3*(t1-t0):.1f} ms, "
          f"all done {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
