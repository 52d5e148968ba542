"""D2H of one step's store snapshot (56 B x 2^20) into host arrays: fresh pageable,
pre-touched pageable, registered (cudaHostRegister) -- where the store time goes."""
import ctypes as C
import time

import numpy as np
import torch

cud = C.CDLL("libcudart.so.12")
n = 1 << 20
steps = 30
src = torch.randn(7 * n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def run(dst, label):
    t0 = time.perf_counter()
    for t in range(steps):
        d = torch.from_numpy(dst[t])
        d.copy_(src, non_blocking=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    print(f"{label:32s} {dt * 1e3:8.3f} ms/step  {7 * n * 8 / dt / 1e9:6.2f} GB/s", flush=True)


run(np.empty((steps, 7 * n)), "fresh pageable")
a = np.empty((steps, 7 * n)); a.fill(0)
run(a, "pre-touched pageable")
b = np.empty((steps, 7 * n))
t0 = time.perf_counter()
rc = cud.cudaHostRegister(C.c_void_p(b.ctypes.data), C.c_size_t(b.nbytes), 0)
print("register", rc, f"{(time.perf_counter() - t0) * 1e3:.1f} ms for {b.nbytes / 1e9:.2f} GB", flush=True)
run(b, "registered (fresh)")
cud.cudaHostUnregister(C.c_void_p(b.ctypes.data))
c = np.empty((steps, 7 * n)); c.fill(0)
t0 = time.perf_counter()
rc = cud.cudaHostRegister(C.c_void_p(c.ctypes.data), C.c_size_t(c.nbytes), 0)
print("register touched", rc, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
run(c, "registered (touched)")
