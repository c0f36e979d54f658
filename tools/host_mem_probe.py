"""Host-side costs for the pageable host path: cudaHostRegister/Unregister of
a 400 MB buffer, and memcpy bandwidth (1..16 threads) into pinned memory."""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

n = 100_000_000
x = np.random.default_rng(1).integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
y = np.empty_like(x)
y[...] = 0
cudart = ctypes.CDLL("libcudart.so") if False else None
torch.cuda.init()
lib = ctypes.CDLL(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so")) \
    if os.path.exists(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so")) else None
if lib is None:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    lib = ctypes.CDLL(cands[0])
for it in range(3):
    t0 = time.perf_counter()
    r = lib.cudaHostRegister(ctypes.c_void_p(y.ctypes.data), ctypes.c_size_t(y.nbytes), 0)
    t1 = time.perf_counter()
    r2 = lib.cudaHostUnregister(ctypes.c_void_p(y.ctypes.data))
    t2 = time.perf_counter()
    print(f"register 400MB: {1e3*(t1-t0):.2f} ms (rc={r})  unregister {1e3*(t2-t1):.2f} ms (rc={r2})")
pinned = torch.empty(n, dtype=torch.uint32).pin_memory().numpy()
for threads in (1, 2, 4, 8, 16, 32):
    def work(i):
        a = i * n // threads
        b = (i + 1) * n // threads
        np.copyto(pinned[a:b], x[a:b])
    best = 1e9
    for _ in range(3):
        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        best = min(best, time.perf_counter() - t0)
    print(f"memcpy pageable->pinned {threads:2d} threads: {x.nbytes / best / 1e9:.1f} GB/s")
print("cpus", os.cpu_count())
