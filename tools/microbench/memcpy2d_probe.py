"""H2D throughput of a column slice of a row-major pinned fp64 block (cudaMemcpy2DAsync) vs the
whole block contiguous: can a features call upload panel B's columns while panel A filters?"""
import ctypes, glob, time, sys
import torch
N, d = 1_000_000, 56
lib = None
for pat in ("/usr/local/cuda/lib64/libcudart.so*", sys.prefix + "/lib/python3*/site-packages/nvidia/cuda_runtime/lib/libcudart.so*"):
    for p in sorted(glob.glob(pat)):
        try:
            lib = ctypes.CDLL(p); break
        except OSError:
            pass
    if lib: break
h = torch.empty((N, d), dtype=torch.float64).pin_memory()
h.normal_()
dev = torch.empty((N, d), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def c2d(ncols, col0=0):
    r = lib.cudaMemcpy2DAsync(ctypes.c_void_p(dev.data_ptr() + col0 * 8), ctypes.c_size_t(ncols * 8),
                              ctypes.c_void_p(h.data_ptr() + col0 * 8), ctypes.c_size_t(d * 8),
                              ctypes.c_size_t(ncols * 8), ctypes.c_size_t(N), 1, ctypes.c_void_p(s))
    assert r == 0, r
for name, fn, nbytes in (("full contiguous", lambda: dev.copy_(h, non_blocking=True), N * d * 8),
                         ("2D 32 of 56 cols", lambda: c2d(32), N * 32 * 8),
                         ("2D 24 of 56 cols", lambda: c2d(24, 32), N * 24 * 8),
                         ("2D 16 of 56 cols", lambda: c2d(16), N * 16 * 8)):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name:20s} {nbytes/1e6:8.1f} MB  {dt*1e3:7.2f} ms  {nbytes/dt/1e9:6.1f} GB/s", flush=True)
