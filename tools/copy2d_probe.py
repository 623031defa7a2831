"""H2D rates: 1-D copy vs the pipeline's 2-D chunk copy (100 rows of a
node-major b x tau pinned array), one stream or split over two.
python tools/copy2d_probe.py"""
import ctypes
import time

import torch

b, tau, chunk = 100, 525600, 36864
host = torch.empty((b, tau), dtype=torch.complex128).pin_memory()
dev = torch.empty((b, chunk), dtype=torch.complex128, device="cuda")
dev2 = torch.empty(b * chunk, dtype=torch.complex128, device="cuda")
flat = torch.empty(b * chunk, dtype=torch.complex128).pin_memory()
cudart = ctypes.CDLL("libcudart.so")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


nbytes = b * chunk * 16
one_d = t(lambda: dev2.copy_(flat, non_blocking=True))
print("1-D  %.1f GB/s" % (nbytes / one_d / 1e9))


def two_d(rows0, rows1, stream):
    cudart.cudaMemcpy2DAsync(ctypes.c_void_p(dev.data_ptr() + rows0 * chunk * 16), ctypes.c_size_t(chunk * 16),
                             ctypes.c_void_p(host.data_ptr() + rows0 * tau * 16), ctypes.c_size_t(tau * 16),
                             ctypes.c_size_t(chunk * 16), ctypes.c_size_t(rows1 - rows0), 1,
                             ctypes.c_void_p(stream.cuda_stream))


print("2-D  %.1f GB/s" % (nbytes / t(lambda: two_d(0, b, s1)) / 1e9))
print("2-D x2 streams %.1f GB/s" % (nbytes / t(lambda: (two_d(0, b // 2, s1), two_d(b // 2, b, s2))) / 1e9))

# both directions at once, as in the pipeline (H2D of one chunk, D2H of another)
hostv = torch.empty((b, tau), dtype=torch.complex128).pin_memory()
devv = torch.empty((b, chunk), dtype=torch.complex128, device="cuda")


def d2h_2d(stream):
    cudart.cudaMemcpy2DAsync(ctypes.c_void_p(hostv.data_ptr()), ctypes.c_size_t(tau * 16),
                             ctypes.c_void_p(devv.data_ptr()), ctypes.c_size_t(chunk * 16),
                             ctypes.c_size_t(chunk * 16), ctypes.c_size_t(b), 2, ctypes.c_void_p(stream.cuda_stream))


flatv = torch.empty(b * chunk, dtype=torch.complex128).pin_memory()
dev2v = torch.empty(b * chunk, dtype=torch.complex128, device="cuda")


def both_1d():
    with torch.cuda.stream(s1):
        dev2.copy_(flat, non_blocking=True)
    with torch.cuda.stream(s2):
        flatv.copy_(dev2v, non_blocking=True)


print("bidirectional 1-D  %.1f GB/s per direction" % (nbytes / t(both_1d) / 1e9))
print("bidirectional 2-D  %.1f GB/s per direction" % (nbytes / t(lambda: (two_d(0, b, s1), d2h_2d(s2))) / 1e9))
