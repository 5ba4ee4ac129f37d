"""Kernel microbenchmarks through st_debug_bench (development)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_19439_b200 as m  # noqa: E402

L = m.lib()
L.st_debug_bench.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                             C.POINTER(C.c_double)]
rp = np.array([0, 1, 2], np.int32)
g = m.TrackerSession(rp, np.array([1, 0], np.int32), np.ones(2), [1.0], np.ones((2, 1)) / np.sqrt(2), k=1)


def bench(which, N, m1, m2, flag=0, iters=10):
    ms = C.c_double()
    rc = L.st_debug_bench(g._h, which, N, m1, m2, flag, iters, C.byref(ms))
    assert rc == 0, L.st_last_error(g._h)
    return ms.value


cases = sys.argv[1:] or ["gram", "nn", "small"]
if "gram" in cases:
    for (N, a, b, sym) in [(200000, 200, 200, 1), (200000, 132, 132, 1), (200000, 164, 164, 0), (200000, 32, 200, 0),
                           (200000, 164, 32, 0), (200000, 32, 32, 0), (1000000, 32, 32, 1)]:
        t = bench(0, N, a, b, sym)
        fl = N * a * (a + 1) if sym else 2 * N * a * b
        print(f"gram N={N} {a}x{b} sym={sym}: {t*1e3:8.1f} us  {fl/t/1e9:6.2f} TF")
if "nn" in cases:
    for (N, a, b, tri) in [(200000, 200, 200, 1), (200000, 200, 100, 0), (200000, 32, 200, 0), (200000, 164, 32, 0),
                           (200000, 32, 32, 0), (1000000, 32, 32, 0)]:
        t = bench(1, N, a, b, tri)
        fl = N * a * (a + 1) if tri else 2 * N * a * b
        print(f"nn   N={N} {a}x{b} tri={tri}: {t*1e3:8.1f} us  {fl/t/1e9:6.2f} TF")
if "small" in cases:
    for w in (32, 132, 164, 200):
        print(f"chol w={w}: {bench(2, 1, w, w)*1e3:8.1f} us  chol+inv: {bench(2, 1, w, w, 1)*1e3:8.1f} us  triinv: {bench(3, 1, w, w)*1e3:8.1f} us   "
              f"eig(want 32): {bench(4, 1, w, 32, iters=3)*1e3:8.1f} us")
if cases and cases[0] == "one":  # one launch for ncu: one <which> N m1 m2 flag
    bench(int(cases[1]), int(cases[2]), int(cases[3]), int(cases[4]), int(cases[5]), iters=1)
if cases and cases[0] == "stepshapes":  # the cfg3 step's Gram/GEMM shapes at p ~ 109K rows
    N = 109268
    for (a, b, sym) in [(200, 200, 1), (164, 100, 0), (64, 200, 0), (100, 100, 1), (64, 100, 0), (32, 200, 0),
                        (64, 64, 1)]:
        t = bench(0, N, a, b, sym)
        fl = N * a * (a + 1) if sym else 2 * N * a * b
        print(f"gram N={N} {a}x{b} sym={sym}: {t*1e3:8.1f} us  {fl/t/1e9:6.2f} TF")
    for (a, b, tri) in [(200, 200, 1), (200, 100, 0), (64, 200, 0), (100, 100, 1), (64, 100, 0), (32, 200, 0),
                        (164, 32, 0)]:
        t = bench(1, N, a, b, tri)
        fl = N * a * (a + 1) if tri else 2 * N * a * b
        print(f"nn   N={N} {a}x{b} tri={tri}: {t*1e3:8.1f} us  {fl/t/1e9:6.2f} TF")
