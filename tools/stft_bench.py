"""Device time of the STFT / inverse STFT on a resident signal (bench hook).

  python tools/stft_bench.py [reps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19388_b200 as d  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
lib = d._capi.load()
a, b = C.c_double(), C.c_double()
for (n, hop, T, M) in [(1024, 256, 626, 12), (4096, 1024, 153, 12)]:
    L = (T - 1) * hop + n
    d._capi.check(lib.dfm_bench_stft(L, M, n, hop, reps, C.byref(a), C.byref(b), 0))
    print(f"window {n} hop {hop} frames {T} channels {M}: forward {a.value:.4f} ms, inverse {b.value:.4f} ms")
