"""Per-band timeline of the banded DP kernel (instrumented build).

Builds libbimine_b200 with -DBM_NW_PROFILE into tools/_prof/, loads it via
BM_LIB_PATH and prints, per (doc, band) item: start, first block, end (us,
relative to the first ticket) and lane 0's boundary wait time.
Usage: python tools/nw_trace.py [--build-only] NxM
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_prof", os.environ.get("BM_PROF_LIB", "libbimine_b200_prof.so"))


def build():
    sys.path.insert(0, ROOT)
    from paper_1509_08639_b200 import _build as B
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    extra = [f"-D{x}" for x in os.environ.get("BM_PROF_DEFS", "").split(",") if x]
    cmd = ["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DBM_NW_PROFILE", *extra, f"-I{B.INCLUDE}", f"-I{B.CSRC}",
           *[os.path.join(B.CSRC, s) for s in B.SOURCES], "-o", OUT]
    subprocess.check_call(cmd)


def main():
    if "--build-only" in sys.argv:
        build()
        return
    os.environ["BM_LIB_PATH"] = OUT
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_1509_08639_b200 import _native as N, engine
    n, m = map(int, sys.argv[1].split("x"))
    S = np.random.default_rng(1).random((n, m))
    St, s_off, pitch, nn, mm = engine.upload_matrices([S])
    for _ in range(2):
        engine.nw_paths(St, s_off, pitch, nn, mm, 0.3)
    torch.cuda.synchronize()
    nb = (n + 127) // 128
    buf = (C.c_ulonglong * (4 * nb))()
    lib = N.lib()
    assert lib.bm_nw_prof(buf, nb) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(nb, 4).astype(np.int64)
    t0 = a[:, 0].min()
    prev_first = None
    for b in range(nb):
        s, f, e, sp = a[b]
        lag = "" if prev_first is None else f"  lag_first={(f - prev_first) / 1e3:8.2f}"
        print(f"band {b:3d} start={(s - t0) / 1e3:8.2f} first={(f - t0) / 1e3:8.2f} end={(e - t0) / 1e3:8.2f} "
              f"wait_us={sp / 1e3:8.2f}{lag}")
        prev_first = f
    print("total us", (a[:, 2].max() - t0) / 1e3)
    if "--chunks" in sys.argv:
        cb = (C.c_ulonglong * (16 * 256 * 3))()
        assert lib.bm_nw_chunks(cb) == 0
        ch = np.frombuffer(cb, dtype=np.uint64).reshape(16, 256, 3).astype(np.int64)
        nch = (m + 31) // 32
        for b in range(1, min(nb, 4)):
            print(f"band {b}: chunk, publish(prev band) -> wait start, wait end (us)")
            for q in range(min(nch, 40)):
                pub = (ch[b - 1, q, 2] - t0) / 1e3
                ws, we = (ch[b, q, 0] - t0) / 1e3, (ch[b, q, 1] - t0) / 1e3
                print(f"  {q:3d} pub={pub:9.2f} start={ws:9.2f} end={we:9.2f} wait={we - ws:7.2f} "
                      f"end-pub={we - pub:7.2f}")


if __name__ == "__main__":
    main()
