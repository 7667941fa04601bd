"""Time the banded DP (nw_band + traceback) on shapes that separate the
per-super-step cost (one band) from the band-to-band lag (many bands)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_08639_b200 import engine

shapes = [(128, 8192), (256, 8192), (1024, 8192), (8192, 8192), (8192, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(map(int, s.split("x"))) for s in sys.argv[1:]]
os.environ.setdefault("BM_ROUTE", "banded")
for n, m in shapes:
    S = np.random.default_rng(1).random((n, m))
    St, s_off, pitch, nn, mm = engine.upload_matrices([S])
    engine.nw_paths(St, s_off, pitch, nn, mm, 0.3)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); engine.nw_paths(St, s_off, pitch, nn, mm, 0.3); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(json.dumps({"n": n, "m": m, "ms": float(np.median(ts))}), flush=True)
