"""Host enqueue timeline vs GPU timeline of one device-resident bm_mine on C3
(BM_TRACE=1): is the GPU waiting for the host's planning?
python tools/c3_host_trace.py [docs]"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


class A:
    c3_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    c2_docs, c5_docs = 10000, 100000


ctx = bench.Ctx(A, 0, 1, 0)
w = bench.MineWorkload(ctx, "c3")
torch = ctx.torch
for _ in range(3):
    w.mine()
torch.cuda.synchronize()
t0 = time.perf_counter()
w.mine()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3 * (t1 - t0):.1f} ms, until GPU done {1e3 * (t2 - t0):.1f} ms", file=sys.stderr)
os.environ["BM_TRACE"] = "1"
w.mine()
torch.cuda.synchronize()
