"""Time the host and device parts of one bm_mine + bm_compact step (C2)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_08639_b200 import _native as N, engine, hostapi, synth
from paper_1509_08639_b200.classifier import load_model

lib = N.lib()
sc = synth.make_corpus(*synth.c2_shape(10000), seed=1)
c = sc.packed
plex = sc.world.packed_lexicon()
dc = engine.DeviceCorpus.upload(c); dl = engine.DeviceLexicon.upload(plex)
view = engine.DocView.of(c)
n_h, m_h = view.n, view.m
amax = np.ascontiguousarray(view.token_max(c), dtype=np.int32)
dev = torch.device("cuda")
rec_off = engine.record_offsets(n_h, m_h); cap = int(np.minimum(n_h, m_h).sum())
rec = torch.empty(cap * 24, dtype=torch.uint8, device=dev); dense = torch.empty_like(rec)
cnt = torch.zeros(c.n_docs, dtype=torch.int32, device=dev); cost = torch.empty(c.n_docs, dtype=torch.float64, device=dev)
total = torch.zeros(1, dtype=torch.int64, device=dev); rod = engine.to_dev(rec_off, dev)
model = load_model("tests/golden/model5k_fwd.json")
ms = N.model_struct(model)
st = torch.cuda.current_stream(); sp = int(st.cuda_stream)
def mine():
    N.check(lib.bm_mine(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data, m_h.ctypes.data, amax.ctypes.data, C.byref(dl.lex), C.byref(ms), 0.5, 0.2, engine._ptr(rod), engine._ptr(rec), engine._ptr(cnt), engine._ptr(cost), sp))
def compact():
    N.check(lib.bm_compact(engine._ptr(rec), engine._ptr(rod), engine._ptr(cnt), c.n_docs, engine._ptr(dense), engine._ptr(total), sp))
pb = hostapi.PinnedBatch(c, plex, pin=True)
def e2e():
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
def h2d_only():
    t = torch.empty(pb.h2d_bytes, dtype=torch.uint8, device=dev)
    src = torch.from_numpy(np.frombuffer(pb.arrs["tok_id"], dtype=np.uint8))
for f, name in ((mine, "bm_mine"), (compact, "bm_compact"), (e2e, "bm_mine_host")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    hs, ds = [], []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); a.record(st); f(); t1 = time.perf_counter(); b.record(st); b.synchronize()
        hs.append(1e3 * (t1 - t0)); ds.append(a.elapsed_time(b))
    print(f"{name}: host call {np.median(hs):.2f} ms, event span {np.median(ds):.2f} ms")
# raw pinned H2D bandwidth of the batch
big = torch.empty(pb.h2d_bytes, dtype=torch.uint8, pin_memory=True); dbig = torch.empty_like(big, device=dev)
for _ in range(2): dbig.copy_(big, non_blocking=True)
torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(st); dbig.copy_(big, non_blocking=True); b.record(st); b.synchronize()
print(f"pinned H2D {pb.h2d_bytes/1e6:.1f} MB in {a.elapsed_time(b):.2f} ms = {pb.h2d_bytes/a.elapsed_time(b)/1e6:.1f} GB/s")
