"""Time the host and device parts of one bm_mine + bm_compact step."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1509_08639_b200 import _native as N, engine, synth
from paper_1509_08639_b200.classifier import load_model

lib = N.lib()
sc = synth.make_corpus(*synth.c2_shape(10000), seed=1)
c = sc.packed
dc = engine.DeviceCorpus.upload(c); dl = engine.DeviceLexicon.upload(sc.world.packed_lexicon())
view = engine.DocView.of(c)
n_h, m_h = view.n, view.m
amax = np.ascontiguousarray(view.alpha_max(c), dtype=np.int32)
dev = torch.device("cuda")
rec_off = engine.record_offsets(n_h, m_h); cap = int(np.minimum(n_h, m_h).sum())
rec = torch.empty(cap * 24, dtype=torch.uint8, device=dev); dense = torch.empty_like(rec)
cnt = torch.zeros(c.n_docs, dtype=torch.int32, device=dev); cost = torch.empty(c.n_docs, dtype=torch.float64, device=dev)
total = torch.zeros(1, dtype=torch.int64, device=dev); rod = engine.to_dev(rec_off, dev)
model = N.model_struct(load_model("tests/golden/model5k_fwd.json"))
sp = int(torch.cuda.current_stream().cuda_stream)
def mine():
    N.check(lib.bm_mine(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data, m_h.ctypes.data, amax.ctypes.data, C.byref(dl.lex), C.byref(model), 0.5, 0.2, engine._ptr(rod), engine._ptr(rec), engine._ptr(cnt), engine._ptr(cost), sp))
def compact():
    N.check(lib.bm_compact(engine._ptr(rec), engine._ptr(rod), engine._ptr(cnt), c.n_docs, engine._ptr(dense), engine._ptr(total), sp))
for f, name in ((mine, "bm_mine"), (compact, "bm_compact")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{name}: host call {1e3*(t1-t0):.2f} ms, until done {1e3*(t2-t0):.2f} ms")
