"""Timeline of the C3 end-to-end call (bm_mine_host_packed, BM_TRACE=1) vs
the device-resident bm_mine on the same documents: python tools/e2e_c3_trace.py [docs]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1509_08639_b200 import engine, hostapi, synth  # noqa: E402
from paper_1509_08639_b200.classifier import load_model  # noqa: E402

n_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
g, a, b = synth.c2_shape(n_docs) if "--c2" in sys.argv else synth.c3_shape(n_docs, seed=2026)
sc = synth.make_corpus_native(g, a, b, seed=2026)
model = load_model(os.path.join(ROOT, "tests", "golden", "model5k_fwd.json"))
plex = sc.world.packed_lexicon()
pb = hostapi.PinnedBatch(sc.packed, plex, pin=True)
sp = int(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
torch.cuda.synchronize()
print(f"e2e {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms per call, h2d {pb.h2d_bytes / 1e9:.2f} GB",
      file=sys.stderr)
dc = engine.DeviceCorpus.upload(sc.packed)
dl = engine.DeviceLexicon.upload(plex)
view = engine.DocView.of(sc.packed)
for _ in range(2):
    engine.mine_device(dc, dl, view, model, 0.5, 0.2)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    engine.mine_device(dc, dl, view, model, 0.5, 0.2)
torch.cuda.synchronize()
print(f"device-resident {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms per call", file=sys.stderr)
if "--trace" in sys.argv:
    os.environ["BM_TRACE"] = "1"
    engine.mine_device(dc, dl, view, model, 0.5, 0.2)
    torch.cuda.synchronize()
    del os.environ["BM_TRACE"]
    for k in range(3):  # the last of three traced calls is the steady state
        if k == 2:
            os.environ["BM_TRACE"] = "1"
        hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
        torch.cuda.synchronize()
