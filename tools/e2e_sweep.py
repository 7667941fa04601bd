"""Wall time of bm_mine_host_packed on C2 (one setting per process: the
BM_CHUNK_CELLS / BM_MINE_STREAMS knobs are read once)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1509_08639_b200 import hostapi, synth
from paper_1509_08639_b200.classifier import load_model

sc = synth.make_corpus(*synth.c2_shape(10000), seed=1)
model = load_model(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "model5k_fwd.json"))
pb = hostapi.PinnedBatch(sc.packed, sc.world.packed_lexicon(), pin=True)
sp = int(torch.cuda.current_stream().cuda_stream)
for _ in range(5):
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    t = time.perf_counter()
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
    ts.append(time.perf_counter() - t)
ts.sort()
print(f"{os.environ.get('BM_CHUNK_CELLS', '-')} {os.environ.get('BM_FIRST_CHUNK_CELLS', '-')} {os.environ.get('BM_MINE_STREAMS', '-')} "
      f"median {ts[15]*1e3:.3f} ms  min {ts[0]*1e3:.3f} ms")
