"""GPU timeline of one bm_mine_host_wire call on C2 (BM_TRACE=1 output)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BM_TRACE"] = "1"
import torch
from paper_1509_08639_b200 import hostapi, synth
from paper_1509_08639_b200.classifier import load_model

n_docs = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
sc = synth.make_corpus(*synth.c2_shape(n_docs), seed=1)
model = load_model(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "model5k_fwd.json"))
pb = hostapi.PinnedBatch(sc.packed, sc.world.packed_lexicon(), pin=True)
sp = int(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    hostapi.mine_pinned(pb, model, 0.5, 0.2, sp)
torch.cuda.synchronize()
print("h2d bytes", pb.h2d_bytes, file=sys.stderr)
