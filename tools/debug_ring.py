"""Debug helper: ring-kernel costs/records vs the oracle on a few docs."""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")]
import numpy as np
import oracle
import paper_1509_08639_b200 as bm
from paper_1509_08639_b200 import engine, synth

sc = synth.make_corpus([3, 60], [2, 40], [2, 40], seed=3)
model = bm.load_model("tests/golden/model5k_fwd.json")
plex = sc.world.packed_lexicon()
recs, cost = engine.mine(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                         engine.DocView.of(sc.packed), model, 0.5, 0.2)
want, wcost = oracle.mine(oracle.HostBatch(sc.packed, plex), model, 0.5, 0.2, threads=4)
print("gpu cost", cost, "oracle", wcost)
print("gpu recs", len(recs), "oracle", len(want))
print(recs[:5]); print(want[:5])
from paper_1509_08639_b200.pack import PackedCorpus
import ctypes
os.environ["BM_RING_DEBUG"] = "1"
recs, cost = engine.mine(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                         engine.DocView.of(sc.packed), model, 0.5, 0.2)
print("hit sums (hf + 1000 hr)", cost)
S = bm.aligner  # expected from K1 path
from paper_1509_08639_b200 import engine as E
Sbuf, s_off, pitch, _, _ = E.score(E.DeviceCorpus.upload(sc.packed), E.DeviceLexicon.upload(plex), E.DocView.of(sc.packed), model)
mats = E.matrices_from_buffer(Sbuf, s_off, pitch, sc.packed.n, sc.packed.m)
print("K1 S sums", [float(x.sum()) for x in mats], "max", [float(x.max()) for x in mats])
os.environ["BM_RING_DEBUG"] = "2"
recs, cost = engine.mine(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                         engine.DocView.of(sc.packed), model, 0.5, 0.2)
print("consumer sum(1-S)", cost, "expected", [x.size - float(x.sum()) for x in mats])
for mode in ("5", "6"):
    os.environ["BM_RING_DEBUG"] = mode
    recs, cost = engine.mine(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                             engine.DocView.of(sc.packed), model, 0.5, 0.2)
    print("mode", mode, "mismatches", cost)
