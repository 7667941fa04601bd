"""Debug: streamed mine_corpus_file vs the oracle-based emission on a C3 JSONL
file; prints the first differing lines (tools/c3_parity.py --parts stream)."""
import hashlib
import io
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1509_08639_b200 as bm  # noqa: E402
from paper_1509_08639_b200 import synth  # noqa: E402
from paper_1509_08639_b200.ingest import NativeCorpus  # noqa: E402

n_docs = int(sys.argv[1])
path = "/tmp/c3_dbg.jsonl"
fwd = bm.load_model(os.path.join(ROOT, "tests/golden/model5k_fwd.json"))
bwd = bm.load_model(os.path.join(ROOT, "tests/golden/model5k_bwd.json"))
lex = synth.SynthWorld(5000).lexicon()
g, a, b = synth.c3_shape(n_docs, seed=2026)
synth.write_jsonl_native(path, g, a, b, seed=2026)
cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
out = io.StringIO()
bm.mine_corpus_file(path, fwd, bwd, lex, cfg, out)
got = out.getvalue().encode()
nc = NativeCorpus.load(path)
c = nc.packed
plex = nc.lexicon(lex)
wf, _ = oracle.mine(oracle.HostBatch(c, plex), fwd, 0.5, 0.2, threads=16)
wb, _ = oracle.mine(oracle.HostBatch(c, plex.swapped(), c.tgt0, c.m, c.src0, c.n), bwd, 0.5, 0.2,
                    threads=16)
k = c.n_docs
want, _ = nc.emit(wf, wb, np.zeros(k, np.uint8), np.ones(k, np.uint8), np.zeros(k, np.uint8))
print("equal", got == want, len(got), len(want))
if got != want:
    gl, wl = got.split(b"\n"), want.split(b"\n")
    for q, (x, y) in enumerate(zip(gl, wl)):
        if x != y:
            print("line", q)
            print(" got ", x[:300])
            print(" want", y[:300])
            break
# the same emission from the GPU's own records (host merge) vs the device merge
