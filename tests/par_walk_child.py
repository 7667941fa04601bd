"""Child process of test_gpu_large's routing tests: BM_PAR_WALK_MIN (the
band-parallel extraction threshold) and BM_BAND_FUSED / BM_BAND_MIN_ITEMS (the
fused banded tier) are read once per process, so each setting needs its own
process. Mines the C3 tail corpus and exits 0 when records and costs equal the
oracle's."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.join(os.path.dirname(HERE), "oracle"), HERE]

import oracle  # noqa: E402  (checker only)
import paper_1509_08639_b200 as bm  # noqa: E402
from paper_1509_08639_b200 import engine  # noqa: E402
from test_gpu_large import _c3_tail_corpus  # noqa: E402
from conftest import golden  # noqa: E402


def main():
    sc = _c3_tail_corpus(int(sys.argv[1]))
    c = sc.packed
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    hb = oracle.HostBatch(c, plex)
    for t, p in ((0.5, 0.2), (0.4, 0.8), (0.0, 0.05), (0.3, float("inf"))):
        recs, cost = engine.mine(dc, dl, view, model, t, p)
        want, wcost = oracle.mine(hb, model, t, p, threads=os.cpu_count() or 8)
        assert np.array_equal(cost.view(np.uint64), wcost.view(np.uint64)), (t, p)
        assert recs.tobytes() == want.tobytes(), (t, p)
    print("records equal")


if __name__ == "__main__":
    main()
