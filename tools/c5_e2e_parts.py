"""Where the C5 end-to-end time goes: hostapi.tune_pinned as is, with the
sweep skipped (copies only) and with the copies skipped (sweep only)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1509_08639_b200 import _native as N, engine, hostapi, synth  # noqa: E402
from paper_1509_08639_b200.classifier import load_model  # noqa: E402

PENS = [0.05, 0.1, 0.2, 0.3, 0.4, 0.6, 0.8, 1.6]
THRS = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
sc = synth.make_corpus_native(*synth.c2_shape(100000), seed=5)
c = sc.packed
model = load_model(os.path.join(ROOT, "tests", "golden", "model5k_fwd.json"))
dl = engine.DeviceLexicon.upload(sc.world.packed_lexicon())
gk, goff = engine.pack_gold(sc.gold_keys())
tp = hostapi.TunePinned(c, gk, goff)


def timed(label, reps=5):
    for _ in range(2):
        hostapi.tune_pinned(tp, dl, model, PENS, THRS)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        hostapi.tune_pinned(tp, dl, model, PENS, THRS)
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / reps * 1e3:.1f} ms", flush=True)


timed("tune_pinned")
lib = N.lib()
real = lib.bm_tune


class NoTune:
    def __getattr__(self, k):
        return getattr(lib, k)

    def bm_tune(self, *a):
        return 0


N_lib = N.lib
N.lib = lambda: NoTune()
timed("copies only")
N.lib = N_lib
cp = hostapi.TunePinned.device_buffers
orig_copy = torch.Tensor.copy_
torch.Tensor.copy_ = lambda self, src, non_blocking=False: self
timed("sweep only (copies skipped)")
torch.Tensor.copy_ = orig_copy
dc = engine.DeviceCorpus.upload(c)
view = engine.DocView.of(c)
gold = engine.DeviceGold(gk, goff)
for _ in range(2):
    engine.tune_counts_device(dc, dl, view, model, PENS, THRS, gold)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    p, h = engine.tune_counts_device(dc, dl, view, model, PENS, THRS, gold)
    p.cpu()
torch.cuda.synchronize()
print(f"device-resident one call: {(time.perf_counter() - t0) / 5 * 1e3:.1f} ms")

# host time of each bm_tune call inside tune_pinned (a blocking call shows up here)
times = []


class TimedLib:
    def __getattr__(self, k):
        return getattr(lib, k)

    def bm_tune(self, *a):
        t = time.perf_counter()
        r = lib.bm_tune(*a)
        times.append((time.perf_counter() - t) * 1e3)
        return r


N.lib = lambda: TimedLib()
torch.cuda.synchronize()
t0 = time.perf_counter()
hostapi.tune_pinned(tp, dl, model, PENS, THRS)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("bm_tune host ms per chunk:", [round(x, 2) for x in times], f"call {(t1 - t0) * 1e3:.1f} ms")
N.lib = N_lib
