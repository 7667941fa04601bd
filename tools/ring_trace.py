"""Per-document phase timeline of mine_ring_kernel on C2 (a BM_RING_PROFILE
variant). Build here: python tools/ring_trace.py --build-only [extra -D...]
Run on the GPU box:   python tools/ring_trace.py [lib]
Prints the mean per-document duration of each phase (load: hits TMA +
sentence staging, DP with the score producers, traceback, extract) and the
kernel span."""
import ctypes as C, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "--build-only":
    defs = ["BM_RING_PROFILE"] + sys.argv[2:]
    name = "ring_prof" + "".join("_" + d.split("=")[0].lower() for d in sys.argv[2:])
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), name, *defs])
    sys.exit(0)

lib_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tools", "_prof", "ring_prof.so")
os.environ["BM_LIB_PATH"] = lib_path
import numpy as np, torch  # noqa: E402
from paper_1509_08639_b200 import _native as N, engine, synth  # noqa: E402
from paper_1509_08639_b200.classifier import load_model  # noqa: E402

lib = N.lib()
sc = synth.make_corpus(*synth.c2_shape(10000), seed=1)
c, plex = sc.packed, sc.world.packed_lexicon()
dc, dl = engine.DeviceCorpus.upload(c), engine.DeviceLexicon.upload(plex)
view = engine.DocView.of(c)
model = load_model(os.path.join(ROOT, "tests", "golden", "model5k_fwd.json"))
for _ in range(3):
    engine.mine(dc, dl, view, model, 0.5, 0.2)
torch.cuda.synchronize()
n = min(c.n_docs, 16384)
buf = np.zeros((n, 6), dtype=np.uint64)
fn = lib.bm_ring_prof
fn.argtypes = [C.c_void_p, C.c_int]
assert fn(buf.ctypes.data, n) == 0
t = buf[:, :5].astype(np.int64)
t -= t[:, 0].min()
ph = np.diff(t, axis=1) / 1e3  # us
names = ["load", "dp", "traceback", "extract"]
print(f"docs {n}  span {t[:, 4].max() / 1e3:.1f} us  SMs {len(np.unique(buf[:, 5]))}")
for k, nm in enumerate(names):
    print(f"  {nm:10s} mean {ph[:, k].mean():7.2f} us  p50 {np.median(ph[:, k]):7.2f}  p99 {np.percentile(ph[:, k], 99):7.2f}")
tot = ph.sum(axis=1)
print(f"  per doc    mean {tot.mean():7.2f} us;  docs resident on average "
      f"{tot.sum() / (t[:, 4].max() / 1e3) / len(np.unique(buf[:, 5])):.2f} per SM")
