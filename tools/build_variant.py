"""Build libbimine_b200 with extra -D flags into tools/_prof/<name>.so (A/B
experiments: BM_LIB_PATH=tools/_prof/<name>.so python bench.py ...)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1509_08639_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "_prof", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
subprocess.check_call(["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, *[f"-D{d}" for d in defs],
                       f"-I{B.INCLUDE}", f"-I{B.CSRC}", *[os.path.join(B.CSRC, s) for s in B.SOURCES], "-o", out])
print(out)
