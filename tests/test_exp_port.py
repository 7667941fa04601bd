"""The CUDA kernels' exp (csrc/glibc_exp.cuh) is a bit-exact port of glibc's.

Pinned on the CPU: the header is compiled for the host and compared with
(a) the reference's own math.exp outputs frozen in tests/golden/exp_golden.npz
and (b) this host's libm on millions of random inputs.
"""

import math
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

CSRC = os.path.join(ROOT, "paper_1509_08639_b200", "csrc")

HARNESS = r"""
#include "glibc_exp.cuh"
#include <stdio.h>
#include <stdlib.h>
static const uint64_t T[256] = BM_EXP_TABLE_INIT;
int main(int argc, char** argv) {
  if (argc > 1) {  /* random sweep against libm */
    unsigned long long s = 88172645463325252ull; long bad = 0, n = atol(argv[1]);
    for (long k = 0; k < n; ++k) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      double x;
      if (k % 3 == 0) { memcpy(&x, &s, 8); }
      else if (k % 3 == 1) { x = -745.0 * (double)(s >> 11) / 9007199254740992.0; }
      else { x = 80.0 * ((double)(s >> 11) / 9007199254740992.0 - 0.5); }
      double a = exp(x), b = bmexp::exp_glibc(x, T);
      if (memcmp(&a, &b, 8) != 0 && !(a != a && b != b)) ++bad;
    }
    printf("%ld\n", bad);
    return 0;
  }
  double x;
  while (fread(&x, 8, 1, stdin) == 1) { double y = bmexp::exp_glibc(x, T); fwrite(&y, 8, 1, stdout); }
  return 0;
}
"""


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    d = tmp_path_factory.mktemp("exp")
    src = d / "h.cpp"
    src.write_text(HARNESS)
    exe = d / "h"
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", f"-I{CSRC}", str(src), "-o", str(exe), "-lm"])
    return str(exe)


def test_table_generator_matches_header():
    import importlib.util

    spec = importlib.util.spec_from_file_location("gen", os.path.join(CSRC, "gen_exp_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    text = open(os.path.join(CSRC, "glibc_exp_table.h")).read()
    for v in gen.table()[:8]:
        assert f"0x{v:016x}ull" in text


def test_port_matches_reference_math_exp(harness):
    z = np.load(golden("exp_golden.npz"))
    out = subprocess.run([harness], input=z["z"].astype(np.float64).tobytes(), capture_output=True, check=True)
    got = np.frombuffer(out.stdout, dtype=np.uint64)
    assert got.shape == z["exp_bits"].shape
    assert np.array_equal(got, z["exp_bits"])


def test_port_matches_host_libm_random(harness):
    out = subprocess.run([harness, "3000000"], capture_output=True, check=True, text=True)
    assert int(out.stdout.strip()) == 0


def test_host_math_exp_is_the_reference_exp():
    # the golden bits came from CPython math.exp on the build host; the CPU
    # baseline assumes this host's libm agrees
    z = np.load(golden("exp_golden.npz"))
    for x, b in list(zip(z["z"], z["exp_bits"]))[::37]:
        assert struct.unpack("<Q", struct.pack("<d", math.exp(float(x))))[0] == int(b)


ONE_MINUS = r"""
#include "glibc_exp.cuh"
#include <stdio.h>
#include <string.h>
static const uint64_t T[256] = BM_EXP_TABLE_INIT;
int main() {
  /* the DP's diagonal cost 1 - S without the lower clamp == 1 - clamped S */
  unsigned long long s = 2463534242ull; long bad = 0, n = 0;
  double zs[] = {0.0, -0.0, 1e-300, -1e-300, 36.0, 37.0, 38.0, 40.0, 700.0, 800.0, -690.0,
                 -700.0, -745.0, -746.0, -800.0, 1e308, -1e308, 0.0 / 0.0};
  for (double z : zs) {
    double a = 1.0 - bmexp::confidence_from_z(z, T), b = bmexp::one_minus_confidence(z, T);
    n++; if (memcmp(&a, &b, 8) != 0 && !(a != a && b != b)) ++bad;
  }
  for (long k = 0; k < 2000000; ++k) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double z = 1600.0 * ((double)(s >> 11) / 9007199254740992.0 - 0.5);
    double a = 1.0 - bmexp::confidence_from_z(z, T), b = bmexp::one_minus_confidence(z, T);
    n++; if (memcmp(&a, &b, 8) != 0) ++bad;
  }
  printf("%ld %ld\n", bad, n);
  return 0;
}
"""


def test_ring_cost_without_lower_clamp_is_exact(tmp_path):
    """one_minus_confidence (the ring producers' 1 - S) equals 1 - S with both
    clamps for every z, including the underflow and saturation ends."""
    src = tmp_path / "om.cpp"
    src.write_text(ONE_MINUS)
    exe = tmp_path / "om"
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", f"-I{CSRC}", str(src), "-o", str(exe), "-lm"])
    bad, n = map(int, subprocess.check_output([str(exe)]).split())
    assert n > 2_000_000 and bad == 0
