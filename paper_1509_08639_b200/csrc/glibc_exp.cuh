// Bit-exact replica of glibc 2.39 exp() as dispatched on x86-64 hosts with
// FMA+AVX2 (the "__exp_fma" ifunc variant of sysdeps/ieee754/dbl-64/e_exp.c).
//
// The reference scores every cell through CPython math.exp -> glibc exp
// (bimine/classifier.py:100-104). glibc's exp is NOT correctly rounded, so a
// CUDA exp() or a correctly rounded exp would drift by 1 ulp on ~1e-3 of the
// inputs and could flip a DP tie or a printed %.6f digit. This file restates
// the algorithm (2^(k/128) table + degree-5 polynomial) with the exact
// multiply/add/FMA pattern of the compiled FMA variant:
//
//   kd   = fma(x, InvLn2N, Shift); ki = bits(kd); kd -= Shift
//   r    = fma(kd, NegLn2loN, fma(kd, NegLn2hiN, x))
//   tmp  = fma(r2*r2, fma(r,C5,C4), fma(fma(r,C3,C2), r2, r + tail))
//   exp  = fma(scale, tmp, scale)
//
// Every non-FMA operation is an explicitly rounded intrinsic so nvcc cannot
// contract it. tests/test_exp_port.py compiles this header for the host and
// compares it with libm bit-for-bit.
#pragma once
#include <stdint.h>

#include "glibc_exp_table.h"

#if defined(__CUDACC__)
#define BM_HD __host__ __device__ __forceinline__
#else
#define BM_HD static inline
#include <math.h>
#include <string.h>
#endif

namespace bmexp {

BM_HD uint64_t asu64(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}

BM_HD double asdbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

BM_HD double fma_(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}

BM_HD double add_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}

BM_HD double sub_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

BM_HD double mul_(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}

// e_exp.c: specialcase() for 512 <= |x| < 1024 (k carries the exponent).
BM_HD double special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    double scale = asdbl(sbits);
    return mul_(fma_(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;
  double scale = asdbl(sbits);
  double st = mul_(scale, tmp);
  double y = add_(scale, st);
  if (y < 1.0) {
    double hi = add_(y, 1.0);
    double lo = add_(sub_(scale, y), st);
    double t = add_(add_(sub_(1.0, hi), y), lo);
    y = sub_(add_(t, hi), 1.0);
    if (y == 0.0) return 0.0;
  }
  return mul_(y, 0x1p-1022);
}

#if defined(__CUDACC__)
// Device copies of the polynomial constants: read from the constant bank they
// are direct DFMA operands instead of being rebuilt in registers per call.
__constant__ double c_exp_k[8] = {0x1.71547652b82fep7,  0x1.8p52,
                                  -0x1.62e42fefa0000p-8, -0x1.cf79abc9e3b3ap-47,
                                  0x1.ffffffffffdbdp-2,  0x1.555555555543cp-3,
                                  0x1.55555cf172b91p-5,  0x1.1111167a4d017p-7};
#endif
#if defined(__CUDA_ARCH__)
#define BM_EXPK(i, lit) c_exp_k[i]
#else
#define BM_EXPK(i, lit) (lit)
#endif

// T: the 256-entry table (glibc_exp_table.h); on the GPU it is staged in
// shared memory because lanes index it divergently.
// Table access: a plain pointer (host, global or generic shared memory), or on
// the device a 32-bit shared-window address read with ld.shared (the cell
// loops of the scoring kernels: no generic-to-shared conversion per lookup).
BM_HD void tab_pair(const uint64_t* T, uint32_t i, uint64_t& a, uint64_t& b) {
  a = T[i];
  b = T[i + 1];
}
#if defined(__CUDACC__)
struct SmemTab {
  uint32_t addr;  // __cvta_generic_to_shared of the staged table
};
__device__ __forceinline__ void tab_pair(SmemTab T, uint32_t i, uint64_t& a, uint64_t& b) {
  // not volatile: a read-only table, so independent lookups may be scheduled
  // freely (several cells' exp chains interleave)
  asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(T.addr + i * 8u));
}
#endif

template <class Tab>
BM_HD double exp_glibc(double x, Tab T) {
  const double InvLn2N = BM_EXPK(0, 0x1.71547652b82fep7);
  const double Shift = BM_EXPK(1, 0x1.8p52);
  const double NegLn2hiN = BM_EXPK(2, -0x1.62e42fefa0000p-8);
  const double NegLn2loN = BM_EXPK(3, -0x1.cf79abc9e3b3ap-47);
  const double C2 = BM_EXPK(4, 0x1.ffffffffffdbdp-2);
  const double C3 = BM_EXPK(5, 0x1.555555555543cp-3);
  const double C4 = BM_EXPK(6, 0x1.55555cf172b91p-5);
  const double C5 = BM_EXPK(7, 0x1.1111167a4d017p-7);

  uint32_t abstop = (uint32_t)(asu64(x) >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return add_(x, 1.0);  // |x| < 2^-54
    if (abstop >= 0x409u) {                                   // |x| >= 1024
      if (asu64(x) == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return add_(x, 1.0);
      if (asu64(x) >> 63) return 0.0;                         // underflow
      return asdbl(0x7ff0000000000000ull);                    // overflow
    }
    abstop = 0;                                               // 512 <= |x| < 1024
  }
  double kd = fma_(x, InvLn2N, Shift);
  uint64_t ki = asu64(kd);
  kd = sub_(kd, Shift);
  double r = fma_(kd, NegLn2hiN, x);
  r = fma_(kd, NegLn2loN, r);
  uint32_t idx = 2u * (uint32_t)(ki & 127u);
  uint64_t top = ki << 45;
  uint64_t w0, w1;
  tab_pair(T, idx, w0, w1);
  double tail = asdbl(w0);
  uint64_t sbits = w1 + top;
  double r2 = mul_(r, r);
  double p23 = fma_(r, C3, C2);
  double p45 = fma_(r, C5, C4);
  double t1 = fma_(p23, r2, add_(r, tail));
  double r4 = mul_(r2, r2);
  double tmp = fma_(r4, p45, t1);
  if (abstop == 0) return special(tmp, sbits, ki);
  double scale = asdbl(sbits);
  return fma_(scale, tmp, scale);
}

// bimine/classifier.py:100-117: sigmoid, then clamp into [1e-300, 1-2^-53]
// with Python's min/max semantics (first argument wins unless strictly beaten).
// The unclamped sigmoid (classifier.py:100-104), p in [0, 1] or NaN.
template <class Tab>
BM_HD double sigmoid_glibc(double z, Tab T) {
  // Branch-free form of the two sigmoid branches: exactly one exp and one
  // division per call, so lanes of a warp with mixed signs do not execute both.
  //   z >= 0: 1 / (1 + exp(-z))      z < 0 (or NaN): exp(z) / (1 + exp(z))
  const bool nonneg = z >= 0.0;
  const double e = exp_glibc(nonneg ? -z : z, T);
  const double num = nonneg ? 1.0 : e;
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(num, add_(1.0, e));
#else
  return num / (1.0 + e);
#endif
}

template <class Tab>
BM_HD double confidence_from_z(double z, Tab T) {
  const double p = sigmoid_glibc(z, T);
  const double PMIN = 1e-300;
  const double PMAX = 1.0 - 0x1p-53;
  double lo = (PMIN > p) ? PMIN : p;   // max(p, PMIN)
  return (PMAX < lo) ? PMAX : lo;      // min(lo, PMAX)
}

// 1 - confidence_from_z(z): the DP's diagonal cost. The lower clamp is not
// needed here: for 0 <= p < 2^-54 both 1 - p and 1 - 1e-300 round to 1.0.
template <class Tab>
BM_HD double one_minus_confidence(double z, Tab T) {
  const double p = sigmoid_glibc(z, T);
  const double PMAX = 1.0 - 0x1p-53;
  return sub_(1.0, (PMAX < p) ? PMAX : p);
}

}  // namespace bmexp
