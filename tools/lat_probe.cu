// Dependent-chain latency of the FP64 ops on the DP critical path (one warp).
#include <cstdio>
#include <cstdint>
__global__ void probe(double* out, long long* cyc, double a, double b, int iters) {
  double x = a, y = b;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, -b); }
  t1 = clock64(); cyc[0] = t1 - t0;
  // compare+select chain (min)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { double c = x + 0.0; x = (y < x) ? y : x; y = (x < y) ? x : y; (void)c; }
  t1 = clock64(); cyc[1] = t1 - t0;
  // fmin chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = fmin(x, y); y = fmin(y, x); }
  t1 = clock64(); cyc[2] = t1 - t0;
  // shfl chain (64-bit)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); }
  t1 = clock64(); cyc[3] = t1 - t0;
  // full cell chain: lcand = l+p; b = d; if (lcand<b) b=lcand; if (u<b) b=u; l = b
  double l = x, d = y + 1.0, u = y + 2.0, p = b;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double lc = __dadd_rn(l, p); double bb = d; if (lc < bb) bb = lc; if (u < bb) bb = u; l = bb;
    lc = __dadd_rn(l, p); bb = d; if (lc < bb) bb = lc; if (u < bb) bb = u; l = bb;
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  out[threadIdx.x] = x + y + l;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 64);
  const int it = 4096;
  probe<<<1, 32>>>(o, c, 1.0, 0.5, it); cudaDeviceSynchronize();
  probe<<<1, 32>>>(o, c, 1.0, 0.5, it); cudaDeviceSynchronize();
  const char* nm[] = {"DADD", "DSETP+FSEL min", "fmin", "SHFL.UP f64", "cell (DADD+2 min)"};
  for (int k = 0; k < 5; ++k) printf("%-20s %.1f cycles per dependent op\n", nm[k], c[k] / (2.0 * it));
  return 0;
}
