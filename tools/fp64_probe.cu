// Latency / throughput probe of the FP64 operations on the DP critical path
// (B200 sm_100a). One warp for latencies, many warps for throughput.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double cell_old(double dg, double up, double lf, double om, double p, unsigned& code) {
  const double dc = __dadd_rn(dg, om), lc = __dadd_rn(lf, p), uc = __dadd_rn(up, p);
  double b = dc; if (lc < b) b = lc; if (uc < b) b = uc;
  code = b == dc ? 0u : (b == uc ? 1u : 2u);
  return b;
}
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  double x = a, y = b;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, b); x = __dadd_rn(x, -b); }
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = (y < x) ? y : x; y = (x < y) ? x : y; }
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); }
  t1 = clock64(); cyc[2] = t1 - t0;
  // old cell chain along a row: l feeds the next cell
  double l = x, d = y + 1.0, u = y + 2.0, p = b; unsigned cs = 0, c;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    l = cell_old(d, u, l, 0.25, p, c); cs += c;
    l = cell_old(d, u, l, 0.25, p, c); cs += c;
  }
  t1 = clock64(); cyc[3] = t1 - t0;
  // new cell: vp = v + p carried; m2 = min(lc, uc); best = dc <= m2 ? dc : m2
  double vp = l + p;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double dc = __dadd_rn(d, 0.25), uc = __dadd_rn(u, p);
      const bool g = uc <= vp; const double m2 = g ? uc : vp;
      const bool dd = dc <= m2; const double bst = dd ? dc : m2;
      cs += dd ? 0u : (g ? 1u : 2u);
      vp = __dadd_rn(bst, p);
    }
  }
  t1 = clock64(); cyc[4] = t1 - t0;
  // integer-pipe chain for reference (IADD)
  int q = (int)x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { q = q + (int)b; q = q ^ 3; }
  t1 = clock64(); cyc[5] = t1 - t0;
  // LDS chain
  __shared__ int sm[64];
  sm[threadIdx.x] = threadIdx.x; sm[threadIdx.x + 32] = 0;
  __syncwarp();
  int z = threadIdx.x & 1;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { z = sm[z]; z = sm[z + 32]; }
  t1 = clock64(); cyc[6] = t1 - t0;
  out[threadIdx.x] = x + y + l + vp + cs + q + z;
}
__global__ void thr_dadd(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __dadd_rn(a[k], 1e-12);
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 42.0) out[0] = s;
}
__global__ void thr_dsetp(double* out, int iters, double y) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (y < a[k]) ? y + a[k] * 0 : a[k];
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 42.0) out[0] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMallocManaged(&c, 64);
  const int it = 4096;
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(o, c, 1.0, 0.5, it); cudaDeviceSynchronize(); }
  const char* nm[] = {"DADD", "DSETP+FSEL min", "SHFL.UP f64", "cell old (per cell)", "cell new (per cell)", "IADD+LOP", "LDS"};
  for (int k = 0; k < 7; ++k) printf("%-22s %.1f cycles per dependent op\n", nm[k], c[k] / (2.0 * it));
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) {
    int blocks = sms * 8, iters = 8192; float ms;
    thr_dadd<<<blocks, 256>>>(o, iters); cudaEventRecord(a); thr_dadd<<<blocks, 256>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (w) printf("DADD throughput  %.2f T/s\n", 8.0 * 256 * blocks * (double)iters / (ms * 1e-3) / 1e12);
    thr_dsetp<<<blocks, 256>>>(o, iters, 0.5); cudaEventRecord(a); thr_dsetp<<<blocks, 256>>>(o, iters, 0.5); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (w) printf("DSETP+sel throughput  %.2f T/s\n", 8.0 * 256 * blocks * (double)iters / (ms * 1e-3) / 1e12);
  }
  return 0;
}
