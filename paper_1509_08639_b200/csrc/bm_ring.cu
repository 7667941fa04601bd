// Fused miner, producer/consumer form ("ring" kernel): score -> NW DP ->
// traceback -> threshold -> records for one document per CTA, nothing but the
// records leaving the SM (miner.py:84-128, aligner.py:116-206, 342-368).
//
// CTA = 4 warps.
//   1. all 128 threads: dictionary join -> per-cell coverage hit counts (smem)
//   2. warps 1-3 (producers): score exactly the cells the DP wavefront needs,
//      in wavefront-step order, and write (1 - S) into a shared-memory ring of
//      K steps x 32 lanes x R rows; warp 0 (consumer) runs the lane-skewed
//      anti-diagonal DP over the ring. Full/empty mbarriers per block of
//      kGroup steps hand ring slots back and forth, so the FP64-heavy scoring
//      runs on 96 threads at full lane utilisation while the latency-bound DP
//      chain runs on its own warp.
//   3. thread 0: traceback over the 2-bit codes in smem (tie order D > GS > GT)
//   4. all threads: re-score the diagonal cells of the path, threshold, and
//      compact them in path order.
// Same arithmetic, operation for operation, as bm_kernels.cu's kernels.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bm_kernels.cuh"

namespace bm {

constexpr int kRingThreads = 128;
constexpr int kProducers = kRingThreads - WARP;
constexpr int kRingBytes = 32 * 1024;
constexpr int kGroup = 8;       // wavefront steps per mbarrier block
constexpr int kFixedBytes = kExpTableWords * 8 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(b))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n"
      " bra WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__host__ __device__ constexpr int ring_depth(int R) { return kRingBytes / (WARP * R * 8); }

// Per-document variable shared memory (must match the device carve below).
__host__ __device__ inline size_t ring_var_bytes(int n, int m, int R) {
  const int cpw = 16 / R;
  size_t b = align16(((size_t)n * m + 1) / 2 * 4);   // hits (16-bit cells)
  b += align16((size_t)m * 8);                        // column positions
  b += align16((size_t)n * 8);                        // row positions
  b += align16((size_t)((m + cpw - 1) / cpw) * WARP * 4);  // direction codes
  b += align16((size_t)(n < m ? n : m) * 4);          // diagonal cells of the path
  return b;
}

size_t ring_slice_bytes(int n, int m, int R) {
  return kFixedBytes + kRingBytes + ring_var_bytes(n, m, R);
}

template <int R>
__global__ void __launch_bounds__(kRingThreads, 1) mine_ring_kernel(FusedArgs a) {
  constexpr int K = ring_depth(R);   // ring depth in steps
  constexpr int NB = K / kGroup;     // mbarrier blocks in the ring
  constexpr int CPW = 16 / R;        // columns per direction word
  static_assert(NB >= 2, "ring too shallow");
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const bm_sentences& S = a.S;

  uint64_t* exp_tab = (uint64_t*)smem;
  uint64_t* bar_full = (uint64_t*)(smem + kExpTableWords * 8);
  uint64_t* bar_empty = bar_full + NB;
  int* misc = (int*)(bar_empty + NB);
  double* ring = (double*)(smem + kFixedBytes);
  uint8_t* var = smem + kFixedBytes + kRingBytes;
  stage_exp_table(exp_tab, tid, kRingThreads);

  for (int item = blockIdx.x; item < a.n_list; item += gridDim.x) {
    const int doc = a.list[item];
    const int n = a.D.n[doc], m = a.D.m[doc];
    const int s0 = a.D.src0[doc], t0 = a.D.tgt0[doc];
    const double p = a.p;
    uint32_t* hits = (uint32_t*)var;
    double* cpos = (double*)(var + align16(((size_t)n * m + 1) / 2 * 4));
    double* rpos = (double*)((uint8_t*)cpos + align16((size_t)m * 8));
    uint32_t* dirs = (uint32_t*)((uint8_t*)rpos + align16((size_t)n * 8));
    const int ncg = (m + CPW - 1) / CPW;
    int32_t* dlist = (int32_t*)((uint8_t*)dirs + align16((size_t)ncg * WARP * 4));

    __syncthreads();  // the previous document is completely done with smem
    if (tid == 0) {
      for (int q = 0; q < NB; ++q) {
        mbar_init(bar_full + q, kProducers);
        mbar_init(bar_empty + q, 1);
      }
    }
    for (int j = tid; j < m; j += kRingThreads) cpos[j] = doc_pos(j, m);
    for (int i = tid; i < n; i += kRingThreads) rpos[i] = doc_pos(i, n);
    JoinSmem js = carve_join((uint8_t*)ring);  // the ring is idle during the join
    tile_join<true>(CtaGroup(), S, a.L, s0, n, t0, m, hits, js);  // ends with __syncthreads

    if (a.debug == 1) {
      if (tid == 0) {
        double sum = 0.0;
        for (int c = 0; c < n * m; ++c) {
          int hf, hr;
          read_hits<true>(hits, c, hf, hr);
          sum += hf + 1000.0 * hr;
        }
        a.cost[doc] = sum;
        a.rec_count[doc] = 0;
      }
      continue;
    }
    const int nl = (n + R - 1) / R;
    const int steps = m + nl - 1;
    const int nblocks = (steps + kGroup - 1) / kGroup;

    if (warp == 0) {
      // ------------------------------------------------------------ DP warp
      const int i0 = lane * R;
      const int my_rows = lane < nl ? min(R, n - i0) : 0;
      double left[R];
#pragma unroll
      for (int r = 0; r < R; ++r) left[r] = (double)(i0 + r + 1) * p;
      double bot = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r == my_rows - 1) bot = left[r];
      double prev_recv = (double)i0 * p;
      uint32_t dword = 0;
      double dbg_acc = 0.0;
      for (int b = 0; b < nblocks; ++b) {
        mbar_wait(bar_full + (b % NB), (uint32_t)((b / NB) & 1));
        const int s_end = min(steps, (b + 1) * kGroup);
        for (int s = b * kGroup; s < s_end; ++s) {
          const int j = s - lane;
          const double recv = __shfl_up_sync(FULL, bot, 1);
          double up, dg;
          if (lane == 0) {
            up = (double)(j + 1) * p;
            dg = (double)j * p;
          } else {
            up = recv;
            dg = prev_recv;
          }
          prev_recv = recv;
          if (lane < nl && j >= 0 && j < m) {
            const double* om = ring + ((size_t)(s % K) * WARP + lane) * R;
            double omv[R];
#pragma unroll
            for (int r = 0; r < R; ++r) omv[r] = om[r];
            if (a.debug == 2)
              for (int r = 0; r < R; ++r)
                if (r < my_rows) dbg_acc += omv[r];
            if (a.debug >= 5)
              for (int r = 0; r < R; ++r)
                if (r < my_rows) {
                  int hf, hr;
                  read_hits<true>(hits, (i0 + r) * m + j, hf, hr);
                  const double sv = cell_score(S, a.M, exp_tab, load_scalars(S, s0 + i0 + r),
                                               load_scalars(S, t0 + j), hf, hr, rpos[i0 + r], cpos[j]);
                  dbg_acc += (__dsub_rn(1.0, sv) != omv[r]) ? 1.0 : 0.0;
                }
            uint32_t codes = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if (r < my_rows) {
                const double dcand = __dadd_rn(dg, omv[r]);
                const double lcand = __dadd_rn(left[r], p);
                // min(d, u, l) with the reference's comparison semantics; l is
                // folded in first because it does not depend on the row above
                double best = dcand;
                if (lcand < best) best = lcand;
                const double ucand = __dadd_rn(up, p);
                if (ucand < best) best = ucand;
                const uint32_t code = best == dcand ? 0u : (best == ucand ? 1u : 2u);
                codes |= code << (2 * r);
                dg = left[r];
                left[r] = best;
                up = best;
              }
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r == my_rows - 1) bot = left[r];
            const int slot = j % CPW;
            dword |= codes << (2 * R * slot);
            if (slot == CPW - 1 || j == m - 1) {
              dirs[(j / CPW) * WARP + lane] = dword;
              dword = 0;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty + (b % NB));
      }
      if (lane == (n - 1) / R) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (i0 + r == n - 1) a.cost[doc] = left[r];
      }
      if (a.debug == 2 || a.debug >= 5) {
        for (int o = 16; o > 0; o >>= 1) dbg_acc += __shfl_xor_sync(FULL, dbg_acc, o);
        if (lane == 0) a.cost[doc] = dbg_acc;
      }
    } else {
      // ------------------------------------------------------ score warps
      const int ptid = tid - WARP;
      for (int b = 0; b < nblocks; ++b) {
        if (b >= NB) mbar_wait(bar_empty + (b % NB), (uint32_t)(((b / NB) - 1) & 1));
        if (a.debug == 6) __nanosleep(20000);
        // valid (lane, row) slots of each step of the block, prefix-summed
        int cnt[kGroup];
        int total = 0;
#pragma unroll
        for (int g = 0; g < kGroup; ++g) {
          const int s = b * kGroup + g;
          const int L0 = max(0, s - (m - 1));
          const int L1 = min(nl - 1, s);
          cnt[g] = (s < steps && L1 >= L0) ? (L1 - L0 + 1) * R : 0;
          total += cnt[g];
        }
        for (int f = ptid; f < total; f += kProducers) {
          int g = 0, rem = f;
#pragma unroll
          for (int q = 0; q < kGroup - 1; ++q) {
            if (g == q && rem >= cnt[q]) {
              rem -= cnt[q];
              g = q + 1;
            }
          }
          const int s = b * kGroup + g;
          const int L = max(0, s - (m - 1)) + rem / R;
          const int r = rem - (rem / R) * R;
          const int i = L * R + r;
          if (i < n) {
            const int j = s - L;
            int hf, hr;
            read_hits<true>(hits, i * m + j, hf, hr);
            const double sv = cell_score(S, a.M, exp_tab, load_scalars(S, s0 + i),
                                         load_scalars(S, t0 + j), hf, hr, rpos[i], cpos[j]);
            ring[((size_t)(s % K) * WARP + L) * R + r] = __dsub_rn(1.0, sv);
          }
        }
        mbar_arrive(bar_full + (b % NB));
      }
    }
    __syncthreads();  // DP complete: dirs final

    if (tid == 0) {
      int k = 0, i = n, j = m;
      while (i > 0 && j > 0) {
        const int ci = i - 1, cj = j - 1;
        const uint32_t wv = dirs[(cj / CPW) * WARP + ci / R];
        const uint32_t op = (wv >> (2 * R * (cj % CPW) + 2 * (ci % R))) & 3u;
        if (op == BM_MOVE_D) {
          dlist[k++] = ci * m + cj;
          --i;
          --j;
        } else if (op == BM_MOVE_GS) {
          --i;
        } else {
          --j;
        }
      }
      misc[0] = k;
    }
    __syncthreads();
    const int K_path = misc[0];

    // threshold + order-preserving block compaction (extract_pairs)
    bm_record* out = a.rec + a.rec_off[doc];
    int base = 0;
    for (int f0 = 0; f0 < K_path; f0 += kRingThreads) {
      const int f = f0 + tid;
      bool keep = false;
      int ci = 0, cj = 0;
      double sv = 0.0;
      if (f < K_path) {
        const int cell = dlist[K_path - 1 - f];
        ci = cell / m;
        cj = cell - ci * m;
        int hf, hr;
        read_hits<true>(hits, cell, hf, hr);
        sv = cell_score(S, a.M, exp_tab, load_scalars(S, s0 + ci), load_scalars(S, t0 + cj), hf,
                        hr, rpos[ci], cpos[cj]);
        keep = sv >= a.threshold;
      }
      const unsigned mask = __ballot_sync(FULL, keep);
      if (lane == 0) misc[4 + warp] = __popc(mask);
      __syncthreads();
      int before = 0, chunk = 0;
#pragma unroll
      for (int w = 0; w < kRingThreads / WARP; ++w) {
        const int c = misc[4 + w];
        before += w < warp ? c : 0;
        chunk += c;
      }
      if (keep) {
        bm_record r;
        r.doc = doc;
        r.i = ci;
        r.j = cj;
        r.pad = 0;
        r.conf = sv;
        out[base + before + __popc(mask & ((1u << lane) - 1u))] = r;
      }
      base += chunk;
      __syncthreads();  // misc reused by the next chunk
    }
    if (tid == 0) a.rec_count[doc] = base;
  }
}

cudaError_t launch_ring(const FusedArgs& a, int R, size_t smem, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  cudaError_t e;
#define BM_LAUNCH_RING(RR)                                                                   \
  e = cudaFuncSetAttribute(mine_ring_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                       \
  if (e != cudaSuccess) return e;                                                            \
  mine_ring_kernel<RR><<<a.n_list, kRingThreads, smem, st>>>(a);
  switch (R) {
    case 1: BM_LAUNCH_RING(1); break;
    case 2: BM_LAUNCH_RING(2); break;
    case 4: BM_LAUNCH_RING(4); break;
    case 8: BM_LAUNCH_RING(8); break;
    default: return cudaErrorInvalidValue;
  }
#undef BM_LAUNCH_RING
  e = cudaGetLastError();
  if (e == cudaSuccess) g_launches += 1;
  return e;
}

}  // namespace bm
