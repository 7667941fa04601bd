// Fused miner for documents with n <= 256 rows: score -> NW DP -> traceback
// -> threshold -> records (miner.py:84-128, aligner.py:116-206, 342-368).
//
// Two kernels:
//   hits_kernel       one CTA per document: the dictionary join (lexicon.py:
//                     88-105) into dense per-cell coverage hit counts, written
//                     to HBM scratch (2 B/cell). High occupancy hides the
//                     dependent lexicon lookups.
//   mine_ring_kernel  one CTA (4 warps) per document. The document's hit
//                     counts arrive in shared memory by one TMA bulk copy
//                     (cp.async.bulk + mbarrier complete_tx). Warps 1-3
//                     (producers) score exactly the cells the DP wavefront
//                     needs, in wavefront-step order, into a shared-memory ring
//                     of (1 - S) values; warp 0 runs the lane-skewed
//                     anti-diagonal DP over the ring (full/empty mbarriers per
//                     block of kGroup steps). Thread 0 then walks the 2-bit
//                     codes (tie order D > GS > GT) and all threads re-score
//                     the diagonal cells of the path, threshold them and
//                     compact them in path order.
// The similarity matrix never exists in memory; every value is computed with
// the same operation order as bm_kernels.cu (bit-identical to the reference).
#include <cuda_runtime.h>
#include <stdint.h>

#include "bm_kernels.cuh"

namespace bm {

constexpr int kRingThreads = 128;
constexpr int kProducers = kRingThreads - WARP;
constexpr int kGroup = 8;  // wavefront steps per mbarrier block
constexpr int kFixedBytes = kExpTableWords * 8 + 256;
constexpr int kHitsThreads = 64;

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

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(bytes)
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

// TMA 1-D bulk copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Ring of (1 - S) values: at least two mbarrier blocks of kGroup steps.
// Same as mbar_wait but sleeps between polls: the DP warp idles on the
// producers and must not steal their issue slots.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}

__host__ __device__ constexpr int ring_bytes(int R) {
  return (2 * kGroup * WARP * R * 8) > 16384 ? 2 * kGroup * WARP * R * 8 : 16384;
}
__host__ __device__ constexpr int ring_depth(int R) { return ring_bytes(R) / (WARP * R * 8); }

__host__ __device__ inline size_t hits_bytes(int n, int m) { return align16(((size_t)n * m + 1) / 2 * 4); }

// Per-document shared memory of the ring kernel (must match the carve below).
__host__ __device__ inline size_t ring_var_bytes(int n, int m, int R) {
  const int cpw = 16 / R;
  size_t b = hits_bytes(n, m);
  b += (size_t)(n + m) * 16;                                   // SPack per sentence
  b += align16((size_t)((m + cpw - 1) / cpw) * WARP * 4);      // direction codes
  b += align16((size_t)(n < m ? n : m) * 4);                   // path diagonal cells
  return b;
}

size_t ring_slice_bytes(int n, int m, int R) {
  return kFixedBytes + ring_bytes(R) + ring_var_bytes(n, m, R);
}

size_t hits_kernel_smem(int n, int m) {
  return align16(join_smem_bytes()) + align16((size_t)(n + m + 2) * 4) + (size_t)kJoinEmax * 2;
}

// ---------------------------------------------------------------------------
// hits_kernel: dictionary join of one document -> HBM scratch
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kHitsThreads, 8) hits_kernel(bm_sentences S, bm_docs D,
                                                            bm_lexicon L, const int32_t* list,
                                                            int n_list, const int64_t* hit_off,
                                                            uint8_t* hits_out) {
  // hit counters accumulate straight into the (pre-zeroed) HBM scratch with
  // L2 atomics: no per-document smem matrix, so many documents fit per SM
  extern __shared__ __align__(16) uint8_t smem[];
  const int item = blockIdx.x;
  if (item >= n_list) return;
  const int doc = list[item];
  const int n = D.n[doc], m = D.m[doc];
  JoinSmem js = carve_join(smem);
  int32_t* offS = (int32_t*)(smem + align16(join_smem_bytes()));
  int32_t* offT = offS + n + 1;
  uint16_t* chunk_owner = (uint16_t*)((uint8_t*)offS + align16((size_t)(n + m + 2) * 4));
  const int s0 = D.src0[doc], t0 = D.tgt0[doc];
  for (int k = threadIdx.x; k <= n + m + 1; k += blockDim.x) {
    if (k <= n)
      offS[k] = __ldg(S.tok_off + s0 + k);
    else
      offT[k - n - 1] = __ldg(S.tok_off + t0 + (k - n - 1));
  }
  __syncthreads();
  uint32_t* hits = (uint32_t*)(hits_out + hit_off[doc]);
  tile_join_entries<true>(CtaGroup(), S, L, s0, n, t0, m, offS, offT, hits, js, chunk_owner,
                          /*zero_hits=*/false);
}

// One sentence as the fused kernel stages it in shared memory (16 bytes):
// T, P, |A|, |D| in one byte each (routing guarantees T <= 255 and T bounds
// the other three), the offset of its digit set, its document position.
struct __align__(16) SPack {
  uint32_t tpad;  // T | P << 8 | nA << 16 | nD << 24
  int32_t d0;
  double pos;
};

// Features of one cell from staged sentences (same values, operation by
// operation, as bm_device.cuh cell_features / margin / confidence_from_z).
__device__ __forceinline__ double staged_score(const bm_sentences& S, const Model& M,
                                               const uint64_t* exp_tab, const PairTables& tb,
                                               const SPack a, const SPack b, int hf, int hr) {
  // every count is < 256 here (routing: T <= 255 bounds P, |A|, |D| and hits)
  const int aT = a.tpad & 0xff, aP = (a.tpad >> 8) & 0xff, aA = (a.tpad >> 16) & 0xff,
            aD = a.tpad >> 24;
  const int bT = b.tpad & 0xff, bP = (b.tpad >> 8) & 0xff, bA = (b.tpad >> 16) & 0xff,
            bD = b.tpad >> 24;
  double f[7];
  f[0] = __ldg(tb.ratio2 + aT * kPairMax + bT);
  f[1] = __ldg(tb.frac2 + hf * kPairMax + aA);
  f[2] = __ldg(tb.frac2 + hr * kPairMax + bA);
  if ((aD | bD) == 0) {
    f[3] = 1.0;
  } else if (aD == 0 || bD == 0) {
    f[3] = 0.0;  // 0 / |D_s | D_t|
  } else {
    const int inter = sorted_intersection(S.dig_id + a.d0, aD, S.dig_id + b.d0, bD);
    f[3] = frac_or_zero(inter, aD + bD - inter);
  }
  f[4] = __ldg(tb.ratio2 + aP * kPairMax + bP);
  f[5] = __dsub_rn(1.0, fabs(__dsub_rn(a.pos, b.pos)));
  f[6] = 1.0;
  return bmexp::confidence_from_z(margin(M, f), exp_tab);
}

// Valid (lane, row) slots of wavefront step s: lanes max(0, s-m+1) ..
// min(nl-1, s), R rows each.
__device__ __forceinline__ int step_slots(int s, int steps, int m, int nl, int R) {
  if (s >= steps) return 0;
  const int L0 = max(0, s - (m - 1));
  const int L1 = min(nl - 1, s);
  return (L1 - L0 + 1) * R;
}

template <int R>
__global__ void __launch_bounds__(kRingThreads, 5) mine_ring_kernel(FusedArgs a) {
  constexpr int K = ring_depth(R);  // ring depth in steps
  constexpr int NB = K / kGroup;    // mbarrier blocks in the ring
  constexpr int CPW = 16 / R;       // columns per direction word
  static_assert(NB >= 2, "ring too shallow");
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const bm_sentences& S = a.S;

  uint64_t* exp_tab = (uint64_t*)smem;
  uint64_t* bar_full = (uint64_t*)(smem + kExpTableWords * 8);
  uint64_t* bar_empty = bar_full + NB;
  uint64_t* bar_load = bar_empty + NB;
  int* misc = (int*)(bar_load + 1);
  double* ring = (double*)(smem + kFixedBytes);
  uint8_t* var = smem + kFixedBytes + ring_bytes(R);
  stage_exp_table(exp_tab, tid, kRingThreads);

  for (int item = blockIdx.x; item < a.n_list; item += gridDim.x) {
    const int doc = a.list[item];
    const int n = a.D.n[doc], m = a.D.m[doc];
    const int s0 = a.D.src0[doc], t0 = a.D.tgt0[doc];
    const double p = a.p;
    const int ncg = (m + CPW - 1) / CPW;
    uint32_t* hits = (uint32_t*)var;
    SPack* sp = (SPack*)(var + hits_bytes(n, m));
    uint32_t* dirs = (uint32_t*)((uint8_t*)sp + (size_t)(n + m) * 16);
    int32_t* dlist = (int32_t*)((uint8_t*)dirs + align16((size_t)ncg * WARP * 4));

    __syncthreads();  // the previous document is done with every buffer
    if (tid == 0) {
      for (int q = 0; q < NB; ++q) {
        mbar_init(bar_full + q, kProducers);
        mbar_init(bar_empty + q, 1);
      }
      mbar_init(bar_load, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t bytes = (uint32_t)hits_bytes(n, m);
      mbar_arrive_expect_tx(bar_load, bytes);
      bulk_g2s(hits, a.hits + a.hit_off[doc], bytes, bar_load);
    }
    // sentences of the document (rows 0..n-1, then columns)
    for (int k = tid; k < n + m; k += kRingThreads) {
      const bool row = k < n;
      const int g = row ? s0 + k : t0 + (k - n);
      const SentScalars v = load_scalars(S, g);
      SPack q;
      q.tpad = (uint32_t)v.T | ((uint32_t)v.P << 8) | ((uint32_t)v.nA << 16) | ((uint32_t)v.nD << 24);
      q.d0 = v.d0;
      q.pos = row ? doc_pos(k, n) : doc_pos(k - n, m);
      sp[k] = q;
    }
    __syncthreads();
    mbar_wait(bar_load, 0);

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
      for (int b = 0; b < nblocks; ++b) {
        mbar_wait_sleep(bar_full + (b % NB), (uint32_t)((b / NB) & 1));
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
                bot = best;  // the last valid row of the lane ends the chain
              }
            }
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
    } else {
      // ------------------------------------------------------ score warps
      const int ptid = tid - WARP;
      for (int b = 0; b < nblocks; ++b) {
        if (b >= NB) mbar_wait(bar_empty + (b % NB), (uint32_t)(((b / NB) - 1) & 1));
        const int s_end = min(steps, (b + 1) * kGroup);
        // walk this thread's slots (stride kProducers over the concatenated
        // valid slots of the block's steps); the step state (s, first valid
        // lane L0, slot count) only changes when the walk crosses a step
        int s = b * kGroup, rem = ptid;
        int L0 = max(0, s - (m - 1));
        int cnt = step_slots(s, steps, m, nl, R);
        while (s < s_end && rem >= cnt) {
          rem -= cnt;
          ++s;
          L0 = max(0, s - (m - 1));
          cnt = step_slots(s, steps, m, nl, R);
        }
        while (s < s_end) {
          const int L = L0 + rem / R;
          const int r = rem % R;
          const int i = L * R + r;
          if (i < n) {
            const int j = s - L;
            const uint32_t hv = ((const uint16_t*)hits)[i * m + j];
            const double sv = staged_score(S, a.M, exp_tab, a.tabs, sp[i], sp[n + j], hv & 0xff, hv >> 8);
            ring[((s % K) * WARP + L) * R + r] = __dsub_rn(1.0, sv);
          }
          rem += kProducers;
          while (rem >= cnt && s < s_end) {
            rem -= cnt;
            ++s;
            L0 = max(0, s - (m - 1));
            cnt = step_slots(s, steps, m, nl, R);
          }
        }
        mbar_arrive(bar_full + (b % NB));
      }
    }
    __syncthreads();  // DP complete: direction codes final

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
        const uint32_t hv = ((const uint16_t*)hits)[cell];
        sv = staged_score(S, a.M, exp_tab, a.tabs, sp[ci], sp[n + cj], hv & 0xff, hv >> 8);
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

cudaError_t launch_hits(const FusedArgs& a, size_t smem, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(hits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(hits_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  hits_kernel<<<a.n_list, kHitsThreads, smem, st>>>(a.S, a.D, a.L, a.list, a.n_list, a.hit_off,
                                                     a.hits);
  (void)0;
  e = cudaGetLastError();
  if (e == cudaSuccess) g_launches += 1;
  return e;
}

cudaError_t launch_ring(const FusedArgs& a, int R, size_t smem, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  cudaError_t e;
#define BM_LAUNCH_RING(RR)                                                                   \
  e = cudaFuncSetAttribute(mine_ring_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)smem);                                                       \
  if (e != cudaSuccess) return e;                                                            \
  e = cudaFuncSetAttribute(mine_ring_kernel<RR>,                                             \
                           cudaFuncAttributePreferredSharedMemoryCarveout, 100);             \
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
