// Fused miner for documents with n <= 256 rows: score -> NW DP -> traceback
// -> threshold -> records (miner.py:84-128, aligner.py:116-206, 342-368).
//
// Two kernels:
//   hits_kernel       one CTA per document: the dictionary join (lexicon.py:
//                     88-105) into dense per-cell coverage hit counts, written
//                     to HBM scratch (2 B/cell). High occupancy hides the
//                     dependent lexicon lookups.
//   mine_ring_kernel  one CTA (5 warps) per document. The document's hit
//                     counts arrive in shared memory by one TMA bulk copy
//                     (cp.async.bulk + mbarrier complete_tx). Warps 1-4
//                     (producers) score the R x 4 lane blocks the DP needs,
//                     super-step by super-step, as 32-cell tasks dealt
//                     round-robin, into a 4-slot shared-memory ring of
//                     (1 - S); warp 0 runs the blocked wavefront DP of
//                     nw_band_kernel over it (full/empty mbarriers per slot,
//                     waits suspend in hardware). Thread 0 then walks the
//                     2-bit codes (tie order D > GS > GT) and all threads
//                     re-score the diagonal cells of the path, threshold them
//                     and compact them in path order.
// The similarity matrix never exists in memory; every value is computed with
// the same operation order as bm_kernels.cu (bit-identical to the reference).
#include <mutex>
#include <unordered_map>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "bm_kernels.cuh"

namespace bm {

constexpr int kProdWarps = 4;
constexpr int kRingThreads = (kProdWarps + 1) * WARP;  // warp 0: DP, warps 1..4: scoring
constexpr int kProducers = kProdWarps * WARP;
#ifndef BM_RING_SLOTS
#define BM_RING_SLOTS 2
#endif
// scoring warps: one full-barrier arrival per warp; empty-slot waits sleep up
// to BM_RING_SLEEP_NS (0: try_wait loop)
#ifndef BM_RING_WARP_ARRIVE
#define BM_RING_WARP_ARRIVE 0
#endif
#ifndef BM_RING_SLEEP_NS
#define BM_RING_SLEEP_NS 0
#endif
// cells per scoring thread and task (one row of a lane block: 4; half a row:
// 2; one cell: 1)
#ifndef BM_RING_CPT
#define BM_RING_CPT 1
#endif
#ifndef BM_RING_MINB
#define BM_RING_MINB 6
#endif
constexpr int kSlots = BM_RING_SLOTS;  // ring depth in super-steps
constexpr int kFixedBytes = kExpTableWords * 8 + 256;
#ifndef BM_HITS_THREADS
#define BM_HITS_THREADS 64
#endif
constexpr int kHitsThreads = BM_HITS_THREADS;

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

// Waits that suspend the thread in hardware (try_wait with a suspend-time
// hint) until the phase completes, instead of polling: a warp stalled on its
// partner must not take issue slots from the other CTAs on the SM.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}

// A wait that does not spin on the issue slots: a non-blocking phase test,
// then a sleep that doubles up to max_ns. For warps whose wait is not on the
// critical path (scoring warps ahead of their DP warp): try_wait with a
// suspend hint wakes at every mbarrier event of the CTA, and the producers'
// retry loop took a quarter of the fused banded kernel's issue slots.
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred P1;\n mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      " selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t max_ns) {
  uint32_t ns = 32;
  while (!mbar_test(b, parity)) {
    __nanosleep(ns);
    ns = ns < max_ns ? 2 * ns : max_ns;
  }
}

__host__ __device__ constexpr int ring_lane(int R) { return R * 4 + 2; }
// slots hold only the document's nl active DP lanes (smem decides how many
// CTAs share an SM)
__host__ __device__ constexpr int ring_slot_doubles(int R, int nl) { return nl * ring_lane(R); }
__host__ __device__ inline size_t ring_bytes(int R, int nl) {
  return align16((size_t)kSlots * ring_slot_doubles(R, nl) * 8);
}
// 2-bit codes of one lane block (R rows x 4 columns, bit 2*(c*R + r))
__host__ __device__ constexpr int code_bytes(int R) { return R == 8 ? 8 : 4; }

__host__ __device__ inline size_t hits_bytes(int n, int m) { return align16(((size_t)n * m + 1) / 2 * 4); }

// Per-document shared memory of the ring kernel (must match the carve below).
// BM_RING_FUSED_JOIN=1: each CTA runs its document's dictionary join itself
// (hit counts accumulate in shared memory; the join's scratch shares the ring's
// space, which is free until scoring starts). 0 (default): the hits_kernel
// writes the counts to HBM scratch and the CTA loads them with one TMA bulk
// copy. Measured on C2: fused 1.78 ms vs 0.33 + 1.11 ms split -- the join's
// dependent lexicon lookups need the hits kernel's occupancy (15 small CTAs
// per SM) to hide their latency.
#ifndef BM_RING_FUSED_JOIN
#define BM_RING_FUSED_JOIN 0
#endif

// join scratch of the fused CTA: bucket table, staged offsets, owner tables
__host__ __device__ inline size_t join_scratch_bytes(int n, int m) {
  return align16(join_smem_bytes()) + align16((size_t)(n + m + 2) * 4) + (size_t)kJoinEmax * 4;
}

// bytes of the region shared by the join scratch and the ring
__host__ __device__ inline size_t union_bytes(int n, int m, int R) {
  const size_t rb = ring_bytes(R, (n + R - 1) / R);
  if (!BM_RING_FUSED_JOIN) return rb;
  const size_t jb = align16(join_scratch_bytes(n, m));
  return rb > jb ? rb : jb;
}

__host__ __device__ inline size_t ring_var_bytes(int n, int m, int R) {
  size_t b = hits_bytes(n, m);
  b += (size_t)(n + m) * 16;                                         // SPack per sentence
  b += align16((size_t)((m + 3) / 4) * WARP * code_bytes(R));        // direction codes
  b += align16((size_t)(n < m ? n : m) * 4);                         // path diagonal cells
  return b;
}

size_t ring_slice_bytes(int n, int m, int R) {
  return kFixedBytes + union_bytes(n, m, R) + ring_var_bytes(n, m, R);
}

size_t hits_kernel_smem(int n, int m) {
  return align16(join_smem_bytes()) + align16((size_t)(n + m + 2) * 4) + (size_t)kJoinEmax * 4;
}

// ---------------------------------------------------------------------------
// hits_kernel: dictionary join of one document -> HBM scratch
// ---------------------------------------------------------------------------
#ifndef BM_HITS_MINB
#define BM_HITS_MINB 8
#endif
__global__ void __launch_bounds__(kHitsThreads, BM_HITS_MINB) hits_kernel(bm_sentences S, bm_docs D,
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
  uint16_t* a_owner = chunk_owner + kJoinEmax;
  const int s0 = D.src0[doc], t0 = D.tgt0[doc];
  for (int k = threadIdx.x; k <= n + m + 1; k += blockDim.x) {
    if (k <= n)
      offS[k] = __ldg(S.tok_off + s0 + k);
    else
      offT[k - n - 1] = __ldg(S.tok_off + t0 + (k - n - 1));
  }
  __syncthreads();
  uint32_t* hits = (uint32_t*)(hits_out + hit_off[doc]);
  tile_join_entries<true>(CtaGroup(), S, L, s0, n, t0, m, offS, offT, hits, js, chunk_owner, a_owner,
                          /*zero_hits=*/false);
}

// One sentence as the fused kernel stages it in shared memory (16 bytes):
// T, P, |A|, |D| in one byte each (routing guarantees T <= 255 and T bounds
// the other three), the offset of its digit set, its document position.
struct __align__(16) SPack {
  uint32_t tpad;  // T | P << 8 | nA << 16 | nD << 24
  uint32_t dx;    // digit word (digit_word: signature, or kDigMany | offset)
  double pos;
};

// One staged sentence as a single 16-byte shared-memory load.
__device__ __forceinline__ SPack ld_spack(const SPack* p) {
  const int4 v = *reinterpret_cast<const int4*>(p);
  SPack q;
  q.tpad = (uint32_t)v.x;
  q.dx = (uint32_t)v.y;
  q.pos = __hiloint2double(v.w, v.z);
  return q;
}

// Features of one cell from staged sentences (same values, operation by
// operation, as bm_device.cuh cell_features / margin / confidence_from_z).
// BM_RING_FOLD=1: the margin from the model's folded tables (ModelTables):
// z = z1[aT,bT] + p1[hf,|A_s|] + p2[hr,|A_t|] + w3*f3 + p4[aP,bP] + w5*f5 + w6,
// the same additions in the same order as margin(), whose products the tables
// hold (w*1.0 == w, so f6 and the common f3 = 1 need no multiply).
#ifndef BM_RING_FOLD
#define BM_RING_FOLD 1
#endif
__device__ __forceinline__ double staged_margin(const bm_sentences& S, const Model& M,
                                                const PairTables& tb, const ModelTables& mt,
                                                const SPack a, const SPack b, int hf, int hr) {
  // every count is < 256 here (routing: T <= 255 bounds P, |A|, |D| and hits)
  const int aT = a.tpad & 0xff, aP = (a.tpad >> 8) & 0xff, aA = (a.tpad >> 16) & 0xff,
            aD = a.tpad >> 24;
  const int bT = b.tpad & 0xff, bP = (b.tpad >> 8) & 0xff, bA = (b.tpad >> 16) & 0xff,
            bD = b.tpad >> 24;
#if BM_RING_FOLD
  double z = __ldg(mt.z1 + aT * kPairMax + bT);
  z = __dadd_rn(z, __ldg(mt.p1 + hf * kPairMax + aA));
  z = __dadd_rn(z, __ldg(mt.p2 + hr * kPairMax + bA));
  z = __dadd_rn(z, digit_term_w(S, M, __dmul_rn(M.w[3], 0.0), a.dx, b.dx, aD, bD));
  z = __dadd_rn(z, __ldg(mt.p4 + aP * kPairMax + bP));
  z = __dadd_rn(z, __dmul_rn(M.w[5], __dsub_rn(1.0, fabs(__dsub_rn(a.pos, b.pos)))));
  z = __dadd_rn(z, M.w[6]);  // w6 * 1.0
  return z;
#else
  double f[7];
  f[0] = __ldg(tb.ratio2 + aT * kPairMax + bT);
  f[1] = __ldg(tb.frac2 + hf * kPairMax + aA);
  f[2] = __ldg(tb.frac2 + hr * kPairMax + bA);
  if ((aD | bD) == 0) {
    f[3] = 1.0;
  } else if (aD == 0 || bD == 0) {
    f[3] = 0.0;  // 0 / |D_s | D_t|
  } else {
    const int inter = digit_inter(S, a.dx, b.dx, aD, bD);
    f[3] = frac_or_zero(inter, aD + bD - inter);
  }
  f[4] = __ldg(tb.ratio2 + aP * kPairMax + bP);
  f[5] = __dsub_rn(1.0, fabs(__dsub_rn(a.pos, b.pos)));
  f[6] = 1.0;
  return margin(M, f);
#endif
}

__device__ __forceinline__ double staged_score(const bm_sentences& S, const Model& M,
                                               const uint64_t* exp_tab, const PairTables& tb,
                                               const ModelTables& mt, const SPack a,
                                               const SPack b, int hf, int hr) {
  return bmexp::confidence_from_z(staged_margin(S, M, tb, mt, a, b, hf, hr), exp_tab);
}

// Lanes of the DP warp active at super-step t (lane L works on column group
// t - L): [L0, L1], empty when L0 > L1.
__device__ __forceinline__ int2 active_lanes(int t, int ngroups, int nl) {
  return make_int2(max(0, t - ngroups + 1), min(nl - 1, t));
}

// 5 CTAs per SM (smem slices of C2-shaped documents fit 5); R = 8 blocks need
// the registers of 4
#ifdef BM_RING_PROFILE
// tools/ring_trace.py: per document (first 16384 of a launch) globaltimer
// stamps [start, loaded, DP done, traceback done, end] and the SM id
__device__ unsigned long long g_ring_prof[16384][6];
__device__ __forceinline__ unsigned long long ring_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define RING_PROF(slot)                                                   \
  if (tid == 0 && item < 16384) {                                         \
    g_ring_prof[item][slot] = ring_timer();                               \
    if (slot == 0) {                                                      \
      unsigned s;                                                         \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(s));                      \
      g_ring_prof[item][5] = s;                                           \
    }                                                                     \
  }
#else
#define RING_PROF(slot)
#endif

template <int R>
__global__ void __launch_bounds__(kRingThreads, R == 8 ? 4 : BM_RING_MINB) mine_ring_kernel(FusedArgs a) {
  using CodeT = typename std::conditional<R == 8, uint64_t, uint32_t>::type;
  constexpr int RL = ring_lane(R);
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bm_sentences& S = a.S;

  uint64_t* exp_tab = (uint64_t*)smem;
  uint64_t* bar_full = (uint64_t*)(smem + kExpTableWords * 8);
  uint64_t* bar_empty = bar_full + kSlots;
  uint64_t* bar_load = bar_empty + kSlots;
  int* misc = (int*)(bar_load + 1);
  double* ring = (double*)(smem + kFixedBytes);
  stage_exp_table(exp_tab, tid, kRingThreads);

  for (int item = blockIdx.x; item < a.n_list; item += gridDim.x) {
    const int doc = a.list[item];
    const int n = a.D.n[doc], m = a.D.m[doc];
    const int s0 = a.D.src0[doc], t0 = a.D.tgt0[doc];
    const double p = a.p;
    const int ngroups = (m + 3) >> 2;
    const int nl = (n + R - 1) / R;
    const int slot_d = ring_slot_doubles(R, nl);
    uint8_t* var = smem + kFixedBytes + union_bytes(n, m, R);
    uint32_t* hits = (uint32_t*)var;
    SPack* sp = (SPack*)(var + hits_bytes(n, m));
    const uint16_t* hits16 = (const uint16_t*)hits;
    CodeT* dirs = (CodeT*)((uint8_t*)sp + (size_t)(n + m) * 16);
    int32_t* dlist = (int32_t*)((uint8_t*)dirs + align16((size_t)ngroups * WARP * sizeof(CodeT)));

    __syncthreads();  // the previous document is done with every buffer
    RING_PROF(0)
    if (tid == 0) {
      for (int q = 0; q < kSlots; ++q) {
        mbar_init(bar_full + q, BM_RING_WARP_ARRIVE ? kProdWarps : kProducers);
        mbar_init(bar_empty + q, 1);
      }
      mbar_init(bar_load, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#if !BM_RING_FUSED_JOIN
      const uint32_t bytes = (uint32_t)hits_bytes(n, m);
      mbar_arrive_expect_tx(bar_load, bytes);
      bulk_g2s(hits, a.hits + a.hit_off[doc], bytes, bar_load);
#endif
    }
#if BM_RING_FUSED_JOIN
    // the document's dictionary join: hit counts accumulate in shared memory
    // (the join's scratch lives in the ring's space, unused until scoring)
    uint8_t* uni = smem + kFixedBytes;
    JoinSmem js = carve_join(uni);
    int32_t* offS = (int32_t*)(uni + align16(join_smem_bytes()));
    int32_t* offT = offS + n + 1;
    uint16_t* chunk_owner = (uint16_t*)((uint8_t*)offS + align16((size_t)(n + m + 2) * 4));
    uint16_t* a_owner = chunk_owner + kJoinEmax;
    {
      const int nw = (int)(hits_bytes(n, m) / 4);
      for (int q = tid; q < nw; q += kRingThreads) hits[q] = 0u;
      for (int q = tid; q <= n + m + 1; q += kRingThreads) {
        if (q <= n)
          offS[q] = __ldg(S.tok_off + s0 + q);
        else
          offT[q - n - 1] = __ldg(S.tok_off + t0 + (q - n - 1));
      }
    }
    __syncthreads();
    tile_join_entries<true>(CtaGroup(), S, a.L, s0, n, t0, m, offS, offT, hits, js, chunk_owner,
                            a_owner, /*zero_hits=*/false);
#endif
    // sentences of the document (rows 0..n-1, then columns)
    for (int k = tid; k < n + m; k += kRingThreads) {
      const bool row = k < n;
      const int g = row ? s0 + k : t0 + (k - n);
      const SentScalars v = load_scalars(S, g);
      SPack q;
      q.tpad = (uint32_t)v.T | ((uint32_t)v.P << 8) | ((uint32_t)v.nA << 16) | ((uint32_t)v.nD << 24);
      q.dx = digit_word(S, v.nD, v.d0);
      q.pos = row ? doc_pos(k, n) : doc_pos(k - n, m);
      sp[k] = q;
    }
    __syncthreads();
#if !BM_RING_FUSED_JOIN
    mbar_wait(bar_load, 0);
#endif
    RING_PROF(1)

    const int steps = ngroups + nl - 1;

    if (warp == 0) {
      // ------------------------------------------------------------ DP warp
      // blocked wavefront (see nw_band_kernel): lane L owns rows RL..RL+R-1
      // and at super-step t computes the R x 4 block of column group t - L
      const int i0 = lane * R;
      const bool lane_on = lane < nl;
      double lf[R];
#pragma unroll
      for (int r = 0; r < R; ++r) lf[r] = (double)(i0 + r + 1) * p;
      double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
      double dgn = (double)i0 * p;
      const int cost_lane = (n - 1) / R;
      for (int t = 0; t < steps; ++t) {
        const int g = t - lane;
        double u[4];
        u[0] = __shfl_up_sync(kFull, b0, 1);
        u[1] = __shfl_up_sync(kFull, b1, 1);
        u[2] = __shfl_up_sync(kFull, b2, 1);
        u[3] = __shfl_up_sync(kFull, b3, 1);
        if (lane == 0) {  // row 0 border C[0][j] = j * p
          u[0] = (double)(4 * g + 1) * p;
          u[1] = (double)(4 * g + 2) * p;
          u[2] = (double)(4 * g + 3) * p;
          u[3] = (double)(4 * g + 4) * p;
          dgn = (double)(4 * g) * p;
        }
        mbar_wait_backoff(bar_full + (t % kSlots), (uint32_t)((t / kSlots) & 1));
        const bool act = lane_on && (unsigned)g < (unsigned)ngroups;
        if (act) {
          const double* om = ring + (size_t)(t % kSlots) * slot_d + lane * RL;
          double v[R][4];
          CodeT codes = 0;
#pragma unroll
          for (int dd = 0; dd < R + 3; ++dd) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int c = dd - r;
              if (c < 0 || c > 3) continue;
              const double dgv = r == 0 ? (c == 0 ? dgn : u[c - 1]) : (c == 0 ? lf[r - 1] : v[r - 1][c - 1]);
              const double upv = r == 0 ? u[c] : v[r - 1][c];
              const double lfv = c == 0 ? lf[r] : v[r][c - 1];
              uint32_t kc;
              nw_cell(dgv, upv, lfv, om[r * 4 + c], p, v[r][c], kc);
              codes |= (CodeT)kc << (2 * (c * R + r));
            }
          }
          dirs[g * WARP + lane] = codes;
          if (lane == cost_lane && g == ngroups - 1) {
            const int r = n - 1 - i0, c = m - 1 - 4 * g;
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
              for (int cc = 0; cc < 4; ++cc)
                if (rr == r && cc == c) a.cost[doc] = v[rr][cc];
          }
          dgn = u[3];
#pragma unroll
          for (int r = 0; r < R; ++r) lf[r] = v[r][3];
          b0 = v[R - 1][0];
          b1 = v[R - 1][1];
          b2 = v[R - 1][2];
          b3 = v[R - 1][3];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty + (t % kSlots));
      }
    } else {
      // ------------------------------------------------------ score warps
      // a task is 32 / R lane blocks of one super-step; a thread scores one row
      // of its R x 4 block (4 cells: the row's sentence and hit words loaded
      // once). The tasks of all super-steps form one sequence and producer
      // warp w takes every 4th (w, w + 4, ...), which balances the ragged
      // fill/drain super-steps. Rows past the matrix are skipped; a column
      // past m re-scores column m - 1 (never read by the DP).
      static_assert(kProdWarps == 4, "task striding assumes 4 producer warps");
      constexpr int CPT = BM_RING_CPT;              // cells per thread and task
      constexpr int TPB = R * (4 / CPT);            // threads per R x 4 lane block
      constexpr int TL = WARP / TPB;                // lane blocks per task
      const int pw = warp - 1;
      const int sub = lane / TPB, r = (lane % TPB) / (4 / CPT), c0 = (lane % (4 / CPT)) * CPT;
      const double w3z = __dmul_rn(a.M.w[3], 0.0);
      int q0 = 0;  // sequence index of super-step t's first task
      for (int t = 0; t < steps; ++t) {
        if (t >= kSlots) {
          if (BM_RING_SLEEP_NS > 0)
            mbar_wait_sleep(bar_empty + (t % kSlots), (uint32_t)(((t / kSlots) - 1) & 1), BM_RING_SLEEP_NS);
          else
            mbar_wait_backoff(bar_empty + (t % kSlots), (uint32_t)(((t / kSlots) - 1) & 1));
        }
        const int2 la = active_lanes(t, ngroups, nl);
        const int ntask = (la.y - la.x + TL) / TL;
        double* slot = ring + (size_t)(t % kSlots) * slot_d;
        for (int kt = (pw - q0) & 3; kt < ntask; kt += kProdWarps) {
          const int L = la.x + kt * TL + sub;
          const int i = L * R + r, j0 = 4 * (t - L) + c0;
          if (L <= la.y && i < n) {
            const SPack sa = ld_spack(sp + i);
            const uint16_t* hrow = hits16 + i * m;
            double o[CPT];
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
              const int j = min(j0 + c, m - 1);
              const uint32_t hv = hrow[j];
#ifdef BM_PROF_FAKE_SCORE  // timing experiment only: DP side lower bound
              o[c] = __dsub_rn(1.0, (double)(hv & 0xff) * 0.01 + sa.pos);
#else
              o[c] = bmexp::one_minus_confidence(
                  staged_margin(S, a.M, a.tabs, a.mt, sa, ld_spack(sp + n + j), hv & 0xff, hv >> 8),
                  exp_tab);
#endif
            }
            double* dst = slot + L * RL + r * 4 + c0;
            if (CPT == 1) {
              dst[0] = o[0];
            } else {
#pragma unroll
              for (int c = 0; c < CPT; c += 2)
                *reinterpret_cast<double2*>(dst + c) = make_double2(o[c], o[(c + 1) % CPT]);
            }
          }
        }
        q0 += ntask;
        if (BM_RING_WARP_ARRIVE) {
          __syncwarp();  // the warp's ring stores before lane 0's (release) arrival
          if (lane == 0) mbar_arrive(bar_full + (t % kSlots));
        } else {
          mbar_arrive(bar_full + (t % kSlots));
        }
      }
    }
    __syncthreads();  // DP complete: direction codes final
    RING_PROF(2)

    if (tid == 0) {
      // block walk: load an R x 4 block's code word once, then step in
      // registers (bit offset sh = 2 (c R + r) moves by a constant per move
      // kind) until the path leaves the block through its top or left edge
      int k = 0, ci = n - 1, cj = m - 1;
      while (ci >= 0 && cj >= 0) {
        const CodeT wv = dirs[(cj >> 2) * WARP + ci / R];
        int r = ci % R, c = cj & 3;
        int sh = 2 * (c * R + r);
        for (;;) {
          const uint32_t op = (uint32_t)(wv >> sh) & 3u;
          if (op == BM_MOVE_D) {
            dlist[k++] = (ci << 16) | cj;
            --ci;
            --cj;
            --r;
            --c;
            sh -= 2 * (R + 1);
            if ((r | c) < 0) break;
          } else if (op == BM_MOVE_GS) {
            --ci;
            --r;
            sh -= 2;
            if (r < 0) break;
          } else {
            --cj;
            --c;
            sh -= 2 * R;
            if (c < 0) break;
          }
        }
      }
      misc[0] = k;
    }
    __syncthreads();
    RING_PROF(3)
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
        const int cell = dlist[K_path - 1 - f];  // ci << 16 | cj
        ci = cell >> 16;
        cj = cell & 0xffff;
        const uint32_t hv = hits16[ci * m + cj];
        sv = staged_score(S, a.M, exp_tab, a.tabs, a.mt, ld_spack(sp + ci), ld_spack(sp + n + cj),
                          hv & 0xff, hv >> 8);
        keep = sv >= a.threshold;
      }
      const unsigned mask = __ballot_sync(kFull, keep);
      if (lane == 0) misc[4 + warp] = __popc(mask);
      __syncthreads();
      int before = 0, chunk = 0;
#pragma unroll
      for (int w = 0; w < kRingThreads / WARP; ++w) {
        const int cw = misc[4 + w];
        before += w < warp ? cw : 0;
        chunk += cw;
      }
      if (keep) {
        bm_record rec;
        rec.doc = doc;
        rec.i = ci;
        rec.j = cj;
        rec.pad = 0;
        rec.conf = sv;
        out[base + before + __popc(mask & ((1u << lane) - 1u))] = rec;
      }
      base += chunk;
      __syncthreads();  // misc reused by the next chunk
    }
    if (tid == 0) a.rec_count[doc] = base;
    RING_PROF(4)
  }
}

// Raise a kernel's dynamic shared memory limit (and prefer the shared-memory
// carveout) once per size: the attribute calls cost microseconds of host time
// per launch, and the host entry launches per chunk.
// The attribute belongs to the current device's context, so the cache is keyed
// by (device, function).
cudaError_t smem_attr(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> set[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  auto it = set[dev].find(fn);
  if (it != set[dev].end() && it->second >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  set[dev][fn] = smem;
  return cudaSuccess;
}

cudaError_t launch_hits(const FusedArgs& a, size_t smem, cudaStream_t st) {
  if (a.n_list == 0) return cudaSuccess;
  cudaError_t e = smem_attr((const void*)hits_kernel, smem);
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
#define BM_LAUNCH_RING(RR)                                  \
  e = smem_attr((const void*)mine_ring_kernel<RR>, smem);   \
  if (e != cudaSuccess) return e;                           \
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

#ifdef BM_RING_PROFILE
extern "C" int bm_ring_prof(unsigned long long* host, int n_items) {
  return (int)cudaMemcpyFromSymbol(host, g_ring_prof, sizeof(unsigned long long) * 6 * n_items);
}
#endif
}  // namespace bm
