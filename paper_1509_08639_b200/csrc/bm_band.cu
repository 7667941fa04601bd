// Fused banded tier: score -> NW DP for the 128-row bands of documents too
// large for the ring kernel (aligner.py:313-339 fused with :116-173).
//
// The unfused banded tier wrote the similarity matrix to HBM (score_hits_kernel,
// 8 B/cell) and read it back in the DP (nw_band_kernel): two kernels that each
// held the whole GPU in turn -- the scoring issue-bound, the DP latency-bound,
// never overlapping. Here one CTA runs one (document, band) item at a time:
//   warp 0       the blocked wavefront DP of nw_band_kernel (lane L owns rows
//                4L..4L+3 of the band and at super-step t computes the 4 x 4
//                block of column group t - L), reading 1 - S from a
//                shared-memory ring of kBandSlots super-steps; bottom rows go
//                to the band below through global memory exactly as in
//                nw_band_kernel (sentinel-valued boundary rows, same codes,
//                same cost), so extraction is unchanged;
//   warps 1..P   score the blocks each super-step needs: one thread scores
//                BM_BAND_CPT cells of one row of a 4 x 4 lane block (one hit
//                count load, the row's staged sentence once); the tasks of
//                all super-steps form one sequence dealt round-robin to the
//                scoring warps, so the wavefront's fill and drain leave few
//                threads idle. Full / empty mbarriers per slot.
// The hit counts come from the document-level join (hits_doc_kernel) in rows
// of pitch_of(m) words. The matrix never exists; extraction re-scores the
// path's diagonal cells (extract_kernel<true>). Documents with a sentence over
// 255 tokens (the folded tables' range) keep the unfused tier.
//
// Opt-in (BM_BAND_FUSED=1, bm_api.cu): parity-green but slower than the
// unfused tier on C3 (70.6 vs 68.5 ms for 200k documents). A CTA's progress is
// its one DP warp's: with 8 scoring warps per DP warp only ~3 DP warps run per
// SM (nw_band_kernel keeps ~12), so the scoring warps wait on their rings
// (profiles/r02g_c3_band_ncu_full_summary.txt).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "bm_kernels.cuh"

namespace bm {

// BM_BAND_CPT cells per scoring thread and super-step (4: one row of a 4 x 4
// block, 4 scoring warps; 2: half a row, 8 scoring warps -- more warps to hide
// the table lookups' latency, less ILP per thread)
#ifndef BM_BAND_CPT
#define BM_BAND_CPT 2
#endif
#ifndef BM_BAND_SLOTS
#define BM_BAND_SLOTS 4
#endif
// scoring warps per DP warp (a CTA runs one (doc, band) item)
#ifndef BM_BAND_PROD_WARPS
#define BM_BAND_PROD_WARPS (16 / BM_BAND_CPT)
#endif
#ifndef BM_BAND_MINB
#define BM_BAND_MINB \
  (BM_BAND_PROD_WARPS == 1 ? 8 : BM_BAND_PROD_WARPS == 2 ? 6 : BM_BAND_PROD_WARPS == 4 ? 5 : 3)
#endif
// scoring warps: one arrival per warp on the full barriers (fewer mbarrier
// events wake fewer sleeping waiters); empty-slot waits sleep up to
// BM_BAND_SLEEP_NS instead of retrying try_wait (0: try_wait loop)
#ifndef BM_BAND_WARP_ARRIVE
#define BM_BAND_WARP_ARRIVE 1
#endif
#ifndef BM_BAND_SLEEP_NS
#define BM_BAND_SLEEP_NS 256
#endif
constexpr int kBandCpt = BM_BAND_CPT;
static_assert(kBandCpt == 4 || kBandCpt == 2, "2 or 4 cells per thread");
constexpr int kBandProdWarps = BM_BAND_PROD_WARPS;
constexpr int kBandThreads = (1 + kBandProdWarps) * WARP;
constexpr int kBandSlots = BM_BAND_SLOTS;
constexpr int kBandLaneD = kBandR * 4 + 2;  // doubles per DP lane in a slot (+2: banks)
constexpr int kBandSlotD = WARP * kBandLaneD;
constexpr int kBandThrPerBlock = 16 / kBandCpt;      // threads per 4 x 4 lane block
constexpr int kBandTaskLanes = WARP / kBandThrPerBlock;  // lane blocks per 32-thread task

// One staged sentence (16 B): T | P << 8 | |A| << 16 | |D| << 24, the digit
// word (0: no digit token; id + 1: exactly one; kDigMany | dig_off: two or
// more), the document position.
struct __align__(16) BandSent {
  uint32_t tpad;
  uint32_t dx;
  double pos;
};

// Column window: the target sentences of column groups [t - 31 - kBandSlots,
// t + kBandAhead] are in use while producers score super-step t (a ring of
// kBandWinGroups groups, so shared memory does not grow with m). Group
// t + kBandAhead is staged by one producer warp during super-step t; since
// kBandAhead >= kBandSlots, every other producer warp reaches super-step
// t + kBandAhead only after the DP consumed super-step t + kBandAhead -
// kBandSlots >= t, i.e. after the staging warp arrived on that full barrier.
constexpr int kBandAhead = kBandSlots;
constexpr int kBandWinGroups = 64;
static_assert(kBandAhead >= kBandSlots, "staging must precede the other warps' use");
static_assert(WARP + 2 * kBandSlots + kBandAhead <= kBandWinGroups, "column window too small");
__host__ __device__ constexpr size_t band_fixed_smem() {
  return (size_t)kExpTableWords * 8 + 128 /* barriers, misc */ + WARP * 8 /* boundary chunk */ +
         (size_t)kBandSlots * kBandSlotD * 8 + (size_t)kBandRows * sizeof(BandSent) +
         (size_t)kBandWinGroups * 4 * sizeof(BandSent);
}
size_t band_smem_bytes(int) { return band_fixed_smem(); }

__device__ __forceinline__ BandSent band_sent(const bm_sentences& S, int g, double pos) {
  const SentScalars v = load_scalars(S, g);
  BandSent b;
  b.tpad = (uint32_t)v.T | ((uint32_t)v.P << 8) | ((uint32_t)v.nA << 16) | ((uint32_t)v.nD << 24);
  b.dx = digit_word(S, v.nD, v.d0);
  b.pos = pos;
  return b;
}

// 1 - S of one cell: folded_margin's additions in margin()'s order, then
// the glibc sigmoid (bit-identical to score_hits_kernel).
__device__ __forceinline__ double band_cost(const bm_sentences& S, const Model& M,
                                            const ModelTables& mt, double w3z, bmexp::SmemTab tab,
                                            uint32_t ta, uint32_t ax, double pos_s, uint32_t tb,
                                            uint32_t bx, double pos_t, uint32_t hv) {
  const uint32_t hf = hv & 0xffffu, hr = hv >> 16;
  double z = __ldg(mt.z1 + (((ta & 0xffu) << 8) | (tb & 0xffu)));
  z = __dadd_rn(z, __ldg(mt.p1 + ((hf << 8) | ((ta >> 16) & 0xffu))));
  z = __dadd_rn(z, __ldg(mt.p2 + ((hr << 8) | ((tb >> 16) & 0xffu))));
  z = __dadd_rn(z, digit_term_w(S, M, w3z, ax, bx, (int)(ta >> 24), (int)(tb >> 24)));
  z = __dadd_rn(z, __ldg(mt.p4 + ((ta & 0xff00u) | ((tb >> 8) & 0xffu))));
  z = __dadd_rn(z, __dmul_rn(M.w[5], __dsub_rn(1.0, fabs(__dsub_rn(pos_s, pos_t)))));
  z = __dadd_rn(z, M.w[6]);  // w6 * 1.0
  return bmexp::one_minus_confidence(z, tab);
}

template <bool kFin>
__global__ void __launch_bounds__(kBandThreads, BM_BAND_MINB) mine_band_kernel(BandArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* exp_tab = (uint64_t*)smem;
  uint64_t* bar_full = (uint64_t*)(smem + kExpTableWords * 8);
  uint64_t* bar_empty = bar_full + kBandSlots;
  int* misc = (int*)(bar_empty + kBandSlots);
  double* bnd_s = (double*)(smem + kExpTableWords * 8 + 128);
  double* ring = bnd_s + WARP;
  BandSent* rows = (BandSent*)(ring + kBandSlots * kBandSlotD);
  BandSent* cols = rows + kBandRows;
  stage_exp_table(exp_tab, tid, kBandThreads);
  const double p = a.p;
  const bm_sentences& S = a.S;

  for (;;) {
    __syncthreads();  // the previous item is done with every buffer
    if (tid == 0) {
      misc[0] = (int)atomicAdd(a.ticket, 1u);
      for (int q = 0; q < kBandSlots; ++q) {
        mbar_init(bar_full + q, BM_BAND_WARP_ARRIVE ? kBandProdWarps : kBandProdWarps * WARP);
        mbar_init(bar_empty + q, 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int it = misc[0];
    if (it >= a.n_items) return;
    const WorkItem w = a.items[it];
    const int d = w.doc, band = w.band;
    const int n = a.D.n[d], m = a.D.m[d];
    const int row0 = band * kBandRows;
    const int nrow = min(kBandRows, n - row0);
    const int nl = (nrow + kBandR - 1) / kBandR;
    const int nbands = (n + kBandRows - 1) / kBandRows;
    const int ngroups = (m + 3) >> 2;
    const int steps = ngroups + nl - 1;
    {
      const int s0 = a.D.src0[d] + row0, t0 = a.D.tgt0[d];
      // rows of the band, and the column window's first kBandAhead groups
      const int nc = min(m, 4 * kBandAhead);
      for (int k = tid; k < nrow + nc; k += kBandThreads) {
        if (k < nrow)
          rows[k] = band_sent(S, s0 + k, doc_pos(row0 + k, n));
        else
          cols[k - nrow] = band_sent(S, t0 + (k - nrow), doc_pos(k - nrow, m));
      }
    }
    __syncthreads();

    if (warp == 0) {
      // ------------------------------------------------------------ DP warp
      // nw_band_kernel<., 1, kFin>'s super-step with 1 - S from the ring
      uint32_t* dirs = a.dirs + a.dir_off[d] + (int64_t)band * ngroups * WARP + lane;
      const double* bnd_up = band > 0 ? a.bnd + a.bnd_off[d] + (int64_t)(band - 1) * m : nullptr;
      double* bnd_me = band < nbands - 1 ? a.bnd + a.bnd_off[d] + (int64_t)band * m : nullptr;
      const int i0 = row0 + lane * kBandR;
      const bool lane_on = lane < nl;
      const bool pub_lane = bnd_me != nullptr && lane == nl - 1;
      const int cost_lane = (band == nbands - 1) ? (n - 1 - row0) / kBandR : -1;
      const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + (uint32_t)(lane * kBandLaneD * 8);
      double l[4], b[4], dgn = (double)i0 * p;
      uint64_t pre = kBndSentinel;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        l[r] = (double)(i0 + r + 1) * p;
        b[r] = 0.0;
      }
#pragma unroll 1
      for (int t = 0; t < steps; ++t) {
        const int g = t - lane;
        if ((t & (kNwChunkG - 1)) == 0 && 4 * t < m) {
          // lane 0's next kNwChunkG groups of the row above (band 0: border)
          const int c = lane < 4 * kNwChunkG ? 4 * t + lane : m;
          double v = 0.0;
          if (c < m) {
            if (band == 0) {
              v = (double)(c + 1) * p;
            } else {
              uint64_t x = pre;
              while (x == kBndSentinel && (x = ld_relaxed_u64(bnd_up + c)) == kBndSentinel)
                __nanosleep(32);
              v = __longlong_as_double((long long)x);
            }
          }
          __syncwarp();
          bnd_s[lane] = v;
          __syncwarp();
        }
        if (band > 0 && (t & (kNwChunkG - 1)) == kNwChunkG / 2) {
          const int c = lane < 4 * kNwChunkG ? 4 * (t + kNwChunkG / 2) + lane : m;
          pre = c < m ? ld_relaxed_u64(bnd_up + c) : kBndSentinel;
        }
        double u[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) u[c] = __shfl_up_sync(kFull, b[c], 1);
        {
          const double2 x = *(const double2*)(bnd_s + 4 * (t & (kNwChunkG - 1)));
          const double2 y = *(const double2*)(bnd_s + 4 * (t & (kNwChunkG - 1)) + 2);
          if (lane == 0) {
            u[0] = x.x;
            u[1] = x.y;
            u[2] = y.x;
            u[3] = y.y;
          }
        }
        if (g == 0) {  // the lane's first block: the left border of its rows
#pragma unroll
          for (int r = 0; r < 4; ++r) l[r] = (double)(i0 + r + 1) * p;
          dgn = (double)i0 * p;
        }
        const int slot = t % kBandSlots;
        mbar_wait_backoff(bar_full + slot, (uint32_t)((t / kBandSlots) & 1));
        double om[16];
        {
          const uint32_t src = ring_s + (uint32_t)(slot * kBandSlotD * 8);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                         : "=d"(om[2 * q]), "=d"(om[2 * q + 1])
                         : "r"(src + 16u * q));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_empty + slot);
        double v[4][4], vp[4][4], upp[4], lfp[4];
        uint32_t codes = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          upp[k] = __dadd_rn(u[k], p);
          lfp[k] = __dadd_rn(l[k], p);
        }
#pragma unroll
        for (int dd = 0; dd < 7; ++dd) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int c = dd - r;
            if (c < 0 || c > 3) continue;
            const double dgv = r == 0 ? (c == 0 ? dgn : u[c - 1]) : (c == 0 ? l[r - 1] : v[r - 1][c - 1]);
            const double upv = r == 0 ? upp[c] : vp[r - 1][c];
            const double lfv = c == 0 ? lfp[r] : vp[r][c - 1];
            uint32_t kc;
            nw_cell2<kFin>(dgv, upv, lfv, om[4 * r + c], p, v[r][c], vp[r][c], kc);
            codes |= kc << (8 * c + 2 * r);
          }
        }
        const bool act = lane_on && (unsigned)g < (unsigned)ngroups;
        const int cmax = m - 4 * g;
        dgn = u[3];
#pragma unroll
        for (int r = 0; r < 4; ++r) l[r] = v[r][3];
#pragma unroll
        for (int c = 0; c < 4; ++c) b[c] = v[3][c];
        if (act) dirs[(int64_t)g * WARP] = codes;
        if (act && pub_lane) {
          double* dst = bnd_me + 4 * g;
          st_relaxed_f64(dst, b[0]);
          if (cmax > 1) st_relaxed_f64(dst + 1, b[1]);
          if (cmax > 2) st_relaxed_f64(dst + 2, b[2]);
          if (cmax > 3) st_relaxed_f64(dst + 3, b[3]);
        }
        if (act && lane == cost_lane && g == ngroups - 1) {
          const int r = n - 1 - i0;
          double row[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) row[c] = r == 0 ? v[0][c] : r == 1 ? v[1][c] : r == 2 ? v[2][c] : v[3][c];
          a.cost[d] = cmax == 1 ? row[0] : cmax == 2 ? row[1] : cmax == 3 ? row[2] : row[3];
        }
      }
    } else {
      // ------------------------------------------------------ score warps
      const int pw = warp - 1;
      const int sub = lane / kBandThrPerBlock, r = (lane % kBandThrPerBlock) / (4 / kBandCpt);
      const int c0 = (lane % (4 / kBandCpt)) * kBandCpt;  // first column of the thread in the block
      const uint32_t* hd = a.hits + a.h_off[d];
      const int64_t hp = a.pitch[d];
      const double w3z = __dmul_rn(a.M.w[3], 0.0);
      const uint32_t zz = (uint32_t)hp >> 31;  // 0, opaque to the compiler (keeps bases in registers)
      const bmexp::SmemTab tab{(uint32_t)__cvta_generic_to_shared(exp_tab) + zz};
      const uint32_t cols_s = (uint32_t)__cvta_generic_to_shared(cols) + zz;
      const uint32_t rows_s = (uint32_t)__cvta_generic_to_shared(rows) + zz;
      const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + zz;
      // this warp's tasks: every P-th of the sequence of all super-steps'
      // tasks; the next task's hit words are loaded before the current task
      // is scored
      struct Task {
        int t, kt, L, il, j0;
        bool on;
      };
      auto ntask_of = [&](int t) {
        const int lx = max(0, t - ngroups + 1), ly = min(nl - 1, t);
        return (ly - lx + kBandTaskLanes) / kBandTaskLanes;
      };
      // (t, kt) -> the first own task at or after it (t == steps: none)
      auto task_at = [&](int t, int kt) {
        while (t < steps) {
          const int nt = ntask_of(t);
          if (kt < nt) break;
          kt -= nt;
          ++t;
        }
        Task k;
        k.t = t;
        k.kt = kt;
        const int lx = max(0, t - ngroups + 1), ly = min(nl - 1, t);
        k.L = lx + kt * kBandTaskLanes + sub;
        k.il = k.L * kBandR + r;
        k.j0 = 4 * (t - k.L) + c0;
        k.on = t < steps && k.L <= ly && k.il < nrow;
        return k;
      };
      auto hits_of = [&](const Task& k) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (k.on) {
          const uint32_t* q = hd + (int64_t)(row0 + k.il) * hp + k.j0;
          if (kBandCpt == 4) {
            v = ld_stream_v4(q);
          } else {
            const uint2 w2 = ld_stream_v2(q);
            v.x = w2.x;
            v.y = w2.y;
          }
        }
        return v;
      };
      Task k = task_at(0, pw);
      uint4 hv = hits_of(k);
#pragma unroll 1
      for (int t = 0; t < steps; ++t) {
        const int slot = t % kBandSlots;
        if (t >= kBandSlots) {
          if (BM_BAND_SLEEP_NS > 0)
            mbar_wait_sleep(bar_empty + slot, (uint32_t)(((t / kBandSlots) - 1) & 1), BM_BAND_SLEEP_NS);
          else
            mbar_wait_backoff(bar_empty + slot, (uint32_t)(((t / kBandSlots) - 1) & 1));
        }
        if (pw == t % kBandProdWarps && lane < 4) {
          const int j = 4 * (t + kBandAhead) + lane;
          if (j < m)
            cols[j & (4 * kBandWinGroups - 1)] = band_sent(S, a.D.tgt0[d] + j, doc_pos(j, m));
        }
        __syncwarp();
#pragma unroll 1
        while (k.t == t) {
          const Task nk = task_at(k.t, k.kt + kBandProdWarps);
          const uint4 nh = hits_of(nk);
          const int L = k.L, il = k.il;
          if (k.on) {
            const int j0 = k.j0;
            uint32_t ta, ax;
            double pos_s;
            {
              const uint32_t ra = rows_s + (uint32_t)il * 16u;
              asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(ta), "=r"(ax) : "r"(ra));
              asm("ld.shared.f64 %0, [%1];" : "=d"(pos_s) : "r"(ra + 8u));
            }
            // the cells are independent chains: no branches between them
            // (a column past m re-scores column m - 1; the DP never reads it)
            double o[kBandCpt];
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int c = 0; c < kBandCpt; ++c) {
              uint32_t tb, bx;
              double pos_t;
              const uint32_t ca =
                  cols_s + (uint32_t)(min(j0 + c, m - 1) & (4 * kBandWinGroups - 1)) * 16u;
              asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(tb), "=r"(bx) : "r"(ca));
              asm("ld.shared.f64 %0, [%1];" : "=d"(pos_t) : "r"(ca + 8u));
              o[c] = band_cost(S, a.M, a.mt, w3z, tab, ta, ax, pos_s, tb, bx, pos_t, hw[c]);
            }
            const uint32_t dst =
                ring_s + (uint32_t)((slot * kBandSlotD + L * kBandLaneD + r * 4 + (j0 & 3)) * 8);
#pragma unroll
            for (int c = 0; c < kBandCpt; c += 2)
              asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(dst + 8u * c), "d"(o[c]),
                           "d"(o[c + 1])
                           : "memory");
          }
          k = nk;
          hv = nh;
        }
        if (BM_BAND_WARP_ARRIVE) {
          // the warp's ring stores are ordered before lane 0's (release)
          // arrival by the warp barrier
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_full + slot);
        } else {
          mbar_arrive(bar_full + slot);
        }
      }
    }
  }
}

cudaError_t launch_band(const BandArgs& a, int m_max, cudaStream_t st) {
  if (a.n_items == 0) return cudaSuccess;
  const size_t smem = band_smem_bytes(m_max);
  const bool fin = std::isfinite(a.p);
  const void* fn = fin ? (const void*)mine_band_kernel<true> : (const void*)mine_band_kernel<false>;
  cudaError_t e = smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBandThreads, smem);
  if (e != cudaSuccess) return e;
  const int grid = std::min(a.n_items, sms * std::max(per_sm, 1));
  if (fin)
    mine_band_kernel<true><<<grid, kBandThreads, smem, st>>>(a);
  else
    mine_band_kernel<false><<<grid, kBandThreads, smem, st>>>(a);
  return counted(cudaGetLastError());
}

}  // namespace bm
