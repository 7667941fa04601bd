// K2 for runs of single-band documents (n <= 128 rows): the blocked
// wavefront of nw_band_kernel over several documents laid end to end along
// the columns (aligner.py:116-173, one DP per document and penalty).
//
// A 100 x 100 document alone keeps a warp for 25 + 25 - 1 = 49 super-steps,
// of which each lane works 25 (the wavefront's fill and drain): 40 % of the
// lane-steps. Concatenated, lane L moves on to the next document's first
// column group as soon as it finishes the previous one, so the fill and drain
// are paid once per run. Nothing crosses a document border: at a document's
// first group every lane restarts from the left border of its rows, lane 0's
// row above is the top border, and codes, costs and S are addressed per
// document exactly as in nw_band_kernel (same code words, same order D > GS >
// GT), so tune_count_kernel / extraction read the results unchanged.
#include <cuda_runtime.h>
#include <stdint.h>

#include "bm_kernels.cuh"

namespace bm {

constexpr int kSeqMaxDocs = 32;  // documents per run (the per-warp table)

struct __align__(16) SeqDoc {
  int start;   // first column group of the document in the run
  int m;
  int n;
  int pitch;
  int64_t s_off;
  int64_t dir_off;
};

__host__ __device__ constexpr int nw_seq_smem(int D, int NP) {
  return D * kNwSlotBytes + NP * WARP * 8 + kSeqMaxDocs * (int)sizeof(SeqDoc);
}

template <int D, int NP, bool kFin>
__global__ void __launch_bounds__(WARP, 1) nw_seq_kernel(NwArgs a) {
  static_assert((D & (D - 1)) == 0, "ring depth must be a power of two");
  extern __shared__ __align__(16) double nw_ring[];
  const int lane = threadIdx.x;
  double* bnd_s = nw_ring + D * WARP * kNwLane;  // NP x 32-column top-border chunks
  SeqDoc* tab = (SeqDoc*)(bnd_s + NP * WARP);
  const double* ring_l = nw_ring + (size_t)lane * kNwLane;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring_l);
  double pq[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) pq[q] = NP == 1 ? a.p : a.pv[q];
  for (;;) {
    int it = 0;
    if (lane == 0) it = (int)atomicAdd(a.ticket, 1u);
    it = __shfl_sync(kFull, it, 0);
    if (it >= a.n_seq) return;
    const int d0 = a.seq_off[2 * it], nd = a.seq_off[2 * it + 1] - d0;
    // the run's table: per document its first group, shape and offsets
    int tg = 0, nlmax = 0;
    {
      int gl = 0, nlv = 0;
      if (lane < nd) {
        const int d = d0 + lane;
        gl = (a.m[d] + 3) >> 2;
        nlv = (a.n[d] + kBandR - 1) / kBandR;
      }
      int incl = gl;
#pragma unroll
      for (int o = 1; o < WARP; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane < nd) {
        const int d = d0 + lane;
        SeqDoc e;
        e.start = incl - gl;
        e.m = a.m[d];
        e.n = a.n[d];
        e.pitch = a.pitch[d];
        e.s_off = a.s_off[d];
        e.dir_off = a.dir_off[d];
        tab[lane] = e;
      }
      tg = __shfl_sync(kFull, incl, WARP - 1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nlv = max(nlv, __shfl_xor_sync(kFull, nlv, o));
      nlmax = nlv;
    }
    __syncwarp();
    const int i0 = lane * kBandR;
    // prefetch cursor: the document of group pg (groups issued in order)
    int pd = 0, pend = (tab[0].m + 3) >> 2;
    const double* src[4];
    auto set_src = [&](int k) {
      const SeqDoc& e = tab[k];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        src[r] = a.S + e.s_off + (int64_t)min(i0 + r, e.n - 1) * e.pitch - 4 * (int64_t)e.start;
    };
    set_src(0);
    // one commit per call on every lane (nw_band_kernel's accounting); a group
    // outside [0, tg) copies the first document's row starts
    auto issue = [&](int gi) {
      const bool ok = (unsigned)gi < (unsigned)tg;
      if (ok) {
        while (gi >= pend) {
          ++pd;
          pend = tab[pd].start + ((tab[pd].m + 3) >> 2);
          set_src(pd);
        }
      }
      const int c = ok ? gi * 4 : 4 * tab[pd].start;
      const uint32_t dst = ring_s + (uint32_t)((gi & (D - 1)) * kNwSlotBytes);
      cp_async16_s(dst + 0, src[0] + c);
      cp_async16_s(dst + 16, src[0] + c + 2);
      cp_async16_s(dst + 32, src[1] + c);
      cp_async16_s(dst + 48, src[1] + c + 2);
      cp_async16_s(dst + 64, src[2] + c);
      cp_async16_s(dst + 80, src[2] + c + 2);
      cp_async16_s(dst + 96, src[3] + c);
      cp_async16_s(dst + 112, src[3] + c + 2);
      cp_async_commit();
    };
    auto load = [&](int gi, double(&o)[16]) {
      const double* cur = ring_l + (size_t)(gi & (D - 1)) * (WARP * kNwLane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 s = *(const double2*)(cur + 2 * q);
        o[2 * q] = __dsub_rn(1.0, s.x);
        o[2 * q + 1] = __dsub_rn(1.0, s.y);
      }
    };
#pragma unroll 1
    for (int q = 0; q < D; ++q) issue(q - lane);
    cp_async_wait_depth<D>();
    double oA[16], oB[16];
    load(-lane, oA);

    // compute cursor: the document of group t - lane
    int cd = 0, cstart = 0, cend = (tab[0].m + 3) >> 2;
    double l[NP][4], b[NP][4], dgn[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        l[q][r] = (double)(i0 + r + 1) * pq[q];
        b[q][r] = 0.0;
      }
      dgn[q] = (double)i0 * pq[q];
    }

    auto step = [&](const int t, double(&oc)[16], double(&on)[16]) {
      const int gg = t - lane;
      if ((unsigned)gg < (unsigned)tg) {
        while (gg >= cend) {
          ++cd;
          cstart = cend;
          cend = cstart + ((tab[cd].m + 3) >> 2);
        }
      }
      if ((t & (kNwChunkG - 1)) == 0 && t < tg) {
        // lane 0's next kNwChunkG groups: the top border C[0][j] = j * p of
        // whichever document each group belongs to (from lane 0's cursor)
        int k = __shfl_sync(kFull, cd, 0);
        const int e = lane < 4 * kNwChunkG ? lane : 0;
        const int grp = t + (e >> 2);
        int kend = tab[k].start + ((tab[k].m + 3) >> 2);
        while (grp >= kend && k + 1 < nd) {
          ++k;
          kend = tab[k].start + ((tab[k].m + 3) >> 2);
        }
        const int c = 4 * (grp - tab[k].start) + (e & 3);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NP; ++q) bnd_s[q * WARP + lane] = (double)(c + 1) * pq[q];
        __syncwarp();
      }
      const int g = gg - cstart;  // the lane's group within its document
      double u[NP][4];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
#pragma unroll
        for (int c = 0; c < 4; ++c) u[q][c] = __shfl_up_sync(kFull, b[q][c], 1);
        const double2 x = *(const double2*)(bnd_s + q * WARP + 4 * (t & (kNwChunkG - 1)));
        const double2 y = *(const double2*)(bnd_s + q * WARP + 4 * (t & (kNwChunkG - 1)) + 2);
        if (lane == 0) {
          u[q][0] = x.x;
          u[q][1] = x.y;
          u[q][2] = y.x;
          u[q][3] = y.y;
        }
        if (g == 0) {  // a document's first block: the left border of its rows
#pragma unroll
          for (int r = 0; r < 4; ++r) l[q][r] = (double)(i0 + r + 1) * pq[q];
          dgn[q] = (double)i0 * pq[q];
        }
      }
      issue(gg + D);
      cp_async_wait_depth<D>();  // block gg+1 has landed
      load(gg + 1, on);

      double v[NP][4][4], vp[NP][4][4], upp[NP][4], lfp[NP][4];
      uint32_t codes[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        codes[q] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          upp[q][k] = __dadd_rn(u[q][k], pq[q]);
          lfp[q][k] = __dadd_rn(l[q][k], pq[q]);
        }
      }
#pragma unroll
      for (int dd = 0; dd < 7; ++dd) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int c = dd - r;
          if (c < 0 || c > 3) continue;
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            const double dgv = r == 0 ? (c == 0 ? dgn[q] : u[q][c - 1])
                                      : (c == 0 ? l[q][r - 1] : v[q][r - 1][c - 1]);
            const double upv = r == 0 ? upp[q][c] : vp[q][r - 1][c];
            const double lfv = c == 0 ? lfp[q][r] : vp[q][r][c - 1];
            uint32_t kc;
            nw_cell2<kFin>(dgv, upv, lfv, oc[4 * r + c], pq[q], v[q][r][c], vp[q][r][c], kc);
            codes[q] |= kc << (8 * c + 2 * r);
          }
        }
      }
      const SeqDoc& e = tab[cd];
      const bool act = (unsigned)gg < (unsigned)tg && lane < (e.n + kBandR - 1) / kBandR;
      const int ngroups = (e.m + 3) >> 2;
      const int cmax = e.m - 4 * g;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        dgn[q] = u[q][3];
#pragma unroll
        for (int r = 0; r < 4; ++r) l[q][r] = v[q][r][3];
#pragma unroll
        for (int c = 0; c < 4; ++c) b[q][c] = v[q][3][c];
        if (act) a.dirs[q * a.dir_stride + e.dir_off + (int64_t)g * WARP + lane] = codes[q];
        if (act && lane == (e.n - 1) / kBandR && g == ngroups - 1) {
          const int r = e.n - 1 - i0;
          double row[4];
#pragma unroll
          for (int c = 0; c < 4; ++c)
            row[c] = r == 0 ? v[q][0][c] : r == 1 ? v[q][1][c] : r == 2 ? v[q][2][c] : v[q][3][c];
          a.cost[q * a.cost_stride + d0 + cd] =
              cmax == 1 ? row[0] : cmax == 2 ? row[1] : cmax == 3 ? row[2] : row[3];
        }
      }
    };
    const int steps = tg + nlmax - 1;
#pragma unroll 1
    for (int t = 0; t < steps; t += 2) {
      step(t, oA, oB);
      step(t + 1, oB, oA);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
  }
}

template <int NP, bool kFin>
cudaError_t launch_seq_np(const NwArgs& a, cudaStream_t st) {
  constexpr int D = 2;
  const int smem = nw_seq_smem(D, NP);
  cudaError_t e = cudaFuncSetAttribute(nw_seq_kernel<D, NP, kFin>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaFuncSetAttribute(nw_seq_kernel<D, NP, kFin>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nw_seq_kernel<D, NP, kFin>, WARP, smem);
  if (e != cudaSuccess) return e;
  nw_seq_kernel<D, NP, kFin><<<std::min(a.n_seq, sms * std::max(per_sm, 1)), WARP, smem, st>>>(a);
  return counted(cudaGetLastError());
}

template <int NP>
cudaError_t launch_seq_fin(const NwArgs& a, cudaStream_t st) {
  bool fin = true;
  for (int q = 0; q < NP; ++q) fin &= std::isfinite(NP == 1 ? a.p : a.pv[q]);
  return fin ? launch_seq_np<NP, true>(a, st) : launch_seq_np<NP, false>(a, st);
}

cudaError_t launch_nw_seq(const NwArgs& a, cudaStream_t st) {
  if (a.n_seq == 0) return cudaSuccess;
  switch (a.np) {
    case 1: return launch_seq_fin<1>(a, st);
    case 2: return launch_seq_fin<2>(a, st);
    case 4: return launch_seq_fin<4>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bm
