// Device building blocks shared by the kernels: per-cell features and score
// (bimine/classifier.py:54-117, aligner.py:332-338) and the dictionary join
// that turns token ids into per-cell coverage hit counts (lexicon.py:88-105).
//
// Arithmetic order is the reference's, operation by operation:
//   features are int/int true divisions (correctly rounded == __ddiv_rn),
//   z = bias; z += w_k * f_k  (separately rounded multiply and add, no FMA),
//   S = clamp(sigmoid(z)) with the glibc exp replica.
#pragma once
#include <stdint.h>

#include "bimine_b200.h"
#include "glibc_exp.cuh"

namespace bm {

constexpr int WARP = 32;
constexpr int kExpTableWords = 256;

struct Model {
  double w[7];
  double bias;
};

// Correctly rounded quotients k/d for 0 <= k <= d <= kQuotMax (Python's
// int/int true division of small counts), filled once by the host. The five
// count ratios of a cell are table loads instead of IEEE divisions; a zero
// numerator never reaches a division (its slow path is a called subroutine).
constexpr int kQuotMax = 64;
constexpr int kQuotStride = kQuotMax + 1;
constexpr int kQuotEntries = kQuotStride * kQuotStride;  // [den][num]
static __device__ double g_quot[kQuotEntries];  // filled by ensure_quot_table()

// Branch-free feature tables for counts < kPairMax, indexed by the two counts
// as they occur (global memory, filled once per device by ensure_quot_table()
// with host IEEE division; read through L1):
//   ratio2[a * kPairMax + b] = min(a,b)/max(a,b), 1.0 for a = b = 0 (classifier.py:62-65)
//   frac2[k * kPairMax + d]  = k/d, 0.0 for d = 0              (lexicon.py:96-105)
constexpr int kPairMax = 256;
struct PairTables {
  const double* ratio2;
  const double* frac2;
};

// Per-model tables of the margin's table-driven terms with the weights already
// applied by the same roundings margin() performs (bm_kernels.cu
// model_tables): z1 = bias + w0*ratio(aT, bT), p1 = w1*frac(h, A),
// p2 = w2*frac(h, A), p4 = w4*ratio(aP, bP); kPairMax x kPairMax each.
struct ModelTables {
  const double* z1;
  const double* p1;
  const double* p2;
  const double* p4;
};

__device__ __forceinline__ double quot(int num, int den) {  // 0 < num <= den
  if (den <= kQuotMax) return __ldg(&g_quot[den * kQuotStride + num]);
  return __ddiv_rn((double)num, (double)den);
}

// min(a,b)/max(a,b), 1.0 when both are zero (classifier.py:62-65).
__device__ __forceinline__ double ratio_min_max(int a, int b);
__device__ __forceinline__ double frac_or_zero(int num, int den);


__device__ __forceinline__ double ratio_min_max(int a, int b) {
  int lo = a < b ? a : b;
  int hi = a < b ? b : a;
  if (hi == 0) return 1.0;
  if (lo == 0) return 0.0;
  return quot(lo, hi);
}

// Python int/int true division; 0.0 for an empty denominator (lexicon.py:96-97).
__device__ __forceinline__ double frac_or_zero(int num, int den) {
  if (den == 0 || num == 0) return 0.0;
  return quot(num, den);
}

// |D_s & D_t| for two ascending id lists (classifier.py:82-87).
__device__ __forceinline__ int sorted_intersection(const int32_t* a, int na, const int32_t* b,
                                                   int nb) {
  int i = 0, j = 0, k = 0;
  while (i < na && j < nb) {
    int x = __ldg(a + i), y = __ldg(b + j);
    k += (x == y);
    i += (x <= y);
    j += (y <= x);
  }
  return k;
}

// Per-sentence scalars the score needs (loaded once per row / column).
struct SentScalars {
  int T, P, nA, nD, d0;
};

__device__ __forceinline__ SentScalars load_scalars(const bm_sentences& S, int g) {
  SentScalars r;
  r.T = __ldg(S.n_tok + g);
  r.P = __ldg(S.n_punct + g);
  r.nA = __ldg(S.n_alpha + g);
  r.d0 = __ldg(S.dig_off + g);
  r.nD = __ldg(S.dig_off + g + 1) - r.d0;
  return r;
}

// Feature vector of one cell (classifier.py:68-97). hf/hr: coverage hit counts.
__device__ __forceinline__ void cell_features(const bm_sentences& S, const SentScalars& a,
                                              const SentScalars& b, int hf, int hr,
                                              double pos_s, double pos_t, double f[7]) {
  f[0] = ratio_min_max(a.T, b.T);
  f[1] = frac_or_zero(hf, a.nA);
  f[2] = frac_or_zero(hr, b.nA);
  if (a.nD == 0 && b.nD == 0) {
    f[3] = 1.0;
  } else {
    int inter = (a.nD && b.nD) ? sorted_intersection(S.dig_id + a.d0, a.nD, S.dig_id + b.d0, b.nD)
                               : 0;
    f[3] = frac_or_zero(inter, a.nD + b.nD - inter);
  }
  f[4] = ratio_min_max(a.P, b.P);
  f[5] = __dsub_rn(1.0, fabs(__dsub_rn(pos_s, pos_t)));
  f[6] = 1.0;
}

// z = bias; z += w_k * f_k (classifier.py:114-116), each op separately rounded.
__device__ __forceinline__ double margin(const Model& M, const double f[7]) {
  double z = M.bias;
#pragma unroll
  for (int k = 0; k < 7; ++k) z = __dadd_rn(z, __dmul_rn(M.w[k], f[k]));
  return z;
}

__device__ __forceinline__ double cell_score(const bm_sentences& S, const Model& M,
                                             const uint64_t* exp_tab, const SentScalars& a,
                                             const SentScalars& b, int hf, int hr, double pos_s,
                                             double pos_t) {
  double f[7];
  cell_features(S, a, b, hf, hr, pos_s, pos_t, f);
  return bmexp::confidence_from_z(margin(M, f), exp_tab);
}

// i / max(1, n-1): document position of a sentence (aligner.py:332-333).
__device__ __forceinline__ double doc_pos(int i, int n) {
  return __ddiv_rn((double)i, (double)(n > 1 ? n - 1 : 1));
}

// ---------------------------------------------------------------------------
// Dictionary join. For a tile of source sentences [s0, s0+ns) x target
// sentences [t0, t0+nt) it accumulates, per cell,
//   hf(s,t) = sum over alpha entries a of s (with multiplicity) of
//             [ FWD[a] intersects U_t ]                 (coverage src->tgt)
//   hr(s,t) = same with the target's alpha entries, REV and U_s.
// One side's U entries are bucketed by id (a counting sort into a chained hash
// table in shared memory, chunked so any sentence length fits), the other
// side's candidates probe it. Counts are added with shared-memory atomics into
// packed counters: hits are order independent, so the result is deterministic.
// ---------------------------------------------------------------------------

struct JoinSmem {
  int32_t* key;      // [emax] bucketed token ids
  uint16_t* owner;   // [emax] local sentence index of each bucketed id
  int32_t* bstart;   // [nbuckets + 1]
  int32_t* bfill;    // [nbuckets]
  int emax;
  int nbuckets;      // power of two
  int bshift;        // 32 - log2(nbuckets)
};

__device__ __forceinline__ uint32_t bucket_of(int32_t id, int bshift) {
  return ((uint32_t)id * 0x9E3779B1u) >> bshift;
}

// Thread groups: whole CTA or a single warp.
struct CtaGroup {
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
  __device__ bool scanner() const { return threadIdx.x < WARP; }
};
struct WarpGroup {
  __device__ int rank() const { return threadIdx.x & (WARP - 1); }
  __device__ int size() const { return WARP; }
  __device__ void sync() const { __syncwarp(); }
  __device__ bool scanner() const { return true; }
};

// Is id present in the ascending list [p, p+n)?
__device__ __forceinline__ bool sorted_contains(const int32_t* p, int n, int32_t id) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int v = __ldg(p + mid);
    if (v < id)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n && __ldg(p + lo) == id;
}

// One direction of the join: index side B (sentences [b0, b0+nb_sent)), probe
// with the alpha entries of side A (sentences [a0, a0+na_sent)) through the
// lexicon CSR (off, cand). add(la, lb, w) accumulates hits for local indices.
template <class G, class AddFn>
__device__ void join_direction(G g, const bm_sentences& S, const int32_t* off,
                               const int32_t* cand, int a0, int na_sent, int b0, int nb_sent,
                               JoinSmem& js, AddFn add) {
  const int e_begin = __ldg(S.tok_off + b0);
  const int e_end = __ldg(S.tok_off + b0 + nb_sent);
  for (int c0 = e_begin; c0 < e_end; c0 += js.emax) {
    const int c1 = min(e_end, c0 + js.emax);
    // 1. bucket counts
    for (int b = g.rank(); b < js.nbuckets; b += g.size()) js.bfill[b] = 0;
    g.sync();
    for (int k = g.rank(); k < nb_sent; k += g.size()) {
      int e0 = max(c0, __ldg(S.tok_off + b0 + k));
      int e1 = min(c1, __ldg(S.tok_off + b0 + k + 1));
      for (int e = e0; e < e1; ++e) atomicAdd(&js.bfill[bucket_of(__ldg(S.tok_id + e), js.bshift)], 1);
    }
    g.sync();
    if (g.scanner()) {
      // counts live in bfill; scan into bstart and reset bfill to the starts
      int lane = threadIdx.x & (WARP - 1);
      int per = (js.nbuckets + WARP - 1) / WARP;
      int q0 = lane * per, q1 = min(js.nbuckets, q0 + per);
      int sum = 0;
      for (int b = q0; b < q1; ++b) sum += js.bfill[b];
      int incl = sum;
#pragma unroll
      for (int o = 1; o < WARP; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int run = incl - sum;
      for (int b = q0; b < q1; ++b) {
        int c = js.bfill[b];
        js.bstart[b] = run;
        js.bfill[b] = run;
        run += c;
      }
      if (lane == WARP - 1) js.bstart[js.nbuckets] = incl;
    }
    g.sync();
    // 2. scatter ids into buckets
    for (int k = g.rank(); k < nb_sent; k += g.size()) {
      int e0 = max(c0, __ldg(S.tok_off + b0 + k));
      int e1 = min(c1, __ldg(S.tok_off + b0 + k + 1));
      for (int e = e0; e < e1; ++e) {
        int32_t id = __ldg(S.tok_id + e);
        int slot = atomicAdd(&js.bfill[bucket_of(id, js.bshift)], 1);
        js.key[slot] = id;
        js.owner[slot] = (uint16_t)k;
      }
    }
    g.sync();
    // 3. probe with side A's alpha entries
    for (int k = g.rank(); k < na_sent; k += g.size()) {
      const int e0 = __ldg(S.tok_off + a0 + k);
      const int e1 = __ldg(S.tok_off + a0 + k + 1);
      for (int e = e0; e < e1; ++e) {
        const int w = __ldg(S.tok_alpha + e);
        if (w == 0) continue;
        const int32_t id = __ldg(S.tok_id + e);
        const int q0 = __ldg(off + id), q1 = __ldg(off + id + 1);
        for (int q = q0; q < q1; ++q) {
          const int32_t c = __ldg(cand + q);
          const uint32_t bk = bucket_of(c, js.bshift);
          for (int slot = js.bstart[bk]; slot < js.bstart[bk + 1]; ++slot) {
            if (js.key[slot] != c) continue;
            const int lb = js.owner[slot];
            // an entry hits a sentence once however many candidates it holds:
            // skip if an earlier candidate of this entry is also in U_lb
            bool dup = false;
            if (q > q0) {
              const int u0 = __ldg(S.tok_off + b0 + lb);
              const int un = __ldg(S.tok_off + b0 + lb + 1) - u0;
              for (int qq = q0; qq < q && !dup; ++qq) dup = sorted_contains(S.tok_id + u0, un, __ldg(cand + qq));
            }
            if (!dup) add(k, lb, w);
          }
        }
      }
    }
    g.sync();
  }
}

// Entry-parallel form of join_direction: every loop runs over token entries
// (coalesced loads, all lanes busy) instead of over sentences. offA / offB are
// the two sides' tok_off slices staged in shared memory (na+1 / nb+1 ints).
// First sentence k of [0, ns) whose entries reach past e (off[k+1] > e).
__device__ __forceinline__ int first_sentence_after(const int32_t* off, int ns, int e) {
  int lo = 0, hi = ns;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (off[mid + 1] <= e)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// One chunk [c0, c1) of side B's entries: bucket it, then probe with every
// alpha entry of side A (in chunks with an owner table). offA / offB: the
// sides' tok_off slices (shared or global memory), na / nb sentences.
template <class G, class AddFn>
__device__ void join_chunk_entries(G g, const bm_sentences& S, const int32_t* off,
                                   const int32_t* cand, const int32_t* offA, int na,
                                   const int32_t* offB, int b0, int nb, int c0, int c1,
                                   JoinSmem& js, uint16_t* chunk_owner, uint16_t* a_owner,
                                   AddFn add) {
  const int eA0 = offA[0], eA1 = offA[na];
  for (int b = g.rank(); b < js.nbuckets; b += g.size()) js.bfill[b] = 0;
  g.sync();
  // the bucket passes load kFill ids per thread before using any of them,
  // so the global-load latencies overlap (ids are >= 0; -1 marks no entry)
  constexpr int kFill = 4;
  for (int eb = c0 + g.rank(); eb < c1; eb += kFill * g.size()) {
    int idv[kFill];
#pragma unroll
    for (int u = 0; u < kFill; ++u) {
      const int e = eb + u * g.size();
      idv[u] = e < c1 ? __ldg(S.tok_id + e) : -1;
    }
#pragma unroll
    for (int u = 0; u < kFill; ++u)
      if (idv[u] >= 0) atomicAdd(&js.bfill[bucket_of(idv[u], js.bshift)], 1);
  }
  // owner sentence of every entry of the chunk (stores only)
  {
    const int kb0 = first_sentence_after(offB, nb, c0);
    for (int k = kb0 + g.rank(); k < nb; k += g.size()) {
      const int bk = offB[k];
      if (bk >= c1) break;
      const int e0 = max(c0, bk), e1 = min(c1, offB[k + 1]);
      for (int e = e0; e < e1; ++e) chunk_owner[e - c0] = (uint16_t)k;
    }
  }
  g.sync();
  if (g.scanner()) {
    int lane = threadIdx.x & (WARP - 1);
    int per = (js.nbuckets + WARP - 1) / WARP;
    int q0 = lane * per, q1 = min(js.nbuckets, q0 + per);
    int sum = 0;
    for (int b = q0; b < q1; ++b) sum += js.bfill[b];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < WARP; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - sum;
    for (int b = q0; b < q1; ++b) {
      int c = js.bfill[b];
      js.bstart[b] = run;
      js.bfill[b] = run;
      run += c;
    }
    if (lane == WARP - 1) js.bstart[js.nbuckets] = incl;
  }
  g.sync();
  for (int eb = c0 + g.rank(); eb < c1; eb += kFill * g.size()) {
    int idv[kFill];
#pragma unroll
    for (int u = 0; u < kFill; ++u) {
      const int e = eb + u * g.size();
      idv[u] = e < c1 ? __ldg(S.tok_id + e) : -1;
    }
#pragma unroll
    for (int u = 0; u < kFill; ++u) {
      if (idv[u] < 0) continue;
      const int slot = atomicAdd(&js.bfill[bucket_of(idv[u], js.bshift)], 1);
      js.key[slot] = idv[u];
      js.owner[slot] = chunk_owner[eb + u * g.size() - c0];
    }
  }
  g.sync();
  // probe side in chunks of emax entries, each with an owner table (a
  // per-entry binary search over the offsets cost more than the probes)
  for (int a0 = eA0; a0 < eA1; a0 += js.emax) {
    const int a1 = min(eA1, a0 + js.emax);
    {
      const int ka0 = first_sentence_after(offA, na, a0);
      for (int k = ka0 + g.rank(); k < na; k += g.size()) {
        const int ak = offA[k];
        if (ak >= a1) break;
        const int e0 = max(a0, ak), e1 = min(a1, offA[k + 1]);
        for (int e = e0; e < e1; ++e) a_owner[e - a0] = (uint16_t)k;
      }
    }
    g.sync();
    // kBatch entries per thread at a time: each level of the dependent
    // lookups (entry -> lexicon offsets -> first candidate) is issued for
    // all of them before any is used, so their latencies overlap
#ifndef BM_HITS_BATCH
#define BM_HITS_BATCH 4
#endif
    constexpr int kBatch = BM_HITS_BATCH;
    for (int eb = a0 + g.rank(); eb < a1; eb += kBatch * g.size()) {
      int wv[kBatch], idv[kBatch], q0v[kBatch], q1v[kBatch], lav[kBatch], c0v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int e = eb + u * g.size();
        const bool ok = e < a1;
        wv[u] = ok ? __ldg(S.tok_alpha + e) : 0;
        idv[u] = ok ? __ldg(S.tok_id + e) : 0;
        lav[u] = ok ? a_owner[e - a0] : 0;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        q0v[u] = wv[u] ? __ldg(off + idv[u]) : 0;
        q1v[u] = wv[u] ? __ldg(off + idv[u] + 1) : 0;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) c0v[u] = q0v[u] < q1v[u] ? __ldg(cand + q0v[u]) : 0;
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int w = wv[u], la = lav[u], q0 = q0v[u], q1 = q1v[u];
        for (int q = q0; q < q1; ++q) {
          const int32_t c = q == q0 ? c0v[u] : __ldg(cand + q);
          const uint32_t bk = bucket_of(c, js.bshift);
          const int s1 = js.bstart[bk + 1];
          for (int slot = js.bstart[bk]; slot < s1; ++slot) {
            if (js.key[slot] != c) continue;
            const int lb = js.owner[slot];
            // an entry hits a sentence once however many candidates it holds
            bool dup = false;
            if (q > q0) {
              const int u0 = __ldg(S.tok_off + b0 + lb);
              const int un = __ldg(S.tok_off + b0 + lb + 1) - u0;
              for (int qq = q0; qq < q && !dup; ++qq) dup = sorted_contains(S.tok_id + u0, un, __ldg(cand + qq));
            }
            if (!dup) add(la, lb, w);
          }
        }
      }
    }
    g.sync();
  }
}

template <class G, class AddFn>
__device__ void join_direction_entries(G g, const bm_sentences& S, const int32_t* off,
                                       const int32_t* cand, const int32_t* offA, int na,
                                       const int32_t* offB, int b0, int nb, JoinSmem& js,
                                       uint16_t* chunk_owner, uint16_t* a_owner, AddFn add) {
  const int eB0 = offB[0], eB1 = offB[nb];
  for (int c0 = eB0; c0 < eB1; c0 += js.emax)
    join_chunk_entries(g, S, off, cand, offA, na, offB, b0, nb, c0, min(eB1, c0 + js.emax), js,
                       chunk_owner, a_owner, add);
}

// Entry-parallel full join; offS / offT: staged tok_off slices (ns+1 / nt+1).
template <bool kPacked16, class G>
__device__ void tile_join_entries(G g, const bm_sentences& S, const bm_lexicon& L, int s0,
                                  int ns, int t0, int nt, const int32_t* offS,
                                  const int32_t* offT, uint32_t* hits, JoinSmem& js,
                                  uint16_t* chunk_owner, uint16_t* a_owner, bool zero_hits = true) {
  const int ncell = ns * nt;
  const int nwords = kPacked16 ? (ncell + 1) / 2 : 2 * ncell;
  if (zero_hits) {
    for (int k = g.rank(); k < nwords; k += g.size()) hits[k] = 0u;
    g.sync();
  }
  join_direction_entries(g, S, L.fwd_off, L.fwd_cand, offS, ns, offT, t0, nt, js, chunk_owner,
                         a_owner, [&](int ls, int lt, int w) {
                           int cell = ls * nt + lt;
                           if (kPacked16)
                             atomicAdd(&hits[cell >> 1], (uint32_t)w << ((cell & 1) * 16));
                           else
                             atomicAdd(&hits[cell], (uint32_t)w);
                         });
  join_direction_entries(g, S, L.rev_off, L.rev_cand, offT, nt, offS, s0, ns, js, chunk_owner,
                         a_owner, [&](int lt, int ls, int w) {
                           int cell = ls * nt + lt;
                           if (kPacked16)
                             atomicAdd(&hits[cell >> 1], (uint32_t)w << ((cell & 1) * 16 + 8));
                           else
                             atomicAdd(&hits[ncell + cell], (uint32_t)w);
                         });
}

// Full join for a tile. Hits are packed per cell into `hits` words:
//   kPacked16: 16-bit cells, hf in bits 0-7, hr in bits 8-15 (counts <= 255)
//   otherwise: full 32-bit counts, hf in hits[cell], hr in hits[ns*nt + cell]
//              (any sentence length: counts are bounded by |A| < 2^31)
template <bool kPacked16, class G>
__device__ void tile_join(G g, const bm_sentences& S, const bm_lexicon& L, int s0, int ns,
                          int t0, int nt, uint32_t* hits, JoinSmem& js) {
  const int ncell = ns * nt;
  const int nwords = kPacked16 ? (ncell + 1) / 2 : 2 * ncell;
  for (int k = g.rank(); k < nwords; k += g.size()) hits[k] = 0u;
  g.sync();
  // forward: source alpha entries through FWD into target U sets
  join_direction(g, S, L.fwd_off, L.fwd_cand, s0, ns, t0, nt, js, [&](int ls, int lt, int w) {
    int cell = ls * nt + lt;
    if (kPacked16)
      atomicAdd(&hits[cell >> 1], (uint32_t)w << ((cell & 1) * 16));
    else
      atomicAdd(&hits[cell], (uint32_t)w);
  });
  // reverse: target alpha entries through REV into source U sets
  join_direction(g, S, L.rev_off, L.rev_cand, t0, nt, s0, ns, js, [&](int lt, int ls, int w) {
    int cell = ls * nt + lt;
    if (kPacked16)
      atomicAdd(&hits[cell >> 1], (uint32_t)w << ((cell & 1) * 16 + 8));
    else
      atomicAdd(&hits[ncell + cell], (uint32_t)w);
  });
}

template <bool kPacked16>
__device__ __forceinline__ void read_hits(const uint32_t* hits, int cell, int ncell, int& hf,
                                          int& hr) {
  if (kPacked16) {
    uint32_t v = hits[cell >> 1] >> ((cell & 1) * 16);
    hf = v & 0xff;
    hr = (v >> 8) & 0xff;
  } else {
    hf = (int)hits[cell];
    hr = (int)hits[ncell + cell];
  }
}

}  // namespace bm
