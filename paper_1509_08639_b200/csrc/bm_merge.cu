// bidirectional_merge on the device (bimine/miner.py:131-155).
//
// Per document, the forward-model records F and the backward-model records B
// (each in its pass's path order, (i, j) in that pass's orientation) become
// the pair's merged record list: re-oriented to the pair's (source, target)
// frame (miner.py:115-128; a pass that read the pair swapped is labelled
// "backward"), keyed on the normalized text of both sentences, one record per
// key -- the reference's scan over F then B keeps the first record unless a
// later one has a higher confidence, or the same confidence and the label
// "forward" over "backward" -- and sorted by (source index, target index).
//
// One CTA per document, deterministic:
//   1. every record claims its key's slot in an open-addressing table and
//      raises the slot's best confidence (atomicMax on the bit pattern: the
//      confidences are positive doubles, ordered like their bits);
//   2. records holding the best confidence lower the slot's rank
//      ((label != forward) << 31 | position in F-then-B order) with atomicMin;
//   3. the record whose rank is the slot's rank is the winner -- exactly the
//      record the sequential scan ends with;
//   4. F's and B's winners are each already in (i, j) order (a path's diagonal
//      cells increase in both coordinates, in either orientation), so a
//      winner's output position is its rank among its own list's winners plus
//      the number of the other list's winners before it (binary search).
#include <cuda_runtime.h>
#include <stdint.h>

#include "bm_kernels.cuh"

namespace bm {

constexpr int kMergeThreads = 256;
constexpr uint64_t kEmptyKey = ~0ull;

struct MergeArgs {
  const bm_record* fwd;
  const bm_record* bwd;
  const int64_t* f_off;     // [n_docs + 1] record offsets of each document
  const int64_t* b_off;
  const int32_t* src0;      // [n_docs] first source / target sentence
  const int32_t* tgt0;
  const int32_t* norm_key;  // [n_sent] normalized-text id of every sentence
  const uint8_t* swap_f;    // [n_docs] the pass read the pair swapped
  const uint8_t* swap_b;
  int n_docs;
  // scratch: document d's table at 4 * (f_off + b_off) (capacity < 4 k), its
  // records' slots and winners at f_off + b_off
  uint64_t* slot_key;
  uint64_t* slot_conf;
  uint32_t* slot_rank;
  uint32_t* rec_slot;
  int64_t* win_ij;          // compacted winners' (i << 32 | j), F then B
  bm_record* out;           // per document at f_off[d] + b_off[d]
  int32_t* out_cnt;
  int64_t* out_off;         // [n_docs] = f_off[d] + b_off[d]
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

// exclusive CTA scan of a 0/1 flag; returns the prefix and the total
__device__ __forceinline__ int cta_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  int base = 0;
  total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    base += w < wid ? warp_tot[w] : 0;
    total += warp_tot[w];
  }
  __syncthreads();
  return base + incl - v;
}

__global__ void __launch_bounds__(kMergeThreads) merge_bidir_kernel(MergeArgs a) {
  __shared__ int warp_tot[kMergeThreads / 32];
  __shared__ int nw_f_sh;
  const int d = blockIdx.x;
  const int64_t f0 = a.f_off[d], kf = a.f_off[d + 1] - f0;
  const int64_t b0 = a.b_off[d], kb = a.b_off[d + 1] - b0;
  const int64_t k = kf + kb;
  const int64_t base = f0 + b0;  // this document's scratch / output region
  if (threadIdx.x == 0) a.out_off[d] = base;
  if (k == 0) {
    if (threadIdx.x == 0) a.out_cnt[d] = 0;
    return;
  }
  int64_t cap = 1;
  while (cap < 2 * k) cap <<= 1;  // 2k <= cap < 4k
  uint64_t* skey = a.slot_key + 4 * base;
  uint64_t* sconf = a.slot_conf + 4 * base;
  uint32_t* srank = a.slot_rank + 4 * base;
  uint32_t* rslot = a.rec_slot + base;
  const int32_t s0 = a.src0[d], t0 = a.tgt0[d];
  const bool swf = a.swap_f[d] != 0, swb = a.swap_b[d] != 0;
  auto rec_at = [&](int64_t q, int32_t& si, int32_t& tj, bool& fwd_label, double& conf) {
    const bool from_f = q < kf;
    const bm_record r = from_f ? a.fwd[f0 + q] : a.bwd[b0 + (q - kf)];
    const bool sw = from_f ? swf : swb;
    si = sw ? r.j : r.i;
    tj = sw ? r.i : r.j;
    fwd_label = !sw;
    conf = r.conf;
  };
  for (int64_t s = threadIdx.x; s < cap; s += blockDim.x) {
    skey[s] = kEmptyKey;
    sconf[s] = 0ull;
    srank[s] = 0xffffffffu;
  }
  __syncthreads();
  // 1. claim the key's slot, raise its best confidence
  for (int64_t q = threadIdx.x; q < k; q += blockDim.x) {
    int32_t si, tj;
    bool fl;
    double conf;
    rec_at(q, si, tj, fl, conf);
    const uint64_t key = ((uint64_t)(uint32_t)a.norm_key[s0 + si] << 32) |
                         (uint32_t)a.norm_key[t0 + tj];
    uint64_t s = mix64(key) & (uint64_t)(cap - 1);
    for (;;) {
      const unsigned long long prev =
          atomicCAS((unsigned long long*)(skey + s), (unsigned long long)kEmptyKey,
                    (unsigned long long)key);
      if (prev == kEmptyKey || prev == key) break;
      s = (s + 1) & (uint64_t)(cap - 1);
    }
    rslot[q] = (uint32_t)s;
    atomicMax((unsigned long long*)(sconf + s), (unsigned long long)__double_as_longlong(conf));
  }
  __syncthreads();
  // 2. among the best-confidence records: forward label first, then first seen
  for (int64_t q = threadIdx.x; q < k; q += blockDim.x) {
    int32_t si, tj;
    bool fl;
    double conf;
    rec_at(q, si, tj, fl, conf);
    const uint32_t s = rslot[q];
    if ((uint64_t)__double_as_longlong(conf) == sconf[s])
      atomicMin(srank + s, (fl ? 0u : 0x80000000u) | (uint32_t)q);
  }
  __syncthreads();
  // 3. winners, compacted per list in (i, j) order
  int64_t* wij = a.win_ij + base;
  int nw_f = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int64_t lo = pass == 0 ? 0 : kf, hi = pass == 0 ? kf : k;
    int carry = 0;
    for (int64_t c0 = lo; c0 < hi; c0 += blockDim.x) {
      const int64_t q = c0 + threadIdx.x;
      int win = 0;
      int32_t si = 0, tj = 0;
      if (q < hi) {
        bool fl;
        double conf;
        rec_at(q, si, tj, fl, conf);
        win = (srank[rslot[q]] & 0x7fffffffu) == (uint32_t)q;
      }
      int total;
      const int pos = cta_scan(win, warp_tot, total);
      if (win) wij[(pass == 0 ? 0 : nw_f) + carry + pos] = ((int64_t)si << 32) | (uint32_t)tj;
      carry += total;
    }
    if (pass == 0) nw_f = carry;
    else if (threadIdx.x == 0) nw_f_sh = carry;  // winners of B
  }
  __syncthreads();
  const int nw_b = nw_f_sh;
  // 4. merge the two (i, j)-ordered winner lists
  bm_record* out = a.out + base;
  for (int q = threadIdx.x; q < nw_f + nw_b; q += blockDim.x) {
    const bool in_f = q < nw_f;
    const int64_t v = wij[q];
    const int64_t* other = in_f ? wij + nw_f : wij;
    int lo = 0, hi = in_f ? nw_b : nw_f;
    while (lo < hi) {  // other-list winners before v
      const int mid = (lo + hi) >> 1;
      if (other[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    const int pos = (in_f ? q : q - nw_f) + lo;
    bm_record r;
    r.doc = d;
    r.i = (int32_t)(v >> 32);
    r.j = (int32_t)(uint32_t)v;
    r.pad = 0;
    r.conf = 0.0;
    out[pos] = r;
  }
  __syncthreads();
  // confidences and labels of the winners (one more pass over the records)
  for (int64_t q = threadIdx.x; q < k; q += blockDim.x) {
    if ((srank[rslot[q]] & 0x7fffffffu) != (uint32_t)q) continue;
    int32_t si, tj;
    bool fl;
    double conf;
    rec_at(q, si, tj, fl, conf);
    const int64_t v = ((int64_t)si << 32) | (uint32_t)tj;
    int lo = 0, hi = nw_f + nw_b;  // out is sorted by (i, j): find v
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const int64_t w = ((int64_t)out[mid].i << 32) | (uint32_t)out[mid].j;
      if (w < v) lo = mid + 1;
      else hi = mid;
    }
    out[lo].conf = conf;
    out[lo].pad = fl ? 0 : 1;  // direction: 0 forward, 1 backward
  }
  if (threadIdx.x == 0) a.out_cnt[d] = nw_f + nw_b;
}

// per-document record offsets of a document-ordered stream (lower bounds)
__global__ void doc_offsets_kernel(const bm_record* __restrict__ r, int64_t n, int n_docs,
                                   int64_t* __restrict__ off) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d > n_docs) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (r[mid].doc < d) lo = mid + 1;
    else hi = mid;
  }
  off[d] = lo;
}

cudaError_t launch_merge_bidir(const MergeArgs& a, cudaStream_t st) {
  if (a.n_docs == 0) return cudaSuccess;
  merge_bidir_kernel<<<a.n_docs, kMergeThreads, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) g_launches += 1;
  return e;
}

cudaError_t launch_doc_offsets(const bm_record* r, int64_t n, int n_docs, int64_t* off,
                               cudaStream_t st) {
  doc_offsets_kernel<<<(n_docs + 1 + 255) / 256, 256, 0, st>>>(r, n, n_docs, off);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) g_launches += 1;
  return e;
}

}  // namespace bm
