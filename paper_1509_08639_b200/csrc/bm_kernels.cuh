// Kernel declarations and launch-shape constants shared by bm_kernels.cu and
// bm_api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include <vector>

#include "bm_device.cuh"

namespace bm {

// K1 tile shape and join capacity.
constexpr int kTile = 64;              // 64 x 64 cells per CTA
constexpr int kTileThreads = 256;
#ifndef BM_JOIN_EMAX
#define BM_JOIN_EMAX 1024
#endif
constexpr int kJoinEmax = BM_JOIN_EMAX;  // bucketed ids per join chunk
#ifndef BM_JOIN_BUCKETS
#define BM_JOIN_BUCKETS 512
#endif
constexpr int kJoinBuckets = BM_JOIN_BUCKETS;
__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v / 2); }
static_assert((kJoinBuckets & (kJoinBuckets - 1)) == 0, "bucket count must be a power of two");

// Banded NW (K2/K3): 4 rows per lane, 128 rows per warp band.
constexpr int kBandR = 4;
constexpr int kBandRows = WARP * kBandR;
constexpr int kBandCols = 16 / kBandR;   // columns per packed direction word
constexpr int kPublish = 16;             // boundary publication granularity

// Fused miner limits (warp per document, everything in shared memory).
constexpr int kFusedMaxRows = 256;       // n <= 32 * 8
constexpr int kFusedMaxSmem = 64 * 1024;  // larger slices run 1-3 CTAs/SM: the banded tier is faster

struct WorkItem {
  int32_t doc;
  int32_t band;
};

__host__ __device__ constexpr size_t join_smem_bytes(int emax = kJoinEmax,
                                                     int buckets = kJoinBuckets) {
  return (size_t)emax * 4 + (size_t)emax * 2 + (size_t)(buckets + 1) * 4 + (size_t)buckets * 4;
}
__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

static __device__ const uint64_t g_exp_table[kExpTableWords] = BM_EXP_TABLE_INIT;

__device__ __forceinline__ void stage_exp_table(uint64_t* dst, int rank, int size) {
  for (int k = rank; k < kExpTableWords; k += size) dst[k] = g_exp_table[k];
}

__device__ __forceinline__ JoinSmem carve_join(uint8_t* p, int emax = kJoinEmax,
                                               int buckets = kJoinBuckets) {
  JoinSmem js;
  js.key = (int32_t*)p;
  p += emax * 4;
  js.bstart = (int32_t*)p;
  p += (buckets + 1) * 4;
  js.bfill = (int32_t*)p;
  p += buckets * 4;
  js.owner = (uint16_t*)p;
  js.emax = emax;
  js.nbuckets = buckets;
  js.bshift = 32 - ilog2(buckets);
  return js;
}

int fused_rows_per_lane(int n);

__host__ __device__ inline int64_t band_dirs_words(int32_t n, int32_t m) {
  int64_t nb = (n + kBandRows - 1) / kBandRows;
  int64_t ncg = (m + kBandCols - 1) / kBandCols;
  return nb * ncg * WARP;
}

struct NwArgs {
  const double* S;
  const int64_t* s_off;
  const int32_t* pitch;
  const int32_t* n;
  const int32_t* m;
  double p;
  uint32_t* dirs;
  const int64_t* dir_off;
  double* cost;
  const WorkItem* items;
  int n_items;
  unsigned int* ticket;
  double* bnd;               // boundary rows
  const int64_t* bnd_off;    // per doc: start of its (nb-1) x m boundary rows
  // multi-penalty passes (tuner): penalty q of a pass uses pv[q] and writes
  // dirs + q * dir_stride, bnd + q * bnd_stride, cost + q * cost_stride
  int np = 1;
  double pv[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t dir_stride = 0, bnd_stride = 0;
  int cost_stride = 0;
  // runs of single-band documents (nw_seq_kernel): run r is the plan's
  // documents [seq_off[2r], seq_off[2r + 1]), at most kSeqMaxDocs
  const int32_t* seq_off = nullptr;
  int n_seq = 0;
  // scoring overlapped with the DP: per (doc, band) count of scored 64 x 64
  // tiles (ready[band_base[d] + band]); nullptr when S is complete at launch
  const int* ready = nullptr;
  const int32_t* band_base = nullptr;
};
cudaError_t launch_nw_seq(const NwArgs& a, cudaStream_t st);

struct FusedArgs {
  bm_sentences S;
  bm_docs D;
  bm_lexicon L;
  Model M;
  double threshold;
  double p;
  const int32_t* list;
  int n_list;
  const int64_t* rec_off;
  bm_record* rec;
  int32_t* rec_count;
  double* cost;
  PairTables tabs;         // branch-free feature tables (device pointers)
  ModelTables mt;          // the model's folded margin tables (model_tables)
  uint8_t* hits;           // per-doc dense coverage hit counts (hits_kernel output)
  const int64_t* hit_off;  // byte offset of each doc's hits (16-byte aligned)
};

// Fused banded tier (bm_band.cu): (doc, band) items of a banded plan, scored
// from the document-level join's hit counts and aligned in one kernel.
struct BandArgs {
  bm_sentences S;
  bm_docs D;                 // the plan's documents (local indices)
  Model M;
  ModelTables mt;
  const uint32_t* hits;      // hf | hr << 16 per cell, rows of pitch[d] words
  const int64_t* h_off;
  const int32_t* pitch;
  double p;
  uint32_t* dirs;
  const int64_t* dir_off;
  double* cost;
  const WorkItem* items;
  int n_items;
  unsigned int* ticket;
  double* bnd;
  const int64_t* bnd_off;
};
size_t band_smem_bytes(int m_max);
cudaError_t launch_band(const BandArgs& a, int m_max, cudaStream_t st);

// Where extraction reads a path cell's confidence: the similarity matrix
// (S != nullptr), or -- for the fused banded tier, which never stores it --
// re-scored from the hit counts and the sentences (same value, bit for bit).
struct CellSrc {
  const double* S = nullptr;
  const int64_t* s_off = nullptr;
  bm_sentences sent;
  bm_docs D;
  Model M;
  const uint32_t* hits = nullptr;
  const int64_t* h_off = nullptr;
};

cudaError_t launch_score(const bm_sentences&, const bm_docs&, const bm_lexicon&, const Model&,
                         const int4*, int, const int64_t*, const int32_t*, double*, cudaStream_t);
cudaError_t launch_features(const bm_sentences&, const bm_lexicon&, const int32_t*, const int32_t*,
                            const double*, const double*, int, double*, cudaStream_t);
cudaError_t launch_confidence(const double*, int, const Model&, double*, cudaStream_t);
cudaError_t launch_nw(const NwArgs&, cudaStream_t);
cudaError_t launch_traceback(const uint32_t*, const int64_t*, const int32_t*, const int32_t*, int,
                             const int64_t*, int8_t*, int32_t*, int32_t*, int32_t*, cudaStream_t);
cudaError_t launch_extract(const uint32_t*, const int64_t*, const CellSrc&,
                           const int32_t*, const int32_t*, const int32_t*, int, double,
                           const int64_t*, bm_record*, int32_t*, cudaStream_t,
                           const uint8_t* skip = nullptr);
// Band-parallel extraction of the long documents of a banded plan (local
// indices big[0, n_big)); device arrays, see band_exit_kernel.
constexpr int kGatherMaxBands = 1024;  // bands per document (n <= 131072)
struct BandedExtract {
  int n_big = 0;
  int max_bands = 0;            // max bands over the big documents
  int64_t max_exit_walks = 0;   // max (bands - 1) * m over the big documents
  const int32_t* big = nullptr;
  const int64_t* e_off = nullptr;   // exit-map offset per big document ((bands) x (m + 1))
  int32_t* exits = nullptr;
  int32_t* entry = nullptr;         // per band slot: the true path's entry column
  const int64_t* b_off = nullptr;   // first band slot per big document
  bm_record* slots = nullptr;       // kBandRows records per band
  int32_t* slot_cnt = nullptr;
};
cudaError_t launch_extract_banded(const uint32_t* dirs, const int64_t* dir_off, const CellSrc& cs,
                                  const int32_t* pitch, const int32_t* n,
                                  const int32_t* m, const BandedExtract& bx, double thr,
                                  const int64_t* rec_off, bm_record* rec, int32_t* cnt,
                                  cudaStream_t st);
cudaError_t launch_tune_count(const uint32_t*, const int64_t*, const double*, const int64_t*,
                              const int32_t*, const int32_t*, const int32_t*, int, const double*,
                              int, const int64_t*, const int64_t*, unsigned long long*,
                              unsigned long long*, cudaStream_t);
void join_items(const int32_t* n, const int32_t* m, int nd, std::vector<int4>& items);
cudaError_t launch_score_hits(const bm_sentences& S, const bm_docs& D, const bm_lexicon& L,
                              const Model& M, const ModelTables& mt, const int4* items, int n_items, uint32_t* hits,
                              const int64_t* h_off, const int4* tiles, int n_tiles,
                              const int64_t* s_off, const int32_t* pitch, double* out,
                              cudaStream_t st, int* ready = nullptr,
                              const int32_t* band_base = nullptr);
cudaError_t launch_compact(const bm_record*, const int64_t*, const int32_t*, int, int64_t*,
                           int64_t*, bm_record*, int64_t* bsum, cudaStream_t, int doc0 = 0);
cudaError_t launch_scan_counts(const int32_t* cnt, int n, int64_t* off, int64_t* total,
                               int64_t* bsum, cudaStream_t st);
size_t scan_scratch_count(int n);
struct MergeArgs;
cudaError_t launch_merge_bidir(const MergeArgs& a, cudaStream_t st);
cudaError_t launch_doc_offsets(const bm_record* r, int64_t n, int n_docs, int64_t* off,
                               cudaStream_t st);
cudaError_t launch_merge_shards(const bm_record* rec, int64_t stride, const int64_t* len, int world,
                                int n_docs, int32_t* counts, int64_t* src_start, int64_t* goff,
                                int64_t* total, int64_t* bsum, bm_record* out, cudaStream_t st);
size_t score_smem_bytes();
cudaError_t preload_score_hits();
cudaError_t launch_fp64_probe(double*, int, int, cudaStream_t);
long long launches();
cudaError_t ensure_quot_table();
PairTables pair_tables();
cudaError_t model_tables(const Model& M, ModelTables* out);
cudaError_t launch_unpack_wire(const uint8_t*, const uint8_t*, const uint8_t*, const uint16_t*,
                               const uint8_t*, const uint16_t*, int, int, int64_t, int64_t, int64_t,
                               int64_t, int32_t*, int32_t*, int32_t*, int32_t*, uint32_t*, int32_t*,
                               cudaStream_t);
cudaError_t launch_unpack_packed(const uint32_t*, const int32_t*, const int32_t*, const uint16_t*,
                                 const uint16_t*, int, int, int32_t*, int32_t*, int32_t*, int32_t*,
                                 int32_t*, uint32_t*, int32_t*, int32_t*, cudaStream_t);
size_t ring_slice_bytes(int n, int m, int R);
size_t hits_kernel_smem(int n, int m);
cudaError_t launch_hits(const FusedArgs& a, size_t smem, cudaStream_t st);
cudaError_t launch_ring(const FusedArgs& a, int R, size_t smem, cudaStream_t st);
extern std::atomic<long long> g_launches;
cudaError_t launch_select(const double*, int64_t, const int32_t*, const int32_t*, int, double,
                          double*, uint8_t*, cudaStream_t);

}  // namespace bm
