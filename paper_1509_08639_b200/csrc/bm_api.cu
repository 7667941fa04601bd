// C ABI of libbimine_b200.so (declared in include/bimine_b200.h).
//
// Host-side planning only: which kernel tier each document goes to, tile and
// band work lists, offsets into stream-ordered scratch (cudaMallocAsync), and
// error mapping. No arithmetic of the hot path happens here.
#include <deque>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bimine_b200.h"
#include "bm_kernels.cuh"


using namespace bm;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? BM_ENOMEM : BM_ECUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define BM_CK(expr, what)                        \
  do {                                           \
    cudaError_t _e = (expr);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

constexpr int kMaxMineStreams = 4;

// Page-locked staging for host -> device uploads of host-built plans. A
// cudaMemcpyAsync from pageable memory may wait for the stream's earlier work
// before it returns (measured: the banded tier's 9 MB of tiles held the host
// until the fused tier's kernels finished), so larger uploads are copied into
// a page-locked block first; a block is reused once the event recorded after
// its copy has completed.
// (The blocks live as long as the thread: no CUDA calls at process teardown.)
// Plan uploads are copied by a kernel that reads the page-locked block over
// the bus (mapped through unified addressing), not by the copy engine: the
// engine serves H2D copies of all streams in submission order, so an upload
// queued on a busy stream behind its kernels would hold up the bulk copies of
// another stream submitted after it (and those would hold up the next plan
// upload), serialising copies and kernels (hostapi.tune_pinned: 31 + 38 ms).
__global__ void h2d_plan_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16,
                                const uint8_t* __restrict__ src_b, uint8_t* __restrict__ dst_b,
                                int tail) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n16; k += stride)
    dst[k] = src[k];
  if (blockIdx.x == 0 && (int)threadIdx.x < tail) dst_b[threadIdx.x] = src_b[threadIdx.x];
}

class PinnedPool {
 public:
  // copies bytes into a free block and enqueues the H2D copy on st
  cudaError_t upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    Block* blk = nullptr;
    // blocks are taken round robin (their uploads complete roughly in order),
    // so the search usually stops at the first block it queries
    const size_t nb = blocks_.size();
    for (size_t q = 0; q < nb && blk == nullptr; ++q) {
      Block& b = blocks_[(next_ + q) % nb];
      if (b.cap >= bytes && cudaEventQuery(b.ev) == cudaSuccess) {
        blk = &b;
        next_ = (next_ + q + 1) % nb;
      }
    }
    if (blk == nullptr) {
      size_t cap = 1 << 12;
      while (cap < bytes) cap <<= 1;
      Block b;
      cudaError_t e = cudaHostAlloc((void**)&b.p, cap, cudaHostAllocMapped | cudaHostAllocPortable);
      if (e != cudaSuccess) return e;
      e = cudaHostGetDevicePointer((void**)&b.d, b.p, 0);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
      if (e != cudaSuccess) {
        cudaFreeHost(b.p);
        return e;
      }
      b.cap = cap;
      blocks_.push_back(b);
      blk = &blocks_.back();
    }
    memcpy(blk->p, src, bytes);
    cudaError_t e;
    static const bool by_kernel =
        getenv("BM_PLAN_COPY_KERNEL") ? atoi(getenv("BM_PLAN_COPY_KERNEL")) != 0 : true;
    if (by_kernel && ((uintptr_t)dst & 15) == 0) {
      const size_t n16 = bytes / 16;
      const int tail = (int)(bytes - n16 * 16);
      const int grid = (int)std::min<size_t>(256, std::max<size_t>(1, (n16 + 255) / 256));
      h2d_plan_kernel<<<grid, 256, 0, st>>>((const uint4*)blk->d, (uint4*)dst, n16,
                                            (const uint8_t*)blk->d + n16 * 16,
                                            (uint8_t*)dst + n16 * 16, tail);
      e = cudaGetLastError();
      if (e == cudaSuccess) bm::g_launches += 1;
    } else {
      e = cudaMemcpyAsync(dst, blk->p, bytes, cudaMemcpyHostToDevice, st);
    }
    if (e != cudaSuccess) return e;
    return cudaEventRecord(blk->ev, st);
  }

 private:
  struct Block {
    char* p = nullptr;  // host address
    char* d = nullptr;  // device address of the mapped block
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
  };
  std::deque<Block> blocks_;  // stable addresses
  size_t next_ = 0;
};

PinnedPool& pinned_pool() {
  static thread_local PinnedPool pool;
  return pool;
}

// Stream-ordered scratch: allocated on `st`, freed on `st` when it goes out of
// scope, so it stays valid for every kernel enqueued before the free.
class Scratch {
 public:
  explicit Scratch(cudaStream_t st) : st_(st) {}
  ~Scratch() {
    for (void* p : ptrs_) cudaFreeAsync(p, st_);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st_);
    if (e != cudaSuccess) return e;
    ptrs_.push_back(p);
    *out = (T*)p;
    return cudaSuccess;
  }
  template <class T>
  cudaError_t upload(T** out, const std::vector<T>& v) {
    cudaError_t e = alloc(out, v.size());
    if (e != cudaSuccess || v.empty()) return e;
    const size_t bytes = v.size() * sizeof(T);
    return pinned_pool().upload(*out, v.data(), bytes, st_);
  }

 private:
  cudaStream_t st_;
  std::vector<void*> ptrs_;
};

// Grow-only device workspaces for the large per-call scratch (similarity
// matrices, hit counts, direction codes, boundary rows), one set per stream of
// the calling thread: work on one stream is ordered, so a buffer is reused by
// the next group or chunk on that stream without a free / malloc round trip
// (pool growth between calls cost tens of milliseconds on C3), and a buffer
// that must grow is released stream-ordered on its own stream.
enum WsSlot { kWsS, kWsDirs, kWsBnd, kWsHits, kWsHits16, kWsSlots };
struct Workspace {
  cudaStream_t st;
  int dev;
  void* buf[kWsSlots];
  size_t cap[kWsSlots];
};

std::vector<Workspace>& workspaces() {
  static thread_local std::vector<Workspace> spaces;
  return spaces;
}

// Releases a workspace set (the rare eviction path and bm_trim): its stream
// may be gone, so the device is synchronized and the buffers freed directly.
void ws_release(Workspace& w) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(w.dev);
  cudaDeviceSynchronize();
  for (int k = 0; k < kWsSlots; ++k)
    if (w.buf[k]) cudaFree(w.buf[k]);
  cudaSetDevice(cur);
}

template <class T>
cudaError_t ws_get(cudaStream_t st, WsSlot slot, T** out, size_t count) {
  std::vector<Workspace>& spaces = workspaces();
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  Workspace* w = nullptr;
  for (Workspace& x : spaces)
    if (x.st == st && x.dev == dev) w = &x;
  if (w == nullptr) {
    if (spaces.size() >= 8) {  // bounded: release the oldest stream's set
      ws_release(spaces.front());
      spaces.erase(spaces.begin());
    }
    Workspace fresh{};
    fresh.st = st;
    fresh.dev = dev;
    spaces.push_back(fresh);
    w = &spaces.back();
  }
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  if (w->cap[slot] < bytes) {
    if (w->buf[slot]) cudaFreeAsync(w->buf[slot], st);
    w->buf[slot] = nullptr;
    w->cap[slot] = 0;
    const size_t grow = bytes + bytes / 8;  // headroom: groups differ slightly in size
    e = cudaMallocAsync(&w->buf[slot], grow, st);
    if (e != cudaSuccess) return e;
    w->cap[slot] = grow;
  }
  *out = (T*)w->buf[slot];
  return cudaSuccess;
}

void note_launch() { bm::g_launches += 1; }

Model to_model(const bm_model* m) {
  Model M;
  for (int k = 0; k < 7; ++k) M.w[k] = m->w[k];
  M.bias = m->bias;
  return M;
}

inline int32_t pitch_of(int32_t m) { return (m + 3) & ~3; }

// Unfused general path for a subset of documents: K1 -> K2/K3 -> consumer.
struct GeneralPlan {
  std::vector<int32_t> docs;  // indices into the batch
  std::vector<int64_t> s_off, dir_off, bnd_off;
  std::vector<int32_t> pitch, n, m;
  std::vector<int4> tiles;    // doc field = local index
  std::vector<WorkItem> items;
  int64_t s_total = 0, dir_total = 0, bnd_total = 0;

  void add(int32_t d, int32_t nd, int32_t md) {
    const int32_t local = (int32_t)docs.size();
    docs.push_back(d);
    n.push_back(nd);
    m.push_back(md);
    pitch.push_back(pitch_of(md));
    s_off.push_back(s_total);
    s_total += (int64_t)nd * pitch_of(md);
    dir_off.push_back(dir_total);
    dir_total += band_dirs_words(nd, md);
    const int nb = (nd + kBandRows - 1) / kBandRows;
    bnd_off.push_back(bnd_total);
    bnd_total += (int64_t)(nb - 1) * md;
    for (int r0 = 0; r0 < nd; r0 += kTile)
      for (int c0 = 0; c0 < md; c0 += kTile) tiles.push_back(make_int4(local, r0, c0, 0));
    for (int b = 0; b < nb; ++b) items.push_back(WorkItem{local, b});
  }
};

// Device copies of a GeneralPlan plus the subset's own bm_docs view.
struct GeneralDev {
  int64_t *s_off, *dir_off, *bnd_off;
  int32_t *pitch, *n, *m, *src0, *tgt0;
  int4* tiles;
  WorkItem* items;
  double *S, *bnd;
  uint32_t* dirs;
  unsigned int* ticket;
  uint32_t* hits = nullptr;     // document-level join output (doc_join plans)
  int64_t* h_off = nullptr;
  std::vector<WorkItem> order;  // the DP's (doc, band) work order (host copy)
};

// Gathers src0/tgt0/n/m of the subset on the device from the batch arrays.
__global__ void gather_docs_kernel(bm_docs D, const int32_t* idx, int k, int32_t* src0,
                                   int32_t* tgt0) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < k) {
    src0[q] = D.src0[idx[q]];
    tgt0[q] = D.tgt0[idx[q]];
  }
}

__global__ void scatter_results_kernel(const int32_t* idx, int k, const double* cost_local,
                                       double* cost, const bm_record* rec_local,
                                       const int64_t* rec_off_local, const int32_t* cnt_local,
                                       const int64_t* rec_off, bm_record* rec, int32_t* cnt) {
  int q = blockIdx.x;
  if (q >= k) return;
  const int d = idx[q];
  if (threadIdx.x == 0) {
    cost[d] = cost_local[q];
    cnt[d] = cnt_local[q];
  }
  for (int t = threadIdx.x; t < cnt_local[q]; t += blockDim.x) {
    bm_record r = rec_local[rec_off_local[q] + t];
    r.doc = d;
    rec[rec_off[d] + t] = r;
  }
}

// BM_TRACE=1: host-side phase timings of the planning code on stderr.
struct HostTrace {
  bool on;
  std::chrono::steady_clock::time_point t0;
  const char* fn;
  explicit HostTrace(const char* f) : on(getenv("BM_TRACE") != nullptr), t0(std::chrono::steady_clock::now()), fn(f) {}
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[bm trace] %s %-24s %8.3f ms\n", fn, what,
            std::chrono::duration<double, std::milli>(t - t0).count());
  }
};

int general_prepare(const GeneralPlan& g, const bm_docs* docs, Scratch& sc, GeneralDev& dv,
                    cudaStream_t st, bool store_s = true) {
  const int k = (int)g.docs.size();
  HostTrace tr("general_prepare");
  int32_t* idx = nullptr;
  BM_CK(sc.upload(&idx, g.docs), "upload");
  BM_CK(sc.upload(&dv.s_off, g.s_off), "upload");
  BM_CK(sc.upload(&dv.dir_off, g.dir_off), "upload");
  BM_CK(sc.upload(&dv.bnd_off, g.bnd_off), "upload");
  BM_CK(sc.upload(&dv.pitch, g.pitch), "upload");
  BM_CK(sc.upload(&dv.n, g.n), "upload");
  BM_CK(sc.upload(&dv.m, g.m), "upload");
  BM_CK(sc.upload(&dv.tiles, g.tiles), "upload");
  tr.mark("plan uploads");
  // (doc, band) work order of the banded DP. A band waits for the band above
  // to publish its bottom row; BM_NW_STAGGER = K places band b of the q-th
  // document at position q + b * K instead of next to band b - 1 (K = 0), so
  // the persistent warps spend less time spinning on bands that have barely
  // started (C3 200k: 74.0 -> 72.8 ms at K = 512). Band b - 1 always
  // precedes band b (deadlock freedom).
  static const int kStagger = getenv("BM_NW_STAGGER") ? atoi(getenv("BM_NW_STAGGER")) : 512;
  if (kStagger > 0 && g.items.size() > 1) {
    std::vector<std::pair<int64_t, int>> key(g.items.size());
    for (size_t q = 0; q < g.items.size(); ++q)
      key[q] = {(int64_t)g.items[q].doc + (int64_t)g.items[q].band * kStagger, (int)q};
    std::stable_sort(key.begin(), key.end());
    dv.order.resize(g.items.size());
    for (size_t q = 0; q < dv.order.size(); ++q) dv.order[q] = g.items[key[q].second];
  } else {
    dv.order = g.items;
  }
  BM_CK(sc.upload(&dv.items, dv.order), "upload");
  tr.mark("items");
  BM_CK(sc.alloc(&dv.src0, k), "alloc");
  BM_CK(sc.alloc(&dv.tgt0, k), "alloc");
  dv.S = nullptr;  // the fused banded tier never stores the matrix
  if (store_s) BM_CK(ws_get(st, kWsS, &dv.S, (size_t)g.s_total), "alloc S");
  tr.mark("S workspace");
  BM_CK(ws_get(st, kWsDirs, &dv.dirs, (size_t)g.dir_total), "alloc dirs");
  BM_CK(ws_get(st, kWsBnd, &dv.bnd, (size_t)g.bnd_total), "alloc boundary");
  BM_CK(sc.alloc(&dv.ticket, 1), "alloc ticket");
  tr.mark("workspaces");
  gather_docs_kernel<<<(k + 255) / 256, 256, 0, st>>>(*docs, idx, k, dv.src0, dv.tgt0);
  BM_CK(cudaGetLastError(), "gather_docs");
  note_launch();
  return BM_OK;
}

bm_docs local_docs(const GeneralDev& dv, int k) {
  bm_docs D;
  D.n_docs = k;
  D.src0 = dv.src0;
  D.n = dv.n;
  D.tgt0 = dv.tgt0;
  D.m = dv.m;
  return D;
}

int general_nw(const GeneralPlan& g, GeneralDev& dv, double penalty, double* cost,
               cudaStream_t st) {
  BM_CK(cudaMemsetAsync(dv.ticket, 0, 4, st), "memset");
  // boundary rows start as the sentinel (negative) pattern consumers spin on
  BM_CK(cudaMemsetAsync(dv.bnd, 0xde, std::max<int64_t>(g.bnd_total, 1) * 8, st), "memset");
  NwArgs a;
  a.S = dv.S;
  a.s_off = dv.s_off;
  a.pitch = dv.pitch;
  a.n = dv.n;
  a.m = dv.m;
  a.p = penalty;
  a.dirs = dv.dirs;
  a.dir_off = dv.dir_off;
  a.cost = cost;
  a.items = dv.items;
  a.n_items = (int)g.items.size();
  a.ticket = dv.ticket;
  a.bnd = dv.bnd;
  a.bnd_off = dv.bnd_off;
  BM_CK(launch_nw(a, st), "nw_band_kernel");
  return BM_OK;
}

bool check_penalty(double p) { return p >= 0.0; }

// Largest ring-kernel smem slice a document may need and still take the fused
// tier (BM_FUSED_MAX_SMEM overrides; experiments).
size_t fused_max_smem() {
  static const size_t v =
      getenv("BM_FUSED_MAX_SMEM") ? (size_t)atoll(getenv("BM_FUSED_MAX_SMEM")) : (size_t)kFusedMaxSmem;
  return v;
}  // NaN fails (aligner.py:209-213)


// Banded tier for the documents of `g` (K1 -> K2/K3 -> K4, then scatter into
// the caller's per-document record slots).
// K1 over a banded plan: the document-level join + scoring kernels when every
// document's counts fit 16 bits (doc_join: max tokens per sentence <= 65535,
// checked by the caller; sides <= 65535 sentences, checked here), else the
// per-tile kernel.
int score_general(const GeneralPlan& g, const bm_sentences* sent, const bm_docs& D,
                  const bm_lexicon* lex, const Model& M, GeneralDev& dv, bool doc_join,
                  Scratch& sc, cudaStream_t st, bool join_only = false) {
  const int k = (int)g.docs.size();
  for (int q = 0; q < k && doc_join; ++q) doc_join = g.n[q] <= 65535 && g.m[q] <= 65535;
  if (!doc_join) {
    BM_CK(launch_score(*sent, D, *lex, M, dv.tiles, (int)g.tiles.size(), dv.s_off, dv.pitch, dv.S,
                       st),
          "score_tile_kernel");
    return BM_OK;
  }
  std::vector<int64_t> hoff(k);
  int64_t ht = 0;
  for (int q = 0; q < k; ++q) {
    hoff[q] = ht;  // rows of pitch_of(m) words: 16-byte aligned rows
    ht += (int64_t)g.n[q] * g.pitch[q];
  }
  std::vector<int4> items;
  join_items(g.n.data(), g.m.data(), k, items);
  uint32_t* hits = nullptr;
  int64_t* dho = nullptr;
  int4* dit = nullptr;
  BM_CK(ws_get(st, kWsHits, &hits, (size_t)ht), "alloc hits");
  BM_CK(cudaMemsetAsync(hits, 0, (size_t)ht * 4, st), "memset hits");
  BM_CK(sc.upload(&dho, hoff), "upload");
  BM_CK(sc.upload(&dit, items), "upload");
  ModelTables mt;
  BM_CK(model_tables(M, &mt), "model tables");
  BM_CK(launch_score_hits(*sent, D, *lex, M, mt, dit, (int)items.size(), hits, dho, dv.tiles,
                          join_only ? 0 : (int)g.tiles.size(), dv.s_off, dv.pitch,
                          join_only ? nullptr : dv.S, st),
        "score_hits_kernel");
  dv.hits = hits;
  dv.h_off = dho;
  return BM_OK;
}

// `after` waits for everything enqueued on `before` so far.
static cudaError_t stream_after(cudaStream_t after, cudaStream_t before) {
  cudaEvent_t e;
  cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (r != cudaSuccess) return r;
  r = cudaEventRecord(e, before);
  if (r == cudaSuccess) r = cudaStreamWaitEvent(after, e, 0);
  cudaEventDestroy(e);
  return r;
}

// BM_DP_OVERLAP=1: a few long documents' DP starts each band as soon as its
// tiles are scored (opt-in: measured on C4 2.81 -> 4.5 ms -- the 64 DP warps
// share their SMs' schedulers with the scoring CTAs and their latency chain
// slows by more than the scoring time it hides)
static bool dp_overlap_on() {
  static const bool v = getenv("BM_DP_OVERLAP") ? atoi(getenv("BM_DP_OVERLAP")) != 0 : false;
  return v;
}

// BM_NW_SEQ=0: the tuner's single-band documents keep one DP item each
static bool nw_seq_on() {
  static const bool v = getenv("BM_NW_SEQ") ? atoi(getenv("BM_NW_SEQ")) != 0 : true;
  return v;
}

static bool dp_prio_on() {
  static const bool v = getenv("BM_DP_PRIO") ? atoi(getenv("BM_DP_PRIO")) != 0 : false;
  return v;
}

// The high-priority companion stream of a mining stream (one per stream and
// device, created on first use, kept for the thread's lifetime).
static cudaStream_t dp_stream(cudaStream_t st) {
  static thread_local std::vector<std::pair<std::pair<cudaStream_t, int>, cudaStream_t>> map;
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& e : map)
    if (e.first.first == st && e.first.second == dev) return e.second;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) return st;
  map.push_back({{st, dev}, s});
  return s;
}

// Band-parallel extraction (launch_extract_banded): documents whose path is at
// least BM_PAR_WALK_MIN moves long (default 8192; 0 disables), while the exit
// maps of the plan stay within kParWalkBudget walks (one walk per band and
// entry column; 2M ~ four 8192^2 documents, ~0.1 ms of the whole GPU).
constexpr int64_t kParWalkBudget = 2 << 20;
int64_t par_walk_min() {
  static const int64_t v = getenv("BM_PAR_WALK_MIN") ? atoll(getenv("BM_PAR_WALK_MIN")) : 8192;
  return v > 0 ? v : INT64_MAX;
}

int mine_general(const GeneralPlan& g, const bm_sentences* sent, const bm_docs* docs,
                 const bm_lexicon* lex, const Model& M, double threshold, double penalty,
                 const int64_t* rec_off, bm_record* rec, int32_t* rec_count, double* cost,
                 bool doc_join, Scratch& sc, cudaStream_t st, bool fused = false) {
  {
    HostTrace tr("mine_general");
    const int k = (int)g.docs.size();
    for (int q = 0; q < k && fused; ++q) fused = g.n[q] <= 65535 && g.m[q] <= 65535;
    fused = fused && doc_join;
    // a few long documents (C4: 64 bands of one 8192^2 pair) leave most SMs to
    // the scoring kernel while their DP runs: the DP starts each band as soon
    // as the band's tiles are scored (readiness counters) instead of after the
    // whole matrix. Only with at most one band per SM, so the spinning DP
    // warps can never take the resources the scoring CTAs need.
    bool dj = doc_join;
    for (int q = 0; q < k && dj; ++q) dj = g.n[q] <= 65535 && g.m[q] <= 65535;
    int sms = 0;
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const bool overlap = !fused && dj && dp_overlap_on() && (int64_t)g.items.size() <= sms;
    GeneralDev dv;
    int rc = general_prepare(g, docs, sc, dv, st, /*store_s=*/!fused);
    if (rc) return rc;
    tr.mark("prepare");
    const bm_docs D = local_docs(dv, k);
    rc = score_general(g, sent, D, lex, M, dv, doc_join, sc, st, /*join_only=*/fused || overlap);
    if (rc) return rc;
    tr.mark("score enqueued");
    int* ready = nullptr;
    int32_t* band_base = nullptr;
    if (overlap) {
      BM_CK(preload_score_hits(), "load score_hits_kernel");
      std::vector<int32_t> bb(k);
      int32_t nb = 0;
      for (int q = 0; q < k; ++q) {
        bb[q] = nb;
        nb += (g.n[q] + kBandRows - 1) / kBandRows;
      }
      BM_CK(sc.upload(&band_base, bb), "upload");
      BM_CK(sc.alloc(&ready, (size_t)nb), "alloc");
      BM_CK(cudaMemsetAsync(ready, 0, (size_t)nb * 4, st), "memset");
    }
    // every buffer of the DP and extraction phase is allocated and uploaded on
    // st first; the phase itself may then run on the high-priority DP stream
    double* cost_l = nullptr;
    BM_CK(sc.alloc(&cost_l, k), "alloc");
    BM_CK(cudaMemsetAsync(dv.ticket, 0, 4, st), "memset");
    // boundary rows start as the sentinel (negative) pattern consumers spin on
    BM_CK(cudaMemsetAsync(dv.bnd, 0xde, std::max<int64_t>(g.bnd_total, 1) * 8, st), "memset");
    std::vector<int64_t> roff(k);
    int64_t rt = 0;
    for (int q = 0; q < k; ++q) {
      roff[q] = rt;
      rt += std::min(g.n[q], g.m[q]);
    }
    int64_t* droff = nullptr;
    bm_record* rl = nullptr;
    int32_t* cl = nullptr;
    int32_t* idx = nullptr;
    BM_CK(sc.upload(&droff, roff), "upload");
    BM_CK(sc.alloc(&rl, (size_t)rt), "alloc");
    BM_CK(sc.alloc(&cl, k), "alloc");
    BM_CK(sc.upload(&idx, g.docs), "upload");
    // long paths (n + m >= kParWalkMin) take the band-parallel extraction
    // while the exit maps stay small next to the rest of the plan's work
    std::vector<int32_t> big;
    std::vector<int64_t> e_off, b_off;
    std::vector<uint8_t> skip;
    BandedExtract bx;
    {
      std::vector<int32_t> cand;
      for (int q = 0; q < k; ++q)
        if ((int64_t)g.n[q] + g.m[q] >= par_walk_min() && g.n[q] > 4 * kBandRows &&
            (g.n[q] + kBandRows - 1) / kBandRows <= kGatherMaxBands)
          cand.push_back(q);
      std::sort(cand.begin(), cand.end(), [&](int a, int b) {
        return (int64_t)g.n[a] + g.m[a] > (int64_t)g.n[b] + g.m[b];
      });
      int64_t walks = 0, et = 0, bt = 0;
      for (int q : cand) {
        const int nb = (g.n[q] + kBandRows - 1) / kBandRows;
        const int64_t w = (int64_t)(nb - 1) * g.m[q];
        if (walks + w > kParWalkBudget) break;
        walks += w;
        big.push_back(q);
        e_off.push_back(et);
        b_off.push_back(bt);
        et += (int64_t)nb * (g.m[q] + 1);
        bt += nb;
        bx.max_bands = std::max(bx.max_bands, nb);
        bx.max_exit_walks = std::max(bx.max_exit_walks, w);
      }
      if (!big.empty()) {
        skip.assign(k, 0);
        for (int q : big) skip[q] = 1;
        bx.n_big = (int)big.size();
        int32_t* dbig = nullptr;
        int64_t *deo = nullptr, *dbo = nullptr;
        BM_CK(sc.upload(&dbig, big), "upload");
        BM_CK(sc.upload(&deo, e_off), "upload");
        BM_CK(sc.upload(&dbo, b_off), "upload");
        BM_CK(sc.alloc(&bx.exits, (size_t)et), "alloc");
        BM_CK(sc.alloc(&bx.slots, (size_t)bt * kBandRows), "alloc");
        BM_CK(sc.alloc(&bx.slot_cnt, (size_t)bt), "alloc");
        BM_CK(sc.alloc(&bx.entry, (size_t)bt), "alloc");
        bx.big = dbig;
        bx.e_off = deo;
        bx.b_off = dbo;
      }
    }
    uint8_t* dskip = nullptr;
    if (bx.n_big) BM_CK(sc.upload(&dskip, skip), "upload");
    ModelTables mt;
    BM_CK(model_tables(M, &mt), "model tables");
    // BM_DP_PRIO: the latency-bound phase (DP, extraction) on a high-priority
    // stream, so its CTAs are dispatched next to the scoring kernels of other
    // groups instead of queueing behind their waves (experiments)
    cudaStream_t sd = st;
    if (dp_prio_on() || overlap) {
      sd = dp_stream(st);
      BM_CK(stream_after(sd, st), "event");
    }
    struct Rejoin {
      cudaStream_t st, sd;
      ~Rejoin() {
        if (sd != st && stream_after(st, sd) != cudaSuccess) cudaStreamSynchronize(sd);
      }
    } rejoin{st, sd};
    if (fused) {
      // score + DP per (doc, band) item in one kernel (bm_band.cu)
      BandArgs a;
      a.S = *sent;
      a.D = D;
      a.M = M;
      a.mt = mt;
      a.hits = dv.hits;
      a.h_off = dv.h_off;
      a.pitch = dv.pitch;
      a.p = penalty;
      a.dirs = dv.dirs;
      a.dir_off = dv.dir_off;
      a.cost = cost_l;
      a.items = dv.items;
      a.n_items = (int)g.items.size();
      a.ticket = dv.ticket;
      a.bnd = dv.bnd;
      a.bnd_off = dv.bnd_off;
      const int m_max = *std::max_element(g.m.begin(), g.m.end());
      BM_CK(launch_band(a, m_max, sd), "mine_band_kernel");
    } else {
      NwArgs a;
      a.S = dv.S;
      a.s_off = dv.s_off;
      a.pitch = dv.pitch;
      a.n = dv.n;
      a.m = dv.m;
      a.p = penalty;
      a.dirs = dv.dirs;
      a.dir_off = dv.dir_off;
      a.cost = cost_l;
      a.items = dv.items;
      a.n_items = (int)g.items.size();
      a.ticket = dv.ticket;
      a.bnd = dv.bnd;
      a.bnd_off = dv.bnd_off;
      a.ready = ready;
      a.band_base = band_base;
      BM_CK(launch_nw(a, sd), "nw_band_kernel");
      if (overlap) {
        // the scoring kernel beside the DP; extraction reads S after both
        BM_CK(launch_score_hits(*sent, D, *lex, M, mt, nullptr, 0, dv.hits, dv.h_off, dv.tiles,
                                (int)g.tiles.size(), dv.s_off, dv.pitch, dv.S, st, ready, band_base),
              "score_hits_kernel");
        BM_CK(stream_after(sd, st), "event");
      }
    }
    tr.mark("nw enqueued");
    CellSrc cs;
    cs.S = dv.S;
    cs.s_off = dv.s_off;
    cs.sent = *sent;
    cs.D = D;
    cs.M = M;
    cs.hits = dv.hits;
    cs.h_off = dv.h_off;
    BM_CK(launch_extract(dv.dirs, dv.dir_off, cs, dv.pitch, dv.n, dv.m, k, threshold,
                         droff, rl, cl, sd, dskip),
          "extract_kernel");
    BM_CK(launch_extract_banded(dv.dirs, dv.dir_off, cs, dv.pitch, dv.n, dv.m, bx,
                                threshold, droff, rl, cl, sd),
          "band-parallel extraction");
    scatter_results_kernel<<<k, 128, 0, sd>>>(idx, k, cost_l, cost, rl, droff, cl, rec_off, rec,
                                              rec_count);
    BM_CK(cudaGetLastError(), "scatter_results");
    note_launch();
  }
  return BM_OK;
}

}  // namespace

extern "C" {

int bm_abi_version(void) { return BM_ABI_VERSION; }

int bm_trim(void) {
  for (Workspace& w : workspaces()) ws_release(w);
  workspaces().clear();
  return BM_OK;
}

const char* bm_last_error(void) { return g_err.c_str(); }

int bm_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int64_t bm_dirs_words(int32_t n, int32_t m) { return band_dirs_words(n, m); }

int64_t bm_launches(void) { return (int64_t)launches(); }

int bm_probe_fp64(double* out, int32_t iters, int32_t blocks, void* stream) {
  BM_CK(launch_fp64_probe(out, iters, blocks, (cudaStream_t)stream), "fp64_probe_kernel");
  return BM_OK;
}

int bm_score(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
             const int32_t* m_host, const bm_lexicon* lex, const bm_model* model,
             const int64_t* s_off, const int32_t* pitch, double* S, void* stream) {
  BM_CK(ensure_quot_table(), "quotient table");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int4> tiles;
  for (int d = 0; d < docs->n_docs; ++d)
    for (int r0 = 0; r0 < n_host[d]; r0 += kTile)
      for (int c0 = 0; c0 < m_host[d]; c0 += kTile) tiles.push_back(make_int4(d, r0, c0, 0));
  Scratch sc(st);
  int4* dt = nullptr;
  BM_CK(sc.upload(&dt, tiles), "upload tiles");
  BM_CK(launch_score(*sent, *docs, *lex, to_model(model), dt, (int)tiles.size(), s_off, pitch, S, st),
        "score_tile_kernel");
  return BM_OK;
}

int bm_features(const bm_sentences* sent, const bm_lexicon* lex, const int32_t* q_src,
                const int32_t* q_tgt, const double* q_pos_s, const double* q_pos_t, int32_t n_q,
                double* feats, void* stream) {
  BM_CK(ensure_quot_table(), "quotient table");
  BM_CK(launch_features(*sent, *lex, q_src, q_tgt, q_pos_s, q_pos_t, n_q, feats,
                        (cudaStream_t)stream),
        "features_kernel");
  return BM_OK;
}

int bm_confidence(const double* feats, int32_t n_q, const bm_model* model, double* conf,
                  void* stream) {
  BM_CK(launch_confidence(feats, n_q, to_model(model), conf, (cudaStream_t)stream),
        "confidence_kernel");
  return BM_OK;
}

int bm_nw(const double* S, const int64_t* s_off, const int32_t* pitch, const int32_t* n,
          const int32_t* m, const int32_t* n_host, const int32_t* m_host, int32_t n_docs,
          double penalty, uint32_t* dirs, const int64_t* dir_off, double* cost, void* stream) {
  if (!check_penalty(penalty)) return fail(BM_EINVAL, "penalty must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<WorkItem> items;
  std::vector<int64_t> bnd_off(n_docs);
  int64_t bt = 0;
  for (int d = 0; d < n_docs; ++d) {
    const int nb = (n_host[d] + kBandRows - 1) / kBandRows;
    bnd_off[d] = bt;
    bt += (int64_t)std::max(nb - 1, 0) * m_host[d];
    for (int b = 0; b < nb; ++b) items.push_back(WorkItem{d, b});
  }
  Scratch sc(st);
  NwArgs a;
  WorkItem* di = nullptr;
  int64_t* dbo = nullptr;
  BM_CK(sc.upload(&di, items), "upload");
  BM_CK(sc.upload(&dbo, bnd_off), "upload");
  double* bnd = nullptr;
  unsigned int* ticket = nullptr;
  BM_CK(sc.alloc(&bnd, (size_t)bt), "alloc");
  BM_CK(sc.alloc(&ticket, 1), "alloc");
  BM_CK(cudaMemsetAsync(ticket, 0, 4, st), "memset");
  BM_CK(cudaMemsetAsync(bnd, 0xde, std::max<int64_t>(bt, 1) * 8, st), "memset");
  a.S = S;
  a.s_off = s_off;
  a.pitch = pitch;
  a.n = n;
  a.m = m;
  a.p = penalty;
  a.dirs = dirs;
  a.dir_off = dir_off;
  a.cost = cost;
  a.items = di;
  a.n_items = (int)items.size();
  a.ticket = ticket;
  a.bnd = bnd;
  a.bnd_off = dbo;
  BM_CK(launch_nw(a, st), "nw_band_kernel");
  return BM_OK;
}

int bm_traceback(const uint32_t* dirs, const int64_t* dir_off, const int32_t* n, const int32_t* m,
                 int32_t n_docs, const int64_t* mv_off, int8_t* mv_op, int32_t* mv_i,
                 int32_t* mv_j, int32_t* mv_len, void* stream) {
  BM_CK(launch_traceback(dirs, dir_off, n, m, n_docs, mv_off, mv_op, mv_i, mv_j, mv_len,
                         (cudaStream_t)stream),
        "traceback_kernel");
  return BM_OK;
}

int bm_extract(const uint32_t* dirs, const int64_t* dir_off, const double* S, const int64_t* s_off,
               const int32_t* pitch, const int32_t* n, const int32_t* m, int32_t n_docs,
               double threshold, const int64_t* rec_off, bm_record* rec, int32_t* rec_count,
               void* stream) {
  if (S == nullptr && n_docs > 0) return fail(BM_EINVAL, "S is null");
  CellSrc cs;
  cs.S = S;
  cs.s_off = s_off;
  BM_CK(launch_extract(dirs, dir_off, cs, pitch, n, m, n_docs, threshold, rec_off, rec,
                       rec_count, (cudaStream_t)stream),
        "extract_kernel");
  return BM_OK;
}

int bm_select(const double* S, int64_t pitch, const int32_t* ci, const int32_t* cj, int32_t k,
              double threshold, double* conf, uint8_t* keep, void* stream) {
  BM_CK(launch_select(S, pitch, ci, cj, k, threshold, conf, keep, (cudaStream_t)stream),
        "select_kernel");
  return BM_OK;
}

// Extra compute streams of the calling thread: bm_mine_host deals chunks
// round-robin over the caller's stream and these, so a chunk's kernel tails
// overlap the next chunks' kernels.
static cudaStream_t side_stream(int q) {
  static thread_local cudaStream_t s[kMaxMineStreams] = {};
  static thread_local int dev_of = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_of != dev) {
    for (auto& x : s) x = nullptr;
    dev_of = dev;
  }
  if (s[q] == nullptr) cudaStreamCreateWithFlags(&s[q], cudaStreamNonBlocking);
  return s[q];
}

// Ring-kernel shared-memory buckets (bytes of a document's slice): 9 / 7 / 5 /
// 3 / fewer CTAs per SM. BM_RING_BUCKETS=0: one launch per R (a launch's slice is its
// largest document's).
constexpr int kRingSmemBuckets = 5;
static int ring_smem_bucket(size_t sl) {
  static const bool on = getenv("BM_RING_BUCKETS") ? atoi(getenv("BM_RING_BUCKETS")) != 0 : true;
  if (!on) return kRingSmemBuckets - 1;
  return sl <= 24 * 1024 ? 0 : sl <= 32 * 1024 ? 1 : sl <= 44 * 1024 ? 2 : sl <= 64 * 1024 ? 3 : 4;
}

// Fused banded tier (bm_band.cu) routing, opt-in: BM_BAND_FUSED=1 sends the
// banded documents whose sentences fit the folded tables there instead of
// score_hits_kernel -> nw_band_kernel. Measured on C3 200k:
// 70.6 ms fused vs 68.5 ms unfused -- the fused kernel issues at ~45-50 %
// against score_hits' 67 %, which the saved S round trip does not make up.
// BM_BAND_MIN_ITEMS: (doc, band) items a group needs for the fused tier
// (default 4 per SM: fewer bands leave the scoring warps idle; C4's 64 bands
// ran 2.9 -> 9 ms fused).
static bool band_fused_on() {
  static const bool v = getenv("BM_BAND_FUSED") ? atoi(getenv("BM_BAND_FUSED")) != 0 : false;
  return v;
}
static int64_t band_fused_min_items() {
  static const int64_t v = getenv("BM_BAND_MIN_ITEMS") ? atoll(getenv("BM_BAND_MIN_ITEMS")) : 4 * 148;
  return v;
}

// Documents per bm_mine group: consecutive documents up to this many cells
// share one routing pass and one set of scratch buffers (2 B/cell of hit
// counts for the fused tier, 4 + 8 B/cell for the banded tier), freed
// stream-ordered before the next group allocates, so any batch size fits.
static int64_t mine_group_cells() {
  static const int64_t v =
      getenv("BM_GROUP_CELLS") ? atoll(getenv("BM_GROUP_CELLS")) : (int64_t)1 << 30;
  return std::max<int64_t>(v, 1);
}

// One group: the fused tier's kernels on stream sf, the banded tier's on sb
// (bm_mine rotates groups over its streams, so one group's latency-bound DP
// runs next to another's issue-bound scoring).
static int mine_group(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
               const int32_t* m_host, const int32_t* amax_host, const bm_lexicon* lex,
               const Model& M, double threshold, double penalty, const int64_t* rec_off,
               bm_record* rec, int32_t* rec_count, double* cost, int d_lo, int d_hi,
               HostTrace& tr, cudaStream_t sf, cudaStream_t sb) {
  // fused tier: one launch per (rows per lane R, shared-memory bucket): a
  // launch's slice is its largest document's, so a few documents with large
  // hit-count matrices would otherwise cut every CTA of the class to 3 per SM
  constexpr int kNB = kRingSmemBuckets;
  std::vector<int32_t> fused[4 * kNB];
  size_t fused_smem[4 * kNB] = {}, hits_smem[4 * kNB] = {};
  std::vector<int64_t> hit_off;  // per document of [d_lo, d_hi)
  int64_t hit_total = 0;
  std::vector<int32_t> banded;  // planned after the fused tier is launched
  // BM_ROUTE=banded forces every document onto the K1 -> K2/K3 -> K4 tier
  // (benchmarking / testing both tiers on the same workload).
  const char* route = getenv("BM_ROUTE");
  const bool force_banded = route != nullptr && strcmp(route, "banded") == 0;
  hit_off.assign((size_t)(d_hi - d_lo), 0);
  int pn = -1, pm = -1, pq = -1;  // the last shape's class (batches repeat shapes)
  size_t sl = 0, hs = 0;
  for (int d = d_lo; d < d_hi; ++d) {
    const int n = n_host[d], m = m_host[d];
    if (n <= 0 || m <= 0) continue;
    if (n != pn || m != pm) {
      const int R = fused_rows_per_lane(n);
      sl = ring_slice_bytes(n, m, R);
      hs = hits_kernel_smem(n, m);
      pq = (!force_banded && n <= kFusedMaxRows && sl <= fused_max_smem())
               ? (R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3)
               : -1;
      pn = n;
      pm = m;
    }
    if (pq >= 0 && amax_host[d] <= 255) {
      const int q = pq;
      const int qq = q * kNB + ring_smem_bucket(sl);
      fused[qq].push_back(d);
      fused_smem[qq] = std::max(fused_smem[qq], sl);
      hits_smem[qq] = std::max(hits_smem[qq], hs);
      hit_off[d - d_lo] = hit_total;
      hit_total += (int64_t)align16(((size_t)n * m + 1) / 2 * 4);
    } else {
      banded.push_back(d);
    }
  }
  tr.mark("route");
  Scratch sc(sf), scb(sb);
  cudaStream_t st = sf;
  if (hit_total > 0) {
    uint8_t* hits = nullptr;
    int64_t* dho = nullptr;
    if (!BM_RING_FUSED_JOIN) {
      BM_CK(ws_get(st, kWsHits16, &hits, (size_t)hit_total), "alloc hits");
      BM_CK(cudaMemsetAsync(hits, 0, (size_t)hit_total, st), "memset hits");
      BM_CK(sc.upload(&dho, hit_off), "upload");
      tr.mark("alloc hits");
    }
    // per rows-per-lane class: one hits_kernel over all of its documents,
    // then one ring launch per shared-memory bucket (a sub-range of the list)
    for (int c = 0; c < 4; ++c) {
      std::vector<int32_t> all;
      int boff[kNB + 1];
      size_t hs = 0;
      for (int b = 0; b < kNB; ++b) {
        boff[b] = (int)all.size();
        all.insert(all.end(), fused[c * kNB + b].begin(), fused[c * kNB + b].end());
        hs = std::max(hs, hits_smem[c * kNB + b]);
      }
      boff[kNB] = (int)all.size();
      if (all.empty()) continue;
      int32_t* list = nullptr;
      BM_CK(sc.upload(&list, all), "upload");
      FusedArgs a;
      a.S = *sent;
      a.D = *docs;
      a.L = *lex;
      a.M = M;
      a.threshold = threshold;
      a.p = penalty;
      a.list = list;
      a.n_list = (int)all.size();
      a.rec_off = rec_off;
      a.rec = rec;
      a.rec_count = rec_count;
      a.cost = cost;
      a.hits = hits;
      a.hit_off = dho - d_lo;  // indexed by the batch's document index
      a.tabs = pair_tables();
      BM_CK(model_tables(M, &a.mt), "model tables");
      if (!BM_RING_FUSED_JOIN) BM_CK(launch_hits(a, hs, st), "hits_kernel");
      for (int b = 0; b < kNB; ++b) {
        if (boff[b + 1] == boff[b]) continue;
        a.list = list + boff[b];
        a.n_list = boff[b + 1] - boff[b];
        BM_CK(launch_ring(a, 1 << c, fused_smem[c * kNB + b], st), "mine_ring_kernel");
      }
      tr.mark("launch fused tier");
    }
  }
  // banded tier: the document-level join keeps 16-bit hit counts (every
  // sentence <= 65535 tokens); longer sentences take the per-tile scoring
  // kernel with 32-bit counts
  // every sentence <= 255 tokens (the folded tables' range): the fused banded
  // tier (bm_band.cu) when the group has enough bands to fill the GPU with its
  // CTAs; a few long documents (C4) keep the unfused tier, whose DP runs a
  // warp per band without waiting on 4 scoring warps per band
  GeneralPlan gf, g, gw;
  for (int32_t d : banded) {
    const int32_t md = m_host[d];
    GeneralPlan& t = amax_host[d] > 65535 ? gw
                     : (!band_fused_on() || amax_host[d] > 255 || md > 65535) ? g
                     : gf;
    t.add(d, n_host[d], md);
  }
  if (!gf.docs.empty() && (int64_t)gf.items.size() < band_fused_min_items()) {
    for (size_t q = 0; q < gf.docs.size(); ++q) g.add(gf.docs[q], gf.n[q], gf.m[q]);
    gf = GeneralPlan();
  }
  for (GeneralPlan* gp : {&gf, &g, &gw}) {
    if (gp->docs.empty()) continue;
    int rc = mine_general(*gp, sent, docs, lex, M, threshold, penalty, rec_off, rec, rec_count,
                          cost, gp != &gw, scb, sb, gp == &gf);
    if (rc) return rc;
    tr.mark("banded tier enqueued");
  }
  return BM_OK;
}

int bm_mine(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
            const int32_t* m_host, const int32_t* amax_host, const bm_lexicon* lex,
            const bm_model* model, double threshold, double penalty, const int64_t* rec_off,
            bm_record* rec, int32_t* rec_count, double* cost, void* stream) {
  BM_CK(ensure_quot_table(), "quotient table");
  if (!check_penalty(penalty)) return fail(BM_EINVAL, "penalty must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  HostTrace tr("bm_mine");
  const int nd = docs->n_docs;
  BM_CK(cudaMemsetAsync(rec_count, 0, std::max(nd, 1) * sizeof(int32_t), st), "memset");
  const Model M = to_model(model);
  const int64_t budget = mine_group_cells();
  // the caller's stream and two side streams take the groups' tiers in turn;
  // every side stream starts after the memset and is joined back into st on
  // every exit path (before the per-group scratch on it is reused)
  cudaStream_t ss[3] = {st, side_stream(1), side_stream(2)};
  struct Join {
    cudaStream_t st;
    cudaStream_t* side;
    ~Join() {
      for (int q = 1; q < 3; ++q) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventRecord(e, side[q]) == cudaSuccess && cudaStreamWaitEvent(st, e, 0) == cudaSuccess)
          cudaEventDestroy(e);
        else
          cudaStreamSynchronize(side[q]);
      }
    }
  } join{st, ss};
  {
    cudaEvent_t e0;
    BM_CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming), "event");
    BM_CK(cudaEventRecord(e0, st), "event");
    BM_CK(cudaStreamWaitEvent(ss[1], e0, 0), "event");
    BM_CK(cudaStreamWaitEvent(ss[2], e0, 0), "event");
    cudaEventDestroy(e0);
  }
  // BM_TRACE: GPU timeline of the groups (both tiers done, relative to the start)
  cudaEvent_t tl0 = nullptr;
  std::vector<cudaEvent_t> tl_a, tl_b;
  if (tr.on) {
    cudaEventCreate(&tl0);
    cudaEventRecord(tl0, st);
  }
  int unit = 0;
  for (int d0 = 0; d0 < nd;) {
    int d1 = d0;
    int64_t cells = 0;
    while (d1 < nd && (d1 == d0 || cells + (int64_t)n_host[d1] * m_host[d1] <= budget))
      cells += (int64_t)n_host[d1] * m_host[d1], ++d1;
    int rc = mine_group(sent, docs, n_host, m_host, amax_host, lex, M, threshold, penalty,
                        rec_off, rec, rec_count, cost, d0, d1, tr, ss[unit % 3],
                        ss[(unit + 1) % 3]);
    if (rc) return rc;
    if (tr.on) {
      cudaEvent_t ea, eb;
      cudaEventCreate(&ea);
      cudaEventCreate(&eb);
      cudaEventRecord(ea, ss[unit % 3]);
      cudaEventRecord(eb, ss[(unit + 1) % 3]);
      tl_a.push_back(ea);
      tl_b.push_back(eb);
    }
    unit += 2;
    d0 = d1;
  }
  if (tr.on) {
    tr.mark("groups enqueued");
    cudaDeviceSynchronize();
    for (size_t q = 0; q < tl_a.size(); ++q) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, tl0, tl_a[q]);
      cudaEventElapsedTime(&b, tl0, tl_b[q]);
      fprintf(stderr, "[bm trace] gpu group %2zu  fused tier %8.3f ms  banded tier %8.3f ms\n", q, a, b);
      cudaEventDestroy(tl_a[q]);
      cudaEventDestroy(tl_b[q]);
    }
    cudaEventDestroy(tl0);
  }
  return BM_OK;
}

int bm_compact(const bm_record* rec, const int64_t* rec_off, const int32_t* rec_count,
               int32_t n_docs, bm_record* dense, int64_t* total, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc(st);
  int64_t *doff = nullptr, *bsum = nullptr;
  BM_CK(sc.alloc(&doff, n_docs), "alloc");
  BM_CK(sc.alloc(&bsum, scan_scratch_count(n_docs)), "alloc");
  BM_CK(launch_compact(rec, rec_off, rec_count, n_docs, doff, total, dense, bsum, st), "compact");
  return BM_OK;
}

int bm_merge_bidir(const bm_record* fwd, int64_t n_fwd, const bm_record* bwd, int64_t n_bwd,
                   int32_t n_docs, const int32_t* src0, const int32_t* tgt0,
                   const int32_t* norm_key, const uint8_t* swap_f, const uint8_t* swap_b,
                   bm_record* out, int64_t* total, void* stream) {
  if (n_docs < 0 || n_fwd < 0 || n_bwd < 0) return fail(BM_EINVAL, "bad merge sizes");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_docs == 0) {
    BM_CK(cudaMemsetAsync(total, 0, sizeof(int64_t), st), "memset");
    return BM_OK;
  }
  Scratch sc(st);
  const int64_t k = n_fwd + n_bwd;
  MergeArgs a;
  int64_t *f_off = nullptr, *b_off = nullptr, *out_off = nullptr, *win = nullptr, *bsum = nullptr,
          *dense_off = nullptr;
  uint64_t *skey = nullptr, *sconf = nullptr;
  uint32_t *srank = nullptr, *rslot = nullptr;
  bm_record* tmp = nullptr;
  int32_t* cnt = nullptr;
  BM_CK(sc.alloc(&f_off, (size_t)n_docs + 1), "alloc");
  BM_CK(sc.alloc(&b_off, (size_t)n_docs + 1), "alloc");
  BM_CK(sc.alloc(&out_off, (size_t)n_docs), "alloc");
  BM_CK(sc.alloc(&skey, 4 * (size_t)k), "alloc");
  BM_CK(sc.alloc(&sconf, 4 * (size_t)k), "alloc");
  BM_CK(sc.alloc(&srank, 4 * (size_t)k), "alloc");
  BM_CK(sc.alloc(&rslot, (size_t)k), "alloc");
  BM_CK(sc.alloc(&win, (size_t)k), "alloc");
  BM_CK(sc.alloc(&tmp, (size_t)k), "alloc");
  BM_CK(sc.alloc(&cnt, (size_t)n_docs), "alloc");
  BM_CK(sc.alloc(&dense_off, (size_t)n_docs), "alloc");
  BM_CK(sc.alloc(&bsum, scan_scratch_count(n_docs)), "alloc");
  BM_CK(launch_doc_offsets(fwd, n_fwd, n_docs, f_off, st), "doc_offsets");
  BM_CK(launch_doc_offsets(bwd, n_bwd, n_docs, b_off, st), "doc_offsets");
  a.fwd = fwd;
  a.bwd = bwd;
  a.f_off = f_off;
  a.b_off = b_off;
  a.src0 = src0;
  a.tgt0 = tgt0;
  a.norm_key = norm_key;
  a.swap_f = swap_f;
  a.swap_b = swap_b;
  a.n_docs = n_docs;
  a.slot_key = skey;
  a.slot_conf = sconf;
  a.slot_rank = srank;
  a.rec_slot = rslot;
  a.win_ij = win;
  a.out = tmp;
  a.out_cnt = cnt;
  a.out_off = out_off;
  BM_CK(launch_merge_bidir(a, st), "merge_bidir_kernel");
  BM_CK(launch_compact(tmp, out_off, cnt, n_docs, dense_off, total, out, bsum, st), "compact");
  return BM_OK;
}

int bm_merge_shards(const bm_record* rec, int64_t stride, const int64_t* part_len, int32_t world,
                    int32_t n_docs, bm_record* out, int64_t* total, void* stream) {
  if (world < 1 || stride < 0 || n_docs < 0) return fail(BM_EINVAL, "bad shard layout");
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc(st);
  int32_t* counts = nullptr;
  int64_t *src_start = nullptr, *goff = nullptr, *bsum = nullptr;
  BM_CK(sc.alloc(&counts, n_docs), "alloc");
  BM_CK(sc.alloc(&src_start, n_docs), "alloc");
  BM_CK(sc.alloc(&goff, n_docs), "alloc");
  BM_CK(sc.alloc(&bsum, scan_scratch_count(n_docs)), "alloc");
  BM_CK(launch_merge_shards(rec, stride, part_len, world, n_docs, counts, src_start, goff, total,
                            bsum, out, st),
        "merge_shards");
  return BM_OK;
}

// Copy stream of the calling thread on the current device (H2D of chunk k+1
// overlaps the kernels of chunk k in bm_mine_host).
static cudaStream_t copy_stream() {
  static thread_local cudaStream_t s = nullptr;
  static thread_local int dev_of = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (s == nullptr || dev_of != dev) {
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    dev_of = dev;
  }
  return s;
}

// Page-locked per-chunk record counts of the calling thread (grown on demand).
static int64_t* pinned_counts(size_t n) {
  static thread_local int64_t* buf = nullptr;
  static thread_local size_t cap = 0;
  if (n > cap) {
    if (buf) cudaFreeHost(buf);
    cap = std::max<size_t>(n, 256);
    if (cudaHostAlloc((void**)&buf, cap * sizeof(int64_t), cudaHostAllocDefault) != cudaSuccess) {
      buf = nullptr;
      cap = 0;
    }
  }
  return buf;
}

// Host source of a streamed batch: either the plain bm_sentences arrays or the
// compact wire format (narrow types, widened on the device per chunk).
struct HostSource {
  int32_t n_sent;
  const int32_t* tok_off;  // host, [n_sent + 1]
  const int32_t* dig_off;  // host, [n_sent + 1]
  const bm_sentences* full;
  const bm_wire* wire;
  const bm_wire_packed* pk = nullptr;
  int32_t tok_max(int k) const {
    return full ? full->n_tok[k] : wire ? (int32_t)wire->n_tok[k] : (int32_t)(pk->counts[k] & 0xff);
  }
};

static int mine_host_impl(const HostSource& src, const bm_docs* dh, const bm_lexicon* lh,
                   const bm_model* model, double threshold, double penalty, bm_record* rec_out,
                   int64_t rec_cap, int64_t* n_rec, double* cost_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  HostTrace tr("bm_mine_host");
  BM_CK(ensure_quot_table(), "device init");
  cudaStream_t cs = copy_stream();
  const int ns = src.n_sent, nd = dh->n_docs;
  const int64_t ne = ns ? src.tok_off[ns] : 0;
  const int64_t ndig = ns ? src.dig_off[ns] : 0;
  const int nid = lh->n_ids;
  // routing input: per-doc max token count; one vectorisable pass decides
  // whether any document can exceed the fused kernel's 8-bit counters at all
  int32_t gmax = 0;
  if (src.full) {
    for (int k = 0; k < ns; ++k) gmax = std::max(gmax, src.full->n_tok[k]);
  }
  std::vector<int32_t> amax(nd, 0);
  if (gmax > 255) {
    for (int d = 0; d < nd; ++d) {
      int v = 0;
      for (int k = 0; k < dh->n[d]; ++k) v = std::max(v, src.tok_max(dh->src0[d] + k));
      for (int k = 0; k < dh->m[d]; ++k) v = std::max(v, src.tok_max(dh->tgt0[d] + k));
      amax[d] = v;
    }
  }
  std::vector<int64_t> roff(nd);
  int64_t rt = 0;
  for (int d = 0; d < nd; ++d) {
    roff[d] = rt;
    rt += std::max(0, std::min(dh->n[d], dh->m[d]));
  }
  if (!check_penalty(penalty)) return fail(BM_EINVAL, "penalty must be >= 0");
  tr.mark("host prep");
  Scratch sc(st);
  // declared after the scratch, so destroyed before it: an early return never
  // frees scratch (stream-ordered on st) under copies still queued on cs
  struct CopyFence {
    cudaStream_t s;
    ~CopyFence() { cudaStreamSynchronize(s); }
  } fence{cs};
  // Every exit path (early error returns included) joins the side mining
  // streams back into st before ~Scratch frees on st: their queued kernels
  // still read and write the scratch. Declared after the scratch, so it runs
  // first; the events it and the chunk loop create are released on exit.
  struct StreamJoin {
    cudaStream_t st;
    std::vector<cudaStream_t> side;
    std::vector<cudaEvent_t> events;
    cudaEvent_t event() {
      cudaEvent_t e = nullptr;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
      events.push_back(e);
      return e;
    }
    cudaError_t join() {
      cudaError_t err = cudaSuccess;
      for (cudaStream_t s : side) {
        cudaEvent_t e = event();
        cudaError_t r = e ? cudaEventRecord(e, s) : cudaErrorMemoryAllocation;
        if (r == cudaSuccess) r = cudaStreamWaitEvent(st, e, 0);
        if (r != cudaSuccess) {
          cudaStreamSynchronize(s);  // cannot order it: wait for it instead
          if (err == cudaSuccess) err = r;
        }
      }
      side.clear();
      return err;
    }
    ~StreamJoin() {
      join();
      for (cudaEvent_t e : events) cudaEventDestroy(e);
    }
  } joiner{st, {}, {}};
  bm_sentences sd;
  sd.n_sent = ns;
  int32_t *a0, *a1, *a2, *a3, *a4, *a5, *a6;
  uint32_t* a7;
  BM_CK(sc.alloc(&a0, ns), "alloc");
  BM_CK(sc.alloc(&a1, ns), "alloc");
  BM_CK(sc.alloc(&a2, ns), "alloc");
  BM_CK(sc.alloc(&a3, ns + 1), "alloc");
  BM_CK(sc.alloc(&a4, ne), "alloc");
  BM_CK(sc.alloc(&a7, ne), "alloc");
  BM_CK(sc.alloc(&a5, ns + 1), "alloc");
  BM_CK(sc.alloc(&a6, ndig), "alloc");
  sd.n_tok = a0;
  sd.n_punct = a1;
  sd.n_alpha = a2;
  sd.tok_off = a3;
  sd.tok_id = a4;
  sd.tok_alpha = a7;
  sd.dig_off = a5;
  sd.dig_id = a6;
  // device staging of the narrow wire arrays
  uint8_t *w_t = nullptr, *w_p = nullptr, *w_a = nullptr, *w_al = nullptr;
  uint16_t *w_id = nullptr, *w_dg = nullptr;
  uint32_t* w_cnt = nullptr;
  int32_t *w_o32 = nullptr, *w_d32 = nullptr;
  if (src.pk) {
    BM_CK(sc.alloc(&w_cnt, ns), "alloc");
    BM_CK(sc.alloc(&w_o32, ns / 32 + 1), "alloc");
    BM_CK(sc.alloc(&w_d32, ns / 32 + 1), "alloc");
    BM_CK(sc.alloc(&w_id, ne), "alloc");
    BM_CK(sc.alloc(&w_dg, ndig), "alloc");
  }
  if (src.wire) {
    BM_CK(sc.alloc(&w_t, ns), "alloc");
    BM_CK(sc.alloc(&w_p, ns), "alloc");
    BM_CK(sc.alloc(&w_a, ns), "alloc");
    BM_CK(sc.alloc(&w_id, ne), "alloc");
    BM_CK(sc.alloc(&w_al, ne), "alloc");
    BM_CK(sc.alloc(&w_dg, ndig), "alloc");
  }
  bm_docs dd;
  dd.n_docs = nd;
  int32_t *b0, *b1, *b2, *b3;
  BM_CK(sc.alloc(&b0, nd), "alloc");
  BM_CK(sc.alloc(&b1, nd), "alloc");
  BM_CK(sc.alloc(&b2, nd), "alloc");
  BM_CK(sc.alloc(&b3, nd), "alloc");
  dd.src0 = b0;
  dd.n = b1;
  dd.tgt0 = b2;
  dd.m = b3;
  bm_lexicon ld;
  ld.n_ids = nid;
  int32_t *c0, *c1, *c2, *c3;
  const int64_t nf = nid ? lh->fwd_off[nid] : 0, nr = nid ? lh->rev_off[nid] : 0;
  BM_CK(sc.alloc(&c0, nid + 1), "alloc");
  BM_CK(sc.alloc(&c1, nf), "alloc");
  BM_CK(sc.alloc(&c2, nid + 1), "alloc");
  BM_CK(sc.alloc(&c3, nr), "alloc");
  ld.fwd_off = c0;
  ld.fwd_cand = c1;
  ld.rev_off = c2;
  ld.rev_cand = c3;
  int64_t* droff = nullptr;
  bm_record *rec = nullptr, *dense = nullptr;
  int32_t* cnt = nullptr;
  double* cost = nullptr;
  BM_CK(sc.alloc(&droff, nd), "alloc");
  BM_CK(sc.alloc(&rec, (size_t)rt), "alloc");
  BM_CK(sc.alloc(&dense, (size_t)rt), "alloc");
  BM_CK(sc.alloc(&cnt, nd), "alloc");
  BM_CK(sc.alloc(&cost, nd), "alloc");
  int64_t* doff = nullptr;
  BM_CK(sc.alloc(&doff, nd), "alloc");
  // chunk count upper bound: every chunk but the last holds >= 1 document
  int64_t* ctot = nullptr;
  BM_CK(sc.alloc(&ctot, nd + 1), "alloc");
  int64_t* bsum_all = nullptr;  // per-chunk scan scratch (see enqueue_kernels)
  BM_CK(sc.alloc(&bsum_all, 2 * (size_t)nd + 2), "alloc");
  tr.mark("allocs");
  int64_t* hcnt = pinned_counts((size_t)nd + 1);
  if (hcnt == nullptr) return fail(BM_ENOMEM, "pinned count buffer");
  // the copy stream may only touch the scratch once it is allocated on st
  cudaEvent_t ready = joiner.event();
  if (ready == nullptr) return fail(BM_ECUDA, "event create failed");
  BM_CK(cudaEventRecord(ready, st), "event");
  BM_CK(cudaStreamWaitEvent(cs, ready, 0), "event");
  auto h2d = [&](void* dst, const void* from, size_t bytes) -> cudaError_t {
    return bytes ? cudaMemcpyAsync(dst, from, bytes, cudaMemcpyHostToDevice, cs) : cudaSuccess;
  };
  BM_CK(h2d(c0, lh->fwd_off, (nid + 1) * 4), "h2d");
  BM_CK(h2d(c1, lh->fwd_cand, nf * 4), "h2d");
  BM_CK(h2d(c2, lh->rev_off, (nid + 1) * 4), "h2d");
  BM_CK(h2d(c3, lh->rev_cand, nr * 4), "h2d");
  BM_CK(h2d(droff, roff.data(), nd * 8), "h2d");
  BM_CK(h2d(b0, dh->src0, nd * 4), "h2d");
  BM_CK(h2d(b1, dh->n, nd * 4), "h2d");
  BM_CK(h2d(b2, dh->tgt0, nd * 4), "h2d");
  BM_CK(h2d(b3, dh->m, nd * 4), "h2d");
  tr.mark("alloc + small h2d");
  // chunks of documents: H2D the sentence range each chunk touches on the
  // copy stream, mine it on the compute stream once its copy event fired
  // (16M cells per chunk; large batches use ~16 chunks of at most
  // mine_group_cells(): a chunk's banded DP must hold enough (doc, band) items
  // for its persistent grid -- C3 200k in 64 chunks took 181 ms, in groups 75)
  int64_t all_cells = 0;
  for (int d = 0; d < nd; ++d) all_cells += (int64_t)dh->n[d] * dh->m[d];
  static const int64_t kChunkEnv = getenv("BM_CHUNK_CELLS") ? atoll(getenv("BM_CHUNK_CELLS")) : 0;
  const int64_t kChunkCells =
      kChunkEnv > 0 ? kChunkEnv
                    : std::min(mine_group_cells(), std::max<int64_t>(16ll << 20, all_cells / 16));
  static const int64_t kFirstEnv =
      getenv("BM_FIRST_CHUNK_CELLS") ? atoll(getenv("BM_FIRST_CHUNK_CELLS")) : 0;
  const int64_t kFirstChunkCells = kFirstEnv > 0 ? kFirstEnv : (4ll << 20);
  // per chunk: docs [d0, d1), compacted into dense + roff[d0], count -> ctot[k]
  std::vector<int> ch_d0, ch_d1;
  std::vector<cudaEvent_t> ch_ev;
  // BM_TRACE: GPU timeline (copy done / mined per chunk, relative to t_start)
  std::vector<cudaEvent_t> tl_copy, tl_mine, tl_start, tl_fused;
  cudaEvent_t tl0 = nullptr;
  if (tr.on) {
    cudaEventCreate(&tl0);
    cudaEventRecord(tl0, cs);
  }
  // pass 1: the chunks' bulk copies (kernels wait on each chunk's copy event).
  // Chunk 0 goes first so its DMA overlaps the routing below; the rest follow
  // the small list uploads, which would otherwise queue behind the bulk DMA.
  struct Chunk {
    int d0, d1, lo, hi;
    cudaEvent_t copied;
  };
  std::vector<Chunk> chunks;
  int d0 = 0;
  auto enqueue_copies = [&](size_t upto) -> int {
    while (d0 < nd && chunks.size() < upto) {
      int d1 = d0;
      int64_t cells = 0;
      int lo = ns, hi = 0;
      // a small first chunk starts the GPU early; later chunks amortise launches
      const int64_t want = chunks.empty() ? kFirstChunkCells : kChunkCells;
      while (d1 < nd && (d1 == d0 || cells < want)) {
        cells += (int64_t)dh->n[d1] * dh->m[d1];
        if (dh->n[d1] > 0) {
          lo = std::min(lo, dh->src0[d1]);
          hi = std::max(hi, dh->src0[d1] + dh->n[d1]);
        }
        if (dh->m[d1] > 0) {
          lo = std::min(lo, dh->tgt0[d1]);
          hi = std::max(hi, dh->tgt0[d1] + dh->m[d1]);
        }
        ++d1;
      }
      if (hi > lo) {
        const int64_t e0 = src.tok_off[lo], e1 = src.tok_off[hi];
        const int64_t g0 = src.dig_off[lo], g1 = src.dig_off[hi];
        const size_t cntS = (size_t)(hi - lo);
        if (src.pk) {
          // counts from the chunk's first 32-sentence block, bases through hi's
          const bm_wire_packed* w = src.pk;
          const int l32 = lo & ~31;
          BM_CK(h2d(w_cnt + l32, w->counts + l32, (size_t)(hi - l32) * 4), "h2d");
          BM_CK(h2d(w_o32 + (lo >> 5), w->tok_off32 + (lo >> 5), (size_t)((hi >> 5) - (lo >> 5) + 1) * 4), "h2d");
          BM_CK(h2d(w_d32 + (lo >> 5), w->dig_off32 + (lo >> 5), (size_t)((hi >> 5) - (lo >> 5) + 1) * 4), "h2d");
          BM_CK(h2d(w_id + e0, w->tok_pk + e0, (size_t)(e1 - e0) * 2), "h2d");
          BM_CK(h2d(w_dg + g0, w->dig_id + g0, (size_t)(g1 - g0) * 2), "h2d");
        } else {
          BM_CK(h2d(a3 + lo, src.tok_off + lo, (cntS + 1) * 4), "h2d");
          BM_CK(h2d(a5 + lo, src.dig_off + lo, (cntS + 1) * 4), "h2d");
        }
        if (src.full) {
          const bm_sentences* sh = src.full;
          BM_CK(h2d(a0 + lo, sh->n_tok + lo, cntS * 4), "h2d");
          BM_CK(h2d(a1 + lo, sh->n_punct + lo, cntS * 4), "h2d");
          BM_CK(h2d(a2 + lo, sh->n_alpha + lo, cntS * 4), "h2d");
          BM_CK(h2d(a4 + e0, sh->tok_id + e0, (size_t)(e1 - e0) * 4), "h2d");
          BM_CK(h2d(a7 + e0, sh->tok_alpha + e0, (size_t)(e1 - e0) * 4), "h2d");
          BM_CK(h2d(a6 + g0, sh->dig_id + g0, (size_t)(g1 - g0) * 4), "h2d");
        } else if (src.wire) {
          const bm_wire* w = src.wire;
          BM_CK(h2d(w_t + lo, w->n_tok + lo, cntS), "h2d");
          BM_CK(h2d(w_p + lo, w->n_punct + lo, cntS), "h2d");
          BM_CK(h2d(w_a + lo, w->n_alpha + lo, cntS), "h2d");
          BM_CK(h2d(w_id + e0, w->tok_id + e0, (size_t)(e1 - e0) * 2), "h2d");
          BM_CK(h2d(w_al + e0, w->tok_alpha + e0, (size_t)(e1 - e0)), "h2d");
          BM_CK(h2d(w_dg + g0, w->dig_id + g0, (size_t)(g1 - g0) * 2), "h2d");
        }
      }
      cudaEvent_t ev = joiner.event();
      if (ev == nullptr) return fail(BM_ECUDA, "event create failed");
      BM_CK(cudaEventRecord(ev, cs), "event");
      if (tr.on) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, cs);
        tl_copy.push_back(e);
      }
      chunks.push_back(Chunk{d0, d1, lo, hi, ev});
      d0 = d1;
    }
    return BM_OK;
  };
  if (int rc = enqueue_copies(1)) return rc;
  tr.mark("chunk 0 copies enqueued");
  // the chunks are mined like bm_mine's groups (mine_group: routing, fused
  // tier on one stream, banded tier on the next), rotating over the mining
  // streams, each chunk once its copies have landed
  const Model M = to_model(model);
  BM_CK(cudaMemsetAsync(cnt, 0, std::max(nd, 1) * sizeof(int32_t), st), "memset");
  {
    ModelTables mt;  // built (once per model and device) before any stream uses it
    BM_CK(model_tables(M, &mt), "model tables");
  }
  tr.mark("memsets");
  // the mining streams start after the memsets on st
  cudaEvent_t planned = joiner.event();
  if (planned == nullptr) return fail(BM_ECUDA, "event create failed");
  BM_CK(cudaEventRecord(planned, st), "event");
  static const int n_ms = std::max(1, std::min(kMaxMineStreams,
      getenv("BM_MINE_STREAMS") ? atoi(getenv("BM_MINE_STREAMS")) : 4));
  std::vector<cudaStream_t> ms(1, st);
  for (int q = 1; q < n_ms; ++q) {
    ms.push_back(side_stream(q));
    BM_CK(cudaStreamWaitEvent(ms.back(), planned, 0), "event");
    joiner.side.push_back(ms.back());
  }
  // pass 2: per chunk, widen + mine + compact on the mining streams; chunk 0's
  // kernels are enqueued before the remaining copies so the GPU starts early
  auto enqueue_kernels = [&](size_t kc) -> int {
    const int d0 = chunks[kc].d0, d1 = chunks[kc].d1, lo = chunks[kc].lo, hi = chunks[kc].hi;
    cudaEvent_t ev = chunks[kc].copied;
    // chunk k: fused tier on stream k + 1, banded tier on stream k + 3 (mod
    // the stream count): every stream takes fused tiers in turn, and a chunk's
    // fused tier queues behind the banded tier of the chunk two before it, not
    // the one just before (chunk 0 on a side stream). The chunk's compaction
    // follows its fused tier on the same stream once the banded tier is done.
    const size_t u = ch_d0.size() + 1;
    cudaStream_t sk = ms[u % ms.size()];
    cudaStream_t sb = ms.size() > 1 ? ms[(u + (ms.size() > 2 ? 2 : 1)) % ms.size()] : sk;
    cudaStream_t sc_ = sk, so_ = sb;
    BM_CK(cudaStreamWaitEvent(sk, ev, 0), "event");
    // the copy stream only moves bytes: widening the wire arrays is a few
    // microseconds of compute and runs in order on the compute stream (on the
    // copy stream it would queue behind the mining CTAs and stall the DMA)
    if (src.pk && hi > lo)
      BM_CK(launch_unpack_packed(w_cnt, w_o32, w_d32, w_id, w_dg, lo, hi, a0, a1, a2, a3, a4, a7,
                                 a5, a6, sk),
            "unpack_packed_kernel");
    if (src.wire && hi > lo) {
      const int64_t e0 = src.tok_off[lo], e1 = src.tok_off[hi];
      const int64_t g0 = src.dig_off[lo], g1 = src.dig_off[hi];
      BM_CK(launch_unpack_wire(w_t, w_p, w_a, w_id, w_al, w_dg, lo, hi, e0, e1, g0, g1, a0, a1,
                               a2, a4, a7, a6, sk),
            "unpack_wire_kernel");
    }
    if (sb != sk) {  // the banded tier starts once the chunk's arrays are ready
      cudaEvent_t ready_b = joiner.event();
      if (ready_b == nullptr) return fail(BM_ECUDA, "event create failed");
      BM_CK(cudaEventRecord(ready_b, sk), "event");
      BM_CK(cudaStreamWaitEvent(sb, ready_b, 0), "event");
    }
    if (tr.on) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, sk);
      tl_start.push_back(e);
    }
    {
      int rc = mine_group(&sd, &dd, dh->n, dh->m, amax.data(), &ld, M, threshold, penalty, droff,
                          rec, cnt, cost, d0, d1, tr, sk, sb);
      if (rc) return rc;
    }
    if (tr.on) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, sk);
      tl_fused.push_back(e);
    }
    if (sb != sk) {  // compaction after both tiers
      cudaEvent_t done_f = joiner.event();
      if (done_f == nullptr) return fail(BM_ECUDA, "event create failed");
      BM_CK(cudaEventRecord(done_f, so_), "event");
      BM_CK(cudaStreamWaitEvent(sc_, done_f, 0), "event");
    }
    // compact the chunk into its own region of `dense` (starting at its first
    // document's record slot) and fetch its record count; the host copies the
    // records out as soon as the count arrives, overlapping later chunks
    {
      const int kq = (int)ch_d0.size();
      // chunk kq's scan scratch: [d0 + kq, d1 + kq] (>= its block count + 1)
      BM_CK(launch_compact(rec, droff + d0, cnt + d0, d1 - d0, doff + d0, ctot + kq,
                           dense + roff[d0], bsum_all + d0 + kq, sc_, d0),
            "compact");
      BM_CK(cudaMemcpyAsync(hcnt + kq, ctot + kq, sizeof(int64_t), cudaMemcpyDeviceToHost, sc_),
            "d2h");
      cudaEvent_t ce = joiner.event();
      if (ce == nullptr) return fail(BM_ECUDA, "event create failed");
      BM_CK(cudaEventRecord(ce, sc_), "event");
      ch_d0.push_back(d0);
      ch_d1.push_back(d1);
      ch_ev.push_back(ce);
    }
    if (tr.on) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, sc_);
      tl_mine.push_back(e);
    }
    return BM_OK;
  };
  // the bulk copies run kCopyAhead chunks ahead of the kernels enqueued so
  // far: the copy engine serves H2D copies in submission order, so a chunk's
  // small plan uploads (on its mining stream) would otherwise queue behind all
  // of the batch's bulk copies (C3 1M: the first chunks' kernels waited ~70 ms)
  static const size_t kCopyAhead =
      getenv("BM_COPY_AHEAD") ? (size_t)atoll(getenv("BM_COPY_AHEAD")) : 1;
  if (int rc = enqueue_copies(1 + kCopyAhead)) return rc;
  if (int rc = enqueue_kernels(0)) return rc;
  for (size_t kc = 1; kc < chunks.size(); ++kc) {
    if (int rc = enqueue_copies(kc + 1 + kCopyAhead)) return rc;
    if (int rc = enqueue_kernels(kc)) return rc;
  }
  tr.mark("copies enqueued");
  // join the side streams back into the caller's stream
  BM_CK(joiner.join(), "stream join");
  tr.mark("chunks enqueued");
  int64_t tot = 0;
  for (size_t q = 0; q < ch_ev.size(); ++q) {
    BM_CK(cudaEventSynchronize(ch_ev[q]), "sync");
    const int64_t c = hcnt[q];
    if (tot + c > rec_cap) {
      cudaStreamSynchronize(cs);
      return fail(BM_ELIMIT, "record buffer too small");
    }
    if (c) BM_CK(cudaMemcpyAsync(rec_out + tot, dense + roff[ch_d0[q]], c * sizeof(bm_record),
                                 cudaMemcpyDeviceToHost, cs),
                 "d2h");
    tot += c;
  }
  tr.mark("mined + compacted");
  if (cost_out) BM_CK(cudaMemcpyAsync(cost_out, cost, nd * sizeof(double), cudaMemcpyDeviceToHost, st), "d2h");
  BM_CK(cudaStreamSynchronize(cs), "sync");
  BM_CK(cudaStreamSynchronize(st), "sync");
  tr.mark("records d2h");
  if (tr.on) {
    for (size_t q = 0; q < tl_copy.size(); ++q) {
      float a = 0.f, b = 0.f, c = 0.f, f = 0.f;
      cudaEventElapsedTime(&a, tl0, tl_copy[q]);
      cudaEventElapsedTime(&c, tl0, tl_start[q]);
      cudaEventElapsedTime(&f, tl0, tl_fused[q]);
      cudaEventElapsedTime(&b, tl0, tl_mine[q]);
      fprintf(stderr, "[bm trace] gpu chunk %2zu copied %8.3f ms  started %8.3f  fused %8.3f  mined %8.3f ms\n",
              q, a, c, f, b);
      cudaEventDestroy(tl_copy[q]);
      cudaEventDestroy(tl_mine[q]);
      cudaEventDestroy(tl_start[q]);
      cudaEventDestroy(tl_fused[q]);
    }
    cudaEventDestroy(tl0);
  }
  *n_rec = tot;
  return BM_OK;
}

int bm_mine_host(const bm_sentences* sh, const bm_docs* dh, const bm_lexicon* lh,
                 const bm_model* model, double threshold, double penalty, bm_record* rec_out,
                 int64_t rec_cap, int64_t* n_rec, double* cost_out, void* stream) {
  HostSource src{sh->n_sent, sh->tok_off, sh->dig_off, sh, nullptr};
  return mine_host_impl(src, dh, lh, model, threshold, penalty, rec_out, rec_cap, n_rec, cost_out,
                        stream);
}

int bm_mine_host_packed(const bm_wire_packed* ph, const bm_docs* dh, const bm_lexicon* lh,
                        const bm_model* model, double threshold, double penalty,
                        bm_record* rec_out, int64_t rec_cap, int64_t* n_rec, double* cost_out,
                        void* stream) {
  if (lh->n_ids > 16384) return fail(BM_EINVAL, "packed format: more than 16384 ids");
  HostSource src{ph->n_sent, ph->tok_off, ph->dig_off, nullptr, nullptr, ph};
  return mine_host_impl(src, dh, lh, model, threshold, penalty, rec_out, rec_cap, n_rec, cost_out,
                        stream);
}

int bm_mine_host_wire(const bm_wire* wh, const bm_docs* dh, const bm_lexicon* lh,
                      const bm_model* model, double threshold, double penalty, bm_record* rec_out,
                      int64_t rec_cap, int64_t* n_rec, double* cost_out, void* stream) {
  HostSource src{wh->n_sent, wh->tok_off, wh->dig_off, nullptr, wh};
  return mine_host_impl(src, dh, lh, model, threshold, penalty, rec_out, rec_cap, n_rec, cost_out,
                        stream);
}

int bm_tune(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
            const int32_t* m_host, const bm_lexicon* lex, const bm_model* model,
            const double* penalties_host, int32_t n_pen, const double* thresholds, int32_t n_thr,
            const int64_t* gold, const int64_t* gold_off, unsigned long long* pred,
            unsigned long long* hit, int32_t token_bound, void* stream) {
  BM_CK(ensure_quot_table(), "quotient table");
  cudaStream_t st = (cudaStream_t)stream;
  for (int k = 0; k < n_pen; ++k)
    if (!check_penalty(penalties_host[k])) return fail(BM_EINVAL, "penalty must be >= 0");
  if (n_thr > 64) return fail(BM_EINVAL, "at most 64 thresholds per call");
  GeneralPlan g;
  for (int d = 0; d < docs->n_docs; ++d) g.add(d, n_host[d], m_host[d]);
  Scratch sc(st);
  GeneralDev dv;
  int rc = general_prepare(g, docs, sc, dv, st);
  if (rc) return rc;
  const int k = (int)g.docs.size();
  const bm_docs D = local_docs(dv, k);
  rc = score_general(g, sent, D, lex, to_model(model), dv,
                     token_bound >= 0 && token_bound <= 65535, sc, st);
  if (rc) return rc;
  // Penalties run in passes of up to 4 (nw_band_kernel<D, NP>): one pass
  // stages S once for all of its penalties; each penalty has its own codes and
  // boundary rows. The pass width shrinks when the codes would not fit.
  int width = n_pen >= 4 ? 4 : n_pen >= 2 ? 2 : 1;
  const size_t dir_bytes = (size_t)std::max<int64_t>(g.dir_total, 1) * 4;
  while (width > 1 && (size_t)width * dir_bytes > ((size_t)16 << 30)) width /= 2;
  double* cost_l = nullptr;
  BM_CK(sc.alloc(&cost_l, (size_t)k * width), "alloc");
  uint32_t* dirs = dv.dirs;
  double* bnd = dv.bnd;
  const int64_t dstride = std::max<int64_t>(g.dir_total, 1), bstride = std::max<int64_t>(g.bnd_total, 1);
  if (width > 1) {
    BM_CK(sc.alloc(&dirs, (size_t)dstride * width), "alloc dirs");
    BM_CK(sc.alloc(&bnd, (size_t)bstride * width), "alloc boundary");
  }
  // single-band documents (n <= 128) run end to end in runs (nw_seq_kernel:
  // the wavefront's fill and drain once per run instead of once per
  // document); the others keep their (doc, band) items
  std::vector<int32_t> seq_off;  // (begin, end) plan indices per run
  std::vector<WorkItem> multi;
  if (nw_seq_on()) {
    int64_t single = 0;
    for (int q = 0; q < k; ++q) single += g.n[q] <= kBandRows;
    // about 4 runs per resident DP warp (8 per SM at 4 penalties): runs long
    // enough to amortise the fill, numerous enough to balance the warps
    // (BM_NW_SEQ_RUN, read per call: a fixed run length, for tests)
    const char* fr = getenv("BM_NW_SEQ_RUN");
    const int run = fr ? std::max(1, std::min(kSeqMaxDocs, atoi(fr)))
                       : (int)std::max<int64_t>(1, std::min<int64_t>(kSeqMaxDocs, single / (4 * 8 * 148)));
    for (int q = 0; q < k;) {
      if (g.n[q] > kBandRows) {
        ++q;
        continue;
      }
      const int q1 = q;
      while (q < k && q - q1 < run && g.n[q] <= kBandRows) ++q;
      seq_off.push_back(q1);
      seq_off.push_back(q);
    }
    for (const WorkItem& w : dv.order)
      if (g.n[w.doc] > kBandRows) multi.push_back(w);
  }
  int32_t* d_seq = nullptr;
  WorkItem* d_multi = nullptr;
  unsigned int* seq_ticket = nullptr;
  const int n_runs = (int)seq_off.size() / 2;
  if (n_runs > 0) {
    BM_CK(sc.upload(&d_seq, seq_off), "upload");
    BM_CK(sc.upload(&d_multi, multi), "upload");
    BM_CK(sc.alloc(&seq_ticket, 1), "alloc");
  }
  for (int q0 = 0; q0 < n_pen;) {
    int np = width;
    while (q0 + np > n_pen) np /= 2;
    BM_CK(cudaMemsetAsync(dv.ticket, 0, 4, st), "memset");
    if (n_runs > 0) BM_CK(cudaMemsetAsync(seq_ticket, 0, 4, st), "memset");
    BM_CK(cudaMemsetAsync(bnd, 0xde, (size_t)bstride * np * 8, st), "memset");
    NwArgs a;
    a.S = dv.S;
    a.s_off = dv.s_off;
    a.pitch = dv.pitch;
    a.n = dv.n;
    a.m = dv.m;
    a.p = penalties_host[q0];
    a.np = np;
    for (int q = 0; q < np; ++q) a.pv[q] = penalties_host[q0 + q];
    a.dirs = dirs;
    a.dir_stride = dstride;
    a.dir_off = dv.dir_off;
    a.cost = cost_l;
    a.cost_stride = k;
    a.items = dv.items;
    a.n_items = (int)g.items.size();
    a.ticket = dv.ticket;
    a.bnd = bnd;
    a.bnd_stride = bstride;
    a.bnd_off = dv.bnd_off;
    if (n_runs > 0) {
      a.items = d_multi;
      a.n_items = (int)multi.size();
      BM_CK(launch_nw(a, st), "nw_band_kernel");
      NwArgs b = a;
      b.ticket = seq_ticket;
      b.seq_off = d_seq;
      b.n_seq = n_runs;
      BM_CK(launch_nw_seq(b, st), "nw_seq_kernel");
    } else {
      BM_CK(launch_nw(a, st), "nw_band_kernel");
    }
    for (int q = 0; q < np; ++q) {
      const size_t pq = (size_t)(q0 + q) * n_thr;
      BM_CK(launch_tune_count(dirs + (size_t)q * dstride, dv.dir_off, dv.S, dv.s_off, dv.pitch,
                              dv.n, dv.m, k, thresholds, n_thr, gold, gold_off, pred + pq,
                              hit + pq, st),
            "tune_count_kernel");
    }
    q0 += np;
  }
  return BM_OK;
}

}  // extern "C"

#ifdef BM_NW_PROFILE
extern "C" int bm_nw_prof(unsigned long long* host, int n_items) {
  return (int)cudaMemcpyFromSymbol(host, bm::g_nw_prof, sizeof(unsigned long long) * 4 * n_items);
}
extern "C" int bm_nw_chunks(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, bm::g_nw_chunk, sizeof(unsigned long long) * 16 * 256 * 3);
}
#endif
