/*
 * bimine_b200.h -- C ABI of the B200 comparable-corpus miner (libbimine_b200.so).
 *
 * Hot path of the reference package `bimine` (arXiv 1509.08639 reproduction):
 *   score     build_similarity_matrix   bimine/aligner.py:313-339   (+ classifier.py:54-117,
 *                                                                    lexicon.py:88-105)
 *   align     nw_align / _nw_costs      bimine/aligner.py:116-134, 176-206, 216-220
 *             nw_align_wavefront        bimine/aligner.py:137-173, 223-241
 *   extract   extract_pairs             bimine/aligner.py:342-368
 *   tune      tune / f_measure          bimine/tuner.py:67-154
 *
 * The reference has no FFI: its only compiled boundary is the numba kernel
 * `_nw_costs(S: float64[n,m], penalty) -> float64[n+1,m+1]` (aligner.py:116).
 * Every entry point below replaces one of the Python/numba functions above; the
 * file:line each replaces is given on the declaration. INTEGRATION.md shows the
 * ctypes binding a bimine maintainer would add.
 *
 * Conventions
 *  - Plain C types only. Pointers inside the bm_* structs passed to the
 *    *device* entry points are DEVICE pointers; the `_host` entry points take
 *    HOST pointers and do their own H2D/D2H copies.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and does not synchronize unless documented.
 *  - Return 0 on success or a negative BM_E* code; bm_last_error() returns a
 *    thread-local message for the last failure.
 *  - Arithmetic is IEEE fp64 with the exact operation order of the reference
 *    (no FMA contraction, glibc-exact exp) so results are bit-identical.
 */
#ifndef BIMINE_B200_H
#define BIMINE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 2  /* 2: tok_alpha widened to uint32 (any sentence length) */

#define BM_OK 0
#define BM_EINVAL -1   /* bad argument (maps to ValueError)            */
#define BM_ECUDA -2    /* CUDA runtime error                           */
#define BM_ENOMEM -3   /* device allocation failed                     */
#define BM_ELIMIT -4   /* size over a hard bound (ResourceLimitError)  */
#define BM_EUNSUPPORTED -5 /* input outside the native ingest subset:  run
                              the Python path (bm_ingest_jsonl only)      */

/* Move codes (bimine/aligner.py:76-82): diagonal, skip-source, skip-target. */
#define BM_MOVE_D 0
#define BM_MOVE_GS 1
#define BM_MOVE_GT 2

/*
 * Packed sentences. Token strings are interned into one id space per pack
 * (normalized tokens and raw digit tokens share it; equal strings = equal id).
 * Per sentence (bimine/classifier.py:54-97, lexicon.py:95-98):
 *   n_tok   = len(tokens)                                  (T)
 *   n_punct = #tokens with no alphanumeric character        (P)
 *   n_alpha = #tokens with str.isalpha()                    (|A|)
 *   tok_*   = the set U of normalize(token) ids, ascending, with the number
 *             of isalpha() tokens that normalize to each id (A as multiplicities)
 *   dig_*   = the set D of raw isdigit() token ids, ascending
 */
typedef struct bm_sentences {
  int32_t n_sent;
  const int32_t* n_tok;
  const int32_t* n_punct;
  const int32_t* n_alpha;
  const int32_t* tok_off;    /* [n_sent + 1] */
  const int32_t* tok_id;     /* [tok_off[n_sent]] */
  const uint32_t* tok_alpha; /* [tok_off[n_sent]] */
  const int32_t* dig_off;    /* [n_sent + 1] */
  const int32_t* dig_id;     /* [dig_off[n_sent]] */
} bm_sentences;

/* Document pairs: source sentences [src0, src0+n), target [tgt0, tgt0+m). */
typedef struct bm_docs {
  int32_t n_docs;
  const int32_t* src0;
  const int32_t* n;
  const int32_t* tgt0;
  const int32_t* m;
} bm_docs;

/*
 * Lexicon over the same id space (bimine/lexicon.py:16-46): fwd = the model's
 * lexicon (source word -> candidate target words), rev = lex.reversed().
 * Only candidates that occur in the id space are kept (others can never hit).
 */
typedef struct bm_lexicon {
  int32_t n_ids;
  const int32_t* fwd_off; /* [n_ids + 1] */
  const int32_t* fwd_cand;
  const int32_t* rev_off; /* [n_ids + 1] */
  const int32_t* rev_cand;
} bm_lexicon;

/* Linear classifier (bimine/classifier.py:41-49,107-117). */
typedef struct bm_model {
  double w[7];
  double bias;
} bm_model;

/* One mined pair (bimine/aligner.py:103-113 minus the Sentence objects). */
typedef struct bm_record {
  int32_t doc;  /* index into bm_docs */
  int32_t i;    /* source sentence index (src_index) */
  int32_t j;    /* target sentence index (tgt_index) */
  int32_t pad;
  double conf;  /* S[i, j] */
} bm_record;

int bm_abi_version(void);
const char* bm_last_error(void);
/* Number of CUDA devices visible (0 = no GPU). */
int bm_device_count(void);
/* Kernels this library has launched since it was loaded (instrumentation). */
int64_t bm_launches(void);
/* FP64 pipe probe (8 DFMA chains x 256 threads x blocks x iters); used by the
 * benchmark to measure the FP64 roof of the device. Not part of the path. */
int bm_probe_fp64(double* out, int32_t iters, int32_t blocks, void* stream);

/*
 * K1 -- replaces build_similarity_matrix (aligner.py:313-339) for a batch:
 * S[d] is written row-major with row pitch `pitch[d]` doubles at S + s_off[d].
 * pitch[d] must be a multiple of 4 and S + s_off[d] 32-byte aligned (the NW
 * kernel reads S with 16-byte vector loads). n_host/m_host: host copies of
 * docs->n / docs->m (used to plan the tile grid).
 */
int bm_score(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
             const int32_t* m_host, const bm_lexicon* lex, const bm_model* model,
             const int64_t* s_off, const int32_t* pitch, double* S, void* stream);

/*
 * Feature vectors / confidences for explicit (src, tgt, pos_s, pos_t) tuples:
 * replaces extract_features (classifier.py:68-97) and confidence (:107-117).
 * feats: [n_q, 7]; conf: [n_q] (either may be NULL).
 */
int bm_features(const bm_sentences* sent, const bm_lexicon* lex, const int32_t* q_src,
                const int32_t* q_tgt, const double* q_pos_s, const double* q_pos_t,
                int32_t n_q, double* feats, void* stream);
int bm_confidence(const double* feats, int32_t n_q, const bm_model* model, double* conf,
                  void* stream);

/*
 * K2/K3 -- replaces _nw_costs / _nw_costs_wavefront + the fill half of
 * nw_align (aligner.py:116-173, 216-241) for a batch of matrices.
 * S: as written by bm_score. dirs: 2-bit traceback codes, layout private to
 * the library, sized by bm_dirs_words(n, m) uint32 words at dirs + dir_off[d].
 * cost[d] = C[n, m].
 */
int64_t bm_dirs_words(int32_t n, int32_t m);
int bm_nw(const double* S, const int64_t* s_off, const int32_t* pitch, const int32_t* n,
          const int32_t* m, const int32_t* n_host, const int32_t* m_host, int32_t n_docs,
          double penalty, uint32_t* dirs, const int64_t* dir_off, double* cost, void* stream);

/*
 * K4a -- the traceback of aligner.py:176-206 (tie order D > GS > GT): the
 * moves of doc d are written at mv_off[d] (capacity n+m) in REVERSE path
 * order; mv_op = BM_MOVE_*, mv_i / mv_j = cell indices (-1 where the move has
 * none: GS has no j, GT no i), mv_len[d] = path length.
 */
int bm_traceback(const uint32_t* dirs, const int64_t* dir_off, const int32_t* n,
                 const int32_t* m, int32_t n_docs, const int64_t* mv_off, int8_t* mv_op,
                 int32_t* mv_i, int32_t* mv_j, int32_t* mv_len, void* stream);

/*
 * K4b -- extract_pairs (aligner.py:342-368) fused with the traceback: every
 * diagonal move with S[i,j] >= threshold becomes a record, in path order.
 * Records of doc d land at rec + rec_off[d] (capacity min(n,m)); rec_count[d].
 */
int bm_extract(const uint32_t* dirs, const int64_t* dir_off, const double* S,
               const int64_t* s_off, const int32_t* pitch, const int32_t* n, const int32_t* m,
               int32_t n_docs, double threshold, const int64_t* rec_off, bm_record* rec,
               int32_t* rec_count, void* stream);

/*
 * extract_pairs for an explicit path (aligner.py:352-357): conf[q] =
 * S[ci[q], cj[q]] (row pitch `pitch` doubles), keep[q] = conf[q] >= threshold.
 */
int bm_select(const double* S, int64_t pitch, const int32_t* ci, const int32_t* cj, int32_t k,
              double threshold, double* conf, uint8_t* keep, void* stream);

/*
 * Fused score -> NW -> traceback -> threshold for a batch (mine_document,
 * miner.py:84-128, forward orientation). Records land at rec + rec_off[d]
 * (capacity min(n,m)), counts in rec_count, path costs C[n,m] in cost. Docs of
 * any size are accepted: the library routes each one either to the fused
 * warp-per-document kernel (no similarity matrix is materialised) or to the
 * banded K1 -> K2/K3 -> K4 path. n_host/m_host/amax_host are host arrays
 * (amax = the largest n_tok of any sentence of the doc; <= 255 allows the
 * fused tier). Scratch is
 * stream-ordered (cudaMallocAsync on `stream`).
 */
int bm_mine(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
            const int32_t* m_host, const int32_t* amax_host, const bm_lexicon* lex,
            const bm_model* model, double threshold, double penalty, const int64_t* rec_off,
            bm_record* rec, int32_t* rec_count, double* cost, void* stream);

/*
 * Same as bm_mine but every array (sentences, docs, lexicon) is in HOST
 * memory: the call copies inputs to the device, mines, compacts the records
 * and copies them back into rec_out (capacity rec_cap) in document order.
 * *n_rec receives the record count. Synchronizes `stream` before returning.
 * This is the end-to-end entry point a foreign-language binding would call.
 */
int bm_mine_host(const bm_sentences* sent_h, const bm_docs* docs_h, const bm_lexicon* lex_h,
                 const bm_model* model, double threshold, double penalty, bm_record* rec_out,
                 int64_t rec_cap, int64_t* n_rec, double* cost_out, void* stream);

/*
 * Compact host wire format for bm_mine_host_wire: same content as
 * bm_sentences, narrower types (valid when the id space has <= 65536 ids and
 * every count is <= 255). Halves the host->device bytes of a batch.
 */
typedef struct bm_wire {
  int32_t n_sent;
  const uint8_t* n_tok;
  const uint8_t* n_punct;
  const uint8_t* n_alpha;
  const int32_t* tok_off;   /* [n_sent + 1] */
  const uint16_t* tok_id;
  const uint8_t* tok_alpha;
  const int32_t* dig_off;   /* [n_sent + 1] */
  const uint16_t* dig_id;
} bm_wire;

/* bm_mine_host with the compact wire format (host pointers). */
int bm_mine_host_wire(const bm_wire* wire_h, const bm_docs* docs_h, const bm_lexicon* lex_h,
                      const bm_model* model, double threshold, double penalty,
                      bm_record* rec_out, int64_t rec_cap, int64_t* n_rec, double* cost_out,
                      void* stream);

/*
 * Packed host format for bm_mine_host_packed: the same content in 4 bytes per
 * sentence plus 2 bytes per distinct token (valid when the id space has
 * <= 16384 ids, every count is <= 255 and no token occurs more than 3 times
 * as an alphabetic token in one sentence). Offsets are rebuilt on the device
 * from the per-sentence counts and one base offset per 32 sentences, so
 * tok_off / dig_off are read by the host planner only and never copied.
 * counts[s] = n_tok | n_punct << 8 | n_uniq << 16 | n_dig << 24 with
 * n_uniq = tok_off[s+1] - tok_off[s], n_dig = dig_off[s+1] - dig_off[s];
 * n_alpha is the sum of the sentence's alphabetic counts.
 */
typedef struct bm_wire_packed {
  int32_t n_sent;
  const int32_t* tok_off;    /* [n_sent + 1] host planning only */
  const int32_t* dig_off;    /* [n_sent + 1] host planning only */
  const uint32_t* counts;    /* [n_sent] */
  const int32_t* tok_off32;  /* [n_sent / 32 + 1]: tok_off[32 b] */
  const int32_t* dig_off32;  /* [n_sent / 32 + 1]: dig_off[32 b] */
  const uint16_t* tok_pk;    /* [tok_off[n_sent]]: tok_id << 2 | tok_alpha */
  const uint16_t* dig_id;    /* [dig_off[n_sent]] */
} bm_wire_packed;

/* bm_mine_host with the packed format (host pointers). */
int bm_mine_host_packed(const bm_wire_packed* pk_h, const bm_docs* docs_h, const bm_lexicon* lex_h,
                        const bm_model* model, double threshold, double penalty,
                        bm_record* rec_out, int64_t rec_cap, int64_t* n_rec, double* cost_out,
                        void* stream);

/*
 * K5 -- tune (tuner.py:87-154): for every penalty p_k and threshold t_l,
 * pred[k*n_thr + l] += #diagonal moves with S >= t_l over all docs, and
 * hit[k*n_thr + l] += those whose (i, j) is in the doc's gold set.
 * gold: per doc ascending keys i*m + j at gold + gold_off[d] (gold_off[n_docs]).
 * token_bound: an upper bound of the token count of every sentence of the
 * docs (enables the document-level join for scoring), or -1 if unknown.
 */
int bm_tune(const bm_sentences* sent, const bm_docs* docs, const int32_t* n_host,
            const int32_t* m_host, const bm_lexicon* lex, const bm_model* model,
            const double* penalties_host, int32_t n_pen, const double* thresholds, int32_t n_thr,
            const int64_t* gold, const int64_t* gold_off, unsigned long long* pred,
            unsigned long long* hit, int32_t token_bound, void* stream);

/* The large mining scratch (similarity matrices, hit counts, codes) is kept
 * per stream of the calling thread and reused by later calls (grow-only, at
 * most 8 streams); bm_trim synchronizes the device and releases it. */
int bm_trim(void);

/* Exclusive-scan compaction of per-doc record slots into a dense,
 * document-ordered array; *total (device) receives the record count. */
int bm_compact(const bm_record* rec, const int64_t* rec_off, const int32_t* rec_count,
               int32_t n_docs, bm_record* dense, int64_t* total, void* stream);

/* bidirectional_merge on the device (miner.py:131-155).
 * fwd / bwd: the two passes' compacted records (document-ordered, doc = batch
 * index, (i, j) in the pass's orientation, path order). swap_f[d] / swap_b[d]:
 * the pass read pair d swapped (its records are re-oriented and labelled
 * "backward", miner.py:115-128). norm_key: per sentence an id of its
 * normalized text (equal ids <=> equal texts within a document). Writes the
 * merged records -- one per (source text, target text) key: the higher
 * confidence, "forward" over "backward" on an exact tie, else the first seen
 * in F-then-B order -- sorted by (document, source index, target index) in
 * the pair's orientation, with pad = 0 (forward) / 1 (backward); *total
 * (device) receives their number. All pointers are device pointers; out
 * holds n_fwd + n_bwd records. */
int bm_merge_bidir(const bm_record* fwd, int64_t n_fwd, const bm_record* bwd, int64_t n_bwd,
                   int32_t n_docs, const int32_t* src0, const int32_t* tgt0,
                   const int32_t* norm_key, const uint8_t* swap_f, const uint8_t* swap_b,
                   bm_record* out, int64_t* total, void* stream);

/* Multi-GPU result gather, rank 0 (the reference's ordered
 * pool.map, bimine/miner.py:236-245): the compacted records of `world` ranks
 * sit in a padded [world][stride] device layout with part_len[r] (device)
 * valid records each; every rank mined its own documents, ordered by global
 * document index (record.doc). Writes all of them to out in global document
 * order (path order within a document) and their number to *total (device). */
int bm_merge_shards(const bm_record* rec, int64_t stride, const int64_t* part_len, int32_t world,
                    int32_t n_docs, bm_record* out, int64_t* total, void* stream);

/* ------------------------------------------------------------------------
 * Native corpus path: host C++, no device work.
 * Replaces, for ASCII JSONL input, bimine/corpus.py:129-193 load_document_pairs
 * (+ segment_sentences :92-126, tokenize :28, normalize :38-40), the packing
 * of pack.py, bimine/miner.py:131-155 bidirectional_merge and :253-260
 * format_pair_line. Anything outside the accepted subset (non-ASCII bytes,
 * JSON the validator refuses, non-string/int ids or langs, missing fields,
 * equal langs) returns BM_EUNSUPPORTED with the reason in `why`; the caller
 * then runs the Python path, which reproduces the reference exactly
 * (including its DataError messages).
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t n_sent, n_docs, n_ids, n_skipped;
  int64_t n_tok_entries, n_dig_entries;
  const int32_t *n_tok, *n_punct, *n_alpha, *tok_off, *tok_id;
  const uint32_t* tok_alpha;
  const int32_t *dig_off, *dig_id;
  const int32_t *src0, *n, *tgt0, *m;
} bm_ingest_arrays;

/* Parse + segment + tokenize + intern a JSONL file of document pairs; pairs
 * with an empty side are dropped (listed by bm_ingest_skipped). *handle owns
 * every array until bm_ingest_free. */
int bm_ingest_jsonl(const char* path, void** handle, char* why, int32_t why_len);
void bm_ingest_free(void* handle);
/* Gold set (tuner.py:157-203 load_gold_set, §8(f)-4): the same reader for
 * document-pair JSONL whose lines also hold "gold": [[i, j], ...]. Lines with
 * an empty side, a missing or malformed "gold", or pairs out of bounds -- where
 * load_gold_set raises -- and empty files return BM_EUNSUPPORTED (the Python
 * reader then raises the reference's DataError). bm_ingest_gold: per document
 * d the ascending unique keys i * m + j at keys[off[d] .. off[d + 1]). */
int bm_ingest_gold_jsonl(const char* path, void** handle, char* why, int32_t why_len);
int bm_ingest_gold(void* handle, const int64_t** keys, const int64_t** off, int64_t* n_keys);
int bm_ingest_view(void* handle, bm_ingest_arrays* out);
int bm_ingest_doc(void* handle, int32_t k, const char** id, const char** src_lang,
                  const char** tgt_lang);
int bm_ingest_skipped(void* handle, int32_t q, int64_t* lineno, const char** id,
                      const char** side);
/* Lexicon (src_words[q] -> tgt_words[q]) as forward/reverse CSR over the
 * handle's id space (pack.py pack_lexicon); arrays owned by the handle. */
int bm_ingest_lexicon(void* handle, const char* const* src_words, const char* const* tgt_words,
                      int64_t n_entries, bm_lexicon* out);
/* Re-orient, merge (when has_bwd) and format the mined records as TSV bytes
 * in document order; report = {pairs, forward, backward, unique src tokens,
 * unique tgt tokens, docs mined}. *out stays valid until the next call. */
int bm_ingest_emit(void* handle, const bm_record* fwd, int64_t n_fwd, const bm_record* bwd,
                   int64_t n_bwd, int32_t has_bwd, const uint8_t* swap_f, const uint8_t* swap_b,
                   const uint8_t* skip, const char** out, int64_t* out_len, int64_t* report);
/* The same emission for records bm_merge_bidir already re-oriented and merged
 * (pad = 0 forward / 1 backward; doc = the handle's document index). */
int bm_ingest_emit_merged(void* handle, const bm_record* recs, int64_t n, const uint8_t* skip,
                          const char** out, int64_t* out_len, int64_t* report);
/* Per sentence of the handle, an id of its normalized text (equal ids <=>
 * equal texts within one document): bm_merge_bidir's key. */
int bm_ingest_norm_keys(void* handle, const int32_t** keys);
/* Streaming (mine_corpus_file over large files): ingest the lines of bytes
 * [b0, b1) of the file (b0 at a line start, b1 < 0: to the end), numbering
 * them from line0 + 1; *n_lines receives the number of lines of the range. */
int bm_ingest_jsonl_range(const char* path, int64_t b0, int64_t b1, int64_t line0, void** handle,
                          int64_t* n_lines, char* why, int32_t why_len);
/* After an emit: the normalized token strings of the emitted pairs' source
 * (which = 0) / target (1) sentences, NUL-separated (miner.py:253-260). */
int bm_ingest_seen(void* handle, int32_t which, const char** buf, int64_t* len);

#ifdef __cplusplus
}
#endif

#endif /* BIMINE_B200_H */
