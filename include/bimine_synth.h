/* Native synthetic-corpus generator for the benchmark workloads (bench input
 * generation only; NOT part of the drop-in mining boundary of bimine_b200.h).
 *
 * Draws the distributions of the reference's test generator
 * (pkg/tests/synthgen.py:19-145, restated in paper_1509_08639_b200/synth.py)
 * per document, from a stream keyed by (seed, global document index), and
 * emits the packed bm_sentences layout directly. */
#ifndef BIMINE_SYNTH_H
#define BIMINE_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bm_synth_spec {
  int32_t vocab;      /* words per language (synthgen.make_vocab) */
  double noise;       /* target-word noise of translation pairs */
  double digit_rate;  /* probability of a year token in a translation pair */
  uint64_t seed;
} bm_synth_spec;

typedef struct bm_synth_arrays {
  int64_t n_sent, n_docs, n_tok_entries, n_dig_entries, n_gold;
  const int32_t *n_tok, *n_punct, *n_alpha, *tok_off, *tok_id;
  const uint32_t* tok_alpha;
  const int32_t *dig_off, *dig_id;
  const int32_t *src0, *n, *tgt0, *m;
  const int64_t* gold_off; /* [n_docs + 1] into gold_i / gold_j */
  const int32_t *gold_i, *gold_j;
} bm_synth_arrays;

/* Documents ids[q] (q < k) with g[q] translation pairs and a[q] / b[q] source
 * / target distractors, in the order given; threads <= 0: all host threads.
 * Returns 0, -1 on bad arguments, -4 when the corpus exceeds int32 offsets. */
int bm_synth_generate(const bm_synth_spec* spec, const int64_t* ids, const int32_t* g,
                      const int32_t* a, const int32_t* b, int64_t k, int32_t threads,
                      void** handle);
int bm_synth_view(void* handle, bm_synth_arrays* out);
void bm_synth_free(void* handle);
/* The same documents rendered as document-pair JSONL (ids "doc%07d" of the
 * global index, languages xx / yy, sentences as lists): tokenizing the file
 * gives back exactly the arrays bm_synth_generate packs. */
int bm_synth_jsonl(const bm_synth_spec* spec, const int64_t* ids, const int32_t* g,
                   const int32_t* a, const int32_t* b, int64_t k, int32_t threads,
                   const char* path);

#ifdef __cplusplus
}
#endif

#endif /* BIMINE_SYNTH_H */
