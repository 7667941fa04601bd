// Synthetic comparable corpora for the benchmark workloads, generated natively
// and per document (BENCH INPUT GENERATION; not part of the mining path).
//
// Same distributions as synth.make_corpus (the numpy restatement of the
// reference's test generator, pkg/tests/synthgen.py:19-145): a document with
// g translation pairs and a / b one-sided distractors is g + a + b events in
// random order; an event is a sentence of 4-9 words from a V-word vocabulary
// (translation pairs: distinct words, target words replaced by a random word
// with probability `noise`, a year token with probability `digit_rate`), ended
// by ".". Ids: source word k -> k, target word k -> V + k, "." -> 2V, year y ->
// 2V + 1 + (y - 1900).
//
// Every document draws from its own counter-based stream (splitmix64 of the
// seed and the document's GLOBAL index), so a rank generates exactly the
// documents of its shard and a document's text never depends on how a corpus
// is split. Threads take contiguous ranges of the requested documents.
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bimine_synth.h"

namespace {

constexpr int kYear0 = 1900, kYears = 131;

struct Rng {  // xoshiro256** seeded by splitmix64
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  Rng(uint64_t seed, uint64_t doc) {
    uint64_t x = seed * 0xD1B54A32D192ED03ull ^ (doc + 0x632BE59BD9B4E019ull);
    for (auto& v : s) v = splitmix(x);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  uint32_t below(uint32_t n) { return (uint32_t)(((next() >> 32) * (uint64_t)n) >> 32); }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

template <class T>
struct Buf {  // append-only buffer without zero-fill (sized to an upper bound)
  T* p = nullptr;
  size_t n = 0;
  void init(size_t cap) { p = (T*)malloc(std::max<size_t>(cap, 1) * sizeof(T)); }
  ~Buf() { free(p); }
  void push(T v) { p[n++] = v; }
  size_t size() const { return n; }
};

struct Part {  // one thread's documents, sentence and entry offsets local
  Buf<int32_t> n_tok, n_punct, n_alpha, tok_off, tok_id, dig_off, dig_id;
  Buf<uint32_t> tok_alpha;
  std::vector<int32_t> src0, n, tgt0, m;
  std::vector<int64_t> gold_off{0};
  std::vector<int32_t> gold_i, gold_j;
};

struct Corpus {
  std::vector<int32_t> n_tok, n_punct, n_alpha, tok_off, tok_id, dig_off, dig_id;
  std::vector<uint32_t> tok_alpha;
  std::vector<int32_t> src0, n, tgt0, m;
  std::vector<int64_t> gold_off;
  std::vector<int32_t> gold_i, gold_j;
};

struct Event {
  uint8_t type;  // 0 translation pair, 1 source distractor, 2 target distractor
  uint8_t k;     // words
  int16_t year;  // -1: none
  int32_t w[9];  // source word ids (type 0/1) or target words before + V (type 2)
  int32_t t[9];  // target word ids of a translation pair (noised)
};

// one sentence: words (+ year) + "."; U = ascending unique ids with alpha counts
void emit_sentence(Part& p, const int32_t* words, int k, int year_id, int dot) {
  int32_t ids[11];
  for (int q = 0; q < k; ++q) {  // insertion sort (k <= 9)
    const int32_t v = words[q];
    int u = q;
    for (; u > 0 && ids[u - 1] > v; --u) ids[u] = ids[u - 1];
    ids[u] = v;
  }
  int32_t* out = p.tok_id.p + p.tok_id.n;
  uint32_t* cnt = p.tok_alpha.p + p.tok_alpha.n;
  int nu = 0;
  for (int q = 0; q < k; ++q) {
    if (nu > 0 && out[nu - 1] == ids[q]) {
      ++cnt[nu - 1];
    } else {
      out[nu] = ids[q];
      cnt[nu++] = 1;
    }
  }
  out[nu] = dot;  // ids: words < 2V = dot < years
  cnt[nu++] = 0;
  if (year_id >= 0) {
    out[nu] = year_id;
    cnt[nu++] = 0;
    p.dig_id.push(year_id);
  }
  p.tok_id.n += nu;
  p.tok_alpha.n += nu;
  p.tok_off.push((int32_t)p.tok_id.n);
  p.dig_off.push((int32_t)p.dig_id.n);
  p.n_tok.push(k + (year_id >= 0 ? 1 : 0) + 1);
  p.n_punct.push(1);
  p.n_alpha.push(k);
}

void gen_doc(Part& p, const bm_synth_spec& sp, int64_t doc, int32_t g, int32_t a, int32_t b,
             std::vector<Event>& ev) {
  Rng r(sp.seed, (uint64_t)doc);
  const int V = sp.vocab, dot = 2 * V;
  const int E = g + a + b;
  ev.resize(E);
  for (int e = 0; e < E; ++e) ev[e].type = e < g ? 0 : e < g + a ? 1 : 2;
  for (int e = E - 1; e > 0; --e) std::swap(ev[e].type, ev[r.below((uint32_t)e + 1)].type);
  for (int e = 0; e < E; ++e) {
    Event& x = ev[e];
    x.k = (uint8_t)(4 + r.below(6));
    for (int q = 0; q < x.k; ++q) x.w[q] = (int32_t)r.below((uint32_t)V);
    x.year = -1;
    if (x.type == 0) {
      // distinct words in a translation pair (synth.make_corpus redraws)
      for (int q = 1; q < x.k; ++q)
        for (int u = 0; u < q; ++u)
          if (x.w[u] == x.w[q]) {
            x.w[q] = (int32_t)r.below((uint32_t)V);
            u = -1;  // re-check against every earlier word
          }
      for (int q = 0; q < x.k; ++q)
        x.t[q] = V + (r.uniform() < sp.noise ? (int32_t)r.below((uint32_t)V) : x.w[q]);
      if (r.uniform() < sp.digit_rate) x.year = (int16_t)r.below(kYears);
    }
  }
  const int32_t s_base = (int32_t)p.n_tok.size();
  int ns = 0, nt = 0;
  for (const Event& x : ev) ns += x.type != 2;
  for (const Event& x : ev) nt += x.type != 1;
  p.src0.push_back(s_base);
  p.n.push_back(ns);
  p.tgt0.push_back(s_base + ns);
  p.m.push_back(nt);
  for (const Event& x : ev) {  // source side: events 0 / 1 in order
    if (x.type == 2) continue;
    emit_sentence(p, x.w, x.k, x.year >= 0 ? dot + 1 + x.year : -1, dot);
  }
  int i = 0, j = 0;
  for (const Event& x : ev) {  // target side: events 0 / 2 in order
    if (x.type == 1) {
      ++i;
      continue;
    }
    int32_t tw[9];
    for (int q = 0; q < x.k; ++q) tw[q] = x.type == 0 ? x.t[q] : V + x.w[q];
    emit_sentence(p, tw, x.k, x.year >= 0 ? dot + 1 + x.year : -1, dot);
    if (x.type == 0) {
      p.gold_i.push_back(i);
      p.gold_j.push_back(j);
      ++i;
    }
    ++j;
  }
  p.gold_off.push_back((int64_t)p.gold_i.size());
}

// JSONL text of one document (synth.SynthCorpus.doc_pairs rendering: the
// words, then the year, then "." -- tokenize() gives back the packed tokens).
void letters3(int k, char* out) {
  out[2] = (char)('a' + k % 26);
  k /= 26;
  out[1] = (char)('a' + k % 26);
  k /= 26;
  out[0] = (char)('a' + k % 26);
}

void jsonl_doc(std::string& o, const bm_synth_spec& sp, int64_t doc, int32_t g, int32_t a,
               int32_t b, std::vector<Event>& ev) {
  Part scratch;  // reuse gen_doc's event draws: same stream, same events
  const int V = sp.vocab;
  // regenerate the events exactly as gen_doc does (the draws are identical)
  Rng r(sp.seed, (uint64_t)doc);
  const int E = g + a + b;
  ev.resize(E);
  for (int e = 0; e < E; ++e) ev[e].type = e < g ? 0 : e < g + a ? 1 : 2;
  for (int e = E - 1; e > 0; --e) std::swap(ev[e].type, ev[r.below((uint32_t)e + 1)].type);
  for (int e = 0; e < E; ++e) {
    Event& x = ev[e];
    x.k = (uint8_t)(4 + r.below(6));
    for (int q = 0; q < x.k; ++q) x.w[q] = (int32_t)r.below((uint32_t)V);
    x.year = -1;
    if (x.type == 0) {
      for (int q = 1; q < x.k; ++q)
        for (int u = 0; u < q; ++u)
          if (x.w[u] == x.w[q]) {
            x.w[q] = (int32_t)r.below((uint32_t)V);
            u = -1;
          }
      for (int q = 0; q < x.k; ++q)
        x.t[q] = V + (r.uniform() < sp.noise ? (int32_t)r.below((uint32_t)V) : x.w[q]);
      if (r.uniform() < sp.digit_rate) x.year = (int16_t)r.below(kYears);
    }
  }
  char buf[32];
  snprintf(buf, sizeof(buf), "%07lld", (long long)doc);
  o += "{\"id\": \"doc";
  o += buf;
  o += "\", \"src_lang\": \"xx\", \"tgt_lang\": \"yy\", \"src\": [";
  auto sentence = [&](const int32_t* words, int k, int year, bool tgt) {
    o += '"';
    for (int q = 0; q < k; ++q) {
      if (q) o += ' ';
      char w[4];
      w[0] = tgt ? 'v' : 'w';
      letters3(words[q] - (tgt ? V : 0), w + 1);
      o.append(w, 4);
    }
    if (year >= 0) {
      snprintf(buf, sizeof(buf), " %d", kYear0 + year);
      o += buf;
    }
    o += ".\"";
  };
  bool first = true;
  for (const Event& x : ev) {
    if (x.type == 2) continue;
    if (!first) o += ", ";
    first = false;
    sentence(x.w, x.k, x.year, false);
  }
  o += "], \"tgt\": [";
  first = true;
  for (const Event& x : ev) {
    if (x.type == 1) continue;
    if (!first) o += ", ";
    first = false;
    int32_t tw[9];
    for (int q = 0; q < x.k; ++q) tw[q] = x.type == 0 ? x.t[q] : V + x.w[q];
    sentence(tw, x.k, x.year, true);
  }
  o += "]}\n";
  (void)scratch;
}

template <class T>
T src_at(const std::vector<T>& v, size_t q) { return v[q]; }
template <class T>
T src_at(const Buf<T>& v, size_t q) { return v.p[q]; }
template <class T, class S>
void append(std::vector<T>& dst, size_t at, const S& src, T add, size_t skip = 0) {
  for (size_t q = skip; q < src.size(); ++q) dst[at + q - skip] = src_at(src, q) + add;
}

}  // namespace

extern "C" {

int bm_synth_generate(const bm_synth_spec* spec, const int64_t* ids, const int32_t* g,
                      const int32_t* a, const int32_t* b, int64_t k, int32_t threads,
                      void** handle) {
  if (spec == nullptr || handle == nullptr || k < 0 || spec->vocab < 1) return -1;
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(k, 1));
  std::vector<Part> parts(nt);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      const int64_t lo = k * t / nt, hi = k * (t + 1) / nt;
      int64_t sents = 0;
      for (int64_t q = lo; q < hi; ++q) sents += 2 * (int64_t)g[q] + a[q] + b[q];
      Part& p = parts[t];
      for (auto* v : {&p.n_tok, &p.n_punct, &p.n_alpha, &p.tok_off, &p.dig_off, &p.dig_id})
        v->init(sents + 1);
      p.tok_id.init(sents * 11);
      p.tok_alpha.init(sents * 11);
      p.tok_off.push(0);
      p.dig_off.push(0);
      std::vector<Event> ev;
      for (int64_t q = lo; q < hi; ++q) gen_doc(parts[t], *spec, ids[q], g[q], a[q], b[q], ev);
    });
  for (auto& th : pool) th.join();
  // concatenate (parallel copies at precomputed bases)
  std::vector<int64_t> sb(nt + 1, 0), eb(nt + 1, 0), db(nt + 1, 0), gb(nt + 1, 0), kb(nt + 1, 0);
  for (int t = 0; t < nt; ++t) {
    sb[t + 1] = sb[t] + (int64_t)parts[t].n_tok.size();
    eb[t + 1] = eb[t] + (int64_t)parts[t].tok_id.size();
    db[t + 1] = db[t] + (int64_t)parts[t].dig_id.size();
    gb[t + 1] = gb[t] + (int64_t)parts[t].gold_i.size();
    kb[t + 1] = kb[t] + (int64_t)parts[t].n.size();
  }
  if (sb[nt] > INT32_MAX || eb[nt] > INT32_MAX) return -4;  // int32 offsets of bm_sentences
  auto* c = new Corpus();
  c->n_tok.resize(sb[nt]);
  c->n_punct.resize(sb[nt]);
  c->n_alpha.resize(sb[nt]);
  c->tok_off.resize(sb[nt] + 1);
  c->dig_off.resize(sb[nt] + 1);
  c->tok_id.resize(eb[nt]);
  c->tok_alpha.resize(eb[nt]);
  c->dig_id.resize(db[nt]);
  c->src0.resize(kb[nt]);
  c->n.resize(kb[nt]);
  c->tgt0.resize(kb[nt]);
  c->m.resize(kb[nt]);
  c->gold_off.resize(kb[nt] + 1);
  c->gold_i.resize(gb[nt]);
  c->gold_j.resize(gb[nt]);
  c->tok_off[0] = c->dig_off[0] = 0;
  c->gold_off[0] = 0;
  pool.clear();
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      Part& p = parts[t];
      const int32_t s0 = (int32_t)sb[t], e0 = (int32_t)eb[t], d0 = (int32_t)db[t];
      append(c->n_tok, sb[t], p.n_tok, 0);
      append(c->n_punct, sb[t], p.n_punct, 0);
      append(c->n_alpha, sb[t], p.n_alpha, 0);
      append(c->tok_off, sb[t] + 1, p.tok_off, e0, 1);
      append(c->dig_off, sb[t] + 1, p.dig_off, d0, 1);
      append(c->tok_id, eb[t], p.tok_id, 0);
      append(c->tok_alpha, eb[t], p.tok_alpha, 0u);
      append(c->dig_id, db[t], p.dig_id, 0);
      append(c->src0, kb[t], p.src0, s0);
      append(c->n, kb[t], p.n, 0);
      append(c->tgt0, kb[t], p.tgt0, s0);
      append(c->m, kb[t], p.m, 0);
      append(c->gold_off, kb[t] + 1, p.gold_off, (int64_t)gb[t], 1);
      append(c->gold_i, gb[t], p.gold_i, 0);
      append(c->gold_j, gb[t], p.gold_j, 0);
    });
  for (auto& th : pool) th.join();
  *handle = c;
  return 0;
}

int bm_synth_view(void* handle, bm_synth_arrays* out) {
  if (handle == nullptr || out == nullptr) return -1;
  Corpus* c = (Corpus*)handle;
  out->n_sent = (int64_t)c->n_tok.size();
  out->n_docs = (int64_t)c->n.size();
  out->n_tok_entries = (int64_t)c->tok_id.size();
  out->n_dig_entries = (int64_t)c->dig_id.size();
  out->n_gold = (int64_t)c->gold_i.size();
  out->n_tok = c->n_tok.data();
  out->n_punct = c->n_punct.data();
  out->n_alpha = c->n_alpha.data();
  out->tok_off = c->tok_off.data();
  out->tok_id = c->tok_id.data();
  out->tok_alpha = c->tok_alpha.data();
  out->dig_off = c->dig_off.data();
  out->dig_id = c->dig_id.data();
  out->src0 = c->src0.data();
  out->n = c->n.data();
  out->tgt0 = c->tgt0.data();
  out->m = c->m.data();
  out->gold_off = c->gold_off.data();
  out->gold_i = c->gold_i.data();
  out->gold_j = c->gold_j.data();
  return 0;
}

void bm_synth_free(void* handle) { delete (Corpus*)handle; }

int bm_synth_jsonl(const bm_synth_spec* spec, const int64_t* ids, const int32_t* g,
                   const int32_t* a, const int32_t* b, int64_t k, int32_t threads,
                   const char* path) {
  if (spec == nullptr || path == nullptr || k < 0 || spec->vocab < 1 || spec->vocab > 17576)
    return -1;
  FILE* f = fopen(path, "wb");
  if (f == nullptr) return -2;
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  // blocks of documents rendered in parallel, written in order
  const int64_t block = 4096;
  std::vector<std::string> buf((size_t)nt);
  int rc = 0;
  for (int64_t b0 = 0; b0 < k && rc == 0; b0 += block * nt) {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        buf[t].clear();
        std::vector<Event> ev;
        const int64_t lo = b0 + block * t, hi = std::min(k, lo + block);
        for (int64_t q = lo; q < hi; ++q) jsonl_doc(buf[t], *spec, ids[q], g[q], a[q], b[q], ev);
      });
    for (auto& th : pool) th.join();
    for (int t = 0; t < nt && rc == 0; ++t)
      if (!buf[t].empty() && fwrite(buf[t].data(), 1, buf[t].size(), f) != buf[t].size()) rc = -3;
  }
  if (fclose(f) != 0 && rc == 0) rc = -3;
  return rc;
}

}  // extern "C"
