// Native corpus path: JSONL document pairs ->
// packed id arrays (the bm_sentences / bm_docs / bm_lexicon inputs of the
// kernels) -> after mining, the bidirectional merge and the TSV bytes.
//
// It restates, for ASCII input, the host side of the reference:
//   corpus.py:28,38-60     tokenize ([^\W_]+|\S), normalize (NFC, lower, ws)
//   corpus.py:92-126       segment_sentences (abbreviations, . ! ? rules)
//   corpus.py:129-193      load_document_pairs (JSON fields, empty-side skip)
//   pack.py                the packed per-sentence features (T, P, |A|, U, D)
//   miner.py:131-155       bidirectional_merge (normalized-text key)
//   miner.py:183-194,253   format_pair_line, _sanitize, unique-token counts
// Exactness contract: the native path accepts a file only when it is valid
// UTF-8, its JSON stays inside a simple, fully validated subset, and all text
// passes the checks below; otherwise bm_ingest_jsonl returns BM_EUNSUPPORTED
// and the caller runs the Python path (which also produces the reference's
// error messages). Character properties come from tables generated from the
// reference's own CPython (gen_unicode_tables.py -> unicode_tables.h):
//   SPACE (str.isspace = re \s = split/strip), ALNUM (isalnum = re \w minus
//   '_'), ALPHA, DIGIT, UPPER, NFC quick-check Yes, combining class 0, and the
//   one-code-point lowercase map. Accepted text has every code point NFC-QC
//   Yes with no two adjacent non-starters -- so NFC(text) == text (UAX #15
//   quick check) -- and every code point lowercases to one code point of the
//   same classes (no final-sigma U+03A3), so str.lower() is the per-character
//   map and lowering never moves a token boundary. Real text (e.g. Polish or
//   English) passes; anything else goes to Python.
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include "bimine_b200.h"
#include "unicode_tables.h"

namespace bm_ingest {

inline uint8_t uprops(uint32_t cp) {
  return bm_unicode::kBlocks[bm_unicode::kBlockIndex[cp >> 8]][cp & 255];
}
inline bool is_space(uint32_t c) {
  return c < 128 ? ((c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x20)) : (uprops(c) & bm_unicode::SPACE) != 0;
}
inline bool is_alpha(uint32_t c) {
  return c < 128 ? ((c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z')) : (uprops(c) & bm_unicode::ALPHA) != 0;
}
inline bool is_digit(uint32_t c) {
  return c < 128 ? (c >= '0' && c <= '9') : (uprops(c) & bm_unicode::DIGIT) != 0;
}
inline bool is_alnum(uint32_t c) {
  return c < 128 ? (is_alpha(c) || is_digit(c)) : (uprops(c) & bm_unicode::ALNUM) != 0;
}
inline bool is_upper(uint32_t c) {
  return c < 128 ? (c >= 'A' && c <= 'Z') : (uprops(c) & bm_unicode::UPPER) != 0;
}
// str.lower() of one accepted code point (LOWOK: a single code point)
inline uint32_t lower_cp(uint32_t c) {
  if (c < 128) return (c >= 'A' && c <= 'Z') ? c + 32 : c;
  int lo = 0, hi = bm_unicode::kLowerCount;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bm_unicode::kLower[mid][0] < c)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < bm_unicode::kLowerCount && bm_unicode::kLower[lo][0] == c) ? bm_unicode::kLower[lo][1] : c;
}

// UTF-8 of validated text: the code point at s[i], i advanced past it
inline uint32_t decode(const char* s, size_t& i) {
  const unsigned char c = (unsigned char)s[i];
  if (c < 0x80) {
    ++i;
    return c;
  }
  const unsigned char* u = (const unsigned char*)s + i;
  if (c < 0xE0) {
    i += 2;
    return ((uint32_t)(c & 0x1F) << 6) | (u[1] & 0x3F);
  }
  if (c < 0xF0) {
    i += 3;
    return ((uint32_t)(c & 0x0F) << 12) | ((uint32_t)(u[1] & 0x3F) << 6) | (u[2] & 0x3F);
  }
  i += 4;
  return ((uint32_t)(c & 0x07) << 18) | ((uint32_t)(u[1] & 0x3F) << 12) |
         ((uint32_t)(u[2] & 0x3F) << 6) | (u[3] & 0x3F);
}
// start of the code point that ends at byte i (i > 0)
inline size_t prev_start(const char* s, size_t i) {
  --i;
  while (i > 0 && ((unsigned char)s[i] & 0xC0) == 0x80) --i;
  return i;
}
inline void encode(std::string& o, uint32_t c) {
  if (c < 0x80) {
    o.push_back((char)c);
  } else if (c < 0x800) {
    o.push_back((char)(0xC0 | (c >> 6)));
    o.push_back((char)(0x80 | (c & 0x3F)));
  } else if (c < 0x10000) {
    o.push_back((char)(0xE0 | (c >> 12)));
    o.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
    o.push_back((char)(0x80 | (c & 0x3F)));
  } else {
    o.push_back((char)(0xF0 | (c >> 18)));
    o.push_back((char)(0x80 | ((c >> 12) & 0x3F)));
    o.push_back((char)(0x80 | ((c >> 6) & 0x3F)));
    o.push_back((char)(0x80 | (c & 0x3F)));
  }
}

// the next 8 bytes exist and are all ASCII
inline bool ascii8(const void* p, size_t left) {
  if (left < 8) return false;
  uint64_t w;
  memcpy(&w, p, 8);
  return (w & 0x8080808080808080ull) == 0;
}

// Python's strict UTF-8 decoding (no surrogates, no overlongs, <= U+10FFFF)
bool valid_utf8(const char* d, size_t n) {
  const unsigned char* s = (const unsigned char*)d;
  size_t i = 0;
  while (i < n) {
    if (ascii8(s + i, n - i)) {
      i += 8;
      continue;
    }
    const unsigned char c = s[i];
    if (c < 0x80) {
      ++i;
      continue;
    }
    int len;
    uint32_t cp, minv;
    if (c >= 0xC2 && c <= 0xDF) {
      len = 2, cp = c & 0x1F, minv = 0x80;
    } else if (c >= 0xE0 && c <= 0xEF) {
      len = 3, cp = c & 0x0F, minv = 0x800;
    } else if (c >= 0xF0 && c <= 0xF4) {
      len = 4, cp = c & 0x07, minv = 0x10000;
    } else {
      return false;
    }
    if (i + (size_t)len > n) return false;
    for (int q = 1; q < len; ++q) {
      if ((s[i + q] & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (s[i + q] & 0x3F);
    }
    if (cp < minv || cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF)) return false;
    i += (size_t)len;
  }
  return true;
}

// Text the native path can normalize exactly (see the contract above).
bool text_ok(const char* s, size_t n) {
  size_t i = 0;
  bool prev_nonstarter = false;
  while (i < n) {
    if (ascii8(s + i, n - i)) {
      i += 8;
      prev_nonstarter = false;
      continue;
    }
    const uint32_t cp = decode(s, i);
    if (cp < 128) {
      prev_nonstarter = false;
      continue;
    }
    const uint8_t p = uprops(cp);
    if (!(p & bm_unicode::NFCYES) || !(p & bm_unicode::LOWOK)) return false;
    const bool ns = !(p & bm_unicode::CCC0);
    if (ns && prev_nonstarter) return false;
    prev_nonstarter = ns;
  }
  return true;
}

// Open-addressing table of byte strings (arena-backed, looked up by pointer
// + length, no allocation per lookup) -> int32 value.
struct StrTable {
  struct E {
    uint64_t h;
    uint32_t off, len;
    int32_t val;
  };
  std::vector<uint32_t> slot;  // entry index + 1; 0 = empty
  std::vector<E> ents;
  std::string arena;
  uint32_t mask = 0;
  StrTable() { rehash(1u << 12); }
  static uint64_t hash(const char* s, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull ^ n;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      memcpy(&w, s + i, 8);
      h = (h ^ w) * 0x100000001b3ull;
      h ^= h >> 29;
    }
    uint64_t w = 0;
    memcpy(&w, s + i, n - i);
    h = (h ^ w) * 0x100000001b3ull;
    h ^= h >> 32;
    return h * 0x9E3779B97F4A7C15ull;
  }
  void rehash(uint32_t cap) {
    slot.assign(cap, 0);
    mask = cap - 1;
    for (uint32_t q = 0; q < ents.size(); ++q) {
      uint32_t s = (uint32_t)(ents[q].h >> 32) & mask;
      while (slot[s]) s = (s + 1) & mask;
      slot[s] = q + 1;
    }
  }
  // value of the string, or -1
  int32_t find(const char* s, size_t n, uint64_t h) const {
    uint32_t q = (uint32_t)(h >> 32) & mask;
    while (slot[q]) {
      const E& e = ents[slot[q] - 1];
      if (e.h == h && e.len == n && memcmp(arena.data() + e.off, s, n) == 0) return e.val;
      q = (q + 1) & mask;
    }
    return -1;
  }
  int32_t find(const char* s, size_t n) const { return find(s, n, hash(s, n)); }
  // insert a string known to be absent
  void insert(const char* s, size_t n, uint64_t h, int32_t val) {
    if ((ents.size() + 1) * 2 > slot.size()) rehash((uint32_t)slot.size() * 2);
    E e{h, (uint32_t)arena.size(), (uint32_t)n, val};
    arena.append(s, n);
    ents.push_back(e);
    uint32_t q = (uint32_t)(h >> 32) & mask;
    while (slot[q]) q = (q + 1) & mask;
    slot[q] = (uint32_t)ents.size();
  }
  size_t size() const { return ents.size(); }
};

struct Doc {
  std::string id, src_lang, tgt_lang;
  int32_t src0 = 0, n = 0, tgt0 = 0, m = 0;
};

// std::vector without value-initialization on resize (the merge fills every
// slot, so zeroing hundreds of MB first would only cost time)
template <class T>
struct NoInit : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInit<U>;
  };
  NoInit() = default;
  template <class U>
  NoInit(const NoInit<U>&) {}
  template <class U>
  void construct(U* p) noexcept {
    ::new ((void*)p) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new ((void*)p) U(std::forward<A>(a)...);
  }
};
template <class T>
using pvec = std::vector<T, NoInit<T>>;

struct Ingest {
  // packed sentences (pack.py layout)
  pvec<int32_t> n_tok, n_punct, n_alpha, tok_off{0}, tok_id, dig_off{0}, dig_id;
  pvec<uint32_t> tok_alpha;
  pvec<int32_t> src0, n, tgt0, m;
  // interned token strings (normalized tokens and raw digit tokens) -> id
  StrTable ids;
  // per sentence: raw text and the interned id of its normalized text (merge
  // key; unique within a chunk -- keys are only compared inside one document)
  std::string raw;
  pvec<int64_t> raw_off{0};
  pvec<int32_t> norm_key;
  StrTable norm_ids;
  std::string norm_tmp;
  // after ingest: every sentence's raw text (a merged ingest keeps each
  // chunk's text buffer in raw_store instead of copying them together)
  std::vector<std::string> raw_store;
  pvec<const char*> sent_ptr;
  pvec<int32_t> sent_len;
  std::vector<Doc> docs;
  std::vector<int64_t> skipped_lines;  // empty-side pairs dropped at load
  std::vector<std::string> skipped_ids, skipped_side;
  // lexicon CSR over the id space (bm_ingest_lexicon)
  std::vector<int32_t> fwd_off, fwd_cand, rev_off, rev_cand;
  // raw token -> (normalized id, digit id, isalpha, punctuation-only)
  struct TokInfo {
    int32_t nid, did;
    bool alpha, punct;
  };
  StrTable tok_cache;
  std::vector<TokInfo> tok_info;
  std::string out;  // TSV bytes of bm_ingest_emit
  std::string err;
  // gold sets (bm_ingest_gold_jsonl, tuner.py:157-203): per document the
  // ascending unique keys i * m + j of its "gold" pairs
  bool gold_mode = false;
  int64_t n_lines = 0;                 // lines of the ingested byte range
  std::string seen_src, seen_tgt;      // bm_ingest_seen: NUL-separated strings
  pvec<int64_t> gold_keys;
  std::vector<int64_t> gold_cnt;  // per document (merged into gold_off)
  std::vector<int64_t> gold_off;
  std::vector<std::pair<int32_t, int32_t>> alpha_scratch;
  std::vector<int32_t> digit_scratch;
  std::string tmp;

  int32_t intern(const char* s, size_t n) {
    const uint64_t h = StrTable::hash(s, n);
    const int32_t v = ids.find(s, n, h);
    if (v >= 0) return v;
    const int32_t k = (int32_t)ids.size();
    ids.insert(s, n, h, k);
    return k;
  }
};

// ------------------------------------------------------------------ tokens
// tokenize (corpus.py:28): maximal alnum runs ([^\W_]+) or one non-space char
template <class F>
void for_tokens(const char* s, size_t len, F&& f) {
  size_t i = 0;
  while (i < len) {
    const size_t st = i;
    const uint32_t c = decode(s, i);
    if (is_space(c)) continue;
    if (is_alnum(c)) {
      size_t j = i;
      while (j < len) {
        size_t k2 = j;
        if (!is_alnum(decode(s, k2))) break;
        j = k2;
      }
      f(s + st, j - st);
      i = j;
    } else {
      f(s + st, i - st);
    }
  }
}

// normalize (corpus.py:38-40): NFC (identity on accepted text), lower(),
// " ".join(split()); appended to o
void normalize_into(std::string& o, const char* s, size_t len) {
  const size_t start = o.size();
  size_t i = 0;
  bool pending_space = false;
  while (i < len) {
    const uint32_t c = decode(s, i);
    if (is_space(c)) {
      pending_space = o.size() > start;
      continue;
    }
    if (pending_space) {
      o.push_back(' ');
      pending_space = false;
    }
    encode(o, lower_cp(c));
  }
}

// Packer.add_sentence (pack.py) for one raw sentence
bool add_sentence(Ingest& g, const char* s, size_t len) {
  int32_t T = 0, P = 0, A = 0;
  auto& alpha = g.alpha_scratch;  // (normalized id, isalpha count)
  auto& digits = g.digit_scratch;
  alpha.clear();
  digits.clear();
  for_tokens(s, len, [&](const char* t, size_t tl) {
    const uint64_t h = StrTable::hash(t, tl);
    int32_t ix = g.tok_cache.find(t, tl, h);
    if (ix < 0) {
      Ingest::TokInfo ti;
      g.tmp.clear();
      normalize_into(g.tmp, t, tl);
      ti.nid = g.intern(g.tmp.data(), g.tmp.size());
      bool all_alpha = tl > 0, all_digit = tl > 0, any_alnum = false;
      for (size_t q = 0; q < tl;) {
        const uint32_t c = decode(t, q);
        all_alpha &= is_alpha(c);
        all_digit &= is_digit(c);
        any_alnum |= is_alnum(c);
      }
      ti.did = all_digit ? g.intern(t, tl) : -1;
      ti.alpha = all_alpha;
      ti.punct = !any_alnum;
      ix = (int32_t)g.tok_info.size();
      g.tok_info.push_back(ti);
      g.tok_cache.insert(t, tl, h, ix);
    }
    const Ingest::TokInfo ti = g.tok_info[ix];
    ++T;
    P += ti.punct ? 1 : 0;
    bool found = false;
    for (auto& pr : alpha)
      if (pr.first == ti.nid) {
        pr.second += ti.alpha ? 1 : 0;
        found = true;
        break;
      }
    if (!found) alpha.emplace_back(ti.nid, ti.alpha ? 1 : 0);
    if (ti.alpha) ++A;
    if (ti.did >= 0 && std::find(digits.begin(), digits.end(), ti.did) == digits.end())
      digits.push_back(ti.did);
  });
  std::sort(alpha.begin(), alpha.end());
  std::sort(digits.begin(), digits.end());
  for (auto& pr : alpha) {
    g.tok_id.push_back(pr.first);
    g.tok_alpha.push_back((uint32_t)pr.second);
  }
  g.n_tok.push_back(T);
  g.n_punct.push_back(P);
  g.n_alpha.push_back(A);
  g.tok_off.push_back((int32_t)g.tok_id.size());
  g.dig_id.insert(g.dig_id.end(), digits.begin(), digits.end());
  g.dig_off.push_back((int32_t)g.dig_id.size());
  // raw + normalized text of the Sentence object
  g.raw.append(s, len);
  g.raw_off.push_back((int64_t)g.raw.size());
  g.norm_tmp.clear();
  normalize_into(g.norm_tmp, s, len);
  const char* nm = g.norm_tmp.data();
  const size_t nl = g.norm_tmp.size();
  const uint64_t h = StrTable::hash(nm, nl);
  int32_t nk = g.norm_ids.find(nm, nl, h);
  if (nk < 0) {
    nk = (int32_t)g.norm_ids.size();
    g.norm_ids.insert(nm, nl, h, nk);
  }
  g.norm_key.push_back(nk);
  return true;
}

const char* const kAbbrev[] = {"dr", "mr", "mrs", "ms", "prof", "st", "no", "vs", "etc"};

bool is_abbrev(const char* s, size_t len) {
  for (const char* a : kAbbrev) {
    const size_t al = strlen(a);
    size_t i = 0, q = 0;
    bool eq = true;
    while (i < len && q < al && eq) eq = lower_cp(decode(s, i)) == (uint32_t)(unsigned char)a[q++];
    if (eq && i == len && q == al) return true;
  }
  return false;
}

// segment_sentences (corpus.py:92-126): sentence spans [begin, end) of text
// (byte offsets at code-point boundaries)
void segment(const std::string& text, std::vector<std::pair<size_t, size_t>>& spans) {
  const size_t size = text.size();
  const char* s = text.data();
  size_t pos = 0;
  while (pos < size) {
    size_t nx = pos;
    if (!is_space(decode(s, nx))) break;
    pos = nx;
  }
  size_t begin = pos;
  while (pos < size) {
    size_t next = pos;
    const uint32_t ch = decode(s, next);
    if (ch != '.' && ch != '!' && ch != '?') {
      pos = next;
      continue;
    }
    if (ch == '.') {
      size_t st = pos;
      while (st > 0) {
        const size_t ps = prev_start(s, st);
        size_t q = ps;
        if (!is_alpha(decode(s, q))) break;
        st = ps;
      }
      if (is_abbrev(s + st, pos - st)) {
        pos = next;
        continue;
      }
    }
    size_t nxt = pos + 1;
    size_t q = nxt;
    if (nxt < size && is_space(decode(s, q))) {
      nxt = q;
      while (nxt < size) {
        size_t r = nxt;
        if (!is_space(decode(s, r))) break;
        nxt = r;
      }
      size_t r = nxt;
      if (nxt < size) {
        const uint32_t c2 = decode(s, r);
        if (is_upper(c2) || is_digit(c2)) {
          spans.emplace_back(begin, pos + 1);
          begin = pos = nxt;
          continue;
        }
      }
    }
    pos = next;
  }
  size_t end = size;
  while (end > begin) {
    const size_t ps = prev_start(s, end);
    size_t q = ps;
    if (!is_space(decode(s, q))) break;
    end = ps;
  }
  if (end > begin) spans.emplace_back(begin, end);
}

// ------------------------------------------------------------------ JSON
// A validating parser for the subset the native path accepts. Anything it
// does not accept makes the whole file fall back to Python (which then also
// raises the reference's DataError for genuinely malformed input).
struct Json {
  const char* p;
  const char* e;
  bool ok = true;
  void ws() {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool lit(const char* w) {
    const size_t l = strlen(w);
    if ((size_t)(e - p) >= l && memcmp(p, w, l) == 0) {
      p += l;
      return true;
    }
    return false;
  }
  bool hex4(unsigned& v) {
    if (e - p < 4) return false;
    v = 0;
    for (int q = 0; q < 4; ++q) {
      const char h = *p++;
      v <<= 4;
      if (h >= '0' && h <= '9') v |= (unsigned)(h - '0');
      else if (h >= 'a' && h <= 'f') v |= (unsigned)(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') v |= (unsigned)(h - 'A' + 10);
      else return false;
    }
    return true;
  }
  // JSON string -> UTF-8 (raw control chars and lone surrogates: fail)
  bool str(std::string& out) {
    out.clear();
    if (p >= e || *p != '"') return false;
    ++p;
    while (p < e) {
      const unsigned char c = (unsigned char)*p++;
      if (c == '"') return true;
      if (c < 0x20) return false;
      if (c != '\\') {
        out.push_back((char)c);  // raw UTF-8 (the file was validated)
        continue;
      }
      if (p >= e) return false;
      const char x = *p++;
      switch (x) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          unsigned v;
          if (!hex4(v)) return false;
          if (v >= 0xD800 && v <= 0xDBFF) {  // a surrogate pair or nothing
            unsigned lo;
            if (e - p < 6 || p[0] != '\\' || p[1] != 'u') return false;
            p += 2;
            if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return false;
            v = 0x10000 + ((v - 0xD800) << 10) + (lo - 0xDC00);
          } else if (v >= 0xDC00 && v <= 0xDFFF) {
            return false;
          }
          encode(out, v);
          break;
        }
        default: return false;
      }
    }
    return false;
  }
  // JSON number; *is_int: matches -?(0|[1-9][0-9]*) with no fraction/exponent
  bool num(std::string& text, bool* is_int) {
    const char* b = p;
    if (p < e && *p == '-') ++p;
    if (p >= e) return false;
    if (*p == '0') {
      ++p;
    } else if (*p >= '1' && *p <= '9') {
      while (p < e && is_digit((unsigned char)*p)) ++p;
    } else {
      return false;
    }
    *is_int = true;
    if (p < e && *p == '.') {
      *is_int = false;
      ++p;
      if (p >= e || !is_digit((unsigned char)*p)) return false;
      while (p < e && is_digit((unsigned char)*p)) ++p;
    }
    if (p < e && (*p == 'e' || *p == 'E')) {
      *is_int = false;
      ++p;
      if (p < e && (*p == '+' || *p == '-')) ++p;
      if (p >= e || !is_digit((unsigned char)*p)) return false;
      while (p < e && is_digit((unsigned char)*p)) ++p;
    }
    text.assign(b, p);
    return true;
  }
  // any value, validated and discarded (NaN/Infinity are refused)
  bool skip(int depth = 0) {
    if (depth > 64) return false;
    ws();
    if (p >= e) return false;
    std::string tmp;
    if (*p == '"') return str(tmp);
    if (*p == '{') {
      ++p;
      ws();
      if (p < e && *p == '}') {
        ++p;
        return true;
      }
      for (;;) {
        ws();
        if (!str(tmp)) return false;
        ws();
        if (p >= e || *p != ':') return false;
        ++p;
        if (!skip(depth + 1)) return false;
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == '}') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (*p == '[') {
      ++p;
      ws();
      if (p < e && *p == ']') {
        ++p;
        return true;
      }
      for (;;) {
        if (!skip(depth + 1)) return false;
        ws();
        if (p < e && *p == ',') {
          ++p;
          continue;
        }
        if (p < e && *p == ']') {
          ++p;
          return true;
        }
        return false;
      }
    }
    if (lit("true") || lit("false") || lit("null")) return true;
    bool is_int;
    return num(tmp, &is_int);
  }
};

// A text field: a string (segmented) or a list of strings (one sentence each,
// blank ones dropped). kind: 0 absent, 1 string, 2 list.
struct Field {
  int kind = 0;
  std::string text;
  std::vector<std::string> items;
};

bool parse_field(Json& js, Field& f) {
  js.ws();
  if (js.p < js.e && *js.p == '"') {
    f.kind = 1;
    f.items.clear();
    return js.str(f.text);
  }
  if (js.p < js.e && *js.p == '[') {
    f.kind = 2;
    f.items.clear();
    ++js.p;
    js.ws();
    if (js.p < js.e && *js.p == ']') {
      ++js.p;
      return true;
    }
    for (;;) {
      js.ws();
      std::string s;
      if (!js.str(s)) return false;  // non-string items: Python raises DataError
      f.items.push_back(std::move(s));
      js.ws();
      if (js.p < js.e && *js.p == ',') {
        ++js.p;
        continue;
      }
      if (js.p < js.e && *js.p == ']') {
        ++js.p;
        return true;
      }
      return false;
    }
  }
  return false;
}

// str(value) for id / lang: strings and integers only
bool parse_scalar(Json& js, std::string& out) {
  js.ws();
  if (js.p < js.e && *js.p == '"') return js.str(out);
  bool is_int = false;
  std::string t;
  if (!js.num(t, &is_int) || !is_int) return false;
  // str(int): no leading '-0'
  if (t == "-0") t = "0";
  out = t;
  return true;
}

// A "gold" value: a list of [i, j] integer pairs. Anything else (floats,
// booleans, nesting, numbers past int32) is left to the Python reader, which
// raises the reference's error.
bool parse_gold(Json& js, std::vector<std::pair<int64_t, int64_t>>& out) {
  out.clear();
  js.ws();
  if (js.p >= js.e || *js.p != '[') return false;
  ++js.p;
  js.ws();
  if (js.p < js.e && *js.p == ']') {
    ++js.p;
    return true;
  }
  for (;;) {
    js.ws();
    if (js.p >= js.e || *js.p != '[') return false;
    ++js.p;
    int64_t v[2];
    for (int q = 0; q < 2; ++q) {
      js.ws();
      std::string t;
      bool is_int = false;
      if (!js.num(t, &is_int) || !is_int || t.size() > 10) return false;
      v[q] = strtoll(t.c_str(), nullptr, 10);
      if (v[q] < INT32_MIN || v[q] > INT32_MAX) return false;
      js.ws();
      if (q == 0) {
        if (js.p >= js.e || *js.p != ',') return false;
        ++js.p;
      }
    }
    if (js.p >= js.e || *js.p != ']') return false;
    ++js.p;
    out.emplace_back(v[0], v[1]);
    js.ws();
    if (js.p < js.e && *js.p == ',') {
      ++js.p;
      continue;
    }
    if (js.p < js.e && *js.p == ']') {
      ++js.p;
      return true;
    }
    return false;
  }
}

// The sentences of a field as (pointer, length) spans: a string is
// segmented, a list contributes its non-blank items (corpus.py:114-121).
void field_spans(const Field& f, std::vector<std::pair<const char*, size_t>>& out) {
  out.clear();
  if (f.kind == 1) {
    std::vector<std::pair<size_t, size_t>> sp;
    segment(f.text, sp);
    for (auto& x : sp) out.emplace_back(f.text.data() + x.first, x.second - x.first);
    return;
  }
  for (const std::string& s : f.items) {
    bool blank = true;
    for (size_t i = 0; i < s.size() && blank;) blank = is_space(decode(s.data(), i));
    if (!blank) out.emplace_back(s.data(), s.size());
  }
}

// One line: returns 1 = document added, 0 = skipped (empty side), -1 = fallback
int parse_line(Ingest& g, const char* b, const char* e, int64_t lineno) {
  Json js{b, e};
  js.ws();
  if (js.p >= js.e || *js.p != '{') return -1;
  ++js.p;
  std::string key, id, sl, tl;
  bool has_id = false, has_sl = false, has_tl = false, has_gold = false;
  Field src, tgt;
  std::vector<std::pair<int64_t, int64_t>> gold;
  js.ws();
  if (js.p < js.e && *js.p == '}') return -1;  // missing fields: Python raises
  for (;;) {
    js.ws();
    if (!js.str(key)) return -1;
    js.ws();
    if (js.p >= js.e || *js.p != ':') return -1;
    ++js.p;
    // duplicate keys: the last occurrence wins (json.loads)
    if (key == "id") {
      if (!parse_scalar(js, id)) return -1;
      has_id = true;
    } else if (key == "src_lang") {
      if (!parse_scalar(js, sl)) return -1;
      has_sl = true;
    } else if (key == "tgt_lang") {
      if (!parse_scalar(js, tl)) return -1;
      has_tl = true;
    } else if (key == "src") {
      if (!parse_field(js, src)) return -1;
    } else if (key == "tgt") {
      if (!parse_field(js, tgt)) return -1;
    } else if (g.gold_mode && key == "gold") {
      if (!parse_gold(js, gold)) return -1;
      has_gold = true;
    } else if (!js.skip()) {
      return -1;
    }
    js.ws();
    if (js.p < js.e && *js.p == ',') {
      ++js.p;
      continue;
    }
    if (js.p < js.e && *js.p == '}') {
      ++js.p;
      break;
    }
    return -1;
  }
  js.ws();
  if (js.p != js.e) return -1;  // trailing data
  if (!has_id || !has_sl || !has_tl || src.kind == 0 || tgt.kind == 0) return -1;
  if (sl == tl) return -1;
  // ids and languages cross the C ABI as NUL-terminated strings
  for (const std::string* s : {&id, &sl, &tl})
    if (s->find('\0') != std::string::npos) return -1;
  // text the native normalizer reproduces exactly (else: Python path)
  for (const Field* f : {&src, &tgt}) {
    if (f->kind == 1 && !text_ok(f->text.data(), f->text.size())) return -1;
    for (const std::string& it : f->items)
      if (!text_ok(it.data(), it.size())) return -1;
  }
  Doc d;
  d.id = id;
  d.src_lang = sl;
  d.tgt_lang = tl;
  std::vector<std::pair<const char*, size_t>> ss, ts;
  field_spans(src, ss);
  field_spans(tgt, ts);
  if (g.gold_mode) {
    // load_gold_set raises for an empty side, a missing "gold" or a pair out
    // of bounds: the Python reader reproduces the message
    if (ss.empty() || ts.empty() || !has_gold) return -1;
    const int64_t n = (int64_t)ss.size(), m = (int64_t)ts.size();
    const size_t k0 = g.gold_keys.size();
    for (auto& c : gold) {
      if (c.first < 0 || c.first >= n || c.second < 0 || c.second >= m) return -1;
      g.gold_keys.push_back(c.first * m + c.second);
    }
    std::sort(g.gold_keys.begin() + (long)k0, g.gold_keys.end());
    g.gold_keys.resize((size_t)(std::unique(g.gold_keys.begin() + (long)k0, g.gold_keys.end()) -
                                g.gold_keys.begin()));
    g.gold_cnt.push_back((int64_t)(g.gold_keys.size() - k0));
  }
  if (ss.empty() || ts.empty()) {
    // load_document_pairs skips the pair before anything is packed
    g.skipped_lines.push_back(lineno);
    g.skipped_ids.push_back(d.id);
    g.skipped_side.push_back(ss.empty() ? "src" : "tgt");
    return 0;
  }
  d.src0 = (int32_t)g.n_tok.size();
  d.n = (int32_t)ss.size();
  for (auto& x : ss)
    if (!add_sentence(g, x.first, x.second)) return -1;
  d.tgt0 = (int32_t)g.n_tok.size();
  d.m = (int32_t)ts.size();
  for (auto& x : ts)
    if (!add_sentence(g, x.first, x.second)) return -1;
  g.src0.push_back(d.src0);
  g.n.push_back(d.n);
  g.tgt0.push_back(d.tgt0);
  g.m.push_back(d.m);
  g.docs.push_back(std::move(d));
  return 1;
}

// Merge chunks parsed independently (local id spaces) into part[0]. Local
// ids are in first-appearance order within their chunk, so re-interning each
// chunk's strings in chunk order gives exactly the ids one sequential pass
// assigns (sequential, cheap: unique token strings only). The arrays are then
// rewritten chunk-parallel into preallocated global slices, each sentence's
// id lists re-sorted under the new ids.
void merge_parts(std::vector<Ingest*>& part) {
  const size_t np = part.size();
  Ingest& G = *part[0];
  const bool trace = getenv("BM_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[bm trace]   merge %-10s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  };
  std::vector<std::vector<int32_t>> rid(np);
  for (size_t t = 1; t < np; ++t) {
    Ingest& L = *part[t];
    rid[t].resize(L.ids.size());
    for (const StrTable::E& e : L.ids.ents)
      rid[t][(size_t)e.val] = G.intern(L.ids.arena.data() + e.off, e.len);
  }
  lap("intern");
  // slice bases
  std::vector<size_t> sb(np + 1, 0), tb(np + 1, 0), db(np + 1, 0), kb(np + 1, 0);
  for (size_t t = 0; t < np; ++t) {
    Ingest& L = *part[t];
    sb[t + 1] = sb[t] + L.n_tok.size();
    tb[t + 1] = tb[t] + L.tok_id.size();
    db[t + 1] = db[t] + L.dig_id.size();
    kb[t + 1] = kb[t] + L.docs.size();
  }
  // chunk texts move (no copy); sentence pointers into them are set below
  G.raw_store.resize(np);
  for (size_t t = 0; t < np; ++t) G.raw_store[t] = std::move(part[t]->raw);
  G.sent_ptr.resize(sb[np]);
  G.sent_len.resize(sb[np]);
  G.n_tok.resize(sb[np]);
  G.n_punct.resize(sb[np]);
  G.n_alpha.resize(sb[np]);
  G.norm_key.resize(sb[np]);
  G.tok_off.resize(sb[np] + 1);
  G.dig_off.resize(sb[np] + 1);
  G.tok_id.resize(tb[np]);
  G.tok_alpha.resize(tb[np]);
  G.dig_id.resize(db[np]);
  G.docs.resize(kb[np]);
  G.src0.resize(kb[np]);
  G.n.resize(kb[np]);
  G.tgt0.resize(kb[np]);
  G.m.resize(kb[np]);
  lap("resize");
  auto fill = [&](size_t t) {
    Ingest& L = *part[t];
    const size_t ns = L.n_tok.size(), s0 = sb[t];
    std::copy(L.n_tok.begin(), L.n_tok.end(), G.n_tok.begin() + s0);
    std::copy(L.n_punct.begin(), L.n_punct.end(), G.n_punct.begin() + s0);
    std::copy(L.n_alpha.begin(), L.n_alpha.end(), G.n_alpha.begin() + s0);
    const char* text = G.raw_store[t].data();
    for (size_t s = 0; s < ns; ++s) {
      G.sent_ptr[s0 + s] = text + L.raw_off[s];
      G.sent_len[s0 + s] = (int32_t)(L.raw_off[s + 1] - L.raw_off[s]);
    }
    std::vector<std::pair<int32_t, uint32_t>> ta;
    for (size_t s = 0; s < ns; ++s) {
      const int32_t a = L.tok_off[s], b = L.tok_off[s + 1];
      ta.clear();
      for (int32_t q = a; q < b; ++q) ta.emplace_back(rid[t][(size_t)L.tok_id[q]], L.tok_alpha[q]);
      std::sort(ta.begin(), ta.end());
      for (int32_t q = a; q < b; ++q) {
        G.tok_id[tb[t] + (size_t)q] = ta[(size_t)(q - a)].first;
        G.tok_alpha[tb[t] + (size_t)q] = ta[(size_t)(q - a)].second;
      }
      G.tok_off[s0 + s + 1] = (int32_t)(tb[t] + (size_t)b);
      const int32_t c = L.dig_off[s], d = L.dig_off[s + 1];
      for (int32_t q = c; q < d; ++q) G.dig_id[db[t] + (size_t)q] = rid[t][(size_t)L.dig_id[q]];
      std::sort(G.dig_id.begin() + (long)(db[t] + (size_t)c), G.dig_id.begin() + (long)(db[t] + (size_t)d));
      G.dig_off[s0 + s + 1] = (int32_t)(db[t] + (size_t)d);
      // merge keys are compared only within a document, and a document never
      // spans chunks: chunk-local keys need no remapping
      G.norm_key[s0 + s] = L.norm_key[s];
    }
    for (size_t q = 0; q < L.docs.size(); ++q) {
      Doc D = std::move(L.docs[q]);
      D.src0 += (int32_t)s0;
      D.tgt0 += (int32_t)s0;
      const size_t k = kb[t] + q;
      G.src0[k] = D.src0;
      G.n[k] = D.n;
      G.tgt0[k] = D.tgt0;
      G.m[k] = D.m;
      G.docs[k] = std::move(D);
    }
  };
  {
    std::vector<std::thread> th;
    for (size_t t = 1; t < np; ++t) th.emplace_back(fill, t);
    // part 0 is G itself: its arrays are in place, only its pointers are new
    const char* text = G.raw_store[0].data();
    for (size_t s = 0; s < sb[1]; ++s) {
      G.sent_ptr[s] = text + G.raw_off[s];
      G.sent_len[s] = (int32_t)(G.raw_off[s + 1] - G.raw_off[s]);
    }
    for (auto& x : th) x.join();
  }
  G.raw_off.clear();
  G.raw_off.shrink_to_fit();
  lap("fill");
  if (G.gold_mode) {  // documents keep their order: concatenate the key lists
    for (size_t t = 1; t < np; ++t) {
      Ingest& L = *part[t];
      G.gold_keys.insert(G.gold_keys.end(), L.gold_keys.begin(), L.gold_keys.end());
      G.gold_cnt.insert(G.gold_cnt.end(), L.gold_cnt.begin(), L.gold_cnt.end());
    }
    G.gold_off.assign(G.gold_cnt.size() + 1, 0);
    for (size_t k = 0; k < G.gold_cnt.size(); ++k) G.gold_off[k + 1] = G.gold_off[k] + G.gold_cnt[k];
  }
  for (size_t t = 1; t < np; ++t) {
    Ingest& L = *part[t];
    G.skipped_lines.insert(G.skipped_lines.end(), L.skipped_lines.begin(), L.skipped_lines.end());
    G.skipped_ids.insert(G.skipped_ids.end(), L.skipped_ids.begin(), L.skipped_ids.end());
    G.skipped_side.insert(G.skipped_side.end(), L.skipped_side.begin(), L.skipped_side.end());
  }
}

}  // namespace bm_ingest

using bm_ingest::Ingest;

extern "C" {

// [b0, b1) of the file (b1 < 0: to the end), its first line numbered line0 + 1
static int ingest_impl(const char* path, bool gold, int64_t b0, int64_t b1, int64_t line0,
                       void** handle, char* why, int32_t why_len) {
  auto fail_why = [&](const char* w) {
    if (why && why_len > 0) snprintf(why, (size_t)why_len, "%s", w);
    return BM_EUNSUPPORTED;
  };
  *handle = nullptr;
  const bool trace = getenv("BM_TRACE") != nullptr;
  auto tr0 = std::chrono::steady_clock::now();
  // the file is mapped read-only (nothing keeps pointers into it past this
  // call: sentence texts are copied into the chunk buffers)
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail_why("cannot open file");
  struct stat sb;
  if (fstat(fd, &sb) != 0) {
    close(fd);
    return fail_why("cannot stat file");
  }
  const size_t fsize = (size_t)sb.st_size;
  void* map = fsize ? mmap(nullptr, fsize, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0) : nullptr;
  close(fd);
  if (fsize && map == MAP_FAILED) return fail_why("cannot map file");
  struct Unmap {
    void* p;
    size_t n;
    ~Unmap() {
      if (p) munmap(p, n);
    }
  } unmap{fsize ? map : nullptr, fsize};
  if (b0 < 0 || (size_t)b0 > fsize) return fail_why("bad byte range");
  const size_t end = (b1 < 0 || (size_t)b1 > fsize) ? fsize : (size_t)b1;
  if ((size_t)b0 > end) return fail_why("bad byte range");
  const struct {
    const char* p;
    size_t n;
    const char* data() const { return p; }
    size_t size() const { return n; }
  } data{fsize ? (const char*)map + b0 : "", end - (size_t)b0};
  if (!bm_ingest::valid_utf8(data.data(), data.size())) return fail_why("not valid UTF-8");
  // lines: text-mode splitting, \n, \r\n and \r end a line
  struct Line {
    size_t b, e;
  };
  std::vector<Line> lines;
  {
    const char* base = data.data();
    size_t i = 0;
    const size_t size = data.size();
    while (i < size) {
      size_t q = i;
      while (q < size && base[q] != '\n' && base[q] != '\r') ++q;
      lines.push_back(Line{i, q});
      if (q < size && base[q] == '\r' && q + 1 < size && base[q + 1] == '\n') ++q;
      i = q + 1;
    }
  }
  // chunks of about equal bytes, parsed in parallel into local id spaces
  const size_t nlines = lines.size();
  unsigned hw = std::thread::hardware_concurrency();
  const char* env = getenv("BM_INGEST_THREADS");
  if (env) hw = (unsigned)atoi(env);
  const size_t nthr = std::max<size_t>(1, std::min<size_t>({(size_t)std::max(hw, 1u), (size_t)32,
                                                            nlines / 64 + 1}));
  std::vector<size_t> cut(nthr + 1, nlines);
  cut[0] = 0;
  {
    const size_t per = data.size() / nthr + 1;
    size_t t = 1;
    for (size_t q = 0; q < nlines && t < nthr; ++q)
      if (lines[q].b >= t * per) cut[t++] = q;
    for (; t < nthr; ++t) cut[t] = nlines;
  }
  std::vector<Ingest*> part(nthr, nullptr);
  std::vector<int64_t> bad(nthr, -1);
  auto work = [&](size_t t) {
    Ingest* L = new Ingest();
    L->gold_mode = gold;
    part[t] = L;
    const char* base = data.data();
    for (size_t q = cut[t]; q < cut[t + 1]; ++q) {
      const char* b = base + lines[q].b;
      const char* e = base + lines[q].e;
      bool blank = true;
      for (size_t i = 0; i < (size_t)(e - b) && blank;) blank = bm_ingest::is_space(bm_ingest::decode(b, i));
      if (blank) continue;
      if (bm_ingest::parse_line(*L, b, e, line0 + (int64_t)q + 1) < 0) {
        bad[t] = line0 + (int64_t)q + 1;
        return;
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  if (trace)
    fprintf(stderr, "[bm trace] ingest read + validate + lines %.3f ms\n",
            std::chrono::duration<double, std::milli>(t0 - tr0).count());
  if (nthr == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < nthr; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  for (size_t t = 0; t < nthr; ++t) {
    if (bad[t] >= 0) {
      char msg[160];
      snprintf(msg, sizeof(msg), "line %lld: %s", (long long)bad[t],
               part[t]->err.empty() ? "outside the native JSON subset" : part[t]->err.c_str());
      for (Ingest* x : part) delete x;
      return fail_why(msg);
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  Ingest* g = part[0];
  bm_ingest::merge_parts(part);  // also sets the sentence text pointers
  for (size_t t = 1; t < nthr; ++t) delete part[t];
  if (trace) {
    auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[bm trace] ingest %zu threads: parse %.3f ms, merge %.3f ms\n", nthr,
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  g->n_lines = (int64_t)nlines;
  *handle = g;
  return BM_OK;
}

int bm_ingest_jsonl(const char* path, void** handle, char* why, int32_t why_len) {
  return ingest_impl(path, false, 0, -1, 0, handle, why, why_len);
}

int bm_ingest_jsonl_range(const char* path, int64_t b0, int64_t b1, int64_t line0, void** handle,
                          int64_t* n_lines, char* why, int32_t why_len) {
  const int rc = ingest_impl(path, false, b0, b1, line0, handle, why, why_len);
  if (rc == BM_OK) *n_lines = ((Ingest*)*handle)->n_lines;
  return rc;
}

int bm_ingest_gold_jsonl(const char* path, void** handle, char* why, int32_t why_len) {
  const int rc = ingest_impl(path, true, 0, -1, 0, handle, why, why_len);
  if (rc == BM_OK && ((Ingest*)*handle)->docs.empty()) {  // load_gold_set raises
    bm_ingest_free(*handle);
    *handle = nullptr;
    if (why && why_len > 0) snprintf(why, (size_t)why_len, "%s", "empty gold set");
    return BM_EUNSUPPORTED;
  }
  return rc;
}

int bm_ingest_gold(void* h, const int64_t** keys, const int64_t** off, int64_t* n_keys) {
  Ingest* g = (Ingest*)h;
  if (!g->gold_mode) return BM_EINVAL;
  *keys = g->gold_keys.data();
  *off = g->gold_off.data();
  *n_keys = (int64_t)g->gold_keys.size();
  return BM_OK;
}

void bm_ingest_free(void* h) { delete (Ingest*)h; }

int bm_ingest_view(void* h, bm_ingest_arrays* v) {
  Ingest* g = (Ingest*)h;
  v->n_sent = (int32_t)g->n_tok.size();
  v->n_docs = (int32_t)g->docs.size();
  v->n_ids = (int32_t)g->ids.size();
  v->n_tok_entries = (int64_t)g->tok_id.size();
  v->n_dig_entries = (int64_t)g->dig_id.size();
  v->n_tok = g->n_tok.data();
  v->n_punct = g->n_punct.data();
  v->n_alpha = g->n_alpha.data();
  v->tok_off = g->tok_off.data();
  v->tok_id = g->tok_id.data();
  v->tok_alpha = g->tok_alpha.data();
  v->dig_off = g->dig_off.data();
  v->dig_id = g->dig_id.data();
  v->src0 = g->src0.data();
  v->n = g->n.data();
  v->tgt0 = g->tgt0.data();
  v->m = g->m.data();
  v->n_skipped = (int32_t)g->skipped_lines.size();
  return BM_OK;
}

// Document k: id / src_lang / tgt_lang as NUL-terminated strings.
int bm_ingest_doc(void* h, int32_t k, const char** id, const char** src_lang,
                  const char** tgt_lang) {
  Ingest* g = (Ingest*)h;
  if (k < 0 || k >= (int32_t)g->docs.size()) return BM_EINVAL;
  *id = g->docs[k].id.c_str();
  *src_lang = g->docs[k].src_lang.c_str();
  *tgt_lang = g->docs[k].tgt_lang.c_str();
  return BM_OK;
}

// Skipped (empty-side) pair q: line number, id, side ("src"/"tgt").
int bm_ingest_skipped(void* h, int32_t q, int64_t* lineno, const char** id, const char** side) {
  Ingest* g = (Ingest*)h;
  if (q < 0 || q >= (int32_t)g->skipped_lines.size()) return BM_EINVAL;
  *lineno = g->skipped_lines[q];
  *id = g->skipped_ids[q].c_str();
  *side = g->skipped_side[q].c_str();
  return BM_OK;
}

// Lexicon lowered to CSR over the batch's id space (pack.py pack_lexicon):
// forward = (src word -> candidates) from `n` (src, tgt) entries, reverse is
// its transpose (Lexicon.reversed); candidates outside the batch are dropped;
// per id the candidate ids are ascending and unique (pack.py _csr).
int bm_ingest_lexicon(void* h, const char* const* src_words, const char* const* tgt_words,
                      int64_t n_entries, bm_lexicon* out) {
  Ingest* g = (Ingest*)h;
  const int32_t nid = (int32_t)g->ids.size();
  std::vector<std::vector<int32_t>> fw(nid), rv(nid);
  for (int64_t q = 0; q < n_entries; ++q) {
    const int32_t ia = g->ids.find(src_words[q], strlen(src_words[q]));
    if (ia < 0) continue;
    const int32_t ib = g->ids.find(tgt_words[q], strlen(tgt_words[q]));
    if (ib < 0) continue;
    fw[ia].push_back(ib);
    rv[ib].push_back(ia);
  }
  auto csr = [&](std::vector<std::vector<int32_t>>& lists, std::vector<int32_t>& off,
                 std::vector<int32_t>& cand) {
    off.assign((size_t)nid + 1, 0);
    cand.clear();
    for (int32_t k = 0; k < nid; ++k) {
      auto& l = lists[k];
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
      cand.insert(cand.end(), l.begin(), l.end());
      off[k + 1] = (int32_t)cand.size();
    }
  };
  csr(fw, g->fwd_off, g->fwd_cand);
  csr(rv, g->rev_off, g->rev_cand);
  out->n_ids = nid;
  out->fwd_off = g->fwd_off.data();
  out->fwd_cand = g->fwd_cand.data();
  out->rev_off = g->rev_off.data();
  out->rev_cand = g->rev_cand.data();
  return BM_OK;
}

// After mining: per document the forward records (oriented as mined; swapped
// documents re-oriented), optionally merged with the backward records
// (miner.py:131-155), formatted as TSV lines (miner.py:253-260) in document
// order. fwd/bwd: compacted records of the batch (doc-ordered, path order);
// swap_f/swap_b: per-doc orientation flags; skip: per-doc 1 = not mined
// (ResourceLimitError), its records are absent. Counts go to report[0..5]:
// pairs, forward, backward, unique src tokens, unique tgt tokens, docs mined.
// merged: fwd holds records already oriented and merged (bm_merge_bidir: pad =
// 0 forward / 1 backward, (i, j) in the pair's own orientation).
static int emit_impl(void* h, const bm_record* fwd, int64_t n_fwd, const bm_record* bwd,
                     int64_t n_bwd, int32_t has_bwd, const uint8_t* swap_f, const uint8_t* swap_b,
                     const uint8_t* skip, bool merged, const char** out, int64_t* out_len,
                     int64_t* report) {
  Ingest* g = (Ingest*)h;
  const int32_t nd = (int32_t)g->docs.size();
  const size_t nid = g->ids.size();
  // documents are independent: ranges of documents (about equal record
  // counts) are formatted on separate threads and concatenated in order
  unsigned hw = std::thread::hardware_concurrency();
  if (const char* env = getenv("BM_INGEST_THREADS")) hw = (unsigned)atoi(env);
  const int64_t nrec = n_fwd + (has_bwd ? n_bwd : 0);
  const int nthr = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)std::max(hw, 1u), 32,
                                                                 nrec / 4096 + 1, (int64_t)nd}));
  auto doc_lb = [](const bm_record* r, int64_t n, int32_t d) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (r[mid].doc < d)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  std::vector<int32_t> cut(nthr + 1, nd);
  cut[0] = 0;
  for (int t = 1; t < nthr; ++t) {  // split the forward stream evenly
    const int64_t q = n_fwd * t / nthr;
    cut[t] = q < n_fwd ? fwd[q].doc : nd;
    cut[t] = std::max(cut[t], cut[t - 1]);
  }
  struct Part {
    std::string o;
    std::vector<uint8_t> src_seen, tgt_seen;
    int64_t pairs = 0, nf = 0, nb = 0, mined = 0;
  };
  std::vector<Part> parts(nthr);
  auto work = [&](int t) {
    Part& P = parts[t];
    std::string& o = P.o;
    P.src_seen.assign(nid, 0);
    P.tgt_seen.assign(nid, 0);
    // unique-token counts (miner.py count_unique_tokens): on accepted text
    // tokenize(normalize(raw)) is exactly the sentence's set U of normalized
    // token ids, so the sets are bitmaps over the id space
    auto mark = [&](std::vector<uint8_t>& seen, int32_t s) {
      for (int32_t q = g->tok_off[s]; q < g->tok_off[s + 1]; ++q) seen[(size_t)g->tok_id[q]] = 1;
    };
    struct Rec {
      int32_t si, tj;  // src / tgt sentence index in the pair's own orientation
      double conf;
      bool forward;
      uint64_t key;
    };
    const int32_t d_lo = cut[t], d_hi = cut[t + 1];
    int64_t pf = doc_lb(fwd, n_fwd, d_lo);
    int64_t pb = has_bwd ? doc_lb(bwd, n_bwd, d_lo) : 0;
    std::vector<Rec> recs, outr;
    std::vector<uint32_t> ord;
    // _sanitize (miner.py:253-258): tab / newline / carriage return -> space
    auto put_sanitized = [&](const char* s, size_t n) {
      const size_t o0 = o.size();
      o.append(s, n);
      for (size_t q = o0; q < o.size(); ++q)
        if (o[q] == '\t' || o[q] == '\n' || o[q] == '\r') o[q] = ' ';
    };
    auto put_raw = [&](int32_t s) {
      put_sanitized(g->sent_ptr[s], (size_t)g->sent_len[s]);
    };
    char num[64];
    for (int32_t d = d_lo; d < d_hi; ++d) {
      const bm_ingest::Doc& D = g->docs[d];
      // records of doc d (both streams are doc-ordered)
      const int64_t f0 = pf;
      while (pf < n_fwd && fwd[pf].doc == d) ++pf;
      const int64_t b0 = pb;
      if (has_bwd)
        while (pb < n_bwd && bwd[pb].doc == d) ++pb;
      if (skip[d]) continue;
      ++P.mined;
      recs.clear();
      auto take = [&](const bm_record& r, bool swapped) {
        Rec x;
        // oriented source is the pair's target when swapped (miner.py:117-128)
        x.si = swapped ? r.j : r.i;
        x.tj = swapped ? r.i : r.j;
        x.conf = r.conf;
        x.forward = !swapped;
        x.key = ((uint64_t)(uint32_t)g->norm_key[D.src0 + x.si] << 32) |
                (uint32_t)g->norm_key[D.tgt0 + x.tj];
        recs.push_back(x);
      };
      if (merged) {
        for (int64_t q = f0; q < pf; ++q) {
          Rec x;
          x.si = fwd[q].i;
          x.tj = fwd[q].j;
          x.conf = fwd[q].conf;
          x.forward = fwd[q].pad == 0;
          x.key = 0;
          recs.push_back(x);
        }
      } else {
        for (int64_t q = f0; q < pf; ++q) take(fwd[q], swap_f[d] != 0);
      }
      const std::vector<Rec>* emit = &recs;
      if (has_bwd) {
        for (int64_t q = b0; q < pb; ++q) take(bwd[q], swap_b[d] != 0);
        // bidirectional_merge (miner.py:131-155): per normalized-text key the
        // first record wins unless a later one is better (higher confidence,
        // or forward over backward on an exact tie); then sort by indices
        ord.resize(recs.size());
        for (uint32_t q = 0; q < ord.size(); ++q) ord[q] = q;
        std::stable_sort(ord.begin(), ord.end(),
                         [&](uint32_t a, uint32_t b) { return recs[a].key < recs[b].key; });
        outr.clear();
        for (size_t q = 0; q < ord.size();) {
          size_t w = q;
          size_t r = q + 1;
          for (; r < ord.size() && recs[ord[r]].key == recs[ord[q]].key; ++r) {
            const Rec& x = recs[ord[r]];
            const Rec& cur = recs[ord[w]];
            const bool better = x.conf != cur.conf ? x.conf > cur.conf : (x.forward && !cur.forward);
            if (better) w = r;
          }
          outr.push_back(recs[ord[w]]);
          q = r;
        }
        std::sort(outr.begin(), outr.end(), [](const Rec& a, const Rec& b) {
          return a.si != b.si ? a.si < b.si : a.tj < b.tj;
        });
        emit = &outr;
      }
      for (const Rec& x : *emit) {
        const int32_t ss = D.src0 + x.si, ts = D.tgt0 + x.tj;
        put_raw(ss);
        o += '\t';
        put_raw(ts);
        o += '\t';
        const int nc = snprintf(num, sizeof(num), "%.6f", x.conf);
        o.append(num, (size_t)nc);
        o += '\t';
        put_sanitized(D.id.data(), D.id.size());
        o += x.forward ? "\tforward\n" : "\tbackward\n";
        ++P.pairs;
        (x.forward ? P.nf : P.nb) += 1;
        mark(P.src_seen, ss);
        mark(P.tgt_seen, ts);
      }
    }
  };
  if (nthr == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nthr; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
  }
  std::string& o = g->out;
  size_t total = 0;
  for (const Part& P : parts) total += P.o.size();
  o.clear();
  o.reserve(total);
  int64_t pairs = 0, nf = 0, nb = 0, mined = 0, n_src_tok = 0, n_tgt_tok = 0;
  for (Part& P : parts) {
    o += P.o;
    pairs += P.pairs;
    nf += P.nf;
    nb += P.nb;
    mined += P.mined;
  }
  g->seen_src.clear();
  g->seen_tgt.clear();
  std::vector<const bm_ingest::StrTable::E*> by_id(nid, nullptr);
  for (const auto& e : g->ids.ents) by_id[(size_t)e.val] = &e;
  for (size_t id = 0; id < nid; ++id) {
    uint8_t s = 0, tg = 0;
    for (const Part& P : parts) {
      s |= P.src_seen[id];
      tg |= P.tgt_seen[id];
    }
    n_src_tok += s;
    n_tgt_tok += tg;
    // the token strings themselves (streamed files: unique counts across chunks)
    if (s) g->seen_src.append(g->ids.arena.data() + by_id[id]->off, by_id[id]->len).push_back('\0');
    if (tg) g->seen_tgt.append(g->ids.arena.data() + by_id[id]->off, by_id[id]->len).push_back('\0');
  }
  *out = o.data();
  *out_len = (int64_t)o.size();
  report[0] = pairs;
  report[1] = nf;
  report[2] = nb;
  report[3] = n_src_tok;
  report[4] = n_tgt_tok;
  report[5] = mined;
  return BM_OK;
}

int bm_ingest_emit(void* h, const bm_record* fwd, int64_t n_fwd, const bm_record* bwd,
                   int64_t n_bwd, int32_t has_bwd, const uint8_t* swap_f, const uint8_t* swap_b,
                   const uint8_t* skip, const char** out, int64_t* out_len, int64_t* report) {
  return emit_impl(h, fwd, n_fwd, bwd, n_bwd, has_bwd, swap_f, swap_b, skip, false, out, out_len,
                   report);
}

int bm_ingest_emit_merged(void* h, const bm_record* recs, int64_t n, const uint8_t* skip,
                          const char** out, int64_t* out_len, int64_t* report) {
  return emit_impl(h, recs, n, nullptr, 0, 0, nullptr, nullptr, skip, true, out, out_len, report);
}

int bm_ingest_seen(void* h, int32_t which, const char** buf, int64_t* len) {
  Ingest* g = (Ingest*)h;
  const std::string& s = which == 0 ? g->seen_src : g->seen_tgt;
  *buf = s.data();
  *len = (int64_t)s.size();
  return BM_OK;
}

int bm_ingest_norm_keys(void* h, const int32_t** keys) {
  *keys = ((Ingest*)h)->norm_key.data();
  return BM_OK;
}

}  // extern "C"
