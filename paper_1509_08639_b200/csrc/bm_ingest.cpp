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
// Exactness contract: the native path accepts a file only when every byte is
// ASCII and the JSON stays inside a simple, fully validated subset; otherwise
// bm_ingest_jsonl returns BM_EUNSUPPORTED and the caller runs the Python path
// (which also produces the reference's error messages). Under that contract
// Python's Unicode-aware str methods reduce to fixed ASCII tables:
//   whitespace (str.isspace, re \s, split, strip) = 09-0D, 1C-1F, 20
//   alnum / regex word chars without '_'        = [0-9A-Za-z]
// and NFC is the identity.
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <unordered_map>
#include <vector>

#include "bimine_b200.h"

namespace bm_ingest {

inline bool is_space(unsigned char c) { return (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f) || c == 0x20; }
inline bool is_alpha(unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z'); }
inline bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }
inline bool is_alnum(unsigned char c) { return is_alpha(c) || is_digit(c); }
inline bool is_upper(unsigned char c) { return c >= 'A' && c <= 'Z'; }
inline char lower(char c) { return (c >= 'A' && c <= 'Z') ? (char)(c + 32) : c; }

struct Doc {
  std::string id, src_lang, tgt_lang;
  int32_t src0 = 0, n = 0, tgt0 = 0, m = 0;
};

struct Ingest {
  // packed sentences (pack.py layout)
  std::vector<int32_t> n_tok, n_punct, n_alpha, tok_off{0}, tok_id, dig_off{0}, dig_id;
  std::vector<uint16_t> tok_alpha;
  std::vector<int32_t> src0, n, tgt0, m;
  // interned token strings (normalized tokens and raw digit tokens)
  std::vector<std::string> strings;
  std::unordered_map<std::string, int32_t> ids;
  // per sentence: raw text, normalized text and its interned id (merge key)
  std::string raw, norm;
  std::vector<int64_t> raw_off{0}, norm_off{0};
  std::vector<int32_t> norm_key;
  std::unordered_map<std::string, int32_t> norm_ids;
  std::vector<Doc> docs;
  std::vector<int64_t> skipped_lines;  // empty-side pairs dropped at load
  std::vector<std::string> skipped_ids, skipped_side;
  // lexicon CSR over the id space (bm_ingest_lexicon)
  std::vector<int32_t> fwd_off, fwd_cand, rev_off, rev_cand;
  // token scratch
  struct TokInfo {
    int32_t nid, did;
    bool alpha, punct;
  };
  std::unordered_map<std::string, TokInfo> tok_cache;
  std::string out;  // TSV bytes of bm_ingest_emit
  std::string err;

  int32_t intern(const std::string& s) {
    auto it = ids.find(s);
    if (it != ids.end()) return it->second;
    const int32_t k = (int32_t)strings.size();
    ids.emplace(s, k);
    strings.push_back(s);
    return k;
  }
};

// ------------------------------------------------------------------ tokens
// tokenize (corpus.py:28): maximal [0-9A-Za-z] runs or one non-space char
template <class F>
void for_tokens(const char* s, size_t len, F&& f) {
  size_t i = 0;
  while (i < len) {
    const unsigned char c = (unsigned char)s[i];
    if (is_space(c)) {
      ++i;
    } else if (is_alnum(c)) {
      size_t j = i + 1;
      while (j < len && is_alnum((unsigned char)s[j])) ++j;
      f(s + i, j - i);
      i = j;
    } else {
      f(s + i, 1);
      ++i;
    }
  }
}

// normalize (corpus.py:38-40): NFC (identity on ASCII), lower, " ".join(split())
std::string normalize(const char* s, size_t len) {
  std::string o;
  o.reserve(len);
  size_t i = 0;
  while (i < len) {
    while (i < len && is_space((unsigned char)s[i])) ++i;
    if (i >= len) break;
    if (!o.empty()) o.push_back(' ');
    while (i < len && !is_space((unsigned char)s[i])) o.push_back(lower(s[i++]));
  }
  return o;
}

// Packer.add_sentence (pack.py) for one raw sentence
bool add_sentence(Ingest& g, const char* s, size_t len) {
  int32_t T = 0, P = 0, A = 0;
  std::vector<std::pair<int32_t, int32_t>> alpha;  // (normalized id, isalpha count)
  std::vector<int32_t> digits;
  std::string key;
  for_tokens(s, len, [&](const char* t, size_t tl) {
    key.assign(t, tl);
    auto it = g.tok_cache.find(key);
    if (it == g.tok_cache.end()) {
      Ingest::TokInfo ti;
      ti.nid = g.intern(normalize(t, tl));
      bool all_alpha = tl > 0, all_digit = tl > 0, any_alnum = false;
      for (size_t q = 0; q < tl; ++q) {
        const unsigned char c = (unsigned char)t[q];
        all_alpha &= is_alpha(c);
        all_digit &= is_digit(c);
        any_alnum |= is_alnum(c);
      }
      ti.did = all_digit ? g.intern(key) : -1;
      ti.alpha = all_alpha;
      ti.punct = !any_alnum;
      it = g.tok_cache.emplace(key, ti).first;
    }
    const Ingest::TokInfo& ti = it->second;
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
    if (pr.second > 65535) {
      g.err = "a sentence repeats one token more than 65535 times";
      return false;
    }
    g.tok_id.push_back(pr.first);
    g.tok_alpha.push_back((uint16_t)pr.second);
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
  std::string nm = normalize(s, len);
  auto nit = g.norm_ids.find(nm);
  int32_t nk;
  if (nit == g.norm_ids.end()) {
    nk = (int32_t)g.norm_ids.size();
    g.norm_ids.emplace(nm, nk);
  } else {
    nk = nit->second;
  }
  g.norm_key.push_back(nk);
  g.norm.append(nm);
  g.norm_off.push_back((int64_t)g.norm.size());
  return true;
}

const char* const kAbbrev[] = {"dr", "mr", "mrs", "ms", "prof", "st", "no", "vs", "etc"};

bool is_abbrev(const char* s, size_t len) {
  for (const char* a : kAbbrev) {
    if (strlen(a) != len) continue;
    bool eq = true;
    for (size_t q = 0; q < len; ++q) eq &= lower(s[q]) == a[q];
    if (eq) return true;
  }
  return false;
}

// segment_sentences (corpus.py:92-126): sentence spans [begin, end) of text
void segment(const std::string& text, std::vector<std::pair<size_t, size_t>>& spans) {
  const size_t size = text.size();
  const char* s = text.data();
  size_t pos = 0;
  while (pos < size && is_space((unsigned char)s[pos])) ++pos;
  size_t begin = pos;
  while (pos < size) {
    const char ch = s[pos];
    if (ch != '.' && ch != '!' && ch != '?') {
      ++pos;
      continue;
    }
    if (ch == '.') {
      size_t st = pos;
      while (st > 0 && is_alpha((unsigned char)s[st - 1])) --st;
      if (is_abbrev(s + st, pos - st)) {
        ++pos;
        continue;
      }
    }
    size_t nxt = pos + 1;
    if (nxt < size && is_space((unsigned char)s[nxt])) {
      while (nxt < size && is_space((unsigned char)s[nxt])) ++nxt;
      if (nxt < size && (is_upper((unsigned char)s[nxt]) || is_digit((unsigned char)s[nxt]))) {
        spans.emplace_back(begin, pos + 1);
        begin = pos = nxt;
        continue;
      }
    }
    ++pos;
  }
  size_t end = size;
  while (end > begin && is_space((unsigned char)s[end - 1])) --end;
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
  // JSON string -> ASCII bytes (\u escapes above 0x7f, raw control chars: fail)
  bool str(std::string& out) {
    out.clear();
    if (p >= e || *p != '"') return false;
    ++p;
    while (p < e) {
      const unsigned char c = (unsigned char)*p++;
      if (c == '"') return true;
      if (c < 0x20) return false;
      if (c != '\\') {
        out.push_back((char)c);
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
          if (e - p < 4) return false;
          unsigned v = 0;
          for (int q = 0; q < 4; ++q) {
            const char h = *p++;
            v <<= 4;
            if (h >= '0' && h <= '9') v |= (unsigned)(h - '0');
            else if (h >= 'a' && h <= 'f') v |= (unsigned)(h - 'a' + 10);
            else if (h >= 'A' && h <= 'F') v |= (unsigned)(h - 'A' + 10);
            else return false;
          }
          if (v >= 0x80) return false;  // non-ASCII text: Python path
          out.push_back((char)v);
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
    for (char ch : s) blank &= is_space((unsigned char)ch);
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
  bool has_id = false, has_sl = false, has_tl = false;
  Field src, tgt;
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
  Doc d;
  d.id = id;
  d.src_lang = sl;
  d.tgt_lang = tl;
  std::vector<std::pair<const char*, size_t>> ss, ts;
  field_spans(src, ss);
  field_spans(tgt, ts);
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

}  // namespace bm_ingest

using bm_ingest::Ingest;

extern "C" {

int bm_ingest_jsonl(const char* path, void** handle, char* why, int32_t why_len) {
  auto fail_why = [&](const char* w) {
    if (why && why_len > 0) snprintf(why, (size_t)why_len, "%s", w);
    return BM_EUNSUPPORTED;
  };
  *handle = nullptr;
  FILE* fh = fopen(path, "rb");
  if (!fh) return fail_why("cannot open file");
  std::string data;
  char buf[1 << 16];
  size_t r;
  while ((r = fread(buf, 1, sizeof(buf), fh)) > 0) data.append(buf, r);
  fclose(fh);
  for (unsigned char c : data)
    if (c >= 0x80) return fail_why("non-ASCII input");
  Ingest* g = new Ingest();
  const char* s = data.data();
  const char* end = s + data.size();
  int64_t lineno = 0;
  while (s < end) {
    // text-mode line splitting: \n, \r\n and \r end a line
    const char* q = s;
    while (q < end && *q != '\n' && *q != '\r') ++q;
    ++lineno;
    bool blank = true;
    for (const char* t = s; t < q; ++t) blank &= bm_ingest::is_space((unsigned char)*t);
    if (!blank) {
      const int rc = bm_ingest::parse_line(*g, s, q, lineno);
      if (rc < 0) {
        char msg[160];
        snprintf(msg, sizeof(msg), "line %lld: %s", (long long)lineno,
                 g->err.empty() ? "outside the native JSON subset" : g->err.c_str());
        delete g;
        return fail_why(msg);
      }
    }
    if (q < end && *q == '\r' && q + 1 < end && q[1] == '\n') ++q;
    s = q + 1;
  }
  *handle = g;
  return BM_OK;
}

void bm_ingest_free(void* h) { delete (Ingest*)h; }

int bm_ingest_view(void* h, bm_ingest_arrays* v) {
  Ingest* g = (Ingest*)h;
  v->n_sent = (int32_t)g->n_tok.size();
  v->n_docs = (int32_t)g->docs.size();
  v->n_ids = (int32_t)g->strings.size();
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
  const int32_t nid = (int32_t)g->strings.size();
  std::vector<std::vector<int32_t>> fw(nid), rv(nid);
  std::string a, b;
  for (int64_t q = 0; q < n_entries; ++q) {
    a = src_words[q];
    b = tgt_words[q];
    auto ia = g->ids.find(a);
    auto ib = g->ids.find(b);
    if (ia == g->ids.end() || ib == g->ids.end()) continue;
    fw[ia->second].push_back(ib->second);
    rv[ib->second].push_back(ia->second);
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
int bm_ingest_emit(void* h, const bm_record* fwd, int64_t n_fwd, const bm_record* bwd,
                   int64_t n_bwd, int32_t has_bwd, const uint8_t* swap_f, const uint8_t* swap_b,
                   const uint8_t* skip, const char** out, int64_t* out_len, int64_t* report) {
  Ingest* g = (Ingest*)h;
  const int32_t nd = (int32_t)g->docs.size();
  std::string& o = g->out;
  o.clear();
  int64_t pairs = 0, nf = 0, nb = 0, mined = 0;
  std::unordered_map<std::string, char> src_tok, tgt_tok;
  struct Rec {
    int32_t si, tj;  // src / tgt sentence index in the pair's own orientation
    double conf;
    bool forward;
  };
  int64_t pf = 0, pb = 0;
  std::vector<Rec> recs;
  std::unordered_map<uint64_t, size_t> best;
  auto sent_raw = [&](int32_t s) {
    return std::string(g->raw.data() + g->raw_off[s], (size_t)(g->raw_off[s + 1] - g->raw_off[s]));
  };
  auto sanitize = [](std::string t) {
    for (char& c : t)
      if (c == '\t' || c == '\n' || c == '\r') c = ' ';
    return t;
  };
  char num[64];
  for (int32_t d = 0; d < nd; ++d) {
    const bm_ingest::Doc& D = g->docs[d];
    // records of doc d (both streams are doc-ordered)
    const int64_t f0 = pf;
    while (pf < n_fwd && fwd[pf].doc == d) ++pf;
    const int64_t b0 = pb;
    if (has_bwd)
      while (pb < n_bwd && bwd[pb].doc == d) ++pb;
    if (skip[d]) continue;
    ++mined;
    recs.clear();
    auto take = [&](const bm_record& r, bool swapped, bool forward) {
      Rec x;
      // oriented source is the pair's target when swapped (miner.py:117-128)
      x.si = swapped ? r.j : r.i;
      x.tj = swapped ? r.i : r.j;
      x.conf = r.conf;
      x.forward = forward;
      recs.push_back(x);
    };
    for (int64_t q = f0; q < pf; ++q) take(fwd[q], swap_f[d] != 0, !swap_f[d]);
    std::vector<Rec> outr;
    if (!has_bwd) {
      outr = recs;
    } else {
      for (int64_t q = b0; q < pb; ++q) take(bwd[q], swap_b[d] != 0, !swap_b[d]);
      best.clear();
      std::vector<Rec> uniq;
      for (const Rec& x : recs) {
        const uint64_t key = ((uint64_t)(uint32_t)g->norm_key[D.src0 + x.si] << 32) |
                             (uint32_t)g->norm_key[D.tgt0 + x.tj];
        auto it = best.find(key);
        if (it == best.end()) {
          best.emplace(key, uniq.size());
          uniq.push_back(x);
        } else {
          Rec& cur = uniq[it->second];
          const bool better = x.conf != cur.conf ? x.conf > cur.conf : (x.forward && !cur.forward);
          if (better) cur = x;
        }
      }
      std::stable_sort(uniq.begin(), uniq.end(), [](const Rec& a, const Rec& b) {
        return a.si != b.si ? a.si < b.si : a.tj < b.tj;
      });
      outr.swap(uniq);
    }
    const std::string did = sanitize(D.id);
    for (const Rec& x : outr) {
      const int32_t ss = D.src0 + x.si, ts = D.tgt0 + x.tj;
      o += sanitize(sent_raw(ss));
      o += '\t';
      o += sanitize(sent_raw(ts));
      o += '\t';
      snprintf(num, sizeof(num), "%.6f", x.conf);
      o += num;
      o += '\t';
      o += did;
      o += x.forward ? "\tforward\n" : "\tbackward\n";
      ++pairs;
      (x.forward ? nf : nb) += 1;
      const char* ns = g->norm.data() + g->norm_off[ss];
      bm_ingest::for_tokens(ns, (size_t)(g->norm_off[ss + 1] - g->norm_off[ss]),
                            [&](const char* t, size_t tl) { src_tok.emplace(std::string(t, tl), 1); });
      const char* nt = g->norm.data() + g->norm_off[ts];
      bm_ingest::for_tokens(nt, (size_t)(g->norm_off[ts + 1] - g->norm_off[ts]),
                            [&](const char* t, size_t tl) { tgt_tok.emplace(std::string(t, tl), 1); });
    }
  }
  *out = o.data();
  *out_len = (int64_t)o.size();
  report[0] = pairs;
  report[1] = nf;
  report[2] = nb;
  report[3] = (int64_t)src_tok.size();
  report[4] = (int64_t)tgt_tok.size();
  report[5] = mined;
  return BM_OK;
}

}  // extern "C"
