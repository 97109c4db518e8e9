// text.cu — host-side text pipeline (§8(f) row f3): the fastBPE-style subword codec the
// paper swapped in for the Python tool ("replacing the Python subword tool with the C++
// implementation") and the shared vocabulary of the jointly BPE-encoded data
// ("jointly byte pair encoded with 32K merge operations using a shared vocabulary ...
// After decoding, we removed the BPE separators").  Reading R28:
// pretokenised input split on ASCII whitespace; a word starts as its UTF-8 characters;
// the adjacent pair of lowest merge rank is merged at every non-overlapping occurrence,
// left to right, until no pair is in the table; non-final subwords carry "@@".
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/nmt.h"
#include "engine.h"

struct nmt_text {
  std::unordered_map<std::string, int> rank;   // "a\x01b" -> merge rank
  std::unordered_map<std::string, int> tok2id;
  std::vector<std::string> id2tok;             // [vocab_size]; reserved ids have ""
};

namespace nmt {
namespace {

constexpr int kPad = 0, kUnk = 1, kBos = 2, kEos = 3;

inline bool ascii_ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f';
}

std::vector<std::string> split_ws(const char* p, size_t n) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < n) {
    while (i < n && ascii_ws(p[i])) ++i;
    size_t j = i;
    while (j < n && !ascii_ws(p[j])) ++j;
    if (j > i) out.emplace_back(p + i, j - i);
    i = j;
  }
  return out;
}

// UTF-8 characters of a word (a malformed lead byte is one character)
std::vector<std::string> utf8_chars(const std::string& w) {
  std::vector<std::string> out;
  size_t i = 0;
  while (i < w.size()) {
    const unsigned char c = (unsigned char)w[i];
    size_t len = c < 0x80 ? 1 : (c >> 5) == 6 ? 2 : (c >> 4) == 14 ? 3 : (c >> 3) == 30 ? 4 : 1;
    len = std::min(len, w.size() - i);
    out.push_back(w.substr(i, len));
    i += len;
  }
  return out;
}

inline std::string key(const std::string& a, const std::string& b) {
  std::string k;
  k.reserve(a.size() + b.size() + 1);
  k += a;
  k += '\x01';
  k += b;
  return k;
}

// BPE of one word -> subword tokens (separators attached)
void bpe_word(const nmt_text* t, const std::string& w, std::vector<std::string>& out) {
  std::vector<std::string> sym = utf8_chars(w);
  while (sym.size() > 1) {
    int best = -1;
    for (size_t i = 0; i + 1 < sym.size(); ++i) {
      auto it = t->rank.find(key(sym[i], sym[i + 1]));
      if (it != t->rank.end() && (best < 0 || it->second < best)) best = it->second;
    }
    if (best < 0) break;
    std::vector<std::string> nx;
    nx.reserve(sym.size());
    for (size_t i = 0; i < sym.size();) {
      if (i + 1 < sym.size()) {
        auto it = t->rank.find(key(sym[i], sym[i + 1]));
        if (it != t->rank.end() && it->second == best) {
          nx.push_back(sym[i] + sym[i + 1]);
          i += 2;
          continue;
        }
      }
      nx.push_back(sym[i]);
      ++i;
    }
    sym.swap(nx);
  }
  for (size_t i = 0; i < sym.size(); ++i) out.push_back(i + 1 < sym.size() ? sym[i] + "@@" : sym[i]);
}

// one line -> ids (+ EOS), with a per-thread word cache (fastBPE caches words too)
void encode_line(const nmt_text* t, const char* p, size_t n,
                 std::unordered_map<std::string, std::vector<int>>& cache, std::vector<int>& ids) {
  ids.clear();
  std::vector<std::string> toks;
  for (const std::string& w : split_ws(p, n)) {
    auto it = cache.find(w);
    if (it == cache.end()) {
      toks.clear();
      bpe_word(t, w, toks);
      std::vector<int> v;
      for (const auto& s : toks) {
        auto f = t->tok2id.find(s);
        v.push_back(f == t->tok2id.end() ? kUnk : f->second);
      }
      if (cache.size() < 1000000) it = cache.emplace(w, std::move(v)).first;
      else {
        ids.insert(ids.end(), v.begin(), v.end());
        continue;
      }
    }
    ids.insert(ids.end(), it->second.begin(), it->second.end());
  }
  ids.push_back(kEos);
}

std::vector<std::pair<const char*, size_t>> split_lines(const char* p, size_t n) {
  std::vector<std::pair<const char*, size_t>> out;
  size_t i = 0;
  while (i < n) {
    size_t j = i;
    while (j < n && p[j] != '\n') ++j;
    out.emplace_back(p + i, j - i);
    i = j + 1;
  }
  return out;
}

}  // namespace
}  // namespace nmt

using namespace nmt;

extern "C" {

nmt_status nmt_text_load(const char* vocab, int64_t vocab_len, const char* merges,
                         int64_t merges_len, nmt_text** out) {
  return guard([&] {
    NMT_REQUIRE(vocab && merges && out && vocab_len >= 0 && merges_len >= 0, NMT_E_ARG,
                "null argument");
    std::unique_ptr<nmt_text> t(new nmt_text());
    int ln = 0, r = 0;
    for (auto& L : split_lines(merges, (size_t)merges_len)) {
      ++ln;
      if (L.second >= 8 && std::strncmp(L.first, "#version", 8) == 0) continue;
      auto parts = split_ws(L.first, L.second);
      if (parts.empty()) continue;
      NMT_REQUIRE(parts.size() == 2, NMT_E_FORMAT,
                  "merges line " + std::to_string(ln) + ": expected two symbols");
      NMT_REQUIRE(t->rank.emplace(key(parts[0], parts[1]), r).second, NMT_E_FORMAT,
                  "merges line " + std::to_string(ln) + ": duplicate pair");
      ++r;
    }
    t->id2tok.assign(4, std::string());
    ln = 0;
    for (auto& L : split_lines(vocab, (size_t)vocab_len)) {
      ++ln;
      size_t a = 0, b = L.second;
      while (a < b && (L.first[a] == ' ' || L.first[a] == '\t' || L.first[a] == '\r')) ++a;
      while (b > a && (L.first[b - 1] == ' ' || L.first[b - 1] == '\t' || L.first[b - 1] == '\r')) --b;
      if (b == a) continue;
      std::string tok(L.first + a, b - a);
      const int id = (int)t->id2tok.size();
      NMT_REQUIRE(t->tok2id.emplace(tok, id).second, NMT_E_FORMAT,
                  "vocab line " + std::to_string(ln) + ": duplicate token");
      t->id2tok.push_back(tok);
    }
    *out = t.release();
  });
}

void nmt_text_free(nmt_text* t) { delete t; }

int32_t nmt_text_vocab_size(const nmt_text* t) { return t ? (int32_t)t->id2tok.size() : 0; }

nmt_status nmt_text_encode(const nmt_text* t, const char* text, int64_t len, int32_t n_threads,
                           int32_t* h_ids, int64_t cap, int64_t* h_off, int64_t max_lines,
                           int64_t* n_lines) {
  return guard([&] {
    NMT_REQUIRE(t && text && h_ids && h_off && n_lines && len >= 0, NMT_E_ARG, "null argument");
    auto lines = split_lines(text, (size_t)len);
    const int64_t n = (int64_t)lines.size();
    NMT_REQUIRE(n <= max_lines, NMT_E_SHAPE,
                std::to_string(n) + " lines > max_lines " + std::to_string(max_lines));
    std::vector<std::vector<int>> ids(n);
    const int T = std::max(1, std::min<int>(n_threads, 64));
    auto work = [&](int w) {
      std::unordered_map<std::string, std::vector<int>> cache;
      for (int64_t i = w; i < n; i += T) encode_line(t, lines[i].first, lines[i].second, cache, ids[i]);
    };
    if (T == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int w = 0; w < T; ++w) th.emplace_back(work, w);
      for (auto& x : th) x.join();
    }
    int64_t pos = 0;
    h_off[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
      NMT_REQUIRE(pos + (int64_t)ids[i].size() <= cap, NMT_E_SHAPE, "ids cap too small");
      std::copy(ids[i].begin(), ids[i].end(), h_ids + pos);
      pos += ids[i].size();
      h_off[i + 1] = pos;
    }
    *n_lines = n;
  });
}

nmt_status nmt_text_decode(const nmt_text* t, const int32_t* h_ids, const int64_t* h_off,
                           int64_t n, char* out, int64_t cap, int64_t* out_len) {
  return guard([&] {
    NMT_REQUIRE(t && h_ids && h_off && out && out_len && n >= 0, NMT_E_ARG, "null argument");
    const int V = (int)t->id2tok.size();
    std::string s;
    for (int64_t i = 0; i < n; ++i) {
      std::string line;
      for (int64_t k = h_off[i]; k < h_off[i + 1]; ++k) {
        const int id = h_ids[k];
        NMT_REQUIRE(id >= 0 && id < V, NMT_E_INPUT, "id " + std::to_string(id) + " out of range");
        if (id == kEos) break;
        if (id < 4) continue;   // PAD / UNK / BOS are never emitted
        if (!line.empty()) line += ' ';
        line += t->id2tok[id];
      }
      // remove the separators: every "@@ " (separator + space)
      std::string o;
      o.reserve(line.size());
      for (size_t q = 0; q < line.size();) {
        if (line.compare(q, 3, "@@ ") == 0) q += 3;
        else o += line[q++];
      }
      s += o;
      s += '\n';
    }
    NMT_REQUIRE((int64_t)s.size() <= cap, NMT_E_SHAPE, "text cap too small");
    std::memcpy(out, s.data(), s.size());
    *out_len = (int64_t)s.size();
  });
}

}  // extern "C"
