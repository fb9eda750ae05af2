// Host ingest in C++ (SURVEY.md §8f rank 1): the FNV-1a-64 word-hash tokenizer and the shared-
// prefix varlen packer, so host-side work keeps up with 8 B200s of scoring.
//
// Tokenizer — bit-identical to the reference tokenizer.encode (/root/reference/pkg/src/prefrank/
// tokenizer.py:119-134): text is lowercased (Python str.lower()), then scanned left to right
// with the template tags matched first (longest first, tokenizer.py:98-101) and otherwise
// maximal [a-z0-9]+ runs; a word's id is its special id ("yes"=1, "no"=2) or
// reserved + FNV-1a-64(word) mod (size - reserved) (tokenizer.py:72-76).  Input is UTF-8.  The
// only non-ASCII code points whose lowercase contains [a-z0-9] are U+0130 (-> "i" U+0307) and
// U+212A (-> "k"); every other non-ASCII code point is a separator (checked exhaustively over
// all code points in tests/test_host_ingest.py).
//
// Packer — bit-identical to prefixcache.split_shared_prefix + pack_requests.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/prefill_sm100.h"

namespace {

constexpr uint64_t kFnvOffset = 14695981039346656037ull;
constexpr uint64_t kFnvPrime = 1099511628211ull;

struct TagSpec {
  const char* text;
  int len;
  int id;
};
// tokenizer.py:27-37 (ids 3..11), sorted longest first as the reference scanner does
const TagSpec kTags[] = {
    {"<|/meta|>", 9, 8}, {"<|/desc|>", 9, 10}, {"<|/sys|>", 8, 4}, {"<|meta|>", 8, 7}, {"<|desc|>", 8, 9},
    {"<|sys|>", 7, 3},   {"<|ans|>", 7, 11},   {"<|/q|>", 6, 6},   {"<|q|>", 5, 5},
};

// UTF-8 -> the lowercase stream the regex sees, restricted to what can matter: ASCII is
// lowercased, U+0130 -> 'i' + separator, U+212A -> 'k', any other code point -> separator (0x01).
void lower_stream(const char* s, size_t n, std::string& out) {
  out.clear();
  out.reserve(n);
  const unsigned char* p = reinterpret_cast<const unsigned char*>(s);
  size_t i = 0;
  while (i < n) {
    const unsigned char c = p[i];
    if (c < 0x80) {
      out.push_back((c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : static_cast<char>(c));
      ++i;
      continue;
    }
    int len = (c >= 0xF0) ? 4 : (c >= 0xE0) ? 3 : (c >= 0xC0) ? 2 : 1;
    if (i + len > n) len = static_cast<int>(n - i);
    if (len == 2 && c == 0xC4 && p[i + 1] == 0xB0) {          // U+0130 LATIN CAPITAL I WITH DOT
      out.push_back('i');
      out.push_back('\x01');
    } else if (len == 3 && c == 0xE2 && p[i + 1] == 0x84 && p[i + 2] == 0xAA) {   // U+212A KELVIN
      out.push_back('k');
    } else {
      out.push_back('\x01');
    }
    i += len;
  }
}

inline bool is_word(char c) { return (c >= 'a' && c <= 'z') || (c >= '0' && c <= '9'); }

// ends (optional): end index of each token in the lowercased string, counted in Python str
// units (code points; U+0130 counts 2), i.e. the span end tokenizer.encode_with_spans reports.
int64_t tokenize_one(const char* text, size_t n, int32_t* out, int64_t cap, int size, int reserved,
                     std::string& buf, int64_t* ends = nullptr) {
  lower_stream(text, n, buf);
  const char* s = buf.data();
  const size_t m = buf.size();
  const uint64_t modulus = static_cast<uint64_t>(size - reserved);
  int64_t k = 0;
  size_t i = 0;
  while (i < m) {
    const char c = s[i];
    if (c == '<') {
      bool hit = false;
      for (const TagSpec& t : kTags) {
        if (i + t.len <= m && std::memcmp(s + i, t.text, t.len) == 0) {
          if (k < cap) {
            out[k] = t.id;
            if (ends) ends[k] = static_cast<int64_t>(i + t.len);
          }
          ++k;
          i += t.len;
          hit = true;
          break;
        }
      }
      if (hit) continue;
      ++i;
      continue;
    }
    if (!is_word(c)) {
      ++i;
      continue;
    }
    size_t j = i;
    uint64_t h = kFnvOffset;
    while (j < m && is_word(s[j])) {
      h = (h ^ static_cast<unsigned char>(s[j])) * kFnvPrime;
      ++j;
    }
    int32_t id;
    const size_t len = j - i;
    if (len == 3 && s[i] == 'y' && s[i + 1] == 'e' && s[i + 2] == 's') id = 1;
    else if (len == 2 && s[i] == 'n' && s[i + 1] == 'o') id = 2;
    else id = static_cast<int32_t>(reserved + h % modulus);
    if (k < cap) {
      out[k] = id;
      if (ends) ends[k] = static_cast<int64_t>(j);
    }
    ++k;
    i = j;
  }
  return k;
}

}  // namespace

extern "C" {

int pf_tokenize(const char* text, size_t len, int vocab_size, int reserved, int32_t* out_ids, int64_t cap,
                int64_t* n_out) {
  if (!text && len) return -1;
  if (vocab_size <= reserved || reserved < 12) return -1;
  std::string buf;
  const int64_t k = tokenize_one(text, len, out_ids, cap, vocab_size, reserved, buf);
  if (n_out) *n_out = k;
  return k > cap ? -5 : 0;
}

int pf_tokenize_spans(const char* text, size_t len, int vocab_size, int reserved, int32_t* out_ids,
                      int64_t* out_ends, int64_t cap, int64_t* n_out) {
  if (!text && len) return -1;
  if (vocab_size <= reserved || reserved < 12) return -1;
  std::string buf;
  const int64_t k = tokenize_one(text, len, out_ids, cap, vocab_size, reserved, buf, out_ends);
  if (n_out) *n_out = k;
  return k > cap ? -5 : 0;
}

int pf_tokenize_batch(const char* data, const int64_t* text_offsets, int n_texts, int vocab_size, int reserved,
                      int32_t* out_ids, int64_t cap, int64_t* out_offsets, int n_threads) {
  if (n_texts < 0 || !text_offsets || !out_offsets) return -1;
  if (vocab_size <= reserved || reserved < 12) return -1;
  // every token consumes >= 1 input byte, so text i's ids fit in its byte-length slot; pass 1
  // tokenizes each text into its own slot (in parallel), pass 2 compacts.
  const int64_t total = text_offsets[n_texts] - text_offsets[0];
  if (cap < total) return -5;
  std::vector<int64_t> counts(static_cast<size_t>(n_texts), 0);
  int nt = n_threads > 0 ? n_threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, n_texts));
  auto work = [&](int t) {
    std::string buf;
    for (int i = t; i < n_texts; i += nt) {
      const int64_t a = text_offsets[i], b = text_offsets[i + 1];
      counts[i] = tokenize_one(data + a, static_cast<size_t>(b - a), out_ids + (a - text_offsets[0]), b - a,
                               vocab_size, reserved, buf);
    }
  };
  if (nt == 1 || total < (1 << 16)) {
    nt = 1;
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  int64_t w = 0;
  out_offsets[0] = 0;
  for (int i = 0; i < n_texts; ++i) {
    const int64_t a = text_offsets[i] - text_offsets[0];
    if (w != a) std::memmove(out_ids + w, out_ids + a, static_cast<size_t>(counts[i]) * sizeof(int32_t));
    w += counts[i];
    out_offsets[i + 1] = w;
  }
  return 0;
}

// Pack requests.  Request r owns token lists [list_begin[r], list_begin[r+1]) of the flat list
// set (ids[list_offsets[k] .. list_offsets[k+1])).  Outputs (caller-allocated, sizes from the
// _sizes call): ids/pos [T], segs [n_seg][4], last_idx [n_items], prefix_lens [R].
int pf_pack_sizes(const int64_t* list_offsets, const int32_t* list_begin, int n_requests, int64_t* T,
                  int64_t* n_seg, int64_t* n_items) {
  int64_t t = 0, s = 0, it = 0;
  for (int r = 0; r < n_requests; ++r) {
    const int n = list_begin[r + 1] - list_begin[r];
    if (n < 1) return -1;
    t += list_offsets[list_begin[r + 1]] - list_offsets[list_begin[r]];
    s += n + 1;
    it += n;
  }
  *T = t;   // upper bound: the prefix is stored once, so the packed length is <= sum of lists
  *n_seg = s;
  *n_items = it;
  return 0;
}

int pf_pack_requests(const int32_t* ids, const int64_t* list_offsets, const int32_t* list_begin, int n_requests,
                     int max_seq, int32_t* out_ids, int32_t* out_pos, int32_t* out_segs, int32_t* out_last,
                     int32_t* out_prefix_lens, int64_t* out_T, int64_t* out_n_seg) {
  int64_t row = 0, seg = 0, item = 0;
  for (int r = 0; r < n_requests; ++r) {
    const int b = list_begin[r], e = list_begin[r + 1];
    if (e <= b) return -1;
    // longest common prefix, moved one left if any list would be left empty
    int64_t lcp = list_offsets[b + 1] - list_offsets[b];
    for (int k = b; k < e; ++k) {
      const int64_t len = list_offsets[k + 1] - list_offsets[k];
      if (len < 1) return -1;
      lcp = std::min(lcp, len);
    }
    const int32_t* first = ids + list_offsets[b];
    for (int k = b + 1; k < e && lcp > 0; ++k) {
      const int32_t* x = ids + list_offsets[k];
      int64_t n = 0;
      while (n < lcp && x[n] == first[n]) ++n;
      lcp = n;
    }
    bool any_equal = false;
    for (int k = b; k < e; ++k) any_equal |= (list_offsets[k + 1] - list_offsets[k]) == lcp;
    if (any_equal) --lcp;
    const int64_t P = lcp;
    out_prefix_lens[r] = static_cast<int32_t>(P);
    const int64_t pre_off = row;
    if (P > 0) {
      for (int64_t i = 0; i < P; ++i) {
        out_ids[row + i] = first[i];
        out_pos[row + i] = static_cast<int32_t>(i);
      }
      int32_t* sg = out_segs + 4 * seg++;
      sg[0] = static_cast<int32_t>(pre_off); sg[1] = 0; sg[2] = static_cast<int32_t>(pre_off);
      sg[3] = static_cast<int32_t>(P);
      row += P;
    }
    for (int k = b; k < e; ++k) {
      const int32_t* x = ids + list_offsets[k] + P;
      const int64_t S = list_offsets[k + 1] - list_offsets[k] - P;
      if (P + S > max_seq) return -2;
      for (int64_t i = 0; i < S; ++i) {
        out_ids[row + i] = x[i];
        out_pos[row + i] = static_cast<int32_t>(P + i);
      }
      int32_t* sg = out_segs + 4 * seg++;
      sg[0] = static_cast<int32_t>(pre_off); sg[1] = static_cast<int32_t>(P); sg[2] = static_cast<int32_t>(row);
      sg[3] = static_cast<int32_t>(S);
      row += S;
      out_last[item++] = static_cast<int32_t>(row - 1);
    }
  }
  *out_T = row;
  *out_n_seg = seg;
  return 0;
}

}  // extern "C"
