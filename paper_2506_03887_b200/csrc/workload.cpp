// workload.cpp — synthetic inputs for tests and bench.py (include/pre3_workload.h).
//
// gmw_synth_vocab restates the reference acceptance gate's bench vocabulary
// generator, WriteBenchVocab (tests/acceptance/acceptance_main.cpp:341-359):
// 27 fixed fragments plus tokens of length {1,2,2,3,3,4,5,6,8} over a 49-byte
// alphabet drawn from mt19937_64(424242) into a std::set until it holds
// `num_tokens` distinct strings; ids are the set's (sorted) order.  With
// num_tokens = 32000 the output is byte-identical to the reference's; larger
// counts (128,255 for the Llama-3-sized configs) continue the same stream.
#include <cstdint>
#include <cstring>
#include <random>
#include <set>
#include <string>

#include "pre3_workload.h"

extern "C" int64_t gmw_synth_vocab(int32_t num_tokens, int32_t flavor, uint8_t* bytes, int64_t bytes_cap,
                                   int64_t* offsets) {
  if (num_tokens < 27) return -1;
  std::string alphabet = "abcdefghijklmnopqrstuvwxyz0123456789{}[],:\" .-+eE_";
  std::set<std::string> toks;
  for (const char* frag : {"true", "false", "null", "{\"", " \"", "\":", "\",", "\"}", "},", "],", "[{", "}}",
                           "]}", "0.", "e+", ", ", "\": \"", "0", "1", "2", "3", "4", "5", "6", "7", "8", "9"}) {
    toks.insert(frag);
  }
  if (flavor == 1) {
    // SQL-flavoured extension for the config-4 grammar.
    alphabet += "ABCDEFGHIJKLMNOPQRSTUVWXYZ()*=<>";
    for (const char* frag : {"SELECT ", "FROM ", "WHERE ", "AND ", "OR ", "ORDER ", "BY ", "ASC", "DESC",
                             "COUNT", "SUM", "MAX", "MIN", "(", ")", "* ", "= ", "< ", "> ", ", "}) {
      toks.insert(frag);
    }
  }
  std::mt19937_64 rng(424242);
  const size_t lens[] = {1, 2, 2, 3, 3, 4, 5, 6, 8};
  while (toks.size() < static_cast<size_t>(num_tokens)) {
    size_t len = lens[rng() % (sizeof(lens) / sizeof(lens[0]))];
    std::string t;
    for (size_t i = 0; i < len; ++i) t.push_back(alphabet[rng() % alphabet.size()]);
    toks.insert(t);
  }
  int64_t total = 0;
  for (const auto& t : toks) total += static_cast<int64_t>(t.size());
  if (bytes == nullptr || offsets == nullptr) return total;
  if (bytes_cap < total) return -2;
  int64_t o = 0, i = 0;
  for (const auto& t : toks) {
    offsets[i++] = o;
    std::memcpy(bytes + o, t.data(), t.size());
    o += static_cast<int64_t>(t.size());
  }
  offsets[i] = o;
  return total;
}

extern "C" int32_t gmw_structural_words(const uint8_t* bytes, const int64_t* offsets, int32_t num_tokens,
                                        uint32_t* words) {
  const int32_t nw = (num_tokens + 1 + 31) / 32;
  std::memset(words, 0, sizeof(uint32_t) * static_cast<size_t>(nw));
  int32_t n = 0;
  for (int32_t t = 0; t < num_tokens; ++t) {
    for (int64_t i = offsets[t]; i < offsets[t + 1]; ++i) {
      if (std::strchr("{}[],:\"", bytes[i]) != nullptr && bytes[i] != 0) {
        words[t >> 5] |= 1u << (t & 31);
        ++n;
        break;
      }
    }
  }
  return n;
}
