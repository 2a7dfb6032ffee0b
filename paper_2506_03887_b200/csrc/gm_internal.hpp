// gm_internal.hpp — host-side structures behind include/pre3_gmask.h.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pre3_gmask.h"

namespace pre3 {

// Thrown inside the library and mapped to a gm_status_code at the C boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Host copy of a compiled automaton (gmask::Dpda, dpda.hpp:97-124), edges
// stored per state in arbitration order (dpda_builder.cpp:327-338).
struct Edge {
  int32_t source = -1;
  uint64_t accepted[4] = {0, 0, 0, 0};
  bool dollar = false;
  uint8_t origin = 0;  // 0 acceptance, 1 reduction, 2 cycle back, 3 merged
  bool dynamic = false;
  int32_t target = -1;
  std::vector<int32_t> match_pop;  // top first
  std::vector<int32_t> push;       // bottom first
  // Composites only (origin 3): the second consumed terminal set.
  uint64_t second[4] = {0, 0, 0, 0};
  bool dollar_second = false;

  bool Accepts(int32_t terminal) const {
    if (terminal == 256) return dollar;
    return (accepted[terminal >> 6] >> (terminal & 63)) & 1u;
  }
};

// A rewritten pumping circuit (gmask::Cycle, dpda.hpp:62-70), bottom first.
struct CycleRec {
  std::vector<int32_t> states;
  int closing_byte = 0;
};

// gmask::BuildStats (dpda.hpp:82-90).
struct BuildStats {
  int64_t states = 0, acceptance = 0, reduction = 0, cycle_back = 0, merged = 0, aggregated_groups = 0,
          edges_before_aggregation = 0;
};

struct Automaton {
  int32_t num_states = 0;
  int32_t initial_state = 0;
  int32_t accept_state = -1;
  uint64_t grammar_hash = 0;
  std::string grammar_text;
  std::vector<int32_t> shift_targets;  // S*256
  std::vector<Edge> edges;
  std::vector<int32_t> edge_begin;  // S+1
  // Build products the runtime never reads but the GMASKDP1 format carries
  // (serialize.cpp:148-196): composites in arbitration order, rewritten
  // circuits, BuildStats.  Absent (zero) for automata loaded from P3DPDA.
  std::vector<Edge> composite_edges;
  std::vector<CycleRec> cycle_list;
  BuildStats stats;
  int64_t composites = 0;  // composite_edges.size() (kept for P3DPDA-only automata: 0)
  int64_t cycles = 0;      // cycle_list.size()

  void Validate() const;  // throws Error(GM_ERR_CORRUPT_INPUT)
};

Automaton LoadFlat(const uint8_t* data, size_t n);
std::vector<uint8_t> SaveFlat(const Automaton& a);
Automaton CompileGrammar(const std::string& text, bool aggregate, bool merge);
// FinalizeEdgeOrder + ValidateDeterminism (dpda_builder.cpp:409-467) over an
// automaton read from disk: edges and composites re-sorted in arbitration
// order, ranges rebuilt; throws Error(GM_ERR_BUILD) when inconsistent.
void FinalizeAndCheck(Automaton* a);
uint64_t GrammarHash(const std::string& normalized_text);
// GMASKDP1 (serialize.cpp): magic line + one sorted-key JSON object.
std::vector<uint8_t> SaveGmaskdp1(const Automaton& a);
Automaton LoadGmaskdp1(const uint8_t* data, size_t n);  // throws Error(GM_ERR_CORRUPT_INPUT)
// LoadVocabulary / UnescapeToken / EscapeToken (serialize.cpp:298-364).
std::vector<std::string> LoadVocabularyJson(const uint8_t* data, size_t n);
std::string EscapeToken(const std::string& s);

// Device-oriented flattening.  For every (state, terminal)
// the candidate edges — those whose accepted set contains the terminal — in
// arbitration order, each as a self-contained record: the condition minus its
// first entry (always the current state, dpda.hpp:45 `front() == source`),
// the push sequence with a dynamic edge's shift target resolved for that
// terminal when the push prefix is non-empty (optimizer.cpp:33-76,
// runtime.cpp:159-164), and the resulting state; the first 16 condition
// entries and 4 pushed states are inlined in the record.
struct CandRec {
  int16_t cond_len;   // full |match_pop| (entry 0 = the source state, implicit)
  int16_t push_len;   // entries to push (resolved dynamic target included)
  int32_t cond_off;   // rec_cond index of entry 1 (entries 1..cond_len-1, top first)
  int32_t push_off;   // rec_push index (bottom first)
  int32_t new_state;  // top after apply; -1: dynamic with an empty push prefix
                      // (target read from the exposed top at apply time)
  int32_t push[4];    // first four pushed entries, bottom first (-1 padded)
  int32_t cond[16];   // condition entries 1..16, top first (-1 padded)
};
// 96 B = 6 x 16 B: one round trip of independent vector loads gives a
// candidate's whole condition (|match_pop| <= 17) and push list (<= 4).
static_assert(sizeof(CandRec) == 96, "CandRec layout");

struct FlatLayout {
  std::vector<int32_t> rec_begin;  // S*257 + 1
  std::vector<CandRec> recs;
  std::vector<int32_t> rec_edge;   // host only: the edge of each record
  std::vector<int32_t> rec_cond;
  std::vector<int32_t> rec_push;
  std::vector<uint32_t> state_any;  // S*9: bytes with any candidate (8 words) + bit0 of word 8 = '$'
  // Dense copy of each (state, terminal)'s first candidate (cond_len 0: none):
  // the candidate that wins ~2/3 of steps arrives in the same round trip as
  // the candidate range, so most byte steps cost one L2 round trip.
  std::vector<CandRec> first;
  // Condition index (FindEdge in O(distinct condition lengths)): for a
  // (state, terminal) with more than kHashMin candidates, the winner is the
  // candidate whose whole condition equals the stack top for the LONGEST
  // such length (arbitration: longer conditions first, dpda_builder.cpp:
  // 327-338; equal conditions keep the lower origin rank, listed first), so
  // a probe per distinct length replaces a serial scan (SQL: up to 864
  // candidates, 20 lengths).  hidx_meta[s*257+t] = {lens offset, count | max
  // length << 16}; lens descending in hidx_lens; hidx_exact maps
  // CondHash(s, t, L, condition) -> candidate; hidx_prefix holds
  // CondHash'(s, t, D, first D entries) of every longer condition (a walk
  // against a key that ends D entries down is undecidable when one matches).
  std::vector<int32_t> hidx_meta;   // S*257*2
  std::vector<int16_t> hidx_lens;
  std::vector<uint64_t> hidx_exact;  // pairs {key, candidate}, power-of-two slots
  std::vector<uint64_t> hidx_prefix; // keys, power-of-two slots
  int32_t max_cond = 0, max_push = 0;
};

constexpr int kHashMin = 6;  // candidates above which a (state, terminal) is indexed

#ifdef __CUDACC__
#define GM_HD __host__ __device__ __forceinline__
#else
#define GM_HD inline
#endif

// Hash of a condition prefix (shared by host and device; identical bits).
GM_HD uint64_t CondMix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// Running hash r_0 = CondSeed(s, t); r_j = CondMix(r_{j-1} ^ entry_{j-1}) over
// the stack top (entry 0 = the state); keys finish r_L with a salt and L.
GM_HD uint64_t CondSeed(int32_t s, int32_t t) {
  return CondMix(0x3c6ef372fe94f82bull ^ (static_cast<uint64_t>(static_cast<uint32_t>(s)) << 24) ^
                 static_cast<uint64_t>(static_cast<uint32_t>(t)));
}
constexpr uint64_t kSaltExact = 0x6a09e667f3bcc909ull, kSaltPrefix = 0xbb67ae8584caa73bull;
GM_HD uint64_t CondKey(uint64_t running, uint64_t salt, int32_t len) {
  return CondMix(running ^ salt ^ static_cast<uint64_t>(len)) | 1ull;
}

FlatLayout Flatten(const Automaton& a);

}  // namespace pre3
