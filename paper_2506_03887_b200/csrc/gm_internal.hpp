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

  bool Accepts(int32_t terminal) const {
    if (terminal == 256) return dollar;
    return (accepted[terminal >> 6] >> (terminal & 63)) & 1u;
  }
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

  void Validate() const;  // throws Error(GM_ERR_CORRUPT_INPUT)
};

Automaton LoadFlat(const uint8_t* data, size_t n);
std::vector<uint8_t> SaveFlat(const Automaton& a);
Automaton CompileGrammar(const std::string& text, bool aggregate, bool merge);

// Device-oriented flattening.
struct DevEdge {
  int32_t cond_off;
  int32_t push_off;
  int16_t cond_len;
  int16_t push_len;
  int32_t flags;  // bit0 dynamic
};
static_assert(sizeof(DevEdge) == 16, "DevEdge layout");

struct FlatLayout {
  std::vector<DevEdge> edges;
  std::vector<int32_t> cond_pool;  // top first
  std::vector<int32_t> push_pool;  // bottom first
  // Candidate edges per (state, terminal), terminal 0..256, in arbitration
  // order: the edges whose accepted set contains the terminal.
  std::vector<int32_t> cand_begin;  // S*257 + 1
  std::vector<int32_t> cand;
  int32_t max_cond = 0, max_push = 0;
};

FlatLayout Flatten(const Automaton& a);

}  // namespace pre3
