// automaton.cpp — P3DPDA v1 load/save, validation, and the device flattening.
//
// The flat format carries exactly the fields of gmask::Dpda the runtime
// consumes (dpda.hpp:97-124): state counts, the byte shift table
// (dpda.hpp:114-116), the single-terminal edges in arbitration order with
// their CSR ranges (dpda_builder.cpp:450-467).  Composites (optimizer.cpp:
// 78-136) are never consulted by Step/ComputeMask and are not stored.
#include <algorithm>
#include <cstring>

#include "gm_internal.hpp"

namespace pre3 {
namespace {

constexpr char kMagic[8] = {'P', '3', 'D', 'P', 'D', 'A', '0', '1'};

struct Reader {
  const uint8_t* p;
  const uint8_t* end;
  template <typename T>
  T Get() {
    if (static_cast<size_t>(end - p) < sizeof(T)) {
      throw Error(GM_ERR_CORRUPT_INPUT, "P3DPDA: truncated input");
    }
    T v;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    return v;
  }
};

template <typename T>
void Put(std::vector<uint8_t>* out, T v) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  out->insert(out->end(), b, b + sizeof(T));
}

void Corrupt(const std::string& why) { throw Error(GM_ERR_CORRUPT_INPUT, "P3DPDA: " + why); }

}  // namespace

Automaton LoadFlat(const uint8_t* data, size_t n) {
  if (n < 8 || std::memcmp(data, kMagic, 8) != 0) Corrupt("bad magic");
  Reader r{data + 8, data + n};
  Automaton a;
  a.num_states = r.Get<int32_t>();
  a.initial_state = r.Get<int32_t>();
  a.accept_state = r.Get<int32_t>();
  a.grammar_hash = r.Get<uint64_t>();
  int32_t tl = r.Get<int32_t>();
  if (a.num_states <= 0 || a.num_states > (1 << 24)) Corrupt("state count out of range");
  if (tl < 0 || tl > r.end - r.p) Corrupt("grammar text length");
  a.grammar_text.assign(reinterpret_cast<const char*>(r.p), static_cast<size_t>(tl));
  r.p += tl;
  size_t S = static_cast<size_t>(a.num_states);
  if (static_cast<size_t>(r.end - r.p) < S * 256 * 4) Corrupt("truncated shift table");
  a.shift_targets.resize(S * 256);
  std::memcpy(a.shift_targets.data(), r.p, S * 256 * 4);
  r.p += S * 256 * 4;
  int32_t ne = r.Get<int32_t>();
  if (ne < 0 || ne > (1 << 28)) Corrupt("edge count out of range");
  // Every edge record takes at least 56 bytes (header + one condition entry):
  // reject a count the remaining input cannot hold before allocating for it.
  if (static_cast<size_t>(ne) > static_cast<size_t>(r.end - r.p) / 56) Corrupt("edge count exceeds the input");
  a.edge_begin.resize(S + 1);
  for (auto& b : a.edge_begin) b = r.Get<int32_t>();
  a.edges.resize(static_cast<size_t>(ne));
  for (Edge& e : a.edges) {
    e.source = r.Get<int32_t>();
    for (auto& w : e.accepted) w = r.Get<uint64_t>();
    e.dollar = r.Get<uint8_t>() != 0;
    e.origin = r.Get<uint8_t>();
    e.dynamic = r.Get<uint8_t>() != 0;
    (void)r.Get<uint8_t>();
    e.target = r.Get<int32_t>();
    int32_t cl = r.Get<int32_t>();
    int32_t pl = r.Get<int32_t>();
    if (cl < 1 || cl > 4096 || pl < 0 || pl > 4096) Corrupt("edge condition/push length");
    e.match_pop.resize(static_cast<size_t>(cl));
    e.push.resize(static_cast<size_t>(pl));
    for (auto& s : e.match_pop) s = r.Get<int32_t>();
    for (auto& s : e.push) s = r.Get<int32_t>();
  }
  if (r.p != r.end) Corrupt("trailing bytes");
  a.Validate();
  return a;
}

std::vector<uint8_t> SaveFlat(const Automaton& a) {
  std::vector<uint8_t> out(kMagic, kMagic + 8);
  Put<int32_t>(&out, a.num_states);
  Put<int32_t>(&out, a.initial_state);
  Put<int32_t>(&out, a.accept_state);
  Put<uint64_t>(&out, a.grammar_hash);
  Put<int32_t>(&out, static_cast<int32_t>(a.grammar_text.size()));
  out.insert(out.end(), a.grammar_text.begin(), a.grammar_text.end());
  for (int32_t t : a.shift_targets) Put<int32_t>(&out, t);
  Put<int32_t>(&out, static_cast<int32_t>(a.edges.size()));
  for (int32_t b : a.edge_begin) Put<int32_t>(&out, b);
  for (const Edge& e : a.edges) {
    Put<int32_t>(&out, e.source);
    for (uint64_t w : e.accepted) Put<uint64_t>(&out, w);
    Put<uint8_t>(&out, e.dollar ? 1 : 0);
    Put<uint8_t>(&out, e.origin);
    Put<uint8_t>(&out, e.dynamic ? 1 : 0);
    Put<uint8_t>(&out, 0);
    Put<int32_t>(&out, e.target);
    Put<int32_t>(&out, static_cast<int32_t>(e.match_pop.size()));
    Put<int32_t>(&out, static_cast<int32_t>(e.push.size()));
    for (int32_t s : e.match_pop) Put<int32_t>(&out, s);
    for (int32_t s : e.push) Put<int32_t>(&out, s);
  }
  return out;
}

// Structural checks in the spirit of DeserializeDpda's re-validation
// (serialize.cpp:284-292) and ValidateDeterminism's well-formedness rules
// (dpda_builder.cpp:409-448): ids in range, CSR ranges consistent, each
// edge's condition starts at its source, dynamic edges resolvable.
void Automaton::Validate() const {
  const int32_t S = num_states;
  auto in_range = [S](int32_t s) { return s >= 0 && s < S; };
  if (!in_range(initial_state)) Corrupt("initial state out of range");
  if (accept_state != -1 && !in_range(accept_state)) Corrupt("accept state out of range");
  if (shift_targets.size() != static_cast<size_t>(S) * 256) Corrupt("shift table size");
  for (int32_t t : shift_targets) {
    if (t != -1 && !in_range(t)) Corrupt("shift target out of range");
  }
  if (static_cast<int32_t>(edge_begin.size()) != S + 1 || edge_begin[0] != 0 ||
      edge_begin[static_cast<size_t>(S)] != static_cast<int32_t>(edges.size())) {
    Corrupt("edge ranges");
  }
  for (int32_t s = 0; s < S; ++s) {
    if (edge_begin[static_cast<size_t>(s)] > edge_begin[static_cast<size_t>(s) + 1]) {
      Corrupt("edge ranges not monotone");
    }
    for (int32_t i = edge_begin[static_cast<size_t>(s)]; i < edge_begin[static_cast<size_t>(s) + 1]; ++i) {
      const Edge& e = edges[static_cast<size_t>(i)];
      if (e.source != s) Corrupt("edge source does not match its range");
      if (e.match_pop.empty() || e.match_pop[0] != s) Corrupt("condition must start at source");
      for (int32_t x : e.match_pop) {
        if (!in_range(x)) Corrupt("condition state out of range");
      }
      for (int32_t x : e.push) {
        if (!in_range(x)) Corrupt("push state out of range");
      }
      if (!e.dynamic && e.push.empty()) Corrupt("static edge pushes nothing");
      if (e.dynamic) {
        if (e.dollar) Corrupt("dynamic edge accepts the end marker");
        for (int b = 0; b < 256; ++b) {
          if (!e.Accepts(b)) continue;
          // The exposed top after the push prefix is either the last pushed
          // state or (empty prefix) the entry under the popped suffix, which
          // is unknown here; check the pushed case only.
          if (!e.push.empty() &&
              shift_targets[static_cast<size_t>(e.push.back()) * 256 + static_cast<size_t>(b)] < 0) {
            Corrupt("dynamic edge without a shift target");
          }
        }
      }
    }
  }
}

namespace {

// Open-addressing insert (linear probing); key 0 = empty.  `pairs`: entries
// are {key, value} pairs.
void HashInsert(std::vector<uint64_t>* tab, size_t slots, bool pairs, uint64_t key, uint64_t value) {
  const size_t stride = pairs ? 2 : 1;
  for (size_t i = key & (slots - 1);; i = (i + 1) & (slots - 1)) {
    uint64_t& k = (*tab)[i * stride];
    if (k == key) return;  // first inserted wins (arbitration order)
    if (k == 0) {
      k = key;
      if (pairs) (*tab)[i * stride + 1] = value;
      return;
    }
  }
}

size_t Pow2Slots(size_t n) {
  size_t s = 16;
  while (s < 2 * n) s <<= 1;
  return s;
}

void BuildConditionIndex(const Automaton& a, FlatLayout* f) {
  const int32_t S = a.num_states;
  f->hidx_meta.assign(static_cast<size_t>(S) * 257 * 2, 0);
  std::vector<std::pair<uint64_t, uint64_t>> exact;
  std::vector<uint64_t> prefix;
  for (int32_t s = 0; s < S; ++s) {
    for (int32_t t = 0; t < 257; ++t) {
      const size_t idx = static_cast<size_t>(s) * 257 + static_cast<size_t>(t);
      const int32_t cb = f->rec_begin[idx], ce = f->rec_begin[idx + 1];
      if (ce - cb <= kHashMin) continue;
      std::vector<int16_t> lens;
      for (int32_t c = cb; c < ce; ++c) {
        const CandRec& r = f->recs[static_cast<size_t>(c)];
        (void)r;
        const Edge& e = a.edges[static_cast<size_t>(f->rec_edge[static_cast<size_t>(c)])];
        const int L = static_cast<int>(e.match_pop.size());
        if (lens.empty() || lens.back() != L) lens.push_back(static_cast<int16_t>(L));  // descending (arbitration)
        uint64_t h = CondSeed(s, t);
        for (int j = 1; j <= L; ++j) {
          h = CondMix(h ^ static_cast<uint32_t>(e.match_pop[static_cast<size_t>(j - 1)]));
          if (j < L) prefix.push_back(CondKey(h, kSaltPrefix, j));  // a shorter known stack matches this prefix
        }
        exact.emplace_back(CondKey(h, kSaltExact, L), static_cast<uint64_t>(c));
      }
      f->hidx_meta[idx * 2] = static_cast<int32_t>(f->hidx_lens.size());
      f->hidx_meta[idx * 2 + 1] = static_cast<int32_t>(lens.size()) | (static_cast<int32_t>(lens.front()) << 16);
      f->hidx_lens.insert(f->hidx_lens.end(), lens.begin(), lens.end());
    }
  }
  std::sort(prefix.begin(), prefix.end());
  prefix.erase(std::unique(prefix.begin(), prefix.end()), prefix.end());
  const size_t es = Pow2Slots(exact.size()), ps = Pow2Slots(prefix.size());
  f->hidx_exact.assign(es * 2, 0);
  f->hidx_prefix.assign(ps, 0);
  for (const auto& kv : exact) HashInsert(&f->hidx_exact, es, true, kv.first, kv.second);
  for (uint64_t k : prefix) HashInsert(&f->hidx_prefix, ps, false, k, 0);
  if (f->hidx_lens.empty()) f->hidx_lens.push_back(0);
}

}  // namespace

FlatLayout Flatten(const Automaton& a) {
  FlatLayout f;
  const int32_t S = a.num_states;
  f.rec_begin.assign(static_cast<size_t>(S) * 257 + 1, 0);
  f.state_any.assign(static_cast<size_t>(S) * 9, 0u);
  // Conditions are shared by all records of an edge; static pushes too.
  // Every list starts on a 16-byte boundary so the device reads it with
  // independent int4 loads (one memory latency per list, not per entry).
  auto align4 = [](std::vector<int32_t>* v) {
    while (v->size() % 4) v->push_back(-1);
  };
  std::vector<int32_t> cond_at(a.edges.size()), push_at(a.edges.size());
  for (size_t i = 0; i < a.edges.size(); ++i) {
    const Edge& e = a.edges[i];
    align4(&f.rec_cond);
    align4(&f.rec_push);
    cond_at[i] = static_cast<int32_t>(f.rec_cond.size());
    for (size_t j = 1; j < e.match_pop.size(); ++j) f.rec_cond.push_back(e.match_pop[j]);
    push_at[i] = static_cast<int32_t>(f.rec_push.size());
    if (!e.dynamic) f.rec_push.insert(f.rec_push.end(), e.push.begin(), e.push.end());
  }
  for (int32_t s = 0; s < S; ++s) {
    for (int32_t t = 0; t < 257; ++t) {
      f.rec_begin[static_cast<size_t>(s) * 257 + static_cast<size_t>(t)] = static_cast<int32_t>(f.recs.size());
      for (int32_t i = a.edge_begin[static_cast<size_t>(s)]; i < a.edge_begin[static_cast<size_t>(s) + 1]; ++i) {
        const Edge& e = a.edges[static_cast<size_t>(i)];
        if (!e.Accepts(t)) continue;
        CandRec r{};
        r.cond_len = static_cast<int16_t>(e.match_pop.size());
        r.cond_off = cond_at[static_cast<size_t>(i)];
        for (int j = 0; j < 16; ++j) {
          r.cond[j] = static_cast<size_t>(j) + 1 < e.match_pop.size() ? e.match_pop[static_cast<size_t>(j) + 1] : -1;
        }
        if (e.dynamic) {
          align4(&f.rec_push);
          r.push_off = static_cast<int32_t>(f.rec_push.size());
          f.rec_push.insert(f.rec_push.end(), e.push.begin(), e.push.end());
          if (e.push.empty()) {
            r.new_state = -1;
          } else {
            const int32_t tgt = a.shift_targets[static_cast<size_t>(e.push.back()) * 256 + static_cast<size_t>(t)];
            f.rec_push.push_back(tgt);
            r.new_state = tgt;
          }
          r.push_len = static_cast<int16_t>(f.rec_push.size() - static_cast<size_t>(r.push_off));
        } else {
          r.push_off = push_at[static_cast<size_t>(i)];
          r.push_len = static_cast<int16_t>(e.push.size());
          r.new_state = e.push.back();
        }
        for (int j = 0; j < 4; ++j) r.push[j] = j < r.push_len ? f.rec_push[static_cast<size_t>(r.push_off + j)] : -1;
        f.max_cond = std::max<int32_t>(f.max_cond, r.cond_len);
        f.max_push = std::max<int32_t>(f.max_push, r.push_len + (r.new_state < 0 ? 1 : 0));
        f.recs.push_back(r);
        f.rec_edge.push_back(i);
        f.state_any[static_cast<size_t>(s) * 9 + static_cast<size_t>(t >> 5)] |= 1u << (t & 31);
      }
    }
  }
  f.rec_begin[static_cast<size_t>(S) * 257] = static_cast<int32_t>(f.recs.size());
  f.first.assign(static_cast<size_t>(S) * 257, CandRec{});
  for (size_t i = 0; i + 1 < f.rec_begin.size(); ++i) {
    if (f.rec_begin[i] < f.rec_begin[i + 1]) f.first[i] = f.recs[static_cast<size_t>(f.rec_begin[i])];
  }
  BuildConditionIndex(a, &f);
  if (f.recs.empty()) f.recs.push_back(CandRec{});
  // Tail padding: vector reads of the last list stay in bounds.
  f.rec_cond.insert(f.rec_cond.end(), 16, -1);
  f.rec_push.insert(f.rec_push.end(), 16, -1);
  align4(&f.rec_cond);
  align4(&f.rec_push);
  return f;
}

}  // namespace pre3
