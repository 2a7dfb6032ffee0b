// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the
// product path).
//
// A thin extern "C" shim over the UNMODIFIED reference matcher ("gmask",
// /root/reference/proj).  The reference sources are compiled where they lie by
// oracle/Makefile into oracle/_ref/libgmask_ref.so; nothing is copied.  The
// shim exposes exactly what the parity tests, the golden-vector generator and
// bench.py's reference arm need:
//
//   * BuildDpda (dpda_builder.cpp:478-522) and an exporter of the resulting
//     `gmask::Dpda` into this repo's flat automaton format (P3DPDA v1, see
//     DESIGN.md §3), plus an importer so the reference Engine can run any flat
//     automaton on the GPU box without /root/reference;
//   * Engine::InitialConfig / Step / AllowedTerminals / ComputeMask /
//     ComputeMaskNaive (runtime.cpp:115-307) and TokenTrie::Build
//     (runtime.cpp:18-61) on opaque handles;
//   * the CPU reference decode loop timed by bench.py (`--impl reference`):
//     per sequence-step ComputeMask + bf16 -inf masking + the synthetic-stream
//     sampler + Step per token byte, batch sharded over std::thread workers.
//     Masking and sampling are NOT in the reference; they
//     are restated here from DESIGN.md §5 so the CPU and GPU arms replay the
//     identical token streams.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "gmask/dpda.hpp"
#include "gmask/grammar.hpp"
#include "gmask/lr1.hpp"
#include "gmask/runtime.hpp"
#ifdef GMASK_WITH_SERIALIZE
#include "gmask/serialize.hpp"
#endif
#include "support/oracle.hpp"

using namespace gmask;

namespace {

// ---------------------------------------------------------------- flat format
// Little-endian; see DESIGN.md §3 (mirrors paper_2506_03887_b200/csrc/automaton.cpp).
constexpr char kMagic[8] = {'P', '3', 'D', 'P', 'D', 'A', '0', '1'};

struct Writer {
  std::vector<uint8_t> out;
  template <typename T>
  void put(T v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    out.insert(out.end(), p, p + sizeof(T));
  }
  void bytes(const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    out.insert(out.end(), b, b + n);
  }
};

struct Reader {
  const uint8_t* p;
  const uint8_t* end;
  template <typename T>
  T get() {
    if (p + sizeof(T) > end) throw std::runtime_error("truncated flat automaton");
    T v;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    return v;
  }
};

std::vector<uint8_t> ExportFlat(const Dpda& d) {
  Writer w;
  w.bytes(kMagic, 8);
  w.put<int32_t>(d.num_states);
  w.put<int32_t>(d.initial_state);
  w.put<int32_t>(d.accept_state);
  w.put<uint64_t>(d.grammar_hash);
  w.put<int32_t>(static_cast<int32_t>(d.grammar_text.size()));
  w.bytes(d.grammar_text.data(), d.grammar_text.size());
  for (StateId t : d.shift_targets) w.put<int32_t>(t);
  w.put<int32_t>(static_cast<int32_t>(d.edges.size()));
  for (int32_t b : d.edge_begin) w.put<int32_t>(b);
  for (const PrefixConditionedEdge& e : d.edges) {
    w.put<int32_t>(e.source);
    for (uint64_t word : e.accepted.bytes.words) w.put<uint64_t>(word);
    w.put<uint8_t>(e.accepted.end_marker ? 1 : 0);
    w.put<uint8_t>(static_cast<uint8_t>(e.origin));
    w.put<uint8_t>(e.push_shift_target ? 1 : 0);
    w.put<uint8_t>(0);
    w.put<int32_t>(e.target);
    w.put<int32_t>(static_cast<int32_t>(e.match_pop.size()));
    w.put<int32_t>(static_cast<int32_t>(e.push.size()));
    for (StateId s : e.match_pop) w.put<int32_t>(s);
    for (StateId s : e.push) w.put<int32_t>(s);
  }
  return w.out;
}

Dpda ImportFlat(const uint8_t* buf, size_t n) {
  Reader r{buf, buf + n};
  if (n < 8 || std::memcmp(buf, kMagic, 8) != 0) throw std::runtime_error("bad magic");
  r.p += 8;
  Dpda d;
  d.num_states = r.get<int32_t>();
  d.initial_state = r.get<int32_t>();
  d.accept_state = r.get<int32_t>();
  d.grammar_hash = r.get<uint64_t>();
  int32_t tl = r.get<int32_t>();
  if (tl < 0 || r.p + tl > r.end) throw std::runtime_error("bad grammar text");
  d.grammar_text.assign(reinterpret_cast<const char*>(r.p), static_cast<size_t>(tl));
  r.p += tl;
  d.shift_targets.resize(static_cast<size_t>(d.num_states) * 256);
  for (auto& t : d.shift_targets) t = r.get<int32_t>();
  int32_t ne = r.get<int32_t>();
  d.edge_begin.resize(static_cast<size_t>(d.num_states) + 1);
  for (auto& b : d.edge_begin) b = r.get<int32_t>();
  d.edges.resize(static_cast<size_t>(ne));
  for (auto& e : d.edges) {
    e.source = r.get<int32_t>();
    for (auto& word : e.accepted.bytes.words) word = r.get<uint64_t>();
    e.accepted.end_marker = r.get<uint8_t>() != 0;
    e.origin = static_cast<PrefixConditionedEdge::Origin>(r.get<uint8_t>());
    e.push_shift_target = r.get<uint8_t>() != 0;
    (void)r.get<uint8_t>();
    e.target = r.get<int32_t>();
    int32_t cl = r.get<int32_t>();
    int32_t pl = r.get<int32_t>();
    e.match_pop.resize(static_cast<size_t>(cl));
    e.push.resize(static_cast<size_t>(pl));
    for (auto& s : e.match_pop) s = r.get<int32_t>();
    for (auto& s : e.push) s = r.get<int32_t>();
  }
  d.composite_begin.assign(static_cast<size_t>(d.num_states) + 1, 0);
  return d;
}

std::vector<std::string> Tokens(const uint8_t* bytes, const int64_t* offs, int32_t n) {
  std::vector<std::string> v(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    v[static_cast<size_t>(i)].assign(reinterpret_cast<const char*>(bytes + offs[i]),
                                     static_cast<size_t>(offs[i + 1] - offs[i]));
  }
  return v;
}

void MaskToWords(const TokenMask& m, uint32_t* words) {
  int32_t nbits = m.num_tokens() + 1;
  int32_t nw = (nbits + 31) / 32;
  std::memset(words, 0, sizeof(uint32_t) * static_cast<size_t>(nw));
  for (int32_t t = 0; t < nbits; ++t) {
    if (m.Test(t)) words[t >> 5] |= 1u << (t & 31);
  }
}

void SetErr(char* err, int errlen, const char* msg) {
  if (!err || errlen <= 0) return;
  std::snprintf(err, static_cast<size_t>(errlen), "%s", msg);
}

// ------------------------------------------------ synthetic stream
inline uint64_t Mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

inline uint64_t StreamDraw(uint64_t seed, uint64_t seq, uint64_t draw) {
  return Mix64(Mix64(seed ^ (seq * 0xD1B54A32D192ED03ull)) ^ draw);
}

// Returns the r-th (0-based) set bit among words[0..nw) & filter (filter may
// be null); bits >= limit are ignored.
int32_t SelectBit(const uint32_t* words, const uint32_t* filter, int32_t limit, uint32_t r) {
  int32_t nw = (limit + 31) / 32;
  for (int32_t w = 0; w < nw; ++w) {
    uint32_t x = words[w] & (filter ? filter[w] : ~0u);
    if (w == nw - 1 && (limit & 31)) x &= (1u << (limit & 31)) - 1;
    uint32_t c = static_cast<uint32_t>(__builtin_popcount(x));
    if (r < c) {
      for (;;) {
        int bit = __builtin_ctz(x);
        if (r == 0) return w * 32 + bit;
        --r;
        x &= x - 1;
      }
    }
    r -= c;
  }
  return -1;
}

int32_t CountBits(const uint32_t* words, const uint32_t* filter, int32_t limit) {
  int32_t nw = (limit + 31) / 32;
  int32_t n = 0;
  for (int32_t w = 0; w < nw; ++w) {
    uint32_t x = words[w] & (filter ? filter[w] : ~0u);
    if (w == nw - 1 && (limit & 31)) x &= (1u << (limit & 31)) - 1;
    n += __builtin_popcount(x);
  }
  return n;
}

// DESIGN.md §5 "stream" sampler: V regular tokens, EOS = bit V.
int32_t StreamPick(const uint32_t* mask, const uint32_t* structural, int32_t V, uint64_t u) {
  int32_t n_all = CountBits(mask, nullptr, V);
  bool eos = (mask[V >> 5] >> (V & 31)) & 1u;
  if (n_all == 0) return eos ? V : -1;
  if (eos && ((u >> 32) & 3u) == 0) return V;  // EOS with probability 1/4
  uint32_t lo = static_cast<uint32_t>(u);
  if ((u >> 34) & 1u) {
    int32_t n_s = structural ? CountBits(mask, structural, V) : 0;
    if (n_s > 0) {
      uint32_t r = static_cast<uint32_t>((static_cast<uint64_t>(lo) * static_cast<uint32_t>(n_s)) >> 32);
      return SelectBit(mask, structural, V, r);
    }
  }
  uint32_t r = static_cast<uint32_t>((static_cast<uint64_t>(lo) * static_cast<uint32_t>(n_all)) >> 32);
  return SelectBit(mask, nullptr, V, r);
}

// Synthetic bf16 logits of config 5 (gmask_port.c gp_synth_logit; the
// device bench fills its rotating buffers with the same function).
uint16_t SynthLogit(uint64_t seed, int32_t k, int32_t b, int32_t t) {
  uint64_t h = Mix64(seed ^ 0x6C6F67697473ull ^ (static_cast<uint64_t>(static_cast<uint32_t>(k)) * 0xA24BAED4963EE407ull) ^
                     (static_cast<uint64_t>(static_cast<uint32_t>(b)) * 0xD1B54A32D192ED03ull));
  uint64_t x = Mix64(h ^ static_cast<uint64_t>(static_cast<uint32_t>(t)));
  return static_cast<uint16_t>((0x3C00u + static_cast<uint32_t>(x & 0x3FFu)) ^ (((x >> 20) & 1u) ? 0x8000u : 0u));
}

// Argmax of the allowed bf16 logits (ties -> lowest id; -1 when nothing is
// allowed) — the device greedy rule (kernels.cu GreedyKey).
int32_t GreedyPick(const uint16_t* row, const uint32_t* mask, int32_t v1) {
  int32_t best = -1;
  uint32_t best_key = 0;
  for (int32_t t = 0; t < v1; ++t) {
    if (!((mask[t >> 5] >> (t & 31)) & 1u)) continue;
    const uint32_t bits = static_cast<uint32_t>(row[t]) << 16;
    const uint32_t key = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
    if (best < 0 || key > best_key) {
      best = t;
      best_key = key;
    }
  }
  return best;
}

// bf16 -inf masking of one logits row (new work).
void MaskRowBf16(uint16_t* row, const uint32_t* mask, int32_t v1) {
  for (int32_t t = 0; t < v1; ++t) {
    if (!((mask[t >> 5] >> (t & 31)) & 1u)) row[t] = 0xFF80u;
  }
}

struct Engines {
  Engine engine;
  explicit Engines(Dpda d) : engine(std::move(d)) {}
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------- automaton
// Returns 0 ok, 2 grammar error, 3 build error, 1 other.
int ref_compile(const char* text, int aggregate, int merge, void** out, char* err, int errlen) {
  try {
    BuildOptions o;
    o.aggregate = aggregate != 0;
    o.merge = merge != 0;
    Grammar g = ParseGrammar(text);
    *out = new Dpda(BuildDpda(g, o));
    return 0;
  } catch (const GrammarError& e) {
    SetErr(err, errlen, e.what());
    return 2;
  } catch (const BuildError& e) {
    SetErr(err, errlen, e.what());
    return 3;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 1;
  }
}

void ref_dpda_free(void* d) { delete static_cast<Dpda*>(d); }

#ifdef GMASK_WITH_SERIALIZE
// SerializeDpda (serialize.cpp:148-196) -> GMASKDP1 bytes (size returned;
// copied when cap suffices).
int64_t ref_dpda_serialize(void* d, uint8_t* buf, int64_t cap) {
  const std::string s = gmask::SerializeDpda(*static_cast<Dpda*>(d));
  if (buf && cap >= static_cast<int64_t>(s.size())) std::memcpy(buf, s.data(), s.size());
  return static_cast<int64_t>(s.size());
}

// DeserializeDpda (serialize.cpp:198-294): 0 ok, 4 SerializeError (message).
int ref_dpda_deserialize(const uint8_t* data, int64_t n, void** out, char* err, int errlen) {
  try {
    *out = new Dpda(gmask::DeserializeDpda(std::string(reinterpret_cast<const char*>(data), static_cast<size_t>(n))));
    return 0;
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return 4;
  }
}

// LoadVocabulary (serialize.cpp:348-364): tokens joined by offsets; returns
// the token count (-1 on error, message in err).
int32_t ref_load_vocabulary(const uint8_t* data, int64_t n, uint8_t* bytes, int64_t cap, int64_t* offs,
                            int32_t max_tokens, char* err, int errlen) {
  try {
    std::vector<std::string> v =
        gmask::LoadVocabulary(std::string(reinterpret_cast<const char*>(data), static_cast<size_t>(n)));
    int64_t o = 0;
    for (size_t i = 0; i < v.size() && static_cast<int32_t>(i) < max_tokens; ++i) {
      if (offs) offs[i] = o;
      if (bytes && o + static_cast<int64_t>(v[i].size()) <= cap) std::memcpy(bytes + o, v[i].data(), v[i].size());
      o += static_cast<int64_t>(v[i].size());
    }
    if (offs && static_cast<int32_t>(v.size()) <= max_tokens) offs[v.size()] = o;
    return static_cast<int32_t>(v.size());
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return -1;
  }
}
#endif

int64_t ref_dpda_flat(void* d, uint8_t* buf, int64_t cap) {
  std::vector<uint8_t> v = ExportFlat(*static_cast<Dpda*>(d));
  if (buf && cap >= static_cast<int64_t>(v.size())) std::memcpy(buf, v.data(), v.size());
  return static_cast<int64_t>(v.size());
}

void ref_dpda_stats(void* dp, int64_t* out /*8*/) {
  const Dpda& d = *static_cast<Dpda*>(dp);
  out[0] = d.num_states;
  out[1] = static_cast<int64_t>(d.edges.size());
  out[2] = static_cast<int64_t>(d.composites.size());
  out[3] = static_cast<int64_t>(d.cycles.size());
  int64_t dyn = 0, maxpop = 0, maxpush = 0;
  for (const auto& e : d.edges) {
    dyn += e.push_shift_target;
    maxpop = std::max<int64_t>(maxpop, static_cast<int64_t>(e.match_pop.size()));
    maxpush = std::max<int64_t>(maxpush, static_cast<int64_t>(e.push.size()));
  }
  out[4] = dyn;
  out[5] = maxpop;
  out[6] = maxpush;
  out[7] = d.stats.edges_before_aggregation;
}

// ---------------------------------------------------------------- engine
void* ref_engine_from_dpda(void* d) { return new Engines(*static_cast<Dpda*>(d)); }

void* ref_engine_from_flat(const uint8_t* buf, int64_t n, char* err, int errlen) {
  try {
    return new Engines(ImportFlat(buf, static_cast<size_t>(n)));
  } catch (const std::exception& e) {
    SetErr(err, errlen, e.what());
    return nullptr;
  }
}

void ref_engine_free(void* e) { delete static_cast<Engines*>(e); }

// err_kind: 0 ok, 1 empty token, 2 duplicate token.
void* ref_trie_new(const uint8_t* bytes, const int64_t* offs, int32_t n, int* err_kind, char* err,
                   int errlen) {
  *err_kind = 0;
  try {
    return new TokenTrie(TokenTrie::Build(Tokens(bytes, offs, n)));
  } catch (const VocabError& e) {
    *err_kind = e.kind() == VocabError::Kind::kEmptyToken ? 1 : 2;
    SetErr(err, errlen, e.what());
    return nullptr;
  }
}

void ref_trie_free(void* t) { delete static_cast<TokenTrie*>(t); }
int32_t ref_trie_nodes(void* t) {
  return static_cast<int32_t>(static_cast<TokenTrie*>(t)->nodes().size());
}

void* ref_cfg_new(void* e) {
  return new RuntimeConfig(static_cast<Engines*>(e)->engine.InitialConfig());
}
void* ref_cfg_clone(void* c) { return new RuntimeConfig(*static_cast<RuntimeConfig*>(c)); }
void ref_cfg_free(void* c) { delete static_cast<RuntimeConfig*>(c); }

// Returns the stack depth; copies min(depth, cap) entries bottom-first.
int32_t ref_cfg_get(void* c, int32_t* state, int32_t* status, int32_t* stack, int32_t cap) {
  const RuntimeConfig& cfg = *static_cast<RuntimeConfig*>(c);
  *state = cfg.state;
  *status = static_cast<int32_t>(cfg.status);
  int32_t n = static_cast<int32_t>(cfg.stack.size());
  for (int32_t i = 0; i < std::min(n, cap); ++i) stack[i] = cfg.stack[static_cast<size_t>(i)];
  return n;
}

void ref_cfg_set(void* c, int32_t status, const int32_t* stack, int32_t depth) {
  RuntimeConfig& cfg = *static_cast<RuntimeConfig*>(c);
  cfg.stack.assign(stack, stack + depth);
  cfg.state = depth > 0 ? stack[depth - 1] : 0;
  cfg.status = static_cast<Status>(status);
}

int ref_step(void* e, void* c, int32_t terminal) {
  return static_cast<Engines*>(e)->engine.Step(static_cast<RuntimeConfig*>(c), terminal) ? 1 : 0;
}

void ref_allowed(void* e, void* c, uint64_t* bytes4, int32_t* dollar) {
  TerminalSet t = static_cast<Engines*>(e)->engine.AllowedTerminals(*static_cast<RuntimeConfig*>(c));
  for (int i = 0; i < 4; ++i) bytes4[i] = t.bytes.words[static_cast<size_t>(i)];
  *dollar = t.end_marker ? 1 : 0;
}

void ref_mask(void* e, void* c, void* trie, uint32_t* words) {
  TokenMask m = static_cast<Engines*>(e)->engine.ComputeMask(*static_cast<RuntimeConfig*>(c),
                                                            *static_cast<TokenTrie*>(trie));
  MaskToWords(m, words);
}

void ref_mask_naive(void* e, void* c, const uint8_t* bytes, const int64_t* offs, int32_t n,
                    uint32_t* words) {
  TokenMask m = static_cast<Engines*>(e)->engine.ComputeMaskNaive(*static_cast<RuntimeConfig*>(c),
                                                                 Tokens(bytes, offs, n));
  MaskToWords(m, words);
}

// --------------------------------------------------- CPU reference decode loop
// One "sequence-step" = ComputeMask + bf16 -inf row masking + stream sampling +
// Step per token byte (EOS: Step(kEndMarker)); finished sequences restart from
// InitialConfig.  Sequences [0, batch) are sharded over `threads`
// std::thread workers; the same engine/trie are shared read-only
// (SPEC.md:416-418).  Stacks deeper than stack_cap count as overflow and
// restart, matching the device's fixed-capacity stacks.
//
// out_stats[0] = seconds of the timed steps, [1] = seq-steps timed, [2] =
// restarts, [3] = FNV-1a digest of the chosen tokens in (sequence, step)
// order, [4] = sum of mask popcounts of the timed steps, [5] = the digest of
// sequences [0, digest_seqs) over the timed steps only, [6] = their mask
// popcounts (EOS bit excluded) — the bench's in-run evidence (both arms print
// [5] and [6]).  logits_row 2 (greedy) reads SynthLogit rows of buffer
// (step % rows).  If `tokens_out` is non-null it receives the
// [batch][steps] chosen tokens; if `final_stacks` is non-null it receives
// per sequence [depth, status, stack...] rows of stride stack_cap + 2.
int ref_decode_run(void* e, void* trie, const uint32_t* structural, int32_t batch, int32_t warmup,
                   int32_t timed, uint64_t seed, int32_t threads, int32_t stack_cap, int32_t logits_row,
                   double* out_stats, int32_t* tokens_out, int32_t* final_stacks, int32_t rows,
                   uint64_t logit_seed, int32_t digest_seqs) {
  const int32_t steps = warmup + timed;
  const Engine& eng = static_cast<Engines*>(e)->engine;
  const TokenTrie& tr = *static_cast<TokenTrie*>(trie);
  // Token bytes for Step: rebuild from the trie (first-child/next-sibling).
  int32_t V = tr.num_tokens();
  std::vector<std::string> toks(static_cast<size_t>(V));
  {
    std::vector<std::pair<int32_t, std::string>> stack{{0, std::string()}};
    const auto& nodes = tr.nodes();
    while (!stack.empty()) {
      auto [n, s] = stack.back();
      stack.pop_back();
      if (nodes[static_cast<size_t>(n)].token >= 0) toks[static_cast<size_t>(nodes[static_cast<size_t>(n)].token)] = s;
      for (int32_t c = nodes[static_cast<size_t>(n)].first_child; c != -1; c = nodes[static_cast<size_t>(c)].next_sibling) {
        stack.push_back({c, s + static_cast<char>(nodes[static_cast<size_t>(c)].byte)});
      }
    }
  }
  int32_t v1 = V + 1;
  int32_t nw = (v1 + 31) / 32;
  if (threads < 1) threads = 1;
  threads = std::min(threads, std::max(batch, 1));
  std::vector<std::vector<int32_t>> chosen(static_cast<size_t>(batch),
                                           std::vector<int32_t>(static_cast<size_t>(steps), -1));
  std::vector<RuntimeConfig> cfgs(static_cast<size_t>(batch), eng.InitialConfig());
  std::vector<int64_t> restarts(static_cast<size_t>(threads), 0), pops(static_cast<size_t>(threads), 0);
  std::vector<uint64_t> draws(static_cast<size_t>(batch), 0);
  std::vector<int64_t> wpops(static_cast<size_t>(threads), 0);
  // Greedy mode (logits_row == 2, config 5): every sequence's SynthLogit row
  // of each rotating buffer, generated ahead (outside the timed steps).
  if (rows < 1) rows = 1;
  std::vector<uint16_t> grows;
  if (logits_row == 2) {
    grows.resize(static_cast<size_t>(batch) * static_cast<size_t>(rows) * static_cast<size_t>(v1));
    for (int32_t b = 0; b < batch; ++b) {
      for (int32_t k = 0; k < rows; ++k) {
        uint16_t* g = &grows[(static_cast<size_t>(b) * static_cast<size_t>(rows) + static_cast<size_t>(k)) * static_cast<size_t>(v1)];
        for (int32_t t = 0; t < v1; ++t) g[t] = SynthLogit(logit_seed, k, b, t);
      }
    }
  }

  auto worker = [&](int32_t tid, int32_t s_begin, int32_t s_end) {
    std::vector<uint32_t> mask(static_cast<size_t>(nw));
    std::vector<uint16_t> row(logits_row ? static_cast<size_t>(v1) : 0, 0x3F80u);
    for (int32_t s = s_begin; s < s_end; ++s) {
      for (int32_t b = tid; b < batch; b += threads) {
        RuntimeConfig& cfg = cfgs[static_cast<size_t>(b)];
        TokenMask m = eng.ComputeMask(cfg, tr);
        MaskToWords(m, mask.data());
        const int64_t pc = static_cast<int64_t>(m.CountSet());
        pops[static_cast<size_t>(tid)] += pc;
        if (b < digest_seqs) wpops[static_cast<size_t>(tid)] += pc - (m.Test(V) ? 1 : 0);
        int32_t tok;
        if (logits_row == 2) {
          tok = GreedyPick(&grows[(static_cast<size_t>(b) * static_cast<size_t>(rows) + static_cast<size_t>(s % rows)) *
                                  static_cast<size_t>(v1)],
                           mask.data(), v1);
        } else {
          if (logits_row) MaskRowBf16(row.data(), mask.data(), v1);
          uint64_t u = StreamDraw(seed, static_cast<uint64_t>(b), draws[static_cast<size_t>(b)]++);
          tok = StreamPick(mask.data(), structural, V, u);
        }
        chosen[static_cast<size_t>(b)][static_cast<size_t>(s)] = tok;
        bool overflow = false;
        if (tok == V) {
          eng.Step(&cfg, kEndMarker);
        } else if (tok >= 0) {
          for (char ch : toks[static_cast<size_t>(tok)]) {
            if (!eng.Step(&cfg, static_cast<uint8_t>(ch))) break;
            if (static_cast<int32_t>(cfg.stack.size()) > stack_cap) {
              overflow = true;
              break;
            }
          }
        }
        if (tok < 0 || overflow || cfg.status != Status::kAlive) {
          cfg = eng.InitialConfig();
          ++restarts[static_cast<size_t>(tid)];
        }
      }
    }
  };
  auto run = [&](int32_t s_begin, int32_t s_end) {
    std::vector<std::thread> pool;
    for (int32_t t = 1; t < threads; ++t) pool.emplace_back(worker, t, s_begin, s_end);
    worker(0, s_begin, s_end);
    for (auto& th : pool) th.join();
  };
  run(0, warmup);
  std::fill(pops.begin(), pops.end(), 0);
  std::fill(wpops.begin(), wpops.end(), 0);
  auto t0 = std::chrono::steady_clock::now();
  run(warmup, steps);
  auto t1 = std::chrono::steady_clock::now();

  uint64_t digest = 1469598103934665603ull;
  for (int32_t b = 0; b < batch; ++b) {
    for (int32_t s = 0; s < steps; ++s) {
      uint32_t v = static_cast<uint32_t>(chosen[static_cast<size_t>(b)][static_cast<size_t>(s)]);
      for (int k = 0; k < 4; ++k) digest = (digest ^ ((v >> (8 * k)) & 0xffu)) * 1099511628211ull;
      if (tokens_out) tokens_out[static_cast<int64_t>(b) * steps + s] = static_cast<int32_t>(v);
    }
  }
  uint64_t wdigest = 1469598103934665603ull;
  for (int32_t b = 0; b < batch && b < digest_seqs; ++b) {
    for (int32_t s = warmup; s < steps; ++s) {
      uint32_t v = static_cast<uint32_t>(chosen[static_cast<size_t>(b)][static_cast<size_t>(s)]);
      for (int k = 0; k < 4; ++k) wdigest = (wdigest ^ ((v >> (8 * k)) & 0xffu)) * 1099511628211ull;
    }
  }
  int64_t r = 0, p = 0, wp = 0;
  for (int32_t t = 0; t < threads; ++t) {
    r += restarts[static_cast<size_t>(t)];
    p += pops[static_cast<size_t>(t)];
    wp += wpops[static_cast<size_t>(t)];
  }
  out_stats[0] = std::chrono::duration<double>(t1 - t0).count();
  out_stats[1] = static_cast<double>(static_cast<int64_t>(batch) * timed);
  out_stats[2] = static_cast<double>(r);
  out_stats[3] = static_cast<double>(digest >> 11);  // 53-bit exact in a double
  out_stats[4] = static_cast<double>(p);
  out_stats[5] = static_cast<double>(wdigest >> 11);
  out_stats[6] = static_cast<double>(wp);
  if (final_stacks) {
    for (int32_t b = 0; b < batch; ++b) {
      int32_t* row = final_stacks + static_cast<int64_t>(b) * (stack_cap + 2);
      const RuntimeConfig& cfg = cfgs[static_cast<size_t>(b)];
      int32_t d = static_cast<int32_t>(cfg.stack.size());
      row[0] = d;
      row[1] = static_cast<int32_t>(cfg.status);
      for (int32_t i = 0; i < std::min(d, stack_cap); ++i) row[2 + i] = cfg.stack[static_cast<size_t>(i)];
    }
  }
  return 0;
}

// SampleSentence (tests/support/oracle.cpp:140-183) over a grammar text with a
// seeded mt19937_64 state carried by the caller (`rng_state` = the seed on
// first use is NOT supported: the caller passes a fresh seed per call).
int32_t ref_sample_sentence(const char* grammar_text, uint64_t seed, int32_t soft_limit, char* out,
                            int32_t cap) {
  try {
    Grammar g = ParseGrammar(grammar_text);
    std::mt19937_64 rng(seed);
    std::string s = gmask::testing::SampleSentence(g, &rng, static_cast<size_t>(soft_limit));
    int32_t n = static_cast<int32_t>(s.size());
    if (out && cap >= n) std::memcpy(out, s.data(), s.size());
    return n;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
