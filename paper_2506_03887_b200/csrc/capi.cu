// capi.cu — the C ABI of include/pre3_gmask.h: engine/batch lifetime, device
// uploads, and launch wrappers.  Host-side only; kernels live in kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <cstdlib>
#include <thread>
#include <unordered_set>
#include <string_view>
#include <vector>

#include "gm_internal.hpp"
#include "kernels.cuh"
#include "pre3_gmask.h"

struct gm_automaton {
  pre3::Automaton a;
};

#ifndef PRE3_HEAVY_PER_SM
#define PRE3_HEAVY_PER_SM 2  // heavy-pass (and first builder) CTAs of a fill grid per SM
#endif

namespace {

thread_local std::string g_last_error;

int Fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

void Check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw pre3::Error(GM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename T>
T* DevAlloc(size_t n, std::vector<void*>* owned) {
  void* p = nullptr;
  Check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  owned->push_back(p);
  return static_cast<T*>(p);
}

template <typename T>
T* DevUpload(const std::vector<T>& v, std::vector<void*>* owned) {
  T* p = DevAlloc<T>(v.size(), owned);
  if (!v.empty()) Check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
  return p;
}

template <typename F>
int Guard(F&& f) {
  try {
    return f();
  } catch (const pre3::Error& e) {
    return Fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return Fail(GM_ERR_USAGE, "host allocation failed");
  } catch (const std::exception& e) {
    return Fail(GM_ERR_USAGE, e.what());
  }
}

// Word-wise 64-bit hash (multiply-xorshift) for snapshot keys and checksums.
uint64_t Hash64(const void* data, size_t n, uint64_t h = 0x243F6A8885A308D3ull) {
  const uint8_t* p = static_cast<const uint8_t*>(data);
  auto mix = [](uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
  };
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = (h ^ mix(w)) * 0x9E3779B97F4A7C15ull;
  }
  uint64_t t = 0;
  std::memcpy(&t, p + i, n - i);
  return mix(h ^ mix(t ^ (static_cast<uint64_t>(n) << 3)));
}

template <typename T>
uint64_t HashVec(const std::vector<T>& v, uint64_t h) {
  return Hash64(v.data(), v.size() * sizeof(T), h);
}

}  // namespace

struct gm_engine {
  int device = 0;
  int32_t V = 0, W = 0, nseg = 0;
  pre3::AutView aut{};
  pre3::VocabView vocab{};
  pre3::CacheView cache{};
  uint32_t* structural = nullptr;
  std::vector<uint32_t> disabled;  // host copy (W words) or empty
  // Snapshot key (gm_engine_snapshot_*): the automaton's grammar hash, a hash
  // of the flattened device layout and one of the vocabulary + logit layout.
  uint64_t grammar_hash = 0, layout_hash = 0, vocab_hash = 0;
  // Eviction: the engine's batches (their seq_slot rows are kept), the keep
  // bytes, the host-mapped free-row count and the auto-eviction threshold.
  std::vector<gm_batch*> batches;
  uint8_t* evict_keep = nullptr;
  int32_t* host_free = nullptr;  // cudaHostAlloc(mapped)
  int32_t auto_evict_free = 0;
  std::vector<void*> owned;
  ~gm_engine() {
    cudaSetDevice(device);
    for (void* p : owned) cudaFree(p);
    if (host_free) cudaFreeHost(host_free);
  }
};

// Host bookkeeping of the two build queues.  Lookups (fused into accepts or
// the fill's tail, or LookupKernel) feed queue[prod]; the next fill drains
// queue[prod].  At most two lookup passes reach a queue before it is drained
// (capacity 2*B*nseg items).
struct gm_batch {
  gm_engine* engine = nullptr;
  // One-shot measurement hook (gm_batch_time_next_fill): events recorded
  // around the next fill kernel launch on its stream, whatever call makes it.
  cudaEvent_t time_fill[2] = {nullptr, nullptr};
  void FillStart(cudaStream_t s) {
    if (time_fill[0]) Check(cudaEventRecord(time_fill[0], s), "event record");
  }
  void FillEnd(cudaStream_t s) {
    if (time_fill[1]) Check(cudaEventRecord(time_fill[1], s), "event record");
    time_fill[0] = time_fill[1] = nullptr;
  }
  pre3::BatchView view{};
  int32_t* seg_counts = nullptr;          // internal scratch for fused decode
  uint32_t* scratch_mask = nullptr;       // internal bitmask when the caller passes none
  unsigned long long* best = nullptr;     // greedy argmax packed keys
  int prod = 0;                           // queue the next fill drains
  int last_consumed = -1;                 // queue the previous fill drained (reset by the next)
  int fill_seq = 0;                       // number of the next fill (heavy-list tags)
  bool slots_valid = false;               // seq_slot matches the stacks
  bool lookup_pending = false;            // queue[prod] got a lookup pass since the last fill
  bool arrivals_pending = false;          // a fill published per-sequence arrivals nobody consumed yet

  // seq_arrive must start at zero for a fused tail or a publishing fill.
  void ClearArrivals(cudaStream_t s) {
    if (arrivals_pending) {
      Check(cudaMemsetAsync(view.seq_arrive, 0, static_cast<size_t>(view.B) * 4, s), "memset");
      arrivals_pending = false;
    }
  }

  // Queue roles of a fill launch (3-queue ring, see kernels.cuh BatchView).
  void BeginFill(pre3::FillArgs* f) const {
    f->consume = prod;
    f->produce = (prod + 1) % 3;
    f->reset = last_consumed;
    f->fill_no = fill_seq;
  }
  void EndFill(bool tail) {
    fill_seq = (fill_seq + 1) % pre3::kFillPeriod;
    last_consumed = prod;
    prod = (prod + 1) % 3;
    // seq_slot / seq_hmask / heavy_index are double-buffered by fill parity
    // and their heavy-list tags recur every kFillPeriod fills: the next fill's
    // rows hold this batch's current contexts only when a lookup pass wrote
    // them for it — the fused tail's, or a later accept's (AcceptLookupQueue).
    // Otherwise the next fill runs LookupKernel first (two fills in a row,
    // a sample without accept), never reading rows written for an older fill.
    slots_valid = tail;
    lookup_pending = tail;  // the tail fed the new queue[prod]
  }

  // Queue for an accept's fused lookup, or -1 (then the next fill looks up).
  int AcceptLookupQueue() {
    if (lookup_pending) {
      slots_valid = false;
      return -1;
    }
    lookup_pending = true;
    slots_valid = true;
    return prod;
  }
  int sms = 148;  // the device's SM count
  bool split_two_kernels = false;  // PRE3_SPLIT_TWO_KERNELS=1 at batch creation (tests, A/B)
  // Split step in one grid (the accepts as CTAs among the fill's light
  // CTAs): measured faster at 256, 1,024 and 4,096 sequences (+9 %, +11 %,
  // +3 %; the PDL accept grid only starts with the fill's last wave).  The
  // fill + accept kernel form stays for PRE3_SPLIT_TWO_KERNELS and batches
  // past PRE3_ONE_GRID_CTAS_PER_SM light CTAs per SM (default: no limit).
  bool OneGridSplit() const {
    return PRE3_SPLIT_ONE_GRID && !split_two_kernels &&
           static_cast<int64_t>(view.B) * engine->nseg <= static_cast<int64_t>(8) * PRE3_ONE_GRID_CTAS_PER_SM * sms;
  }
  cudaStream_t capture_stream = nullptr;  // graph capture (the legacy stream cannot capture)
  std::vector<void*> owned;
  ~gm_batch() {
    cudaSetDevice(engine->device);
    auto& bs = engine->batches;
    bs.erase(std::remove(bs.begin(), bs.end(), this), bs.end());
    if (capture_stream) cudaStreamDestroy(capture_stream);
    // Builds still queued belong to contexts other batches may already use.
    for (int q = 0; q < 3; ++q) pre3::LaunchDrain(engine->aut, engine->vocab, engine->cache, view, q, nullptr);
    cudaDeviceSynchronize();
    for (void* p : owned) cudaFree(p);
  }
};

namespace {

// gm_engine_evict's work, on stream s (every batch of the engine idle).
void Evict(gm_engine* e, cudaStream_t s) {
  std::vector<const int32_t*> ptrs;
  std::vector<int> counts;
  for (gm_batch* b : e->batches) {
    ptrs.push_back(b->view.seq_slot);
    counts.push_back(2 * b->view.B);  // both fill parities
  }
  Check(pre3::LaunchEvict(e->cache, e->nseg, ptrs.data(), counts.data(), static_cast<int>(ptrs.size()),
                          e->evict_keep, s),
        "evict launch");
}

// Auto-eviction check at the start of a batch's fill (never while the
// stream is being captured into a graph): the free-row count the device
// mirrored at its latest pop (or eviction).
void MaybeEvict(gm_batch* b, cudaStream_t s) {
  gm_engine* e = b->engine;
  if (e->auto_evict_free <= 0) return;
  if (*reinterpret_cast<volatile int32_t*>(e->host_free) >= e->auto_evict_free) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  Check(cudaStreamIsCapturing(s, &cap), "capture status");
  if (cap != cudaStreamCaptureStatusNone) return;
  *reinterpret_cast<volatile int32_t*>(e->host_free) = e->cache.C;  // until the eviction writes the real count
  Evict(e, s);
}

}  // namespace

extern "C" {

const char* gm_last_error(void) { return g_last_error.c_str(); }
int gm_abi_version(void) { return GM_ABI_VERSION; }

// ---------------------------------------------------------------- automaton
int gm_automaton_load(const void* data, size_t bytes, gm_automaton** out) {
  return Guard([&]() -> int {
    if (!data || !out) return Fail(GM_ERR_USAGE, "null argument");
    const auto* p = static_cast<const uint8_t*>(data);
    const bool flat = bytes >= 6 && std::memcmp(p, "P3DPDA", 6) == 0;
    auto* a = new gm_automaton{flat ? pre3::LoadFlat(p, bytes) : pre3::LoadGmaskdp1(p, bytes)};
    *out = a;
    return GM_OK;
  });
}

int gm_automaton_compile(const char* text, int aggregate, int merge, gm_automaton** out) {
  return Guard([&]() -> int {
    if (!text || !out) return Fail(GM_ERR_USAGE, "null argument");
    auto* a = new gm_automaton{pre3::CompileGrammar(text, aggregate != 0, merge != 0)};
    *out = a;
    return GM_OK;
  });
}

int gm_automaton_save(const gm_automaton* a, void* buf, size_t cap, size_t* size) {
  return Guard([&]() -> int {
    if (!a || !size) return Fail(GM_ERR_USAGE, "null argument");
    std::vector<uint8_t> v = pre3::SaveFlat(a->a);
    *size = v.size();
    if (buf) {
      if (cap < v.size()) return Fail(GM_ERR_USAGE, "buffer too small");
      std::memcpy(buf, v.data(), v.size());
    }
    return GM_OK;
  });
}

int gm_automaton_save_gmaskdp1(const gm_automaton* a, void* buf, size_t cap, size_t* size) {
  return Guard([&]() -> int {
    if (!a || !size) return Fail(GM_ERR_USAGE, "null argument");
    std::vector<uint8_t> v = pre3::SaveGmaskdp1(a->a);
    *size = v.size();
    if (buf) {
      if (cap < v.size()) return Fail(GM_ERR_USAGE, "buffer too small");
      std::memcpy(buf, v.data(), v.size());
    }
    return GM_OK;
  });
}

int gm_vocab_load_json(const void* data, size_t bytes, uint8_t* tok_bytes, int64_t bytes_cap, int64_t* tok_offsets,
                       int32_t tokens_cap, int32_t* num_tokens, int64_t* total_bytes) {
  return Guard([&]() -> int {
    if (!data || !num_tokens || !total_bytes) return Fail(GM_ERR_USAGE, "null argument");
    const std::vector<std::string> v = pre3::LoadVocabularyJson(static_cast<const uint8_t*>(data), bytes);
    int64_t total = 0;
    for (const std::string& t : v) total += static_cast<int64_t>(t.size());
    *num_tokens = static_cast<int32_t>(v.size());
    *total_bytes = total;
    if (tok_bytes == nullptr || tok_offsets == nullptr) return GM_OK;
    if (bytes_cap < total || tokens_cap < static_cast<int32_t>(v.size())) {
      return Fail(GM_ERR_USAGE, "buffer too small");
    }
    int64_t o = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      tok_offsets[i] = o;
      std::memcpy(tok_bytes + o, v[i].data(), v[i].size());
      o += static_cast<int64_t>(v[i].size());
    }
    tok_offsets[v.size()] = o;
    return GM_OK;
  });
}

int gm_automaton_destroy(gm_automaton* a) {
  delete a;
  return GM_OK;
}

int gm_automaton_compile_stats(const gm_automaton* a, int64_t stats[4]) {
  if (!a || !stats) return Fail(GM_ERR_USAGE, "null argument");
  stats[0] = a->a.composites;
  stats[1] = a->a.cycles;
  stats[2] = 0;
  stats[3] = 0;
  return GM_OK;
}

int gm_automaton_info(const gm_automaton* a, int64_t info[8]) {
  if (!a || !info) return Fail(GM_ERR_USAGE, "null argument");
  int64_t maxpop = 0, maxpush = 0, dyn = 0;
  for (const auto& e : a->a.edges) {
    maxpop = std::max<int64_t>(maxpop, static_cast<int64_t>(e.match_pop.size()));
    maxpush = std::max<int64_t>(maxpush, static_cast<int64_t>(e.push.size()));
    dyn += e.dynamic;
  }
  info[0] = a->a.num_states;
  info[1] = static_cast<int64_t>(a->a.edges.size());
  info[2] = a->a.initial_state;
  info[3] = a->a.accept_state;
  info[4] = maxpop;
  info[5] = maxpush;
  info[6] = dyn;
  info[7] = static_cast<int64_t>(a->a.grammar_hash);
  return GM_OK;
}

// ---------------------------------------------------------------- engine
int gm_engine_create(const gm_automaton* a, const uint8_t* tok_bytes, const int64_t* tok_offsets,
                     int32_t num_tokens, const gm_engine_options* opts, int device,
                     gm_engine** out) {
  return Guard([&]() -> int {
    if (!a || !out || num_tokens < 0 || (num_tokens > 0 && (!tok_bytes || !tok_offsets))) {
      return Fail(GM_ERR_USAGE, "bad argument");
    }
    gm_engine_options o{8, 8192, 0, pre3::kSegWords, 0, 0, nullptr, 0};
    if (opts) {
      if (opts->context_depth) o.context_depth = opts->context_depth;
      if (opts->context_slots) o.context_slots = opts->context_slots;
      if (opts->segment_words) o.segment_words = opts->segment_words;
      o.parent_depth = opts->parent_depth;
      o.num_columns = opts->num_columns;
      o.eos_column = opts->eos_column;
      o.disabled = opts->disabled;
      o.auto_evict_free = opts->auto_evict_free;
    }
    if (o.auto_evict_free < 0) return Fail(GM_ERR_USAGE, "auto_evict_free must be >= 0");
    const int32_t W = (num_tokens + 1 + 31) / 32;
    auto is_disabled = [&](int32_t i) { return o.disabled && ((o.disabled[i >> 5] >> (i & 31)) & 1u); };
    if (o.num_columns < 0) return Fail(GM_ERR_USAGE, "num_columns must be >= 0");
    if (o.num_columns > 0) {
      if (o.eos_column < 0 || o.eos_column >= o.num_columns) return Fail(GM_ERR_USAGE, "eos_column out of range");
      if (o.num_columns < num_tokens) return Fail(GM_ERR_USAGE, "num_columns < V");
      if (o.eos_column < num_tokens && !is_disabled(o.eos_column)) {
        return Fail(GM_ERR_USAGE, "eos_column < V must name a disabled id");
      }
    }
    // Parent key depth R: new contexts keyed K deep are built from the
    // context of the same stack top keyed R deep (0 = default min(4, K-1);
    // negative = off: every new context is built over the whole vocabulary).
    if (o.parent_depth == 0) o.parent_depth = o.context_depth > 1 ? std::min<int64_t>(4, o.context_depth - 1) : -1;
    if (o.parent_depth >= o.context_depth) return Fail(GM_ERR_USAGE, "parent_depth must be < context_depth");
    if (o.parent_depth < 0) o.parent_depth = 0;
    if (o.context_depth < 1 || o.context_depth > pre3::kMaxContext) return Fail(GM_ERR_USAGE, "context_depth must be 1..32");
    if (o.context_slots < 1 || (o.context_slots & (o.context_slots - 1))) return Fail(GM_ERR_USAGE, "context_slots must be a power of two");
    if (o.segment_words != pre3::kSegWords) return Fail(GM_ERR_USAGE, "segment_words must be 256");
    if (tok_offsets && tok_offsets[num_tokens] > (int64_t{1} << 31) - 1) return Fail(GM_ERR_USAGE, "vocabulary bytes exceed 2^31");

    // TokenTrie::Build's vocabulary rules (runtime.cpp:23-53): no empty
    // tokens, no duplicates; the first offending id is reported.
    std::unordered_set<std::string_view> seen;
    seen.reserve(static_cast<size_t>(num_tokens) * 2);
    std::vector<int32_t> offs(static_cast<size_t>(num_tokens) + 1);
    for (int32_t i = 0; i < num_tokens; ++i) {
      const int64_t lo = tok_offsets[i], hi = tok_offsets[i + 1];
      if (hi < lo) return Fail(GM_ERR_USAGE, "token offsets not monotone");
      offs[static_cast<size_t>(i)] = static_cast<int32_t>(lo - tok_offsets[0]);
      if (is_disabled(i)) continue;  // never allowed: bytes ignored, exempt from the trie rules
      if (hi == lo) return Fail(GM_ERR_VOCAB_EMPTY, "EmptyToken: token " + std::to_string(i) + " has no bytes");
      std::string_view sv(reinterpret_cast<const char*>(tok_bytes + lo), static_cast<size_t>(hi - lo));
      if (!seen.insert(sv).second) {
        int32_t first = -1;
        for (int32_t j = 0; j < i; ++j) {
          if (is_disabled(j)) continue;
          if (std::string_view(reinterpret_cast<const char*>(tok_bytes + tok_offsets[j]),
                               static_cast<size_t>(tok_offsets[j + 1] - tok_offsets[j])) == sv) {
            first = j;
            break;
          }
        }
        return Fail(GM_ERR_VOCAB_DUPLICATE, "DuplicateToken: tokens " + std::to_string(first) + " and " +
                                                std::to_string(i) + " are identical");
      }
    }
    offs[static_cast<size_t>(num_tokens)] = num_tokens ? static_cast<int32_t>(tok_offsets[num_tokens] - tok_offsets[0]) : 0;

    Check(cudaSetDevice(device), "cudaSetDevice");
    auto e = std::make_unique<gm_engine>();
    e->device = device;
    pre3::FlatLayout f = pre3::Flatten(a->a);
    e->aut.rec_begin = DevUpload(f.rec_begin, &e->owned);
    e->aut.recs = DevUpload(f.recs, &e->owned);
    e->aut.first = DevUpload(f.first, &e->owned);
    e->aut.hidx_meta = reinterpret_cast<const int2*>(DevUpload(f.hidx_meta, &e->owned));
    e->aut.hidx_lens = DevUpload(f.hidx_lens, &e->owned);
    e->aut.hidx_exact = reinterpret_cast<const unsigned long long*>(DevUpload(f.hidx_exact, &e->owned));
    e->aut.hidx_prefix = reinterpret_cast<const unsigned long long*>(DevUpload(f.hidx_prefix, &e->owned));
    e->aut.hidx_exact_mask = f.hidx_exact.size() / 2 - 1;
    e->aut.hidx_prefix_mask = f.hidx_prefix.size() - 1;
    e->aut.rec_cond = DevUpload(f.rec_cond, &e->owned);
    e->aut.rec_push = DevUpload(f.rec_push, &e->owned);
    e->aut.shift = DevUpload(a->a.shift_targets, &e->owned);
    e->aut.state_any = DevUpload(f.state_any, &e->owned);
    e->aut.num_states = a->a.num_states;
    e->aut.initial = a->a.initial_state;
    e->grammar_hash = a->a.grammar_hash;
    {
      uint64_t h = HashVec(f.rec_begin, 1);
      h = HashVec(f.recs, h);
      h = HashVec(f.rec_cond, h);
      h = HashVec(f.rec_push, h);
      h = HashVec(a->a.shift_targets, h);
      const int64_t ids[2] = {a->a.num_states, a->a.initial_state};
      e->layout_hash = Hash64(ids, sizeof ids, h);
    }

    e->V = num_tokens;
    e->W = (num_tokens + 1 + 31) / 32;
    e->nseg = (e->W + pre3::kSegWords - 1) / pre3::kSegWords;
    std::vector<uint8_t> bytes(num_tokens ? tok_bytes + tok_offsets[0] : tok_bytes,
                               num_tokens ? tok_bytes + tok_offsets[num_tokens] : tok_bytes);
    e->vocab.tok_off = DevUpload(offs, &e->owned);
    e->vocab.tok_bytes = DevUpload(bytes, &e->owned);
    // Token records: offset, length and the first 8 bytes in one 16-B load
    // (a walk's first round trip; longer tokens read the rest from tok_bytes).
    // Entry V is EOS: length 1, no bytes.
    std::vector<int32_t> recs(4 * (static_cast<size_t>(num_tokens) + 1), 0);
    // A disabled id keeps length 0: every walk of it rejects, accepting it
    // kills the sequence.
    for (int32_t i = 0; i < num_tokens; ++i) {
      const int32_t lo = offs[static_cast<size_t>(i)];
      const int32_t len = is_disabled(i) ? 0 : offs[static_cast<size_t>(i) + 1] - lo;
      uint32_t w[2] = {0u, 0u};
      for (int32_t j = 0; j < len && j < 8; ++j) w[j >> 2] |= static_cast<uint32_t>(bytes[static_cast<size_t>(lo + j)]) << (8 * (j & 3));
      recs[4 * static_cast<size_t>(i) + 0] = lo;
      recs[4 * static_cast<size_t>(i) + 1] = len;
      recs[4 * static_cast<size_t>(i) + 2] = static_cast<int32_t>(w[0]);
      recs[4 * static_cast<size_t>(i) + 3] = static_cast<int32_t>(w[1]);
    }
    recs[4 * static_cast<size_t>(num_tokens) + 1] = 1;
    e->vocab.tok_rec = reinterpret_cast<const int4*>(DevUpload(recs, &e->owned));
    e->structural = DevAlloc<uint32_t>(static_cast<size_t>(e->W), &e->owned);
    Check(cudaMemset(e->structural, 0, sizeof(uint32_t) * static_cast<size_t>(e->W)), "memset");
    e->vocab.structural = e->structural;
    e->vocab.V = e->V;
    e->vocab.W = e->W;
    e->vocab.nseg = e->nseg;
    e->vocab.layout = o.num_columns > 0 && !(o.num_columns == num_tokens + 1 && o.eos_column == num_tokens);
    e->vocab.ncols = e->vocab.layout ? o.num_columns : num_tokens + 1;
    e->vocab.eos_col = e->vocab.layout ? o.eos_column : num_tokens;
    if (o.disabled) {
      e->disabled.assign(o.disabled, o.disabled + W);
      e->disabled[static_cast<size_t>(num_tokens >> 5)] &= (1u << (num_tokens & 31)) - 1u;  // ids < V only
    }
    {
      uint64_t h = HashVec(bytes, 2);
      h = HashVec(recs, h);  // offsets and lengths (0 = disabled)
      const int32_t lay[3] = {e->vocab.ncols, e->vocab.eos_col, num_tokens};
      e->vocab_hash = Hash64(lay, sizeof lay, h);
    }

    const size_t C = static_cast<size_t>(o.context_slots);
    auto& c = e->cache;
    c.C = o.context_slots;
    c.IC = 2 * o.context_slots;
    c.K = o.context_depth;
    c.slot_hash = DevAlloc<unsigned long long>(2 * C, &e->owned);
    Check(cudaMemset(c.slot_hash, 0, 2 * C * 8), "memset");
    {
      std::vector<int32_t> fr(C);
      for (size_t i = 0; i < C; ++i) fr[i] = static_cast<int32_t>(C - 1 - i);  // pops hand out rows 0, 1, ...
      c.row_free = DevUpload(fr, &e->owned);
      const int32_t n = o.context_slots;
      c.row_free_n = DevUpload(std::vector<int32_t>{n}, &e->owned);
    }
    c.row_ref = DevAlloc<uint8_t>(C, &e->owned);
    Check(cudaMemset(c.row_ref, 0, C), "memset");
    e->evict_keep = DevAlloc<uint8_t>(C, &e->owned);
    e->auto_evict_free = o.auto_evict_free;
    Check(cudaHostAlloc(reinterpret_cast<void**>(&e->host_free), 4, cudaHostAllocMapped), "host alloc");
    *e->host_free = o.context_slots;
    Check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.host_free), e->host_free, 0), "mapped pointer");
    c.slot_meta = DevAlloc<int32_t>(C, &e->owned);
    c.slot_keys = DevAlloc<int32_t>(C * static_cast<size_t>(pre3::kMaxContext), &e->owned);
    c.ci = DevAlloc<uint32_t>(C * static_cast<size_t>(e->W), &e->owned);
    c.cdb = DevAlloc<uint32_t>(C * static_cast<size_t>(e->W), &e->owned);
    c.cd_cnt = DevAlloc<int32_t>(C * static_cast<size_t>(e->nseg), &e->owned);
    c.seg_done = DevAlloc<int32_t>(C * static_cast<size_t>(e->nseg), &e->owned);
    c.seg_claim = DevAlloc<int32_t>(C * static_cast<size_t>(e->nseg), &e->owned);
    Check(cudaMemset(c.seg_claim, 0, C * static_cast<size_t>(e->nseg) * 4), "memset");
    c.slot_built = DevAlloc<int32_t>(C, &e->owned);
    c.slot_parent = DevAlloc<int32_t>(C, &e->owned);
    Check(cudaMemset(c.slot_parent, 0xff, C * 4), "memset");
    c.R = static_cast<int32_t>(o.parent_depth);
    c.W = e->W;
    c.eos_word = num_tokens >> 5;
    c.eos_bit = 1u << (num_tokens & 31);
    c.eos_segbit = 0u;
    if (e->vocab.layout && e->vocab.eos_col < num_tokens) {
      const int eseg = (e->vocab.eos_col >> 5) / pre3::kSegWords;
      if (eseg < 32) c.eos_segbit = 1u << eseg;
    }
    c.cd_segmask = DevAlloc<uint32_t>(C, &e->owned);
    Check(cudaMemset(c.cd_segmask, 0, C * 4), "memset");
    c.ci_cnt = DevAlloc<int32_t>(C * static_cast<size_t>(e->nseg) * 2, &e->owned);
    Check(cudaMemset(c.ci_cnt, 0, C * static_cast<size_t>(e->nseg) * 8), "memset");
    Check(cudaMemset(c.slot_built, 0, C * 4), "memset");
    c.counters = DevAlloc<unsigned long long>(8, &e->owned);
    Check(cudaMemset(c.slot_meta, 0, C * 4), "memset");
    Check(cudaMemset(c.cd_cnt, 0, C * static_cast<size_t>(e->nseg) * 4), "memset");
    Check(cudaMemset(c.seg_done, 0, C * static_cast<size_t>(e->nseg) * 4), "memset");
    Check(cudaMemset(c.counters, 0, 64), "memset");
    Check(cudaDeviceSynchronize(), "engine upload");
    *out = e.release();
    return GM_OK;
  });
}

int gm_engine_destroy(gm_engine* e) {
  delete e;
  return GM_OK;
}

int gm_engine_info(gm_engine* e, int64_t info[8]) {
  return Guard([&]() -> int {
    if (!e || !info) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    unsigned long long ctr[8];
    Check(cudaMemcpy(ctr, e->cache.counters, 64, cudaMemcpyDeviceToHost), "info");
    info[0] = e->V;
    info[1] = e->W;
    info[2] = e->nseg;
    info[3] = static_cast<int64_t>(ctr[0]);
    info[4] = static_cast<int64_t>(ctr[1]);
    info[5] = static_cast<int64_t>(ctr[2]);
    info[6] = static_cast<int64_t>(ctr[3]);
    info[7] = e->device;
    return GM_OK;
  });
}

int gm_engine_set_structural(gm_engine* e, const uint32_t* host_words) {
  return Guard([&]() -> int {
    if (!e || !host_words) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    std::vector<uint32_t> w(host_words, host_words + e->W);
    w[static_cast<size_t>(e->V >> 5)] &= ~(1u << (e->V & 31));  // EOS is never structural
    for (size_t i = 0; i < e->disabled.size(); ++i) w[i] &= ~e->disabled[i];
    Check(cudaDeviceSynchronize(), "structural: fills in flight");
    Check(cudaMemcpy(e->structural, w.data(), w.size() * 4, cudaMemcpyHostToDevice), "structural");
    // Contexts built before this call counted the old set.
    Check(pre3::LaunchRecountStructural(e->cache, e->vocab), "structural recount");
    Check(cudaDeviceSynchronize(), "structural recount");
    return GM_OK;
  });
}

// ---------------------------------------------------------------- batch
int gm_batch_create(gm_engine* e, int32_t batch, int32_t stack_capacity, gm_batch** out) {
  return Guard([&]() -> int {
    if (!e || !out || batch < 0 || stack_capacity < 1) return Fail(GM_ERR_USAGE, "bad argument");
    if (stack_capacity > 48 * 1024) return Fail(GM_ERR_USAGE, "stack_capacity must be <= 49152");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    auto b = std::make_unique<gm_batch>();
    b->engine = e;
    auto& v = b->view;
    v.B = batch;
    v.cap = stack_capacity;
    v.seq = DevAlloc<pre3::SeqState>(static_cast<size_t>(batch), &b->owned);
    v.stacks = DevAlloc<int32_t>(static_cast<size_t>(batch) * static_cast<size_t>(stack_capacity), &b->owned);
    v.err = DevAlloc<unsigned int>(1, &b->owned);
    v.stats = DevAlloc<unsigned long long>(8, &b->owned);
    v.counters = DevAlloc<unsigned long long>(4, &b->owned);
    v.stats_enabled = 0;
    v.trace = nullptr;
    v.trace_cap = 0;
    const size_t bn = static_cast<size_t>(std::max(batch, 1)) * static_cast<size_t>(e->nseg);
    v.nseg = e->nseg;
    v.seq_slot = DevAlloc<int32_t>(2 * static_cast<size_t>(batch), &b->owned);  // by fill parity
    v.seq_hmask = DevAlloc<uint32_t>(2 * static_cast<size_t>(batch), &b->owned);
    Check(cudaMemset(v.seq_hmask, 0xff, 2 * static_cast<size_t>(batch) * 4), "memset");
    v.priv = DevAlloc<uint32_t>(static_cast<size_t>(batch) * static_cast<size_t>(e->W), &b->owned);
    v.priv_done = DevAlloc<int32_t>(bn, &b->owned);
    v.heavy_index = DevAlloc<int32_t>(2 * bn, &b->owned);  // double-buffered by fill parity
    Check(cudaMemset(v.heavy_index, 0xff, 2 * bn * 4), "memset");
    v.h_cap = static_cast<int32_t>(std::min<size_t>(bn, std::max<size_t>(64, 2 * static_cast<size_t>(batch))));
    Check(cudaMemset(v.priv_done, 0, bn * 4), "memset");
    for (int q = 0; q < 3; ++q) {
      v.queue[q].items = DevAlloc<int4>(4 * bn, &b->owned);  // a new context may queue its parent too
      v.queue[q].n_items = DevAlloc<unsigned int>(1, &b->owned);
      v.queue[q].next_unit = DevAlloc<unsigned int>(1, &b->owned);
      v.queue[q].heavy = DevAlloc<int2>(static_cast<size_t>(v.h_cap), &b->owned);
      v.queue[q].n_heavy = DevAlloc<unsigned int>(1, &b->owned);
      Check(cudaMemset(v.queue[q].n_heavy, 0, 4), "memset");
      Check(cudaMemset(v.queue[q].n_items, 0, 4), "memset");
      Check(cudaMemset(v.queue[q].next_unit, 0, 4), "memset");
    }
    v.seq_arrive = DevAlloc<int32_t>(static_cast<size_t>(batch), &b->owned);
    Check(cudaMemset(v.seq_arrive, 0, static_cast<size_t>(batch) * 4), "memset");
    v.kernel_done = DevAlloc<unsigned int>(1, &b->owned);
    Check(cudaMemset(v.kernel_done, 0, 4), "memset");
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
    v.build_grid = sms * 4;
    v.h_grid = std::min(v.h_cap, PRE3_HEAVY_PER_SM * sms);
    b->sms = sms;
    if (const char* two = std::getenv("PRE3_SPLIT_TWO_KERNELS")) b->split_two_kernels = std::atoi(two) != 0;
    b->seg_counts = DevAlloc<int32_t>(bn * 2, &b->owned);
    b->scratch_mask = DevAlloc<uint32_t>(static_cast<size_t>(batch) * static_cast<size_t>(e->W), &b->owned);
    b->best = DevAlloc<unsigned long long>(static_cast<size_t>(batch), &b->owned);
    Check(cudaMemset(v.err, 0, 4), "memset");
    Check(cudaMemset(v.stats, 0, 64), "memset");
    Check(cudaMemset(v.counters, 0, 32), "memset");
    Check(cudaMemset(b->best, 0, static_cast<size_t>(batch) * 8), "memset");
    Check(pre3::LaunchReset(e->aut, v, nullptr), "reset");
    Check(cudaDeviceSynchronize(), "batch create");
    e->batches.push_back(b.get());
    *out = b.release();
    return GM_OK;
  });
}

int gm_batch_destroy(gm_batch* b) {
  delete b;
  return GM_OK;
}

int gm_batch_reset(gm_batch* b, void* stream) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    Check(pre3::LaunchReset(b->engine->aut, b->view, static_cast<cudaStream_t>(stream)), "reset");
    b->slots_valid = false;
    return GM_OK;
  });
}

int gm_batch_download(gm_batch* b, int32_t seq, int32_t* state, int32_t* status, int32_t* stack,
                      int32_t cap, int32_t* depth) {
  return Guard([&]() -> int {
    if (!b || seq < 0 || seq >= b->view.B) return Fail(GM_ERR_USAGE, "bad sequence index");
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    Check(cudaDeviceSynchronize(), "sync");
    pre3::SeqState st;
    Check(cudaMemcpy(&st, b->view.seq + seq, sizeof(st), cudaMemcpyDeviceToHost), "download");
    if (depth) *depth = st.depth;
    if (status) *status = st.status;
    const int32_t n = std::min(st.depth, cap);
    std::vector<int32_t> tmp(static_cast<size_t>(std::max(st.depth, 1)));
    Check(cudaMemcpy(tmp.data(), b->view.stacks + static_cast<int64_t>(seq) * b->view.cap,
                     sizeof(int32_t) * static_cast<size_t>(std::max(st.depth, 1)), cudaMemcpyDeviceToHost),
          "download");
    if (stack && n > 0) std::memcpy(stack, tmp.data(), sizeof(int32_t) * static_cast<size_t>(n));
    if (state) *state = st.depth > 0 ? tmp[static_cast<size_t>(st.depth - 1)] : -1;
    return GM_OK;
  });
}

int gm_batch_upload(gm_batch* b, int32_t seq, int32_t status, const int32_t* stack, int32_t depth) {
  return Guard([&]() -> int {
    if (!b || seq < 0 || seq >= b->view.B || !stack) return Fail(GM_ERR_USAGE, "bad argument");
    if (depth < 1 || depth > b->view.cap) return Fail(GM_ERR_STACK_OVERFLOW, "stack depth exceeds capacity");
    for (int32_t i = 0; i < depth; ++i) {
      if (stack[i] < 0 || stack[i] >= b->engine->aut.num_states) return Fail(GM_ERR_USAGE, "state out of range");
    }
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    Check(cudaDeviceSynchronize(), "sync");
    pre3::SeqState st;
    Check(cudaMemcpy(&st, b->view.seq + seq, sizeof(st), cudaMemcpyDeviceToHost), "upload");
    st.depth = depth;
    st.status = status;
    Check(cudaMemcpy(b->view.seq + seq, &st, sizeof(st), cudaMemcpyHostToDevice), "upload");
    Check(cudaMemcpy(b->view.stacks + static_cast<int64_t>(seq) * b->view.cap, stack,
                     sizeof(int32_t) * static_cast<size_t>(depth), cudaMemcpyHostToDevice),
          "upload");
    b->slots_valid = false;
    return GM_OK;
  });
}

int gm_batch_check(gm_batch* b, void* stream) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    Check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "stream sync");
    unsigned int err = 0;
    Check(cudaMemcpy(&err, b->view.err, 4, cudaMemcpyDeviceToHost), "check");
    if (err) {
      Check(cudaMemset(b->view.err, 0, 4), "memset");
      if (err & 2u) return Fail(GM_ERR_CUDA, "internal: an accept timed out waiting for its fill's items");
      return Fail(GM_ERR_STACK_OVERFLOW, "a mask walk pushed more than 256 entries above the stack (walk overlay)");
    }
    return GM_OK;
  });
}

int gm_batch_counters(gm_batch* b, int64_t counters[4]) {
  return Guard([&]() -> int {
    if (!b || !counters) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    unsigned long long c[4];
    Check(cudaMemcpy(c, b->view.counters, 32, cudaMemcpyDeviceToHost), "counters");
    for (int i = 0; i < 4; ++i) counters[i] = static_cast<int64_t>(c[i]);
    return GM_OK;
  });
}

int gm_batch_fill_stats(gm_batch* b, int64_t stats[6]) {
  return Guard([&]() -> int {
    if (!b || !stats) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    unsigned long long s[8];
    Check(cudaMemcpy(s, b->view.stats, 64, cudaMemcpyDeviceToHost), "stats");
    for (int i = 0; i < 6; ++i) stats[i] = static_cast<int64_t>(s[i]);
    Check(cudaMemset(b->view.stats, 0, 64), "memset");
    return GM_OK;
  });
}

int gm_batch_time_next_fill(gm_batch* b, void* start_event, void* end_event) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    b->time_fill[0] = static_cast<cudaEvent_t>(start_event);
    b->time_fill[1] = static_cast<cudaEvent_t>(end_event);
    return GM_OK;
  });
}

int gm_batch_set_trace(gm_batch* b, uint64_t* trace, int32_t capacity) {
  if (!b || (trace && capacity <= 0)) return Fail(GM_ERR_USAGE, "bad trace buffer");
  b->view.trace = reinterpret_cast<unsigned long long*>(trace);
  b->view.trace_cap = trace ? capacity : 0;
  return GM_OK;
}

int gm_batch_set_stats(gm_batch* b, int32_t enable) {
  if (!b) return Fail(GM_ERR_USAGE, "null batch");
  b->view.stats_enabled = enable ? 1 : 0;
  return GM_OK;
}

// ---------------------------------------------------------------- hot path
int gm_fill_next_token_bitmask(gm_batch* b, uint32_t* bitmask, int64_t ld_words, void* stream) {
  return gm_fill_and_mask_logits(b, bitmask, ld_words, nullptr, 0, nullptr, stream);
}

int gm_fill_and_mask_logits(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits,
                            int64_t ld, int32_t* seg_counts, void* stream) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    gm_engine* e = b->engine;
    if (bitmask && ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    if (logits && ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MaybeEvict(b, s);
    if (!b->slots_valid) Check(pre3::LaunchLookup(e->cache, b->view, b->prod, b->fill_seq, s), "lookup launch");
    pre3::FillArgs f{};
    f.bitmask = bitmask;
    f.ldw = ld_words;
    f.logits = logits;
    f.ld = ld;
    f.seg_counts = seg_counts;
    f.best = b->best;
    f.publish_arrival = 1;  // lets a following sample/accept start per sequence
    b->ClearArrivals(s);
    b->BeginFill(&f);
    b->FillStart(s);
    Check(pre3::LaunchFill(pre3::kFillMask, pre3::kTailNone, e->aut, e->vocab, e->cache, b->view, f, s), "fill launch");
    b->FillEnd(s);
    b->EndFill(false);
    b->arrivals_pending = true;
    return GM_OK;
  });
}

// One fused decode step: fill + in-place bf16 -inf logits + stream sample +
// accept + next-step context lookup, in a single launch.
int gm_decode_step_stream(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits, int64_t ld,
                          uint64_t seed, int32_t* tokens_out, void* stream) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    gm_engine* e = b->engine;
    if (bitmask && ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    if (logits && ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MaybeEvict(b, s);
    if (!b->slots_valid) Check(pre3::LaunchLookup(e->cache, b->view, b->prod, b->fill_seq, s), "lookup launch");
    pre3::FillArgs f{};
    f.bitmask = bitmask ? bitmask : b->scratch_mask;
    f.ldw = bitmask ? ld_words : e->W;
    f.logits = logits;
    f.ld = ld;
    f.seg_counts = b->seg_counts;
    f.best = b->best;
    f.tokens_out = tokens_out;
    f.seed = seed;
    b->ClearArrivals(s);
    b->BeginFill(&f);
    b->FillStart(s);
    Check(pre3::LaunchFill(pre3::kFillMask, pre3::kTailStream, e->aut, e->vocab, e->cache, b->view, f, s),
          "decode launch");
    b->FillEnd(s);
    b->EndFill(true);
    return GM_OK;
  });
}

// Two-kernel decode step: fill (arrivals only for sequences that are not
// pure CI), then the overlapping sample/accept/lookup kernel, which samples a
// pure-CI sequence from its slot's CI row and counts (the fill writes the same
// words and counts into bitmask/seg_counts) without waiting for the fill.
int gm_decode_step_stream_split(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits, int64_t ld,
                                int32_t* seg_counts, uint64_t seed, int32_t* tokens_out, void* stream) {
  return Guard([&]() -> int {
    if (!b) return Fail(GM_ERR_USAGE, "null batch");
    gm_engine* e = b->engine;
    if (bitmask && ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    if (logits && ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MaybeEvict(b, s);
    if (!b->slots_valid) Check(pre3::LaunchLookup(e->cache, b->view, b->prod, b->fill_seq, s), "lookup launch");
    pre3::FillArgs f{};
    f.bitmask = bitmask ? bitmask : b->scratch_mask;
    f.ldw = bitmask ? ld_words : e->W;
    f.logits = logits;
    f.ld = ld;
    f.seg_counts = seg_counts ? seg_counts : b->seg_counts;
    f.best = b->best;
    f.publish_arrival = 2;
    b->ClearArrivals(s);
    b->BeginFill(&f);
    const bool one_grid = b->OneGridSplit();
    if (!one_grid) {
      b->FillStart(s);
      Check(pre3::LaunchFill(pre3::kFillMask, pre3::kTailNone, e->aut, e->vocab, e->cache, b->view, f, s),
            "fill launch");
      b->FillEnd(s);
    }
    b->EndFill(false);
    pre3::AcceptArgs& g = f.acc;
    g.restart = 1;
    g.bitmask = f.bitmask;
    g.ldw = f.ldw;
    g.seg_counts = f.seg_counts;
    g.seed = seed;
    g.tokens_out = tokens_out;
    g.do_accept = 1;
    g.lookup_queue = b->AcceptLookupQueue();
    g.lookup_tag = b->fill_seq;
    g.wait_fill = 1;
    g.ci_shortcut = 1;
    if (one_grid) {
      // One grid: the accept CTAs run among the light CTAs (FillArgs::accept_ctas).
      f.accept_ctas = 1;
      b->FillStart(s);
      Check(pre3::LaunchFill(pre3::kFillMask, pre3::kTailNone, e->aut, e->vocab, e->cache, b->view, f, s),
            "fill launch");
      b->FillEnd(s);
    } else {
      Check(pre3::LaunchAccept(pre3::kSampleStream, e->aut, e->vocab, e->cache, b->view, g, s), "accept launch");
    }
    return GM_OK;
  });
}

int gm_batch_split_step_launches(gm_batch* b) {
  if (!b) return -Fail(GM_ERR_USAGE, "null batch");
  return b->OneGridSplit() ? 1 : 2;
}

int gm_allowed_terminals(gm_batch* b, uint32_t* out, void* stream) {
  return Guard([&]() -> int {
    if (!b || !out) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    Check(pre3::LaunchAllowed(e->aut, b->view, out, static_cast<cudaStream_t>(stream)), "allowed launch");
    return GM_OK;
  });
}

int gm_accept_tokens(gm_batch* b, const int32_t* tokens, int32_t* status_out, int32_t restart,
                     void* stream) {
  return Guard([&]() -> int {
    if (!b || !tokens) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    pre3::AcceptArgs g{};
    g.tokens = tokens;
    g.status_out = status_out;
    g.restart = restart;
    g.do_accept = 1;
    g.lookup_queue = b->AcceptLookupQueue();
    g.lookup_tag = b->fill_seq;
    Check(pre3::LaunchAccept(pre3::kSampleGiven, e->aut, e->vocab, e->cache, b->view, g,
                             static_cast<cudaStream_t>(stream)),
          "accept launch");
    return GM_OK;
  });
}

int gm_sample_stream_and_accept(gm_batch* b, const uint32_t* bitmask, int64_t ld_words,
                                const int32_t* seg_counts, uint64_t seed, int32_t* tokens_out,
                                void* stream) {
  return Guard([&]() -> int {
    if (!b || !bitmask || !seg_counts) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    if (ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    pre3::AcceptArgs g{};
    g.restart = 1;
    g.bitmask = bitmask;
    g.ldw = ld_words;
    g.seg_counts = seg_counts;
    g.seed = seed;
    g.tokens_out = tokens_out;
    g.do_accept = 1;
    g.lookup_queue = b->AcceptLookupQueue();
    g.lookup_tag = b->fill_seq;
    g.wait_fill = b->arrivals_pending ? 1 : 0;  // start per sequence while the fill finishes
    b->arrivals_pending = false;
    Check(pre3::LaunchAccept(pre3::kSampleStream, e->aut, e->vocab, e->cache, b->view, g,
                             static_cast<cudaStream_t>(stream)),
          "sample launch");
    return GM_OK;
  });
}

int gm_sample_stream(gm_batch* b, const uint32_t* bitmask, int64_t ld_words, const int32_t* seg_counts,
                     uint64_t seed, int32_t* tokens_out, void* stream) {
  return Guard([&]() -> int {
    if (!b || !bitmask || !seg_counts || !tokens_out) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    if (ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    pre3::AcceptArgs g{};
    g.bitmask = bitmask;
    g.ldw = ld_words;
    g.seg_counts = seg_counts;
    g.seed = seed;
    g.tokens_out = tokens_out;
    g.do_accept = 0;
    g.lookup_queue = -1;
    g.wait_fill = b->arrivals_pending ? 1 : 0;
    b->arrivals_pending = false;
    Check(pre3::LaunchAccept(pre3::kSampleStream, e->aut, e->vocab, e->cache, b->view, g,
                             static_cast<cudaStream_t>(stream)),
          "sample launch");
    return GM_OK;
  });
}

int gm_decode_step_greedy(gm_batch* b, const uint16_t* logits, int64_t ld, uint32_t* bitmask,
                          int64_t ld_words, int32_t* tokens_out, void* stream) {
  return Guard([&]() -> int {
    if (!b || !logits) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    if (ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    if (bitmask && ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    MaybeEvict(b, s);
    if (!b->slots_valid) Check(pre3::LaunchLookup(e->cache, b->view, b->prod, b->fill_seq, s), "lookup launch");
    pre3::FillArgs f{};
    f.bitmask = bitmask ? bitmask : b->scratch_mask;
    f.ldw = bitmask ? ld_words : e->W;
    f.logits = const_cast<uint16_t*>(logits);
    f.ld = ld;
    f.best = b->best;
    f.publish_arrival = 1;
    b->ClearArrivals(s);
    b->BeginFill(&f);
    // Two kernels: the argmax fill, then the accept kernel, which starts per
    // sequence while the fill's last wave runs (measured faster than the
    // one-launch fused tail, whose tails hold fill CTA slots).
    b->FillStart(s);
    Check(pre3::LaunchFill(pre3::kFillGreedy, pre3::kTailNone, e->aut, e->vocab, e->cache, b->view, f, s),
          "greedy fill launch");
    b->FillEnd(s);
    b->EndFill(false);
    pre3::AcceptArgs g{};
    g.best = b->best;
    g.tokens_out = tokens_out;
    g.restart = 1;
    g.do_accept = 1;
    g.lookup_queue = b->AcceptLookupQueue();
    g.lookup_tag = b->fill_seq;
    g.wait_fill = 1;
    Check(pre3::LaunchAccept(pre3::kSampleGreedy, e->aut, e->vocab, e->cache, b->view, g, s), "greedy accept launch");
    return GM_OK;
  });
}

namespace {
int SampleCommon(gm_batch* b, const uint16_t* logits, int64_t ld, const uint32_t* bitmask, int64_t ld_words,
                 float temperature, int32_t top_k, float top_p, uint64_t seed, int32_t* tokens_out, bool accept,
                 cudaStream_t s) {
  gm_engine* e = b->engine;
  if (!(temperature > 0.0f) || top_k < 0 || !(top_p > 0.0f)) {
    return Fail(GM_ERR_USAGE, "temperature > 0, top_k >= 0, top_p in (0, 1] required");
  }
  pre3::SampleArgs g{};
  g.bitmask = bitmask;
  g.ldw = ld_words;
  g.logits = logits;
  g.ld = ld;
  g.temperature = temperature;
  g.top_k = top_k;
  g.top_p24 = top_p >= 1.0f ? (1u << 24) : static_cast<uint32_t>(std::floor(static_cast<double>(top_p) * 16777216.0));
  if (g.top_p24 == 0u) g.top_p24 = 1u;
  g.seed = seed;
  g.tokens_out = tokens_out;
  g.do_accept = accept ? 1 : 0;
  g.restart = 1;
  g.lookup_queue = accept ? b->AcceptLookupQueue() : -1;
  g.lookup_tag = b->fill_seq;
  Check(pre3::LaunchSample(e->aut, e->vocab, e->cache, b->view, g, s), "sample launch");
  return GM_OK;
}
}  // namespace

int gm_sample_tokens(gm_batch* b, const uint16_t* logits_bf16, int64_t ld, const uint32_t* bitmask,
                     int64_t ld_words, float temperature, int32_t top_k, float top_p, uint64_t seed,
                     int32_t* tokens_out, int32_t accept, void* stream) {
  return Guard([&]() -> int {
    if (!b || !logits_bf16 || !bitmask) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    if (ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    if (ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    return SampleCommon(b, logits_bf16, ld, bitmask, ld_words, temperature, top_k, top_p, seed, tokens_out,
                        accept != 0, static_cast<cudaStream_t>(stream));
  });
}

int gm_decode_step_sample(gm_batch* b, const uint16_t* logits_bf16, int64_t ld, uint32_t* bitmask,
                          int64_t ld_words, float temperature, int32_t top_k, float top_p, uint64_t seed,
                          int32_t* tokens_out, void* stream) {
  return Guard([&]() -> int {
    if (!b || !logits_bf16) return Fail(GM_ERR_USAGE, "null argument");
    gm_engine* e = b->engine;
    if (ld < e->vocab.ncols) return Fail(GM_ERR_USAGE, "ld < the row's logit columns");
    if (bitmask && ld_words < e->W) return Fail(GM_ERR_USAGE, "ld_words < W");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t* bm = bitmask ? bitmask : b->scratch_mask;
    const int64_t ldw = bitmask ? ld_words : e->W;
    int rc = gm_fill_next_token_bitmask(b, bm, ldw, stream);
    if (rc != GM_OK) return rc;
    return SampleCommon(b, logits_bf16, ld, bm, ldw, temperature, top_k, top_p, seed, tokens_out, true, s);
  });
}

// ---------------------------------------------------------------- CUDA graphs
struct gm_graph {
  gm_batch* batch = nullptr;
  cudaGraphExec_t exec = nullptr;
  int prod0 = 0, last0 = 0, fill0 = 0, steps = 0;
  ~gm_graph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

int gm_decode_graph_create(gm_batch* b, int32_t kind, int32_t steps, uint32_t* const* bitmask, int64_t ld_words,
                           const uint16_t* const* logits, int64_t ld, int32_t* const* seg_counts, uint64_t seed,
                           int32_t* const* tokens_out, gm_graph** out) {
  return Guard([&]() -> int {
    if (!b || !out || steps <= 0 || steps % pre3::kFillPeriod != 0) {
      return Fail(GM_ERR_USAGE, "steps must be a positive multiple of 6");
    }
    if (kind != 0 && kind != 1) return Fail(GM_ERR_USAGE, "kind must be 0 (stream split step) or 1 (greedy)");
    if (kind == 1 && !logits) return Fail(GM_ERR_USAGE, "the greedy step needs logits");
    gm_engine* e = b->engine;
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    if (!b->capture_stream) Check(cudaStreamCreateWithFlags(&b->capture_stream, cudaStreamNonBlocking), "stream");
    cudaStream_t cs = b->capture_stream;
    // Steady state first (not captured): the next fill's context slots are
    // looked up and no arrivals are pending, as after any decode step — so
    // the captured steps launch exactly the fill + accept kernels.
    Check(cudaDeviceSynchronize(), "sync");
    if (!b->slots_valid) {
      Check(pre3::LaunchLookup(e->cache, b->view, b->prod, b->fill_seq, cs), "lookup launch");
      b->slots_valid = true;
      b->lookup_pending = true;
    }
    b->ClearArrivals(cs);
    // A fresh batch has no previously drained queue (reset = -1); every later
    // fill resets the queue drained before it.  Name that ring position now
    // (resetting the untouched queue is a no-op) so the captured first fill
    // is the same as at every replay start.
    if (b->last_consumed < 0) b->last_consumed = (b->prod + 2) % 3;
    Check(cudaStreamSynchronize(cs), "sync");
    auto g = std::make_unique<gm_graph>();
    g->batch = b;
    g->prod0 = b->prod;
    g->last0 = b->last_consumed;
    g->fill0 = b->fill_seq;
    g->steps = steps;
    cudaGraph_t graph = nullptr;
    Check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
    int rc = GM_OK;
    for (int32_t i = 0; i < steps && rc == GM_OK; ++i) {
      uint32_t* bm = bitmask ? bitmask[i] : nullptr;
      int32_t* to = tokens_out ? tokens_out[i] : nullptr;
      if (kind == 1) {
        rc = gm_decode_step_greedy(b, logits[i], ld, bm, ld_words, to, cs);
      } else {
        rc = gm_decode_step_stream_split(b, bm, ld_words, logits ? const_cast<uint16_t*>(logits[i]) : nullptr, ld,
                                         seg_counts ? seg_counts[i] : nullptr, seed, to, cs);
      }
    }
    const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
    if (rc != GM_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    Check(ec, "end capture");
    const cudaError_t ei = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    Check(ei, "graph instantiate");
    // The host bookkeeping advanced by `steps` (a multiple of the period):
    // it is back at the state the graph starts from.
    if (b->prod != g->prod0 || b->last_consumed != g->last0 || b->fill_seq != g->fill0 || !b->slots_valid ||
        !b->lookup_pending || b->arrivals_pending) {
      return Fail(GM_ERR_USAGE, "internal: step bookkeeping not periodic");
    }
    *out = g.release();
    return GM_OK;
  });
}

int gm_graph_launch(gm_graph* g, void* stream) {
  return Guard([&]() -> int {
    if (!g || !g->exec) return Fail(GM_ERR_USAGE, "null graph");
    gm_batch* b = g->batch;
    // The graph bakes in the queue ring position and fill numbers of its
    // capture: replay only from that state (any 6k eager steps return to it).
    if (b->prod != g->prod0 || b->last_consumed != g->last0 || b->fill_seq != g->fill0 || !b->slots_valid ||
        !b->lookup_pending || b->arrivals_pending) {
      return Fail(GM_ERR_USAGE, "batch is not at the graph's start state (run a multiple of 6 eager steps of the "
                                "same kind, or re-capture)");
    }
    Check(cudaSetDevice(b->engine->device), "cudaSetDevice");
    Check(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream)), "graph launch");
    return GM_OK;
  });
}

int gm_graph_destroy(gm_graph* g) {
  delete g;
  return GM_OK;
}

// ---------------------------------------------------------------- snapshots
// Context-table snapshot "P3GMCTX1" (the reference's cache
// precedent is SerializeDpda/DeserializeDpda, src/serialize.cpp:148-294):
// every fully built context row, keyed by (grammar hash
// (dpda_builder.cpp:469-476), device-layout hash, vocabulary + logit-layout
// hash, K, R, rows).  Little-endian:
//   header: magic[8] "P3GMCTX1", u32 version 2, u32 header bytes (96),
//           u64 grammar_hash, u64 layout_hash, u64 vocab_hash,
//           i32 K, R, C (rows), V, W, nseg, n (rows saved), kMaxContext,
//           u64 payload bytes, u64 payload checksum (Hash64), u64 0 (reserved)
//   payload: i32 row[n], i32 meta[n], i32 parent[n], u32 cd_segmask[n], then
//            per row a block of kMaxContext + 3*nseg + 2*W words: key row,
//            cd_cnt[nseg], ci_cnt[nseg][2], ci[W], cdb[W].
// Loading restores the rows at their ids and rebuilds the row index.
namespace {

constexpr char kSnapMagic[8] = {'P', '3', 'G', 'M', 'C', 'T', 'X', '1'};
constexpr uint32_t kSnapHeader = 96;
constexpr uint32_t kSnapVersion = 3;  // 3: chunked payload checksum (SnapChecksum)

struct SnapHeader {
  char magic[8];
  uint32_t version, header_bytes;
  uint64_t grammar_hash, layout_hash, vocab_hash;
  int32_t K, R, C, V, W, nseg, n, max_context;
  uint64_t payload_bytes, checksum, reserved;
};
static_assert(sizeof(SnapHeader) == kSnapHeader, "snapshot header layout");

constexpr int kSnapChunk = 1024;  // rows per gather/scatter launch

// Payload checksum: Hash64 of every 16 MiB chunk (hashed on up to 16 host
// threads), then Hash64 of those chunk hashes seeded with the length — the
// load of a multi-GB table is not held up by one core hashing it.
uint64_t SnapChecksum(const uint8_t* p, uint64_t n) {
  constexpr uint64_t kChunk = 16ull << 20;
  const size_t chunks = static_cast<size_t>((n + kChunk - 1) / kChunk);
  std::vector<uint64_t> hs(chunks);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned nt = static_cast<unsigned>(std::min<size_t>(hw, chunks));
  auto work = [&](unsigned t) {
    for (size_t c = t; c < chunks; c += nt) {
      const uint64_t off = c * kChunk;
      hs[c] = Hash64(p + off, static_cast<size_t>(std::min(kChunk, n - off)), 0x243F6A8885A308D3ull ^ c);
    }
  };
  if (nt <= 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  return Hash64(hs.data(), hs.size() * 8, 0x13198A2E03707344ull ^ n);
}

struct RowTables {
  std::vector<int32_t> meta, built, parent;
  std::vector<uint32_t> segmask;
};

RowTables ReadRowTables(const gm_engine* e) {
  const size_t C = static_cast<size_t>(e->cache.C);
  RowTables t;
  t.meta.resize(C);
  t.built.resize(C);
  t.parent.resize(C);
  t.segmask.resize(C);
  Check(cudaMemcpy(t.meta.data(), e->cache.slot_meta, C * 4, cudaMemcpyDeviceToHost), "snapshot read");
  Check(cudaMemcpy(t.built.data(), e->cache.slot_built, C * 4, cudaMemcpyDeviceToHost), "snapshot read");
  Check(cudaMemcpy(t.parent.data(), e->cache.slot_parent, C * 4, cudaMemcpyDeviceToHost), "snapshot read");
  Check(cudaMemcpy(t.segmask.data(), e->cache.cd_segmask, C * 4, cudaMemcpyDeviceToHost), "snapshot read");
  return t;
}

size_t SnapBlockWords(const gm_engine* e) {
  return static_cast<size_t>(pre3::kMaxContext) + 3 * static_cast<size_t>(e->nseg) + 2 * static_cast<size_t>(e->W);
}

// Gathers (scatter = false: device -> host blocks) or scatters the rows'
// blocks, kSnapChunk rows per launch through a device staging buffer.
void SnapshotRows(gm_engine* e, const std::vector<int32_t>& ids, uint8_t* host, bool scatter) {
  // Rows move in chunks of kSnapChunk through two pinned staging buffers:
  // the host copy of one chunk overlaps the transfer and gather/scatter
  // kernel of the other (the caller's buffer may be a pageable memory map).
  const size_t n = ids.size(), blk = SnapBlockWords(e);
  if (!n) return;
  const size_t cbytes = static_cast<size_t>(kSnapChunk) * blk * 4;
  std::vector<void*> tmp;
  void* pinned[2] = {nullptr, nullptr};
  cudaStream_t st = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  auto release = [&]() {
    if (st) cudaStreamSynchronize(st);
    for (void* q : tmp) cudaFree(q);
    for (void* q : pinned)
      if (q) cudaFreeHost(q);
    for (cudaEvent_t x : ev)
      if (x) cudaEventDestroy(x);
    if (st) cudaStreamDestroy(st);
  };
  try {
    int32_t* d_ids[2] = {DevAlloc<int32_t>(kSnapChunk, &tmp), DevAlloc<int32_t>(kSnapChunk, &tmp)};
    uint32_t* d_blk[2] = {DevAlloc<uint32_t>(kSnapChunk * blk, &tmp), DevAlloc<uint32_t>(kSnapChunk * blk, &tmp)};
    for (int q = 0; q < 2; ++q) {
      Check(cudaHostAlloc(&pinned[q], cbytes, cudaHostAllocDefault), "snapshot staging");
      Check(cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming), "snapshot event");
    }
    Check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "snapshot stream");
    const size_t chunks = (n + kSnapChunk - 1) / kSnapChunk;
    auto rows = [&](size_t k) { return static_cast<int>(std::min<size_t>(kSnapChunk, n - k * kSnapChunk)); };
    auto launch = [&](size_t k) {  // chunk k on the stream (staging buffer k % 2)
      const int q = static_cast<int>(k & 1), m = rows(k);
      const size_t bytes = static_cast<size_t>(m) * blk * 4;
      Check(cudaMemcpyAsync(d_ids[q], ids.data() + k * kSnapChunk, static_cast<size_t>(m) * 4, cudaMemcpyHostToDevice,
                            st), "snapshot");
      if (scatter) Check(cudaMemcpyAsync(d_blk[q], pinned[q], bytes, cudaMemcpyHostToDevice, st), "snapshot");
      Check(pre3::LaunchSnapshotRows(e->cache, e->W, e->nseg, d_ids[q], m, d_blk[q], scatter, st), "snapshot rows");
      if (!scatter) Check(cudaMemcpyAsync(pinned[q], d_blk[q], bytes, cudaMemcpyDeviceToHost, st), "snapshot");
      Check(cudaEventRecord(ev[q], st), "snapshot event");
    };
    if (scatter) {
      for (size_t k = 0; k < chunks; ++k) {
        const int q = static_cast<int>(k & 1);
        if (k >= 2) Check(cudaEventSynchronize(ev[q]), "snapshot");  // chunk k-2 has left this buffer
        std::memcpy(pinned[q], host + k * cbytes, static_cast<size_t>(rows(k)) * blk * 4);
        launch(k);
      }
    } else {
      for (size_t k = 0; k < chunks; ++k) {
        launch(k);  // (its buffer's previous chunk, k-2, was copied out last iteration)
        if (k >= 1) {  // chunk k-1 is back in its buffer while chunk k runs
          Check(cudaEventSynchronize(ev[(k - 1) & 1]), "snapshot");
          std::memcpy(host + (k - 1) * cbytes, pinned[(k - 1) & 1], static_cast<size_t>(rows(k - 1)) * blk * 4);
        }
      }
      const size_t k = chunks - 1;
      Check(cudaEventSynchronize(ev[k & 1]), "snapshot");
      std::memcpy(host + k * cbytes, pinned[k & 1], static_cast<size_t>(rows(k)) * blk * 4);
    }
    Check(cudaStreamSynchronize(st), "snapshot rows");
  } catch (...) {
    release();
    throw;
  }
  release();
}

}  // namespace

int gm_engine_snapshot_save(gm_engine* e, void* buf, uint64_t cap, uint64_t* size) {
  return Guard([&]() -> int {
    if (!e || !size) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    Check(cudaDeviceSynchronize(), "snapshot: work in flight");
    const RowTables t = ReadRowTables(e);
    const int32_t full = e->nseg * pre3::kChunksPerSeg;
    std::vector<int32_t> ids;
    for (int32_t i = 0; i < e->cache.C; ++i) {
      if ((t.meta[static_cast<size_t>(i)] & (1 << 16)) && t.built[static_cast<size_t>(i)] == full) ids.push_back(i);
    }
    const size_t n = ids.size(), blk = SnapBlockWords(e);
    const uint64_t payload = n * 16 + n * blk * 4;
    *size = kSnapHeader + payload;
    if (!buf) return GM_OK;
    if (cap < *size) return Fail(GM_ERR_USAGE, "buffer too small");
    uint8_t* out = static_cast<uint8_t*>(buf);
    uint8_t* p = out + kSnapHeader;
    auto put = [&p](const void* src, size_t bytes) {
      if (bytes) std::memcpy(p, src, bytes);
      p += bytes;
    };
    std::vector<int32_t> meta(n), parent(n);
    std::vector<uint32_t> segmask(n);
    std::unordered_set<int32_t> saved(ids.begin(), ids.end());
    for (size_t k = 0; k < n; ++k) {
      const size_t i = static_cast<size_t>(ids[k]);
      meta[k] = t.meta[i];
      parent[k] = saved.count(t.parent[i]) ? t.parent[i] : -1;  // a link only matters while building
      segmask[k] = t.segmask[i];
    }
    put(ids.data(), n * 4);
    put(meta.data(), n * 4);
    put(parent.data(), n * 4);
    put(segmask.data(), n * 4);
    SnapshotRows(e, ids, p, false);
    SnapHeader h{};
    std::memcpy(h.magic, kSnapMagic, 8);
    h.version = kSnapVersion;
    h.header_bytes = kSnapHeader;
    h.grammar_hash = e->grammar_hash;
    h.layout_hash = e->layout_hash;
    h.vocab_hash = e->vocab_hash;
    h.K = e->cache.K;
    h.R = e->cache.R;
    h.C = e->cache.C;
    h.V = e->V;
    h.W = e->W;
    h.nseg = e->nseg;
    h.n = static_cast<int32_t>(n);
    h.max_context = pre3::kMaxContext;
    h.payload_bytes = payload;
    h.checksum = SnapChecksum(out + kSnapHeader, payload);
    std::memcpy(out, &h, sizeof h);
    return GM_OK;
  });
}

int gm_engine_snapshot_load(gm_engine* e, const void* buf, uint64_t bytes) {
  return Guard([&]() -> int {
    if (!e || !buf) return Fail(GM_ERR_USAGE, "null argument");
    if (bytes < kSnapHeader) return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: truncated header");
    SnapHeader h;
    std::memcpy(&h, buf, sizeof h);
    if (std::memcmp(h.magic, kSnapMagic, 8) != 0) return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: bad magic");
    if (h.version != kSnapVersion || h.header_bytes != kSnapHeader) {
      return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: unknown version");
    }
    const uint8_t* in = static_cast<const uint8_t*>(buf);
    if (h.payload_bytes != bytes - kSnapHeader) return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: size mismatch");
    if (SnapChecksum(in + kSnapHeader, h.payload_bytes) != h.checksum) {
      return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: checksum");
    }
    if (h.grammar_hash != e->grammar_hash || h.layout_hash != e->layout_hash) {
      return Fail(GM_ERR_SNAPSHOT_MISMATCH, "snapshot: taken for another automaton");
    }
    if (h.vocab_hash != e->vocab_hash || h.V != e->V || h.W != e->W || h.nseg != e->nseg) {
      return Fail(GM_ERR_SNAPSHOT_MISMATCH, "snapshot: taken for another vocabulary or logit layout");
    }
    if (h.K != e->cache.K || h.R != e->cache.R || h.C != e->cache.C || h.max_context != pre3::kMaxContext) {
      return Fail(GM_ERR_SNAPSHOT_MISMATCH, "snapshot: taken with other context options (K, R, rows)");
    }
    const size_t n = static_cast<size_t>(h.n), blk = SnapBlockWords(e);
    if (h.n < 0 || h.n > h.C || h.payload_bytes != n * 16 + n * blk * 4) {
      return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: row count");
    }
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    Check(cudaDeviceSynchronize(), "snapshot: work in flight");
    unsigned long long ctr[8];
    Check(cudaMemcpy(ctr, e->cache.counters, 64, cudaMemcpyDeviceToHost), "snapshot");
    if (ctr[0] != 0 || ctr[2] != 0) return Fail(GM_ERR_USAGE, "snapshot: the context table is not empty");
    const uint8_t* p = in + kSnapHeader;
    std::vector<int32_t> ids(n), meta(n), parent(n);
    std::vector<uint32_t> segmask(n);
    auto get = [&p](void* dst, size_t b) {
      if (b) std::memcpy(dst, p, b);
      p += b;
    };
    get(ids.data(), n * 4);
    get(meta.data(), n * 4);
    get(parent.data(), n * 4);
    get(segmask.data(), n * 4);
    RowTables t = ReadRowTables(e);
    const int32_t full = e->nseg * pre3::kChunksPerSeg;
    for (size_t k = 0; k < n; ++k) {
      const int32_t i = ids[k];
      if (i < 0 || i >= h.C || (t.meta[static_cast<size_t>(i)] & (1 << 16)) || !(meta[k] & (1 << 16)) ||
          (meta[k] & 0xff) > e->cache.K || parent[k] < -1 || parent[k] >= h.C) {
        return Fail(GM_ERR_CORRUPT_INPUT, "snapshot: bad row record");
      }
      t.meta[static_cast<size_t>(i)] = meta[k];
      t.built[static_cast<size_t>(i)] = full;
      t.parent[static_cast<size_t>(i)] = parent[k];
      t.segmask[static_cast<size_t>(i)] = segmask[k];
    }
    SnapshotRows(e, ids, const_cast<uint8_t*>(p), true);
    const size_t C = static_cast<size_t>(e->cache.C);
    std::vector<int32_t> seg_done(C * static_cast<size_t>(e->nseg), 0);
    for (size_t k = 0; k < n; ++k) {
      std::fill_n(seg_done.begin() + static_cast<ptrdiff_t>(static_cast<size_t>(ids[k]) * e->nseg), e->nseg,
                  pre3::kChunksPerSeg);
    }
    Check(cudaMemcpy(e->cache.seg_done, seg_done.data(), seg_done.size() * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.seg_claim, seg_done.data(), seg_done.size() * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.slot_built, t.built.data(), C * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.slot_parent, t.parent.data(), C * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.cd_segmask, t.segmask.data(), C * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.slot_meta, t.meta.data(), C * 4, cudaMemcpyHostToDevice), "snapshot");
    // Free list: every row not loaded (in id order: pops hand out the lowest first).
    std::vector<int32_t> fr;
    fr.reserve(C - n);
    for (size_t i = C; i-- > 0;) {
      if (!(t.meta[i] & (1 << 16))) fr.push_back(static_cast<int32_t>(i));
    }
    const int32_t nfree = static_cast<int32_t>(fr.size());
    if (!fr.empty()) Check(cudaMemcpy(e->cache.row_free, fr.data(), fr.size() * 4, cudaMemcpyHostToDevice), "snapshot");
    Check(cudaMemcpy(e->cache.row_free_n, &nfree, 4, cudaMemcpyHostToDevice), "snapshot");
    *e->host_free = nfree;
    ctr[0] = n;
    Check(cudaMemcpy(e->cache.counters, ctr, 64, cudaMemcpyHostToDevice), "snapshot");
    Check(pre3::LaunchReindex(e->cache, nullptr), "snapshot reindex");
    // The CI ∩ structural counts follow the engine's current structural set.
    Check(pre3::LaunchRecountStructural(e->cache, e->vocab), "snapshot recount");
    Check(cudaDeviceSynchronize(), "snapshot load");
    return GM_OK;
  });
}

int gm_engine_evict(gm_engine* e, void* stream) {
  return Guard([&]() -> int {
    if (!e) return Fail(GM_ERR_USAGE, "null engine");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    Evict(e, static_cast<cudaStream_t>(stream));
    return GM_OK;
  });
}

int gm_engine_cache_stats(gm_engine* e, int64_t out[8]) {
  return Guard([&]() -> int {
    if (!e || !out) return Fail(GM_ERR_USAGE, "null argument");
    Check(cudaSetDevice(e->device), "cudaSetDevice");
    unsigned long long ctr[8];
    int32_t nfree = 0;
    Check(cudaMemcpy(ctr, e->cache.counters, 64, cudaMemcpyDeviceToHost), "cache stats");
    Check(cudaMemcpy(&nfree, e->cache.row_free_n, 4, cudaMemcpyDeviceToHost), "cache stats");
    out[0] = e->cache.C;
    out[1] = static_cast<int64_t>(ctr[0]);
    out[2] = std::max(nfree, 0);
    out[3] = e->cache.IC;
    out[4] = static_cast<int64_t>(ctr[4]);
    out[5] = static_cast<int64_t>(ctr[5]);
    out[6] = static_cast<int64_t>(ctr[2]);
    out[7] = static_cast<int64_t>(ctr[1]);
    return GM_OK;
  });
}

int gm_engine_prewarm(gm_engine* e, int32_t batch, int32_t steps, uint64_t seed, int32_t stack_capacity,
                      void* stream) {
  return Guard([&]() -> int {
    if (!e || batch < 1 || steps < 0) return Fail(GM_ERR_USAGE, "bad argument");
    gm_batch* b = nullptr;
    int rc = gm_batch_create(e, batch, stack_capacity > 0 ? stack_capacity : 1024, &b);
    if (rc != GM_OK) return rc;
    std::unique_ptr<gm_batch> guard(b);
    for (int32_t s = 0; s < steps; ++s) {
      if ((rc = gm_decode_step_stream(b, nullptr, 0, nullptr, 0, seed, nullptr, stream)) != GM_OK) return rc;
    }
    return gm_batch_check(b, stream);
  });
}

}  // extern "C"
