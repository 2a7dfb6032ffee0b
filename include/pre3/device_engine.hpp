// include/pre3/device_engine.hpp — header-only C++ wrapper over the C ABI
// (include/pre3_gmask.h) that mirrors the reference runtime's class surface,
// `gmask::Engine` (/root/reference/proj/include/gmask/runtime.hpp:92-166), so a
// reference caller (tools/gmask_main.cpp DoMask/DoBench, test rigs) can switch
// to the device path with the same method names and error behaviour:
// failures throw `pre3::DeviceError` carrying the gm_status_code that maps to
// the reference's GrammarError / BuildError / SerializeError / VocabError.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pre3_gmask.h"

// The single-sequence calls below (ComputeMask, AllowedTerminals,
// AcceptToken) move one configuration through device memory; they are
// available when the CUDA runtime headers are on the include path.
#if __has_include(<cuda_runtime.h>)
#include <cuda_runtime.h>
#define PRE3_DEVICE_ENGINE_SINGLE 1
#endif

namespace pre3 {

class DeviceError : public std::runtime_error {
 public:
  DeviceError(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

inline void Check(int rc) {
  if (rc != GM_OK) throw DeviceError(rc, gm_last_error());
}

// RuntimeConfig (runtime.hpp:23-27): stack bottom first.
struct RuntimeConfig {
  int32_t state = 0;
  int32_t status = GM_ALIVE;
  std::vector<int32_t> stack;
};

class DeviceEngine {
 public:
  // Engine(Dpda) + TokenTrie::Build(vocab) on `device`.
  DeviceEngine(const std::vector<uint8_t>& p3dpda, const std::vector<std::string>& vocab, int device = 0,
               const gm_engine_options* opts = nullptr) {
    Check(gm_automaton_load(p3dpda.data(), p3dpda.size(), &automaton_));
    std::vector<uint8_t> bytes;
    std::vector<int64_t> offs{0};
    for (const auto& t : vocab) {
      bytes.insert(bytes.end(), t.begin(), t.end());
      offs.push_back(static_cast<int64_t>(bytes.size()));
    }
    if (bytes.empty()) bytes.push_back(0);
    Check(gm_engine_create(automaton_, bytes.data(), offs.data(), static_cast<int32_t>(vocab.size()), opts, device,
                           &engine_));
    num_tokens_ = static_cast<int32_t>(vocab.size());
  }
  ~DeviceEngine() {
#ifdef PRE3_DEVICE_ENGINE_SINGLE
    if (dev_words_) cudaFree(dev_words_);
#endif
    if (one_) gm_batch_destroy(one_);
    if (engine_) gm_engine_destroy(engine_);
    if (automaton_) gm_automaton_destroy(automaton_);
  }
  DeviceEngine(const DeviceEngine&) = delete;
  DeviceEngine& operator=(const DeviceEngine&) = delete;

  gm_engine* handle() const { return engine_; }
  int32_t num_tokens() const { return num_tokens_; }
  int32_t mask_words() const { return (num_tokens_ + 1 + 31) / 32; }

  // Engine::InitialConfig (runtime.cpp:115-121).
  RuntimeConfig InitialConfig() const {
    int64_t info[8];
    Check(gm_automaton_info(automaton_, info));
    RuntimeConfig c;
    c.state = static_cast<int32_t>(info[2]);
    c.stack = {c.state};
    return c;
  }

  // A batch of B sequences on the device: the batched hot path.
  gm_batch* NewBatch(int32_t batch, int32_t stack_capacity = 1024) const {
    gm_batch* b = nullptr;
    Check(gm_batch_create(engine_, batch, stack_capacity, &b));
    return b;
  }

  // Context cache (no reference counterpart: the reference recomputes every
  // mask).  Prewarm populates it with synthetic decode steps; a snapshot
  // ("P3GMCTX1") of the built table loads into a fresh engine of the same
  // automaton / vocabulary / options instead (gm_engine_snapshot_*).
  void Prewarm(int32_t batch, int32_t steps, uint64_t seed) const {
    Check(gm_engine_prewarm(engine_, batch, steps, seed, 0, nullptr));
  }
  std::vector<uint8_t> SaveContexts() const {
    uint64_t n = 0;
    Check(gm_engine_snapshot_save(engine_, nullptr, 0, &n));
    std::vector<uint8_t> buf(static_cast<size_t>(n));
    Check(gm_engine_snapshot_save(engine_, buf.data(), n, &n));
    buf.resize(static_cast<size_t>(n));
    return buf;
  }
  void LoadContexts(const std::vector<uint8_t>& snapshot) const {
    Check(gm_engine_snapshot_load(engine_, snapshot.data(), snapshot.size()));
  }
  int64_t ContextsUsed() const {
    int64_t info[8];
    Check(gm_engine_info(engine_, info));
    return info[3];
  }

#ifdef PRE3_DEVICE_ENGINE_SINGLE
  // Engine::ComputeMask (runtime.cpp:280-287) for one configuration: V+1
  // bits in 32-bit words (bit t of word t/32; bit V = EOS), the reference's
  // TokenMask layout.  Runs the CUDA fill on a batch of one.
  std::vector<uint32_t> ComputeMask(const RuntimeConfig& cfg) {
    Load(cfg);
    const int32_t W = mask_words();
    Check(gm_fill_next_token_bitmask(one_, dev_words_, W, nullptr));
    Check(gm_batch_check(one_, nullptr));
    std::vector<uint32_t> out(static_cast<size_t>(W));
    CudaCheck(cudaMemcpy(out.data(), dev_words_, out.size() * 4, cudaMemcpyDeviceToHost));
    return out;
  }

  // Engine::AllowedTerminals (runtime.cpp:188-208): the 256-bit next-byte set
  // (4 x u64) and the end-marker flag.
  std::pair<std::vector<uint64_t>, bool> AllowedTerminals(const RuntimeConfig& cfg) {
    Load(cfg);
    Check(gm_allowed_terminals(one_, dev_words_, nullptr));
    uint32_t w[9];
    CudaCheck(cudaMemcpy(w, dev_words_, sizeof(w), cudaMemcpyDeviceToHost));
    std::vector<uint64_t> set(4);
    for (int i = 0; i < 4; ++i) set[i] = static_cast<uint64_t>(w[2 * i]) | (static_cast<uint64_t>(w[2 * i + 1]) << 32);
    return {set, (w[8] & 1u) != 0};
  }

  // Engine::Step over every byte of `token` (EOS = id V), like the
  // reference callers' loop (tools/gmask_main.cpp:113-118); returns the new
  // configuration (status Dead when a byte has no edge).
  RuntimeConfig AcceptToken(const RuntimeConfig& cfg, int32_t token) {
    Load(cfg);
    CudaCheck(cudaMemcpy(dev_words_, &token, 4, cudaMemcpyHostToDevice));
    Check(gm_accept_tokens(one_, reinterpret_cast<const int32_t*>(dev_words_), nullptr, 0, nullptr));
    Check(gm_batch_check(one_, nullptr));
    RuntimeConfig out;
    out.stack.resize(static_cast<size_t>(capacity_));
    int32_t depth = 0;
    Check(gm_batch_download(one_, 0, &out.state, &out.status, out.stack.data(), capacity_, &depth));
    out.stack.resize(static_cast<size_t>(depth));
    return out;
  }
#endif

 private:
#ifdef PRE3_DEVICE_ENGINE_SINGLE
  static void CudaCheck(cudaError_t e) {
    if (e != cudaSuccess) throw DeviceError(GM_ERR_CUDA, cudaGetErrorString(e));
  }
  // Batch of one holding `cfg`, and a device scratch of max(W, 9) words.
  void Load(const RuntimeConfig& cfg) {
    if (!one_) {
      Check(gm_batch_create(engine_, 1, capacity_, &one_));
      const size_t words = static_cast<size_t>(mask_words() > 9 ? mask_words() : 9);
      CudaCheck(cudaMalloc(reinterpret_cast<void**>(&dev_words_), words * 4));
    }
    Check(gm_batch_upload(one_, 0, cfg.status, cfg.stack.data(), static_cast<int32_t>(cfg.stack.size())));
  }
  uint32_t* dev_words_ = nullptr;
  int32_t capacity_ = 1024;
#endif

  gm_automaton* automaton_ = nullptr;
  gm_engine* engine_ = nullptr;
  gm_batch* one_ = nullptr;
  int32_t num_tokens_ = 0;
};

}  // namespace pre3
