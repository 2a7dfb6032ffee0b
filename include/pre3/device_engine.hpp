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

 private:
  gm_automaton* automaton_ = nullptr;
  gm_engine* engine_ = nullptr;
  gm_batch* one_ = nullptr;
  int32_t num_tokens_ = 0;
};

}  // namespace pre3
