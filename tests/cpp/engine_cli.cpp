// Test driver (tests/test_gpu_parity.py::test_cpp_device_engine_known_answers):
// the reference-side C++ binding include/pre3/device_engine.hpp used the way
// the reference's own test rig uses gmask::Engine (test_runtime.cpp:24-61):
// argv[1] = a P3DPDA file, argv[2..] = the vocabulary; each stdin line is a
// list of token ids accepted from InitialConfig(); for each line it prints
// the ComputeMask words (hex), the end-marker flag of AllowedTerminals and
// the stack.  With PRE3_CLI_SNAPSHOT set it then prewarms the context cache,
// saves it, loads it into a second engine, recomputes every line's mask on
// that engine and prints "snapshot ok <contexts>" when all are identical.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include "pre3/device_engine.hpp"

int main(int argc, char** argv) {
  if (argc < 3) return 64;
  std::ifstream f(argv[1], std::ios::binary);
  std::vector<uint8_t> flat((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<std::string> vocab(argv + 2, argv + argc);
  try {
    pre3::DeviceEngine eng(flat, vocab, 0);
    std::string line;
    std::vector<pre3::RuntimeConfig> cfgs;
    std::vector<std::vector<uint32_t>> masks;
    while (std::getline(std::cin, line)) {
      std::istringstream in(line);
      pre3::RuntimeConfig cfg = eng.InitialConfig();
      int32_t tok;
      while (in >> tok) cfg = eng.AcceptToken(cfg, tok);
      const std::vector<uint32_t> m = eng.ComputeMask(cfg);
      cfgs.push_back(cfg);
      masks.push_back(m);
      const auto allowed = eng.AllowedTerminals(cfg);
      std::printf("mask");
      for (uint32_t w : m) std::printf(" %08x", w);
      std::printf(" eos %d status %d stack", allowed.second ? 1 : 0, cfg.status);
      for (int32_t s : cfg.stack) std::printf(" %d", s);
      std::printf("\n");
    }
    if (std::getenv("PRE3_CLI_SNAPSHOT")) {
      eng.Prewarm(64, 50, 7);
      const std::vector<uint8_t> snap = eng.SaveContexts();
      pre3::DeviceEngine eng2(flat, vocab, 0);
      eng2.LoadContexts(snap);
      bool same = eng2.ContextsUsed() == eng.ContextsUsed();
      for (size_t i = 0; i < cfgs.size(); ++i) same = same && eng2.ComputeMask(cfgs[i]) == masks[i];
      std::printf(same ? "snapshot ok %lld\n" : "snapshot MISMATCH %lld\n", static_cast<long long>(eng2.ContextsUsed()));
    }
  } catch (const pre3::DeviceError& e) {
    std::fprintf(stderr, "DeviceError %d: %s\n", e.code(), e.what());
    return 1;
  }
  return 0;
}
