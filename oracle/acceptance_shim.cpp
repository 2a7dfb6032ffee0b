// oracle/acceptance_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped).
//
// Compiles the reference's acceptance gate UNMODIFIED from where it lies
// (/root/reference/proj/tests/acceptance/acceptance_main.cpp, included below
// with its `main` renamed) so that oracle/make_golden.py can call the
// reference's own workload helpers:
//   * WriteBenchVocab  (acceptance_main.cpp:341-359) — pins the product's
//     synthetic vocabulary generator byte for byte;
//   * SampleVocab / SampleConfigs / MakePipeline (acceptance_main.cpp:63-115)
//     with the seeds of MaskAgreement (acceptance_main.cpp:202-219) — the
//     reference-scale mask-agreement goldens (6 fixtures x 200 configurations
//     x 1,000-token vocabularies).
// Built only where /root/reference exists (oracle/Makefile target `acc`).
#define main gmask_acceptance_main_unused
#include "acceptance/acceptance_main.cpp"
#undef main

#include <cstring>

namespace {

void PutString(const std::string& s, char* out, int64_t cap, int64_t* n) {
  *n = static_cast<int64_t>(s.size());
  if (out != nullptr && cap >= *n) std::memcpy(out, s.data(), s.size());
}

}  // namespace

extern "C" {

// WriteBenchVocab into `path` (the reference writes a JSON array).
int acc_write_bench_vocab(const char* path) {
  try {
    WriteBenchVocab(fs::path(path));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// MaskAgreement's inputs for one fixture: the 1,000-token vocabulary as a
// JSON array of hex strings and the 200 sampled configurations as
// "status depth s0 s1 ...\n" lines, in the reference's own order and seeds.
int acc_mask_agreement_inputs(const char* fixture, char* vocab_out, int64_t vocab_cap, int64_t* vocab_n,
                              char* cfg_out, int64_t cfg_cap, int64_t* cfg_n) {
  try {
    Pipeline p = MakePipeline(fixture, BuildOptions{});
    std::mt19937_64 rng(0xba5e + std::hash<std::string>{}(fixture));
    std::vector<std::string> vocab = SampleVocab(p.grammar, 1000, &rng);
    std::string vs = "[";
    static const char* hex = "0123456789abcdef";
    for (size_t i = 0; i < vocab.size(); ++i) {
      vs += i ? ",\"" : "\"";
      for (unsigned char c : vocab[i]) {
        vs.push_back(hex[c >> 4]);
        vs.push_back(hex[c & 15]);
      }
      vs += "\"";
    }
    vs += "]";
    std::string cs;
    for (const RuntimeConfig& cfg : SampleConfigs(p.engine, 200, 40, &rng)) {
      cs += std::to_string(static_cast<int>(cfg.status)) + " " + std::to_string(cfg.stack.size());
      for (int32_t s : cfg.stack) cs += " " + std::to_string(s);
      cs += "\n";
    }
    PutString(vs, vocab_out, vocab_cap, vocab_n);
    PutString(cs, cfg_out, cfg_cap, cfg_n);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
