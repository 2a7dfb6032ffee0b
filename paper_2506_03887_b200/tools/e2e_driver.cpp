// e2e_driver.cpp — a C++ caller of the C ABI (include/pre3_gmask.h) that runs
// the end-to-end decode loop bench.py reports as `e2e`: host-held token ids
// in, host-visible results out, every step.  It is what a serving loop
// written in the reference's language looks like (one host thread, plain
// CUDA runtime calls) and keeps Python's per-call overhead out of the
// measurement.  Not part of the product library: it only uses the public ABI.
//
// Per step, on the batch's stream:
//   H2D   last step's token ids (pinned host buffer)       [stream mode]
//   gm_accept_tokens(restart = 1)                          [stream mode]
//   gm_fill_and_mask_logits  /  gm_decode_step_greedy
//   gm_sample_stream                                       [stream mode]
//   D2H   the sampled ids (pinned), then wait for them — the next step needs them
// and on a copy stream: D2H of the step's full bitmask into double-buffered
// pinned memory (overlapping the next step's kernels).  The timed region ends
// when the last bitmask copy has landed.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <vector>

#include "pre3_gmask.h"

namespace {

struct Bufs {
  int32_t* tok_host = nullptr;
  int32_t* picked_host = nullptr;
  uint32_t* bm_host[2] = {nullptr, nullptr};
  int32_t* tok_dev = nullptr;
  int32_t* picked_map = nullptr;  // device alias of picked_host (mapped)
  uint32_t* bm_dev[2] = {nullptr, nullptr};
  int32_t* counts = nullptr;
  cudaStream_t s = nullptr, cs = nullptr;
  cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};

  ~Bufs() {
    cudaFreeHost(tok_host);
    cudaFreeHost(picked_host);
    for (int i = 0; i < 2; ++i) {
      cudaFreeHost(bm_host[i]);
      cudaFree(bm_dev[i]);
      if (ready[i]) cudaEventDestroy(ready[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
    cudaFree(tok_dev);
    cudaFree(counts);
    if (s) cudaStreamDestroy(s);
    if (cs) cudaStreamDestroy(cs);
  }
};

#define CK(x)                         \
  do {                                \
    if ((x) != cudaSuccess) return 5; \
  } while (0)
#define GK(x)                 \
  do {                        \
    const int rc_ = (x);      \
    if (rc_ != GM_OK) return rc_; \
  } while (0)

}  // namespace

extern "C" {

// mode 0: stream sampler (host-held ids, accept via gm_accept_tokens);
// mode 1: greedy one-launch step (device logits in, ids + bitmask out).
// logits: R device pointers to bf16 [B][ld] rows, rotated per step.
// *seconds: host wall time of the `steps` timed steps (after `warmup`).
// copy_mask = 0 skips the bitmask D2H (the deployment where the mask is only
// consumed on the device, by the fused logits masking).
int e2e_run(gm_batch* b, int32_t mode, int32_t B, int32_t W, int32_t nseg, const uint64_t* logits, int32_t R,
            int64_t ld, uint64_t seed, int32_t warmup, int32_t steps, int32_t device, int32_t copy_mask,
            double* seconds) {
  CK(cudaSetDevice(device));
  Bufs m;
  const size_t mask_bytes = static_cast<size_t>(B) * static_cast<size_t>(W) * 4;
  CK(cudaHostAlloc(&m.tok_host, B * 4, cudaHostAllocDefault));
  // The sampled ids come back zero-copy: the kernel stores them straight
  // into mapped pinned memory, so the small read-back never queues behind the
  // 16 KB/sequence bitmask copy on the device-to-host copy engine.
  CK(cudaHostAlloc(&m.picked_host, B * 4, cudaHostAllocMapped));
  CK(cudaMalloc(&m.tok_dev, B * 4));
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&m.picked_map), m.picked_host, 0));
  CK(cudaMalloc(&m.counts, static_cast<size_t>(B) * nseg * 2 * 4));
  for (int i = 0; i < 2; ++i) {
    CK(cudaHostAlloc(&m.bm_host[i], mask_bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&m.bm_dev[i], mask_bytes));
    CK(cudaEventCreateWithFlags(&m.ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m.done[i], cudaEventDisableTiming));
  }
  CK(cudaStreamCreateWithFlags(&m.s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&m.cs, cudaStreamNonBlocking));
  for (int i = 0; i < B; ++i) m.tok_host[i] = -1;
  for (int i = 0; i < 2; ++i) CK(cudaEventRecord(m.done[i], m.cs));

  auto step = [&](int i) -> int {
    const int j = i & 1;
    uint16_t* lg = reinterpret_cast<uint16_t*>(logits[i % R]);
    CK(cudaStreamWaitEvent(m.s, m.done[j], 0));  // bitmask buffer j copied out
    if (mode == 0) {
      CK(cudaMemcpyAsync(m.tok_dev, m.tok_host, B * 4, cudaMemcpyHostToDevice, m.s));
      GK(gm_accept_tokens(b, m.tok_dev, nullptr, 1, m.s));
      GK(gm_fill_and_mask_logits(b, m.bm_dev[j], W, lg, ld, m.counts, m.s));
      CK(cudaEventRecord(m.ready[j], m.s));
      GK(gm_sample_stream(b, m.bm_dev[j], W, m.counts, seed, m.picked_map, m.s));
    } else {
      GK(gm_decode_step_greedy(b, lg, ld, m.bm_dev[j], W, m.picked_map, m.s));
      CK(cudaEventRecord(m.ready[j], m.s));
    }
    if (copy_mask) {
      CK(cudaStreamWaitEvent(m.cs, m.ready[j], 0));
      CK(cudaMemcpyAsync(m.bm_host[j], m.bm_dev[j], mask_bytes, cudaMemcpyDeviceToHost, m.cs));
      CK(cudaEventRecord(m.done[j], m.cs));
    }
    CK(cudaStreamSynchronize(m.s));
    if (mode == 0) {
      for (int k = 0; k < B; ++k) m.tok_host[k] = m.picked_host[k];
    }
    return 0;
  };
  for (int i = 0; i < warmup; ++i) {
    const int rc = step(i);
    if (rc) return rc;
  }
  CK(cudaStreamSynchronize(m.cs));
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) {
    const int rc = step(warmup + i);
    if (rc) return rc;
  }
  CK(cudaStreamSynchronize(m.cs));
  const auto t1 = std::chrono::steady_clock::now();
  *seconds = std::chrono::duration<double>(t1 - t0).count();
  return gm_batch_check(b, m.s);
}

}  // extern "C"
