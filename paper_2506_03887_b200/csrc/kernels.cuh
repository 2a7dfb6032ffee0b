// kernels.cuh — device views and kernel launchers (sm_100a).
// §3 (HBM layout) and §4 (kernels).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gm_internal.hpp"

namespace pre3 {

constexpr int kThreads = 256;      // fill CTA size (8 warps)
constexpr int kSegWords = 256;     // mask words per vocab segment (8192 tokens)
constexpr int kMaxContext = 16;    // max K
constexpr int kWalkOverlay = 64;   // per-thread pushed-entry overlay in a mask walk

// Per-sequence device state: {depth, status, draws, reserved}.
struct SeqState {
  int32_t depth;
  int32_t status;
  uint32_t draws;
  int32_t reserved;
};

struct AutView {
  const DevEdge* edges;
  const int32_t* cond;
  const int32_t* push;
  const int32_t* cand_begin;  // S*257+1
  const int32_t* cand;
  const int32_t* shift;  // S*256
  int32_t num_states;
  int32_t initial;
};

struct VocabView {
  const int32_t* tok_off;  // V+1 byte offsets
  const uint8_t* tok_bytes;
  const uint32_t* structural;  // W words
  int32_t V;                   // regular tokens; EOS = V
  int32_t W;                   // ceil((V+1)/32)
  int32_t nseg;                // ceil(W / kSegWords)
};

// Context cache: key = (n = min(depth, K), complete = depth <= K, top-n
// stack entries top first) -> per segment {CI bitset words, CD token list}.
struct CacheView {
  unsigned long long* slot_hash;  // C; 0 = empty
  int32_t* slot_meta;             // C; n | complete << 8 | ready << 16
  int32_t* slot_keys;             // C*K
  uint32_t* seg_state;            // C*nseg; 0 empty, 1 building, 2 ready, 3 failed
  uint32_t* ci;                   // C*W context-independent accept bits
  int32_t* cd_off;                // C*nseg
  int32_t* cd_len;                // C*nseg
  int32_t* cd_pool;
  unsigned long long* pool_top;
  long long pool_cap;
  unsigned long long* counters;  // [0] slots, [1] builds, [2] direct, [3] cd resolved
  int32_t C;
  int32_t K;
};

struct BatchView {
  SeqState* seq;
  int32_t* stacks;  // B*cap, bottom first
  int32_t cap;
  int32_t B;
  unsigned int* err;                  // bit0: walk overlay overflow
  unsigned long long* stats;          // [0] rd bytes, [1] wr bytes, [2] hits, [3] builds, [4] direct, [5] cd
  unsigned long long* counters;       // [0] restarts, [1] draws, [2] fills, [3] accepts
  int32_t stats_enabled;
};

enum FillMode { kFillMask = 0, kFillGreedy = 1 };
enum SampleMode { kSampleGiven = 0, kSampleStream = 1, kSampleGreedy = 2 };

cudaError_t LaunchReset(const AutView& a, const BatchView& b, cudaStream_t s);
cudaError_t LaunchFill(int mode, const AutView& a, const VocabView& v, const CacheView& c,
                       const BatchView& b, uint32_t* bitmask, long long ldw, uint16_t* logits,
                       long long ld, int32_t* seg_counts, unsigned long long* best,
                       cudaStream_t s);
cudaError_t LaunchAccept(int sample, const AutView& a, const VocabView& v, const BatchView& b,
                         const int32_t* tokens, int32_t* status_out, int restart,
                         const uint32_t* bitmask, long long ldw, const int32_t* seg_counts,
                         unsigned long long seed, unsigned long long* best, int32_t* tokens_out,
                         int do_accept, cudaStream_t s);

}  // namespace pre3
