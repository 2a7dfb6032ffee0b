// kernels.cu — sm_100a kernels of the constrained-decoding hot path.
//
//   fill_kernel    Engine::ComputeMask (runtime.cpp:261-287) for a batch,
//                  one CTA per (vocab segment, sequence), fused with in-place
//                  bf16 -inf logit masking (or greedy argmax).  The mask is
//                  assembled from the context cache (CI bits streamed from
//                  HBM/L2 + CD tokens resolved against the sequence's real
//                  stack); cache misses build the entry in the same launch.
//   accept_kernel  Engine::Step over a token's bytes (runtime.cpp:177-186),
//                  one warp per sequence, lanes testing candidate edges in
//                  arbitration order (FindEdge, runtime.cpp:138-146) with
//                  __ballot_sync; optional fused stream/greedy sampling.
//
// Integer/bit work only: no tensor cores (nothing here is a contraction).
#include <cuda/atomic>

#include "kernels.cuh"

namespace pre3 {
namespace {

enum : int { kReject = 0, kAccept = 1, kUnknown = 2, kOverflow = 3 };
enum : int { kNoMatch = 0, kMatch = 1, kCondUnknown = 2 };
enum : int { kAlive = 0, kDead = 1, kAccepted = 2, kStackOverflow = 3 };
enum : uint32_t { kSegEmpty = 0, kSegBuilding = 1, kSegReady = 2, kSegFailed = 3 };

using atomic_u64 = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
using atomic_u32 = cuda::atomic_ref<uint32_t, cuda::thread_scope_device>;
using atomic_i32 = cuda::atomic_ref<int32_t, cuda::thread_scope_device>;

__device__ __forceinline__ unsigned long long Mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ---------------------------------------------------------------------------
// One token walk (the body of ComputeMaskNaive's per-token replay,
// runtime.cpp:289-307, and of the trie walk's FindEdge/Apply chain) against a
// stack given as `base[0..nb)` bottom first plus a private overlay of pushed
// entries.  With complete == false the base is only the top of an unknown
// deeper stack: any condition that reaches below it (after matching every
// known entry) makes the outcome kUnknown — a context-dependent token.
// Arbitration is first match in stored order (dpda_builder.cpp:327-338), so an
// unknown earlier candidate also makes the outcome unknown.
// ---------------------------------------------------------------------------
__device__ int WalkToken(const AutView& A, const VocabView& Vv, int32_t t, const int32_t* base,
                         int nb, bool complete) {
  int32_t loc[kWalkOverlay];
  int nl = 0;
  const bool eos = t == Vv.V;
  const int nterm = eos ? 1 : (__ldg(Vv.tok_off + t + 1) - __ldg(Vv.tok_off + t));
  const uint8_t* bytes = eos ? nullptr : Vv.tok_bytes + __ldg(Vv.tok_off + t);
  int state = base[nb - 1];
  for (int i = 0; i < nterm; ++i) {
    const int x = eos ? 256 : static_cast<int>(__ldg(bytes + i));
    const int cb = __ldg(A.cand_begin + state * 257 + x);
    const int ce = __ldg(A.cand_begin + state * 257 + x + 1);
    int found = -1;
    DevEdge fe;
    for (int c = cb; c < ce; ++c) {
      const int e = __ldg(A.cand + c);
      const int4 raw = __ldg(reinterpret_cast<const int4*>(A.edges) + e);
      DevEdge ed;
      ed.cond_off = raw.x;
      ed.push_off = raw.y;
      ed.cond_len = static_cast<int16_t>(raw.z & 0xffff);
      ed.push_len = static_cast<int16_t>(raw.z >> 16);
      ed.flags = raw.w;
      const int32_t* cond = A.cond + ed.cond_off;
      int r = kMatch;
      for (int j = 0; j < ed.cond_len; ++j) {
        int v;
        if (j < nl) {
          v = loc[nl - 1 - j];
        } else if (j - nl < nb) {
          v = base[nb - 1 - (j - nl)];
        } else {
          r = complete ? kNoMatch : kCondUnknown;
          break;
        }
        if (v != __ldg(cond + j)) {
          r = kNoMatch;
          break;
        }
      }
      if (r == kCondUnknown) return kUnknown;
      if (r == kMatch) {
        found = e;
        fe = ed;
        break;
      }
    }
    if (found < 0) return kReject;
    if (i == nterm - 1) return kAccept;  // the last Step succeeded
    // Apply (runtime.cpp:148-168) on the overlay.
    const int k = fe.cond_len;
    if (k <= nl) {
      nl -= k;
    } else {
      nb -= k - nl;
      nl = 0;
    }
    if (nl + fe.push_len + 1 > kWalkOverlay) return kOverflow;
    for (int j = 0; j < fe.push_len; ++j) loc[nl++] = __ldg(A.push + fe.push_off + j);
    int top = nl > 0 ? loc[nl - 1] : (nb > 0 ? base[nb - 1] : -1);
    if (top < 0) return complete ? kReject : kUnknown;
    if (fe.flags & 1) {
      top = __ldg(A.shift + top * 256 + x);
      if (top < 0) return kReject;  // unreachable for validated automata
      loc[nl++] = top;
    }
    state = top;
  }
  return kAccept;
}

__device__ __forceinline__ int WarpSum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim == kThreads).
__device__ int BlockExclusiveScan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kThreads / 32 ? scratch[lane] : 0;
    int winc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += y;
    }
    if (lane < kThreads / 32) scratch[lane] = winc - w;
    if (lane == kThreads / 32 - 1) scratch[kThreads / 32] = winc;
  }
  __syncthreads();
  int out = scratch[warp] + inc - v;
  *total = scratch[kThreads / 32];
  __syncthreads();
  return out;
}

__device__ unsigned long long KeyHash(const int32_t* key, int n, int complete) {
  unsigned long long h = Mix64(0x5ca1ab1eull ^ static_cast<unsigned long long>(n | (complete << 8)));
  for (int i = 0; i < n; ++i) h = Mix64(h ^ static_cast<uint32_t>(key[i]));
  return h | 1ull;
}

// Finds or inserts the cache slot of a key (thread-0 only).  Returns the slot
// or -1 (table full / key being inserted by another CTA right now).
__device__ int LookupSlot(const CacheView& C, const int32_t* key, int n, int complete) {
  const unsigned long long h = KeyHash(key, n, complete);
  const int meta_want = n | (complete << 8);
  for (int p = 0; p < 64; ++p) {
    const int i = static_cast<int>((h + static_cast<unsigned long long>(p)) & static_cast<unsigned long long>(C.C - 1));
    atomic_u64 slot(C.slot_hash[i]);
    unsigned long long cur = slot.load(cuda::memory_order_relaxed);
    if (cur == 0) {
      unsigned long long expect = 0;
      if (slot.compare_exchange_strong(expect, h, cuda::memory_order_relaxed)) {
        for (int j = 0; j < n; ++j) C.slot_keys[i * C.K + j] = key[j];
        atomic_i32 meta(C.slot_meta[i]);
        meta.store(meta_want | (1 << 16), cuda::memory_order_release);
        atomicAdd(C.counters + 0, 1ull);
        return i;
      }
      cur = expect;
    }
    if (cur != h) continue;
    atomic_i32 meta(C.slot_meta[i]);
    const int m = meta.load(cuda::memory_order_acquire);
    if (!(m & (1 << 16))) return -1;  // being published; compute directly
    if ((m & 0xffff) != meta_want) continue;
    bool same = true;
    for (int j = 0; j < n && same; ++j) same = __ldcg(C.slot_keys + i * C.K + j) == key[j];
    if (same) return i;
  }
  return -1;
}

struct FillShared {
  uint32_t mask[kSegWords];
  uint32_t cd[kSegWords];
  int32_t key[kMaxContext];
  int32_t base[kMaxContext];
  int scratch[kThreads / 32 + 1];
  unsigned long long best[kThreads / 32];
  int status, depth, slot, mode, cd_off, cd_len, fail;
};

}  // namespace

// ---------------------------------------------------------------------------
// fill_kernel: grid (nseg, B), block kThreads.  Dynamic smem = stack copy.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) FillKernel(AutView A, VocabView Vv, CacheView Cc,
                                                       BatchView Bt, uint32_t* __restrict__ bitmask,
                                                       long long ldw, uint16_t* __restrict__ logits,
                                                       long long ld, int32_t* __restrict__ seg_counts,
                                                       unsigned long long* __restrict__ best,
                                                       int vec_ok) {
  __shared__ FillShared sh;
  extern __shared__ int32_t stack_s[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = blockIdx.x, b = blockIdx.y;
  const int w0 = seg * kSegWords;
  const int nwords = min(Vv.W - w0, kSegWords);
  const int t0 = w0 * 32;
  const int t1 = min(Vv.V + 1, t0 + nwords * 32);
  const int32_t* gstack = Bt.stacks + static_cast<long long>(b) * Bt.cap;

  if (tid == 0) {
    SeqState st = Bt.seq[b];
    sh.status = st.status;
    sh.depth = st.depth;
    sh.mode = 0;
    sh.fail = 0;
    sh.cd_len = 0;
  }
  __syncthreads();
  const int depth = sh.depth;
  const bool alive = sh.status == kAlive;
  const int K = Cc.K;
  const int n = min(depth, K);
  const bool complete = depth <= K;
  bool stack_loaded = false;
  auto load_stack = [&]() {
    if (stack_loaded) return;
    for (int i = tid; i < depth; i += kThreads) stack_s[i] = gstack[i];
    __syncthreads();
    stack_loaded = true;
  };
  unsigned long long st_hit = 0, st_build = 0, st_direct = 0, st_cd = 0;

  if (!alive) {
    for (int w = tid; w < nwords; w += kThreads) sh.mask[w] = 0u;
  } else {
    if (tid < n) {
      const int32_t v = gstack[depth - 1 - tid];
      sh.key[tid] = v;              // top first
      sh.base[n - 1 - tid] = v;     // bottom first
    }
    __syncthreads();
    if (tid == 0) {
      int slot = LookupSlot(Cc, sh.key, n, complete ? 1 : 0);
      int mode = 2;  // direct
      if (slot >= 0) {
        atomic_u32 ss(Cc.seg_state[static_cast<long long>(slot) * Vv.nseg + seg]);
        uint32_t s = ss.load(cuda::memory_order_acquire);
        if (s == kSegReady) {
          mode = 0;
          sh.cd_off = Cc.cd_off[static_cast<long long>(slot) * Vv.nseg + seg];
          sh.cd_len = Cc.cd_len[static_cast<long long>(slot) * Vv.nseg + seg];
        } else if (s == kSegEmpty) {
          uint32_t expect = kSegEmpty;
          if (ss.compare_exchange_strong(expect, kSegBuilding, cuda::memory_order_relaxed)) mode = 1;
        }
      }
      sh.slot = slot;
      sh.mode = mode;
    }
    __syncthreads();
    const int mode = sh.mode;
    const int slot = sh.slot;

    if (mode == 0) {
      // ---- hit: CI bits + resolve CD tokens against the real stack.
      const uint32_t* ci = Cc.ci + static_cast<long long>(slot) * Vv.W + w0;
      for (int w = tid; w < nwords; w += kThreads) sh.mask[w] = __ldcg(ci + w);
      const int cd_len = sh.cd_len;
      __syncthreads();  // CI words in place before CD bits are OR-ed in
      if (cd_len > 0) {
        load_stack();
        const int32_t* pool = Cc.cd_pool + sh.cd_off;
        for (int i = tid; i < cd_len; i += kThreads) {
          const int t = __ldcg(pool + i);
          const int r = WalkToken(A, Vv, t, stack_s, depth, true);
          if (r == kAccept) atomicOr(&sh.mask[(t - t0) >> 5], 1u << ((t - t0) & 31));
          if (r == kOverflow) atomicOr(Bt.err, 1u);
        }
      }
      st_hit = 1;
      st_cd = static_cast<unsigned long long>(cd_len);
    } else {
      // ---- build (mode 1) or direct (mode 2): walk every token of the segment.
      load_stack();
      const int ntok_r = nwords * 32;
      for (int base_t = 0; base_t < ntok_r; base_t += kThreads) {
        const int t = t0 + base_t + tid;
        int r = kReject;
        if (t < t1) {
          r = mode == 1 ? WalkToken(A, Vv, t, sh.base, n, complete)
                        : WalkToken(A, Vv, t, stack_s, depth, true);
        }
        const unsigned acc = __ballot_sync(0xffffffffu, r == kAccept);
        const unsigned cd = __ballot_sync(0xffffffffu, r == kUnknown);
        if (__any_sync(0xffffffffu, r == kOverflow) && lane == 0) atomicOr(Bt.err, 1u);
        if (lane == 0) {
          sh.mask[(base_t >> 5) + warp] = acc;
          sh.cd[(base_t >> 5) + warp] = cd;
        }
      }
      __syncthreads();
      if (mode == 1) {
        // Publish CI bits, then the CD list (prefix-summed word popcounts).
        uint32_t* ci = Cc.ci + static_cast<long long>(slot) * Vv.W + w0;
        for (int w = tid; w < nwords; w += kThreads) ci[w] = sh.mask[w];
        const int c = tid < nwords ? __popc(sh.cd[tid]) : 0;
        int total = 0;
        const int excl = BlockExclusiveScan(c, sh.scratch, &total);
        if (tid == 0) {
          unsigned long long off = atomicAdd(Cc.pool_top, static_cast<unsigned long long>(total));
          if (static_cast<long long>(off + total) > Cc.pool_cap) {
            sh.fail = 1;
          } else {
            sh.cd_off = static_cast<int>(off);
            sh.cd_len = total;
          }
        }
        __syncthreads();
        if (!sh.fail && tid < nwords) {
          uint32_t x = sh.cd[tid];
          int o = sh.cd_off + excl;
          while (x) {
            const int bit = __ffs(x) - 1;
            Cc.cd_pool[o++] = t0 + tid * 32 + bit;
            x &= x - 1;
          }
        }
        __syncthreads();
        // Resolve this sequence's CD tokens against its real stack.
        if (!sh.fail) {
          const int32_t* pool = Cc.cd_pool + sh.cd_off;
          for (int i = tid; i < sh.cd_len; i += kThreads) {
            const int t = pool[i];
            const int r = WalkToken(A, Vv, t, stack_s, depth, true);
            if (r == kAccept) atomicOr(&sh.mask[(t - t0) >> 5], 1u << ((t - t0) & 31));
            if (r == kOverflow) atomicOr(Bt.err, 1u);
          }
        } else {
          for (int w = tid; w < nwords; w += kThreads) {
            uint32_t x = sh.cd[w];
            while (x) {
              const int bit = __ffs(x) - 1;
              const int t = t0 + w * 32 + bit;
              if (WalkToken(A, Vv, t, stack_s, depth, true) == kAccept) atomicOr(&sh.mask[w], 1u << bit);
              x &= x - 1;
            }
          }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
          const long long si = static_cast<long long>(slot) * Vv.nseg + seg;
          if (!sh.fail) {
            Cc.cd_off[si] = sh.cd_off;
            Cc.cd_len[si] = sh.cd_len;
          }
          atomic_u32 ss(Cc.seg_state[si]);
          ss.store(sh.fail ? kSegFailed : kSegReady, cuda::memory_order_release);
          atomicAdd(Cc.counters + 1, 1ull);
        }
        st_build = 1;
        st_cd = static_cast<unsigned long long>(sh.fail ? 0 : sh.cd_len);
      } else {
        // Direct: the CD bits were resolved with the full stack already.
        if (tid == 0) atomicAdd(Cc.counters + 2, 1ull);
        st_direct = 1;
      }
    }
  }
  __syncthreads();

  // ---- outputs: bitmask words, sampler counts, logits.
  if (bitmask != nullptr) {
    uint32_t* out = bitmask + static_cast<long long>(b) * ldw + w0;
    for (int w = tid; w < nwords; w += kThreads) out[w] = sh.mask[w];
  }
  const int eos_w = Vv.V >> 5;
  if (seg_counts != nullptr) {
    int ca = 0, cs = 0;
    for (int w = tid; w < nwords; w += kThreads) {
      uint32_t m = sh.mask[w];
      if (w0 + w == eos_w) m &= ~(1u << (Vv.V & 31));
      ca += __popc(m);
      cs += __popc(m & __ldg(Vv.structural + w0 + w));
    }
    ca = WarpSum(ca);
    cs = WarpSum(cs);
    if (lane == 0) {
      sh.scratch[warp] = ca;
      sh.best[warp] = static_cast<unsigned long long>(cs);
    }
    __syncthreads();
    if (tid == 0) {
      int ta = 0;
      long long ts = 0;
      for (int i = 0; i < kThreads / 32; ++i) ta += sh.scratch[i], ts += static_cast<long long>(sh.best[i]);
      seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 0] = ta;
      seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 1] = static_cast<int32_t>(ts);
    }
    __syncthreads();
  }
  unsigned long long rd = 0, wr = 0;
  if (MODE == kFillMask && logits != nullptr) {
    uint16_t* row = logits + static_cast<long long>(b) * ld;
    const int nchunks = (t1 - t0 + 7) >> 3;
    for (int c = tid; c < nchunks; c += kThreads) {
      const int tb = t0 + c * 8;
      const uint32_t byte = (sh.mask[c >> 2] >> ((c & 3) * 8)) & 0xffu;
      const int valid = min(8, t1 - tb);
      if (valid == 8 && vec_ok) {
        if (byte == 0xffu) continue;
        uint4* p = reinterpret_cast<uint4*>(row + tb);
        if (byte == 0u) {
          __stcs(p, make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u));
          wr += 16;
        } else {
          uint4 v = __ldcs(p);
          uint32_t* vv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t lo = (byte >> (2 * j)) & 1u, hi = (byte >> (2 * j + 1)) & 1u;
            uint32_t keep = (lo ? 0x0000FFFFu : 0u) | (hi ? 0xFFFF0000u : 0u);
            vv[j] = (vv[j] & keep) | (0xFF80FF80u & ~keep);
          }
          __stcs(p, v);
          rd += 16;
          wr += 16;
        }
      } else {
        for (int j = 0; j < valid; ++j) {
          if (!((byte >> j) & 1u)) row[tb + j] = 0xFF80u;
        }
        wr += 2 * valid;
      }
    }
  } else if (MODE == kFillGreedy) {
    const uint16_t* row = logits + static_cast<long long>(b) * ld;
    const int nchunks = (t1 - t0 + 7) >> 3;
    unsigned long long mine = 0;
    for (int c = tid; c < nchunks; c += kThreads) {
      const int tb = t0 + c * 8;
      const uint32_t byte = (sh.mask[c >> 2] >> ((c & 3) * 8)) & 0xffu;
      if (byte == 0u) continue;
      const int valid = min(8, t1 - tb);
      uint16_t vals[8];
      if (valid == 8 && vec_ok) {
        uint4 v = __ldcs(reinterpret_cast<const uint4*>(row + tb));
        const uint16_t* pv = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) vals[j] = pv[j];
        rd += 16;
      } else {
        for (int j = 0; j < valid; ++j) vals[j] = row[tb + j];
        rd += 2 * valid;
      }
      for (int j = 0; j < valid; ++j) {
        if (!((byte >> j) & 1u)) continue;
        uint32_t bits = static_cast<uint32_t>(vals[j]) << 16;
        uint32_t key = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
        unsigned long long packed = (static_cast<unsigned long long>(key) << 32) |
                                    static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(tb + j));
        mine = packed > mine ? packed : mine;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(0xffffffffu, mine, o);
      mine = y > mine ? y : mine;
    }
    if (lane == 0) sh.best[warp] = mine;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0;
      for (int i = 0; i < kThreads / 32; ++i) m = sh.best[i] > m ? sh.best[i] : m;
      if (m) atomicMax(best + b, m);
    }
  }
  if (Bt.stats_enabled) {
    rd = static_cast<unsigned long long>(WarpSum(static_cast<int>(rd)));
    wr = static_cast<unsigned long long>(WarpSum(static_cast<int>(wr)));
    if (lane == 0 && (rd | wr)) {
      atomicAdd(Bt.stats + 0, rd);
      atomicAdd(Bt.stats + 1, wr);
    }
    if (tid == 0) {
      if (st_hit) atomicAdd(Bt.stats + 2, 1ull);
      if (st_build) atomicAdd(Bt.stats + 3, 1ull);
      if (st_direct) atomicAdd(Bt.stats + 4, 1ull);
      if (st_cd) atomicAdd(Bt.stats + 5, st_cd);
    }
  }
  if (tid == 0 && seg == 0) atomicAdd(Bt.counters + 2, 1ull);
}

// ---------------------------------------------------------------------------
// accept_kernel: one warp per sequence.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ResetSeq(const AutView& A, const BatchView& Bt, int b, int lane,
                                         SeqState* st) {
  if (lane == 0) Bt.stacks[static_cast<long long>(b) * Bt.cap] = A.initial;
  st->depth = 1;
  st->status = kAlive;
}

template <int SAMPLE>
__global__ void __launch_bounds__(128) AcceptKernel(AutView A, VocabView Vv, BatchView Bt,
                                                    const int32_t* __restrict__ tokens,
                                                    int32_t* __restrict__ status_out, int restart,
                                                    const uint32_t* __restrict__ bitmask, long long ldw,
                                                    const int32_t* __restrict__ seg_counts,
                                                    unsigned long long seed,
                                                    unsigned long long* __restrict__ best,
                                                    int32_t* __restrict__ tokens_out, int do_accept) {
  const int lane = threadIdx.x & 31;
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= Bt.B) return;
  SeqState st = Bt.seq[b];
  int32_t* stack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
  int tok = -1;
  if (SAMPLE == kSampleGiven) {
    tok = tokens[b];
  } else if (SAMPLE == kSampleGreedy) {
    const unsigned long long p = best[b];
    tok = p ? static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(p)) : -1;
    __syncwarp();
    if (lane == 0) best[b] = 0ull;
  } else {
    // Synthetic stream; identical rule in oracle/gmask_port.c.
    int na = 0, ns = 0;
    for (int s = lane; s < Vv.nseg; s += 32) {
      na += seg_counts[(static_cast<long long>(b) * Vv.nseg + s) * 2];
      ns += seg_counts[(static_cast<long long>(b) * Vv.nseg + s) * 2 + 1];
    }
    na = WarpSum(na);
    ns = WarpSum(ns);
    const uint32_t* row = bitmask + static_cast<long long>(b) * ldw;
    const bool eos = (row[Vv.V >> 5] >> (Vv.V & 31)) & 1u;
    const unsigned long long u = Mix64(Mix64(seed ^ (static_cast<unsigned long long>(b) * 0xD1B54A32D192ED03ull)) ^
                                       static_cast<unsigned long long>(st.draws));
    st.draws += 1;
    if (na == 0) {
      tok = eos ? Vv.V : -1;
    } else if (eos && ((u >> 32) & 3ull) != 0) {
      tok = Vv.V;
    } else {
      const bool use_s = ((u >> 34) & 1ull) && ns > 0;
      const uint32_t nsel = static_cast<uint32_t>(use_s ? ns : na);
      uint32_t r = static_cast<uint32_t>((static_cast<unsigned long long>(static_cast<uint32_t>(u)) * nsel) >> 32);
      // Segment holding the r-th selected bit.
      int seg = 0;
      for (; seg < Vv.nseg; ++seg) {
        const int c = seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + (use_s ? 1 : 0)];
        if (r < static_cast<uint32_t>(c)) break;
        r -= static_cast<uint32_t>(c);
      }
      const int w0 = seg * kSegWords;
      const int w1 = min(Vv.W, w0 + kSegWords);
      tok = -1;
      for (int wb = w0; wb < w1 && tok < 0; wb += 32) {
        const int w = wb + lane;
        uint32_t x = 0;
        if (w < w1) {
          x = row[w];
          if (w == (Vv.V >> 5)) x &= ~(1u << (Vv.V & 31));
          if (use_s) x &= __ldg(Vv.structural + w);
        }
        const int c = __popc(x);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        if (r < static_cast<uint32_t>(total)) {
          const unsigned hit = __ballot_sync(0xffffffffu, static_cast<uint32_t>(inc) > r);
          const int src = __ffs(hit) - 1;
          if (lane == src) {
            uint32_t rr = r - static_cast<uint32_t>(inc - c);
            while (rr--) x &= x - 1;
            tok = w * 32 + __ffs(x) - 1;
          }
          tok = __shfl_sync(0xffffffffu, tok, src);
        } else {
          r -= static_cast<uint32_t>(total);
        }
      }
    }
  }
  if (tokens_out != nullptr && lane == 0) tokens_out[b] = tok;
  if (!do_accept) {
    if (lane == 0) {
      Bt.seq[b].draws = st.draws;
      if (SAMPLE == kSampleStream) atomicAdd(Bt.counters + 1, 1ull);
    }
    return;
  }

  if (tok >= 0 && st.status == kAlive) {
    const bool eos = tok == Vv.V;
    const int nterm = eos ? 1 : (Vv.tok_off[tok + 1] - Vv.tok_off[tok]);
    const uint8_t* bytes = eos ? nullptr : Vv.tok_bytes + Vv.tok_off[tok];
    int depth = st.depth;
    for (int i = 0; i < nterm; ++i) {
      const int x = eos ? 256 : static_cast<int>(bytes[i]);
      const int state = stack[depth - 1];
      const int cb = A.cand_begin[state * 257 + x];
      const int ce = A.cand_begin[state * 257 + x + 1];
      int found = -1;
      for (int c0 = cb; c0 < ce && found < 0; c0 += 32) {
        const int c = c0 + lane;
        bool match = false;
        if (c < ce) {
          const DevEdge ed = A.edges[A.cand[c]];
          match = ed.cond_len <= depth;
          for (int j = 0; j < ed.cond_len && match; ++j) match = stack[depth - 1 - j] == A.cond[ed.cond_off + j];
        }
        const unsigned m = __ballot_sync(0xffffffffu, match);
        if (m) found = A.cand[c0 + __ffs(m) - 1];
      }
      if (found < 0) {
        st.status = kDead;  // earlier bytes stay applied (runtime.cpp:179-183)
        break;
      }
      const DevEdge ed = A.edges[found];
      const int nd = depth - ed.cond_len + ed.push_len + (ed.flags & 1);
      if (nd > Bt.cap) {
        st.status = kStackOverflow;
        break;
      }
      const int base = depth - ed.cond_len;
      for (int j = lane; j < ed.push_len; j += 32) stack[base + j] = A.push[ed.push_off + j];
      __syncwarp();
      if (ed.flags & 1) {
        if (lane == 0) {
          const int top = stack[base + ed.push_len - 1];
          stack[base + ed.push_len] = A.shift[top * 256 + x];
        }
        __syncwarp();
      }
      depth = nd;
      if (eos) st.status = kAccepted;
    }
    st.depth = depth;
  }
  if (status_out != nullptr && lane == 0) status_out[b] = st.status;
  if (restart && st.status != kAlive) {
    ResetSeq(A, Bt, b, lane, &st);
    if (lane == 0) atomicAdd(Bt.counters + 0, 1ull);
  }
  if (lane == 0) {
    Bt.seq[b] = st;
    atomicAdd(Bt.counters + 3, 1ull);
    if (SAMPLE == kSampleStream) atomicAdd(Bt.counters + 1, 1ull);
  }
}

__global__ void ResetKernel(AutView A, BatchView Bt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= Bt.B) return;
  Bt.stacks[static_cast<long long>(b) * Bt.cap] = A.initial;
  SeqState st;
  st.depth = 1;
  st.status = kAlive;
  st.draws = 0;
  st.reserved = 0;
  Bt.seq[b] = st;
}

// ---------------------------------------------------------------------------
cudaError_t LaunchReset(const AutView& a, const BatchView& b, cudaStream_t s) {
  ResetKernel<<<(b.B + 127) / 128, 128, 0, s>>>(a, b);
  return cudaGetLastError();
}

cudaError_t LaunchFill(int mode, const AutView& a, const VocabView& v, const CacheView& c,
                       const BatchView& b, uint32_t* bitmask, long long ldw, uint16_t* logits,
                       long long ld, int32_t* seg_counts, unsigned long long* best,
                       cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  const int vec_ok = logits != nullptr && (ld % 8) == 0 &&
                     (reinterpret_cast<uintptr_t>(logits) % 16) == 0;
  const size_t dyn = static_cast<size_t>(b.cap) * sizeof(int32_t);
  dim3 grid(static_cast<unsigned>(v.nseg), static_cast<unsigned>(b.B));
  if (mode == kFillGreedy) {
    if (dyn > 48 * 1024) {
      cudaFuncSetAttribute(FillKernel<kFillGreedy>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(dyn));
    }
    FillKernel<kFillGreedy><<<grid, kThreads, dyn, s>>>(a, v, c, b, bitmask, ldw, logits, ld, seg_counts,
                                                        best, vec_ok);
  } else {
    if (dyn > 48 * 1024) {
      cudaFuncSetAttribute(FillKernel<kFillMask>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(dyn));
    }
    FillKernel<kFillMask><<<grid, kThreads, dyn, s>>>(a, v, c, b, bitmask, ldw, logits, ld, seg_counts,
                                                      best, vec_ok);
  }
  return cudaGetLastError();
}

cudaError_t LaunchAccept(int sample, const AutView& a, const VocabView& v, const BatchView& b,
                         const int32_t* tokens, int32_t* status_out, int restart,
                         const uint32_t* bitmask, long long ldw, const int32_t* seg_counts,
                         unsigned long long seed, unsigned long long* best, int32_t* tokens_out,
                         int do_accept, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  const int threads = 128;
  const int blocks = (b.B * 32 + threads - 1) / threads;
  switch (sample) {
    case kSampleGiven:
      AcceptKernel<kSampleGiven><<<blocks, threads, 0, s>>>(a, v, b, tokens, status_out, restart, bitmask,
                                                           ldw, seg_counts, seed, best, tokens_out, do_accept);
      break;
    case kSampleStream:
      AcceptKernel<kSampleStream><<<blocks, threads, 0, s>>>(a, v, b, tokens, status_out, restart, bitmask,
                                                            ldw, seg_counts, seed, best, tokens_out, do_accept);
      break;
    default:
      AcceptKernel<kSampleGreedy><<<blocks, threads, 0, s>>>(a, v, b, tokens, status_out, restart, bitmask,
                                                            ldw, seg_counts, seed, best, tokens_out, do_accept);
      break;
  }
  return cudaGetLastError();
}

}  // namespace pre3
