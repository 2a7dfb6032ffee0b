// kernels.cu — sm_100a kernels of the constrained-decoding hot path.
//
// A decode step is ONE launch of FillKernel (grid: vocab segment x sequence):
//   1. help build: CTAs first drain the build queue produced by the previous
//      step's lookups — each unit classifies 256 tokens against a new context
//      key (accept / reject / context-dependent) into the slot's CI and CD
//      bitsets.  Empty in the steady state.
//   2. fill: CTA (seg, b) streams its 256 CI words, walks only the CD tokens
//      against the sequence's real stack (Engine::ComputeMask,
//      runtime.cpp:261-287), writes the 32-bit mask words and, fused, the
//      bf16 -inf logits (or a greedy argmax partial).
//   3. tail: the last CTA to finish a sequence samples its token (synthetic
//      stream or greedy), accepts it — Engine::Step per byte
//      (runtime.cpp:177-186), one warp, lanes over candidate edges in
//      arbitration order (FindEdge, runtime.cpp:138-146) — and looks up the
//      context slot of the next step, queueing builds for new contexts.
// The same pieces run standalone for the reference-shaped API
// (LookupKernel, AcceptKernel, FillKernel without a tail).
//
// Integer/bit work only: no tensor cores (nothing here is a contraction).
#include <cuda/atomic>
#include <algorithm>
#include <utility>

#include "kernels.cuh"

#ifndef PRE3_FILL_MIN_BLOCKS
#define PRE3_FILL_MIN_BLOCKS 4  // fill CTAs resident per SM (64 registers)
#endif
#ifndef PRE3_BULK_SPANS
#define PRE3_BULK_SPANS 0xFF  // span positions whose fully masked spans go to the TMA engine (the rest: LSU stores)
#endif
#ifndef PRE3_BULK_RUN
#define PRE3_BULK_RUN 1  // masked spans per bulk store (a run of adjacent ones: one TMA op)
#endif
#ifndef PRE3_BULK_EVICT_FIRST
#define PRE3_BULK_EVICT_FIRST 1  // -inf bulk stores with an L2 evict-first hint
#endif
#ifndef PRE3_COMPACT_GREEDY
#define PRE3_COMPACT_GREEDY 0  // greedy light pass: allowed chunks in one round trip, packed 16-bit keys
#endif
#ifndef PRE3_COMPACT_MIXED
#define PRE3_COMPACT_MIXED 0  // light pass: all mixed chunks of a segment copied in one round trip
#endif
#ifndef PRE3_DIAG_NO_MIXED
#define PRE3_DIAG_NO_MIXED 0  // (diagnostics only, wrong logits) every full span bulk-stored as -inf
#endif
// Register caps (A/B): a fill at 64 registers x 4 CTAs fills the register
// file, so no accept CTA can be resident beside it until fill CTAs retire.
#ifndef PRE3_FILL_BOUNDS
#define PRE3_FILL_BOUNDS __launch_bounds__(kThreads, PRE3_FILL_MIN_BLOCKS)
#endif
#ifndef PRE3_ACCEPT_BOUNDS
#define PRE3_ACCEPT_BOUNDS __launch_bounds__(128)
#endif
#ifndef PRE3_LIGHT_PER_CTA
#define PRE3_LIGHT_PER_CTA 0  // light items per fill CTA (0: chosen per launch, LightPerCta)
#endif
#ifndef PRE3_FILL_SMEM_PAD
#define PRE3_FILL_SMEM_PAD 0  // (A/B) extra dynamic shared memory per fill CTA: fewer fill CTAs per SM
#endif
#ifndef PRE3_SAMPLE_BATCH
#define PRE3_SAMPLE_BATCH 2  // sampler pass 1: chunks whose loads are issued together per thread
#endif
#ifndef PRE3_LIGHT_BUILD_UNITS
#define PRE3_LIGHT_BUILD_UNITS -1  // build units a light fill CTA takes before its items (-1: until none is left)
#endif
#ifndef PRE3_ACCEPT_SPREAD
#define PRE3_ACCEPT_SPREAD 5  // merged split step: accept CTAs interleaved over this many eighths of the light CTAs
#endif
#ifndef PRE3_ARRIVE_FENCE
#define PRE3_ARRIVE_FENCE 0  // (A/B) item arrivals behind a full __threadfence() instead of a release add
#endif
#ifndef PRE3_BULK_MASKED
#define PRE3_BULK_MASKED 1  // fully masked spans as one bulk (TMA) store
#endif

namespace pre3 {
namespace {

enum : int { kReject = 0, kAccept = 1, kUnknown = 2, kOverflow = 3 };
enum : int { kAlive = 0, kDead = 1, kAccepted = 2, kStackOverflow = 3 };

using atomic_u64 = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
using atomic_i32 = cuda::atomic_ref<int32_t, cuda::thread_scope_device>;

__device__ __forceinline__ unsigned long long Mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Token ids at the ABI vs mask bits (VocabView::layout): with a model logit
// layout the ABI speaks columns (EOS = eos_col); bits stay the reference's
// (EOS = V).  An id that is no token maps past V (the accept kills it).
__device__ __forceinline__ int IdToBit(const VocabView& Vv, int id) {
  if (!Vv.layout || id < 0) return id;
  if (id == Vv.eos_col) return Vv.V;
  return id < Vv.V ? id : Vv.V + 1;
}
__device__ __forceinline__ int BitToId(const VocabView& Vv, int t) { return (Vv.layout && t == Vv.V) ? Vv.eos_col : t; }

// A candidate record in registers: header, first 4 pushed states, condition
// entries 1..16 — six independent 16-B loads (one round trip).
struct Rec {
  int cond_len, push_len, cond_off, push_off, new_state;
  int4 p;     // push[0..3]
  int4 c[4];  // cond entries 1..16
};

__device__ __forceinline__ Rec LoadRec(const CandRec* rp) {
  const int4* q = reinterpret_cast<const int4*>(rp);
  const int4 h = __ldg(q);
  Rec r;
  r.p = __ldg(q + 1);
#pragma unroll
  for (int v = 0; v < 4; ++v) r.c[v] = __ldg(q + 2 + v);
  r.cond_len = h.x & 0xffff;
  r.push_len = h.x >> 16;
  r.cond_off = h.y;
  r.push_off = h.z;
  r.new_state = h.w;
  return r;
}

__device__ __forceinline__ int Lane4(const int4& q, int i) {
  return i == 0 ? q.x : i == 1 ? q.y : i == 2 ? q.z : q.w;
}

// Condition entry j (1-based, j <= 16 inline, else from the pool).
// Byte j (< 8) of a token record (VocabView::tok_rec).
__device__ __forceinline__ int TokByte(const int4& tr, int j) {
  return static_cast<int>(((j < 4 ? static_cast<uint32_t>(tr.z) : static_cast<uint32_t>(tr.w)) >> (8 * (j & 3))) & 0xffu);
}

// Byte `lane` of a token for a warp walk (256 past the end / for EOS): the
// first 8 from the record, the rest from tok_bytes.
__device__ __forceinline__ int TokLaneByte(const int4& tr, const uint8_t* tok_bytes, int lane, int nterm, bool eos) {
  if (eos || lane >= nterm) return 256;
  return lane < 8 ? TokByte(tr, lane) : static_cast<int>(__ldg(tok_bytes + tr.x + lane));
}

__device__ __forceinline__ int CondEntry(const Rec& r, const int32_t* rec_cond, int j) {
  return j <= 16 ? Lane4(r.c[(j - 1) >> 2], (j - 1) & 3) : __ldg(rec_cond + r.cond_off + j - 1);
}

// Device-scope relaxed load (L2; neither a stale L1 hit nor a system-scope
// volatile access).
template <typename T>
__device__ __forceinline__ T LoadRelaxed(const T* p) {
  return cuda::atomic_ref<T, cuda::thread_scope_device>(*const_cast<T*>(p)).load(cuda::memory_order_relaxed);
}

template <typename T>
__device__ __forceinline__ T LoadAcquire(const T* p) {
  return cuda::atomic_ref<T, cuda::thread_scope_device>(*const_cast<T*>(p)).load(cuda::memory_order_acquire);
}

template <typename T>
__device__ __forceinline__ void StoreRelease(T* p, T v) {
  cuda::atomic_ref<T, cuda::thread_scope_device>(*p).store(v, cuda::memory_order_release);
}

// Publishes an item's arrival: the group's (warp's / CTA's) stores were
// ordered before the calling thread by the barrier that precedes this call,
// and the release makes them visible with the count (MEMBAR.ALL, no L1
// invalidate — a full __threadfence() is MEMBAR.SC + CCTL.IVALL).
__device__ __forceinline__ int ArriveRelease(int* p) {
#if PRE3_ARRIVE_FENCE
  __threadfence();
  return atomicAdd(p, 1);
#else
  return cuda::atomic_ref<int, cuda::thread_scope_device>(*p).fetch_add(1, cuda::memory_order_release);
#endif
}

// Queue q of the batch, selected without indexing the by-value parameter
// struct (a dynamic index would copy the whole BatchView to local memory).
__device__ __forceinline__ BuildQueue QueueOf(const BatchView& Bt, int q) {
  return q == 0 ? Bt.queue[0] : (q == 1 ? Bt.queue[1] : Bt.queue[2]);
}


// Programmatic dependent launch: every kernel of a step waits here for the
// previous kernel on the stream to finish (its memory visible), then lets the
// next one be scheduled — so a kernel's launch and CTA ramp-up overlap the
// tail of its predecessor instead of following it.
__device__ __forceinline__ void PdlEnter() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ unsigned long long NowNs() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Appends one diagnostics record (BatchView::trace); call from one thread.
__device__ __forceinline__ void TraceEvent(const BatchView& Bt, int kind, int b, int seg, unsigned long long t0,
                                           unsigned long long extra) {
  if (Bt.trace == nullptr) return;
  const unsigned long long i = atomicAdd(Bt.trace, 1ull);
  if (i >= static_cast<unsigned long long>(Bt.trace_cap)) return;
  unsigned long long* r = Bt.trace + 4 * (i + 1);
  r[0] = static_cast<unsigned long long>(kind) | (static_cast<unsigned long long>(seg & 0xffffff) << 8) |
         (static_cast<unsigned long long>(static_cast<uint32_t>(b)) << 32);
  r[1] = t0;
  r[2] = NowNs();
  r[3] = extra;
}

// ---------------------------------------------------------------------------
// One token walk: the body of ComputeMaskNaive's per-token replay
// (runtime.cpp:289-307) — Step per byte with FindEdge's first match in
// arbitration order and Apply's pop/push — against a stack given as
// base[0..nb) (bottom first) plus a private overlay of pushed entries.
// complete == false: base is only the top of an unknown deeper stack; a
// condition that reaches below it (after matching every known entry), or a
// dynamic target read from below it, makes the outcome kUnknown.  Because
// arbitration is first-match, an unknown earlier candidate is also unknown.
// ---------------------------------------------------------------------------
// Out of line (one copy of the code, shared by the build, heavy and light
// paths: the fill kernel is i-cache bound otherwise); the automaton and
// vocabulary arrays are passed as scalars so no parameter struct is copied to
// local memory.
// Indexed FindEdge for a (state, terminal) with many candidates (the
// FlatLayout::hidx_* tables): the winner is the candidate whose condition
// equals the stack top for the longest such length; with an incomplete stack
// of D known entries, a longer condition whose first D entries match makes
// the outcome unknown (it comes first in arbitration order).  Returns the
// candidate index, -1 (no edge), -2 (unknown) or -3 (hash collision: scan).
// Entry j of the virtual stack: j < nl ? loc[nl-1-j] : base[nb-1-(j-nl)].
__device__ __forceinline__ int IndexedFindEdge(const int16_t* hlens,
                                               const unsigned long long* hexact, unsigned long long emask,
                                               const unsigned long long* hprefix, unsigned long long pmask,
                                               int2 meta, int state, int x, const int32_t* loc, int nl,
                                               const int32_t* base, int nb, bool complete) {
  const int nlen = meta.y & 0xffff;
  const int maxl = meta.y >> 16;
  const int D = nl + nb;
  const int H = min(maxl, D);
  unsigned long long r = CondSeed(state, x);
  int li = nlen - 1;  // lens are descending: walk from the shortest
  int best = -1;
  for (int j = 1; j <= H; ++j) {
    const int e = j - 1 < nl ? loc[nl - j] : base[nb - 1 - (j - 1 - nl)];
    r = CondMix(r ^ static_cast<uint32_t>(e));
    while (li >= 0 && __ldg(hlens + meta.x + li) < j) --li;
    if (li >= 0 && __ldg(hlens + meta.x + li) == j) {
      const unsigned long long key = CondKey(r, kSaltExact, j);
      for (unsigned long long i = key & emask;; i = (i + 1) & emask) {
        const unsigned long long k = __ldg(hexact + 2 * i);
        if (k == key) {
          best = static_cast<int>(__ldg(hexact + 2 * i + 1));  // longer hits overwrite shorter ones
          break;
        }
        if (k == 0ull) break;
      }
    }
  }
  if (!complete && maxl > D) {
    const unsigned long long key = CondKey(r, kSaltPrefix, D);
    for (unsigned long long i = key & pmask;; i = (i + 1) & pmask) {
      const unsigned long long k = __ldg(hprefix + i);
      if (k == key) return -2;
      if (k == 0ull) break;
    }
  }
  return best;
}

__device__ __noinline__ int WalkTokenImpl(const CandRec* first, const int32_t* rec_begin, const CandRec* recs,
                                          const int32_t* rec_cond, const int32_t* rec_push, const int32_t* shift,
                                          const int4* tok_rec, const uint8_t* tok_bytes, int32_t V, int32_t t,
                                          const int32_t* base, int nb, bool complete, const int2* hmeta,
                                          const int16_t* hlens, const unsigned long long* hexact,
                                          unsigned long long emask, const unsigned long long* hprefix,
                                          unsigned long long pmask) {
  const struct {
    const CandRec* first;
    const int32_t* rec_begin;
    const CandRec* recs;
    const int32_t* rec_cond;
    const int32_t* rec_push;
    const int32_t* shift;
  } A{first, rec_begin, recs, rec_cond, rec_push, shift};
  int32_t loc[kWalkOverlay];
  int nl = 0;
  const bool eos = t == V;
  const int4 tr = __ldg(tok_rec + t);  // offset, length, first 8 bytes: one round trip
  const int nterm = tr.y;
  if (nterm == 0) return kReject;  // a disabled id (gm_engine_options::disabled)
  const uint8_t* bytes = tok_bytes + tr.x;
  int state = base[nb - 1];
  int x_next = eos ? 256 : TokByte(tr, 0);
  for (int i = 0; i < nterm; ++i) {
    const int x = x_next;
    if (i + 1 < nterm) x_next = i + 1 < 8 ? TokByte(tr, i + 1) : static_cast<int>(__ldg(bytes + i + 1));
    // Candidates of (state, x) in arbitration order (the first one from the
    // dense table, in the same round trip as the range); none rejects.
    const int idx = state * 257 + x;
    const int cb = __ldg(A.rec_begin + idx);
    const int ce = __ldg(A.rec_begin + idx + 1);
    const int2 meta = __ldg(hmeta + idx);
    int found = -1;
    Rec fr;
    int c_scan = cb;  // first candidate of the linear scan (ce: none)
    if (meta.y != 0) {
      const int c = IndexedFindEdge(hlens, hexact, emask, hprefix, pmask, meta, state, x, loc, nl, base, nb,
                                    complete);
      if (c == -2) return kUnknown;
      c_scan = ce;
      if (c >= 0) {
        // Verify the hit exactly (a 64-bit key collision falls back to the scan).
        const Rec h = LoadRec(A.recs + c);
        bool same = h.cond_len <= nl + nb;
        for (int j = 1; j < h.cond_len && same; ++j) {
          const int have = j < nl ? loc[nl - 1 - j] : base[nb - 1 - (j - nl)];
          same = have == CondEntry(h, A.rec_cond, j);
        }
        if (same) {
          found = c;
          fr = h;
        } else {
          c_scan = cb;
        }
      }
    }
    Rec r = LoadRec(A.first + idx);
    for (int c = c_scan; c < ce; ++c) {
      if (c > cb) r = LoadRec(A.recs + c);
      // ConditionMatches (runtime.cpp:123-131) for entries 1..k-1 (entry 0 is
      // the current state) against the overlay, then the known base.
      int verdict = 1;  // 1 match, 0 no match, 2 unknown
      for (int j = 1; j < r.cond_len && verdict == 1; ++j) {
        const int want = CondEntry(r, A.rec_cond, j);
        int have;
        if (j < nl) {
          have = loc[nl - 1 - j];
        } else if (j - nl < nb) {
          have = base[nb - 1 - (j - nl)];
        } else {
          verdict = complete ? 0 : 2;  // reaches below the known stack
          break;
        }
        if (have != want) verdict = 0;
      }
      if (verdict == 2) return kUnknown;  // every known entry matched so far
      if (verdict == 1) {
        found = c;
        fr = r;
        break;
      }
    }
    if (found < 0) return kReject;
    if (i == nterm - 1) return kAccept;  // the last Step succeeded
    // Apply (runtime.cpp:148-168) on the overlay.
    const int k = fr.cond_len;
    if (k <= nl) {
      nl -= k;
    } else {
      nb -= k - nl;
      nl = 0;
    }
    // Past the overlay: on a partial key (a shared context slot) the token
    // is context-dependent — the cached row must not reject it for good; each
    // fill then walks it on the sequence's whole stack, where overflowing
    // the overlay again is an error (kOverflow: the caller raises Bt.err).
    if (nl + fr.push_len + 1 > kWalkOverlay) return complete ? kOverflow : kUnknown;
    for (int j = 0; j < fr.push_len; ++j) loc[nl++] = j < 4 ? Lane4(fr.p, j) : __ldg(A.rec_push + fr.push_off + j);
    if (fr.new_state < 0) {
      const int top = nl > 0 ? loc[nl - 1] : (nb > 0 ? base[nb - 1] : -1);
      if (top < 0) return complete ? kReject : kUnknown;
      state = __ldg(A.shift + top * 256 + x);
      if (state < 0) return kReject;  // unreachable for validated automata
      loc[nl++] = state;
    } else {
      state = fr.new_state;
    }
  }
  return kAccept;
}

__device__ __forceinline__ int WalkToken(const AutView& A, const VocabView& Vv, int32_t t, const int32_t* base, int nb,
                                         bool complete) {
  return WalkTokenImpl(A.first, A.rec_begin, A.recs, A.rec_cond, A.rec_push, A.shift, Vv.tok_rec,
                                     Vv.tok_bytes, Vv.V, t, base, nb, complete, A.hidx_meta, A.hidx_lens,
                                     A.hidx_exact, A.hidx_exact_mask, A.hidx_prefix, A.hidx_prefix_mask);
}

// The same walk done by one warp for one token (complete stacks only): lanes
// test the candidate edges of each byte in parallel (FindEdge), so a byte step
// costs about one round trip instead of a serial scan; the pushed overlay
// lives in registers (lane i = overlay entry i, bottom first), the base stack
// in shared or global memory.  Used where few tokens need walking and their
// latency is on the critical path (context-dependent tokens of a step).
// Returns kOverflow when the overlay would pass 32 entries (the caller then
// repeats the walk with WalkToken).
__device__ int WalkWarp(const AutView& A, const VocabView& Vv, int32_t t, const int32_t* base, int nb, int lane) {
  const bool eos = t == Vv.V;
  const int4 tr = __ldg(Vv.tok_rec + t);
  const int off = tr.x;
  const int nterm = tr.y;
  if (nterm == 0) return kReject;  // a disabled id
  const int xb = TokLaneByte(tr, Vv.tok_bytes, lane, nterm, eos);
  int ov = -1;  // overlay entry `lane`
  int nl = 0;
  int state = base[nb - 1];
  for (int i = 0; i < nterm; ++i) {
    const int xs = __shfl_sync(0xffffffffu, xb, i & 31);
    const int x = eos ? 256 : (i < 32 ? xs : static_cast<int>(__ldg(Vv.tok_bytes + off + i)));
    const int idx = state * 257 + x;
    const int cb = __ldg(A.rec_begin + idx);
    const int ce = __ldg(A.rec_begin + idx + 1);
    Rec r;
    r.cond_len = 0;
    r.push_len = 0;
    if (lane == 0) r = LoadRec(A.first + idx);
    int win = -1;
    for (int cbase = cb, round = 0; cbase < ce; cbase = round == 1 ? cb + 1 : cbase + 32) {
      const int c = round == 0 ? (lane == 0 ? cb : ce) : cbase + lane;
      if (round++ > 0) {
        r.cond_len = 0;
        r.push_len = 0;
        if (c < ce) r = LoadRec(A.recs + c);
      }
      bool match = c < ce && r.cond_len <= nl + nb;
      const int jmax = static_cast<int>(__reduce_max_sync(0xffffffffu, match ? static_cast<unsigned>(r.cond_len) : 1u));
#pragma unroll
      for (int j = 1; j <= 16; ++j) {
        if (j >= jmax) break;
        const int sh = __shfl_sync(0xffffffffu, ov, (nl - 1 - j) & 31);
        if (match && j < r.cond_len) {
          const int have = j < nl ? sh : base[nb - 1 - (j - nl)];
          if (have != Lane4(r.c[(j - 1) >> 2], (j - 1) & 3)) match = false;
        }
      }
      for (int j = 17; j < r.cond_len && match; ++j) {  // long conditions: overlay (<= 32) or base
        const int have = j < nl ? -2 : base[nb - 1 - (j - nl)];
        const int want = __ldg(A.rec_cond + r.cond_off + j - 1);
        match = (j < nl) ? true : have == want;
      }
      // An overlay entry deeper than 16 under a long condition: resolve it
      // with warp-uniform shuffles (rare).
      {
        const int maxlen = __reduce_max_sync(0xffffffffu, match ? static_cast<unsigned>(r.cond_len) : 0u);
        for (int j = 17; j < maxlen && j < nl; ++j) {
          const int sh = __shfl_sync(0xffffffffu, ov, (nl - 1 - j) & 31);
          if (match && j < r.cond_len && sh != __ldg(A.rec_cond + r.cond_off + j - 1)) match = false;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, match);
      if (m) {
        win = __ffs(m) - 1;
        break;
      }
    }
    if (win < 0) return kReject;
    if (i == nterm - 1) return kAccept;
    const int cond_len = __shfl_sync(0xffffffffu, r.cond_len, win);
    const int push_len = __shfl_sync(0xffffffffu, r.push_len, win);
    const int push_off = __shfl_sync(0xffffffffu, r.push_off, win);
    const int new_state = __shfl_sync(0xffffffffu, r.new_state, win);
    const int p0 = __shfl_sync(0xffffffffu, r.p.x, win);
    const int p1 = __shfl_sync(0xffffffffu, r.p.y, win);
    const int p2 = __shfl_sync(0xffffffffu, r.p.z, win);
    const int p3 = __shfl_sync(0xffffffffu, r.p.w, win);
    if (cond_len <= nl) {
      nl -= cond_len;
    } else {
      nb -= cond_len - nl;
      nl = 0;
    }
    const int dyn = new_state < 0 ? 1 : 0;
    if (nl + push_len + dyn > 32) return kOverflow;
    const int j = lane - nl;  // pushed entry this lane receives
    if (j >= 0 && j < push_len) {
      ov = j == 0 ? p0 : j == 1 ? p1 : j == 2 ? p2 : j == 3 ? p3 : __ldg(A.rec_push + push_off + j);
    }
    nl += push_len;
    if (dyn) {
      const int sh = __shfl_sync(0xffffffffu, ov, (nl - 1) & 31);
      const int top = nl > 0 ? sh : (nb > 0 ? base[nb - 1] : -1);
      if (top < 0) return kReject;
      state = __ldg(A.shift + top * 256 + x);
      if (state < 0) return kReject;  // unreachable for validated automata
      if (lane == nl) ov = state;
      ++nl;
    } else {
      state = new_state;
    }
  }
  return kAccept;
}

__device__ __forceinline__ int WarpSum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int WarpInclusiveScan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread (blockDim == kThreads).
__device__ int BlockExclusiveScan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int inc = WarpInclusiveScan(v, lane);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = lane < kThreads / 32 ? scratch[lane] : 0;
    const int winc = WarpInclusiveScan(w, lane);
    if (lane < kThreads / 32) scratch[lane] = winc - w;
    if (lane == kThreads / 32 - 1) scratch[kThreads / 32] = winc;
  }
  __syncthreads();
  const int out = scratch[warp] + inc - v;
  *total = scratch[kThreads / 32];
  __syncthreads();
  return out;
}

// Hash of a context key: entries mixed independently (position-salted) and
// XOR-combined, so a warp computes it with one Mix64 per lane and a
// butterfly (KeyHashWarp) instead of a serial chain of n.
__device__ __forceinline__ unsigned long long KeyEntryMix(int32_t v, int i) {
  return Mix64((static_cast<unsigned long long>(static_cast<uint32_t>(v)) << 32) |
               static_cast<unsigned long long>(i + 1));
}
__device__ __forceinline__ unsigned long long KeyHashFinish(unsigned long long x, int n, int complete) {
  return Mix64(x ^ Mix64(0x5ca1ab1eull ^ static_cast<unsigned long long>(n | (complete << 8)))) | 1ull;
}
__device__ unsigned long long KeyHash(const int32_t* key, int n, int complete) {
  unsigned long long x = 0ull;
  for (int i = 0; i < n; ++i) x ^= KeyEntryMix(key[i], i);
  return KeyHashFinish(x, n, complete);
}
// The same for a warp holding entry `lane` in kv (lanes < n).
__device__ __forceinline__ unsigned long long KeyHashWarp(int kv, int n, int complete, int lane) {
  unsigned long long x = lane < n ? KeyEntryMix(kv, lane) : 0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
  return KeyHashFinish(x, n, complete);
}

// Index entry tag of a key hash (bit 63 set: never 0 = empty).
__device__ __forceinline__ unsigned long long EntryTag(unsigned long long h) { return (h | (1ull << 63)) & ~kRowMask; }

// Pops a free row (-1: none left: the caller uses a private row).  The
// count is mirrored to host-mapped memory for the auto-eviction check.
__device__ __forceinline__ int PopRow(const CacheView& C) {
  const int k = atomicSub(C.row_free_n, 1);
  if (k <= 0) return -1;
  if (C.host_free != nullptr) *reinterpret_cast<volatile int32_t*>(C.host_free) = k - 1;
  return __ldcg(C.row_free + (k - 1));
}

// Index entry at position i once its claimant has published the row (the
// row and its key follow the claim immediately); bounded at ~0.5 ms, after
// which the caller falls back to a private row.
__device__ __forceinline__ unsigned long long WaitPublished(const CacheView& C, int i, unsigned long long e) {
  for (int spin = 0; (e & kRowMask) == static_cast<unsigned long long>(kRowPending) && spin < 4096; ++spin) {
    __nanosleep(128);
    e = LoadAcquire(C.slot_hash + i);
  }
  return e;
}

// Claims index position i for `tag`, pops a row, writes its key row and
// meta, publishes tag | row.  Returns the row, -1 when the position was
// taken by someone else, -2 when no row is free (the claim is withdrawn).
__device__ int InsertRow(const CacheView& C, int i, unsigned long long tag, const int32_t* key, int n, int complete) {
  if (atomicCAS(C.slot_hash + i, 0ull, tag | static_cast<unsigned long long>(kRowPending)) != 0ull) return -1;
  const int row = PopRow(C);
  if (row < 0) {
    StoreRelease(C.slot_hash + i, 0ull);
    return -2;
  }
  for (int j = 0; j < kMaxContext; ++j) C.slot_keys[row * kMaxContext + j] = j < n ? key[j] : -1;
  atomic_i32 meta(C.slot_meta[row]);
  meta.store(n | (complete << 8) | (1 << 16), cuda::memory_order_release);
  C.row_ref[row] = 1;
  atomicAdd(C.counters + 0, 1ull);
  StoreRelease(C.slot_hash + i, tag | static_cast<unsigned long long>(row));
  return row;
}

// Finds or inserts the row of a key.  Returns the row (created = true when
// this thread inserted it) or -1 (no free row, or the key is being published
// by another thread right now).
__device__ int LookupSlot(const CacheView& C, const int32_t* key, int n, int complete, bool* created) {
  const unsigned long long h = KeyHash(key, n, complete);
  const unsigned long long tag = EntryTag(h);
  const int meta_want = n | (complete << 8);
  *created = false;
  const unsigned long long imask = static_cast<unsigned long long>(C.IC - 1);
  for (int p = 0; p < 64; ++p) {
    const int i = static_cast<int>((h + static_cast<unsigned long long>(p)) & imask);
    unsigned long long cur = LoadAcquire(C.slot_hash + i);
    if (cur == 0ull) {
      const int r = InsertRow(C, i, tag, key, n, complete);
      if (r >= 0) {
        *created = true;
        return r;
      }
      if (r == -2) return -1;
      cur = LoadAcquire(C.slot_hash + i);
    }
    if ((cur & ~kRowMask) != tag) continue;
    cur = WaitPublished(C, i, cur);
    if ((cur & ~kRowMask) != tag || (cur & kRowMask) == static_cast<unsigned long long>(kRowPending)) return -1;
    const int row = static_cast<int>(cur & kRowMask);
    const int m = LoadAcquire(C.slot_meta + row);
    if ((m & 0x1ffff) != (meta_want | (1 << 16))) continue;
    // Whole key row in independent vector loads.
    const int4* krow = reinterpret_cast<const int4*>(C.slot_keys + row * kMaxContext);
    int4 q[kMaxContext / 4];
#pragma unroll
    for (int v = 0; v < kMaxContext / 4; ++v) q[v] = 4 * v < n ? __ldcg(krow + v) : make_int4(-1, -1, -1, -1);
    bool same = true;
#pragma unroll
    for (int j = 0; j < kMaxContext; ++j) {
      if (j < n && Lane4(q[j >> 2], j & 3) != key[j]) same = false;
    }
    if (same) {
      C.row_ref[row] = 1;
      return row;
    }
  }
  return -1;
}

// seq_slot / seq_hmask rows of fill `fill_no` (double-buffered like
// heavy_index: an accept that overlaps a fill writes the next fill's row
// while that fill's items may still read their own).
__device__ __forceinline__ int32_t* SeqSlot(const BatchView& Bt, int fill_no) {
  return Bt.seq_slot + static_cast<long long>(fill_no & 1) * Bt.B;
}
__device__ __forceinline__ uint32_t* SeqHmask(const BatchView& Bt, int fill_no) {
  return Bt.seq_hmask + static_cast<long long>(fill_no & 1) * Bt.B;
}

// Context slot of sequence b for the next fill (seq_slot[b]); a new shared
// slot or a private row queues one build item per segment into `q`.
// `key` = the top min(depth, K) stack entries, top first.  Returns seq_slot[b].
__device__ int AssignSlotKey(const CacheView& Cc, const BatchView& Bt, int q, int tag, int b, const SeqState& st,
                             int nseg, const int32_t* key) {
  int32_t* slot_out = SeqSlot(Bt, tag) + b;
  if (st.status != kAlive) {
    *slot_out = -2;
    return -2;
  }
  const int n = min(st.depth, Cc.K);
  const int complete = st.depth <= Cc.K ? 1 : 0;
  bool created = false;
  int slot = LookupSlot(Cc, key, n, complete, &created);
  bool wait = true;
  if (slot < 0 || created) {
    // Slots are never reused, so a new slot's counters are still zero.
    const BuildQueue Q = QueueOf(Bt, q);
    if (slot < 0) {
      slot = Cc.C + b;
      for (int s = 0; s < nseg; ++s) Bt.priv_done[static_cast<long long>(b) * nseg + s] = 0;
      atomicAdd(Cc.counters + 2, 1ull);
      __threadfence();  // zeroed counters visible before the items
    } else {
      atomicAdd(Cc.counters + 1, static_cast<unsigned long long>(nseg));
      if (Cc.R > 0 && n > Cc.R) {
        // Parent: the same top keyed R deep (queued first, so its units are
        // dequeued before the child's).
        bool pc = false;
        const int parent = LookupSlot(Cc, key, Cc.R, 0, &pc);
        if (pc) {
          atomicAdd(Cc.counters + 1, static_cast<unsigned long long>(nseg));
          const unsigned int pat = atomicAdd(Q.n_items, static_cast<unsigned int>(nseg));
          for (int s = 0; s < nseg; ++s) Q.items[pat + s] = make_int4(parent, s, b, 0);
        }
        Cc.slot_parent[slot] = parent;
        if (parent >= 0) atomicAdd(Cc.counters + 3, 1ull);
        __threadfence();  // parent link visible before the child's items
      }
    }
    const unsigned int at = atomicAdd(Q.n_items, static_cast<unsigned int>(nseg));
    for (int s = 0; s < nseg; ++s) Q.items[at + s] = make_int4(slot, s, b, 0);
  } else {
    // Existing slot: only one whose build is still queued needs a wait.
    wait = LoadAcquire(Cc.slot_built + slot) < nseg * kChunksPerSeg;
  }
  const int flagged = slot | (wait ? kSlotWait : 0);
  *slot_out = flagged;
  return flagged;
}

// heavy_index entry: (fill number mod 2^15) << 16 | heavy-list index.  Every
// lookup pass rewrites all entries, so an entry is at most one fill stale and
// the tag tells the fill whether it was written for it.
__device__ __forceinline__ int HeavyTag(int fill_no, int idx) { return ((fill_no & 0x7fff) << 16) | idx; }
__device__ __forceinline__ int NextFill(int fill_no) { return fill_no + 1 == kFillPeriod ? 0 : fill_no + 1; }
__device__ __forceinline__ int PrevFill(int fill_no) { return fill_no == 0 ? kFillPeriod - 1 : fill_no - 1; }

// heavy_index is double-buffered by fill parity: the fused tail of fill N
// writes fill N+1's entries while fill N's CTAs may still read their own.
__device__ __forceinline__ int32_t* HeavyIndex(const BatchView& Bt, int fill_no, int nseg) {
  return Bt.heavy_index + static_cast<long long>(fill_no & 1) * Bt.B * nseg;
}

// A logit layout whose EOS column lies among the regular ids needs the EOS
// bit in that column's segment: when the built slot's EOS is context-
// dependent, that segment is heavy too (its item walks EOS on the stack, so
// the split step's accept must wait for it; EosBitOf).  0 otherwise.
__device__ __forceinline__ uint32_t EosSegExtra(const CacheView& Cc, int slot) {
  if (!Cc.eos_segbit) return 0u;
  return (__ldcg(Cc.cdb + static_cast<long long>(slot) * Cc.W + Cc.eos_word) & Cc.eos_bit) ? Cc.eos_segbit : 0u;
}

// Segments of sequence b the next fill should schedule first: those with
// context-dependent tokens (walks) or a pending build (waits).
__device__ uint32_t HeavyMask(const CacheView& Cc, int flagged, int nseg) {
  if (flagged < 0) return 0u;
  const uint32_t all = nseg >= 32 ? 0xffffffffu : ((1u << nseg) - 1u);
  if ((flagged & kSlotWait) || (flagged & ~kSlotWait) >= Cc.C) return all;
  return (LoadRelaxed(Cc.cd_segmask + (flagged & ~kSlotWait)) | EosSegExtra(Cc, flagged & ~kSlotWait)) & all;
}

// Appends b's heavy segments to queue q's heavy list and records, for every
// segment of b, its heavy-list index or -1 (exactly-once scheduling even when
// two lookup passes feed one queue).  `lane`/`nl` split the stores over a warp.
__device__ void PublishHeavy(const BatchView& Bt, int q, int tag, int b, uint32_t mask, int nseg, int lane,
                             int nl) {
  unsigned int base = 0;
  if (lane == 0 && mask) base = atomicAdd(QueueOf(Bt, q).n_heavy, static_cast<unsigned int>(__popc(mask)));
  if (nl > 1) base = __shfl_sync(0xffffffffu, base, 0);
  const BuildQueue Q = QueueOf(Bt, q);
  for (int s = lane; s < nseg; s += nl) {
    int idx = -1;
    if (s < 32 && ((mask >> s) & 1u)) {
      const unsigned int k = base + static_cast<unsigned int>(__popc(mask & ((1u << s) - 1u)));
      if (k < static_cast<unsigned int>(Bt.h_cap)) {
        Q.heavy[k] = make_int2(b, s);
        idx = HeavyTag(tag, static_cast<int>(k));
      }
    }
    HeavyIndex(Bt, tag, nseg)[static_cast<long long>(b) * nseg + s] = idx;
  }
  if (lane == 0) SeqHmask(Bt, tag)[b] = mask;
}

// Bounded wait (one thread) for the build of (slot, seg).  Units of this
// batch's queue were all dequeued by running CTAs before any fill item got
// here, so they finish; a slot whose build sits in another batch's queue may
// not, so the wait gives up after 2 ms and the caller fills directly.
__device__ bool WaitBuilt(const CacheView& Cc, const BatchView& Bt, int slot, int seg, int nseg) {
  const int* done = slot < Cc.C ? Cc.seg_done + static_cast<long long>(slot) * nseg + seg
                                : Bt.priv_done + static_cast<long long>(slot - Cc.C) * nseg + seg;
  bool ok = LoadAcquire(done) >= kChunksPerSeg;
  if (!ok) {
    unsigned long long t_start, t_now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    do {
      __nanosleep(256);
      ok = LoadAcquire(done) >= kChunksPerSeg;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
    } while (!ok && t_now - t_start < 2000000ull);
  }
  return ok;
}

// ---------------------------------------------------------------------------
// Build unit: 256 tokens of one (slot, segment) item, one per thread.
// ---------------------------------------------------------------------------
__device__ void BuildUnit(const AutView& A, const VocabView& Vv, const CacheView& Cc, const BatchView& Bt,
                          const int4 it, int chunk, int32_t* base_s, int* sh_flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int slot = it.x, seg = it.y, b = it.z;
  const bool priv = slot >= Cc.C;
  const unsigned long long t_in = Bt.trace ? NowNs() : 0ull;
  int nb;
  bool complete;
  // Incremental build from the parent context (the same stack top keyed R
  // deep): every token the parent decided keeps its verdict (its walk never
  // looked below the top R entries the child key shares); only the parent's
  // context-dependent tokens are walked with the child's deeper key.
  // A parent whose segment is not built yet (new in the same step) is not
  // waited for: blocking a CTA on another unit's progress costs more than
  // walking this unit's 256 tokens in full.
  int parent = priv ? -1 : __ldcg(Cc.slot_parent + slot);
  if (parent >= 0 && LoadAcquire(Cc.seg_done + static_cast<long long>(parent) * Vv.nseg + seg) < kChunksPerSeg) {
    parent = -1;
  }
  (void)sh_flag;
  __syncthreads();  // base_s reuse
  if (priv) {
    // Private row: the sequence's whole current stack (always complete).
    nb = Bt.seq[b].depth;
    complete = true;
    const int32_t* stack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
    for (int i = tid; i < nb; i += kThreads) base_s[i] = stack[i];
  } else {
    // Shared slot: its stored key (top first), independent of any stack.
    const int meta = __ldcg(Cc.slot_meta + slot);
    nb = meta & 0xff;
    complete = (meta >> 8) & 1;
    for (int i = tid; i < nb; i += kThreads) base_s[i] = __ldcg(Cc.slot_keys + slot * kMaxContext + (nb - 1 - i));
  }
  __syncthreads();
  const int t = seg * kSegTokens + chunk * kThreads + tid;
  int r = kReject;
  if (t <= Vv.V) {
    if (parent >= 0) {
      const uint32_t pcd = __ldcg(Cc.cdb + static_cast<long long>(parent) * Vv.W + (t >> 5));
      const uint32_t pci = __ldcg(Cc.ci + static_cast<long long>(parent) * Vv.W + (t >> 5));
      if ((pcd >> (t & 31)) & 1u) r = WalkToken(A, Vv, t, base_s, nb, complete);
      else r = ((pci >> (t & 31)) & 1u) ? kAccept : kReject;
    } else {
      r = WalkToken(A, Vv, t, base_s, nb, complete);
    }
  }
  const unsigned acc = __ballot_sync(0xffffffffu, r == kAccept);
  const unsigned cd = __ballot_sync(0xffffffffu, r == kUnknown);
  if (__any_sync(0xffffffffu, r == kOverflow) && lane == 0) atomicOr(Bt.err, 1u);
  const int w = seg * kSegWords + chunk * (kThreads / 32) + warp;
  if (lane == 0 && w < Vv.W) {
    if (priv) {
      Bt.priv[static_cast<long long>(slot - Cc.C) * Vv.W + w] = acc;
    } else {
      Cc.ci[static_cast<long long>(slot) * Vv.W + w] = acc;
      Cc.cdb[static_cast<long long>(slot) * Vv.W + w] = cd;
      // The segment's sampler counts of the CI bits (EOS excluded), the
      // counts of a pure-CI mask (LightItem, AcceptKernel's ci_shortcut).
      const uint32_t a = w == (Vv.V >> 5) ? acc & ~(1u << (Vv.V & 31)) : acc;
      const int2 n = make_int2(__popc(a), __popc(a & __ldg(Vv.structural + w)));
      int32_t* cnt = Cc.ci_cnt + (static_cast<long long>(slot) * Vv.nseg + seg) * 2;
      if (n.x) atomicAdd(cnt, n.x);
      if (n.y) atomicAdd(cnt + 1, n.y);
      if (cd) {
        atomicAdd(Cc.cd_cnt + static_cast<long long>(slot) * Vv.nseg + seg, __popc(cd));
        if (seg < 32) atomicOr(Cc.cd_segmask + slot, 1u << seg);
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    int* done = priv ? Bt.priv_done + static_cast<long long>(b) * Vv.nseg + seg
                     : Cc.seg_done + static_cast<long long>(slot) * Vv.nseg + seg;
    atomicAdd(done, 1);
    if (!priv) atomicAdd(Cc.slot_built + slot, 1);
    TraceEvent(Bt, 5, slot, seg, t_in, static_cast<unsigned long long>(parent >= 0));
  }
}

// Drains build queue q (CTA-cooperative).  Items were appended by earlier
// launches, so the count is final here.
__device__ void HelpBuild(const AutView& A, const VocabView& Vv, const CacheView& Cc, const BatchView& Bt, int q,
                          int32_t* base_s, int* sh_unit, int max_units = -1) {
  const BuildQueue Q = QueueOf(Bt, q);
  const unsigned int n_items = LoadRelaxed(Q.n_items);
  if (n_items == 0) return;
  const unsigned int units = n_items * kChunksPerSeg;
  for (int done = 0; max_units < 0 || done < max_units; ++done) {
    if (threadIdx.x == 0) *sh_unit = static_cast<int>(atomicAdd(Q.next_unit, 1u));
    __syncthreads();
    const unsigned int u = static_cast<unsigned int>(*sh_unit);
    __syncthreads();
    if (u >= units) break;
    const int4 it = Q.items[u / kChunksPerSeg];
    int chunk = static_cast<int>(u % kChunksPerSeg);
    if (it.x < Cc.C) {
      // A shared slot's chunks go to whoever claims them first (this queue's
      // units or a helper, HelpSegment): a unit whose claim comes too late
      // has nothing left to build.
      if (threadIdx.x == 0) *sh_unit = atomicAdd(Cc.seg_claim + static_cast<long long>(it.x) * Vv.nseg + it.y, 1);
      __syncthreads();
      chunk = *sh_unit;
      __syncthreads();
      if (chunk >= kChunksPerSeg) continue;
    }
    BuildUnit(A, Vv, Cc, Bt, it, chunk, base_s, sh_unit);
  }
}

// A CTA that needs (slot, seg) built now builds every chunk nobody has
// claimed yet, whichever batch's queue listed it (a batch that stopped
// stepping leaves its queued builds unclaimed; other batches must not wait
// on them).  Chunks claimed by others are being built by running CTAs, so
// the caller's bounded wait then completes.  CTA-cooperative.
__device__ void HelpSegment(const AutView& A, const VocabView& Vv, const CacheView& Cc, const BatchView& Bt, int slot,
                            int seg, int b, int32_t* base_s, int* sh_unit) {
  int* claim = Cc.seg_claim + static_cast<long long>(slot) * Vv.nseg + seg;
  for (;;) {
    if (threadIdx.x == 0) *sh_unit = LoadRelaxed(claim) < kChunksPerSeg ? atomicAdd(claim, 1) : kChunksPerSeg;
    __syncthreads();
    const int chunk = *sh_unit;
    __syncthreads();
    if (chunk >= kChunksPerSeg) break;
    BuildUnit(A, Vv, Cc, Bt, make_int4(slot, seg, b, 0), chunk, base_s, sh_unit);
  }
}

// ---------------------------------------------------------------------------
// Warp-level sampler + accept (+ lookup) of one sequence.  Everything here is
// a chain of dependent L2 round trips, so the code is arranged to issue each
// round trip's loads together: ~2 per token byte, 2 for the sampler, 2 for
// the context lookup.
// ---------------------------------------------------------------------------
// Synthetic stream; identical rule in oracle/gmask_port.c.
// Segment s's mask words and counts come from (row, counts) when bit s of
// `hm` is set, else from (crow, ccounts) — a sequence's context CI row and
// the slot's counts, equal to what the fill writes for its segments without
// context-dependent tokens (hm = ~0: everything from row/counts; segments >=
// 32 always are).
__device__ int SampleStreamWarp(const VocabView& Vv, int b, const uint32_t* row, const int32_t* counts,
                                const uint32_t* crow, const int32_t* ccounts, uint32_t hm,
                                unsigned long long seed, uint32_t draw, int lane) {
  // Round trip 1: the per-segment counts (segments 0..31 stay in registers)
  // and the EOS word.
  int c_all = 0, c_str = 0;
  if (lane < Vv.nseg) {
    const int32_t* src = ((hm >> lane) & 1u) ? counts : ccounts;
    const int2 v = __ldcg(reinterpret_cast<const int2*>(src) + lane);
    c_all = v.x;
    c_str = v.y;
  }
  const int eos_seg = (Vv.V >> 5) / kSegWords;
  const uint32_t eos_word = __ldcg((eos_seg >= 32 || ((hm >> eos_seg) & 1u) ? row : crow) + (Vv.V >> 5));
  int na = c_all, ns = c_str;
  for (int s = lane + 32; s < Vv.nseg; s += 32) {
    na += __ldcg(counts + 2 * s);
    ns += __ldcg(counts + 2 * s + 1);
  }
  na = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(na)));
  ns = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(ns)));
  const bool eos = (eos_word >> (Vv.V & 31)) & 1u;
  const unsigned long long u =
      Mix64(Mix64(seed ^ (static_cast<unsigned long long>(b) * 0xD1B54A32D192ED03ull)) ^
            static_cast<unsigned long long>(draw));
  if (na == 0) return eos ? Vv.V : -1;
  if (eos && ((u >> 32) & 3ull) == 0) return Vv.V;  // EOS with probability 1/4
  const bool use_s = ((u >> 34) & 1ull) && ns > 0;
  const uint32_t nsel = static_cast<uint32_t>(use_s ? ns : na);
  uint32_t r = static_cast<uint32_t>((static_cast<unsigned long long>(static_cast<uint32_t>(u)) * nsel) >> 32);
  // Segment holding the r-th selected token: warp prefix sum over the
  // per-segment counts, 32 segments per round.
  int seg = -1;
  for (int s0 = 0; s0 < Vv.nseg && seg < 0; s0 += 32) {
    const int s = s0 + lane;
    int c = use_s ? c_str : c_all;
    if (s0 > 0) c = s < Vv.nseg ? __ldcg(counts + 2 * s + (use_s ? 1 : 0)) : 0;
    const int inc = WarpInclusiveScan(c, lane);
    const int total = __shfl_sync(0xffffffffu, inc, 31);
    if (r < static_cast<uint32_t>(total)) {
      const int src = __ffs(__ballot_sync(0xffffffffu, static_cast<uint32_t>(inc) > r)) - 1;
      seg = s0 + src;
      r -= static_cast<uint32_t>(__shfl_sync(0xffffffffu, inc - c, src));
    } else {
      r -= static_cast<uint32_t>(total);
    }
  }
  if (seg < 0) return -1;
  // Round trip 2: all of the segment's words (and structural words); lane l
  // holds words 8l..8l+7 of the segment, so one warp scan of the per-lane
  // counts finds the lane, which finds the word and bit alone.
  const int w0 = seg * kSegWords;
  const int w1 = min(Vv.W, w0 + kSegWords);
  const uint32_t* wsrc = (seg >= 32 || ((hm >> seg) & 1u)) ? row : crow;
  uint32_t xs[kSegWords / 32];
  int c = 0;
#pragma unroll
  for (int j = 0; j < kSegWords / 32; ++j) {
    const int w = w0 + lane * (kSegWords / 32) + j;
    uint32_t x = 0;
    if (w < w1) {
      x = __ldcg(wsrc + w);
      if (w == (Vv.V >> 5)) x &= ~(1u << (Vv.V & 31));
      if (use_s) x &= __ldg(Vv.structural + w);
    }
    xs[j] = x;
    c += __popc(x);
  }
  const int inc = WarpInclusiveScan(c, lane);
  const int total = __shfl_sync(0xffffffffu, inc, 31);
  if (r >= static_cast<uint32_t>(total)) return -1;
  const int src = __ffs(__ballot_sync(0xffffffffu, static_cast<uint32_t>(inc) > r)) - 1;
  int tok = -1;
  if (lane == src) {
    uint32_t rr = r - static_cast<uint32_t>(inc - c);
#pragma unroll
    for (int j = 0; j < kSegWords / 32; ++j) {
      const uint32_t pc = static_cast<uint32_t>(__popc(xs[j]));
      if (tok < 0 && rr < pc) tok = (w0 + lane * (kSegWords / 32) + j) * 32 + static_cast<int>(__fns(xs[j], 0, rr + 1));
      if (tok < 0) rr -= pc;
    }
  }
  return __shfl_sync(0xffffffffu, tok, src);
}

// Warp-cooperative LookupSlot: same index protocol (64 linear probes from
// the key hash; insert = claim the position, pop a row, key row + meta, then
// publish tag | row, release), but 32 probes are read in one round trip and
// a hit is verified — key row, meta, build progress and CD segment mask — in
// one more.  `kv` = key entry `lane` (lanes < n).  Returns the row (-1: no
// free row, or the key is being published right now); *created when this
// warp inserted it; *built / *segmask of an existing row.
__device__ int LookupSlotWarp(const CacheView& C, int kv, int n, int complete, int lane, bool* created, int* built,
                              uint32_t* segmask) {
  const unsigned long long h = KeyHashWarp(kv, n, complete, lane);
  const unsigned long long tag = EntryTag(h);
  const int meta_want = n | (complete << 8) | (1 << 16);
  *created = false;
  const unsigned long long imask = static_cast<unsigned long long>(C.IC - 1);
  for (int base = 0; base < 64; base += 32) {
    for (int attempt = 0; attempt < 8; ++attempt) {  // re-read a window after a lost insert race
      const int i = static_cast<int>((h + static_cast<unsigned long long>(base + lane)) & imask);
      const unsigned long long cur = LoadRelaxed(C.slot_hash + i);
      const unsigned hit = __ballot_sync(0xffffffffu, (cur & ~kRowMask) == tag);
      const unsigned empty = __ballot_sync(0xffffffffu, cur == 0ull);
      unsigned cand = hit & (empty ? ((1u << (__ffs(empty) - 1)) - 1u) : 0xffffffffu);
      while (cand) {
        const int src = __ffs(cand) - 1;
        cand &= cand - 1;
        unsigned long long e = __shfl_sync(0xffffffffu, cur, src);
        if ((e & kRowMask) == static_cast<unsigned long long>(kRowPending)) {  // being published right now
          if (lane == 0) e = WaitPublished(C, static_cast<int>((h + static_cast<unsigned long long>(base + src)) & imask), e);
          e = __shfl_sync(0xffffffffu, e, 0);
          if ((e & ~kRowMask) != tag || (e & kRowMask) == static_cast<unsigned long long>(kRowPending)) return -1;
        }
        const int row = static_cast<int>(e & kRowMask);
        // Key row (lane i = entry i), meta, build progress, CD segments: one
        // round trip (the last three are warp-broadcast loads; the row id
        // they index arrived with the published entry).
        const int v = lane < n ? __ldcg(C.slot_keys + row * kMaxContext + lane) : 0;
        const int m = LoadAcquire(C.slot_meta + row);
        const int bt = LoadAcquire(C.slot_built + row);
        const int sm = static_cast<int>(LoadRelaxed(C.cd_segmask + row));
        if ((m & 0x1ffff) != meta_want) continue;
        if (__all_sync(0xffffffffu, lane >= n || v == kv)) {
          if (lane == 0) C.row_ref[row] = 1;
          *built = bt;
          *segmask = static_cast<uint32_t>(sm);
          return row;
        }
      }
      if (!empty) break;  // no free position in this window: probe the next one
      const int src = __ffs(empty) - 1;
      const int pos = static_cast<int>((h + static_cast<unsigned long long>(base + src)) & imask);
      int row = -1;
      if (lane == 0) {
        row = atomicCAS(C.slot_hash + pos, 0ull, tag | static_cast<unsigned long long>(kRowPending)) == 0ull ? -3 : -1;
        if (row == -3) {
          row = PopRow(C);
          if (row < 0) {
            StoreRelease(C.slot_hash + pos, 0ull);  // withdraw the claim: the table is full
            row = -2;
          }
        }
      }
      row = __shfl_sync(0xffffffffu, row, 0);
      if (row == -2) return -1;
      if (row >= 0) {
        if (lane < kMaxContext) C.slot_keys[row * kMaxContext + lane] = lane < n ? kv : -1;
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          atomic_i32 meta(C.slot_meta[row]);
          meta.store(meta_want, cuda::memory_order_release);
          C.row_ref[row] = 1;
          atomicAdd(C.counters + 0, 1ull);
          StoreRelease(C.slot_hash + pos, tag | static_cast<unsigned long long>(row));
        }
        *created = true;
        return row;
      }
    }
  }
  return -1;
}

// AssignSlotKey for a warp: the context slot of sequence b for the next fill
// (seq_slot[b]); a new shared slot or a private row queues one build item per
// segment into queue q.  Returns the segments the next fill must schedule in
// its heavy pass (CD tokens or a pending build).
__device__ uint32_t AssignSlotWarp(const CacheView& Cc, const BatchView& Bt, int q, int tag, int b,
                                   const SeqState& st, int nseg, int kv, int lane) {
  int32_t* slot_out = SeqSlot(Bt, tag) + b;
  if (st.status != kAlive) {
    if (lane == 0) *slot_out = -2;
    return 0u;
  }
  const int n = min(st.depth, Cc.K);
  const int complete = st.depth <= Cc.K ? 1 : 0;
  bool created = false;
  int built = 0;
  uint32_t segmask = 0u;
  int slot = LookupSlotWarp(Cc, kv, n, complete, lane, &created, &built, &segmask);
  bool wait = true;
  if (slot < 0 || created) {
    // Slots are never reused, so a new slot's counters are still zero.
    const BuildQueue Q = QueueOf(Bt, q);
    if (slot < 0) {
      slot = Cc.C + b;
      for (int s = lane; s < nseg; s += 32) Bt.priv_done[static_cast<long long>(b) * nseg + s] = 0;
      __threadfence();  // zeroed counters visible before the items
      __syncwarp();
      if (lane == 0) atomicAdd(Cc.counters + 2, 1ull);
    } else {
      if (lane == 0) atomicAdd(Cc.counters + 1, static_cast<unsigned long long>(nseg));
      if (Cc.R > 0 && n > Cc.R) {
        // Parent: the same top keyed R deep (queued first, so its units are
        // dequeued before the child's); the child walks only its CD tokens.
        bool pc = false;
        int pbuilt = 0;
        uint32_t psm = 0u;
        const int parent = LookupSlotWarp(Cc, kv, Cc.R, 0, lane, &pc, &pbuilt, &psm);
        if (pc) {
          unsigned int pat = 0;
          if (lane == 0) {
            atomicAdd(Cc.counters + 1, static_cast<unsigned long long>(nseg));
            pat = atomicAdd(Q.n_items, static_cast<unsigned int>(nseg));
          }
          pat = __shfl_sync(0xffffffffu, pat, 0);
          for (int s = lane; s < nseg; s += 32) Q.items[pat + s] = make_int4(parent, s, b, 0);
        }
        if (lane == 0) {
          Cc.slot_parent[slot] = parent;
          if (parent >= 0) atomicAdd(Cc.counters + 3, 1ull);
        }
        __threadfence();  // parent link visible before the child's items
        __syncwarp();
      }
    }
    unsigned int at = 0;
    if (lane == 0) at = atomicAdd(Q.n_items, static_cast<unsigned int>(nseg));
    at = __shfl_sync(0xffffffffu, at, 0);
    for (int s = lane; s < nseg; s += 32) Q.items[at + s] = make_int4(slot, s, b, 0);
  } else {
    // Existing slot: only one whose build is still queued needs a wait.
    wait = built < nseg * kChunksPerSeg;
  }
  if (lane == 0) *slot_out = slot | (wait ? kSlotWait : 0);
  const uint32_t all = nseg >= 32 ? 0xffffffffu : ((1u << nseg) - 1u);
  return (wait || slot >= Cc.C) ? all : ((segmask | EosSegExtra(Cc, slot)) & all);
}

// Engine::Step over the bytes of `tok` (EOS = V) on the device stack
// (runtime.cpp:177-186), one warp; then optional restart and (lookup_queue
// >= 0) the context slot of the next fill.
//  * Stack window: lane j holds entry j from the top for j < wv; after each
//    Step the new window is rebuilt by shuffles from the pushed entries and
//    the surviving old entries, so the stack is written but never re-read in
//    the common case (conditions reaching past the window read HBM).
//  * FindEdge (runtime.cpp:138-146): lanes test candidate edges in
//    arbitration order, 32 per round; each candidate lane loads its record,
//    condition list and first four pushed states in one round trip; the
//    winner's fields are broadcast by shuffles (Apply, runtime.cpp:148-168).
// Stack window of sequence b (lane j = entry j from the top, -1 below the
// bottom): AcceptWarp's starting registers, loadable ahead of the sample.
__device__ __forceinline__ int StackWindow(const BatchView& Bt, int b, int depth, int lane) {
  return lane < depth ? Bt.stacks[static_cast<long long>(b) * Bt.cap + depth - 1 - lane] : -1;
}

__device__ void AcceptWarp(const AutView& A, const VocabView& Vv, const CacheView& Cc, const BatchView& Bt, int b,
                           SeqState st, int topv, int tok, int32_t* status_out, int restart, int lookup_queue,
                           int lookup_tag, int lane) {
  int32_t* stack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
  unsigned long long t_ph = Bt.trace ? NowNs() : 0ull;
  int depth = st.depth;
  int wv = min(depth, 32);
  if (tok > Vv.V && st.status == kAlive) {
    st.status = kDead;  // not a token of this vocabulary (ids 0..V-1, EOS = V)
  } else if (tok >= 0 && st.status == kAlive) {
    const bool eos = tok == Vv.V;
    const int4 tr = __ldg(Vv.tok_rec + tok);
    const int nterm = tr.y;
    if (nterm == 0) st.status = kDead;  // a disabled id: never allowed (the loop below is skipped)
    const uint8_t* bytes = Vv.tok_bytes + tr.x;
    const int xb = TokLaneByte(tr, Vv.tok_bytes, lane, nterm, eos);
    for (int i = 0; i < nterm; ++i) {
      const int xs = __shfl_sync(0xffffffffu, xb, i & 31);
      const int x = eos ? 256 : (i < 32 ? xs : static_cast<int>(__ldg(bytes + i)));
      const int state = __shfl_sync(0xffffffffu, topv, 0);
      const int idx = state * 257 + x;
      const int cb = __ldg(A.rec_begin + idx);
      const int ce = __ldg(A.rec_begin + idx + 1);
      int win = -1;
      Rec r;
      r.cond_len = 0;
      r.push_len = 0;
      if (lane == 0) r = LoadRec(A.first + idx);  // same round trip as the range
      // Round 0: the first candidate (lane 0); then the rest, 32 per round.
      for (int cbase = cb, round = 0; cbase < ce; cbase = round == 1 ? cb + 1 : cbase + 32) {
        const int c = round == 0 ? (lane == 0 ? cb : ce) : cbase + lane;
        if (round++ > 0) {
          r.cond_len = 0;
          r.push_len = 0;
          if (c < ce) r = LoadRec(A.recs + c);
        }
        bool match = c < ce && r.cond_len <= depth;
        bool far = false;  // condition entries outside the register window
        // Entries 1..16 against the window, up to the longest live condition.
        const int jmax = static_cast<int>(__reduce_max_sync(0xffffffffu, match ? static_cast<unsigned>(r.cond_len) : 1u));
#pragma unroll
        for (int j = 1; j <= 16; ++j) {
          if (j >= jmax) break;
          const int have = __shfl_sync(0xffffffffu, topv, j);
          if (j < r.cond_len) {
            if (j < wv) {
              if (have != Lane4(r.c[(j - 1) >> 2], (j - 1) & 3)) match = false;
            } else {
              far = true;
            }
          }
        }
        if (match && (far || r.cond_len > 17)) {
          for (int j = 1; j < r.cond_len && match; ++j) {
            if (j <= 16 && j < wv) continue;
            match = stack[depth - 1 - j] == __ldg(A.rec_cond + r.cond_off + j - 1);
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, match);
        if (m) {
          win = __ffs(m) - 1;
          break;
        }
      }
      if (win < 0) {
        st.status = kDead;  // earlier bytes stay applied (runtime.cpp:179-183)
        break;
      }
      const int cond_len = __shfl_sync(0xffffffffu, static_cast<int>(r.cond_len), win);
      const int push_len = __shfl_sync(0xffffffffu, static_cast<int>(r.push_len), win);
      const int push_off = __shfl_sync(0xffffffffu, r.push_off, win);
      const int dyn = __shfl_sync(0xffffffffu, r.new_state, win) < 0 ? 1 : 0;
      const int p0 = __shfl_sync(0xffffffffu, r.p.x, win);
      const int p1 = __shfl_sync(0xffffffffu, r.p.y, win);
      const int p2 = __shfl_sync(0xffffffffu, r.p.z, win);
      const int p3 = __shfl_sync(0xffffffffu, r.p.w, win);
      const int base = depth - cond_len;
      const int P = push_len + dyn;
      const int nd = base + P;
      if (nd > Bt.cap) {
        st.status = kStackOverflow;
        break;
      }
      if (dyn && base + push_len == 0) {
        st.status = kDead;  // no exposed top: unreachable for validated automata
        break;
      }
      if (P > 32) {
        // Very long push (not produced by the fixture or workload grammars):
        // write through memory and reload the window.
        for (int j = lane; j < push_len; j += 32) stack[base + j] = __ldg(A.rec_push + push_off + j);
        __syncwarp();
        int tgt = 0;
        if (dyn) tgt = __ldg(A.shift + stack[base + push_len - 1] * 256 + x);
        if (tgt < 0) {
          st.status = kDead;  // no shift target (the mask walk rejects it too)
          break;
        }
        if (dyn && lane == 0) stack[base + push_len] = tgt;
        __syncwarp();
        topv = lane < nd ? stack[nd - 1 - lane] : -1;
        wv = min(nd, 32);
      } else {
        int pj = -1;  // pushed entry `lane` (bottom first)
        if (lane < push_len) {
          pj = lane == 0 ? p0 : lane == 1 ? p1 : lane == 2 ? p2 : lane == 3 ? p3 : __ldg(A.rec_push + push_off + lane);
        }
        if (dyn) {
          // Dynamic target from the exposed top (optimizer.cpp:33-76).
          const int last_pushed = __shfl_sync(0xffffffffu, pj, (push_len - 1) & 31);
          const int below = __shfl_sync(0xffffffffu, topv, cond_len & 31);
          int top = push_len > 0 ? last_pushed : (cond_len < wv ? below : -1);
          if (top < 0) top = stack[base - 1];
          const int tgt = __ldg(A.shift + top * 256 + x);
          if (tgt < 0) {
            st.status = kDead;  // no shift target (the mask walk rejects it too)
            break;
          }
          if (lane == push_len) pj = tgt;
        }
        if (lane < P) stack[base + lane] = pj;
        const int k = cond_len + lane - P;  // old window index of new entry `lane`
        const int old = __shfl_sync(0xffffffffu, topv, k & 31);
        const int pushed = __shfl_sync(0xffffffffu, pj, (P - 1 - lane) & 31);
        topv = lane < P ? pushed : (k < wv ? old : -1);
        wv = min(32, P + max(0, wv - cond_len));
        __syncwarp();  // stack writes visible to the warp's later reads
      }
      depth = nd;
      if (eos) st.status = kAccepted;
    }
    st.depth = depth;
  }
  if (status_out != nullptr && lane == 0) status_out[b] = st.status;
  // restart 1: finished sequences (accepted, dead, overflow) start over;
  // 2 (a sampled token): so does a dead end — no allowed token and no EOS
  // (tok < 0), like the decode loops of the oracle (gmask_port.c gp_decode_run).
  if (restart && (st.status != kAlive || (restart == 2 && tok < 0))) {
    if (lane == 0) {
      stack[0] = A.initial;
      atomicAdd(Bt.counters + 0, 1ull);
    }
    st.depth = 1;
    st.status = kAlive;
    topv = lane == 0 ? A.initial : -1;
    wv = 1;
  }
  __syncwarp();
  if (lane == 0 && Bt.trace) TraceEvent(Bt, 20, b, 0, t_ph, 0), t_ph = NowNs();
  if (lane == 0) {
    Bt.seq[b] = st;
    atomicAdd(Bt.counters + 3, 1ull);
  }
  if (lookup_queue >= 0) {
    // Key of the next fill's context: lane i holds entry i.
    const int n = st.status == kAlive ? min(st.depth, Cc.K) : 0;
    int kv = topv;
    if (n > wv) kv = lane < n ? stack[st.depth - 1 - lane] : 0;
    const uint32_t mask = AssignSlotWarp(Cc, Bt, lookup_queue, lookup_tag, b, st, Vv.nseg, kv, lane);
    if (lane == 0 && Bt.trace) TraceEvent(Bt, 21, b, 0, t_ph, 0), t_ph = NowNs();
    PublishHeavy(Bt, lookup_queue, lookup_tag, b, mask, Vv.nseg, lane, 32);
    if (lane == 0 && Bt.trace) TraceEvent(Bt, 22, b, 0, t_ph, 0), t_ph = NowNs();
  }
}

}  // namespace

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) LookupKernel(CacheView Cc, BatchView Bt, int q, int tag) {
  PdlEnter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= Bt.B) return;
  const SeqState st = Bt.seq[b];
  const int32_t* stack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
  int32_t key[kMaxContext];
  const int n = st.status == kAlive ? min(st.depth, Cc.K) : 0;
  for (int i = 0; i < n; ++i) key[i] = stack[st.depth - 1 - i];
  const int flagged = AssignSlotKey(Cc, Bt, q, tag, b, st, Bt.nseg, key);
  PublishHeavy(Bt, q, tag, b, HeavyMask(Cc, flagged, Bt.nseg), Bt.nseg, 0, 1);
}

// Builds everything queued in q, then empties q (used when a batch goes away
// or before a standalone fill should not pay for builds).
__global__ void __launch_bounds__(kThreads) DrainKernel(AutView A, VocabView Vv, CacheView Cc, BatchView Bt, int q) {
  PdlEnter();
  extern __shared__ int32_t base_s[];
  __shared__ int unit;
  HelpBuild(A, Vv, Cc, Bt, q, base_s, &unit);
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(Bt.kernel_done, 1u) == gridDim.x - 1) {
    *QueueOf(Bt, q).n_items = 0u;
    *QueueOf(Bt, q).next_unit = 0u;
    *QueueOf(Bt, q).n_heavy = 0u;
    *Bt.kernel_done = 0u;
  }
}

// ---------------------------------------------------------------------------
// Defined with AcceptKernel below; the split step's fill runs it too.
template <int SAMPLE>
__device__ __forceinline__ void AcceptSeq(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                          const BatchView& Bt, const AcceptArgs& G, int b, int lane);

namespace {

constexpr int kWarps = kThreads / 32;     // light items per fill CTA
constexpr int kSpans = kSegWords / 32;    // 1024-token spans per segment

// m[i] for a loop-variable i without indexing the register array (a
// dynamic index would move it to local memory).
template <int N>
__device__ __forceinline__ uint32_t Pick(const uint32_t (&m)[N], int i) {
  uint32_t v = 0u;
#pragma unroll
  for (int k = 0; k < N; ++k) v = k == i ? m[k] : v;
  return v;
}

// Greedy key of bf16 bits at token t: order-preserving float key in the high
// word, 0xFFFFFFFF - t in the low word (ties -> lowest id).
__device__ __forceinline__ unsigned long long GreedyKey(uint16_t v, int t) {
  const uint32_t bits = static_cast<uint32_t>(v) << 16;
  const uint32_t key = (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
  return (static_cast<unsigned long long>(key) << 32) | static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(t));
}

// 16-bit order keys of the two bf16 logits in w (low half = lower token),
// 0 for a masked token (bits0/1 of `bits` = the two tokens' mask bits): key =
// h ^ 0xFFFF for a negative value, h ^ 0x8000 otherwise — the top half of
// GreedyKey's high word (Key32 restores it), so comparing keys compares
// values, and every allowed key is > 0 (the key 0x0000 would be a NaN with
// all payload bits set, 0xFFFF).
__device__ __forceinline__ uint32_t PairKeys(uint32_t w, uint32_t bits) {
  const uint32_t neg = ((w >> 15) & 0x00010001u) * 0x7FFFu;
  const uint32_t key = w ^ (0x80008000u | neg);
  const uint32_t keep = ((bits & 1u) ? 0x0000FFFFu : 0u) | ((bits & 2u) ? 0xFFFF0000u : 0u);
  return key & keep;
}
// GreedyKey's high word from a 16-bit key: (key << 16), low half all ones
// for a negative value (the complement of its zero low bits).
__device__ __forceinline__ uint32_t Key32(uint32_t k16) { return (k16 << 16) | ((k16 & 0x8000u) ? 0u : 0xFFFFu); }

// Mask byte of chunk c = 32k + lane of a 1024-token span whose 32 mask words
// are spread one per lane (`mword`): word c/4, byte c%4.
__device__ __forceinline__ void SpanBytes(uint32_t mword, int lane, uint32_t byte[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = 32 * k + lane;
    byte[k] = (__shfl_sync(0xffffffffu, mword, c >> 2) >> ((c & 3) * 8)) & 0xffu;
  }
}

// In-place bf16 -inf over the span [tw, tw + 1024) ∩ [.., t1): 4 rounds of
// 32 lanes x 16 B, each round one coalesced 512-B stretch of the row.  A fully
// masked chunk is one -inf store (no read); a mixed chunk is read, blended
// and written back whole (partial 2/4-B stores measured 1.5x slower: L2
// merges them sector by sector and still fetches the rest of each sector
// from HBM); an all-allowed chunk is skipped.
__device__ __forceinline__ void MaskSpan(uint16_t* row, int tw, int t1, bool vec_ok, uint32_t mword, int lane,
                                         unsigned* rd, unsigned* wr) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
  if (vec_ok && tw + 1024 <= t1) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (byte[k] != 0u && byte[k] != 0xffu) {
        v[k] = __ldcs(reinterpret_cast<const uint4*>(row + tw + (32 * k + lane) * 8));
        *rd += 16;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (byte[k] == 0xffu) continue;
      uint4 o = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
      if (byte[k] != 0u) {
        // keep-mask per 32-bit pair: low half <- bit 2j, high half <- bit 2j+1
        const uint32_t x = byte[k];
        uint32_t* po = reinterpret_cast<uint32_t*>(&o);
        const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t keep = ((x >> (2 * j)) & 1u ? 0x0000FFFFu : 0u) | ((x >> (2 * j + 1)) & 1u ? 0xFFFF0000u : 0u);
          po[j] = (pv[j] & keep) | (0xFF80FF80u & ~keep);
        }
      }
      __stcs(reinterpret_cast<uint4*>(row + tw + (32 * k + lane) * 8), o);
      *wr += 16;
    }
  } else {  // last (partial) span or unaligned rows: rare, kept compact
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int tb = tw + (32 * k + lane) * 8;
      if (byte[k] == 0xffu || tb >= t1) continue;
      const int valid = min(8, t1 - tb);
#pragma unroll 1
      for (int j = 0; j < valid; ++j) {
        if (!((byte[k] >> j) & 1u)) {
          row[tb + j] = 0xFF80u;
          *wr += 2;
        }
      }
    }
  }
}

// cp.async (LDGSTS) helpers: 16-B global -> shared copies that need no
// registers while in flight.
__device__ __forceinline__ void CpAsync16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void CpAsyncCommit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void CpAsyncWait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void CpAsyncWait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ unsigned LaneMaskLt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Bulk (TMA) shared -> global copies: one instruction stores a whole span of
// -inf from a CTA-shared source, L2 evict-first like the __stcs stores.
__device__ __forceinline__ unsigned long long EvictFirstPolicy() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void BulkStore(void* gmem, const void* smem, int bytes, unsigned long long policy) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
#if PRE3_BULK_EVICT_FIRST
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(gmem),
               "r"(sa), "r"(bytes), "l"(policy)
               : "memory");
#else
  (void)policy;
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem), "r"(sa), "r"(bytes)
               : "memory");
#endif
}
__device__ __forceinline__ void BulkCommit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void BulkWaitRead() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// Mixed chunks of a full span -> this lane's slots of a span buffer.
__device__ __forceinline__ void SpanPrefetch(const uint16_t* row, int tw, uint32_t mword, int lane,
                                             uint4 (*buf)[32]) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (byte[k] != 0u && byte[k] != 0xffu) CpAsync16(&buf[k][lane], row + tw + (32 * k + lane) * 8);
  }
}

// Stores of a full span whose mixed chunks were prefetched into `buf`.
__device__ __forceinline__ void SpanStore(uint16_t* row, int tw, uint32_t mword, int lane, const uint4 (*buf)[32],
                                          unsigned* rd, unsigned* wr) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (byte[k] == 0xffu) continue;
    uint4 o = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    if (byte[k] != 0u) {
      const uint32_t x = byte[k];
      const uint4 v = buf[k][lane];
      uint32_t* po = reinterpret_cast<uint32_t*>(&o);
      const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t keep = ((x >> (2 * j)) & 1u ? 0x0000FFFFu : 0u) | ((x >> (2 * j + 1)) & 1u ? 0xFFFF0000u : 0u);
        po[j] = (pv[j] & keep) | (0xFF80FF80u & ~keep);
      }
      *rd += 16;
    }
    __stcs(reinterpret_cast<uint4*>(row + tw + (32 * k + lane) * 8), o);
    *wr += 16;
  }
}

// Chunks of a full span holding any allowed token -> this lane's slots of a
// span buffer (greedy argmax).
__device__ __forceinline__ void SpanPrefetchAllowed(const uint16_t* row, int tw, uint32_t mword, int lane,
                                                    uint4 (*buf)[32]) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (byte[k] != 0u) CpAsync16(&buf[k][lane], row + tw + (32 * k + lane) * 8);
  }
}

// This lane's best allowed (key, token) of a full span prefetched by
// SpanPrefetchAllowed (0 when none).
__device__ __forceinline__ unsigned long long ArgmaxBuffered(int tw, uint32_t mword, int lane,
                                                             const uint4 (*buf)[32], unsigned* rd) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
  unsigned long long mine = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!byte[k]) continue;
    const uint4 v = buf[k][lane];
    const uint16_t* pv = reinterpret_cast<const uint16_t*>(&v);
    const int tb = tw + (32 * k + lane) * 8;
    *rd += 16;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if ((byte[k] >> j) & 1u) {
        const unsigned long long p = GreedyKey(pv[j], tb + j);
        mine = p > mine ? p : mine;
      }
    }
  }
  return mine;
}

// The two 16-bit order keys of the bf16 pair w (low half = lower token):
// h ^ 0xFFFF for a negative value, h ^ 0x8000 otherwise (PRMT replicates
// each half's sign bit over the half).
__device__ __forceinline__ uint32_t PairOrderKeys(uint32_t w) {
  // prmt's generic mode (a selector nibble with its msb set replicates the
  // sign of the selected byte); __byte_perm masks that bit off.
  uint32_t sgn;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(sgn) : "r"(w));
  return w ^ (sgn | 0x80008000u);
}

// ArgmaxBuffered in 32-bit packed form: (16-bit order key << 16) |
// (0xFFFF - token offset in the segment), 0 when no allowed token — one max
// per token instead of 64-bit keys (an allowed key-0 token, bf16 0xFFFF, still
// packs above 0: offsets are < 8192).  Key32 + the offset restore GreedyKey.
__device__ __forceinline__ uint32_t ArgmaxBufferedPacked(int span_off, uint32_t mword, int lane,
                                                         const uint4 (*buf)[32], unsigned* rd) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
  uint32_t best = 0u;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (!byte[k]) continue;
    const uint4 v = buf[k][lane];
    const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v);
    const uint32_t c0 = 0xFFFFu - static_cast<uint32_t>(span_off + (32 * k + lane) * 8);  // token 0 of the chunk
    *rd += 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t key2 = PairOrderKeys(pv[j]);  // two 16-bit order keys
      const uint32_t lo = (key2 << 16) | (c0 - 2 * j);
      const uint32_t hi = (key2 & 0xFFFF0000u) | (c0 - 2 * j - 1);
      if ((byte[k] >> (2 * j)) & 1u) best = max(best, lo);
      if ((byte[k] >> (2 * j + 1)) & 1u) best = max(best, hi);
    }
  }
  return best;
}

// This lane's best allowed (key, token) of the span (0 when none).
__device__ __forceinline__ unsigned long long ArgmaxSpan(const uint16_t* row, int tw, int t1, bool vec_ok,
                                                         uint32_t mword, int lane, unsigned* rd) {
  uint32_t byte[4];
  SpanBytes(mword, lane, byte);
  unsigned long long mine = 0;
  if (vec_ok && tw + 1024 <= t1) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (byte[k]) {
        v[k] = __ldcs(reinterpret_cast<const uint4*>(row + tw + (32 * k + lane) * 8));
        *rd += 16;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!byte[k]) continue;
      const uint16_t* pv = reinterpret_cast<const uint16_t*>(&v[k]);
      const int tb = tw + (32 * k + lane) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((byte[k] >> j) & 1u) {
          const unsigned long long p = GreedyKey(pv[j], tb + j);
          mine = p > mine ? p : mine;
        }
      }
    }
  } else {  // last (partial) span or unaligned rows: rare, kept compact
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
      const int tb = tw + (32 * k + lane) * 8;
      if (!byte[k] || tb >= t1) continue;
      const int valid = min(8, t1 - tb);
#pragma unroll 1
      for (int j = 0; j < valid; ++j) {
        if ((byte[k] >> j) & 1u) {
          const unsigned long long p = GreedyKey(row[tb + j], tb + j);
          *rd += 2;
          mine = p > mine ? p : mine;
        }
      }
    }
  }
  return mine;
}

__device__ __forceinline__ unsigned long long WarpMax64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y > v ? y : v;
  }
  return v;
}

// The EOS bit (mask bit V) of sequence b for an item of another segment
// (logit layouts whose EOS column lies among the regular ids).  With a
// settled (built, shared) slot whose EOS is context-independent it is the
// slot's CI bit — no walk: the sequence's stack may already be changing under
// the overlapped accept, which waits only for its heavy segments.  Otherwise
// the accept waits for this item (a waiting or private slot makes every
// segment heavy; a context-dependent EOS makes the EOS column's segment heavy,
// EosSegExtra), so the stack is stable and EOS (one terminal) is walked on it —
// Step(kEndMarker) succeeds iff AllowedTerminals reports the end marker.
__device__ __forceinline__ int EosBitOf(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                        const BatchView& Bt, int b, int slot, bool settled) {
  if (settled && slot >= 0 && slot < Cc.C) {
    const long long w = static_cast<long long>(slot) * Vv.W + (Vv.V >> 5);
    if (!((__ldcg(Cc.cdb + w) >> (Vv.V & 31)) & 1u)) return static_cast<int>((__ldcg(Cc.ci + w) >> (Vv.V & 31)) & 1u);
  }
  const SeqState st = Bt.seq[b];
  if (st.status != kAlive) return 0;
  return WalkToken(A, Vv, Vv.V, Bt.stacks + static_cast<long long>(b) * Bt.cap, st.depth, true) == kAccept ? 1 : 0;
}

// Logit columns [V, ncols) of a model layout (specials, EOS column): -inf,
// except the EOS column when EOS is allowed.  Lanes stride the columns.
__device__ __forceinline__ void TailColumns(const VocabView& Vv, uint16_t* row, int eos_bit, int lane, int nlanes,
                                            unsigned* wr) {
  for (int c = Vv.V + lane; c < Vv.ncols; c += nlanes) {
    if (c == Vv.eos_col && eos_bit) continue;
    row[c] = 0xFF80u;
    *wr += 2;
  }
}

// The sequence's last finished fill item: sample (stream or greedy), accept,
// restart, and look up the next step's context slot.  One warp.
template <int TAIL>
__device__ __forceinline__ void SequenceTail(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                             const BatchView& Bt, const FillArgs& F, int b, int lane) {
  const unsigned long long t_in = Bt.trace ? NowNs() : 0ull;
  __threadfence();
  SeqState st = Bt.seq[b];
  int tok;
  if (TAIL == kTailGreedy) {
    const unsigned long long p = __ldcg(F.best + b);
    tok = p ? static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(p)) : -1;
    if (lane == 0) F.best[b] = 0ull;
  } else {
    const uint32_t* brow = F.bitmask + static_cast<long long>(b) * F.ldw;
    const int32_t* bcnt = F.seg_counts + static_cast<long long>(b) * Vv.nseg * 2;
    tok = SampleStreamWarp(Vv, b, brow, bcnt, brow, bcnt, ~0u, F.seed, st.draws, lane);
    st.draws += 1;
    if (lane == 0) atomicAdd(Bt.counters + 1, 1ull);
  }
  if (F.tokens_out != nullptr && lane == 0) F.tokens_out[b] = BitToId(Vv, tok);
  if (lane == 0) Bt.seq_arrive[b] = 0;
  AcceptWarp(A, Vv, Cc, Bt, b, st, StackWindow(Bt, b, st.depth, lane), tok, nullptr, 2, F.produce, NextFill(F.fill_no),
             lane);
  if (lane == 0) TraceEvent(Bt, kTraceTail, b, 0, t_in, static_cast<unsigned long long>(tok + 1));
}

// Light item: one warp fills one (sequence, segment) — the steady state (a
// ready context slot, few or no context-dependent tokens).  Lane j owns mask
// words j, 32+j, ..., 224+j of the segment (registers m[]); span i = words
// [32i, 32i+32) = tokens t0 + [1024i, 1024i+1024).  No CTA barriers.
// Split step in one grid (FillArgs::accept_ctas): the arrivals sequence b's
// accept needs — its heavy segments of a built shared slot, else every
// segment (AcceptSeq's ci_shortcut test; the fill's `publish`).  None: an
// accept CTA runs it; otherwise the item completing them does, so nothing
// in the grid ever waits for another CTA's items.
__device__ __forceinline__ int ArrivalsNeeded(const CacheView& Cc, const VocabView& Vv, int slot, uint32_t hmask) {
  if (slot >= 0 && slot < Cc.C && Vv.nseg <= 32) {
    const uint32_t all = Vv.nseg >= 32 ? 0xffffffffu : ((1u << Vv.nseg) - 1u);
    return __popc(hmask & all);
  }
  return Vv.nseg;
}

template <int MODE, int TAIL>
__device__ __forceinline__ void LightItem(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                          const BatchView& Bt, const FillArgs& F, int b, int seg, int slot,
                                          bool pure, bool publish, int need, int lane, uint4 (*span_buf)[4][32],
                                          const uint4* ninf) {
  const unsigned long long t_in = Bt.trace ? NowNs() : 0ull;
  const int w0 = seg * kSegWords;
  const int nwords = min(Vv.W - w0, kSegWords);
  const int t0 = w0 * 32;
  const int t1 = min(Vv.V + 1, t0 + nwords * 32);
  // Logit columns mapped 1:1 to mask bits (a model layout maps bit V to its
  // EOS column and masks the columns >= V itself, TailColumns).
  const int tl1 = Vv.layout ? min(Vv.V, t1) : t1;
  const bool last_seg = seg == Vv.nseg - 1;
  const bool eos_in_seg = Vv.layout && Vv.eos_col < Vv.V && Vv.eos_col >= t0 && Vv.eos_col < tl1;
  const bool wait = slot >= 0 && (slot & kSlotWait);
  if (slot >= 0) slot &= ~kSlotWait;
  if (wait) {
    int ok = 0;
    if (lane == 0) ok = WaitBuilt(Cc, Bt, slot, seg, Vv.nseg) ? 1 : 0;
    if (!__shfl_sync(0xffffffffu, ok, 0)) slot = -3;  // direct fill
  }
  uint32_t m[kSpans];
  int cd_cnt = 0;
  int2 pc = make_int2(0, 0);  // pure: the slot's counts of this segment
  if (slot >= 0) {
    const uint32_t* src = slot < Cc.C ? Cc.ci + static_cast<long long>(slot) * Vv.W
                                      : Bt.priv + static_cast<long long>(slot - Cc.C) * Vv.W;
#pragma unroll
    for (int i = 0; i < kSpans; ++i) {
      const int w = 32 * i + lane;
      m[i] = w < nwords ? __ldcg(src + w0 + w) : 0u;
    }
    if (pure) {
      pc = __ldcg(reinterpret_cast<const int2*>(Cc.ci_cnt) + static_cast<long long>(slot) * Vv.nseg + seg);
    } else if (slot < Cc.C) {
      cd_cnt = __ldcg(Cc.cd_cnt + static_cast<long long>(slot) * Vv.nseg + seg);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSpans; ++i) m[i] = 0u;
  }
  int n_walks = 0;
  if (slot == -3 || cd_cnt > 0) {
    // Rare in the light pass (the lookups list such segments for the heavy
    // pass; only a full heavy list lands them here): walk against the
    // sequence's stack in HBM.
    // m[] is parked in this warp's (still unused) span buffer during the
    // walks so no register array is live across the out-of-line walk calls.
    uint32_t* wbuf = reinterpret_cast<uint32_t*>(span_buf);
#pragma unroll
    for (int i = 0; i < kSpans; ++i) wbuf[32 * i + lane] = m[i];
    const int depth = Bt.seq[b].depth;
    const int32_t* gstack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
    const uint32_t* cdsrc = Cc.cdb + static_cast<long long>(slot) * Vv.W + w0;
#pragma unroll 1
    for (int i = 0; i < kSpans; ++i) {
      const int w = 32 * i + lane;
      uint32_t add = 0u;
      if (slot == -3) {
#pragma unroll 1
        for (int j = 0; j < 32; ++j) {  // word 32i+j: lane = bit
          const int t = t0 + (32 * i + j) * 32 + lane;
          const int r = t < t1 ? WalkToken(A, Vv, t, gstack, depth, true) : kReject;
          const unsigned acc = __ballot_sync(0xffffffffu, r == kAccept);
          if (__any_sync(0xffffffffu, r == kOverflow) && lane == 0) atomicOr(Bt.err, 1u);
          if (lane == j) add = acc;
        }
        n_walks += 32;
      } else {
        uint32_t x = w < nwords ? __ldcg(cdsrc + w) : 0u;
        n_walks += __popc(x);
        while (x) {
          const int bit = __ffs(x) - 1;
          x &= x - 1;
          const int r = WalkToken(A, Vv, t0 + w * 32 + bit, gstack, depth, true);
          if (r == kAccept) add |= 1u << bit;
          if (r == kOverflow) atomicOr(Bt.err, 1u);
        }
      }
      wbuf[32 * i + lane] |= add;  // lane-private word
    }
#pragma unroll
    for (int i = 0; i < kSpans; ++i) m[i] = wbuf[32 * i + lane];
    __syncwarp();  // the buffer is reused for logits chunks below
  }

  // ---- logits spans by class (MaskSpans): all allowed -> untouched, all
  // masked -> a bulk store, mixed -> the mixed chunks read, blended, stored.
  // The first two mixed spans' chunks are requested now, so their round trip
  // overlaps the bitmask and count stores and the bulk stores below (an EOS
  // column patched into this item's words waits until its bit is known).
  uint32_t masked = 0u, mixed = 0u, pend = 0u;
  const bool spans_early = MODE == kFillMask && F.logits != nullptr && !eos_in_seg;
  uint16_t* lrow = F.logits != nullptr ? F.logits + static_cast<long long>(b) * F.ld : nullptr;
  const int nfull = F.vec_ok ? (tl1 - t0) >> 10 : 0;
  auto classify = [&]() {
#pragma unroll
    for (int i = 0; i < kSpans; ++i) {
      const unsigned nz = __ballot_sync(0xffffffffu, m[i] != 0u);
      const unsigned nf = __ballot_sync(0xffffffffu, m[i] != 0xffffffffu);
      if (i < nfull) {
        if ((!nz || PRE3_DIAG_NO_MIXED) && PRE3_BULK_MASKED && ((PRE3_BULK_SPANS >> i) & 1)) masked |= 1u << i;
        else if (nf) mixed |= 1u << i;  // (a masked span left to the LSU path: -inf chunk stores)
      }
    }
  };
  auto prefetch2 = [&]() {  // the first two mixed spans -> the warp's span buffers 0, 1
    pend = mixed;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (pend) {
        const int i = __ffs(pend) - 1;
        pend &= pend - 1;
        SpanPrefetch(lrow, t0 + 1024 * i, Pick(m, i), lane, span_buf[q]);
      }
      CpAsyncCommit();
    }
  };
#if !PRE3_COMPACT_MIXED
  if (spans_early) {
    classify();
    prefetch2();
  }
#endif

  // ---- bitmask words and sampler counts (a pure item's are the slot's).
  const int eos_word = Vv.V >> 5;
  int ca = 0, cs = 0;
#pragma unroll
  for (int i = 0; i < kSpans; ++i) {
    const int w = 32 * i + lane;
    if (w < nwords) {
      if (F.bitmask != nullptr) F.bitmask[static_cast<long long>(b) * F.ldw + w0 + w] = m[i];
      if (F.seg_counts != nullptr && !pure) {
        uint32_t mm = m[i];
        if (w0 + w == eos_word) mm &= ~(1u << (Vv.V & 31));
        ca += __popc(mm);
        cs += __popc(mm & __ldg(Vv.structural + w0 + w));
      }
    }
  }
  if (F.seg_counts != nullptr) {
    if (pure) {
      ca = pc.x;
      cs = pc.y;
    } else {
      ca = WarpSum(ca);
      cs = WarpSum(cs);
    }
    if (lane == 0) {
      F.seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 0] = ca;
      F.seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 1] = cs;
    }
  }
  if (Bt.trace && lane == 0) TraceEvent(Bt, 14, b, seg, t_in, 0);  // l:head (slot, CI loads, bitmask, counts)
  // ---- model logit layout: the EOS bit where this item needs it (the last
  // segment holds bit V; an EOS column among the regular ids is patched into
  // this item's words for the logits pass below — bitmask rows keep the
  // reference layout).
  int eos_bit = 0;
  if (Vv.layout && (last_seg || eos_in_seg)) {
    if (last_seg) {
      const int we = (Vv.V >> 5) - w0;
      eos_bit = static_cast<int>((__shfl_sync(0xffffffffu, Pick(m, we >> 5), we & 31) >> (Vv.V & 31)) & 1u);
    } else {
      if (lane == 0) {
        // (the raw slot again, rather than keeping `wait` live across the item)
        const bool settled = !(SeqSlot(Bt, F.fill_no)[b] & kSlotWait);
        eos_bit = slot == -2 ? 0 : EosBitOf(A, Vv, Cc, Bt, b, slot, settled);
      }
      eos_bit = __shfl_sync(0xffffffffu, eos_bit, 0);
    }
  }
  unsigned rd = 0, wr = 0;  // this lane's logit bytes (stats)
  if (MODE == kFillGreedy) {
    // Argmax over the allowed entries: only 16-B chunks holding an allowed
    // token are read, two spans in flight (cp.async into the warp's span
    // buffer) so a span's round trip overlaps the previous span's compare.
    const uint16_t* row = F.logits + static_cast<long long>(b) * F.ld;
    unsigned long long mine = 0;
    const int nfull = F.vec_ok ? (tl1 - t0) >> 10 : 0;
    uint32_t live = 0u;
#pragma unroll
    for (int i = 0; i < kSpans; ++i) {
      if (i < nfull && __ballot_sync(0xffffffffu, m[i] != 0u)) live |= 1u << i;
    }
#if PRE3_COMPACT_GREEDY
    // Every 16-B chunk holding an allowed token, packed (span, round, lane)
    // into the warp's 256-chunk buffer and copied in ONE round trip; then the
    // max 16-bit order key two tokens at a time (__vmaxu2 over key pairs,
    // masked tokens key 0), a warp max, and the lowest id holding it.
    uint4* cbuf = &span_buf[0][0][0];
    const unsigned lt = LaneMaskLt();
#pragma unroll 1
    for (uint32_t todo = live; todo;) {
      uint32_t batch = 0u;
      int n = 0;
#pragma unroll 1
      for (uint32_t t = todo; t; t &= t - 1) {
        const int i = __ffs(t) - 1;
        uint32_t byte[4];
        SpanBytes(Pick(m, i), lane, byte);
        unsigned bal[4];
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          bal[k] = __ballot_sync(0xffffffffu, byte[k] != 0u);
          cnt += __popc(bal[k]);
        }
        if (n + cnt > 256) break;  // a span holds <= 128 chunks: a batch takes >= 1 span
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((bal[k] >> lane) & 1u) CpAsync16(&cbuf[n + __popc(bal[k] & lt)], row + t0 + 1024 * i + (32 * k + lane) * 8);
          n += __popc(bal[k]);
        }
        batch |= 1u << i;
      }
      CpAsyncCommit();
      CpAsyncWait0();
      // Pass 1: this lane's max key over its chunks of the batch.
      uint32_t acc = 0u;
      n = 0;
#pragma unroll 1
      for (uint32_t t = batch; t; t &= t - 1) {
        const int i = __ffs(t) - 1;
        uint32_t byte[4];
        SpanBytes(Pick(m, i), lane, byte);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const unsigned bal = __ballot_sync(0xffffffffu, byte[k] != 0u);
          if (byte[k] != 0u) {
            const uint4 v = cbuf[n + __popc(bal & lt)];
            const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc = __vmaxu2(acc, PairKeys(pv[j], byte[k] >> (2 * j)));
            }
            rd += 16;
          }
          n += __popc(bal);
        }
      }
      const uint32_t lmax = max(acc & 0xffffu, acc >> 16);
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, lmax);
      // Pass 2 (lanes holding kmax): the lowest token id with that key.
      uint32_t tmin = 0xffffffffu;
      if (kmax != 0u) {
        n = 0;
#pragma unroll 1
        for (uint32_t t = batch; t; t &= t - 1) {
          const int i = __ffs(t) - 1;
          uint32_t byte[4];
          SpanBytes(Pick(m, i), lane, byte);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const unsigned bal = __ballot_sync(0xffffffffu, byte[k] != 0u);
            if (lmax == kmax && byte[k] != 0u && tmin == 0xffffffffu) {
              const uint4 v = cbuf[n + __popc(bal & lt)];
              const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t kk = PairKeys(pv[j], byte[k] >> (2 * j));
                const uint32_t tb = static_cast<uint32_t>(t0 + 1024 * i + (32 * k + lane) * 8 + 2 * j);
                if (tmin == 0xffffffffu && (kk & 0xffffu) == kmax) tmin = tb;
                if (tmin == 0xffffffffu && (kk >> 16) == kmax) tmin = tb + 1;
              }
            }
            n += __popc(bal);
          }
        }
        tmin = __reduce_min_sync(0xffffffffu, tmin);
        const unsigned long long p = (static_cast<unsigned long long>(Key32(kmax)) << 32) |
                                     static_cast<unsigned long long>(0xFFFFFFFFu - tmin);
        mine = p > mine ? p : mine;
      } else if (n > 0) {
        // Only 0xFFFF NaNs allowed (their key is 0, like a masked token's):
        // the exact 64-bit keys, token by token.
        n = 0;
#pragma unroll 1
        for (uint32_t t = batch; t; t &= t - 1) {
          const int i = __ffs(t) - 1;
          uint32_t byte[4];
          SpanBytes(Pick(m, i), lane, byte);
#pragma unroll 1
          for (int k = 0; k < 4; ++k) {
            const unsigned bal = __ballot_sync(0xffffffffu, byte[k] != 0u);
            if (byte[k] != 0u) {
              const uint4 v = cbuf[n + __popc(bal & lt)];
              const uint16_t* ph = reinterpret_cast<const uint16_t*>(&v);
              for (int j = 0; j < 8; ++j) {
                if ((byte[k] >> j) & 1u) {
                  const unsigned long long p = GreedyKey(ph[j], t0 + 1024 * i + (32 * k + lane) * 8 + j);
                  mine = p > mine ? p : mine;
                }
              }
            }
            n += __popc(bal);
          }
        }
      }
      todo &= ~batch;
      __syncwarp();  // the buffer is refilled by the next batch
    }
#else
    uint4(*buf)[4][32] = span_buf;
    uint32_t pend = live;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (pend) {
        const int i = __ffs(pend) - 1;
        pend &= pend - 1;
        SpanPrefetchAllowed(row, t0 + 1024 * i, Pick(m, i), lane, buf[q]);
      }
      CpAsyncCommit();
    }
    int q = 0;
    uint32_t packed = 0u;  // ArgmaxBufferedPacked over the full spans
#pragma unroll 1
    for (uint32_t todo = live; todo; todo &= todo - 1, q ^= 1) {
      const int i = __ffs(todo) - 1;
      CpAsyncWait1();
      packed = max(packed, ArgmaxBufferedPacked(1024 * i, Pick(m, i), lane, buf[q], &rd));
      if (pend) {
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        SpanPrefetchAllowed(row, t0 + 1024 * j, Pick(m, j), lane, buf[q]);
      }
      CpAsyncCommit();
    }
    packed = __reduce_max_sync(0xffffffffu, packed);
    if (packed != 0u) {
      const int t = t0 + static_cast<int>(0xFFFFu - (packed & 0xFFFFu));
      mine = (static_cast<unsigned long long>(Key32(packed >> 16)) << 32) |
             static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<uint32_t>(t));
    }
#endif
#pragma unroll 1
    for (int i = nfull; i < kSpans; ++i) {
      const int tw = t0 + 1024 * i;
      if (tw >= tl1) break;
      const unsigned long long p = ArgmaxSpan(row, tw, tl1, F.vec_ok, Pick(m, i), lane, &rd);
      mine = p > mine ? p : mine;
    }
    if (Vv.layout && last_seg && eos_bit && lane == 0) {  // EOS competes with its column's logit, as bit V
      const unsigned long long p = GreedyKey(row[Vv.eos_col], Vv.V);
      rd += 2;
      mine = p > mine ? p : mine;
    }
    mine = WarpMax64(mine);
    if (lane == 0 && mine) atomicMax(F.best + b, mine);
  }

  // ---- arrival (fused tail): mask words, counts and argmax partials are
  // made visible first; the bulk logits stores follow.
  bool last = false;
  if (FusedTail(TAIL) || F.publish_arrival == 1 || (F.publish_arrival == 2 && publish)) {
    __syncwarp();
    int l = 0;
    if (lane == 0) l = ArriveRelease(Bt.seq_arrive + b) == need - 1;
    last = __shfl_sync(0xffffffffu, l, 0) != 0;
  }
  if (MODE == kFillMask && F.logits != nullptr) {
    uint16_t* row = F.logits + static_cast<long long>(b) * F.ld;
    if (eos_in_seg) {  // the EOS column carries bit V, not its (disabled) id's bit
      // Branch-free selects (an `if` on i here made ptxas index m[] and move
      // the whole array to local memory).
      const int wi = (Vv.eos_col - t0) >> 5;
      const uint32_t bit = lane == (wi & 31) ? 1u << (Vv.eos_col & 31) : 0u;
      const uint32_t set = eos_bit ? bit : 0u, clr = eos_bit ? 0u : bit;
#pragma unroll
      for (int i = 0; i < kSpans; ++i) {
        const bool hit = i == (wi >> 5);
        m[i] = (m[i] & ~(hit ? clr : 0u)) | (hit ? set : 0u);
      }
    }
    // Full spans by class: all allowed -> untouched; all masked -> one bulk
    // (TMA) store of 2 KB of -inf from shared memory, issued by lane 0;
    // mixed -> 16-B chunks, two spans in flight: the mixed chunks of the next
    // two mixed spans are being copied (cp.async, no registers held) while
    // one is blended and stored.  Then a partial last span, if any.
#if PRE3_COMPACT_MIXED
    const bool late = true;
#else
    const bool late = !spans_early;
#endif
    if (late) classify();
    if (masked && lane == 0) {
      const unsigned long long pol = EvictFirstPolicy();
#if PRE3_BULK_RUN > 1
      // Runs of adjacent masked spans as one bulk store (up to PRE3_BULK_RUN spans).
      for (uint32_t x = masked; x;) {
        const int i = __ffs(x) - 1;
        int len = 1;
        while (len < PRE3_BULK_RUN && ((x >> (i + len)) & 1u)) ++len;
        BulkStore(row + t0 + 1024 * i, ninf, 2048 * len, pol);
        x &= ~(((1u << len) - 1u) << i);
      }
#else
      for (uint32_t x = masked; x; x &= x - 1) BulkStore(row + t0 + 1024 * (__ffs(x) - 1), ninf, 2048, pol);
#endif
      BulkCommit();
      wr += 2048u * static_cast<unsigned>(__popc(masked));
    }
#if PRE3_COMPACT_MIXED
    const unsigned long long t_mx = Bt.trace ? NowNs() : 0ull;
    // Mixed chunks of as many mixed spans as fit the warp's 256-chunk buffer,
    // packed in (span, round, lane) order, are all copied in ONE round trip
    // (cp.async: no registers held), then blended and stored span by span; a
    // segment with more mixed chunks takes another batch.  Each lane reads
    // back only the chunks it copied itself.
    uint4* cbuf = &span_buf[0][0][0];  // 2 * 4 * 32 = 256 chunks
    const unsigned lt = LaneMaskLt();
#pragma unroll 1
    for (uint32_t todo = mixed; todo;) {
      uint32_t batch = 0u;
      int n = 0;
#pragma unroll 1
      for (uint32_t t = todo; t; t &= t - 1) {
        const int i = __ffs(t) - 1;
        uint32_t byte[4];
        SpanBytes(Pick(m, i), lane, byte);
        unsigned bal[4];
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          bal[k] = __ballot_sync(0xffffffffu, byte[k] != 0u && byte[k] != 0xffu);
          cnt += __popc(bal[k]);
        }
        if (n + cnt > 256) break;  // a span holds <= 128 mixed chunks: a batch takes >= 1 span
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((bal[k] >> lane) & 1u) CpAsync16(&cbuf[n + __popc(bal[k] & lt)], row + t0 + 1024 * i + (32 * k + lane) * 8);
          n += __popc(bal[k]);
        }
        batch |= 1u << i;
      }
      CpAsyncCommit();
      CpAsyncWait0();
      n = 0;
#pragma unroll 1
      for (uint32_t t = batch; t; t &= t - 1) {
        const int i = __ffs(t) - 1;
        const int tw = t0 + 1024 * i;
        uint32_t byte[4];
        SpanBytes(Pick(m, i), lane, byte);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool mix = byte[k] != 0u && byte[k] != 0xffu;
          const unsigned bal = __ballot_sync(0xffffffffu, mix);
          if (byte[k] != 0xffu) {
            uint4 o = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
            if (mix) {
              const uint32_t x = byte[k];
              const uint4 v = cbuf[n + __popc(bal & lt)];
              uint32_t* po = reinterpret_cast<uint32_t*>(&o);
              const uint32_t* pv = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t keep =
                    ((x >> (2 * j)) & 1u ? 0x0000FFFFu : 0u) | ((x >> (2 * j + 1)) & 1u ? 0xFFFF0000u : 0u);
                po[j] = (pv[j] & keep) | (0xFF80FF80u & ~keep);
              }
              rd += 16;
            }
            __stcs(reinterpret_cast<uint4*>(row + tw + (32 * k + lane) * 8), o);
            wr += 16;
          }
          n += __popc(bal);
        }
      }
      todo &= ~batch;
      __syncwarp();  // the buffer is refilled by the next batch
    }
#else
    const unsigned long long t_mx = Bt.trace ? NowNs() : 0ull;
    uint4(*buf)[4][32] = span_buf;  // [2][4][32] of this warp
    if (late) prefetch2();
    int q = 0;
#pragma unroll 1
    for (uint32_t todo = mixed; todo; todo &= todo - 1, q ^= 1) {
      const int i = __ffs(todo) - 1;
      CpAsyncWait1();  // this span's group is complete (only the next one's may pend)
      SpanStore(row, t0 + 1024 * i, Pick(m, i), lane, buf[q], &rd, &wr);
      if (pend) {
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        SpanPrefetch(row, t0 + 1024 * j, Pick(m, j), lane, buf[q]);
      }
      CpAsyncCommit();
    }
#endif
#pragma unroll 1
    for (int i = nfull; i < kSpans; ++i) {
      if (t0 + 1024 * i < tl1) MaskSpan(row, t0 + 1024 * i, tl1, F.vec_ok, Pick(m, i), lane, &rd, &wr);
    }
    if (Vv.layout && last_seg) TailColumns(Vv, row, eos_bit, lane, 32, &wr);
    const unsigned long long t_bw = Bt.trace ? NowNs() : 0ull;
    if (masked && lane == 0) BulkWaitRead();  // the -inf source outlives the reads
    if (Bt.trace && lane == 0) {
      TraceEvent(Bt, 15, b, seg, t_mx, static_cast<unsigned long long>(__popc(mixed)));  // l:mixed spans
      TraceEvent(Bt, 16, b, seg, t_bw, static_cast<unsigned long long>(__popc(masked)));  // l:bulk wait
    }
  }
  if (Bt.stats_enabled) {
    rd = static_cast<unsigned long long>(WarpSum(static_cast<int>(rd)));
    wr = static_cast<unsigned long long>(WarpSum(static_cast<int>(wr)));
    n_walks = WarpSum(n_walks);
    if (lane == 0) {
      if (rd | wr) {
        atomicAdd(Bt.stats + 0, rd);
        atomicAdd(Bt.stats + 1, wr);
      }
      if (n_walks) atomicAdd(Bt.stats + 2, static_cast<unsigned long long>(n_walks));
      if (slot >= Cc.C) atomicAdd(Bt.stats + 4, 1ull);
      if (slot == -3) atomicAdd(Bt.stats + 5, 1ull);  // gave up waiting for a build
    }
  }
  if (lane == 0 && seg == 0) atomicAdd(Bt.counters + 2, 1ull);
  if (Bt.trace) {
    // extra: walks | SM id << 32 | the warp's logits bytes << 40 (diagnostics)
    const unsigned bytes = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(rd + wr));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (lane == 0) {
      TraceEvent(Bt, kTraceLight, b, seg, t_in,
                 static_cast<unsigned long long>(n_walks & 0xffffffff) | (static_cast<unsigned long long>(smid) << 32) |
                     (static_cast<unsigned long long>(bytes) << 40));
    }
  }
  if constexpr (FusedTail(TAIL)) {
    if (last) SequenceTail<TAIL>(A, Vv, Cc, Bt, F, b, lane);
  }
  if constexpr (TAIL == kTailSplit) {
    if (F.accept_ctas > 0 && last) AcceptSeq<kSampleStream>(A, Vv, Cc, Bt, F.acc, b, lane);
  }
}

}  // namespace

struct FillShared {
  uint32_t mask[kSegWords];
  uint32_t cd[kSegWords];
  int pre[kSegWords];
  int scratch[kThreads / 32 + 1];
  unsigned long long best[kThreads / 32];
  int unit, last, eos;
};

// Grid: h_grid (<= 2 per SM) heavy CTAs, then ceil(B * nseg / kWarps) light CTAs.
//  * Heavy CTA: one (sequence, segment) listed by the lookups — a segment
//    with context-dependent tokens or a pending build — 256 threads: CD
//    tokens are walked one per thread, a direct fill walks 256 tokens a round.
//  * Light CTA: kWarps consecutive (sequence, segment) items, one per warp,
//    skipping items the heavy pass owns (LightItem).
// Every CTA first helps drain the build queue of new contexts (empty in the
// steady state).
template <int MODE, int TAIL>
__global__ void PRE3_FILL_BOUNDS FillKernel(const __grid_constant__ AutView A, const __grid_constant__ VocabView Vv,
                                            const __grid_constant__ CacheView Cc, const __grid_constant__ BatchView Bt,
                                            const __grid_constant__ FillArgs F) {
  PdlEnter();
  __shared__ FillShared sh;
  __shared__ uint4 span_buf[kWarps][2][4][32];  // light pass: per-warp double buffer of mixed chunks (32 KB)
  __shared__ __align__(128) uint4 ninf_buf[128 * PRE3_BULK_RUN];  // bf16 -inf: the bulk-store source

  extern __shared__ int32_t stack_s[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- the queue drained by the previous fill is free again (nobody
  // produces into it until the fill after next consumes it: 3-queue ring).
  if (F.reset >= 0 && blockIdx.x == 0 && tid == 0) {
    const BuildQueue R = QueueOf(Bt, F.reset);
    *R.n_items = 0u;
    *R.next_unit = 0u;
    *R.n_heavy = 0u;
  }

  const BuildQueue Qc = QueueOf(Bt, F.consume);
  const int bid = static_cast<int>(blockIdx.x);
  const int tag = HeavyTag(F.fill_no, 0);
  const int32_t* hidx = HeavyIndex(Bt, F.fill_no, Vv.nseg);

  if (bid >= Bt.h_grid) {
    int r = bid - Bt.h_grid;
    if constexpr (TAIL == kTailSplit) {
      // ---- split step in one grid: accept CTA i sits after light CTA
      // (i + 1) * accept_period - 1, so the accepts run while the light pass
      // streams (a separate accept grid only starts with the fill's last wave).
      const int P = F.accept_period, q = r / (P + 1);
      if (F.accept_ctas > 0 && q < F.accept_ctas && r - q * (P + 1) == P) {
        const int b = q * kWarps + warp;
        // Sequences whose mask is their slot's CI row (no arrivals needed);
        // the others are accepted by the item completing their arrivals.
        if (b < Bt.B && ArrivalsNeeded(Cc, Vv, SeqSlot(Bt, F.fill_no)[b], SeqHmask(Bt, F.fill_no)[b]) == 0) {
          AcceptSeq<kSampleStream>(A, Vv, Cc, Bt, F.acc, b, lane);
        }
        return;
      }
      if (F.accept_ctas > 0) r -= min(q, F.accept_ctas);
    }
    // ---- light pass.  Loads that only depend on (b, seg) are issued together.
    if (MODE == kFillMask && F.logits != nullptr) {
      for (int i = tid; i < 128 * PRE3_BULK_RUN; i += kThreads) {
        ninf_buf[i] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
      }
      {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // visible to the bulk copies
      }
      __syncthreads();
    }
    const int item = r * F.light_per_cta + warp;
    const bool in_range = warp < F.light_per_cta && item < Bt.B * Vv.nseg;
    const int b = in_range ? item / Vv.nseg : 0;
    const int seg = item - b * Vv.nseg;
    int hi = -1, slot = -2;
    uint32_t hmask = ~0u;
    if (in_range) {
      hi = hidx[static_cast<long long>(b) * Vv.nseg + seg];
      slot = SeqSlot(Bt, F.fill_no)[b];
      hmask = SeqHmask(Bt, F.fill_no)[b];
    }
    // Light CTAs help build at most PRE3_LIGHT_BUILD_UNITS units first (-1:
    // until the queue is empty); the heavy CTAs, resident from the start,
    // always drain it, so every unit is claimed by a running CTA.
    const unsigned int n_items = LoadRelaxed(Qc.n_items);
    if (n_items != 0u && PRE3_LIGHT_BUILD_UNITS != 0) {
      HelpBuild(A, Vv, Cc, Bt, F.consume, stack_s, &sh.unit, PRE3_LIGHT_BUILD_UNITS);  // CTA-uniform
    }
    // Owned by the heavy pass: listed for this fill at a position the grid's
    // h_grid heavy CTAs cover (a longer list spills over to the light pass,
    // whose warps take the rare CD/wait paths themselves).
    if (!in_range || (hi >= 0 && (hi & ~0xffff) == tag && (hi & 0xffff) < Bt.h_grid)) return;
    // Pure CI: a built shared slot and no heavy segment — the mask is the CI
    // row, the counts are the slot's (and with publish_arrival 2 nobody
    // waits for this sequence's items).
    const bool shared_ok = slot >= 0 && slot < Cc.C && Vv.nseg <= 32;
    const bool pure = shared_ok && hmask == 0u;
    // Split step (publish_arrival 2): only the items of a sequence's heavy
    // segments publish arrivals — its accept takes the other segments from the
    // slot's CI row (AcceptKernel's ci_shortcut, the same test).
    const bool publish = !shared_ok || ((hmask >> seg) & 1u);
    // Arrivals that complete the sequence: its accept's (split step in one
    // grid), else every segment (the fused tail's).
    const int need = F.accept_ctas > 0 ? ArrivalsNeeded(Cc, Vv, slot, hmask) : Vv.nseg;
    LightItem<MODE, TAIL>(A, Vv, Cc, Bt, F, b, seg, slot, pure, publish, need, lane, span_buf[warp], ninf_buf);
    return;
  }

  // ---- heavy pass.
  const unsigned long long t_in = Bt.trace ? NowNs() : 0ull;
  if (static_cast<unsigned int>(bid) >= LoadRelaxed(Qc.n_heavy)) return;  // (bid < h_grid <= h_cap)
  const int2 hv = Qc.heavy[bid];
  const int b = hv.x;
  const int seg = hv.y;
  const int hi = hidx[static_cast<long long>(b) * Vv.nseg + seg];
  int slot = SeqSlot(Bt, F.fill_no)[b];
  const unsigned int n_items = LoadRelaxed(Qc.n_items);
  if (hi != (tag | bid)) return;
  const int w0 = seg * kSegWords;
  const int nwords = min(Vv.W - w0, kSegWords);
  const int t0 = w0 * 32;
  const int t1 = min(Vv.V + 1, t0 + nwords * 32);
  static_assert(kSegWords == kThreads, "one mask word per thread");

  unsigned long long t_ph = t_in;
  if (n_items != 0u) HelpBuild(A, Vv, Cc, Bt, F.consume, stack_s, &sh.unit);
  if (tid == 0 && Bt.trace) TraceEvent(Bt, 10, b, seg, t_ph, 0), t_ph = NowNs();

  // Thread tid owns mask word w0 + tid (register `mword`).
  const uint32_t sw = (F.seg_counts != nullptr && tid < nwords) ? __ldg(Vv.structural + w0 + tid) : 0u;
  const bool wait = slot >= 0 && (slot & kSlotWait);
  if (slot >= 0) slot &= ~kSlotWait;
  if (wait) {
    if (slot < Cc.C) HelpSegment(A, Vv, Cc, Bt, slot, seg, b, stack_s, &sh.unit);
    if (tid == 0) sh.unit = WaitBuilt(Cc, Bt, slot, seg, Vv.nseg) ? 1 : 0;
    __syncthreads();
    if (!sh.unit) slot = -3;  // direct fill
  }
  if (tid == 0 && Bt.trace) TraceEvent(Bt, 11, b, seg, t_ph, 0), t_ph = NowNs();
  uint32_t mword = 0u;
  int cd_cnt = 0;
  if (slot >= 0) {
    const uint32_t* src = slot < Cc.C ? Cc.ci + static_cast<long long>(slot) * Vv.W
                                      : Bt.priv + static_cast<long long>(slot - Cc.C) * Vv.W;
    if (tid < nwords) mword = __ldcg(src + w0 + tid);
    if (slot < Cc.C) cd_cnt = __ldcg(Cc.cd_cnt + static_cast<long long>(slot) * Vv.nseg + seg);
  }
  unsigned long long n_walks = 0;
  if (slot == -3 || cd_cnt > 0) {
    sh.mask[tid] = mword;
    const int depth = Bt.seq[b].depth;
    const int32_t* gstack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
    for (int i = tid; i < depth; i += kThreads) stack_s[i] = gstack[i];
    if (slot == -3) {
      // Uncached: walk every token of the segment against the real stack.
      __syncthreads();
      for (int base_t = 0; base_t < nwords * 32; base_t += kThreads) {
        const int t = t0 + base_t + tid;
        const int r = t < t1 ? WalkToken(A, Vv, t, stack_s, depth, true) : kReject;
        const unsigned acc = __ballot_sync(0xffffffffu, r == kAccept);
        if (__any_sync(0xffffffffu, r == kOverflow) && lane == 0) atomicOr(Bt.err, 1u);
        if (lane == 0) sh.mask[(base_t >> 5) + warp] = acc;
      }
      n_walks = t1 - t0;
    } else {
      // Context-dependent tokens: walk them against the sequence's real stack.
      const uint32_t* cdsrc = Cc.cdb + static_cast<long long>(slot) * Vv.W + w0;
      const uint32_t x = tid < nwords ? __ldcg(cdsrc + tid) : 0u;
      sh.cd[tid] = x;
      int total = 0;
      const int excl = BlockExclusiveScan(__popc(x), sh.scratch, &total);  // has barriers
      sh.pre[tid] = excl;
      __syncthreads();
      if (tid == 0 && Bt.trace) TraceEvent(Bt, 12, b, seg, t_ph, 0), t_ph = NowNs();
      const bool by_warp = total <= 2 * kWarps;  // few tokens: latency-bound, walk each with a warp
      for (int q = by_warp ? warp : tid; q < total; q += by_warp ? kWarps : kThreads) {
        int lo = 0, hi2 = kThreads - 1;
        while (lo < hi2) {
          const int mid = (lo + hi2 + 1) >> 1;
          if (sh.pre[mid] <= q) lo = mid; else hi2 = mid - 1;
        }
        uint32_t bits = sh.cd[lo];
        for (int r = q - sh.pre[lo]; r > 0; --r) bits &= bits - 1;
        const int t = t0 + lo * 32 + (__ffs(bits) - 1);
        int r;
        if (by_warp) {
          r = WalkWarp(A, Vv, t, stack_s, depth, lane);
          if (r == kOverflow) r = WalkToken(A, Vv, t, stack_s, depth, true);
          if (lane != 0) continue;
        } else {
          r = WalkToken(A, Vv, t, stack_s, depth, true);
        }
        if (r == kAccept) atomicOr(&sh.mask[lo], 1u << ((t - t0) & 31));
        if (r == kOverflow) atomicOr(Bt.err, 1u);
      }
      n_walks = total;
    }
    __syncthreads();
    if (tid == 0 && Bt.trace) TraceEvent(Bt, 13, b, seg, t_ph, 0), t_ph = NowNs();
    mword = sh.mask[tid];
  }

  // ---- outputs: bitmask words, sampler counts, logits.
  if (F.bitmask != nullptr && tid < nwords) F.bitmask[static_cast<long long>(b) * F.ldw + w0 + tid] = mword;
  if (F.seg_counts != nullptr) {
    int ca = 0, cs = 0;
    if (tid < nwords) {
      uint32_t m = mword;
      if (w0 + tid == (Vv.V >> 5)) m &= ~(1u << (Vv.V & 31));
      ca = __popc(m);
      cs = __popc(m & sw);
    }
    ca = WarpSum(ca);
    cs = WarpSum(cs);
    if (lane == 0) {
      sh.scratch[warp] = ca;
      sh.pre[warp] = cs;
    }
    __syncthreads();
    if (tid == 0) {
      int ta = 0, ts = 0;
      for (int i = 0; i < kThreads / 32; ++i) ta += sh.scratch[i], ts += sh.pre[i];
      F.seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 0] = ta;
      F.seg_counts[(static_cast<long long>(b) * Vv.nseg + seg) * 2 + 1] = ts;
    }
  }
  // Model logit layout (LightItem): the EOS bit where the logits need it.
  const int tl1 = Vv.layout ? min(Vv.V, t1) : t1;
  const bool last_seg = seg == Vv.nseg - 1;
  const bool eos_in_seg = Vv.layout && Vv.eos_col < Vv.V && Vv.eos_col >= t0 && Vv.eos_col < tl1;
  if (Vv.layout && (last_seg || eos_in_seg)) {
    if (last_seg) {
      if (w0 + tid == (Vv.V >> 5)) sh.eos = static_cast<int>((mword >> (Vv.V & 31)) & 1u);
    } else if (tid == 0) {
      const int sl = SeqSlot(Bt, F.fill_no)[b];
      sh.eos = sl == -2 ? 0 : EosBitOf(A, Vv, Cc, Bt, b, sl & ~kSlotWait, !(sl & kSlotWait));
    }
  }
  __syncthreads();
  const int eos_bit = Vv.layout && (last_seg || eos_in_seg) ? sh.eos : 0;
  // Warp w covers words [32w, 32w+32) of the segment = one 1024-token span.
  unsigned rd = 0, wr = 0;  // this lane's logit bytes (stats)
  const int tw = t0 + warp * 1024;
  if (MODE == kFillGreedy) {
    const uint16_t* row = F.logits + static_cast<long long>(b) * F.ld;
    unsigned long long mine = tw < tl1 ? ArgmaxSpan(row, tw, tl1, F.vec_ok, mword, lane, &rd) : 0ull;
    if (Vv.layout && last_seg && eos_bit && tid == 0) {  // EOS competes with its column's logit, as bit V
      const unsigned long long p = GreedyKey(row[Vv.eos_col], Vv.V);
      rd += 2;
      mine = p > mine ? p : mine;
    }
    mine = WarpMax64(mine);
    if (lane == 0) sh.best[warp] = mine;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0;
      for (int i = 0; i < kThreads / 32; ++i) m = sh.best[i] > m ? sh.best[i] : m;
      if (m) atomicMax(F.best + b, m);
    }
  }

  // ---- arrival: the sequence's last item runs the tail.  Only the mask
  // words, counts and argmax partials must be visible to it, so the fence
  // precedes the (bulk) logits stores below.
  bool last = false;
  if (FusedTail(TAIL) || F.publish_arrival) {
    __syncthreads();
    if (tid == 0) {
      const int need = F.accept_ctas > 0
                           ? ArrivalsNeeded(Cc, Vv, SeqSlot(Bt, F.fill_no)[b], SeqHmask(Bt, F.fill_no)[b])
                           : Vv.nseg;
      sh.last = ArriveRelease(Bt.seq_arrive + b) == need - 1;
    }
    __syncthreads();
    last = sh.last;
  }
  if (MODE == kFillMask && F.logits != nullptr) {
    uint16_t* row = F.logits + static_cast<long long>(b) * F.ld;
    if (eos_in_seg && w0 + tid == (Vv.eos_col >> 5)) {  // the EOS column carries bit V
      const uint32_t bit = 1u << (Vv.eos_col & 31);
      mword = eos_bit ? (mword | bit) : (mword & ~bit);
    }
    if (tw < tl1) MaskSpan(row, tw, tl1, F.vec_ok, mword, lane, &rd, &wr);
    if (Vv.layout && last_seg && warp == 0) TailColumns(Vv, row, eos_bit, lane, 32, &wr);
  }
  if (Bt.stats_enabled) {
    rd = static_cast<unsigned long long>(WarpSum(static_cast<int>(rd)));
    wr = static_cast<unsigned long long>(WarpSum(static_cast<int>(wr)));
    if (lane == 0 && (rd | wr)) {
      atomicAdd(Bt.stats + 0, rd);
      atomicAdd(Bt.stats + 1, wr);
    }
    if (tid == 0 && n_walks) atomicAdd(Bt.stats + 2, n_walks);
    if (tid == 0 && slot >= Cc.C) atomicAdd(Bt.stats + 4, 1ull);
    if (tid == 0 && slot == -3) atomicAdd(Bt.stats + 5, 1ull);  // gave up waiting for a build
  }
  if (tid == 0 && seg == 0) atomicAdd(Bt.counters + 2, 1ull);
  if (tid == 0) TraceEvent(Bt, kTraceHeavy, b, seg, t_in, n_walks);
  if constexpr (FusedTail(TAIL)) {
    if (last && warp == 0) SequenceTail<TAIL>(A, Vv, Cc, Bt, F, b, lane);
  }
  if constexpr (TAIL == kTailSplit) {
    if (F.accept_ctas > 0 && last && warp == 0) AcceptSeq<kSampleStream>(A, Vv, Cc, Bt, F.acc, b, lane);
  }
}
// ---------------------------------------------------------------------------
// AcceptKernel: one warp per sequence (standalone accept / sample).
// ---------------------------------------------------------------------------
template <int SAMPLE>
__device__ __forceinline__ void AcceptBody(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                           const BatchView& Bt, const AcceptArgs& G, int b, SeqState st, int topv,
                                           const uint32_t* row, const int32_t* counts, const uint32_t* crow,
                                           const int32_t* ccounts, uint32_t hm, int lane, unsigned long long t_in);

// One sequence's sample + accept (+ the next fill's lookup), one warp: the
// body of AcceptKernel, and of the accept CTAs a split-step fill carries
// (FillArgs::accept_ctas).  wait_fill: the fill producing this step's items
// is still running — wait only for this sequence's (heavy) items.
template <int SAMPLE>
__device__ __forceinline__ void AcceptSeq(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                          const BatchView& Bt, const AcceptArgs& G, int b, int lane) {
  // The sequence's state and stack window are not written by the fill:
  // their loads overlap the wait for its items.
  const SeqState st = Bt.seq[b];
  const int topv = StackWindow(Bt, b, st.depth, lane);
  const uint32_t* row = G.bitmask + static_cast<long long>(b) * G.ldw;
  const int32_t* counts = G.seg_counts + static_cast<long long>(b) * Vv.nseg * 2;
  const uint32_t* crow = row;
  const int32_t* ccounts = counts;
  uint32_t hm = ~0u;  // segments read from the fill's outputs (the rest: the context's CI row)
  int need = Vv.nseg;
  if (G.ci_shortcut) {
    // A built shared slot (the fill's own test, FillKernel): the segments
    // without context-dependent tokens are the slot's CI row and counts —
    // sample from those now; wait only for the heavy segments' items (the
    // only ones that publish arrivals).  Pure CI: no wait at all.
    const int slot = SeqSlot(Bt, PrevFill(G.lookup_tag))[b];
    const uint32_t hmask = SeqHmask(Bt, PrevFill(G.lookup_tag))[b];
    if (slot >= 0 && slot < Cc.C && Vv.nseg <= 32) {
      const uint32_t all = Vv.nseg >= 32 ? 0xffffffffu : ((1u << Vv.nseg) - 1u);
      hm = hmask & all;
      need = __popc(hm);
      crow = Cc.ci + static_cast<long long>(slot) * Vv.W;
      ccounts = Cc.ci_cnt + static_cast<long long>(slot) * Vv.nseg * 2;
    }
  }
  if (G.wait_fill && need > 0) {
    // Bounded (200 ms): a fill that never delivers the items would be an
    // internal error — reported through gm_batch_check, never a hung GPU.
    if (LoadAcquire(Bt.seq_arrive + b) < need) {
      unsigned long long t_start, t_now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      do {
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
      } while (LoadAcquire(Bt.seq_arrive + b) < need && t_now - t_start < 200000000ull);
      if (t_now - t_start >= 200000000ull && lane == 0) atomicOr(Bt.err, 2u);
    }
    __syncwarp();
    if (lane == 0) Bt.seq_arrive[b] = 0;
  }
  AcceptBody<SAMPLE>(A, Vv, Cc, Bt, G, b, st, topv, row, counts, crow, ccounts, hm, lane,
                     Bt.trace ? NowNs() : 0ull);
}

template <int SAMPLE>
__global__ void PRE3_ACCEPT_BOUNDS AcceptKernel(AutView A, VocabView Vv, CacheView Cc, BatchView Bt,
                                                    AcceptArgs G) {
  // wait_fill: the preceding fill (launched just before, publishing
  // per-sequence arrivals) may still be running — each warp starts as soon as
  // its own sequence's items are in; the grid-wide wait moves to the end, so
  // this grid still completes after the fill (the next kernel relies on it).
  if (G.wait_fill) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  } else {
    PdlEnter();
  }
  const int lane = threadIdx.x & 31;
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b < Bt.B) AcceptSeq<SAMPLE>(A, Vv, Cc, Bt, G, b, lane);
  if (G.wait_fill) asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <int SAMPLE>
__device__ __forceinline__ void AcceptBody(const AutView& A, const VocabView& Vv, const CacheView& Cc,
                                           const BatchView& Bt, const AcceptArgs& G, int b, SeqState st, int topv,
                                           const uint32_t* row, const int32_t* counts, const uint32_t* crow,
                                           const int32_t* ccounts, uint32_t hm, int lane, unsigned long long t_in) {
  int tok = -1;
  if (SAMPLE == kSampleGiven) {
    tok = IdToBit(Vv, G.tokens[b]);
  } else if (SAMPLE == kSampleGreedy) {
    const unsigned long long p = G.best[b];
    tok = p ? static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(p)) : -1;
    __syncwarp();
    if (lane == 0) G.best[b] = 0ull;
  } else {
    tok = SampleStreamWarp(Vv, b, row, counts, crow, ccounts, hm, G.seed, st.draws, lane);
    st.draws += 1;
    if (lane == 0) atomicAdd(Bt.counters + 1, 1ull);
  }
  if (G.tokens_out != nullptr && lane == 0) G.tokens_out[b] = BitToId(Vv, tok);
  if (!G.do_accept) {
    if (lane == 0) Bt.seq[b].draws = st.draws;
    return;
  }
  AcceptWarp(A, Vv, Cc, Bt, b, st, topv, tok, G.status_out, (SAMPLE != kSampleGiven && G.restart) ? 2 : G.restart,
             G.lookup_queue, G.lookup_tag, lane);
  if (lane == 0) TraceEvent(Bt, kTraceAccept, b, 0, t_in, static_cast<unsigned long long>(tok + 1));
}

__global__ void ResetKernel(AutView A, BatchView Bt) {
  PdlEnter();
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
// SampleKernel: temperature / top-k / top-p sampling over the allowed tokens
// of each sequence, fused with accept (new work — the
// reference has no sampler).  One CTA per sequence.  Exact integer semantics
// (restated in oracle/gmask_port.c gp_sample_pick):
//   key(t)   16-bit order key of the bf16 logit (monotone in value)
//   kept_k   allowed tokens with key >= the k-th largest key (ties kept;
//            k = 0 or k >= |allowed|: all allowed)
//   W(key)   round(2^32 * 2^(((v - v_max) / T) * log2 e)) with a fixed
//            sequence of correctly rounded fp32 operations (deterministic
//            software exp2), v_max = the largest allowed logit
//   kept_p   kept_k tokens with key >= tau_p, tau_p = the largest key whose
//            weight above-or-at it reaches ceil(S_K * P24 / 2^24)
//   token    r = (u32 * S_P) >> 32 for the sequence's next stream draw u;
//            the token where the cumulative weight in (key desc, id asc)
//            order first exceeds r; S_P = 0 (all weights underflow): the
//            lowest-id token with the largest key.
// Every pass reads only the 16-B logit chunks that hold allowed tokens; the
// histograms are two-level (high byte, low byte of the key), so 3-5 passes
// replace a sort.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ uint32_t SampleKey(uint32_t bits16) {
  return (bits16 & 0x8000u) ? (~bits16 & 0xFFFFu) : (bits16 | 0x8000u);
}

__device__ __forceinline__ float KeyValue(uint32_t key) {
  const uint32_t bits = (key & 0x8000u) ? (key & 0x7FFFu) : (~key & 0xFFFFu);
  return __uint_as_float(bits << 16);
}

// Deterministic weight (identical bit-for-bit to the C restatement).
__device__ unsigned long long SampleWeight(uint32_t key, float vmax, float temperature) {
  const float v = KeyValue(key);
  const float d = __fsub_rn(v, vmax);
  const float x = __fdiv_rn(d, temperature);
  const float y = __fmul_rn(x, 1.44269502f);
  if (!(y >= -64.0f)) return 0ull;  // underflow, NaN
  if (y > 0.0f) return 0ull;        // only v <= vmax
  const float fl = floorf(y);
  const int n = static_cast<int>(fl);
  const float f = __fsub_rn(y, fl);
  float p = 1.54035304e-4f;
  p = __fmaf_rn(p, f, 1.33335581e-3f);
  p = __fmaf_rn(p, f, 9.61812911e-3f);
  p = __fmaf_rn(p, f, 5.55041087e-2f);
  p = __fmaf_rn(p, f, 2.40226507e-1f);
  p = __fmaf_rn(p, f, 6.93147181e-1f);
  p = __fmaf_rn(p, f, 1.0f);
  const float scale = __uint_as_float(static_cast<uint32_t>(n + 32 + 127) << 23);  // 2^(n+32), exact
  return __float2ull_rn(__fmul_rn(p, scale));
}

constexpr int kSampleKeySlots = 24;  // kcnt rows: 24 x 256 x 4 B = the per-warp histograms' 24 KB

struct SampleShared {
  unsigned int cnt_hi[256];
  unsigned long long w_hi[256];
  // Per-warp copies of the two dense histograms: an allowed token's high byte
  // (sign + exponent) takes few values, so one shared copy serializes the
  // CTA's atomics; the copies are summed after each pass (exact: integers).
  // Dense rows with few high bytes instead count every 16-bit key (kcnt) and
  // weigh each distinct key once: sum_t W(key_t) = sum_key cnt(key) * W(key).
  union {
    struct {
      unsigned int cnt_hi_w[kThreads / 32][256];
      unsigned long long w_hi_w[kThreads / 32][256];
    } pw;
    unsigned int kcnt[kSampleKeySlots][256];
  } u;
  signed char hslot[256];          // high byte -> kcnt row (-1: none)
  unsigned char slot_h[kSampleKeySlots];
  int nslots;
  unsigned int cnt_lo[256];
  unsigned long long w_lo[256];
  unsigned int cnt_lo2[256];
  unsigned long long w_lo2[256];
  unsigned int red[kThreads / 32 + 1];
  unsigned long long red64[kThreads / 32];
  int found;
  int claim[256];                  // one-pass key counting: high byte -> kcnt row (-1: none yet, -2: being claimed)
  short row_h[kSampleKeySlots];    // kcnt row -> high byte
  int nclaim;
};

enum : int { kPassHi = 0, kPassWeights = 1, kPassLoBin = 2 };

// One pass over the allowed tokens of row b (chunks of 8 tokens whose mask
// byte is non-zero).  fn(t, key) per allowed token.
// Bit t's logit is column t, except EOS (bit V): column eos_col (the model
// logit layout, VocabView; eos_col = V in the reference layout).
template <typename Fn>
__device__ __forceinline__ void ForAllowed(const uint32_t* mrow, const uint16_t* row, int V, int eos_col, bool vec_ok,
                                           int c_begin, int c_end, int c_step, Fn&& fn) {
  for (int c = c_begin; c < c_end; c += c_step) {
    const uint32_t byte = (__ldg(mrow + (c >> 2)) >> ((c & 3) * 8)) & 0xffu;
    if (!byte) continue;
    const int tb = c * 8;
    if (vec_ok && tb + 8 <= V) {
      const uint4 q = __ldcg(reinterpret_cast<const uint4*>(row + tb));
      const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((byte >> j) & 1u) fn(tb + j, SampleKey((w4[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu));
      }
    } else {
      for (int j = 0; j < 8 && tb + j <= V; ++j) {
        if ((byte >> j) & 1u) fn(tb + j, SampleKey(row[tb + j == V ? eos_col : tb + j]));
      }
    }
  }
}

// ForAllowed with U chunks' mask bytes, then their logit loads, issued
// together (one dependent round trip per U chunks instead of per chunk).
template <int U, typename Fn>
__device__ __forceinline__ void ForAllowedBatched(const uint32_t* mrow, const uint16_t* row, int V, int eos_col,
                                                  bool vec_ok, int c_begin, int c_end, int c_step, Fn&& fn) {
  for (int c0 = c_begin; c0 < c_end; c0 += U * c_step) {
    uint32_t byte[U];
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * c_step;
      byte[u] = c < c_end ? (__ldg(mrow + (c >> 2)) >> ((c & 3) * 8)) & 0xffu : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tb = (c0 + u * c_step) * 8;
      q[u] = byte[u] && vec_ok && tb + 8 <= V ? __ldcg(reinterpret_cast<const uint4*>(row + tb)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!byte[u]) continue;
      const int tb = (c0 + u * c_step) * 8;
      if (vec_ok && tb + 8 <= V) {
        const uint32_t k4[4] = {PairOrderKeys(q[u].x), PairOrderKeys(q[u].y), PairOrderKeys(q[u].z),
                                PairOrderKeys(q[u].w)};  // = SampleKey of each half
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if ((byte[u] >> j) & 1u) fn(tb + j, (k4[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu);
        }
      } else {
        for (int j = 0; j < 8 && tb + j <= V; ++j) {
          if ((byte[u] >> j) & 1u) fn(tb + j, SampleKey(row[tb + j == V ? eos_col : tb + j]));
        }
      }
    }
  }
}

// The 16-bit keys of the allowed tokens of chunks [c_begin, c_end) equal to
// `kappa`, in id order: fn(t) per match.  Four chunks' mask bytes, then their
// logit loads, are issued together (pass 5 walks a contiguous chunk range per
// thread; one load at a time made it a chain of ~60 dependent round trips).
template <typename Fn>
__device__ __forceinline__ void ForKeyMatches(const uint32_t* mrow, const uint16_t* row, int V, int eos_col,
                                              bool vec_ok, int c_begin, int c_end, uint32_t kappa, Fn&& fn) {
  constexpr int U = 4;
  for (int c0 = c_begin; c0 < c_end; c0 += U) {
    uint32_t byte[U];
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      byte[u] = c < c_end ? (__ldg(mrow + (c >> 2)) >> ((c & 3) * 8)) & 0xffu : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tb = (c0 + u) * 8;
      q[u] = byte[u] && vec_ok && tb + 8 <= V ? __ldcg(reinterpret_cast<const uint4*>(row + tb)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!byte[u]) continue;
      const int tb = (c0 + u) * 8;
      if (vec_ok && tb + 8 <= V) {
        const uint32_t w4[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
        // Any of the 8 keys equal to kappa?  Two keys per word: a zero half of
        // keys ^ (kappa, kappa) (the haszero test), most chunks have none.
        const uint32_t k2 = kappa | (kappa << 16);
        uint32_t hit = 0u;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const uint32_t x = PairOrderKeys(w4[p]) ^ k2;
          hit |= (x - 0x00010001u) & ~x & 0x80008000u;
        }
        if (!hit) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (((byte[u] >> j) & 1u) && SampleKey((w4[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu) == kappa) fn(tb + j);
        }
      } else {
        for (int j = 0; j < 8 && tb + j <= V; ++j) {
          if (((byte[u] >> j) & 1u) && SampleKey(row[tb + j == V ? eos_col : tb + j]) == kappa) fn(tb + j);
        }
      }
    }
  }
}

// Warp-parallel descending scan of arr[hi], arr[hi-1], ..., arr[lo]
// (smem, at most 256 entries) starting from c0: the first index i whose
// inclusive running sum reaches `target`, with the running sum before it in
// *excl (-1 when none: *excl = c0 + the whole range).  Lane l takes entries
// hi-8l .. hi-8l-7; every lane returns the same result (each warp of the CTA
// can run it redundantly — no barrier).
template <typename T>
__device__ __forceinline__ int ScanDescWarp(const T* arr, int hi, int lo, T c0, T target, T* excl) {
  const int lane = threadIdx.x & 31;
  T v[8];
  T mine = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = hi - 8 * lane - j;
    v[j] = i >= lo ? arr[i] : T(0);
    mine += v[j];
  }
  T inc = mine;  // inclusive warp scan (exact integers)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const T before = c0 + inc - mine;  // the running sum before this lane's entries
  const unsigned hit = __ballot_sync(0xffffffffu, c0 + inc >= target && hi - 8 * lane >= lo);
  if (!hit) {
    *excl = c0 + __shfl_sync(0xffffffffu, inc, 31);
    return -1;
  }
  const int src = __ffs(hit) - 1;
  int idx = -1;
  T cum = before;
  if (lane == src) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (idx < 0) {
        if (cum + v[j] >= target) idx = hi - 8 * lane - j;
        else cum += v[j];
      }
    }
  }
  *excl = __shfl_sync(0xffffffffu, cum, src);
  return __shfl_sync(0xffffffffu, idx, src);
}

__device__ __forceinline__ unsigned long long MulHi32(unsigned long long a, uint32_t u) {
  // (a * u) >> 32 for a < 2^63
  return __umul64hi(a, static_cast<unsigned long long>(u) << 32);
}

}  // namespace

__global__ void __launch_bounds__(kThreads) SampleKernel(AutView A, VocabView Vv, CacheView Cc, BatchView Bt,
                                                         SampleArgs S) {
  PdlEnter();
  __shared__ SampleShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int V1 = Vv.V + 1;
  const int nchunks = (V1 + 7) >> 3;
  const uint32_t* mrow = S.bitmask + static_cast<long long>(b) * S.ldw;
  const uint16_t* row = S.logits + static_cast<long long>(b) * S.ld;
  for (int i = tid; i < kSampleKeySlots * 256; i += kThreads) sh.u.kcnt[i >> 8][i & 255] = 0u;
  for (int i = tid; i < 256; i += kThreads) {
    sh.cnt_hi[i] = 0u;
    sh.w_hi[i] = 0ull;
    sh.cnt_lo[i] = 0u;
    sh.w_lo[i] = 0ull;
    sh.cnt_lo2[i] = 0u;
    sh.w_lo2[i] = 0ull;
    sh.claim[i] = -1;
  }
  if (tid < kSampleKeySlots) sh.row_h[tid] = -1;
  if (tid == 0) sh.nclaim = 0;
  __syncthreads();
  // ---- pass 1 (one-pass key counting): every allowed token's 16-bit key
  // counted in kcnt, a row per high byte claimed on first sight; max key,
  // |allowed|.  More high bytes than rows: the two-pass path below.
  unsigned int kmax = 0u, n_allowed = 0u;
  int last_h = -1, last_r = 0;  // the previous token's high byte and row (consecutive tokens often share it)
  ForAllowedBatched<PRE3_SAMPLE_BATCH>(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, tid, nchunks, kThreads, [&](int, uint32_t key) {
    const int h = static_cast<int>(key >> 8);
    int r = h == last_h ? last_r : sh.claim[h];
    if (r < 0) {
      // -1 -> -2 (claiming) -> row id; a thread that loses the race waits for
      // the winner's id (independent thread scheduling: the winner progresses).
      if (atomicCAS(&sh.claim[h], -1, -2) == -1) {
        r = atomicAdd(&sh.nclaim, 1);
        atomicExch(&sh.claim[h], r);
      } else {
        // Bounded: past it (a tool that serializes threads), force the
        // two-pass path — the counts are then rebuilt from scratch.
        for (int spin = 0; (r = atomicAdd(&sh.claim[h], 0)) < 0 && spin < 4096; ++spin) {
        }
        if (r < 0) {
          atomicMax(&sh.nclaim, kSampleKeySlots + 1);
          r = kSampleKeySlots;
        }
      }
    }
    last_h = h;
    last_r = r;
    if (r < kSampleKeySlots) atomicAdd(&sh.u.kcnt[r][key & 0xffu], 1u);
    kmax = key > kmax ? key : kmax;
    ++n_allowed;
  });
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  n_allowed = __reduce_add_sync(0xffffffffu, n_allowed);
  if (lane == 0) sh.red[warp] = kmax;
  __syncthreads();
  const bool one_pass = sh.nclaim <= kSampleKeySlots;
  if (one_pass) {
    // Row -> high byte, then the high-byte counts from the rows.
    if (sh.claim[tid] >= 0) sh.row_h[sh.claim[tid]] = static_cast<short>(tid);
    __syncthreads();
    for (int r = 0; r < sh.nclaim; ++r) {
      unsigned int c = sh.u.kcnt[r][tid];
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0 && c) atomicAdd(&sh.cnt_hi[sh.row_h[r]], c);
    }
  } else {
    // Two-pass path: per-warp high-byte histograms (a bf16 logit's sign +
    // exponent byte takes few values: one shared copy would serialize).
    for (int i = tid; i < 256 * (kThreads / 32); i += kThreads) {
      sh.u.pw.cnt_hi_w[i >> 8][i & 255] = 0u;
      sh.u.pw.w_hi_w[i >> 8][i & 255] = 0ull;
    }
    __syncthreads();
    ForAllowed(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, tid, nchunks, kThreads,
               [&](int, uint32_t key) { atomicAdd(&sh.u.pw.cnt_hi_w[warp][key >> 8], 1u); });
    __syncthreads();
    for (int i = tid; i < 256; i += kThreads) {
      unsigned int c = 0u;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) c += sh.u.pw.cnt_hi_w[w][i];
      sh.cnt_hi[i] = c;
    }
  }
  if (tid == 0) {
    unsigned int m = 0u;
    for (int i = 0; i < kThreads / 32; ++i) m = sh.red[i] > m ? sh.red[i] : m;
    sh.red[0] = m;
  }
  __syncthreads();
  kmax = sh.red[0];
  __syncthreads();
  if (lane == 0) sh.red[warp] = n_allowed;
  __syncthreads();
  unsigned int total_allowed = 0u;
  for (int i = 0; i < kThreads / 32; ++i) total_allowed += sh.red[i];
  __syncthreads();

  SeqState st = Bt.seq[b];
  int tok = -1;
  // Per-thread uniform decisions below are computed by every thread from
  // shared histograms (identical results, no broadcast needed).
  if (total_allowed > 0u) {
    const float vmax = KeyValue(kmax);
    const unsigned int k = static_cast<unsigned int>(S.top_k);
    int hi_k = -1;       // bin holding the top-k threshold (-1: everything kept)
    unsigned int need_k = 0u;
    if (k > 0u && k < total_allowed) {
      unsigned int cum = 0u;
      hi_k = ScanDescWarp<unsigned int>(sh.cnt_hi, 255, 0, 0u, k, &cum);
      need_k = k - cum;
    }
    // ---- pass 2: weights per high bin above hi_k; counts + weights per low
    // byte inside hi_k.  Key-count mode: dense rows whose high bytes above
    // hi_k fit kSampleKeySlots rows of kcnt.  After a one-pass count every
    // key's count is on chip already: no pass over the row.
    if (one_pass) {
      if (tid == 0) sh.nslots = sh.nclaim;
      for (int h = tid; h < 256; h += kThreads) sh.hslot[h] = static_cast<signed char>(sh.claim[h]);
      for (int r = tid; r < kSampleKeySlots; r += kThreads) sh.slot_h[r] = static_cast<unsigned char>(sh.row_h[r] < 0 ? 0 : sh.row_h[r]);
      if (hi_k >= 0) {
        const uint32_t c = sh.u.kcnt[sh.claim[hi_k]][tid];
        sh.cnt_lo[tid] = c;
        sh.w_lo[tid] = c ? static_cast<unsigned long long>(c) *
                               SampleWeight((static_cast<uint32_t>(hi_k) << 8) | tid, vmax, S.temperature)
                         : 0ull;
      }
      __syncthreads();
    } else if (tid == 0) {
      int n = 0;
      for (int h = 0; h < 256; ++h) {
        const bool act = h > hi_k && sh.cnt_hi[h] > 0u;
        sh.hslot[h] = static_cast<signed char>(act && n < kSampleKeySlots ? n : -1);
        if (act) {
          if (n < kSampleKeySlots) sh.slot_h[n] = static_cast<unsigned char>(h);
          ++n;
        }
      }
      sh.nslots = (total_allowed >= 2048u && n <= kSampleKeySlots) ? n : -1;
    }
    __syncthreads();
    const int nslots = sh.nslots;
    if (!one_pass) {
      if (nslots >= 0) {
        for (int i = tid; i < kSampleKeySlots * 256; i += kThreads) sh.u.kcnt[i >> 8][i & 255] = 0u;
        __syncthreads();
      }
      ForAllowed(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, tid, nchunks, kThreads, [&](int, uint32_t key) {
        const int h = static_cast<int>(key >> 8);
        if (h > hi_k) {
          if (nslots >= 0) atomicAdd(&sh.u.kcnt[sh.hslot[h]][key & 0xffu], 1u);
          else atomicAdd(&sh.u.pw.w_hi_w[warp][h], SampleWeight(key, vmax, S.temperature));
        } else if (h == hi_k) {
          atomicAdd(&sh.cnt_lo[key & 0xffu], 1u);
          atomicAdd(&sh.w_lo[key & 0xffu], SampleWeight(key, vmax, S.temperature));
        }
      });
      __syncthreads();
    }
    if (nslots >= 0) {
      // Thread t = low byte t: weigh each (high byte, t) key once (bins above
      // hi_k; after a one-pass count every bin has a row — the others' sums
      // are never read).
      for (int sl = 0; sl < nslots; ++sl) {
        if (one_pass && (sh.row_h[sl] < 0 || sh.row_h[sl] <= hi_k)) continue;
        const uint32_t c = sh.u.kcnt[sl][tid];
        unsigned long long w =
            c ? static_cast<unsigned long long>(c) * SampleWeight((static_cast<uint32_t>(sh.slot_h[sl]) << 8) | tid,
                                                                 vmax, S.temperature)
              : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (lane == 0 && w) atomicAdd(&sh.w_hi[sh.slot_h[sl]], w);
      }
    } else {
      for (int i = tid; i < 256; i += kThreads) {
        unsigned long long w = 0ull;
#pragma unroll
        for (int ww = 0; ww < kThreads / 32; ++ww) w += sh.u.pw.w_hi_w[ww][i];
        sh.w_hi[i] = w;
      }
    }
    __syncthreads();
    int lo_k = 0;
    if (hi_k >= 0) {
      unsigned int cum = 0u;
      const int l = ScanDescWarp<unsigned int>(sh.cnt_lo, 255, 0, 0u, need_k, &cum);
      lo_k = l < 0 ? 0 : l;
    }
    unsigned long long s_k = 0ull;
    ScanDescWarp<unsigned long long>(sh.w_hi, 255, hi_k + 1, 0ull, ~0ull, &s_k);  // (a sum: no index reaches ~0)
    if (hi_k >= 0) ScanDescWarp<unsigned long long>(sh.w_lo, 255, lo_k, s_k, ~0ull, &s_k);
    // Threshold tau_p as (bin, low byte); lo_p < 0 = resolve with pass 3.
    int hi_p = hi_k, lo_p = lo_k;
    unsigned long long s_p = s_k;
    if (s_k > 0ull && S.top_p24 < (1u << 24)) {
      const unsigned long long target =
          (__umul64hi(s_k, static_cast<unsigned long long>(S.top_p24) << 40) + (((s_k * S.top_p24) & 0xFFFFFFull) ? 1ull : 0ull));
      // target = ceil(s_k * P24 / 2^24): high part via umul64hi of the product shifted by 40 (2^64 / 2^24)
      unsigned long long cum = 0ull;
      bool done = false;
      const int h = ScanDescWarp<unsigned long long>(sh.w_hi, 255, hi_k + 1, 0ull, target, &cum);
      if (h >= 0) {
        hi_p = h;
        lo_p = -1;
        s_p = cum;  // plus the bin's part, after pass 3
        done = true;
      }
      if (!done && hi_k >= 0) {
        unsigned long long before = 0ull;
        const int l = ScanDescWarp<unsigned long long>(sh.w_lo, 255, lo_k, cum, target, &before);
        if (l >= 0) {
          lo_p = l;
          s_p = before + sh.w_lo[l];
          done = true;
        }
      }
      if (lo_p < 0) {
        // ---- pass 3: low-byte weights inside bin hi_p (fully kept_k).
        const int hp = hi_p;
        if (nslots >= 0) {  // key counts of bin hp are on chip (kcnt)
          const uint32_t c = sh.u.kcnt[sh.hslot[hp]][tid];
          sh.cnt_lo2[tid] = c;
          sh.w_lo2[tid] = c ? static_cast<unsigned long long>(c) *
                                  SampleWeight((static_cast<uint32_t>(hp) << 8) | tid, vmax, S.temperature)
                            : 0ull;
        } else {
          ForAllowed(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, tid, nchunks, kThreads, [&](int, uint32_t key) {
            if (static_cast<int>(key >> 8) == hp) {
              atomicAdd(&sh.cnt_lo2[key & 0xffu], 1u);
              atomicAdd(&sh.w_lo2[key & 0xffu], SampleWeight(key, vmax, S.temperature));
            }
          });
        }
        __syncthreads();
        unsigned long long before = 0ull;
        const int l = ScanDescWarp<unsigned long long>(sh.w_lo2, 255, 0, cum, target, &before);
        if (l >= 0) {
          lo_p = l;
          s_p = before + sh.w_lo2[l];
        }
      }
    }
    // ---- the drawn key: (bin, low byte) and the index within its ties.
    uint32_t kappa = kmax;
    unsigned long long jth = 0ull;
    if (s_p > 0ull) {
      const unsigned long long u =
          Mix64(Mix64(S.seed ^ (static_cast<unsigned long long>(b) * 0xD1B54A32D192ED03ull)) ^
                static_cast<unsigned long long>(st.draws));
      const unsigned long long r = MulHi32(s_p, static_cast<uint32_t>(u));
      // Walk kept_p in key-descending order: bins above the threshold bin
      // are whole; the threshold bin counts low bytes >= lo_p.
      const int hb = hi_p;  // threshold bin (hi_p == hi_k when top-p is off)
      unsigned long long cum = 0ull;
      // (every bin above hb >= hi_k is whole: r < cum + w  <=>  cum + w >= r + 1)
      int h_sel = ScanDescWarp<unsigned long long>(sh.w_hi, 255, hb + 1, 0ull, r + 1ull, &cum);
      const unsigned long long* wl;
      int lmin = 0;
      if (h_sel < 0) {
        h_sel = hb;
        lmin = lo_p;
        wl = (hb == hi_k && hi_k >= 0) ? sh.w_lo : sh.w_lo2;
      } else {
        // ---- pass 4: low-byte histogram of the selected whole bin.
        __syncthreads();
        for (int i = tid; i < 256; i += kThreads) {
          sh.cnt_lo2[i] = 0u;
          sh.w_lo2[i] = 0ull;
        }
        __syncthreads();
        const int hs = h_sel;
        if (nslots >= 0) {  // key counts of bin hs are on chip (kcnt)
          const uint32_t c = sh.u.kcnt[sh.hslot[hs]][tid];
          sh.cnt_lo2[tid] = c;
          sh.w_lo2[tid] = c ? static_cast<unsigned long long>(c) *
                                  SampleWeight((static_cast<uint32_t>(hs) << 8) | tid, vmax, S.temperature)
                            : 0ull;
        } else {
          ForAllowed(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, tid, nchunks, kThreads, [&](int, uint32_t key) {
            if (static_cast<int>(key >> 8) == hs) {
              atomicAdd(&sh.cnt_lo2[key & 0xffu], 1u);
              atomicAdd(&sh.w_lo2[key & 0xffu], SampleWeight(key, vmax, S.temperature));
            }
          });
        }
        __syncthreads();
        wl = sh.w_lo2;
      }
      {
        unsigned long long before = 0ull;
        const int l = ScanDescWarp<unsigned long long>(wl, 255, lmin, cum, r + 1ull, &before);
        if (l >= 0) {
          kappa = (static_cast<uint32_t>(h_sel) << 8) | static_cast<uint32_t>(l);
          jth = (r - before) / SampleWeight(kappa, vmax, S.temperature);
        }
      }
    }
    // ---- pass 5: the jth token (id order) with key kappa: contiguous chunk
    // ranges per thread, counts scanned across the CTA.
    const int per = (nchunks + kThreads - 1) / kThreads;
    const int c0 = tid * per, c1 = min(nchunks, c0 + per);
    // The first two matches of each thread are kept, so the thread holding
    // the jth rarely walks its range again.
    unsigned int mine = 0u;
    int first0 = -1, first1 = -1;
    ForKeyMatches(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, c0, c1, kappa, [&](int t) {
      if (mine == 0u) first0 = t;
      else if (mine == 1u) first1 = t;
      ++mine;
    });
    int total = 0;
    const int excl = BlockExclusiveScan(static_cast<int>(mine), reinterpret_cast<int*>(sh.red), &total);
    if (tid == 0) sh.found = -1;
    __syncthreads();
    if (jth >= static_cast<unsigned long long>(excl) && jth < static_cast<unsigned long long>(excl) + mine) {
      unsigned int want = static_cast<unsigned int>(jth) - static_cast<unsigned int>(excl);
      int hit = -1;
      if (want < 2u) {
        hit = want == 0u ? first0 : first1;
      } else {
        ForKeyMatches(mrow, row, Vv.V, Vv.eos_col, S.vec_ok, c0, c1, kappa, [&](int t) {
          if (want == 0u && hit < 0) hit = t;
          --want;
        });
      }
      sh.found = hit;
    }
    __syncthreads();
    tok = sh.found;
  }
  // ---- accept (warp 0): Step per byte, restart, next context lookup.
  if (warp == 0) {
    st.draws += 1;
    if (S.tokens_out != nullptr && lane == 0) S.tokens_out[b] = BitToId(Vv, tok);
    if (S.do_accept) {
      AcceptWarp(A, Vv, Cc, Bt, b, st, StackWindow(Bt, b, st.depth, lane), tok, nullptr, S.restart ? 2 : 0, S.lookup_queue,
                 S.lookup_tag, lane);
    } else if (lane == 0) {
      Bt.seq[b].draws = st.draws;
    }
  }
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute.
template <typename... KArgs, typename... Args>
static cudaError_t Launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

cudaError_t LaunchSample(const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b,
                         SampleArgs s, cudaStream_t st) {
  if (b.B == 0) return cudaSuccess;
  s.vec_ok = (s.ld % 8) == 0 && (reinterpret_cast<uintptr_t>(s.logits) % 16) == 0;
  return Launch(SampleKernel, dim3(b.B), dim3(kThreads), 0, st, a, v, c, b, s);
}

// ---------------------------------------------------------------------------
// AllowedTerminalsKernel: Engine::AllowedTerminals (runtime.cpp:188-208) for
// every sequence — terminal t (byte or $) is allowed iff some edge of the
// current state accepting t has a condition matching the stack (the OR of the
// accepted sets of all condition-matching edges).  One CTA per sequence,
// thread t scans the candidates of (state, t) against the stack in shared
// memory.  out[b*9 + w]: bytes in words 0..7, $ = bit 0 of word 8.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(288) AllowedTerminalsKernel(AutView A, BatchView Bt, uint32_t* out) {
  PdlEnter();
  extern __shared__ int32_t stk[];
  __shared__ uint32_t words[9];
  const int b = blockIdx.x, t = threadIdx.x;
  const SeqState st = Bt.seq[b];
  const int depth = st.depth;
  const int32_t* gstack = Bt.stacks + static_cast<long long>(b) * Bt.cap;
  for (int i = t; i < depth; i += blockDim.x) stk[i] = gstack[i];
  if (t < 9) words[t] = 0u;
  __syncthreads();
  if (st.status == kAlive && t < 257) {
    const int state = stk[depth - 1];
    const int idx = state * 257 + t;
    const int cb = __ldg(A.rec_begin + idx), ce = __ldg(A.rec_begin + idx + 1);
    bool any = false;
    for (int c = cb; c < ce && !any; ++c) {
      const Rec r = LoadRec(A.recs + c);
      bool match = r.cond_len <= depth;  // ConditionMatches (runtime.cpp:123-131)
      for (int j = 1; j < r.cond_len && match; ++j) match = stk[depth - 1 - j] == CondEntry(r, A.rec_cond, j);
      any = match;
    }
    if (any) atomicOr(&words[t >> 5], 1u << (t & 31));
  }
  __syncthreads();
  if (t < 9) out[static_cast<long long>(b) * 9 + t] = words[t];
}

cudaError_t LaunchAllowed(const AutView& a, const BatchView& b, uint32_t* out, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  const size_t dyn = static_cast<size_t>(b.cap) * sizeof(int32_t);
  static size_t opted = 0;
  if (dyn > 48 * 1024 && dyn > opted) {
    cudaFuncSetAttribute(AllowedTerminalsKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
    opted = dyn;
  }
  return Launch(AllowedTerminalsKernel, dim3(b.B), dim3(288), dyn, s, a, b, out);
}

// ---------------------------------------------------------------------------
cudaError_t LaunchReset(const AutView& a, const BatchView& b, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  return Launch(ResetKernel, dim3((b.B + 127) / 128), dim3(128), 0, s, a, b);
}

// Structural counts of every built context (CacheView::ci_cnt[.][.][1]) after
// the structural token set changed: one warp per (slot, segment).
__global__ void __launch_bounds__(256) RecountStructuralKernel(CacheView Cc, VocabView Vv) {
  const int lane = threadIdx.x & 31;
  const long long units = static_cast<long long>(Cc.C) * Vv.nseg;
  for (long long u = (blockIdx.x * 256ll + threadIdx.x) >> 5; u < units; u += (gridDim.x * 256ll) >> 5) {
    const int slot = static_cast<int>(u / Vv.nseg), seg = static_cast<int>(u % Vv.nseg);
    if (!(__ldcg(Cc.slot_meta + slot) & (1 << 16))) continue;
    int cs = 0;
    for (int w = seg * kSegWords + lane; w < min(Vv.W, (seg + 1) * kSegWords); w += 32) {
      uint32_t a = __ldcg(Cc.ci + static_cast<long long>(slot) * Vv.W + w);
      if (w == (Vv.V >> 5)) a &= ~(1u << (Vv.V & 31));
      cs += __popc(a & Vv.structural[w]);
    }
    cs = WarpSum(cs);
    if (lane == 0) Cc.ci_cnt[u * 2 + 1] = cs;
  }
}

// Context-table snapshots (capi.cu gm_engine_snapshot_*): a slot's rows —
// key row, cd_cnt, ci_cnt, ci, cdb — packed into one block of `blk` words per
// listed slot (gather) or unpacked from it (scatter).  One CTA per slot.
__global__ void SnapshotRowsKernel(CacheView c, int W, int nseg, const int32_t* __restrict__ ids, int n,
                                   uint32_t* __restrict__ blocks, int scatter) {
  const int r = static_cast<int>(blockIdx.x);
  if (r >= n) return;
  const long long slot = ids[r];
  const long long blk = kMaxContext + 3LL * nseg + 2LL * W;
  uint32_t* out = blocks + r * blk;
  struct Part {
    uint32_t* base;
    long long len;
  } parts[5] = {{reinterpret_cast<uint32_t*>(c.slot_keys) + slot * kMaxContext, kMaxContext},
                {reinterpret_cast<uint32_t*>(c.cd_cnt) + slot * nseg, nseg},
                {reinterpret_cast<uint32_t*>(c.ci_cnt) + slot * 2 * nseg, 2LL * nseg},
                {c.ci + slot * W, W},
                {c.cdb + slot * W, W}};
  long long off = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    for (long long i = threadIdx.x; i < parts[k].len; i += blockDim.x) {
      if (scatter) parts[k].base[i] = out[off + i];
      else out[off + i] = parts[k].base[i];
    }
    off += parts[k].len;
  }
}

// ---------------------------------------------------------------------------
// Eviction (CLOCK over rows; the engine is quiescent: no fill, accept or
// lookup of any of its batches in flight).
// ---------------------------------------------------------------------------
// keep[row] for rows in use: referenced since the last eviction, or a build
// still pending (its parent too: the child's build reads the parent's rows).
// Clears the reference bits.
__global__ void EvictMarkRowsKernel(CacheView c, int full, uint8_t* keep) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < c.C; r += gridDim.x * blockDim.x) {
    if (!(c.slot_meta[r] & (1 << 16))) continue;
    const bool pending = c.slot_built[r] < full;
    if (c.row_ref[r] || pending) keep[r] = 1;
    if (pending && c.slot_parent[r] >= 0) keep[c.slot_parent[r]] = 1;
    c.row_ref[r] = 0;
  }
}

// Rows a batch's next fill (or the one in flight, other parity) will read.
__global__ void EvictMarkBatchKernel(CacheView c, const int32_t* seq_slot, int n, uint8_t* keep) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int s = seq_slot[i];
    if (s < 0) continue;
    s &= ~kSlotWait;
    if (s < c.C) keep[s] = 1;
  }
}

__global__ void EvictRepairFreeKernel(CacheView c) {
  if (threadIdx.x == 0 && *c.row_free_n < 0) *c.row_free_n = 0;
}

// Resets and frees every row in use that is not kept.
__global__ void EvictFreeKernel(CacheView c, int nseg, const uint8_t* keep) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < c.C; r += gridDim.x * blockDim.x) {
    if (!(c.slot_meta[r] & (1 << 16)) || keep[r]) continue;
    c.slot_meta[r] = 0;
    c.slot_built[r] = 0;
    c.cd_segmask[r] = 0u;
    c.slot_parent[r] = -1;
    for (int g = 0; g < nseg; ++g) {
      const long long k = static_cast<long long>(r) * nseg + g;
      c.seg_done[k] = 0;
      c.seg_claim[k] = 0;
      c.cd_cnt[k] = 0;
      c.ci_cnt[2 * k] = 0;
      c.ci_cnt[2 * k + 1] = 0;
    }
    c.row_free[atomicAdd(c.row_free_n, 1)] = r;
    atomicAdd(c.counters + 5, 1ull);
    atomicAdd(c.counters + 0, ~0ull);  // one row fewer in use
  }
}

// Index rebuild: one warp per row in use inserts tag | row (the key hash
// of its stored key row).
__global__ void ReindexKernel(CacheView c) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < c.C; r += nw) {
    const int m = c.slot_meta[r];
    if (!(m & (1 << 16))) continue;
    const int n = m & 0xff, complete = (m >> 8) & 1;
    const int kv = lane < n ? c.slot_keys[r * kMaxContext + lane] : 0;
    const unsigned long long h = KeyHashWarp(kv, n, complete, lane);
    if (lane == 0) {
      const unsigned long long e = EntryTag(h) | static_cast<unsigned long long>(r);
      for (unsigned long long p = 0;; ++p) {
        const unsigned long long i = (h + p) & static_cast<unsigned long long>(c.IC - 1);
        if (atomicCAS(c.slot_hash + i, 0ull, e) == 0ull) break;
      }
    }
  }
}

__global__ void EvictFinishKernel(CacheView c) {
  if (threadIdx.x == 0) {
    atomicAdd(c.counters + 4, 1ull);
    if (c.host_free != nullptr) *reinterpret_cast<volatile int32_t*>(c.host_free) = *c.row_free_n;
  }
}

cudaError_t LaunchReindex(const CacheView& c, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(c.slot_hash, 0, static_cast<size_t>(c.IC) * 8, s);
  if (e != cudaSuccess) return e;
  ReindexKernel<<<(c.C + 7) / 8, 256, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t LaunchEvict(const CacheView& c, int nseg, const int32_t* const* seq_slots, const int* counts, int nb,
                        uint8_t* keep, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(keep, 0, static_cast<size_t>(c.C), s);
  if (e != cudaSuccess) return e;
  const int grid = (c.C + 255) / 256;
  EvictMarkRowsKernel<<<grid, 256, 0, s>>>(c, nseg * kChunksPerSeg, keep);
  for (int i = 0; i < nb; ++i) {
    if (counts[i] > 0) EvictMarkBatchKernel<<<(counts[i] + 255) / 256, 256, 0, s>>>(c, seq_slots[i], counts[i], keep);
  }
  EvictRepairFreeKernel<<<1, 32, 0, s>>>(c);
  EvictFreeKernel<<<grid, 256, 0, s>>>(c, nseg, keep);
  e = LaunchReindex(c, s);
  if (e != cudaSuccess) return e;
  EvictFinishKernel<<<1, 32, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t LaunchSnapshotRows(const CacheView& c, int W, int nseg, const int32_t* ids, int n, uint32_t* blocks,
                               bool scatter, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  SnapshotRowsKernel<<<n, 256, 0, s>>>(c, W, nseg, ids, n, blocks, scatter ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t LaunchRecountStructural(const CacheView& c, const VocabView& v) {
  RecountStructuralKernel<<<1184, 256>>>(c, v);
  return cudaGetLastError();
}

cudaError_t LaunchLookup(const CacheView& c, const BatchView& b, int queue, int tag, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  return Launch(LookupKernel, dim3((b.B + 127) / 128), dim3(128), 0, s, c, b, queue, tag);
}

cudaError_t LaunchDrain(const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b, int queue,
                        cudaStream_t s) {
  const size_t dyn = static_cast<size_t>(b.cap > kMaxContext ? b.cap : kMaxContext) * sizeof(int32_t);
  if (dyn > 48 * 1024) {
    cudaFuncSetAttribute(DrainKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
  }
  return Launch(DrainKernel, dim3(b.build_grid), dim3(kThreads), dyn, s, a, v, c, b, queue);
}

// Light items per CTA (<= 8 warps).  Measured: 7 per CTA for config 2's
// 4,096 items (586 CTAs: every SM holds 4, 28 items each) slows the step
// 32.6 -> 37.4 us against 8 (512 CTAs): the slots left free host accept CTAs
// while the fill runs.
static int LightPerCta(unsigned items) {
  (void)items;
  return PRE3_LIGHT_PER_CTA > 0 ? PRE3_LIGHT_PER_CTA : kWarps;
}

template <int MODE, int TAIL>
static void LaunchFillT(const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b,
                        const FillArgs& f, size_t dyn, cudaStream_t s) {
  // Static shared memory (span buffers) + the dynamic stack copy may pass the
  // 48 KB default: opt in to what this launch needs (once per size).
  static size_t opted = 0;
  if (dyn > 8 * 1024 && dyn > opted) {
    cudaFuncSetAttribute(FillKernel<MODE, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
    opted = dyn;
  }
  const unsigned items = static_cast<unsigned>(v.nseg) * static_cast<unsigned>(b.B);
  FillArgs g = f;
  g.light_per_cta = LightPerCta(items);
  const unsigned light = (items + g.light_per_cta - 1) / g.light_per_cta;
  unsigned grid = static_cast<unsigned>(b.h_grid) + light;
  if (g.accept_ctas > 0) {
    // Accept CTAs spread over the first PRE3_ACCEPT_SPREAD/8 of the light
    // CTAs: every accept is done well before the light pass ends.
    g.accept_ctas = (b.B + kWarps - 1) / kWarps;
    const unsigned span = std::max(1u, light * PRE3_ACCEPT_SPREAD / 8u);
    g.accept_period = static_cast<int>(std::max(1u, span / static_cast<unsigned>(g.accept_ctas)));
    grid += static_cast<unsigned>(g.accept_ctas);
  }
  Launch(FillKernel<MODE, TAIL>, dim3(grid), dim3(kThreads), dyn, s, a, v, c, b, g);
}

cudaError_t LaunchFill(int mode, int tail, const AutView& a, const VocabView& v, const CacheView& c,
                       const BatchView& b, FillArgs f, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  f.vec_ok = f.logits != nullptr && (f.ld % 8) == 0 && (reinterpret_cast<uintptr_t>(f.logits) % 16) == 0;
  const size_t dyn = static_cast<size_t>(b.cap > kMaxContext ? b.cap : kMaxContext) * sizeof(int32_t) + PRE3_FILL_SMEM_PAD;
  if (mode == kFillGreedy) {
    if (tail == kTailGreedy) {
      LaunchFillT<kFillGreedy, kTailGreedy>(a, v, c, b, f, dyn, s);
    } else {
      LaunchFillT<kFillGreedy, kTailNone>(a, v, c, b, f, dyn, s);
    }
  } else if (tail == kTailStream) {
    LaunchFillT<kFillMask, kTailStream>(a, v, c, b, f, dyn, s);
  } else if (f.accept_ctas > 0) {
    // The one-grid split step: its own instantiation, so the accept code
    // (and its register pressure) stays out of the plain fill.
    LaunchFillT<kFillMask, kTailSplit>(a, v, c, b, f, dyn, s);
  } else {
    LaunchFillT<kFillMask, kTailNone>(a, v, c, b, f, dyn, s);
  }
  return cudaGetLastError();
}

cudaError_t LaunchAccept(int sample, const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b,
                         const AcceptArgs& g, cudaStream_t s) {
  if (b.B == 0) return cudaSuccess;
  const int threads = 128;
  const int blocks = (b.B * 32 + threads - 1) / threads;
  switch (sample) {
    case kSampleGiven:
      Launch(AcceptKernel<kSampleGiven>, dim3(blocks), dim3(threads), 0, s, a, v, c, b, g);
      break;
    case kSampleStream:
      Launch(AcceptKernel<kSampleStream>, dim3(blocks), dim3(threads), 0, s, a, v, c, b, g);
      break;
    default:
      Launch(AcceptKernel<kSampleGreedy>, dim3(blocks), dim3(threads), 0, s, a, v, c, b, g);
      break;
  }
  return cudaGetLastError();
}

}  // namespace pre3
