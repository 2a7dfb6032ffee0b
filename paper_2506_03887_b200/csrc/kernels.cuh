// kernels.cuh — device views and kernel launchers (sm_100a).
// §3 (HBM layout) and §4 (kernels).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gm_internal.hpp"

namespace pre3 {

constexpr int kThreads = 256;                         // fill / build CTA size (8 warps)
constexpr int kSegWords = 256;                        // mask words per vocab segment
constexpr int kSegTokens = kSegWords * 32;            // 8192 tokens per segment
constexpr int kChunksPerSeg = kSegTokens / kThreads;  // build work units per segment
constexpr int kMaxContext = 32;                       // max K (one warp lane per key entry)
constexpr int kWalkOverlay = 256;                     // per-thread pushed-entry overlay in a mask walk
constexpr int kSlotWait = 1 << 30;                    // seq_slot flag: wait for the slot's build
// Fill numbers (heavy-list tags, double-buffer parity) count modulo 6: a tag
// only has to tell a fill from its neighbours, and a period dividing the
// 3-queue ring and the parity makes the host bookkeeping of any 6k steps
// return to its start state — so captured CUDA graphs of 6k steps replay.
constexpr int kFillPeriod = 6;

// Per-sequence device state: {depth, status, draws, reserved}.
struct SeqState {
  int32_t depth;
  int32_t status;
  uint32_t draws;
  int32_t reserved;
};

struct AutView {
  const int32_t* rec_begin;  // S*257+1
  const CandRec* recs;
  const CandRec* first;      // S*257 dense first candidates
  // Condition index (FlatLayout::hidx_*): {lens offset, count | max len << 16}
  // per (state, terminal) (count 0 = scan), lengths, exact and prefix tables.
  const int2* hidx_meta;
  const int16_t* hidx_lens;
  const unsigned long long* hidx_exact;   // {key, candidate} pairs
  const unsigned long long* hidx_prefix;  // keys
  unsigned long long hidx_exact_mask;     // slots - 1
  unsigned long long hidx_prefix_mask;
  const int32_t* rec_cond;   // 16-B aligned lists
  const int32_t* rec_push;   // 16-B aligned lists
  const int32_t* shift;       // S*256
  const uint32_t* state_any;  // S*9
  int32_t num_states;
  int32_t initial;
};

struct VocabView {
  const int32_t* tok_off;  // V+1 byte offsets
  const uint8_t* tok_bytes;
  const int4* tok_rec;         // V+1: {offset, length, bytes 0-3, bytes 4-7} (entry V: EOS, length 1)
  const uint32_t* structural;  // W words
  int32_t V;                   // regular tokens; EOS = V
  int32_t W;                   // ceil((V+1)/32)
  int32_t nseg;                // ceil(W / kSegWords)
  // The model's logit-row layout (gm_engine_options num_columns/eos_column):
  // column c < ncols holds mask bit V if c == eos_col, else bit c if c < V,
  // else a special token (-inf in every fused logits call).  layout == 0:
  // the reference layout (ncols = V + 1, eos_col = V).  Token ids at the ABI
  // are columns (EOS = eos_col) once a layout is set.
  int32_t ncols;
  int32_t eos_col;
  int32_t layout;
};

// Context cache (engine-wide, shared by batches on the device).  Key =
// (n = min(depth, K), complete = depth <= K, the top n stack entries) ->
// {CI: tokens accepted whatever lies below the key, CD: tokens whose walk
// reaches below the key} as two W-word bitsets, plus per-segment CD counts
// and build-completion counters.
// Rows (the "slots" every other array indexes, seq_slot values) are reached
// through an open-addressing index of IC = 2C positions holding
// tag << 24 | row (0: empty; row kRowPending: claimed, row being published),
// so a row can be evicted and reused without moving any data: eviction
// (EvictKernels, gm_engine_evict) rebuilds the index from the live rows.
constexpr unsigned long long kRowMask = 0xFFFFFFull;
constexpr int kRowPending = 0xFFFFFF;
struct CacheView {
  unsigned long long* slot_hash;  // IC index entries
  int32_t* slot_meta;             // C; n | complete << 8 | ready << 16 (0: a free row)
  int32_t* slot_keys;             // C*kMaxContext (rows padded with -1)
  uint32_t* ci;                   // C*W
  uint32_t* cdb;                  // C*W
  int32_t* cd_cnt;                // C*nseg
  int32_t* seg_done;              // C*nseg completed build units (kChunksPerSeg = built)
  int32_t* seg_claim;             // C*nseg build chunks claimed (queue units and helpers draw from it,
                                  //    so each chunk of a shared slot is built exactly once by whoever
                                  //    gets there first — a batch never waits on another batch's queue)
  int32_t* slot_built;            // C completed build units over all segments
  uint32_t* cd_segmask;           // C: bit s set when segment s has context-dependent tokens
  int32_t* ci_cnt;                // C*nseg*2: per segment, CI tokens (EOS excluded) and CI ∩ structural
  int32_t* slot_parent;           // C: context a new one is built from (-1: full build)
  int32_t* row_free;              // C: free-row stack, entries [0, *row_free_n)
  int32_t* row_free_n;            // free rows left (dips below 0 while pops fail; eviction repairs it)
  uint8_t* row_ref;               // C: reference bits (lookups set, eviction clears: CLOCK)
  int32_t* host_free;             // host-mapped: free rows after the latest pop (auto-eviction trigger)
  unsigned long long* counters;   // [0] rows in use, [1] segment builds, [2] private builds, [3] parent-based
                                  // builds, [4] evictions, [5] rows evicted
  int32_t C;
  int32_t IC;                     // index positions (power of two, 2C)
  int32_t K;
  int32_t R;                      // parent key depth (0: no parents)
  int32_t W;                      // mask words per row
  int32_t eos_word;               // V >> 5 (the EOS bit's word)
  uint32_t eos_bit;               // 1 << (V & 31)
  uint32_t eos_segbit;            // logit layout with the EOS column among the regular ids: bit of that
                                  //    column's segment (EosSegExtra), else 0
};

// Build work queue: items {slot, seg, seq, 0}; units = items * kChunksPerSeg.
// Per-step work descriptor produced by the lookups for the next fill: build
// items {slot, seg, seq, 0} (units = items * kChunksPerSeg) and the "heavy"
// (sequence, segment) pairs — those with context-dependent tokens or a
// pending build — that the fill schedules first.
struct BuildQueue {
  int4* items;
  unsigned int* n_items;
  unsigned int* next_unit;
  int2* heavy;
  unsigned int* n_heavy;
};

struct BatchView {
  SeqState* seq;
  int32_t* stacks;  // B*cap, bottom first
  int32_t cap;
  int32_t B;
  int32_t nseg;
  int32_t* seq_slot;        // [2][B] by fill parity: cache slot, C+b = private row, -2 = not alive;
                            //    | kSlotWait when the slot's build may still be pending
  uint32_t* seq_hmask;      // [2][B] by fill parity: the sequence's heavy segments (0: pure CI —
                            //    its mask is the slot's CI row)
  uint32_t* priv;           // B*W private (uncached) masks
  int32_t* priv_done;       // B*nseg build-completion counters of private rows
  int32_t* heavy_index;     // B*nseg: index in the consumed heavy list, or -1
  int32_t h_cap;            // heavy list capacity
  int32_t h_grid;           // heavy-pass CTAs of a fill grid (they loop over the list)
  BuildQueue queue[3];      // ring: lookups feed queue[p], fill drains it, the next fill resets it
  int32_t* seq_arrive;      // B: fill CTAs finished per sequence (fused tail)
  unsigned int* kernel_done;  // CTAs finished per launch (queue reset)
  unsigned int* err;                  // bit0: walk overlay overflow
  unsigned long long* stats;          // [0] rd bytes, [1] wr bytes, [2] walks, [3] -, [4] private
  unsigned long long* counters;       // [0] restarts, [1] draws, [2] fills, [3] accepts
  int32_t stats_enabled;
  int32_t build_grid;
  // Diagnostics (null = off): per-event records {kind | seg << 8 | b << 32,
  // t_start, t_end, extra} (globaltimer ns); trace[0..3] holds the count.
  unsigned long long* trace;
  int32_t trace_cap;
};

enum TraceKind { kTraceLight = 1, kTraceHeavy = 2, kTraceTail = 3, kTraceAccept = 4 };

#ifndef PRE3_ONE_GRID_CTAS_PER_SM
#define PRE3_ONE_GRID_CTAS_PER_SM (1 << 20)  // one-grid split step up to this many light CTAs per SM (no limit)
#endif
#ifndef PRE3_SPLIT_ONE_GRID
#define PRE3_SPLIT_ONE_GRID 1  // split step: the accepts as CTAs of the fill's grid (0: a PDL accept kernel)
#endif

enum FillMode { kFillMask = 0, kFillGreedy = 1 };
enum FillTail { kTailNone = 0, kTailStream = 1, kTailGreedy = 2, kTailSplit = 3 };  // kTailSplit: the one-grid split step
// The fill's last item of a sequence runs sample + accept (the one-launch steps).
__host__ __device__ constexpr bool FusedTail(int tail) { return tail == kTailStream || tail == kTailGreedy; }
enum SampleMode { kSampleGiven = 0, kSampleStream = 1, kSampleGreedy = 2 };

struct AcceptArgs {
  const int32_t* tokens;
  int32_t* status_out;
  int restart;
  const uint32_t* bitmask;
  long long ldw;
  const int32_t* seg_counts;
  unsigned long long seed;
  unsigned long long* best;
  int32_t* tokens_out;
  int do_accept;     // 0: sample only
  int lookup_queue;  // >= 0: assign next-fill context slots into this queue
  int lookup_tag;    // number of the fill that consumes it
  int wait_fill;     // overlap the preceding fill (publish_arrival): per-sequence start
  int ci_shortcut;   // with wait_fill, bitmask/seg_counts from that fill, unmodified: a pure-CI
                     // sequence samples from its slot's CI row and counts without waiting
};

struct FillArgs {
  uint32_t* bitmask;        // [B][ldw] (never null with a tail)
  long long ldw;
  uint16_t* logits;         // bf16 [B][ld] or null
  long long ld;
  int32_t* seg_counts;      // [B][nseg][2] or null (required by the stream tail)
  unsigned long long* best; // [B] greedy partials
  int32_t* tokens_out;      // tail: sampled ids or null
  unsigned long long seed;  // stream tail
  int consume;              // build queue drained by this launch
  int produce;              // build queue fed by the tail's lookups
  int reset;                // queue drained by the previous fill, emptied here (-1: none)
  int fill_no;              // this fill's number (heavy_index tags; the tail tags fill_no + 1)
  int publish_arrival;      // no tail: still count finished items per sequence (seq_arrive) so a
                            // following AcceptKernel with wait_fill can start per sequence;
                            // 2: only the items of a sequence's heavy segments (the accept's
                            // ci_shortcut takes the other segments from the slot's CI row)
  int vec_ok;               // set by LaunchFill
  int light_per_cta;        // light items per CTA (<= kThreads/32; set by LaunchFill so the
                            // light CTAs fill whole waves of the SMs' CTA slots)
  int accept_ctas;          // split step in one grid: this many CTAs (kThreads/32 sequences
                            // each) run AcceptSeq with `acc`, one after every accept_period
                            // light CTAs (set by LaunchFill; 0: none)
  int accept_period;
  AcceptArgs acc;
};


struct SampleArgs {
  const uint32_t* bitmask;   // [B][ldw], from a preceding fill
  long long ldw;
  const uint16_t* logits;    // bf16 [B][ld]
  long long ld;
  float temperature;         // > 0
  int top_k;                 // 0 = off
  uint32_t top_p24;          // floor(top_p * 2^24); 2^24 = off
  unsigned long long seed;
  int32_t* tokens_out;
  int do_accept;
  int restart;
  int lookup_queue;
  int lookup_tag;
  int vec_ok;                // set by LaunchSample
};

// Temperature / top-k / top-p sampling over the allowed tokens (+ accept).
cudaError_t LaunchSample(const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b,
                         SampleArgs s, cudaStream_t st);
cudaError_t LaunchReset(const AutView& a, const BatchView& b, cudaStream_t s);
// Engine::AllowedTerminals per sequence: out[b*9 .. b*9+8].
cudaError_t LaunchAllowed(const AutView& a, const BatchView& b, uint32_t* out, cudaStream_t s);
cudaError_t LaunchLookup(const CacheView& c, const BatchView& b, int queue, int tag, cudaStream_t s);
cudaError_t LaunchRecountStructural(const CacheView& c, const VocabView& v);
// Eviction (quiescent engine): keep = rows referenced since the last
// eviction, rows with builds pending and their parents, and rows named by
// the given seq_slot arrays; the rest are reset and freed, then the index is
// rebuilt from the live rows.  Returns the launch error.
cudaError_t LaunchEvict(const CacheView& c, int nseg, const int32_t* const* seq_slots, const int* counts, int nb,
                        uint8_t* keep, cudaStream_t s);
// Rebuilds the index from the rows in use (snapshot loads).
cudaError_t LaunchReindex(const CacheView& c, cudaStream_t s);
// Snapshot rows of n listed slots <-> blocks of kMaxContext + 3*nseg + 2*W words.
cudaError_t LaunchSnapshotRows(const CacheView& c, int W, int nseg, const int32_t* ids, int n, uint32_t* blocks,
                               bool scatter, cudaStream_t s);
cudaError_t LaunchDrain(const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b, int queue,
                        cudaStream_t s);
// Help-build + fill (+ bf16 -inf masking or greedy argmax) (+ fused tail).
cudaError_t LaunchFill(int mode, int tail, const AutView& a, const VocabView& v, const CacheView& c,
                       const BatchView& b, FillArgs f, cudaStream_t s);
cudaError_t LaunchAccept(int sample, const AutView& a, const VocabView& v, const CacheView& c, const BatchView& b,
                         const AcceptArgs& g, cudaStream_t s);

}  // namespace pre3
