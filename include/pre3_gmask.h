/*
 * include/pre3_gmask.h — the drop-in C ABI of the B200-native constrained
 * decoding hot path (Pre^3, arxiv 2506.03887).
 *
 * It replaces the reference matcher's per-step runtime, `gmask::Engine`
 * (/root/reference/proj/include/gmask/runtime.hpp:92-166,
 * src/runtime.cpp:92-307), and its CPU "kernels" plugin table
 * (include/gmask/kernels.hpp:31-54) with batched sm_100a CUDA.  Every entry
 * point below names the reference interface it replaces.  Plain C types only:
 * pointers are device pointers unless documented as host pointers; streams
 * are `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 *
 * Conventions:
 *   - V regular tokens, token ids 0..V-1 in vocabulary order; EOS is id V
 *     and mask bit V (runtime.hpp:62-85, TokenMask::SetEos).
 *   - A mask row is W = ceil((V+1)/32) uint32 words; bit t = word t/32,
 *     bit t%32 — the little-endian image of the reference's uint64 words.
 *   - Calls that take a stream are asynchronous and enqueue kernels only;
 *     there is no internal locking: one gm_batch per stream.
 *   - Return value: GM_OK or a GM_ERR_* code; gm_last_error() returns a
 *     thread-local message.  The codes mirror the reference's exception
 *     kinds (GrammarError / BuildError / SerializeError / VocabError) and CLI
 *     exit codes (tools/gmask_main.cpp:317-335).
 */
#ifndef PRE3_GMASK_H_
#define PRE3_GMASK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GM_ABI_VERSION 2

enum gm_status_code {
  GM_OK = 0,
  GM_ERR_GRAMMAR = 2,         /* GrammarError (grammar.hpp:34-49) */
  GM_ERR_BUILD = 3,           /* BuildError (lr1.hpp:20-29) */
  GM_ERR_CORRUPT_INPUT = 4,   /* SerializeError (serialize.hpp:17-25) */
  GM_ERR_CUDA = 5,            /* CUDA runtime failure / no device */
  GM_ERR_STACK_OVERFLOW = 6,  /* a device stack or walk overlay overflowed */
  GM_ERR_VOCAB_EMPTY = 7,     /* VocabError::kEmptyToken (runtime.hpp:29-37) */
  GM_ERR_VOCAB_DUPLICATE = 8, /* VocabError::kDuplicateToken */
  GM_ERR_SNAPSHOT_MISMATCH = 9, /* a context snapshot taken for another automaton / vocabulary / K, R, slots */
  GM_ERR_USAGE = 64           /* bad argument (CLI exit 64) */
};

/* Per-sequence status; 0..2 are runtime.hpp:19 `Status`, 3 is new. */
enum gm_seq_status {
  GM_ALIVE = 0,
  GM_DEAD = 1,
  GM_ACCEPTED = 2,
  GM_OVERFLOW = 3 /* stack exceeded the batch's stack_capacity */
};

typedef struct gm_automaton gm_automaton; /* host: compiled DPDA (gmask::Dpda) */
typedef struct gm_engine gm_engine;       /* device: automaton + vocab + context cache */
typedef struct gm_batch gm_batch;         /* device: B sequences' (state, status, stack) */
typedef struct gm_graph gm_graph;         /* a captured CUDA graph of decode steps of one batch */

const char* gm_last_error(void);
int gm_abi_version(void);

/* ------------------------------------------------------------ automaton */
/* Loads a compiled automaton from a host buffer in either format, told apart
 * by the magic: the reference's GMASKDP1 (DeserializeDpda,
 * src/serialize.cpp:198-294: sorted-key JSON; arbitration order re-derived
 * and determinism re-checked; errors = SerializeError kinds) or the flat
 * P3DPDA v1 of DESIGN.md §3 (shapes, id ranges, edge ranges validated). */
int gm_automaton_load(const void* data, size_t bytes, gm_automaton** out);
/* SerializeDpda (src/serialize.cpp:148-196): byte-identical GMASKDP1 text of
 * an automaton (composites / cycles / stats are empty for one loaded from
 * P3DPDA).  *size receives the length (buf = NULL to query). */
int gm_automaton_save_gmaskdp1(const gm_automaton* a, void* buf, size_t cap, size_t* size);
/* LoadVocabulary (src/serialize.cpp:348-364): a JSON array of strings, each
 * `\xNN` / `\\` unescaped, into tok_bytes / tok_offsets[n+1] (host).  Call
 * with tok_bytes = NULL to get *num_tokens and *total_bytes. */
int gm_vocab_load_json(const void* data, size_t bytes, uint8_t* tok_bytes, int64_t bytes_cap,
                       int64_t* tok_offsets, int32_t tokens_cap, int32_t* num_tokens,
                       int64_t* total_bytes);
/* Compiles grammar text (line-oriented BNF, grammar.hpp:1-10) into an
 * automaton: ParseGrammar + BuildDpda (src/dpda_builder.cpp:478-522).
 * aggregate/merge mirror BuildOptions (dpda.hpp:73-80). */
int gm_automaton_compile(const char* grammar_text, int aggregate, int merge,
                         gm_automaton** out);
/* Serializes to P3DPDA v1 into a host buffer; returns the size via *size
 * (call with buf=NULL to query). */
int gm_automaton_save(const gm_automaton* a, void* buf, size_t cap, size_t* size);
int gm_automaton_destroy(gm_automaton* a);
/* info[0..7] = num_states, num_edges, initial_state, accept_state,
 * max |match_pop|, max |push|, dynamic edges, grammar_hash. */
int gm_automaton_info(const gm_automaton* a, int64_t info[8]);
/* Compile statistics of an automaton made by gm_automaton_compile (zero for
 * loaded ones): stats[0] = two-terminal composites MergeEdges would build
 * (optimizer.cpp:78-136; sequence-runner only, not part of the device
 * automaton), stats[1] = rewritten pumping circuits (DetectCycles,
 * dpda_builder.cpp:340-364), stats[2..3] = 0. */
int gm_automaton_compile_stats(const gm_automaton* a, int64_t stats[4]);

/* ------------------------------------------------------------ engine */
typedef struct gm_engine_options {
  int32_t context_depth;   /* K: stack entries keying the context cache (1..32; default 8) */
  int32_t context_slots;   /* context rows (the cache's capacity), power of two (default 8192); the
                              row index has 2x as many positions */
  int64_t parent_depth;    /* R < K: a new context is built from the context of the same stack
                              top keyed R deep, walking only that context's context-dependent
                              tokens (0 = default min(4, K-1); negative = off) */
  int32_t segment_words;   /* vocab segment size in mask words (default 256) */
  /* ABI v2: the model's logit-row layout (all zero = the
   * reference's: V + 1 columns, EOS in column V). */
  int32_t num_columns;     /* logit columns per row (0 = V + 1) */
  int32_t eos_column;      /* column of the EOS logit = mask bit V (used when num_columns > 0) */
  const uint32_t* disabled; /* host bitmask (W words) of token ids < V that are never allowed (model
                               specials or alias ids among the regular ids; their bytes are ignored
                               and may be empty), or NULL */
  /* Context eviction (CLOCK): when fewer than auto_evict_free rows are free
   * at the start of a batch's fill, rows not referenced since the previous
   * eviction — and not read by any batch's next fill or a pending build —
   * are freed for reuse (gm_engine_evict, run on that batch's stream; the
   * engine's other batches must be idle then).  0 = off: a full table falls
   * back to per-sequence private rows (correct, slower). */
  int32_t auto_evict_free;
} gm_engine_options;

/* Engine::Engine (runtime.cpp:92-113) + TokenTrie::Build (runtime.cpp:18-61)
 * on `device`: uploads the flattened automaton, the vocabulary (host
 * `tok_bytes`, `tok_offsets[num_tokens+1]`) and allocates the context cache.
 * Empty / duplicate tokens fail with GM_ERR_VOCAB_* exactly where
 * TokenTrie::Build throws (disabled ids are exempt).  opts may be NULL.
 *
 * Logit layout (opts->num_columns > 0): every fused logits call (mask,
 * greedy, sample) reads/writes columns [0, num_columns): column eos_column
 * carries mask bit V (EOS), columns c < V carry bit c, every other column is
 * a special token and gets -inf (never sampled).  eos_column < V requires
 * that id to be disabled.  Token ids at the ABI (tokens_out, gm_accept_tokens)
 * are then model columns: EOS = eos_column; ids >= V other than eos_column
 * and disabled ids are invalid (the sequence goes GM_DEAD).  Bitmask rows
 * keep the reference layout (bit V = EOS).  Greedy/sampler ties are broken
 * in mask-bit order (EOS last). */
int gm_engine_create(const gm_automaton* a, const uint8_t* tok_bytes,
                     const int64_t* tok_offsets, int32_t num_tokens,
                     const gm_engine_options* opts, int device, gm_engine** out);
int gm_engine_destroy(gm_engine* e);
/* info[0..7] = V, W, num_segments, context slots used, segment builds,
 * private (uncached) rows built, contexts built from a parent context, device */
int gm_engine_info(gm_engine* e, int64_t info[8]);
/* Host bitmask (W words) of "structural" tokens used by the synthetic
 * stream sampler (tokens containing any of {}[],:" ). */
int gm_engine_set_structural(gm_engine* e, const uint32_t* host_words);
/* Preprocessing: populates the context cache by running `steps` synthetic
 * stream decode steps over `batch` scratch sequences (seeded by `seed`) on
 * the device, stacks of `stack_capacity` entries (<= 0: 1024; overflow
 * restarts a sequence); synchronizes `stream`.  Results of later fills are
 * identical with or without it (the cache only changes speed). */
int gm_engine_prewarm(gm_engine* e, int32_t batch, int32_t steps, uint64_t seed, int32_t stack_capacity,
                      void* stream);

/* Context eviction now (see gm_engine_options::auto_evict_free): every
 * batch of the engine must be idle (their streams synchronized, or all
 * work on `stream`).  Rows never move, so batches, captured graphs and
 * pending builds stay valid; later fills rebuild any evicted context they
 * meet.  Results are unchanged (the cache only changes speed). */
int gm_engine_evict(gm_engine* e, void* stream);
/* Context-table counters: [0] rows, [1] rows in use, [2] free rows,
 * [3] index positions, [4] evictions, [5] rows evicted, [6] private-row
 * builds (table full), [7] segment builds. */
int gm_engine_cache_stats(gm_engine* e, int64_t out[8]);

/* Context-table snapshot "P3GMCTX1" (the reference's cache
 * precedent: SerializeDpda / DeserializeDpda, src/serialize.cpp:148-294).
 * save: every fully built context slot into a host buffer (buf = NULL:
 * query *size); synchronizes the device.  load: into an engine whose
 * context table is still empty, created from the same automaton (grammar
 * hash, dpda_builder.cpp:469-476, + device-layout hash), vocabulary and
 * logit layout, K, R and slot count — else GM_ERR_SNAPSHOT_MISMATCH;
 * truncated or altered data -> GM_ERR_CORRUPT_INPUT (checksummed).  A loaded
 * table gives the same masks as the prewarm that built it (the cache only
 * changes speed), without running it. */
int gm_engine_snapshot_save(gm_engine* e, void* buf, uint64_t cap, uint64_t* size);
int gm_engine_snapshot_load(gm_engine* e, const void* buf, uint64_t bytes);

/* ------------------------------------------------------------ batch */
/* B sequences with fixed-capacity device stacks (reference stacks are
 * unbounded vectors; exceeding capacity yields GM_OVERFLOW). */
int gm_batch_create(gm_engine* e, int32_t batch, int32_t stack_capacity, gm_batch** out);
int gm_batch_destroy(gm_batch* b);
/* Engine::InitialConfig (runtime.cpp:115-121) for every sequence. */
int gm_batch_reset(gm_batch* b, void* stream);
/* Host-side parity helpers (synchronous). */
int gm_batch_download(gm_batch* b, int32_t seq, int32_t* state, int32_t* status,
                      int32_t* stack, int32_t cap, int32_t* depth);
int gm_batch_upload(gm_batch* b, int32_t seq, int32_t status, const int32_t* stack,
                    int32_t depth);
/* Synchronizes `stream` and reports device-side errors (GM_ERR_STACK_OVERFLOW
 * if a mask walk overflowed its overlay; GM_ERR_CUDA if an accept's bounded
 * wait for its fill's per-sequence items expired — an internal error, never
 * raised by a sequence of calls this header allows); clears them. */
int gm_batch_check(gm_batch* b, void* stream);
/* counters[0..3] = restarts, total draws, mask fills, accepts */
int gm_batch_counters(gm_batch* b, int64_t counters[4]);

/* ------------------------------------------------------------ hot path */
/* Engine::ComputeMask (runtime.cpp:280-287) for every sequence:
 * bitmask[b * ld_words + w], ld_words >= W.  Non-alive sequences get an
 * all-zero row (runtime.cpp:282). */
int gm_fill_next_token_bitmask(gm_batch* b, uint32_t* bitmask, int64_t ld_words, void* stream);

/* The same fill fused with bf16 logit masking, in place: logits[b*ld + t] =
 * -inf wherever mask bit t is 0, for t in [0, V]; other entries untouched.
 * bitmask may be NULL.  seg_counts (may be NULL) receives per (sequence,
 * segment) {allowed regular tokens, allowed structural tokens} for the
 * stream sampler. */
int gm_fill_and_mask_logits(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits_bf16,
                            int64_t ld, int32_t* seg_counts, void* stream);

/* One fused decode step in a single launch: the fill above (bitmask and
 * logits may be NULL), then per sequence the synthetic-stream sample
 * (DESIGN.md §5), accept (with restart of finished sequences) and the context
 * lookup of the next step.  Equivalent to gm_fill_and_mask_logits followed by
 * gm_sample_stream_and_accept. */
int gm_decode_step_stream(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits_bf16,
                          int64_t ld, uint64_t seed, int32_t* tokens_out, void* stream);

/* The same step with the sample/accept/lookup overlapping the fill — a
 * sequence whose mask is exactly its context's
 * cached CI row (no context-dependent tokens) samples from that
 * row at once; the others start as soon as their own fill items are in.
 * Same results as gm_decode_step_stream.  seg_counts may be NULL (internal
 * buffer); when given it receives the fill's counts as in
 * gm_fill_and_mask_logits. */
int gm_decode_step_stream_split(gm_batch* b, uint32_t* bitmask, int64_t ld_words, uint16_t* logits_bf16,
                                int64_t ld, int32_t* seg_counts, uint64_t seed, int32_t* tokens_out,
                                void* stream);
/* Kernel launches of one gm_decode_step_stream_split of this batch in the
 * steady state: 1 when the accepts run as CTAs of the fill's grid
 * (interleaved with its light CTAs; the default), 2 for the fill + a
 * programmatically dependent accept kernel (environment
 * PRE3_SPLIT_TWO_KERNELS=1 when the batch was created); -GM_ERR_USAGE for a
 * NULL batch. */
int gm_batch_split_step_launches(gm_batch* b);

/* Engine::AllowedTerminals (runtime.cpp:188-208) for every sequence: the
 * exact next-byte set plus $ — terminal t is allowed iff an edge of the
 * current state accepting t has a condition matching the stack.  out is a
 * device array of B x 9 words: bit t of word t/32 for bytes t < 256, $ = bit 0
 * of word 8.  Non-alive sequences get all zero. */
int gm_allowed_terminals(gm_batch* b, uint32_t* out, void* stream);

/* Engine::Step over every byte of tokens[b] (runtime.cpp:177-186; callers'
 * loop gmask_main.cpp:113-118); tokens[b] == V steps kEndMarker; tokens[b] < 0
 * is a no-op.  status_out (may be NULL) receives gm_seq_status per sequence.
 * restart != 0 re-initializes sequences that end non-alive (decode loops). */
int gm_accept_tokens(gm_batch* b, const int32_t* tokens, int32_t* status_out, int32_t restart,
                     void* stream);

/* Synthetic-stream sampler fused with accept: picks each
 * sequence's token from the bitmask + seg_counts of the preceding
 * gm_fill_and_mask_logits, writes it to tokens_out (may be NULL), accepts it
 * and restarts finished sequences (accepted, dead, overflow) and dead ends
 * (nothing allowed: token -1) from InitialConfig.  `seed` keys the
 * per-sequence streams. */
int gm_sample_stream_and_accept(gm_batch* b, const uint32_t* bitmask, int64_t ld_words,
                                const int32_t* seg_counts, uint64_t seed, int32_t* tokens_out,
                                void* stream);

/* The same sampler without the accept: tokens_out receives each sequence's
 * pick (-1 when nothing is allowed) and the stream advances; the caller
 * accepts them later with gm_accept_tokens (e.g. after a host round trip). */
int gm_sample_stream(gm_batch* b, const uint32_t* bitmask, int64_t ld_words, const int32_t* seg_counts,
                     uint64_t seed, int32_t* tokens_out, void* stream);

/* Greedy decode step (config 5): fill + argmax over allowed bf16 logits (the
 * row is read, not written; ties -> lowest id) + accept + restart (finished
 * sequences and dead ends).  tokens_out receives the chosen ids (-1 when
 * nothing is allowed). */
int gm_decode_step_greedy(gm_batch* b, const uint16_t* logits_bf16, int64_t ld, uint32_t* bitmask,
                          int64_t ld_words, int32_t* tokens_out, void* stream);

/* Temperature / top-k / top-p sampling over each sequence's allowed tokens
 * (new work): keep the allowed tokens whose logit is among the
 * top_k largest (0 = all; ties at the threshold kept), weight them by
 * exp((logit - max) / temperature) in exact 2^-32 fixed point, keep the
 * smallest key-descending prefix holding top_p of the weight (ties kept),
 * and draw from it with the sequence's stream draw (seed, draws).  Integer
 * results are bit-exact with oracle/gmask_port.c gp_sample_pick.  accept != 0
 * also accepts the token (Engine::Step per byte), restarts finished sequences
 * and looks up the next context — no host round trip.  bitmask comes from a
 * preceding fill of the same batch. */
int gm_sample_tokens(gm_batch* b, const uint16_t* logits_bf16, int64_t ld, const uint32_t* bitmask,
                     int64_t ld_words, float temperature, int32_t top_k, float top_p, uint64_t seed,
                     int32_t* tokens_out, int32_t accept, void* stream);
/* One decode step with that sampler: gm_fill_next_token_bitmask (bitmask may
 * be NULL) then gm_sample_tokens(accept = 1). */
int gm_decode_step_sample(gm_batch* b, const uint16_t* logits_bf16, int64_t ld, uint32_t* bitmask,
                          int64_t ld_words, float temperature, int32_t top_k, float top_p, uint64_t seed,
                          int32_t* tokens_out, void* stream);

/* CUDA graph of `steps` decode steps of batch b (a positive multiple of 6:
 * the period of the step bookkeeping), so a serving loop launches N steps
 * with one host call.  kind 0 = gm_decode_step_stream_split, 1 =
 * gm_decode_step_greedy; step i uses bitmask[i], logits[i], seg_counts[i],
 * tokens_out[i] (each array may be NULL: no bitmask output / internal
 * scratch / no ids; logits may be NULL for kind 0 = mask only).  The
 * pointers are baked into the graph.  Capture runs on an internal stream and
 * executes nothing except, if needed, the context lookup of the next step.
 * gm_graph_launch replays the steps on `stream`; the batch must be at the
 * state the graph was captured from (true after every replay and after any
 * 6k eager steps of the same kind), else GM_ERR_USAGE. */
int gm_decode_graph_create(gm_batch* b, int32_t kind, int32_t steps, uint32_t* const* bitmask, int64_t ld_words,
                           const uint16_t* const* logits, int64_t ld, int32_t* const* seg_counts, uint64_t seed,
                           int32_t* const* tokens_out, gm_graph** out);
int gm_graph_launch(gm_graph* g, void* stream);
int gm_graph_destroy(gm_graph* g);

/* Measurement hook (diagnostics): the next fill kernel launched for this
 * batch, by any call, is bracketed by cudaEventRecord(start_event) and
 * cudaEventRecord(end_event) on its stream (cudaEvent_t handles; one-shot).
 * In an overlapped step the following kernel then cannot start under it; a
 * one-grid split step's fill kernel includes its sample/accept CTAs. */
int gm_batch_time_next_fill(gm_batch* b, void* start_event, void* end_event);

/* Statistics accumulated while enabled (gm_batch_set_stats), reset on read:
 * stats[0] = logits bytes read, [1] = logits bytes written (16-B chunk
 * granularity), [2] = context-dependent token walks, [3] = build items,
 * [4] = private segment fills, [5] = segment fills that gave up waiting
 * for a context build and walked every token (should stay 0: a fill builds
 * any unclaimed chunk itself, whichever batch queued it). */
int gm_batch_fill_stats(gm_batch* b, int64_t stats[6]);
int gm_batch_set_stats(gm_batch* b, int32_t enable);
/* Diagnostics: per-item timing records of later fill / accept launches into
 * a device buffer of 4 * (capacity + 1) uint64 (NULL turns tracing off).
 * trace[0] counts records; record i at trace[4*(i+1)] = {kind | seg << 8 |
 * seq << 32, start ns, end ns, extra}; kind 1 light fill item, 2 heavy fill
 * item, 3 fused tail, 4 accept.  The caller zeroes trace[0]. */
int gm_batch_set_trace(gm_batch* b, uint64_t* trace, int32_t capacity);

#ifdef __cplusplus
}
#endif
#endif /* PRE3_GMASK_H_ */
