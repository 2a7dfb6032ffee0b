/* oracle/gmask_port.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference matcher's runtime (the hot path that
 * the CUDA kernels replace), operating on this repo's flat automaton format
 * (P3DPDA v1).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker.
 *
 * Each function cites the reference file:line it restates
 * (/root/reference/proj/...).  The restatement is pinned against the
 * reference itself (oracle/_ref/libgmask_ref.so, built from the reference's
 * own sources) and against the golden vectors in tests/golden/.
 */
#ifndef GMASK_PORT_H_
#define GMASK_PORT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gp_automaton gp_automaton;
typedef struct gp_trie gp_trie;

/* runtime.hpp:19 Status {kAlive, kDead, kAccepted} */
enum { GP_ALIVE = 0, GP_DEAD = 1, GP_ACCEPTED = 2 };

/* runtime.hpp:23-27 RuntimeConfig: stack bottom first; growable. */
typedef struct gp_config {
  int32_t state;
  int32_t status;
  int32_t depth;
  int32_t cap;
  int32_t* stack;
} gp_config;

gp_automaton* gp_automaton_load(const uint8_t* buf, int64_t n);
void gp_automaton_free(gp_automaton* a);
int32_t gp_num_states(const gp_automaton* a);
int32_t gp_num_edges(const gp_automaton* a);

/* err_kind: 0 ok, 1 empty token, 2 duplicate token (runtime.cpp:18-61). */
gp_trie* gp_trie_build(const uint8_t* bytes, const int64_t* offs, int32_t n, int* err_kind);
void gp_trie_free(gp_trie* t);
int32_t gp_trie_nodes(const gp_trie* t);

void gp_config_init(const gp_automaton* a, gp_config* c); /* runtime.cpp:115-121 */
void gp_config_copy(gp_config* dst, const gp_config* src);
void gp_config_free(gp_config* c);

int gp_step(const gp_automaton* a, gp_config* c, int32_t terminal);             /* 177-186 */
void gp_allowed(const gp_automaton* a, const gp_config* c, uint64_t bytes[4], int* dollar); /* 188-208 */
void gp_mask(const gp_automaton* a, const gp_config* c, const gp_trie* t, uint32_t* words); /* 261-287 */
void gp_mask_naive(const gp_automaton* a, const gp_config* c, const uint8_t* bytes,
                   const int64_t* offs, int32_t n, uint32_t* words);               /* 289-307 */

/* DESIGN.md §5 samplers (new work; identical rule on the device). */
uint64_t gp_stream_draw(uint64_t seed, uint64_t seq, uint64_t draw);
int32_t gp_stream_pick(const uint32_t* mask, const uint32_t* structural, int32_t V, uint64_t u);
int32_t gp_greedy_pick(const uint32_t* mask, const uint16_t* logits_bf16, int32_t V);
/* Temperature / top-k / top-p pick (kernels.cu SampleKernel rule); u = the
 * sequence's stream draw; top_p24 = floor(top_p * 2^24) (2^24 = off). */
int32_t gp_sample_pick(const uint32_t* mask, const uint16_t* logits_bf16, int32_t V, float temperature,
                       int32_t top_k, uint32_t top_p24, uint64_t u);
uint64_t gp_sample_weight(uint32_t key, float vmax, float temperature);

/* Options of gp_decode_run (NULL = stream sampler, no window digests). */
typedef struct gp_run_opts {
  int32_t mode;          /* 0: stream sampler; 1: greedy over gp_synth_logit rows */
  int32_t rows;          /* greedy: rotating buffers, step s reads buffer s % rows */
  uint64_t logit_seed;   /* greedy: gp_synth_logit seed */
  int32_t warmup;        /* steps before the digest window */
  int32_t digest_seqs;   /* sequences [0, n) enter stats[5] and stats[6] */
  uint64_t* mask_hash;   /* [batch][steps] gp_mask_hash of every mask, or NULL */
} gp_run_opts;

/* Decode loop over `batch` sequences, `steps` steps, restart on finish (same
 * contract as ref_decode_run in oracle/ref_shim.cpp, single thread).
 * stats: [0] seconds, [1] seq-steps, [2] restarts, [3] token digest>>11,
 * [4] mask popcount sum, [5] token digest>>11 of sequences < digest_seqs over
 * steps >= warmup, [6] their mask popcounts (EOS excluded). */
int gp_decode_run(const gp_automaton* a, const gp_trie* t, const uint8_t* bytes,
                  const int64_t* offs, const uint32_t* structural, int32_t batch, int32_t steps,
                  uint64_t seed, int32_t stack_cap, double* stats, int32_t* tokens_out,
                  int32_t* final_stacks, const gp_run_opts* opts);

/* Workload restatements (see gmask_port.c). */
int64_t gp_synth_vocab(int32_t n, int32_t flavor, uint8_t* bytes, int64_t cap, int64_t* offs);
int32_t gp_structural_words(const uint8_t* bytes, const int64_t* offs, int32_t n, uint32_t* words);
uint16_t gp_synth_logit(uint64_t seed, int32_t k, int32_t b, int32_t t);
void gp_synth_logit_row(uint64_t seed, int32_t k, int32_t b, int32_t n, uint16_t* row);
uint64_t gp_mask_hash(const uint32_t* words, int32_t nw);

#ifdef __cplusplus
}
#endif
#endif
