/* include/pre3_workload.h — synthetic workload helpers (tests and bench.py;
 * not part of the reference-facing ABI). */
#ifndef PRE3_WORKLOAD_H_
#define PRE3_WORKLOAD_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Sorted synthetic vocabulary (acceptance_main.cpp:341-359 extended to
 * num_tokens; flavor 0 = JSON fragments, 1 = + SQL fragments).  Call with
 * bytes == NULL to get the byte count; offsets has num_tokens + 1 entries.
 * Returns the byte count or < 0 on error. */
int64_t gmw_synth_vocab(int32_t num_tokens, int32_t flavor, uint8_t* bytes, int64_t bytes_cap,
                        int64_t* offsets);
/* Mask words (W = ceil((V+1)/32)) of tokens containing any of {}[],:" ;
 * returns how many. */
int32_t gmw_structural_words(const uint8_t* bytes, const int64_t* offsets, int32_t num_tokens,
                             uint32_t* words);
/* Synthetic bf16 logits on the device: row r (< rows) of dst[r * ld + t],
 * t < cols, gets gp_synth_logit(seed, k, row0 + r, t) (oracle/gmask_port.c;
 * config 5's greedy decode loop, identical in the CPU reference arm).
 * Asynchronous on `stream`; returns 0 or -1. */
int32_t gmw_synth_logits(uint16_t* dst, int64_t ld, int32_t rows, int32_t cols, int32_t k, int32_t row0,
                         uint64_t seed, void* stream);
#ifdef __cplusplus
}
#endif
#endif
