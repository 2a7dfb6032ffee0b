// workload_dev.cu — device-side synthetic inputs for bench.py and the tests
// (include/pre3_workload.h; not on the hot path, not part of the drop-in ABI).
//
// gmw_synth_logits fills rotating bf16 logit buffers with the counter-based
// generator restated in oracle/gmask_port.c (gp_synth_logit) and
// oracle/ref_shim.cpp (SynthLogit), so the GPU arm and the CPU reference arm
// of config 5's greedy decode loop see identical logits.
#include <cuda_runtime.h>

#include <cstdint>

#include "pre3_workload.h"

namespace {

__device__ __forceinline__ unsigned long long Mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Row b of buffer k: 8 logits (16 B) per thread, grid-stride over the row.
__global__ void SynthLogitsKernel(uint16_t* dst, long long ld, int32_t cols, int32_t k, int32_t row0,
                                  unsigned long long seed) {
  const int b = blockIdx.y;
  const unsigned long long h =
      Mix64(seed ^ 0x6C6F67697473ull ^ (static_cast<unsigned long long>(static_cast<uint32_t>(k)) * 0xA24BAED4963EE407ull) ^
            (static_cast<unsigned long long>(static_cast<uint32_t>(row0 + b)) * 0xD1B54A32D192ED03ull));
  uint16_t* row = dst + static_cast<long long>(b) * ld;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cols; t += gridDim.x * blockDim.x) {
    const unsigned long long x = Mix64(h ^ static_cast<unsigned long long>(static_cast<uint32_t>(t)));
    row[t] = static_cast<uint16_t>((0x3C00u + static_cast<uint32_t>(x & 0x3FFu)) ^ (((x >> 20) & 1u) ? 0x8000u : 0u));
  }
}

}  // namespace

extern "C" int32_t gmw_synth_logits(uint16_t* dst, int64_t ld, int32_t rows, int32_t cols, int32_t k, int32_t row0,
                                    uint64_t seed, void* stream) {
  if (dst == nullptr || rows < 0 || cols < 0 || ld < cols || rows > 65535) return -1;
  if (rows == 0 || cols == 0) return 0;
  const int blocks_x = (cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64;
  SynthLogitsKernel<<<dim3(blocks_x, rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, ld, cols, k, row0,
                                                                                          seed);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
