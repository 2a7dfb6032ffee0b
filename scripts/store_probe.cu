// Store-path probe (diagnostics, not product): how fast can one B200 write a
// buffer of S bytes as -inf bf16, by path and grid shape?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe scripts/store_probe.cu
//   ./store_probe            (sizes 64 MB: L2-resident, and 256 MB / 1 GB: DRAM)
// Paths: STG.128 per lane (st.global.cs), TMA bulk stores of CHUNK bytes
// from shared memory (cp.async.bulk.global.shared::cta), each warp streaming
// ITEM bytes (like the fill's (sequence, segment) items: 16 KB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void StgKernel(uint4* out, long long n16, int item16) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item16;
  if (base >= n16) return;
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  for (int i = lane; i < item16; i += 32) __stcs(out + base + i, v);
}

template <int CHUNK>
__global__ void BulkKernel(char* out, long long bytes, int item) {
  __shared__ __align__(128) uint4 src[CHUNK / 16];
  for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) src[i] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item;
  if (base >= bytes || lane != 0) return;
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(src));
  for (int off = 0; off < item; off += CHUNK) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(out + base + off), "r"(sa), "r"(CHUNK)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// Items with dependent reads first (like the fill's head: slot -> CI ->
// mixed chunks): NRT round trips of one 16-B load per lane (each address
// depends on the previous value), then the item's stores.  Mixed: 1/MIX of
// the chunks are read back (cp.async-like) and written after the round trip.
template <int NRT, int MIX>
__global__ void ItemKernel(uint4* out, const uint4* in, long long n16, int item16) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item16;
  if (base >= n16) return;
  unsigned dep = 0;
#pragma unroll
  for (int r = 0; r < NRT; ++r) dep += __ldcg(reinterpret_cast<const unsigned*>(in) + ((base + lane + dep * 7) & 0xffff));
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u ^ (dep & 1));
  if (MIX > 0) {
    uint4 rd[4];
    for (int j = 0; j < 4; ++j) {
      const int i = (j * 32 + lane) * MIX;
      if (i < item16) rd[j] = __ldcs(out + base + i);
    }
    for (int i = lane; i < item16; i += 32) {
      uint4 w = v;
      if (i % MIX == 0 && (i / MIX) / 32 < 4) { const uint4 x = rd[(i / MIX) / 32]; w.x &= x.x | 1u; }
      __stcs(out + base + i, w);
    }
  } else {
    for (int i = lane; i < item16; i += 32) __stcs(out + base + i, v);
  }
}

// Clustered mixed chunks (like the fill's): in every 128-chunk span, chunks
// 0..13 (11%) hold allowed tokens and must be read before being written.
// One kernel (read, then write the item) vs two (gather the mixed chunks of
// every item into a side buffer first; then a pure store pass that blends
// them from the side buffer).
__device__ __forceinline__ bool MixedChunk(int i) { return (i & 127) < 14; }
__global__ void MixedOneKernel(uint4* out, long long n16, int item16) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item16;
  if (base >= n16) return;
  uint4 rd[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = r * 128 + lane;
    if (lane < 14 && i < item16) rd[r] = __ldcs(out + base + i);
  }
  for (int i = lane; i < item16; i += 32) {
    uint4 w = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    if (MixedChunk(i)) {
      const uint4 x = rd[(i >> 7) & 7];
      w.x = x.x | 0x10000u;
    }
    __stcs(out + base + i, w);
  }
}
__global__ void GatherKernel(const uint4* out, uint4* side, long long n16, int item16) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item16;
  if (base >= n16 || lane >= 14) return;
  uint4 rd[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) rd[r] = __ldcs(out + base + r * 128 + lane);
#pragma unroll
  for (int r = 0; r < 8; ++r) side[warp * 112 + r * 14 + lane] = rd[r];
}
__global__ void BlendKernel(uint4* out, const uint4* side, long long n16, int item16) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long base = warp * item16;
  if (base >= n16) return;
  for (int i = lane; i < item16; i += 32) {
    uint4 w = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    if (MixedChunk(i)) {
      const uint4 x = __ldcg(side + warp * 112 + ((i >> 7) & 7) * 14 + (i & 127));
      w.x = x.x | 0x10000u;
    }
    __stcs(out + base + i, w);
  }
}
uint4* g_side = nullptr;

// Persistent STG: one CTA per SM slot, grid-stride over the buffer.
__global__ void StgPersistent(uint4* out, long long n16) {
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    __stcs(out + i, v);
}

struct Arg;
extern Arg g;
static void Rotate(int r);
static float TimeIt(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch(arg);
  cudaDeviceSynchronize();
  float best = 1e30f, sum = 0;
  for (int r = 0; r < reps; ++r) {
    Rotate(r);  // a buffer region not written by the previous repetition (cold, like the rotating logits)
    cudaEventRecord(a);
    launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
    sum += ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return sum / reps;
}

struct Arg {
  char* base;
  char* buf;
  long long bytes;
  int item, threads, sms;
};
Arg g;
static void Rotate(int r) {
  const long long slots = (2048ll << 20) / g.bytes;
  g.buf = g.base + (r % slots) * g.bytes;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  g.sms = p.multiProcessorCount;
  const long long sizes[] = {64ll << 20, 256ll << 20, 1024ll << 20};
  char* buf;
  cudaMalloc(&buf, 2048ll << 20);
  cudaMalloc(&g_side, (1024ll << 20) / 16384 * 112 * 16);
  // A second buffer written between repetitions pushes the first out of L2.
  for (long long S : sizes) {
    g.base = buf;
    g.buf = buf;
    g.bytes = S;
    for (int item : {4096, 16384, 65536}) {
      g.item = item;
      g.threads = 256;
      auto stg = [](void*) {
        const long long warps = (g.bytes + g.item - 1) / g.item;
        const long long blocks = (warps * 32 + g.threads - 1) / g.threads;
        StgKernel<<<static_cast<unsigned>(blocks), g.threads>>>(reinterpret_cast<uint4*>(g.buf), g.bytes / 16, g.item / 16);
      };
      auto bulk2k = [](void*) {
        const long long warps = (g.bytes + g.item - 1) / g.item;
        const long long blocks = (warps * 32 + g.threads - 1) / g.threads;
        BulkKernel<2048><<<static_cast<unsigned>(blocks), g.threads>>>(g.buf, g.bytes, g.item);
      };
      auto bulk8k = [](void*) {
        const long long warps = (g.bytes + g.item - 1) / g.item;
        const long long blocks = (warps * 32 + g.threads - 1) / g.threads;
        BulkKernel<8192><<<static_cast<unsigned>(blocks), g.threads>>>(g.buf, g.bytes, g.item);
      };
      const float t1 = TimeIt(stg, nullptr, 20);
      const float t2 = TimeIt(bulk2k, nullptr, 20);
      const float t3 = item >= 8192 ? TimeIt(bulk8k, nullptr, 20) : 0.f;
      printf("S=%5lld MB item=%6d B  stg %8.2f us %6.2f TB/s | bulk2K %8.2f us %6.2f TB/s | bulk8K %8.2f us %6.2f TB/s\n",
             S >> 20, item, t1 * 1e3, S / (t1 * 1e-3) / 1e12, t2 * 1e3, S / (t2 * 1e-3) / 1e12, t3 * 1e3,
             t3 > 0 ? S / (t3 * 1e-3) / 1e12 : 0.0);
    }
    {
      g.item = 16384;
      for (int smem : {0, 48 * 1024}) {
        g.threads = smem;  // (reused as the dynamic smem size: 48 KB -> 4 CTAs/SM)
        auto it0 = [](void*) { const long long w = g.bytes / g.item; ItemKernel<0, 0><<<static_cast<unsigned>((w * 32 + 255) / 256), 256, g.threads>>>(reinterpret_cast<uint4*>(g.buf), reinterpret_cast<const uint4*>(g.base), g.bytes / 16, g.item / 16); };
        auto it2 = [](void*) { const long long w = g.bytes / g.item; ItemKernel<2, 0><<<static_cast<unsigned>((w * 32 + 255) / 256), 256, g.threads>>>(reinterpret_cast<uint4*>(g.buf), reinterpret_cast<const uint4*>(g.base), g.bytes / 16, g.item / 16); };
        auto it2m = [](void*) { const long long w = g.bytes / g.item; ItemKernel<2, 8><<<static_cast<unsigned>((w * 32 + 255) / 256), 256, g.threads>>>(reinterpret_cast<uint4*>(g.buf), reinterpret_cast<const uint4*>(g.base), g.bytes / 16, g.item / 16); };
        if (smem) {
          cudaFuncSetAttribute(ItemKernel<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          cudaFuncSetAttribute(ItemKernel<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          cudaFuncSetAttribute(ItemKernel<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        }
        const float a0 = TimeIt(it0, nullptr, 20), a2 = TimeIt(it2, nullptr, 20), a2m = TimeIt(it2m, nullptr, 20);
        printf("S=%5lld MB 16K items %s: stores only %7.2f us | 2 RTs + stores %7.2f us | 2 RTs + 1/8 chunks read-then-written %7.2f us\n",
               S >> 20, smem ? "4 CTAs/SM" : "8 CTAs/SM", a0 * 1e3, a2 * 1e3, a2m * 1e3);
      }
      g.threads = 256;
    }
    {
      g.item = 16384;
      auto one = [](void*) { const long long w = g.bytes / g.item; MixedOneKernel<<<static_cast<unsigned>((w * 32 + 255) / 256), 256>>>(reinterpret_cast<uint4*>(g.buf), g.bytes / 16, g.item / 16); };
      auto two = [](void*) {
        const long long w = g.bytes / g.item;
        GatherKernel<<<static_cast<unsigned>((w * 32 + 255) / 256), 256>>>(reinterpret_cast<const uint4*>(g.buf), g_side, g.bytes / 16, g.item / 16);
        BlendKernel<<<static_cast<unsigned>((w * 32 + 255) / 256), 256>>>(reinterpret_cast<uint4*>(g.buf), g_side, g.bytes / 16, g.item / 16);
      };
      const float t1 = TimeIt(one, nullptr, 20), t2 = TimeIt(two, nullptr, 20);
      printf("S=%5lld MB 16K items, 11%% clustered mixed chunks: one kernel (read, write) %7.2f us | gather kernel + blend kernel %7.2f us\n",
             S >> 20, t1 * 1e3, t2 * 1e3);
      g.threads = 256;
    }
    auto pers = [](void*) { StgPersistent<<<g.sms * 8, 256>>>(reinterpret_cast<uint4*>(g.buf), g.bytes / 16); };
    const float t4 = TimeIt(pers, nullptr, 20);
    printf("S=%5lld MB persistent stg (8 CTAs/SM) %8.2f us %6.2f TB/s\n", S >> 20, t4 * 1e3, S / (t4 * 1e-3) / 1e12);
  }
  cudaFree(buf);
  return 0;
}
