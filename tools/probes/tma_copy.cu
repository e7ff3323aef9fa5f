// TMA bulk-copy ceiling on one B200 (sm_100a): how fast can a
// cp.async.bulk global -> smem -> global pipeline, shaped like the
// executor's (one producer lane, stages owned round-robin by storer warps,
// a stage released at wait_group.read), copy 4 GiB of random bytes, against
// a 16-byte LD/ST grid-stride copy of the same buffers?
//   variant "landed": each storer waits for its writes to land (wait_group 0)
//                     before taking its next stage (the executor's release
//                     rule: a counter may only be published for landed bytes)
//   variant "stream": storers only wait for the smem read-out
// One JSON line per (tile, stages, CTAs per SM, variant).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tma_copy tma_copy.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(
          s32(b)),
      "r"(par)
      : "memory");
}

template <int NSW, bool LANDED, bool INTERLEAVE = false>
__global__ void __launch_bounds__(32 * (1 + NSW)) k_tma(const char* __restrict__ src, char* __restrict__ dst,
                                                       size_t per_cta, int T, int NST) {
  // INTERLEAVE: tile t of CTA b is global tile t * gridDim.x + b (all CTAs
  // sweep one contiguous front) instead of CTA b's own contiguous slice
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 32;
  char* stage = smem + 1024;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) mb_init(&full[s], 1), mb_init(&empty[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = INTERLEAVE ? size_t(blockIdx.x) * T : size_t(blockIdx.x) * per_cta;
  const size_t step = INTERLEAVE ? size_t(gridDim.x) * T : size_t(T);
  const uint32_t ntiles = uint32_t((per_cta + T - 1) / T);
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t t = 0; t < ntiles; ++t) {
        const int s = t % NST;
        if (t >= uint32_t(NST)) mb_wait(&empty[s], ((t / NST) - 1) & 1);
        const uint32_t n = uint32_t(per_cta - size_t(t) * T < size_t(T) ? per_cta - size_t(t) * T : size_t(T));
        mb_arrive_tx(&full[s], n);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                s32(stage + size_t(s) * T)),
            "l"(src + base + size_t(t) * step), "r"(n), "r"(s32(&full[s]))
            : "memory");
      }
    }
  } else if (lane == 0) {
    const int me = warp - 1;
    for (uint32_t t = 0; t < ntiles; ++t) {
      const int s = t % NST;
      if (s % NSW != me) continue;
      mb_wait(&full[s], (t / NST) & 1);
      const uint32_t n = uint32_t(per_cta - size_t(t) * T < size_t(T) ? per_cta - size_t(t) * T : size_t(T));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + base + size_t(t) * step),
                   "r"(s32(stage + size_t(s) * T)), "r"(n)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mb_arrive(&empty[s]);
      if (LANDED) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

__global__ void k_ldst(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    d[i] = __ldcs(s + i);
}
__global__ void k_fill(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull + 0x1234567ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = z ^ (z >> 31);
  }
}

int main() {
  const size_t bytes = size_t(4) << 30;
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  k_fill<<<1184, 512>>>(reinterpret_cast<uint64_t*>(a), bytes / 8);
  k_fill<<<1184, 512>>>(reinterpret_cast<uint64_t*>(b), bytes / 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10 * 1e-3;
  };
  const double t = time([&] { k_ldst<<<4 * 148, 512>>>((const uint4*)a, (uint4*)b, bytes / 16); });
  printf("{\"variant\": \"ldst\", \"GBps\": %.1f, \"err\": \"%s\"}\n", 2 * bytes / t / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  const double tm = time([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); });
  printf("{\"variant\": \"cudaMemcpyAsync D2D\", \"GBps\": %.1f, \"err\": \"%s\"}\n", 2 * bytes / tm / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  for (int cps = 1; cps <= 2; ++cps) {
    const int grid = 148 * cps, T = 32768, NST = cps == 1 ? 6 : 3;
    const size_t per = (bytes / grid) / T * T;  // whole tiles (interleaved layout)
    const size_t sm = 1024 + size_t(T) * NST;
    auto kern = k_tma<3, true, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    const double tt = time([&] { kern<<<grid, 128, sm>>>(a, b, per, T, NST); });
    printf("{\"variant\": \"tma_landed_interleaved\", \"tile\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           T, NST, cps, 2.0 * per * grid / tt / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  struct Cfg {
    int T, NST, cps;
  } cfgs[] = {{32768, 3, 2}, {32768, 6, 1}, {16384, 6, 2}, {65536, 3, 1}, {16384, 12, 1}, {8192, 12, 2}};
  for (auto c : cfgs) {
    for (int landed = 0; landed < 2; ++landed) {
      const int grid = 148 * c.cps;
      const size_t per = (bytes / grid) / 16 * 16;
      const size_t sm = 1024 + size_t(c.T) * c.NST;
      auto kern = landed ? k_tma<3, true> : k_tma<3, false>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
      const double tt = time([&] { kern<<<grid, 128, sm>>>(a, b, per, c.T, c.NST); });
      printf("{\"variant\": \"tma_%s\", \"tile\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
             landed ? "landed" : "stream", c.T, c.NST, c.cps, 2.0 * per * grid / tt / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
