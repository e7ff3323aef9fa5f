// HBM read / write / copy / 1-read-8-write probe on one B200 (sm_100a).
// Grid = 4 x 148 CTAs x 512 threads, 16-byte vector accesses, grid-stride,
// CUDA-event timed after warm-up, buffers of 4 GiB (>> 126 MB L2).
// Prints one JSON line of GB/s per access mix: the ceiling a collective
// with that read:write ratio can reach.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o hbm_rw hbm_rw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k_write(uint4* __restrict__ d, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) d[i] = v;
}
__global__ void k_read(const uint4* __restrict__ s, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcs(s + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_copy(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    d[i] = __ldcs(s + i);
}
// one read, eight writes (the one-shot allgather / broadcast mix)
__global__ void k_fan8(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const uint4 v = __ldcs(s + i);
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k * n + i] = v;
  }
}

int main() {
  const size_t bytes = size_t(4) << 30, n = bytes / 16;
  uint4 *a, *b;
  uint32_t* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 1, bytes);
  const int grid = 4 * 148, block = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](auto launch, int iters) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / iters * 1e-3;
  };
  const double tw = time([&] { k_write<<<grid, block>>>(b, n); }, 10);
  const double tr = time([&] { k_read<<<grid, block>>>(a, n, sink); }, 10);
  const double tc = time([&] { k_copy<<<grid, block>>>(a, b, n / 2); }, 10);          // 2 GiB -> 2 GiB
  const double tf = time([&] { k_fan8<<<grid, block>>>(a, b, n / 16); }, 10);         // 256 MiB -> 8 x 256 MiB
  printf("{\"write_GBps\": %.1f, \"read_GBps\": %.1f, \"copy_1r1w_GBps\": %.1f, \"fan_1r8w_GBps\": %.1f, "
         "\"err\": \"%s\"}\n",
         bytes / tw / 1e9, bytes / tr / 1e9, bytes / tc / 1e9, 9.0 * (bytes / 16) / tf / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
