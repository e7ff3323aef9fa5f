// Launch floor on one B200: per-kernel time of N back-to-back launches of an
// empty kernel captured in one CUDA graph (the way bench/tune time the
// executor), for 1 CTA and for 1184 CTAs.  The executor's small-message
// latency is this floor plus its own work.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o launch_floor launch_floor.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 1024) *p = 0;
}
template <int N>
struct Big {
  int* p;
  unsigned char pad[N];
};
// reads one word of a large __grid_constant__ parameter block
template <int N>
__global__ void big_kernel(const __grid_constant__ Big<N> b) {
  if (b.p && b.pad[threadIdx.x % N] == 7) *b.p = 0;
}
template <int N>
static double big_us(int grid, int n) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  Big<N> arg{};
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) big_kernel<N><<<grid, 256, 0, st>>>(arg);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3 / n;
}

static double per_launch_us(int grid, int block, int n) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < n; ++i) empty_kernel<<<grid, block, 0, st>>>(nullptr);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3 / n;
}

int main() {
  printf("{\"empty_1cta_us\": %.2f, \"empty_1184cta_256thr_us\": %.2f, \"empty_296cta_352thr_us\": %.2f, "
         "\"param_1KB_64cta_us\": %.2f, \"param_8KB_64cta_us\": %.2f, \"param_16KB_64cta_us\": %.2f, "
         "\"param_30KB_64cta_us\": %.2f, \"err\": \"%s\"}\n",
         per_launch_us(1, 32, 200), per_launch_us(1184, 256, 200), per_launch_us(296, 352, 200), big_us<1024>(64, 200),
         big_us<8192>(64, 200), big_us<16384>(64, 200), big_us<30000>(64, 200), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
