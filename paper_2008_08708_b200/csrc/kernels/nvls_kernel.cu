// NVLS (NVLink SHARP) allreduce: the comparison backend of SURVEY.md 8(f)
// f4 ("NVLS multimem Allreduce").  Not schedule-driven: every rank's buffer
// is bound to one multicast object, and rank r reduces slice r of it in the
// NVSwitch -- multimem.ld_reduce reads the slice from every GPU and returns
// the sum, multimem.st writes the result to every GPU -- so each rank moves
// M/P bytes in and M/P * P out through the switch instead of 2(P-1)/P * M
// per direction over NVLink.  A per-CTA arrival counter, incremented on
// every GPU at once with multimem.red.release, brackets the data phase (the
// inputs are in place before any read; every read is done before any rank
// returns and may overwrite its buffer).
//
// Reduction order: the switch's (f32 accumulation for bf16 / f16), not the
// schedule's -- results are exact for integer-valued data and within the
// stated float tolerance otherwise.
#include <cuda_runtime.h>
#include <stdint.h>

namespace sccl {
namespace {

constexpr int NVLS_NT = 512;

__device__ __forceinline__ void mc_arrive(uint32_t* mc_counter) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_counter), "r"(1u) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spin until the local copy of the counter reaches target (wrap-safe)
__device__ __forceinline__ bool wait_count(const uint32_t* p, uint32_t target, long long timeout_ns, int* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t spins = 0;; ++spins) {
    if (int32_t(ld_acquire_sys_u32(p) - target) >= 0) return true;
    if (spins > 64) __nanosleep(64);
    if ((spins & 1023) == 0 && timeout_ns > 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > timeout_ns) {
        if (err) atomicExch(err, 5);
        return false;
      }
    }
  }
}

template <int DT>
__device__ __forceinline__ uint4 mc_ld_reduce(const void* mc) {
  uint4 v;
  if constexpr (DT == 2)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  else if constexpr (DT == 3)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(void* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

struct NvlsParams {
  char* mc;          // multicast mapping of the bound region
  char* uc;          // this GPU's own mapping of the same region
  uint64_t lo, hi;   // this rank's slice of the data, bytes (16-aligned)
  uint64_t flags;    // offset of the counters: [entry x grid][exit x grid] u32
  uint32_t* epochs;  // per-CTA launch counters (device memory)
  int P;
  int* err;          // host-mapped: 5 on a barrier timeout
  long long timeout_ns;
};

template <int DT>
__global__ void __launch_bounds__(NVLS_NT) nvls_allreduce_kernel(const __grid_constant__ NvlsParams p) {
  const int b = blockIdx.x, G = gridDim.x;
  __shared__ uint32_t s_e;
  __shared__ int s_ok;
  uint32_t* entry_mc = reinterpret_cast<uint32_t*>(p.mc + p.flags) + b;
  uint32_t* entry_uc = reinterpret_cast<uint32_t*>(p.uc + p.flags) + b;
  uint32_t* exit_mc = entry_mc + G;
  uint32_t* exit_uc = entry_uc + G;
  if (threadIdx.x == 0) {
    const uint32_t e = p.epochs[b] + 1;
    s_e = e;
    mc_arrive(entry_mc);  // "my input is in place" on every GPU
    s_ok = wait_count(entry_uc, uint32_t(p.P) * e, p.timeout_ns, p.err);
  }
  __syncthreads();
  if (s_ok) {
    const uint64_t v0 = p.lo / 16, v1 = p.hi / 16;
    for (uint64_t v = v0 + uint64_t(b) * NVLS_NT + threadIdx.x; v < v1; v += uint64_t(G) * NVLS_NT) {
      const uint4 x = mc_ld_reduce<DT>(p.mc + v * 16);
      mc_st(p.mc + v * 16, x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    mc_arrive(exit_mc);  // "my reads and stores are done"
    if (s_ok) wait_count(exit_uc, uint32_t(p.P) * s_e, p.timeout_ns, p.err);
    p.epochs[b] = s_e;
  }
}

}  // namespace

int nvls_threads() { return NVLS_NT; }

cudaError_t launch_nvls(char* mc, char* uc, uint64_t lo, uint64_t hi, uint64_t flags, uint32_t* epochs, int P,
                        int grid, int dtype, int* err, long long timeout_ns, cudaStream_t st) {
  NvlsParams p{mc, uc, lo, hi, flags, epochs, P, err, timeout_ns};
  void* args[] = {&p};
  const void* f = dtype == 2 ? reinterpret_cast<const void*>(nvls_allreduce_kernel<2>)
                  : dtype == 3 ? reinterpret_cast<const void*>(nvls_allreduce_kernel<3>)
                  : dtype == 4 ? reinterpret_cast<const void*>(nvls_allreduce_kernel<4>)
                               : nullptr;
  if (!f) return cudaErrorInvalidValue;
  return cudaLaunchKernel(f, dim3(grid), dim3(NVLS_NT), args, 0, st);
}

}  // namespace sccl
