// sm_100a executor for lowered SCCL channel programs.
//
// Design ancestor: the paper's single fused kernel: all
// S steps of a schedule in one launch, chunks pushed straight into the
// destination rank's memory, a dedicated flag per (chunk, connection) set
// after a system-scope fence, receivers spinning on the flag before they
// forward or reduce.  Here:
//   * one CTA per (rank, channel); a channel is a contiguous 16 B-aligned
//     sub-range of every chunk, so a CTA runs its rank's whole op list on
//     its sub-range and program order covers all intra-rank dependencies;
//   * flags are per (receipt slot, channel) 64-bit counters that count tiles
//     across launches (value (epoch-1)*ntiles + t + 1 after tile t), so a
//     consumer can start forwarding tile t while later tiles are in flight
//     and nothing is ever reset;
//   * data moves as 16 B vectors, loads batched ahead of stores; the
//     reduction of combining receipts is fused into the receive and
//     into the forward of the result (one pass over the inputs, results
//     stored to every destination);
//   * loopback mode (every rank of the schedule on this GPU: one launch of
//     P*nch CTAs) uses gpu-scope release/acquire; multi-process mode (one
//     rank per GPU, peers' buffers mapped through CUDA IPC over NVLink)
//     uses system scope and an entry handshake per (peer, channel) so a
//     rank never writes into a peer that has not yet entered the launch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../sccl/devprog.hpp"

namespace sccl {
namespace {

constexpr int NT = 512;  // threads per CTA
constexpr int U = 4;     // 16 B vectors in flight per thread per input

struct DPart {
  int64_t off, len;
};
__device__ __forceinline__ DPart dsplit16(int64_t L, int64_t K, int64_t i) {
  int64_t Uu = L >> 4;
  int64_t lo = (i * Uu / K) << 4;
  int64_t hi = (i == K - 1) ? L : (((i + 1) * Uu / K) << 4);
  return {lo, hi - lo};
}

// ---------------------------------------------------------------- flags
template <bool SYS>
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void signal(uint64_t* p, uint64_t v) {
  // fence.acq_rel + relaxed store == release; the preceding bar.sync makes
  // the whole CTA's stores of the tile part of what is released.
  if (SYS) asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until *f >= target; returns the value seen.  Watchdog: after
// timeout_ns the diagnostic goes to host-mapped memory and the kernel traps
// (the host maps it to SCCL_PEER_TIMEOUT).
template <bool SYS>
__device__ uint64_t wait_ge(const uint64_t* f, uint64_t target, const KParams& p, int rank, int ch, int op,
                            int slot) {
  uint64_t v = ld_acquire<SYS>(f);
  if (v >= target) return v;
  uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while ((v = ld_acquire<SYS>(f)) < target) {
    if (++spins > 256) __nanosleep(40);
    if ((spins & 1023) == 0 && p.timeout_ns > 0 && (long long)(globaltimer() - t0) > p.timeout_ns) {
      volatile int* e = p.errinfo;
      if (e && atomicCAS(p.errinfo, 0, -1) == 0) {
        e[1] = rank;
        e[2] = ch;
        e[3] = op;
        e[4] = slot;
        e[5] = int(target & 0x7fffffff);
        e[6] = int(v & 0x7fffffff);
        __threadfence_system();
        e[0] = ERR_TIMEOUT;
        __threadfence_system();
      }
      __trap();
    }
  }
  return v;
}

// ---------------------------------------------------------------- data
__device__ __forceinline__ int4 ld_vec(const int4* p, bool nc) { return nc ? __ldg(p) : __ldcg(p); }
__device__ __forceinline__ void st_vec(int4* p, const int4& v) { __stcg(p, v); }

// accumulator of one 16 B vector, per element type
template <int DT>
struct Vec;
template <>
struct Vec<0> {  // u8, wrapping
  uint4 a;
  __device__ void init(int4 v) { a = make_uint4(v.x, v.y, v.z, v.w); }
  __device__ void add(int4 v) {
    a.x = __vadd4(a.x, v.x);
    a.y = __vadd4(a.y, v.y);
    a.z = __vadd4(a.z, v.z);
    a.w = __vadd4(a.w, v.w);
  }
  __device__ int4 out() const { return make_int4(a.x, a.y, a.z, a.w); }
};
template <>
struct Vec<1> {  // i32, two's-complement wrap
  uint4 a;
  __device__ void init(int4 v) { a = make_uint4(v.x, v.y, v.z, v.w); }
  __device__ void add(int4 v) {
    a.x += uint32_t(v.x);
    a.y += uint32_t(v.y);
    a.z += uint32_t(v.z);
    a.w += uint32_t(v.w);
  }
  __device__ int4 out() const { return make_int4(a.x, a.y, a.z, a.w); }
};
template <>
struct Vec<2> {  // f32, adds in input order
  float4 a;
  __device__ void init(int4 v) { a = make_float4(__int_as_float(v.x), __int_as_float(v.y), __int_as_float(v.z), __int_as_float(v.w)); }
  __device__ void add(int4 v) {
    a.x = __fadd_rn(a.x, __int_as_float(v.x));
    a.y = __fadd_rn(a.y, __int_as_float(v.y));
    a.z = __fadd_rn(a.z, __int_as_float(v.z));
    a.w = __fadd_rn(a.w, __int_as_float(v.w));
  }
  __device__ int4 out() const { return make_int4(__float_as_int(a.x), __float_as_int(a.y), __float_as_int(a.z), __float_as_int(a.w)); }
};
template <>
struct Vec<3> {  // bf16: widen, add in f32 in input order, round once
  float a[8];
  __device__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
  __device__ static float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
  __device__ void init(int4 v) {
    uint32_t w[4] = {uint32_t(v.x), uint32_t(v.y), uint32_t(v.z), uint32_t(v.w)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = lo(w[k]);
      a[2 * k + 1] = hi(w[k]);
    }
  }
  __device__ void add(int4 v) {
    uint32_t w[4] = {uint32_t(v.x), uint32_t(v.y), uint32_t(v.z), uint32_t(v.w)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = __fadd_rn(a[2 * k], lo(w[k]));
      a[2 * k + 1] = __fadd_rn(a[2 * k + 1], hi(w[k]));
    }
  }
  __device__ int4 out() const {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(a[2 * k]));
      uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(a[2 * k + 1]));
      w[k] = l | (h << 16);
    }
    return make_int4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Vec<4> {  // f16: widen, add in f32 in input order, round once
  float a[8];
  __device__ void init(int4 v) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __half22float2(h[k]);
      a[2 * k] = f.x;
      a[2 * k + 1] = f.y;
    }
  }
  __device__ void add(int4 v) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __half22float2(h[k]);
      a[2 * k] = __fadd_rn(a[2 * k], f.x);
      a[2 * k + 1] = __fadd_rn(a[2 * k + 1], f.y);
    }
  }
  __device__ int4 out() const {
    int4 r;
    __half2* h = reinterpret_cast<__half2*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __halves2half2(__float2half_rn(a[2 * k]), __float2half_rn(a[2 * k + 1]));
    return r;
  }
};

// element-wise path (unaligned ops and the < 16 B chunk tail)
template <int DT>
__device__ void elem_op(const char* const* in, const uint8_t* nc, int nin, char* const* out, int nout,
                        int64_t off, int64_t nbytes, int tid, int nthr) {
  constexpr int ES = (DT == 0) ? 1 : (DT == 3 || DT == 4) ? 2 : 4;
  for (int64_t i = tid; i < nbytes / ES; i += nthr) {
    const int64_t b = off + i * ES;
    if (DT == 0) {
      uint8_t a = *(const volatile uint8_t*)(in[0] + b);
      for (int k = 1; k < nin; ++k) a = uint8_t(a + *(const volatile uint8_t*)(in[k] + b));
      for (int o = 0; o < nout; ++o) *(volatile uint8_t*)(out[o] + b) = a;
    } else if (DT == 1) {
      uint32_t a = *(const volatile uint32_t*)(in[0] + b);
      for (int k = 1; k < nin; ++k) a += *(const volatile uint32_t*)(in[k] + b);
      for (int o = 0; o < nout; ++o) *(volatile uint32_t*)(out[o] + b) = a;
    } else if (DT == 2) {
      float a = __int_as_float(*(const volatile int*)(in[0] + b));
      for (int k = 1; k < nin; ++k) a = __fadd_rn(a, __int_as_float(*(const volatile int*)(in[k] + b)));
      for (int o = 0; o < nout; ++o) *(volatile int*)(out[o] + b) = __float_as_int(a);
    } else {
      auto widen = [](uint16_t h) -> float {
        if (DT == 3) return __uint_as_float(uint32_t(h) << 16);
        return __half2float(__ushort_as_half(h));
      };
      float a = widen(*(const volatile uint16_t*)(in[0] + b));
      for (int k = 1; k < nin; ++k) a = __fadd_rn(a, widen(*(const volatile uint16_t*)(in[k] + b)));
      uint16_t r = (DT == 3) ? __bfloat16_as_ushort(__float2bfloat16_rn(a)) : __half_as_ushort(__float2half_rn(a));
      for (int o = 0; o < nout; ++o) *(volatile uint16_t*)(out[o] + b) = r;
    }
  }
}

// one tile of a copy op: one input, nout destinations
__device__ __forceinline__ void copy_tile(const char* in, bool nc, char* const* out, int nout, int64_t off,
                                          int64_t nbytes) {
  const int4* src = reinterpret_cast<const int4*>(in + off);
  const int64_t nv = nbytes >> 4;
  for (int64_t i = threadIdx.x; i < nv; i += NT * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * NT < nv) v[u] = ld_vec(src + i + u * NT, nc);
    for (int o = 0; o < nout; ++o) {
      int4* dst = reinterpret_cast<int4*>(out[o] + off);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * NT < nv) st_vec(dst + i + u * NT, v[u]);
    }
  }
}

template <int DT>
__device__ __forceinline__ void reduce_tile(const char* const* in, const uint8_t* nc, int nin, char* const* out,
                                            int nout, int64_t off, int64_t nbytes) {
  const int64_t nv = nbytes >> 4;
  for (int64_t i = threadIdx.x; i < nv; i += NT * U) {
    Vec<DT> acc[U];
    {
      const int4* s = reinterpret_cast<const int4*>(in[0] + off);
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * NT < nv) v[u] = ld_vec(s + i + u * NT, nc[0]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u].init(v[u]);
    }
    for (int k = 1; k < nin; ++k) {
      const int4* s = reinterpret_cast<const int4*>(in[k] + off);
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * NT < nv) v[u] = ld_vec(s + i + u * NT, nc[k]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u].add(v[u]);
    }
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = acc[u].out();
    for (int o = 0; o < nout; ++o) {
      int4* dst = reinterpret_cast<int4*>(out[o] + off);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * NT < nv) st_vec(dst + i + u * NT, r[u]);
    }
  }
}

template <int DT, bool SYS>
__global__ void __launch_bounds__(NT, 1) exec_kernel(const __grid_constant__ KParams p) {
  const int tid = threadIdx.x;
  const int lr = blockIdx.x / p.nch, ch = blockIdx.x % p.nch;
  const int rank = p.rank0 + lr;

  __shared__ uint64_t s_e;
  __shared__ const char* s_inp[kMaxOpIn];
  __shared__ char* s_outp[kMaxOpOut];
  __shared__ uint64_t* s_inflag[kMaxOpIn];
  __shared__ uint64_t* s_sigflag[kMaxOpOut];
  __shared__ uint8_t s_nc[kMaxOpIn];
  __shared__ uint8_t s_every[kMaxOpOut];
  __shared__ uint8_t s_outrank[kMaxOpOut];
  __shared__ uint32_t s_ready[kMaxOpIn];
  __shared__ int32_t s_inslot[kMaxOpIn];
  __shared__ uint32_t s_entry_mask;
  __shared__ int s_any_every;

  if (tid == 0) {
    s_e = p.epochs[blockIdx.x] + 1;
    s_entry_mask = 1u << rank;
  }
  __syncthreads();
  const uint64_t e = s_e;
  uint64_t* const myflags = reinterpret_cast<uint64_t*>(p.base[rank][SP_FLAGS_IDX]);

  if (p.multiprocess)  // "rank `rank`, channel ch entered launch e"
    for (int t = tid; t < p.P; t += NT)
      if (t != rank)
        signal<SYS>(reinterpret_cast<uint64_t*>(p.base[t][SP_FLAGS_IDX]) + p.entry_base + rank * p.nch + ch, e);

  const uint32_t ob = p.prog[rank], oe = p.prog[rank + 1];
  for (uint32_t oi = ob; oi < oe; ++oi) {
    const DevOp op = p.ops[oi];
    if (op.kind == 2) {  // end-of-program waits: every receipt has landed
      for (int i = tid; i < op.nin; i += NT) {
        const DevIn in = p.ins[op.in_begin + i];
        const DPart q = dsplit16(int64_t(in.len), p.nch, ch);
        const uint64_t nt = (q.len + p.tile - 1) / p.tile;
        if (nt) wait_ge<SYS>(myflags + uint64_t(in.flag) * p.nch + ch, e * nt, p, rank, ch, int(oi - ob), in.flag);
      }
      __syncthreads();
      continue;
    }
    const DPart q = dsplit16(int64_t(op.len), p.nch, ch);
    const uint32_t ntiles = uint32_t((q.len + p.tile - 1) / p.tile);
    if (ntiles == 0) continue;  // empty sub-range: nothing sent, nothing awaited
    if (tid < op.nin) {
      const DevIn in = p.ins[op.in_begin + tid];
      s_inp[tid] = p.base[in.rank][in.space] + in.off;
      s_nc[tid] = (in.space == 0 && p.send_readonly) ? 1 : 0;
      s_inslot[tid] = in.flag;
      s_inflag[tid] = in.flag >= 0 ? myflags + uint64_t(in.flag) * p.nch + ch : nullptr;
      s_ready[tid] = 0;
    }
    if (tid == 0) s_any_every = 0;
    __syncthreads();
    if (tid < op.nout) {
      const DevOut o = p.outs[op.out_begin + tid];
      s_outp[tid] = p.base[o.rank][o.space] + o.off;
      s_every[tid] = o.every_tile;
      s_outrank[tid] = o.rank;
      s_sigflag[tid] = o.flag >= 0 ? reinterpret_cast<uint64_t*>(p.base[o.rank][SP_FLAGS_IDX]) + uint64_t(o.flag) * p.nch + ch
                                   : nullptr;
      if (o.flag >= 0 && o.every_tile) s_any_every = 1;
      if (p.multiprocess && o.rank != rank && !(s_entry_mask & (1u << o.rank))) {
        wait_ge<SYS>(myflags + p.entry_base + o.rank * p.nch + ch, e, p, rank, ch, int(oi - ob), -2);
        atomicOr(&s_entry_mask, 1u << o.rank);
      }
    }
    __syncthreads();
    const bool any_every = s_any_every != 0;
    const uint64_t base = (e - 1) * uint64_t(ntiles);

    for (uint32_t t = 0; t < ntiles; ++t) {
      if (tid < op.nin && s_inflag[tid] && s_ready[tid] <= t) {
        uint64_t v = wait_ge<SYS>(s_inflag[tid], base + t + 1, p, rank, ch, int(oi - ob), s_inslot[tid]);
        uint64_t r = v - base;
        s_ready[tid] = uint32_t(r > ntiles ? ntiles : r);
      }
      __syncthreads();
      const int64_t off = q.off + int64_t(t) * p.tile;
      const int64_t nb = min(int64_t(p.tile), q.len - int64_t(t) * p.tile);
      const int64_t nvb = op.vec ? (nb & ~int64_t(15)) : 0;
      if (nvb) {
        if (op.kind == 0) copy_tile(s_inp[0], s_nc[0], s_outp, op.nout, off, nvb);
        else reduce_tile<DT>(s_inp, s_nc, op.nin, s_outp, op.nout, off, nvb);
      }
      if (nb > nvb) {
        if (op.kind == 0) elem_op<0>(s_inp, s_nc, 1, s_outp, op.nout, off + nvb, nb - nvb, tid, NT);
        else elem_op<DT>(s_inp, s_nc, op.nin, s_outp, op.nout, off + nvb, nb - nvb, tid, NT);
      }
      const bool last = t + 1 == ntiles;
      if (last || any_every) {
        __syncthreads();
        if (tid < op.nout && s_sigflag[tid] && (last || s_every[tid])) signal<SYS>(s_sigflag[tid], base + t + 1);
      }
    }
    __syncthreads();
  }
  if (tid == 0) p.epochs[blockIdx.x] = e;
}

template <int DT>
cudaError_t launch_dt(const KParams& p, bool sys, cudaStream_t st) {
  dim3 grid(p.nranks_launch * p.nch), block(NT);
  if (sys) exec_kernel<DT, true><<<grid, block, 0, st>>>(p);
  else exec_kernel<DT, false><<<grid, block, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace

int exec_threads() { return NT; }

cudaError_t launch_exec(const KParams& p, int dtype, bool sys, cudaStream_t st) {
  switch (dtype) {
    case 0: return launch_dt<0>(p, sys, st);
    case 1: return launch_dt<1>(p, sys, st);
    case 2: return launch_dt<2>(p, sys, st);
    case 3: return launch_dt<3>(p, sys, st);
    case 4: return launch_dt<4>(p, sys, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t exec_occupancy(int dtype, bool sys, int* blocks_per_sm) {
  const void* f = nullptr;
#define SCCL_F(D)                                                                                   \
  case D:                                                                                           \
    f = sys ? reinterpret_cast<const void*>(exec_kernel<D, true>) : reinterpret_cast<const void*>(exec_kernel<D, false>); \
    break;
  switch (dtype) {
    SCCL_F(0)
    SCCL_F(1)
    SCCL_F(2)
    SCCL_F(3)
    SCCL_F(4)
    default: return cudaErrorInvalidValue;
  }
#undef SCCL_F
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, NT, 0);
}

}  // namespace sccl
