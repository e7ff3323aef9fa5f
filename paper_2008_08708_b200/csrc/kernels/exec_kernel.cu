// sm_100a executor for lowered SCCL channel programs.
//
// Design ancestor: the paper's single fused kernel: all
// S steps of a schedule in one launch, chunks pushed straight into the
// destination rank's memory, a dedicated flag per (chunk, connection) set
// after a system-scope fence, receivers spinning on the flag before they
// forward or reduce.  B200 form:
//
//  * one CTA per (rank, channel).  A channel is a contiguous 16 B-aligned
//    sub-range of every chunk; the CTA runs its rank's whole op list on that
//    sub-range, so program order replaces intra-rank synchronisation and
//    only cross-rank receipts carry flags;
//  * warp-specialised TMA pipeline over a ring of shared-memory stages
//    (mbarriers full / fullr / ready / empty per stage):
//      warp 0     producer  waits the receipt counters a tile needs, then
//                           cp.async.bulk global->smem for every input;
//      warps 1-3  storers   stage s belongs to warp 1 + s % 3; lane o
//                           issues the cp.async.bulk smem->global store to
//                           output o (local and/or peer HBM) and retires it;
//      warp 4     signaler  releases byte counters in tile order, one fence
//                           per batch (or the storers do it themselves for
//                           latency-bound plans);
//      warps 5+   compute   REDUCE tiles: in-place f32 accumulate of the nin
//                           input tiles in smem (fixed order, one rounding);
//                           copy tiles go from producer to storer directly;
//  * window-major order for launches that stream past L2: every role walks
//    byte window w of every op before window w+1, so relayed receipts are
//    re-read from L2 (bulk copies carry L2 eviction hints);
//  * flags count BYTES of a (receipt, channel) sub-range that have landed:
//    (epoch-1)*len + bytes_done.  Producer and consumer may tile the same
//    chunk differently (copy tiles are a whole stage, reduce tiles a stage
//    divided by fan-in); counters are never reset and each CTA keeps its own
//    epoch in device memory (graph capture safe);
//  * loopback (every rank on this GPU, one launch) uses gpu scope;
//    multi-process (one rank per GPU, peers mapped through CUDA IPC over
//    NVLink) uses sys scope plus an entry handshake per (peer, channel).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../sccl/devprog.hpp"

namespace sccl {
namespace {

constexpr int NSW = kStorerWarps;   // storer warps 1..NSW: stage s belongs to storer warp 1 + s % NSW
constexpr int SIGW = 1 + NSW;        // signaler warp
constexpr int CW0 = SIGW + 1;        // first compute warp
constexpr int NCW = kThreads / 32 - CW0;  // compute warps
constexpr int NT = kThreads;
static_assert(NCW >= 4 && NT == (CW0 + NCW) * 32, "thread layout");
constexpr int NPART = NT - 32;       // threads of the unaligned path (all but the signaler)
constexpr int SIGQ = 64;             // tile completion ring (storers -> signaler), indexed by tile number
constexpr int NSTAGE = kMaxStages;   // barrier sets; stages in use = KParams::nstage (a multiple of NSW)
constexpr int SIGWIN = 8;            // ops the signaler keeps prepared ahead of their completion
constexpr size_t SMEM_HDR = kSmemHdr;
constexpr int kDescCache = 11264;    // bytes of descriptors cached per CTA  // mbarriers, completion ring, signaler op window, discard records
__host__ __device__ constexpr size_t smem_bytes(int tile, int nstage) { return SMEM_HDR + size_t(nstage) * tile; }
struct DPart {
  int64_t off, len;
};
// byte part i of K of an L-byte range in 16-byte units (the host's split16),
// with x / K = umulhi(x, ceil(2^64 / K)), exact for x < 2^64 / K (here
// x < K * L / 16): no 64-bit divide on the per-op path
__device__ __forceinline__ DPart dsplit16m(int64_t L, int K, uint64_t magic, int i) {
  if (K == 1) return {0, L};
  const uint64_t Uu = uint64_t(L) >> 4;
  const int64_t lo = int64_t(__umul64hi(uint64_t(i) * Uu, magic) << 4);
  const int64_t hi = (i == K - 1) ? L : int64_t(__umul64hi(uint64_t(i + 1) * Uu, magic) << 4);
  return {lo, hi - lo};
}
// x / d for the launch geometry (x, d < 2^16) with the host's magic
// floor(2^32 / d) + 1; magic 0 means d == 1
__device__ __forceinline__ int fastdiv(uint32_t x, uint32_t magic) { return int(magic ? __umulhi(x, magic) : x); }
// tiles of T bytes covering n bytes: a shift for power-of-two tiles (copies,
// and reductions of fan-in 2, 4, 8, ...), a divide otherwise
__device__ __forceinline__ uint32_t ntiles_of(uint64_t n, uint32_t T) {
  if ((T & (T - 1)) == 0) return uint32_t((n + T - 1) >> (__ffs(T) - 1));
  return n >> 31 ? uint32_t((n + T - 1) / T) : (uint32_t(n) + T - 1) / T;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
// L2 eviction policies for bulk copies: data read or written for the last
// time is evicted first, so it does not push out receipts that a later op
// of the receiver reads (forwards, reduce inputs).  Those are stored with
// the default policy, or evict-last when the plan discards them after use
// (kL2RelayPlain clear).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_load_hint(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* dst, const void* src_smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes), "l"(pol)
               : "memory");
}
// Drop the fully covered 128-byte L2 lines of [p, p + n) without writing
// them back (discard.global.L2): for receipt slots in scratch that have been
// consumed -- their bytes are dead until the next launch rewrites them.
// (the 32 lanes of a warp split the lines)
__device__ __forceinline__ void l2_discard_warp(const char* p, uint32_t n, int lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p), e = (a + n) & ~uintptr_t(127);
  for (uintptr_t l = ((a + 127) & ~uintptr_t(127)) + uintptr_t(lane) * 128; l < e; l += 32 * 128)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <bool SYS>
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// release fence before a flag store.  fence.release (PTX 8.6) is MEMBAR
// without the L1 invalidation (CCTL.IVALL) that fence.acq_rel adds: every
// use here is a release pattern, the acquire side uses ld.acquire.
template <bool SYS>
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void fence_acq() {  // after a relaxed load that observed a release
  if (SYS) asm volatile("fence.acquire.sys;" ::: "memory");
  else asm volatile("fence.acquire.gpu;" ::: "memory");
}
template <bool SYS>
__device__ __forceinline__ void fence_rel() {
  if (SYS) asm volatile("fence.release.sys;" ::: "memory");
  else asm volatile("fence.release.gpu;" ::: "memory");
}
template <bool SYS>
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  if (SYS) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void named_sync(int id) {  // every warp but the signaler
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "n"(NPART) : "memory");
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// Cooperative abort.  A wait that outlives timeout_ns records a diagnostic
// in host-mapped memory (the host maps it to SCCL_PEER_TIMEOUT), sets the
// launch-wide abort word (device memory) and this CTA's abort flag, and
// returns as if satisfied.  From then on the CTA publishes nothing -- no
// stores to peers or outputs, no counters, no LL words -- so no peer ever
// consumes a value computed from data that never arrived: ranks that depend
// on this one time out in turn (every slow wait also polls the abort word,
// so they give up at once).  Every role still walks its program to the end,
// so the mbarrier pipeline drains and the kernel exits normally: no trap,
// the CUDA context stays usable.  The plan itself is poisoned (its epochs
// and counters are out of step); the host refuses further launches.
__shared__ uint32_t cta_abort;  // per CTA
__device__ __forceinline__ bool cta_aborted() { return *reinterpret_cast<volatile uint32_t*>(&cta_abort) != 0; }
__device__ __forceinline__ bool launch_aborted(const KParams& p) {
  return p.abort && *reinterpret_cast<volatile int*>(p.abort) != 0;
}
__device__ __noinline__ void watchdog_fire(const KParams& p, int rank, int ch, int op, int slot, uint64_t target,
                                           uint64_t seen) {
  volatile int* e = p.errinfo;
  if (e && atomicCAS(p.errinfo, 0, -1) == 0) {
    e[1] = rank;
    e[2] = ch;
    e[3] = op;
    e[4] = slot;
    e[5] = int(target & 0x7fffffff);
    e[6] = int(seen & 0x7fffffff);
    __threadfence_system();
    e[0] = ERR_TIMEOUT;
    __threadfence_system();
  }
  *reinterpret_cast<volatile uint32_t*>(&cta_abort) = 1u;
  if (p.abort) *reinterpret_cast<volatile int*>(p.abort) = 1;
}
// an abort raised elsewhere in the launch: give up this wait too
__device__ __forceinline__ bool join_abort(const KParams& p) {
  if (cta_aborted()) return true;
  if (launch_aborted(p)) {
    *reinterpret_cast<volatile uint32_t*>(&cta_abort) = 1u;
    return true;
  }
  return false;
}

// mbarrier phase wait bounded by the watchdog: a pipeline hand-off that
// never completes (a bug, not a peer) aborts instead of hanging the GPU.
__device__ __noinline__ void mbar_wait_slow(uint64_t* b, uint32_t parity, const KParams& p, int rank, int ch,
                                            int op) {
  uint64_t t0 = 0;  // clock first read after 1024 tries (not on every missed hand-off)
  for (uint32_t spins = 1;; ++spins) {
    if (mbar_try(b, parity)) return;
    if ((spins & 1023) == 0) {
      if (join_abort(p)) return;
      const uint64_t now = globaltimer();
      if (!t0) t0 = now;
      else if (p.timeout_ns > 0 && (long long)(now - t0) > p.timeout_ns) {
        watchdog_fire(p, rank, ch, op, -4, parity, 0);
        return;
      }
    }
  }
}
__device__ __forceinline__ void mbar_wait_wd(uint64_t* b, uint32_t parity, const KParams& p, int rank, int ch,
                                             int op) {
  if (!mbar_try(b, parity)) mbar_wait_slow(b, parity, p, rank, ch, op);
}

// Spin until *f >= target; returns the value seen.  Bounded by timeout_ns.
template <bool SYS>
__device__ uint64_t wait_ge(const uint64_t* f, uint64_t target, const KParams& p, int rank, int ch, int op,
                            int slot) {
  uint64_t v = ld_acquire<SYS>(f);
  if (v >= target) return v;
  if (cta_aborted()) return target;
  // poll with relaxed (strong) loads -- no L1 invalidation per poll -- and
  // acquire once the target is reached.  The launch-wide abort word (a
  // global load) and the clock are first read after 1024 polls: on the
  // first miss they only delayed noticing the value (a dependent global
  // round trip per missed wait); the watchdog then counts from there.
  uint64_t t0 = 0;
  uint32_t spins = 0;
  while ((v = ld_relaxed<SYS>(f)) < target) {
    if (++spins > 64) __nanosleep(32);
    if ((spins & 1023) == 0) {
      if (join_abort(p)) return target;
      const uint64_t now = globaltimer();
      if (!t0) t0 = now;
      else if (p.timeout_ns > 0 && (long long)(now - t0) > p.timeout_ns) {
        watchdog_fire(p, rank, ch, op, slot, target, v);
        return target;
      }
    }
  }
  fence_acq<SYS>();
  return v;
}

// ---------------------------------------------------------------- arithmetic
// accumulator of one 16 B vector, per element type (fixed order, f32 for
// the 16-bit types, one rounding at the end: DESIGN.md "Reduction order")
template <int DT>
struct Vec;
template <>
struct Vec<0> {  // u8, wrapping
  uint4 a;
  __device__ void init(uint4 v) { a = v; }
  __device__ void add(uint4 v) {
    a.x = __vadd4(a.x, v.x);
    a.y = __vadd4(a.y, v.y);
    a.z = __vadd4(a.z, v.z);
    a.w = __vadd4(a.w, v.w);
  }
  __device__ uint4 out() const { return a; }
};
template <>
struct Vec<1> {  // i32, two's-complement wrap
  uint4 a;
  __device__ void init(uint4 v) { a = v; }
  __device__ void add(uint4 v) {
    a.x += v.x;
    a.y += v.y;
    a.z += v.z;
    a.w += v.w;
  }
  __device__ uint4 out() const { return a; }
};
// Two bf16 / f16 inputs: widening both to f32, adding and rounding once
// equals the correctly rounded 16-bit add (the f32 sum of two such values is
// exact unless their exponents differ by more than the f32/16-bit precision
// gap, and then it cannot land on a 16-bit rounding tie), so one packed
// add.rn per two elements gives the Vec<DT> result bit for bit (NaNs come out
// canonical, 0x7fff, as in Vec<DT>::out).
template <int DT>
__device__ __forceinline__ uint32_t add_pair_w(uint32_t a, uint32_t b) {
  uint32_t d;
  if constexpr (DT == 3) asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  else asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
template <int DT>
__device__ __forceinline__ uint4 add_pair(uint4 a, uint4 b) {
  return make_uint4(add_pair_w<DT>(a.x, b.x), add_pair_w<DT>(a.y, b.y), add_pair_w<DT>(a.z, b.z),
                    add_pair_w<DT>(a.w, b.w));
}
template <>
struct Vec<2> {  // f32, adds in input order
  float a[4];
  __device__ void init(uint4 v) {
    a[0] = __uint_as_float(v.x);
    a[1] = __uint_as_float(v.y);
    a[2] = __uint_as_float(v.z);
    a[3] = __uint_as_float(v.w);
  }
  __device__ void add(uint4 v) {
    a[0] = __fadd_rn(a[0], __uint_as_float(v.x));
    a[1] = __fadd_rn(a[1], __uint_as_float(v.y));
    a[2] = __fadd_rn(a[2], __uint_as_float(v.z));
    a[3] = __fadd_rn(a[3], __uint_as_float(v.w));
  }
  __device__ uint4 out() const {
    return make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
  }
};
template <>
struct Vec<3> {  // bf16: widen, add in f32 in input order, round once
  float a[8];
  __device__ void init(uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = __uint_as_float(w[k] << 16);
      a[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
  }
  __device__ void add(uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[2 * k] = __fadd_rn(a[2 * k], __uint_as_float(w[k] << 16));
      a[2 * k + 1] = __fadd_rn(a[2 * k + 1], __uint_as_float(w[k] & 0xffff0000u));
    }
  }
  __device__ uint4 out() const {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t l = __bfloat16_as_ushort(__float2bfloat16_rn(a[2 * k]));
      uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(a[2 * k + 1]));
      w[k] = l | (h << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Vec<4> {  // f16: widen, add in f32 in input order, round once
  float a[8];
  __device__ void init(uint4 v) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __half22float2(h[k]);
      a[2 * k] = f.x;
      a[2 * k + 1] = f.y;
    }
  }
  __device__ void add(uint4 v) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __half22float2(h[k]);
      a[2 * k] = __fadd_rn(a[2 * k], f.x);
      a[2 * k + 1] = __fadd_rn(a[2 * k + 1], f.y);
    }
  }
  __device__ uint4 out() const {
    uint4 r;
    __half2* h = reinterpret_cast<__half2*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __halves2half2(__float2half_rn(a[2 * k]), __float2half_rn(a[2 * k + 1]));
    return r;
  }
};

// element-wise path (unaligned ops, the < 16 B chunk tail): global -> global.
// in(k) / out(o) return input k's / output o's base address.
template <int DT, class In, class Out>
__device__ void elem_op(In in, int nin, Out out, int nout, int64_t off, int64_t nbytes, int tid, int nthr) {
  constexpr int ES = (DT == 0) ? 1 : (DT == 3 || DT == 4) ? 2 : 4;
  for (int64_t i = tid; i < nbytes / ES; i += nthr) {
    const int64_t b = off + i * ES;
    if (DT == 0) {
      uint8_t a = *(const volatile uint8_t*)(in(0) + b);
      for (int k = 1; k < nin; ++k) a = uint8_t(a + *(const volatile uint8_t*)(in(k) + b));
      for (int o = 0; o < nout; ++o) *(volatile uint8_t*)(out(o) + b) = a;
    } else if (DT == 1) {
      uint32_t a = *(const volatile uint32_t*)(in(0) + b);
      for (int k = 1; k < nin; ++k) a += *(const volatile uint32_t*)(in(k) + b);
      for (int o = 0; o < nout; ++o) *(volatile uint32_t*)(out(o) + b) = a;
    } else if (DT == 2) {
      float a = __int_as_float(*(const volatile int*)(in(0) + b));
      for (int k = 1; k < nin; ++k) a = __fadd_rn(a, __int_as_float(*(const volatile int*)(in(k) + b)));
      for (int o = 0; o < nout; ++o) *(volatile int*)(out(o) + b) = __float_as_int(a);
    } else {
      auto widen = [](uint16_t h) -> float {
        if (DT == 3) return __uint_as_float(uint32_t(h) << 16);
        return __half2float(__ushort_as_half(h));
      };
      float a = widen(*(const volatile uint16_t*)(in(0) + b));
      for (int k = 1; k < nin; ++k) a = __fadd_rn(a, widen(*(const volatile uint16_t*)(in(k) + b)));
      uint16_t r = (DT == 3) ? __bfloat16_as_ushort(__float2bfloat16_rn(a)) : __half_as_ushort(__float2half_rn(a));
      for (int o = 0; o < nout; ++o) *(volatile uint16_t*)(out(o) + b) = r;
    }
  }
}

// debug trace (p.trace != nullptr): one record per event, per-CTA region
__device__ __forceinline__ void trace_ev(const KParams& p, uint32_t* cnt, int ev, uint32_t op, uint32_t tile) {
  if (!p.trace) return;
  const uint32_t i = atomicAdd(cnt, 1u);
  if (i >= uint32_t(p.trace_cap)) return;
  uint64_t* r = p.trace + (size_t(blockIdx.x) * p.trace_cap + i) * 2;
  r[0] = globaltimer();
  r[1] = uint64_t(ev) | (uint64_t(op) << 8) | (uint64_t(tile) << 32);
}

// one op prepared by the signaler: output o's counter address (or null),
// the op's per-channel byte range and tiling
struct SigOp {
  uint64_t* sig[kMaxOpOut];
  uint64_t fbase, qlen, wlo, whi;  // the op's counter base and part length; this item's byte window
  uint32_t T, ntiles, every, nout, oi;
};
struct Smem {
  // per stage: full = a COPY tile landed (storer waits), fullr = a REDUCE
  // tile's inputs landed (compute warps wait), ready = reduced tile in smem
  // (storer waits), empty = stage read out (producer waits).  Each barrier
  // counts only the uses that touch it, so no role can alias a phase.
  uint64_t full[NSTAGE], fullr[NSTAGE], ready[NSTAGE], empty[NSTAGE];
  SigOp win[SIGWIN];     // signaler's op window (ring)
  // reduce tile in stage s: input k's global range if it is a scratch receipt
  // read for the last time (producer lane k writes it with the load; the
  // compute warps drop those L2 lines after reducing: dead data, no write-back)
  const char* dsc[NSTAGE][32];
  uint32_t dsn[NSTAGE];
  uint32_t done[SIGQ];   // it + 1 once tile `it`'s writes have landed (storer release, signaler acquire)
  uint32_t published;    // tiles < published are complete and their counters released (in tile order)
  uint32_t entry_mask;   // peers whose entry handshake this CTA has seen
  uint32_t trace_n;      // debug trace records written by this CTA
  // this CTA's op / in / out descriptors, copied in the prologue when they
  // fit (otherwise read from global memory): the per-op descriptor loads of
  // every role hit shared memory instead of L1/L2
  alignas(16) uint8_t dcache[kDescCache];
};
static_assert(sizeof(Smem) <= SMEM_HDR, "smem header");

// Simple (bulk) protocol.  Roles per CTA:
//   warp 0          producer: waits the receipt counters of a tile, then
//                   cp.async.bulk global->smem of every input;
//   warps 1..NSW    storers: stage s belongs to storer warp 1 + s % NSW.
//                   Lane o issues the bulk store to output o, every lane
//                   commits and retires its own bulk group, so a storer
//                   warp has one tile in flight and posts it to the
//                   completion ring the moment its writes have landed;
//   warp SIGW       signaler: walks the program in the same tile order,
//                   with every op's counter addresses loaded (lane o:
//                   output o) before its tiles complete; per batch of
//                   completed tiles of one op, one fence and one relaxed
//                   store of the newest byte count (counters are byte
//                   prefixes, so tiles publish in order);
//   warps CW0..     compute: REDUCE tiles, f32 accumulate in smem.
// p.selfpub = 1 (latency-bound plans): the storer warp that completed a
// tile releases its counters itself once every earlier tile has (no
// hand-off), at the cost of a fence on the store path.
// No role blocks on a peer while holding a completed but unreleased tile,
// so the program order argument of DESIGN.md section 4 gives deadlock
// freedom without draining heuristics.
template <int DT, bool SYS>
__global__ void __launch_bounds__(NT, 2) exec_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  uint8_t* const bufs = smem_raw + SMEM_HDR;
  const size_t STAGE = size_t(p.tile);
  const uint32_t NST = uint32_t(p.nstage);
  __shared__ const char* s_inp[kMaxOpIn];
  __shared__ char* s_outp[kMaxOpOut];
  __shared__ uint64_t s_e;
  __shared__ uint32_t s_nwin;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lr = fastdiv(blockIdx.x, p.nch_magic), ch = int(blockIdx.x) - lr * p.nch;
  const int cb = fastdiv(uint32_t(ch), p.kc_magic), cg = ch - cb * p.kc;  // chunk group, byte part
  const int rank = p.rank0 + lr;
  uint64_t* const myflags = reinterpret_cast<uint64_t*>(p.base[rank][SP_FLAGS_IDX]);

  if (tid == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.fullr[s], 1);
      mbar_init(&S.ready[s], NCW);
      mbar_init(&S.empty[s], 1);
    }
    S.published = S.trace_n = 0;
    cta_abort = 0;
    for (int s = 0; s < NSTAGE; ++s) {
      S.dsn[s] = 0;
      for (int k = 0; k < 32; ++k) S.dsc[s][k] = nullptr;
    }
    S.entry_mask = 1u << rank;
    s_e = p.epochs[blockIdx.x] + 1;
    s_nwin = p.nwin ? p.nwin[blockIdx.x] : 1u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < SIGQ; i += NT) S.done[i] = 0;
  const uint4 d0 = reinterpret_cast<const uint4*>(p.dtab)[(rank * p.kc + cg) * 2],
              d1 = reinterpret_cast<const uint4*>(p.dtab)[(rank * p.kc + cg) * 2 + 1];
  const uint32_t ob = d0.x, oe = d0.y, ib = d0.z, xb = d1.x;
  const uint32_t nb_ops = (oe - ob) * uint32_t(sizeof(DevOp)), nb_ins = (d0.w - ib) * uint32_t(sizeof(DevIn));
  const uint32_t nb_all = nb_ops + nb_ins + (d1.y - xb) * uint32_t(sizeof(DevOut));
  const bool cached = nb_all <= uint32_t(kDescCache) && p.dcache_min_ops && oe - ob >= uint32_t(p.dcache_min_ops);
  if (cached)  // every thread copies 16-byte words; the three ranges load in parallel
    for (uint32_t w = tid; w < nb_all / 16; w += NT) {
      const uint32_t o = w * 16;
      const uint4* src = o < nb_ops ? reinterpret_cast<const uint4*>(p.ops + ob) + w
                         : o < nb_ops + nb_ins ? reinterpret_cast<const uint4*>(p.ins + ib) + (o - nb_ops) / 16
                                               : reinterpret_cast<const uint4*>(p.outs + xb) + (o - nb_ops - nb_ins) / 16;
      reinterpret_cast<uint4*>(S.dcache)[w] = *src;
    }
  // indexed like p.ops / p.ins / p.outs (biased by this CTA's range
  // starts); kept in shared memory, not in registers (80 per thread)
  __shared__ const DevOp* OPS;
  __shared__ const DevIn* INS;
  __shared__ const DevOut* OUTS;
  if (tid == 0) {
    OPS = (cached ? reinterpret_cast<const DevOp*>(S.dcache) : p.ops + ob) - ob;
    INS = (cached ? reinterpret_cast<const DevIn*>(S.dcache + nb_ops) : p.ins + ib) - ib;
    OUTS = (cached ? reinterpret_cast<const DevOut*>(S.dcache + nb_ops + nb_ins) : p.outs + xb) - xb;
  }
  __syncthreads();
  if (tid == 0) trace_ev(p, &S.trace_n, TR_START, 0, 0);
  const uint64_t e = s_e;
  if (p.multiprocess)  // "rank `rank`, channel ch entered launch e"
    for (int t = tid; t < p.P; t += NT)
      if (t != rank) {
        fence_rel<SYS>();
        st_relaxed<SYS>(reinterpret_cast<uint64_t*>(p.base[t][SP_FLAGS_IDX]) + p.entry_base + rank * p.nch + ch, e);
      }

  uint32_t it = 0;  // tile number (same sequence in every role)
  // it % NST and (it / NST) & 1, kept incrementally (NST is a runtime
  // value: a modulo per tile was a divide on every role's tile path)
  uint32_t st = 0, sph = 0;
  auto next_tile = [&]() {
    ++it;
    if (++st == NST) {
      st = 0;
      sph ^= 1u;
    }
  };
  const uint32_t my_stage_class = uint32_t(warp - 1);  // storer warps
  // bit s = parity of stage s's next phase of a barrier that only some uses
  // touch: storers track `full` (copy uses) and `ready` (reduce uses),
  // compute warps `fullr` (reduce uses)
  uint32_t cpar = 0, rpar = 0;
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();

  // entry handshake before the first store into peer d (multi-process only)
  auto await_entry = [&](int d, int opi) {
    if (!(atomicOr(&S.entry_mask, 0u) & (1u << d))) {
      wait_ge<SYS>(myflags + p.entry_base + d * p.nch + ch, e, p, rank, ch, opi, -2);
      atomicOr(&S.entry_mask, 1u << d);
    }
  };

  // Window-major order (p.window > 0): the CTA walks byte window w of every
  // op before window w+1 of any, so a receipt is forwarded or reduced a few
  // tiles after it landed, while it is still in L2, instead of one whole op
  // later.  Every role walks the same (window, op, tile) sequence.
  const uint32_t W = p.window;
  const uint32_t nwin = s_nwin;
  auto item = [&](const DevOp& op, uint32_t w, DPart& q, uint64_t& wlo, uint64_t& whi) -> bool {
    if (op.kind == 2) return false;  // (a CTA's program holds only its chunk group's ops)
    q = dsplit16m(int64_t(op.len), p.kb, p.kb_magic, cb);
    if (q.len == 0) return false;  // empty sub-range: nothing sent, nothing awaited
    wlo = W ? uint64_t(w) * W : 0;
    if (wlo >= uint64_t(q.len)) return false;
    whi = W ? min(uint64_t(q.len), wlo + W) : uint64_t(q.len);
    return true;
  };

  // copy-only aligned programs: the compute warps go straight to the final
  // barrier instead of walking the program (they would only take issue slots)
  if (warp != SIGW) {
    if (!(warp >= CW0 && d1.z))
    for (uint32_t w = 0; w < nwin; ++w)
    for (uint32_t oi = ob; oi < oe; ++oi) {
      const DevOp op = OPS[oi];
      if (op.kind == 2) {  // end-of-program waits (after the last window): every receipt has landed
        if (warp == 0 && w + 1 == nwin)
          for (int i = lane; i < op.nin; i += 32) {
            const DevIn in = INS[op.in_begin + i];
            if (int(in.chunk % uint32_t(p.kc)) != cg) continue;
            const DPart q = dsplit16m(int64_t(in.len), p.kb, p.kb_magic, cb);
            if (q.len) wait_ge<SYS>(myflags + uint64_t(in.flag) * p.nch + ch, e * uint64_t(q.len), p, rank, ch,
                                    int(oi - ob), in.flag);
          }
        continue;
      }
      DPart q;
      uint64_t wlo, whi;
      if (!item(op, w, q, wlo, whi)) continue;
      const uint64_t fbase = (e - 1) * uint64_t(q.len);

      if (!op.vec) {
        // ---- unaligned op (op-major plans only): whole CTA (but the signaler),
        // element-wise, synchronous.  Every earlier tile's stores are
        // complete: each storer warp retires its tile before it moves on.
        const int ptid = tid < 32 * SIGW ? tid : tid - 32;
        named_sync(1);
        if (tid < op.nin) {
          const DevIn in = INS[op.in_begin + tid];
          s_inp[tid] = p.base[in.rank][in.space] + in.off;
          if (in.flag >= 0)
            wait_ge<SYS>(myflags + uint64_t(in.flag) * p.nch + ch, fbase + uint64_t(q.len), p, rank, ch,
                         int(oi - ob), in.flag);
        }
        if (tid < op.nout) {
          const DevOut d = OUTS[op.out_begin + tid];
          s_outp[tid] = p.base[d.rank][d.space] + d.off;
          if (p.multiprocess && d.rank != rank) await_entry(d.rank, int(oi - ob));
        }
        named_sync(1);
        if (!cta_aborted()) {
          auto in = [&](int k) { return s_inp[k]; };
          auto out = [&](int o) { return s_outp[o]; };
          if (op.kind == 0) elem_op<0>(in, 1, out, op.nout, q.off, q.len, ptid, NPART);
          else elem_op<DT>(in, op.nin, out, op.nout, q.off, q.len, ptid, NPART);
        }
        named_sync(1);
        if (tid == 32 && !cta_aborted()) {
          fence_rel<SYS>();
          for (int o = 0; o < op.nout; ++o) {
            const DevOut d = OUTS[op.out_begin + o];
            if (d.flag >= 0)
              st_relaxed<SYS>(reinterpret_cast<uint64_t*>(p.base[d.rank][SP_FLAGS_IDX]) + uint64_t(d.flag) * p.nch + ch,
                              fbase + uint64_t(q.len));
          }
        }
        named_sync(1);
        continue;
      }

      // ---- pipelined op: tiles of this window ----
      const uint32_t T = op.tile;  // (host-computed: stage, or stage / fan-in for reductions)
      const uint32_t ntiles = ntiles_of(whi - wlo, T);

      if (warp == 0) {
        // ================= producer =================
        uint64_t ready = 0;  // lane k tracks input k's counter (k < 32)
        const char* src = nullptr;
        int32_t flag = -1;
        bool dead_after = false;  // a scratch receipt: consumed by this read
        if (lane < op.nin) {
          const DevIn in = INS[op.in_begin + lane];
          src = p.base[in.rank][in.space] + in.off + q.off;
          flag = in.flag;
          dead_after = p.discard && in.dead_after;
        }
        if (op.raw && lane == 0)  // input written by an earlier tile of this CTA
          while (ld_acquire_cta(&S.published) < it) __nanosleep(32);
        __syncwarp();
        if (lane == 0) trace_ev(p, &S.trace_n, TR_ENTRY, oi, 0);  // producer: op descriptors read
        for (uint32_t t = 0; t < ntiles; ++t, next_tile()) {
          const uint32_t s = st, ph = sph;
          const uint64_t lo = wlo + uint64_t(t) * T;
          const uint32_t n = uint32_t(min(uint64_t(T), whi - lo));
          const uint32_t nv = n & ~15u;
          if (flag >= 0) {
            const uint64_t need = fbase + lo + n;
            if (ready < need)
              ready = wait_ge<SYS>(myflags + uint64_t(flag) * p.nch + ch, need, p, rank, ch, int(oi - ob), flag);
          }
          __syncwarp();
          if (p.trace) {  // (tile bit 31: some input of this tile has a receipt counter)
            const bool waited = __any_sync(0xffffffffu, flag >= 0);
            if (lane == 0) trace_ev(p, &S.trace_n, TR_FLAG, oi, t | (waited ? 0x80000000u : 0u));
          }
          uint64_t* const fb = op.kind == 1 ? &S.fullr[s] : &S.full[s];
          if (lane == 0) {
            mbar_wait_wd(&S.empty[s], ph ^ 1, p, rank, ch, int(oi - ob));
            trace_ev(p, &S.trace_n, TR_EMPTY, oi, t);
          }
          __syncwarp();
          if (p.discard && op.kind == 1) {  // dead scratch receipts of this reduce tile
            S.dsc[s][lane] = (dead_after && nv) ? src + lo : nullptr;
            if (lane == 0) S.dsn[s] = nv;
          }
          if (lane == 0) mbar_arrive_tx(fb, nv * op.nin);
          __syncwarp();
          if (lane < op.nin && nv) {
            fence_proxy_async_global();  // generic acquire above -> async-proxy reads below
            if (p.l2hint) bulk_load_hint(bufs + size_t(s) * STAGE + size_t(lane) * T, src + lo, nv, fb, pol_first);
            else bulk_load(bufs + size_t(s) * STAGE + size_t(lane) * T, src + lo, nv, fb);
          }
          if (p.trace) {
            __syncwarp();
            if (lane == 0) trace_ev(p, &S.trace_n, TR_ISSUED, oi, t);
          }
        }
      } else if (warp >= CW0) {
        // ================= compute (REDUCE tiles; copy tiles go straight to the storer) =================
        for (uint32_t t = 0; t < ntiles; ++t, next_tile()) {
          const uint32_t s = st;
          if (op.kind == 1) {
            mbar_wait_wd(&S.fullr[s], (rpar >> s) & 1u, p, rank, ch, int(oi - ob));
            rpar ^= 1u << s;
            if (warp == CW0 && lane == 0) trace_ev(p, &S.trace_n, TR_FULL, oi, t);
            const uint64_t lo = wlo + uint64_t(t) * T;
            const uint32_t nv = uint32_t(min(uint64_t(T), whi - lo)) >> 4;
            uint4* b0 = reinterpret_cast<uint4*>(bufs + size_t(s) * STAGE);
            if ((DT == 3 || DT == 4) && op.nin == 2) {  // bf16 / f16 pair: one packed add per 2 elements
              const uint4* b1 = reinterpret_cast<const uint4*>(bufs + size_t(s) * STAGE + size_t(T));
              for (uint32_t v = tid - CW0 * 32; v < nv; v += NCW * 32) b0[v] = add_pair<DT>(b0[v], b1[v]);
            } else {
              // two vectors per thread in flight (same operands, same order;
              // float types only: the integer kernels keep their registers)
              const uint32_t step = NCW * 32;
              uint32_t v = tid - CW0 * 32;
              if constexpr (DT >= 2)
              for (; v + step < nv; v += 2 * step) {
                Vec<DT> acc0, acc1;
                acc0.init(b0[v]);
                acc1.init(b0[v + step]);
                for (int k = 1; k < op.nin; ++k) {
                  const uint4* bk = reinterpret_cast<const uint4*>(bufs + size_t(s) * STAGE + size_t(k) * T);
                  const uint4 x0 = bk[v], x1 = bk[v + step];
                  acc0.add(x0);
                  acc1.add(x1);
                }
                b0[v] = acc0.out();
                b0[v + step] = acc1.out();
              }
              for (; v < nv; v += step) {
                Vec<DT> acc;
                acc.init(b0[v]);
                for (int k = 1; k < op.nin; ++k)
                  acc.add(reinterpret_cast<const uint4*>(bufs + size_t(s) * STAGE + size_t(k) * T)[v]);
                b0[v] = acc.out();
              }
            }
            if (p.discard) {  // dead scratch receipts of this tile: drop their L2 lines (no write-back)
              const uint32_t dn = S.dsn[s];
              for (int k = warp - CW0; k < op.nin; k += NCW)
                if (const char* d = S.dsc[s][k]) l2_discard_warp(d, dn, lane);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.ready[s]);
          }
        }
      } else {
        // ================= storer warp (stages s with s % NSW == warp - 1) =================
        char* outp = nullptr;
        uint64_t* sig = nullptr;  // output `lane`'s counter at its destination, if it has one
        bool every = false;
        if (lane < op.nout) {
          const DevOut d = OUTS[op.out_begin + lane];
          outp = p.base[d.rank][d.space] + d.off + q.off;
          if (d.flag >= 0) {
            sig = reinterpret_cast<uint64_t*>(p.base[d.rank][SP_FLAGS_IDX]) + uint64_t(d.flag) * p.nch + ch;
            every = d.every_tile;
          }
          if (p.multiprocess && d.rank != rank) await_entry(d.rank, int(oi - ob));
        }
        __syncwarp();
        for (uint32_t t = 0; t < ntiles; ++t, next_tile()) {
          const uint32_t s = st;
          if (s % NSW != my_stage_class) continue;
          const uint64_t lo = wlo + uint64_t(t) * T;
          const uint32_t n = uint32_t(min(uint64_t(T), whi - lo));
          const uint32_t nv = n & ~15u;
          if (op.kind == 1) {  // reduce: the compute warps' result
            mbar_wait_wd(&S.ready[s], (rpar >> s) & 1u, p, rank, ch, int(oi - ob));
            rpar ^= 1u << s;
          } else {  // copy: the loaded tile itself
            mbar_wait_wd(&S.full[s], (cpar >> s) & 1u, p, rank, ch, int(oi - ob));
            cpar ^= 1u << s;
            if (lane == 0) trace_ev(p, &S.trace_n, TR_FULL, oi, t);
          }
          if (lane == 0) trace_ev(p, &S.trace_n, TR_READY, oi, t);
          const bool ab = cta_aborted();  // aborted: publish nothing (see watchdog_fire)
          if (n > nv && lane == 0 && !ab) {  // < 16 B chunk tail: element-wise, global -> global
            // addresses from the descriptors per element (no pointer arrays on the stack)
            const DevIn* ins = INS + op.in_begin;
            const DevOut* outs = OUTS + op.out_begin;
            const int64_t qo = q.off;
            auto in = [&](int k) -> const char* { return p.base[ins[k].rank][ins[k].space] + ins[k].off + qo; };
            auto out = [&](int o) -> char* { return p.base[outs[o].rank][outs[o].space] + outs[o].off + qo; };
            if (op.kind == 0) elem_op<0>(in, 1, out, op.nout, int64_t(lo + nv), n - nv, 0, 1);
            else elem_op<DT>(in, op.nin, out, op.nout, int64_t(lo + nv), n - nv, 0, 1);
          }
          if (outp && nv && !ab) {
            if (p.l2hint && !((p.l2hint & kL2RelayPlain) && every))
              bulk_store_hint(outp + lo, bufs + size_t(s) * STAGE, nv, every ? pol_last : pol_first);
            else bulk_store(outp + lo, bufs + size_t(s) * STAGE, nv);
          }
          bulk_commit();
          bulk_wait_read<0>();  // smem read: the stage goes back to the producer
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.empty[s]);
          bulk_wait<0>();               // writes landed
          fence_proxy_async_global();   // async-proxy writes -> generic observers
          __syncwarp();                 // (and lane 0's tail writes -> every lane)
          if (p.selfpub) {
            if (lane == 0) {
              trace_ev(p, &S.trace_n, TR_DONE, oi, t);
              while (ld_acquire_cta(&S.published) != it) {  // earlier tiles publish first
              }
            }
            __syncwarp();
            if (sig && (every || lo + n == uint64_t(q.len)) && !ab) {
              fence_rel<SYS>();
              st_relaxed<SYS>(sig, fbase + lo + n);
            }
            __syncwarp();
            if (lane == 0) {
              trace_ev(p, &S.trace_n, TR_PUB, oi, uint32_t(lo + n));
              st_release_cta(&S.published, it + 1);
            }
          } else if (lane == 0) {
            trace_ev(p, &S.trace_n, TR_DONE, oi, t);
            while (it - ld_acquire_cta(&S.published) >= SIGQ) {  // ring back-pressure
            }
            st_release_cta(&S.done[it % SIGQ], it + 1);
          }
        }
      }
    }
  } else if (!p.selfpub) {
    // ================= signaler =================
    // Walks the same (window, op, tile) sequence as the other roles.  Up to
    // SIGWIN items ahead of completion are prepared in shared memory (lane o
    // loads output o's counter address), so nothing on the signal path waits
    // for a global load.  Each batch of consecutive completed tiles -- across
    // item boundaries -- gets one release fence, then one relaxed store of
    // the newest byte count per counter.
    uint32_t nw = ob < oe ? 0 : nwin, next_oi = ob, wh = 0, wt = 0, t0 = 0, wtiles = 0;  // items [wh, wt)
    for (;;) {
      while (wt - wh < uint32_t(SIGWIN) && nw < nwin) {  // prepare items ahead
        const uint32_t oi = next_oi, w = nw;
        if (++next_oi == oe) {
          next_oi = ob;
          ++nw;
        }
        if (oi >= oe) continue;
        const DevOp op = OPS[oi];
        DPart q;
        uint64_t wlo, whi;
        if (!op.vec || !item(op, w, q, wlo, whi)) continue;
        SigOp& x = S.win[wt % SIGWIN];
        bool every = false;
        if (lane < op.nout) {
          const DevOut d = OUTS[op.out_begin + lane];
          x.sig[lane] = d.flag >= 0 ? reinterpret_cast<uint64_t*>(p.base[d.rank][SP_FLAGS_IDX]) +
                                          uint64_t(d.flag) * p.nch + ch
                                    : nullptr;
          every = d.every_tile;
        }
        const uint32_t em = __ballot_sync(0xffffffffu, every);
        const uint32_t T = op.tile;
        const uint32_t nt = ntiles_of(whi - wlo, T);
        if (lane == 0) {
          x.fbase = (e - 1) * uint64_t(q.len);
          x.qlen = uint64_t(q.len);
          x.wlo = wlo;
          x.whi = whi;
          x.T = T;
          x.ntiles = nt;
          x.every = em;
          x.nout = op.nout;
          x.oi = oi;
        }
        wtiles += nt;
        ++wt;
      }
      __syncwarp();
      if (wh == wt) break;  // every tile published
      uint32_t k = 0;       // tiles it, it+1, ... that have landed
      if (lane == 0)
        while (k < wtiles && k < uint32_t(SIGQ) && ld_acquire_cta(&S.done[(it + k) % SIGQ]) == it + k + 1) ++k;
      k = __shfl_sync(0xffffffffu, k, 0);
      if (k == 0) continue;
      fence_rel<SYS>();
      const bool ab = cta_aborted();  // aborted: advance, publish nothing
      for (uint32_t left = k; left;) {
        const SigOp& x = S.win[wh % SIGWIN];
        const uint32_t take = min(left, x.ntiles - t0);
        const uint32_t tl = t0 + take - 1;  // newest published tile of this item
        const bool item_done = tl + 1 == x.ntiles;
        const uint64_t end = min(x.wlo + uint64_t(tl + 1) * x.T, x.whi);
        const bool last = end == x.qlen;  // the op's final byte
        if (lane < int(x.nout)) {
          uint64_t* f = x.sig[lane];
          if (f && (((x.every >> lane) & 1u) || last) && !ab) st_relaxed<SYS>(f, x.fbase + end);
        }
        if (lane == 0) trace_ev(p, &S.trace_n, TR_PUB, x.oi, uint32_t(end));
        t0 += take;
        left -= take;
        if (item_done) {
          ++wh;
          t0 = 0;
        }
      }
      __syncwarp();
      wtiles -= k;
      it += k;
      if (lane == 0) st_release_cta(&S.published, it);
    }
  }
  __syncthreads();
  if (tid == 0) {
    trace_ev(p, &S.trace_n, TR_END, 0, 0);
    p.epochs[blockIdx.x] = e;
  }
}


// ============================================================================
// LL protocol (small messages).  Every receipt slot holds (4 data bytes,
// 4 flag bytes) words; the sender stores data and the launch epoch together
// with one 8-byte-atomic half of a 16-byte store, the receiver polls the
// words themselves.  No counters, no fences, per-word pipelining across
// hops; 2x the bytes, so only for small chunks.
// ============================================================================
constexpr int LL_NT = kLLThreads;

template <int DT>
struct Acc8;  // 8 data bytes, same arithmetic as Vec<DT>
template <>
struct Acc8<0> {
  uint32_t a[2];
  __device__ void init(uint2 v) { a[0] = v.x, a[1] = v.y; }
  __device__ void add(uint2 v) { a[0] = __vadd4(a[0], v.x), a[1] = __vadd4(a[1], v.y); }
  __device__ uint2 out() const { return make_uint2(a[0], a[1]); }
};
template <>
struct Acc8<1> {
  uint32_t a[2];
  __device__ void init(uint2 v) { a[0] = v.x, a[1] = v.y; }
  __device__ void add(uint2 v) { a[0] += v.x, a[1] += v.y; }
  __device__ uint2 out() const { return make_uint2(a[0], a[1]); }
};
template <>
struct Acc8<2> {
  float a[2];
  __device__ void init(uint2 v) { a[0] = __uint_as_float(v.x), a[1] = __uint_as_float(v.y); }
  __device__ void add(uint2 v) {
    a[0] = __fadd_rn(a[0], __uint_as_float(v.x));
    a[1] = __fadd_rn(a[1], __uint_as_float(v.y));
  }
  __device__ uint2 out() const { return make_uint2(__float_as_uint(a[0]), __float_as_uint(a[1])); }
};
template <>
struct Acc8<3> {
  float a[4];
  __device__ void init(uint2 v) {
    a[0] = __uint_as_float(v.x << 16), a[1] = __uint_as_float(v.x & 0xffff0000u);
    a[2] = __uint_as_float(v.y << 16), a[3] = __uint_as_float(v.y & 0xffff0000u);
  }
  __device__ void add(uint2 v) {
    a[0] = __fadd_rn(a[0], __uint_as_float(v.x << 16));
    a[1] = __fadd_rn(a[1], __uint_as_float(v.x & 0xffff0000u));
    a[2] = __fadd_rn(a[2], __uint_as_float(v.y << 16));
    a[3] = __fadd_rn(a[3], __uint_as_float(v.y & 0xffff0000u));
  }
  __device__ uint2 out() const {
    auto b = [](float f) { return uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(f))); };
    return make_uint2(b(a[0]) | (b(a[1]) << 16), b(a[2]) | (b(a[3]) << 16));
  }
};
template <>
struct Acc8<4> {
  float a[4];
  __device__ static float h(uint32_t w, int hi) { return __half2float(__ushort_as_half(uint16_t(hi ? w >> 16 : w))); }
  __device__ void init(uint2 v) { a[0] = h(v.x, 0), a[1] = h(v.x, 1), a[2] = h(v.y, 0), a[3] = h(v.y, 1); }
  __device__ void add(uint2 v) {
    a[0] = __fadd_rn(a[0], h(v.x, 0));
    a[1] = __fadd_rn(a[1], h(v.x, 1));
    a[2] = __fadd_rn(a[2], h(v.y, 0));
    a[3] = __fadd_rn(a[3], h(v.y, 1));
  }
  __device__ uint2 out() const {
    auto b = [](float f) { return uint32_t(__half_as_ushort(__float2half_rn(f))); };
    return make_uint2(b(a[0]) | (b(a[1]) << 16), b(a[2]) | (b(a[3]) << 16));
  }
};

__device__ __forceinline__ uint4 ld_ll(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_ll(void* p, uint2 d, uint32_t f) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(d.x), "r"(f), "r"(d.y), "r"(f)
               : "memory");
}

// 8 data bytes of an LL slot at pair index; waits for the epoch flag of
// every valid word (gives up under the watchdog / an abort: the caller then
// stores nothing, cta_abort is set)
template <bool SYS>
__device__ uint2 ll_read(const char* slot, int64_t pair, bool two, uint32_t ef, const KParams& p, int rank, int ch,
                         int op, bool& ok) {
  const char* a = slot + pair * 16;
  uint4 v = ld_ll(a);
  if (v.y == ef && (!two || v.w == ef)) return make_uint2(v.x, v.z);
  if (cta_aborted()) {
    ok = false;
    return make_uint2(0, 0);
  }
  uint64_t t0 = 0;  // (abort word and clock first read after 1024 polls, as in wait_ge)
  uint32_t spins = 0;
  for (;;) {
    v = ld_ll(a);
    if (v.y == ef && (!two || v.w == ef)) return make_uint2(v.x, v.z);
    if (++spins > 32) __nanosleep(20);
    if ((spins & 1023) == 0) {
      if (join_abort(p)) {
        ok = false;
        return make_uint2(0, 0);
      }
      const uint64_t now = globaltimer();
      if (!t0) t0 = now;
      else if (p.timeout_ns > 0 && (long long)(now - t0) > p.timeout_ns) {
        watchdog_fire(p, rank, ch, op, -3, ef, v.y);
        ok = false;
        return make_uint2(0, 0);
      }
    }
  }
}

// plain 8 bytes (n valid, rest zero)
__device__ __forceinline__ uint2 ld_plain8(const char* a, int n, bool aligned) {
  if (n == 8 && aligned) {
    uint2 v;
    asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a) : "memory");
    return v;
  }
  uint32_t w[2] = {0, 0};
  for (int i = 0; i < n; ++i) w[i >> 2] |= uint32_t(*(const volatile uint8_t*)(a + i)) << (8 * (i & 3));
  return make_uint2(w[0], w[1]);
}
__device__ __forceinline__ void st_plain8(char* a, uint2 v, int n, bool aligned) {
  if (n == 8 && aligned) {
    asm volatile("st.volatile.global.v2.u32 [%0], {%1,%2};" ::"l"(a), "r"(v.x), "r"(v.y) : "memory");
    return;
  }
  const uint32_t w[2] = {v.x, v.y};
  for (int i = 0; i < n; ++i) *(volatile uint8_t*)(a + i) = uint8_t(w[i >> 2] >> (8 * (i & 3)));
}

template <int DT, bool SYS>
__global__ void __launch_bounds__(LL_NT) exec_ll_kernel(const __grid_constant__ KParams p) {
  const int tid = threadIdx.x;
  const int lr = fastdiv(blockIdx.x, p.nch_magic), ch = int(blockIdx.x) - lr * p.nch;
  const int cb = fastdiv(uint32_t(ch), p.kc_magic), cg = ch - cb * p.kc;  // (no divides in the prologue)
  const int rank = p.rank0 + lr;
  __shared__ uint64_t s_e;
  __shared__ uint64_t s_spar;  // scratch slot-set offset of this launch (epoch parity)
  __shared__ uint32_t s_entry_mask;
  __shared__ const char* s_inp[kMaxOpIn];
  __shared__ char* s_outp[kMaxOpOut];
  __shared__ uint8_t s_inll[kMaxOpIn], s_outll[kMaxOpOut];
  __shared__ uint32_t s_trace_n;
  __shared__ uint32_t s_ob, s_oe;
  __shared__ DevOp s_op[2];  // this op and the next one (prefetched while this one moves data)
  // Prologue round trips in parallel: the epoch (thread 0) and the program
  // range plus its first op (thread PF) -- they used to be three dependent
  // loads after the epoch.
  constexpr int PF = LL_NT - 32;  // the prefetching thread (not one of the descriptor threads below)
  if (tid == 0) {
    s_trace_n = 0;
    trace_ev(p, &s_trace_n, TR_START, 0, 0);
    s_e = p.epochs[blockIdx.x] + 1;
    s_spar = (s_e & 1) * p.ll_parity;
    s_entry_mask = 1u << rank;
    cta_abort = 0;
  }
  if (tid == PF) {
    const uint32_t b = p.prog[rank * p.kc + cg], en = p.prog[rank * p.kc + cg + 1];
    s_ob = b;
    s_oe = en;
    if (b < en) s_op[0] = p.ops[b];
  }
  __syncthreads();
  if (tid == 0) trace_ev(p, &s_trace_n, TR_FLAG, 0, 0);  // epoch known
  const uint64_t e = s_e;
  const uint32_t ef = uint32_t(e);
  // epoch-parity slot sets (one rank per GPU, plan.cpp ll_parity_safe):
  // launch e reads and writes scratch set e & 1 and skips the entry
  // handshake -- no flag stores at entry, no waits before the first store
  // (kept in shared memory, read where an address is formed: as a register
  // live across the op loop it cost the kernel 8-22 registers)
  auto sc = [&](int space) -> uint64_t {
    return space == SP_SCRATCH_IDX ? *reinterpret_cast<volatile uint64_t*>(&s_spar) : 0;
  };
  const bool handshake = p.multiprocess && !p.ll_parity;
  if (handshake)
    for (int t = tid; t < p.P; t += LL_NT)
      if (t != rank) {
        fence_rel<SYS>();
        st_relaxed<SYS>(reinterpret_cast<uint64_t*>(p.base[t][SP_FLAGS_IDX]) + p.entry_base + rank * p.nch + ch, e);
      }

  const uint32_t ob = s_ob, oe = s_oe;
  for (uint32_t oi = ob; oi < oe; ++oi) {
    __syncthreads();  // s_op[cur] (prefetched last iteration) visible; s_op[next] no longer read
    const DevOp op = s_op[(oi - ob) & 1];
    if (tid == PF && oi + 1 < oe) s_op[(oi + 1 - ob) & 1] = p.ops[oi + 1];
    if (op.kind == 2) {  // receipts nobody forwards: consume them
      for (int i = 0; i < op.nin; ++i) {
        const DevIn in = p.ins[op.in_begin + i];
        if (int(in.chunk % uint32_t(p.kc)) != cg) continue;
        const DPart q = dsplit16m(int64_t(in.len), p.kb, p.kb_magic, cb);
        const char* slot = p.base[in.rank][in.space] + sc(in.space) + in.off + 2 * q.off;
        const int64_t npair = (q.len + 7) / 8;
        bool ok = true;  // (a consumed receipt: nothing to publish either way)
        for (int64_t k = tid; k < npair; k += LL_NT)
          ll_read<SYS>(slot, k, q.len - 8 * k > 4, ef, p, rank, ch, int(oi - ob), ok);
      }
      continue;
    }
    if (int(op.chunk % uint32_t(p.kc)) != cg) continue;
    const DPart q = dsplit16m(int64_t(op.len), p.kb, p.kb_magic, cb);
    if (q.len == 0) continue;
    if (tid < op.nin) {
      const DevIn in = p.ins[op.in_begin + tid];
      s_inll[tid] = in.flag >= 0;
      s_inp[tid] = p.base[in.rank][in.space] + sc(in.space) + in.off + (in.flag >= 0 ? 2 * q.off : q.off);
    }
    if (tid >= 32 && tid < 32 + op.nout) {  // outputs on warp 1: loaded in parallel with the inputs
      const int o = tid - 32;
      const DevOut d = p.outs[op.out_begin + o];
      s_outll[o] = d.flag >= 0;
      s_outp[o] = p.base[d.rank][d.space] + sc(d.space) + d.off + (d.flag >= 0 ? 2 * q.off : q.off);
      if (handshake && d.rank != rank && !(atomicOr(&s_entry_mask, 0u) & (1u << d.rank))) {
        wait_ge<SYS>(reinterpret_cast<uint64_t*>(p.base[rank][SP_FLAGS_IDX]) + p.entry_base + d.rank * p.nch + ch, e,
                     p, rank, ch, int(oi - ob), -2);
        atomicOr(&s_entry_mask, 1u << d.rank);
      }
    }
    __syncthreads();
    if (tid == 0) trace_ev(p, &s_trace_n, TR_FULL, oi, 0);  // descriptors read
    const int64_t npair = (q.len + 7) / 8;
    for (int64_t k = tid; k < npair; k += LL_NT) {
      const int n = int(min(int64_t(8), q.len - 8 * k));
      const bool two = n > 4;
      bool ok = true;  // every input word of this element arrived (a read that gave up clears it)
      uint2 v = s_inll[0] ? ll_read<SYS>(s_inp[0], k, two, ef, p, rank, ch, int(oi - ob), ok)
                          : ld_plain8(s_inp[0] + 8 * k, n, op.vec);
      if (op.kind == 1) {
        Acc8<DT> acc;
        acc.init(v);
        for (int i = 1; i < op.nin; ++i)
          acc.add(s_inll[i] ? ll_read<SYS>(s_inp[i], k, two, ef, p, rank, ch, int(oi - ob), ok)
                            : ld_plain8(s_inp[i] + 8 * k, n, op.vec));
        v = acc.out();
      }
      // a read above gave up (watchdog / abort): publish nothing computed
      // from it (see watchdog_fire); values whose inputs all arrived are
      // correct and may still go out.  (A per-thread register, not the
      // CTA's shared abort word: no shared load per element.)
      if (!ok) continue;
      for (int o = 0; o < op.nout; ++o) {
        if (s_outll[o]) st_ll(s_outp[o] + 16 * k, v, ef);
        else st_plain8(s_outp[o] + 8 * k, v, n, op.vec);
      }
    }
    // (no barrier here: the next op's first barrier already keeps its
    // descriptor writes behind every thread's data loop of this op; the
    // debug trace wants the op's end, so it alone pays for one)
    if (p.trace) {
      __syncthreads();
      if (tid == 0) trace_ev(p, &s_trace_n, TR_DONE, oi, 0);  // op's data moved
    }
  }
  __syncthreads();
  if (tid == 0) {
    trace_ev(p, &s_trace_n, TR_END, 0, 0);
    p.epochs[blockIdx.x] = e;
  }
}

template <int DT>
const void* kernel_ptr(bool sys, bool ll) {
  if (ll)
    return sys ? reinterpret_cast<const void*>(exec_ll_kernel<DT, true>)
               : reinterpret_cast<const void*>(exec_ll_kernel<DT, false>);
  return sys ? reinterpret_cast<const void*>(exec_kernel<DT, true>) : reinterpret_cast<const void*>(exec_kernel<DT, false>);
}

const void* kernel_for(int dtype, bool sys, bool ll) {
  switch (dtype) {
    case 0: return kernel_ptr<0>(sys, ll);
    case 1: return kernel_ptr<1>(sys, ll);
    case 2: return kernel_ptr<2>(sys, ll);
    case 3: return kernel_ptr<3>(sys, ll);
    case 4: return kernel_ptr<4>(sys, ll);
  }
  return nullptr;
}

cudaError_t prepare(const void* f) {
  // once per kernel instantiation (10 of them; the driver call is not free)
  static const void* done[16] = {};
  for (auto& d : done)
    if (d == f) return cudaSuccess;
  cudaError_t err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_HDR + kStageBudget));
  if (err == cudaSuccess)
    for (auto& d : done)
      if (!d) {
        d = f;
        break;
      }
  return err;
}

}  // namespace

int exec_threads() { return NT; }

cudaError_t launch_exec(const KParams& p, int dtype, bool sys, cudaStream_t st) {
  const void* f = kernel_for(dtype, sys, p.ll != 0);
  if (!f) return cudaErrorInvalidValue;
  void* args[] = {const_cast<KParams*>(&p)};
  if (p.ll) return cudaLaunchKernel(f, dim3(p.nranks_launch * p.nch), dim3(LL_NT), args, 0, st);
  cudaError_t err = prepare(f);
  if (err != cudaSuccess) return err;
  return cudaLaunchKernel(f, dim3(p.nranks_launch * p.nch), dim3(NT), args, smem_bytes(p.tile, p.nstage), st);
}


cudaError_t exec_occupancy(int dtype, bool sys, int tile, int nstage, int* blocks_per_sm) {
  // tile == 0: the LL kernel (no dynamic shared memory)
  const void* f = kernel_for(dtype, sys, tile == 0);
  if (!f) return cudaErrorInvalidValue;
  if (tile == 0) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, LL_NT, 0);
  cudaError_t err = prepare(f);
  if (err != cudaSuccess) return err;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, NT, smem_bytes(tile, nstage));
}

}  // namespace sccl
