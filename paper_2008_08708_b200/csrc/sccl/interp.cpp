// TEST HOOK, not an execution path: a CPU interpreter of the lowered channel
// program (one std::thread per (rank, channel), std::atomic counters for the
// flags) used by the CPU test suite to check the LOWERING against the
// oracle without a GPU (SURVEY.md section 4, T0 "lowering interpreter").
// sccl_launch / sccl_launch_loopback never call it; the GPU path has no CPU
// fallback.  Declared in include/sccl_debug.h.
#include <atomic>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "../../../include/sccl_debug.h"
#include "../../../include/sccl_exec.h"
#include "error.hpp"
#include "plan.hpp"

namespace {

thread_local std::string g_ierr;

inline float bf16f(uint16_t h) {
  uint32_t u = uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline uint16_t f2bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fff;
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
inline float canon_nan_f32() {
  const uint32_t u = 0x7fffffffu;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

void elem_range(int dtype, const char* const* in, int nin, char* const* out, int nout, int64_t off, int64_t nbytes) {
  const int es = dtype == 0 ? 1 : (dtype == 3 || dtype == 4) ? 2 : 4;
  for (int64_t b = off; b < off + nbytes; b += es) {
    char tmp[4];
    if (nin == 1) {
      std::memcpy(tmp, in[0] + b, es);
    } else if (dtype == 0) {
      uint8_t a = uint8_t(in[0][b]);
      for (int k = 1; k < nin; ++k) a = uint8_t(a + uint8_t(in[k][b]));
      tmp[0] = char(a);
    } else if (dtype == 1) {
      uint32_t a, x;
      std::memcpy(&a, in[0] + b, 4);
      for (int k = 1; k < nin; ++k) {
        std::memcpy(&x, in[k] + b, 4);
        a += x;
      }
      std::memcpy(tmp, &a, 4);
    } else if (dtype == 2) {
      float a, x;
      std::memcpy(&a, in[0] + b, 4);
      for (int k = 1; k < nin; ++k) {
        std::memcpy(&x, in[k] + b, 4);
        a = a + x;
      }
      if (a != a) a = canon_nan_f32();  // canonical NaN (GPU arithmetic)
      std::memcpy(tmp, &a, 4);
    } else if (dtype == 3) {
      uint16_t h;
      std::memcpy(&h, in[0] + b, 2);
      float a = bf16f(h);
      for (int k = 1; k < nin; ++k) {
        std::memcpy(&h, in[k] + b, 2);
        a = a + bf16f(h);
      }
      h = f2bf16(a);
      std::memcpy(tmp, &h, 2);
    } else {
      _Float16 h;
      std::memcpy(&h, in[0] + b, 2);
      float a = float(h);
      for (int k = 1; k < nin; ++k) {
        std::memcpy(&h, in[k] + b, 2);
        a = a + float(h);
      }
      h = _Float16(a);
      uint16_t u;
      std::memcpy(&u, &h, 2);
      if (a != a) u = 0x7fff;  // canonical NaN (PTX cvt)
      std::memcpy(tmp, &u, 2);
    }
    for (int o = 0; o < nout; ++o) std::memcpy(out[o] + b, tmp, es);
  }
}

}  // namespace

extern "C" const char* sccl_debug_last_error(void) { return g_ierr.c_str(); }

extern "C" int sccl_debug_interpret_loopback(sccl_plan* p, const void* const* sendbufs, void* const* recvbufs,
                                             double timeout_s) {
  using namespace sccl;
  if (!p || !p->loopback) {
    g_ierr = "needs a loopback plan";
    return SCCL_INVALID_ARGUMENT;
  }
  const int P = p->nranks, nch = p->nch, kc = p->kc, kb = p->kb;
  const int64_t tile = p->tile;
  const size_t nflags = size_t(p->entry_base + P * nch);
  std::vector<std::vector<std::atomic<uint64_t>>> flags(P);
  std::vector<std::vector<char>> scratch(P);
  for (int r = 0; r < P; ++r) {
    flags[r] = std::vector<std::atomic<uint64_t>>(nflags);
    for (auto& f : flags[r]) f.store(0);
    scratch[r].assign(size_t(p->pg.scratch_bytes) + 16, 0);
  }
  auto base = [&](int rank, int space) -> char* {
    if (space == SP_SEND) return const_cast<char*>(static_cast<const char*>(sendbufs[rank]));
    if (space == SP_RECV) return static_cast<char*>(recvbufs[rank]);
    return scratch[rank].data();
  };
  std::atomic<int> failed{0};
  const uint64_t e = 1;
  auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  auto wait_ge = [&](std::atomic<uint64_t>& f, uint64_t target) -> uint64_t {
    uint64_t v;
    while ((v = f.load(std::memory_order_acquire)) < target) {
      if (failed.load()) return target;
      if (std::chrono::steady_clock::now() > deadline) {
        failed.store(1);
        return target;
      }
      std::this_thread::yield();
    }
    return v;
  };

  const uint32_t ef = uint32_t(e);
  // LL word pair k of a slot: two 8-byte words (data | flag << 32)
  auto ll_read = [&](const char* slot, int64_t k, bool two, char* out8) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(slot + 16 * k);
    uint64_t a, b = 0;
    for (;;) {
      a = __atomic_load_n(w, __ATOMIC_ACQUIRE);
      if (two) b = __atomic_load_n(w + 1, __ATOMIC_ACQUIRE);
      if (uint32_t(a >> 32) == ef && (!two || uint32_t(b >> 32) == ef)) break;
      if (failed.load()) return;
      if (std::chrono::steady_clock::now() > deadline) {
        failed.store(1);
        return;
      }
      std::this_thread::yield();
    }
    uint32_t d[2] = {uint32_t(a), uint32_t(b)};
    std::memcpy(out8, d, 8);
  };
  auto ll_write = [&](char* slot, int64_t k, const char* in8) {
    uint32_t d[2];
    std::memcpy(d, in8, 8);
    uint64_t* w = reinterpret_cast<uint64_t*>(slot + 16 * k);
    __atomic_store_n(w, uint64_t(d[0]) | (uint64_t(ef) << 32), __ATOMIC_RELEASE);
    __atomic_store_n(w + 1, uint64_t(d[1]) | (uint64_t(ef) << 32), __ATOMIC_RELEASE);
  };

  auto run = [&](int rank, int ch) {
    const int cg = ch % kc, cb = ch / kc;  // same channel map as the kernel
    for (uint32_t oi = p->prog[size_t(rank) * kc + cg]; oi < p->prog[size_t(rank) * kc + cg + 1]; ++oi) {
      const DevOp& op = p->ops[oi];
      if (op.kind == OP_WAIT) {
        for (int i = 0; i < op.nin; ++i) {
          const DevIn& in = p->ins[op.in_begin + i];
          if (int(in.chunk % uint32_t(kc)) != cg) continue;
          Part q = split16(int64_t(in.len), kb, cb);
          if (p->ll) {
            char tmp[8];
            for (int64_t k = 0; k < (q.len + 7) / 8; ++k)
              ll_read(base(in.rank, in.space) + in.off + 2 * q.off, k, q.len - 8 * k > 4, tmp);
          } else if (q.len) {
            wait_ge(flags[rank][size_t(in.flag) * nch + ch], e * uint64_t(q.len));
          }
        }
        continue;
      }
      if (int(op.chunk % uint32_t(kc)) != cg) continue;
      Part q = split16(int64_t(op.len), kb, cb);
      if (q.len == 0) continue;
      std::vector<const char*> inp(op.nin);
      std::vector<char*> outp(op.nout);
      for (int i = 0; i < op.nin; ++i) {
        const DevIn& in = p->ins[op.in_begin + i];
        inp[i] = base(in.rank, in.space) + in.off + (p->ll && in.flag >= 0 ? 2 * q.off : q.off);
      }
      for (int o = 0; o < op.nout; ++o) {
        const DevOut& out = p->outs[op.out_begin + o];
        outp[o] = base(out.rank, out.space) + out.off + (p->ll && out.flag >= 0 ? 2 * q.off : q.off);
      }
      if (p->ll) {  // LL: 8 data bytes at a time, flags in the data
        const int dt = op.kind == OP_COPY ? 0 : p->dtype;
        const int nin = op.kind == OP_COPY ? 1 : op.nin;
        std::vector<char> ibuf(8 * size_t(nin));
        std::vector<const char*> ip(nin);
        char obuf[8];
        char* op8[1] = {obuf};
        for (int64_t k = 0; k < (q.len + 7) / 8; ++k) {
          const int n = int(std::min<int64_t>(8, q.len - 8 * k));
          for (int i = 0; i < nin; ++i) {
            char* b8 = ibuf.data() + 8 * i;
            std::memset(b8, 0, 8);
            if (p->ins[op.in_begin + i].flag >= 0) ll_read(inp[i], k, n > 4, b8);
            else std::memcpy(b8, inp[i] + 8 * k, n);
            ip[i] = b8;
          }
          if (failed.load()) return;
          elem_range(dt, ip.data(), nin, op8, 1, 0, 8);
          for (int o = 0; o < op.nout; ++o) {
            if (p->outs[op.out_begin + o].flag >= 0) ll_write(outp[o], k, obuf);
            else std::memcpy(outp[o] + 8 * k, obuf, n);
          }
        }
        continue;
      }
      // same tiling rule as the kernel: copy tiles of `tile`, reduce tiles
      // of tile/nin; counters count bytes so the two sides may differ
      const int64_t T = op.kind == OP_COPY ? tile : std::max<int64_t>(16, (tile / op.nin) & ~int64_t(15));
      const int64_t ntiles = (q.len + T - 1) / T;
      const uint64_t b0 = (e - 1) * uint64_t(q.len);
      for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t lo = t * T, nb = std::min<int64_t>(T, q.len - lo);
        for (int i = 0; i < op.nin; ++i) {
          const DevIn& in = p->ins[op.in_begin + i];
          if (in.flag >= 0) wait_ge(flags[rank][size_t(in.flag) * nch + ch], b0 + uint64_t(lo + nb));
        }
        if (failed.load()) return;
        elem_range(op.kind == OP_COPY ? 0 : p->dtype, inp.data(), op.kind == OP_COPY ? 1 : op.nin, outp.data(),
                   op.nout, lo, nb);
        bool last = t + 1 == ntiles;
        for (int o = 0; o < op.nout; ++o) {
          const DevOut& out = p->outs[op.out_begin + o];
          if (out.flag >= 0 && (last || out.every_tile))
            flags[out.rank][size_t(out.flag) * nch + ch].store(b0 + uint64_t(lo + nb), std::memory_order_release);
        }
      }
    }
  };
  std::vector<std::thread> th;
  for (int r = 0; r < P; ++r)
    for (int c = 0; c < nch; ++c) th.emplace_back(run, r, c);
  for (auto& t : th) t.join();
  if (failed.load()) {
    g_ierr = "interpreter: a wait never completed (deadlock or missing signal)";
    return SCCL_PEER_TIMEOUT;
  }
  return SCCL_OK;
}

extern "C" int sccl_debug_set_trace(sccl_plan* p, void* buf, int records_per_cta) {
  if (!p || (buf && records_per_cta <= 0)) {
    g_ierr = "bad trace arguments";
    return SCCL_INVALID_ARGUMENT;
  }
  p->d_trace = static_cast<uint64_t*>(buf);
  p->trace_cap = buf ? records_per_cta : 0;
  return SCCL_OK;
}
