// Plans and the C-ABI (include/sccl_exec.h).
#include "plan.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "../../../include/sccl_exec.h"
#include "error.hpp"
#include "layout.hpp"
#include "abi.hpp"
#include "driver.hpp"
#include "policy.hpp"

namespace sccl {
cudaError_t launch_exec(const KParams& p, int dtype, bool sys, cudaStream_t st);
cudaError_t exec_occupancy(int dtype, bool sys, int tile, int nstage, int* blocks_per_sm);
int exec_threads();
}  // namespace sccl

using sccl::cu_check;
using sccl::Vmm;
using sccl::vmm_api;
using sccl::vmm_map;

using sccl::cuda_check;
using sccl::g_err;
using sccl::guarded;

namespace {

void put_string(const std::string& s, char* out, size_t* len) {
  if (!len) throw sccl::invalid_argument_error("len must not be NULL");
  size_t need = s.size() + 1;
  if (out && *len >= need) std::memcpy(out, s.c_str(), need);
  else if (out) {
    *len = need;
    throw sccl::invalid_argument_error("output buffer too small");
  }
  *len = need;
}

int esize_of(int dtype) {
  switch (dtype) {
    case SCCL_U8: return 1;
    case SCCL_I32: return 4;
    case SCCL_F32: return 4;
    case SCCL_BF16: return 2;
    case SCCL_F16: return 2;
  }
  throw sccl::invalid_argument_error("unknown dtype");
}

bool loopback_sys() {  // SCCL_LOOPBACK_SYS=1: loopback launches use system scope (measurement only)
  static const bool v = [] {
    const char* e = std::getenv("SCCL_LOOPBACK_SYS");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

// The policy table whose protocol constants price a plan: system-scope
// signalling (multi-process, or loopback under SCCL_LOOPBACK_SYS) makes every
// bulk-protocol step dearer.
const sccl::ModePolicy& signal_policy(bool loopback) { return sccl::mode_policy(loopback && !loopback_sys()); }

// predicted time (us) of a lowered program, see plan_build_host
double predict_us(const sccl::Program& pg, int steps, bool ll, const sccl::ModePolicy& pol) {
  double mb = 0;
  for (auto& rp : pg.ranks)
    for (auto& op : rp.ops)
      if (op.kind != sccl::OP_WAIT) mb += double(op.len) * double(op.ins.size() + op.outs.size());
  mb /= 1e6;
  if (ll) return pol.ll_c + pol.ll_alpha * steps + pol.ll_beta * mb;
  return pol.simple_c + pol.simple_alpha * steps + pol.simple_beta * mb;
}

struct IpcBlob {
  char magic[8];
  char fingerprint[24];
  int32_t rank, nranks, nch, kc, kb, tile;
  int32_t dtype, redop;  // the program fingerprint covers the element size, not the format
  int32_t ll_parity, pad;  // LL slot sets by launch parity (no entry handshake): every rank or none
  uint64_t region_bytes;
  cudaIpcMemHandle_t handle;
};

// A caller buffer registered as a multi-process plan's receive target: the
// CUDA IPC handle of the allocation that holds it plus the offset inside.
struct RegBlob {
  char magic[8];
  int32_t rank, pad;
  uint64_t bytes, offset;
  cudaIpcMemHandle_t handle;
};

}  // namespace

namespace sccl {

namespace {

// Facts about a lowered program the plan policies below are decided from.
struct ProgramStats {
  int steps = 0;            // schedule steps, all phases
  int max_fanin = 1;        // widest REDUCE
  double bytes = 0;         // reads + writes of the lowered ops (this rank's share when multi-process)
  bool rereads = false;     // some op reads a receipt (a relay or a reduction)
  bool reduces = false;
  size_t nops_rank0 = 0;    // rank 0's non-WAIT ops
  int work_chunks = 0;      // most distinct chunks any one rank has non-WAIT ops on
};

ProgramStats program_stats(const Schedule& sched, const Program& pg, bool loopback) {
  ProgramStats st;
  for (auto* ph : sched.flat()) st.steps += ph->S;
  for (size_t r = 0; r < pg.ranks.size(); ++r) {
    std::vector<int> chunks;
    for (auto& op : pg.ranks[r].ops)
      if (op.kind != OP_WAIT) chunks.push_back(op.chunk);
    std::sort(chunks.begin(), chunks.end());
    st.work_chunks = std::max(st.work_chunks, int(std::unique(chunks.begin(), chunks.end()) - chunks.begin()));
  }
  for (size_t r = 0; r < pg.ranks.size(); ++r)
    for (auto& op : pg.ranks[r].ops) {
      if (op.kind == OP_WAIT) continue;
      st.bytes += double(op.len) * double(op.ins.size() + op.outs.size());
      if (op.kind == OP_REDUCE) {
        st.reduces = true;
        st.max_fanin = std::max(st.max_fanin, int(op.ins.size()));
      }
      for (auto& in : op.ins) st.rereads |= in.flag >= 0;
      if (r == 0) ++st.nops_rank0;
    }
  if (!loopback) st.bytes /= double(sched.P);
  return st;
}

// A launch streams when its program moves > ModePolicy::stream_bytes (1 GB):
// past the 126 MB L2, the window-major order, L2 hints, receipt discards and
// the stage choice for streaming reductions pay; below it the data stays
// L2-resident.

// Protocol (auto): lower both ways and take the smaller predicted time
// t = c + alpha*S + beta*MB (S = schedule steps, MB = bytes the lowered
// program reads + writes).  Constants: a relative-error least-squares fit
// to the B200 loopback crossover sweep (tools/gpu_runs/r01/proto_round1i.sh:
// 7 schedules x 16 KiB-16 MiB x both protocols; mean regret vs the
// per-point best 1.9 %); system scope uses its own fit.
bool choose_ll(sccl_plan& p, int64_t bytes, int es, int protocol, bool loopback, bool pull) {
  if (protocol < 0 || protocol > 2) throw invalid_argument_error("protocol must be 0 (auto), 1 (simple), 2 (ll)");
  if (protocol != 0) {
    p.pg = lower(p.sched, bytes, es, protocol == 2, pull);
    return protocol == 2;
  }
  int steps = 0;
  for (auto* ph : p.sched.flat()) steps += ph->S;
  Program a = lower(p.sched, bytes, es, true, pull), b = lower(p.sched, bytes, es, false, pull);
  const ModePolicy& pol = signal_policy(loopback);
  const bool ll = predict_us(a, steps, true, pol) < predict_us(b, steps, false, pol);
  p.pg = ll ? std::move(a) : std::move(b);
  return ll;
}

// Epoch-parity LL slots (one rank per GPU).  The entry handshake exists so
// that a sender in launch e never overwrites a receiver's slot before the
// receiver has read that slot's launch e-1 word.  With two slot sets, launch
// e writing set e & 1, the hazard moves to set reuse two launches apart:
// sender S in launch e needs receiver R past launch e-2.  S starting launch
// e means S finished e-1, i.e. every receipt of its launch e-1 landed; if
// one of those receipts had to wait for R's own launch e-1 to run (R's data
// reached S through a chain of sends, each reading the value its sender
// held at that step), then R had entered e-1 and so finished e-2 (launches
// of a plan are stream-ordered on every rank).  The condition, checked for
// every cross-rank send S -> R of the flattened schedule: R is in S's
// completion set.  Holds for allgather, alltoall, reduce-scatter and
// allreduce (every output depends on every rank); fails for rooted kinds
// (a broadcast root depends on nobody), which keep the handshake.  Only LL:
// its receipts are scratch slots the receiver unpacks itself, while the
// simple protocol stores final values into the peer's receive buffer, whose
// previous contents the peer's stream may still be reading.
bool ll_parity_safe(const Schedule& s) {
  const int P = s.P;
  const auto phases = s.flat();
  int G = 0;
  for (auto* ph : phases) G = std::max(G, ph->G);
  std::vector<uint32_t> dep(size_t(G) * P, 0);  // ranks the value of chunk c at node n waited for
  std::vector<uint32_t> done(P, 0);             // ranks node n's launch completion waits for
  for (auto* ph : phases)
    for (int st = 0; st < ph->S; ++st) {
      std::vector<uint32_t> nd = dep;  // sends at step st read the values at its start
      for (const Send& t : ph->sends)
        if (t.step == st) {
          const uint32_t m = dep[size_t(t.chunk) * P + t.src] | (1u << t.src);
          nd[size_t(t.chunk) * P + t.dst] |= m;
          done[t.dst] |= m;
        }
      dep.swap(nd);
    }
  for (auto* ph : phases)
    for (const Send& t : ph->sends)
      if (!((done[t.src] >> t.dst) & 1u)) return false;
  return true;
}

// Stage (= copy tile) size and pipeline depth.  Streaming copies and
// 2-input reductions: 3 x 32 KiB at 2 CTAs/SM.  Wide reductions (fan-in
// >= 4) that fit L2: 3 x 64 KiB at 1 CTA/SM (8 KiB per input at fan-in 8);
// streaming ones run window-major with receipt discards and do better at
// 2 CTAs/SM with 3 x 32 KiB (AR (8,2,2) 64 MiB 298 -> 280 us, 256 MiB
// 1109 -> 1081 us); with chunks up to 256 KiB they use 16 KiB tiles.
// Small chunks: the smallest power of two that holds one.  Stages come in
// multiples of the storer-warp count (each storer warp owns the stages s
// with s % kStorerWarps == its index): 3 or 6.
void choose_stages(sccl_plan& p, const ProgramStats& st, int64_t maxlen, const ChannelRequest& req,
                   const ModePolicy& pol) {
  const bool wide = st.max_fanin >= 4 && !(st.bytes > pol.stream_bytes && !p.ll);
  int tile = req.tile;
  if (tile <= 0) {
    // wide reductions with small chunks: 16 KiB tiles (6 stages, 2 CTAs/SM)
    // put twice the CTAs on the chunks (AR (8,2,2) 512 KiB-2 MiB per rank:
    // -13..-26 %, tools/gpu_runs/r01/midtile2_round1w.sh)
    tile = wide ? (maxlen <= (256 << 10) ? 16384 : kMaxTile) : 32768;
    // pull-lowered ones (the loopback one-shot allreduce: one fan-in-P op
    // per rank, nothing re-read) keep 16 KiB tiles up to 512 KiB chunks and
    // again from 250 MB of program traffic to the streaming threshold: AR
    // (8,2,2) bf16 at 4 / 16 / 32 / 48 MiB per rank 19.7 / 54.0 / 101.5 /
    // 148.5 -> 15.3 / 53.3 / 95.9 / 138.2 us; 8 and 12 MiB keep 64 KiB
    // (27.0 vs 31.6, 41.0 vs 42.4 us) (tools/gpu_runs/r02/s2_ar822_tile.sh)
    // Re-measured with the session-3 kernels (cheaper per-tile path, two
    // vectors in flight in the wide reduce loop): up to 512 KiB chunks 32
    // KiB tiles now beat 16 KiB, AR (8,2,2) bf16 at 512 KiB / 1 / 4 MiB per
    // rank 9.16 / 10.24 / 14.41 -> 8.39 / 9.28 / 13.89 us, 2 MiB even
    // (profiles/r02/s3_ar822_mid.jsonl); the streaming range keeps 16 KiB.
    if (wide && p.pg.pull && st.reduces && !st.rereads && maxlen <= (512 << 10)) tile = 32768;
    else if (wide && p.pg.pull && st.reduces && !st.rereads && st.bytes >= 250e6) tile = 16384;
    // one-shot copies (one fan-out op per rank, nothing re-read) up to
    // 512 KiB: two 16 KiB tiles per CTA overlap the load of one with the
    // stores of the other (AG (1,1,1) 256 / 512 KiB: -27 / -16 %)
    if (!st.rereads && !st.reduces && st.nops_rank0 <= 2 && maxlen <= (512 << 10)) tile = 16384;
    if (maxlen < tile) {
      tile = 1024;
      while (tile < maxlen) tile *= 2;
    }
  }
  if (tile % 16 || tile > kMaxTile || tile < 256)
    throw invalid_argument_error("tile_bytes must be a multiple of 16 in [256, 65536]");
  // SCCL_STAGE_BUDGET (bytes of stages per CTA) trades depth for CTAs per SM
  int budget = wide ? kStageBudget : kStageBudget / 2;
  if (const char* env = std::getenv("SCCL_STAGE_BUDGET")) budget = std::max(2 * 256, std::min(kStageBudget, std::atoi(env)));
  if (req.stage_budget > 0) budget = std::min(kStageBudget, req.stage_budget);
  p.tile = tile;
  p.nstage = budget / tile >= 2 * kStorerWarps ? 2 * kStorerWarps : kStorerWarps;
}

// Channels: channel j = (chunk group j % kc, byte part j / kc).  Large
// chunks are cut into byte parts so every SM streams (one stage per part:
// fewer, longer parts lost more to idle SMs than they gained in
// pipelining); small chunks are spread over chunk groups so independent
// chunks travel in parallel instead of queueing in one CTA.  With
// ModePolicy::group_split (off in both default tables since round 2.1) a
// streaming, copy-only relay schedule with >= 4 ops per step splits into
// two chunk groups, so a CTA's window holds fewer ops per step: round 1's
// (7,7,7) at 128 MiB/rank went 1979 -> 1869 us with it; the round-2
// pipeline runs one group faster (1752 -> 1730 us; policy.cpp).
void choose_channels(sccl_plan& p, const ProgramStats& st, int64_t maxlen, const ChannelRequest& req, bool loopback,
                     const ModePolicy& pol) {
  const int bps = req.blocks_per_sm ? req.blocks_per_sm(req.ctx, p.ll ? 0 : p.tile, p.nstage)
                  : p.ll ? 2048 / kLLThreads
                         : std::max(1, std::min(2, int((227 << 10) / (p.nstage * p.tile + kSmemHdr))));
  const int resident = std::max(1, req.sms * std::max(1, bps));
  // pull-lowered wide reductions (every input read in place, no receipt
  // re-read): each CTA streams nin reads and nout writes, and one CTA per SM
  // keeps DRAM busiest (AR (8,2,2) bf16 at 64 MiB/rank: 144 CTAs 182 us,
  // 192: 199, 296: 190, 96: 232; 256 MiB: 714 / 769 / -- / 893 us;
  // tools/gpu_runs/r02/abort_reg.sh)
  const bool pull_stream = loopback && !p.ll && p.pg.pull && st.reduces && !st.rereads && st.max_fanin >= 4 &&
                           st.bytes >= pol.stream_bytes / 8;  // (small launches are latency-bound: more CTAs)
  const int cap = pol.max_ctas_per_rank > 0 ? pol.max_ctas_per_rank
                                            : std::max(1, (pull_stream ? req.sms : resident) / p.sched.P);
  const int64_t part = p.ll ? kLLPart : p.tile;
  int kb, kc;
  if (req.nchannels > 0) {
    kb = req.nchannels;
    kc = req.chunk_groups > 0 ? req.chunk_groups : 1;
  } else {
    kb = int(std::max<int64_t>(1, std::min<int64_t>(cap, (maxlen + part - 1) / part)));
    kc = req.chunk_groups > 0 ? req.chunk_groups : std::max(1, std::min(p.pg.G, cap / kb));
    // simple protocol: receipts land in place (only LL unpacks them in an op
    // of the receiver), so a rank has work in as many chunk groups as it has
    // chunks with data ops -- one for one-shot copies and pulled one-shot
    // reductions.  Groups past that only wait; give their CTAs to byte parts
    // instead, down to 8 KiB per CTA: AG (1,1,1) at 64 KiB per rank 9.9 ->
    // 7.1 us (8 x 4 -> 1 x 8 CTAs per rank; tools/gpu_runs/r02/s2_ll_audit.sh)
    if (!p.ll && req.chunk_groups <= 0 && st.work_chunks >= 1 && kc > st.work_chunks) {
      kc = st.work_chunks;
      while (2 * kc * kb <= cap && maxlen / (2 * kb) >= (8 << 10)) kb *= 2;
    }
    if (req.chunk_groups <= 0 && kc == 1 && kb >= 4 && !p.ll && pol.group_split && st.bytes > 4 * pol.stream_bytes &&
        st.rereads &&
        !st.reduces && double(st.nops_rank0) >= 4.0 * st.steps) {
      kc = 2;
      kb /= 2;
    }
    // LL: cap / kb rounding down can leave CTA slots idle (ring AG at
    // 256 KiB: 1 x 64 of 111 per rank); take the chunk-group count that
    // fills the most slots (fewest groups on ties) when that is 25 % more:
    // ring / one-shot AG 256 KiB -22 / -9 % (tools/gpu_runs/r01/llgrid4_round1w.sh)
    if (p.ll && req.chunk_groups <= 0 && 4 * kc * kb < 3 * cap) {
      int bc = kc, bb = kb;
      for (int c = kc + 1; c <= std::min(p.pg.G, cap); ++c) {
        const int b = std::min(kb, cap / c);
        if (c * b > bc * bb) bc = c, bb = b;
      }
      if (4 * bc * bb >= 5 * kc * kb) kc = bc, kb = bb;
    }
    // LL relay / reduce chains (>= 4 steps) with many chunks (>= 32) of up
    // to 40 KiB: one chunk per CTA (kc = G, kb = 1) instead of byte parts of
    // several chunks, so each CTA forwards one chunk down its chain without
    // queueing behind the others' hops: (7,7,7) 64-256 KiB -24..-31 %,
    // (56,14,14) 256 KiB-2 MiB -6..-32 % (tools/gpu_runs/r01/llgrid2_round1w.sh;
    // at 75 KiB chunks the byte parts win again)
    if (p.ll && req.chunk_groups <= 0 && st.rereads && st.steps >= 4 && p.pg.G >= 32 && p.pg.G <= cap &&
        maxlen <= (40 << 10)) {
      kc = p.pg.G;
      kb = 1;
    }
    // LL plans whose chunk groups are exhausted (kc = G) but leave CTAs
    // idle: split the chunks further, down to 2 KiB per CTA, up to 64 CTAs
    // per rank (a larger LL grid lost: (7,7,7) 16 KiB with 896 CTAs +29 %).
    // AR (8,2,2) 64 / 128 KiB -28 / -26 %, one-shot AG 4-16 KiB -14..-16 %
    // (tools/gpu_runs/r01/llpart_round1w.sh, llgrow_round1w.sh).
    if (p.ll && req.chunk_groups <= 0) {
      const int grid_cap = loopback ? std::min(cap, 512 / std::max(1, p.sched.P)) : cap;
      while (2 * kc * kb <= grid_cap && maxlen / (2 * kb) >= 2048) kb *= 2;
    }
  }
  if (kc < 1 || kb < 1) throw invalid_argument_error("channels must be positive");
  p.kc = kc;
  p.kb = kb;
  p.nch = kc * kb;
  p.resident_cap = loopback ? resident : 0;
}

// Chunk groups: every rank's CTA (rank, channel) runs the ops of the chunks
// in its group, and a chunk's group must be the same at every rank (its
// receipt counters are per channel).  `chunk % kc` put all of a rank's
// alltoall chunks (ids i*P + rank) into one group whenever kc divided P;
// such plans assign chunks greedily, largest first, to the group that keeps
// the busiest (rank, group) lightest (A2A 4 MiB per rank: 17.7 -> 12.8 us).
// The modulo map stays unless it loads some (rank, group) 25 % above the
// mean and the greedy map is 3 % better: the (7,7,7) allgather at 128 MiB
// (modulo 1.09x the mean, greedy 1.03x) ran 1.3 % slower greedy -- it is
// HBM-bound, and the modulo order is the one its L2 reuse was tuned on
// (tools/gpu_runs/r01/groups_ab_round1w.sh, groups2_ab_round1w.sh).
void assign_groups(sccl_plan& p) {
  const int P = int(p.pg.ranks.size());
  int maxc = 0;
  for (auto& rp : p.pg.ranks)
    for (auto& op : rp.ops) {
      maxc = std::max(maxc, op.chunk);
      for (auto& in : op.ins) maxc = std::max(maxc, in.chunk);
    }
  p.group_of.assign(size_t(maxc) + 1, 0);
  for (int c = 0; c <= maxc; ++c) p.group_of[size_t(c)] = c % p.kc;
  if (p.kc == 1) return;
  std::vector<double> w(size_t(maxc + 1) * P, 0.0);  // [chunk][rank] bytes moved
  for (int r = 0; r < P; ++r)
    for (auto& op : p.pg.ranks[size_t(r)].ops)
      if (op.kind != OP_WAIT)
        w[size_t(std::max(0, op.chunk)) * P + r] += double(op.len) * double(op.ins.size() + op.outs.size());
  std::vector<int> order(size_t(maxc) + 1);
  for (int c = 0; c <= maxc; ++c) order[size_t(c)] = c;
  auto peak = [&](int c) { return *std::max_element(w.begin() + size_t(c) * P, w.begin() + size_t(c + 1) * P); };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return peak(a) > peak(b); });
  std::vector<double> load(size_t(p.kc) * P, 0.0);  // [group][rank]
  for (int c = 0; c <= maxc; ++c)
    for (int r = 0; r < P; ++r) load[size_t(c % p.kc) * P + r] += w[size_t(c) * P + r];
  const double modulo_max = *std::max_element(load.begin(), load.end());
  std::fill(load.begin(), load.end(), 0.0);
  std::vector<int> greedy(p.group_of);
  for (int c : order) {
    if (peak(c) <= 0) continue;  // no work (WAIT-only chunk ids keep c % kc)
    int best = 0;
    double best_max = 0, best_sum = 0;
    for (int g = 0; g < p.kc; ++g) {
      double mx = 0, sum = 0;
      for (int r = 0; r < P; ++r) {
        mx = std::max(mx, load[size_t(g) * P + r] + w[size_t(c) * P + r]);
        sum += load[size_t(g) * P + r];
      }
      if (g == 0 || mx < best_max || (mx == best_max && sum < best_sum)) best = g, best_max = mx, best_sum = sum;
    }
    greedy[size_t(c)] = best;
    for (int r = 0; r < P; ++r) load[size_t(best) * P + r] += w[size_t(c) * P + r];
  }
  double total = 0;
  for (double x : w) total += x;
  const double mean = total / double(size_t(p.kc) * P);
  p.groups_balanced = modulo_max > 1.25 * mean && *std::max_element(load.begin(), load.end()) < 0.97 * modulo_max;
  if (p.groups_balanced) p.group_of = std::move(greedy);
}

int group_of(const sccl_plan& p, int chunk) {
  const int c = std::max(0, chunk);
  return size_t(c) < p.group_of.size() ? p.group_of[size_t(c)] : c % p.kc;
}

// Counter release: latency-bound plans (<= 16 tiles per CTA) let each
// storer warp release its own tile's counters (no hand-off, ~0.3 us less
// per hop); longer ones keep the fence off the store path in the signaler
// warp, batched across ops (tools/gpu_runs/r01/winsig_round1h.sh).  System scope
// makes the fence on the store path ~3x dearer, so only very short plans
// self-publish there (<= 4 tiles; tools/gpu_runs/r01/sys_pub_round1n.sh).
void choose_release(sccl_plan& p, bool loopback) {
  const ModePolicy& pol = signal_policy(loopback);
  int64_t max_tiles = 0;
  for (auto& rp : p.pg.ranks)
    for (int g = 0; g < p.kc; ++g) {
      int64_t n = 0;
      for (auto& op : rp.ops) {
        if (op.kind == OP_WAIT || group_of(p, op.chunk) != g) continue;
        const int64_t part = split16(op.len, p.kb, p.kb - 1).len;  // the last part is the longest
        const int64_t T = op.kind == OP_COPY ? p.tile : std::max<int64_t>(16, (p.tile / int64_t(op.ins.size())) & ~int64_t(15));
        n += (part + T - 1) / T;
      }
      max_tiles = std::max(max_tiles, n);
    }
  p.selfpub = max_tiles <= pol.selfpub_max_tiles;
  if (const char* env = std::getenv("SCCL_SELFPUB")) p.selfpub = std::atoi(env) != 0;
}

// Device encoding: one op list per (rank, chunk group) -- a CTA walks only
// its own ops (ops of different chunks never depend on each other within a
// rank); end-of-program waits are split by chunk group the same way.  A
// scratch receipt with one reader is marked dead_after (the kernel may drop
// it from L2 once that reader has loaded it).
void encode_program(sccl_plan& p) {
  const int P = p.sched.P;
  p.ops.clear();
  p.ins.clear();
  p.outs.clear();
  p.prog.assign(size_t(P) * p.kc + 1, 0);
  std::vector<std::vector<int>> readers(P);
  for (int r = 0; r < P; ++r) {
    readers[r].assign(size_t(std::max(1, p.pg.ranks[r].nslots)), 0);
    for (const Op& op : p.pg.ranks[r].ops)
      if (op.kind != OP_WAIT)
        for (auto& in : op.ins)
          if (in.flag >= 0 && in.flag < int(readers[r].size())) ++readers[r][size_t(in.flag)];
  }
  auto encode = [&](int r, const Op& op, const std::vector<OpIn>& ins) {
    if (op.kind != OP_WAIT && (ins.size() > size_t(kMaxOpIn) || op.outs.size() > size_t(kMaxOpOut)))
      throw invalid_argument_error("op fan-in/fan-out exceeds executor limits (32)");
    DevOp d{};
    d.len = uint64_t(op.len);
    d.chunk = uint32_t(group_of(p, op.chunk));  // the kernel only needs chunk % kc
    d.kind = uint8_t(op.kind);
    d.in_begin = uint32_t(p.ins.size());
    d.out_begin = uint32_t(p.outs.size());
    d.nin = uint16_t(ins.size());
    d.nout = uint16_t(op.outs.size());
    // the kernel's tile of this op (exec_kernel.cu: copies move a whole
    // stage, reductions stage / fan-in rounded down to 16 bytes)
    d.tile = op.kind == OP_COPY ? uint32_t(p.tile) : std::max(16u, uint32_t(p.tile / std::max<size_t>(1, ins.size())) & ~15u);
    bool vec = true;
    for (auto& in : ins) {
      // remote reads only of untouched SEND buffers, and only in pull mode
      if (in.loc.rank != r && !(p.pg.pull && in.loc.space == SP_SEND && in.flag < 0))
        throw invalid_argument_error("internal: op reads remote memory");
      DevIn x{};
      x.off = uint64_t(in.loc.off);
      x.len = uint64_t(in.len);
      x.flag = in.flag;
      x.chunk = uint32_t(group_of(p, in.chunk));
      x.rank = uint8_t(in.loc.rank);
      x.space = uint8_t(in.loc.space);
      x.dead_after = op.kind != OP_WAIT && in.flag >= 0 && in.loc.space == SP_SCRATCH &&
                     in.flag < int(readers[r].size()) && readers[r][size_t(in.flag)] == 1;
      vec &= in.loc.off % 16 == 0;
      if (in.flag < 0 && in.loc.space != SP_SEND) d.raw = 1;
      p.ins.push_back(x);
    }
    for (auto& o : op.outs) {
      DevOut x{};
      x.off = uint64_t(o.loc.off);
      x.flag = o.flag;
      x.rank = uint8_t(o.loc.rank);
      x.space = uint8_t(o.loc.space);
      x.every_tile = o.every_tile ? 1 : 0;
      vec &= o.loc.off % 16 == 0;
      p.outs.push_back(x);
    }
    d.vec = vec ? 1 : 0;
    p.ops.push_back(d);
  };
  for (int r = 0; r < P; ++r)
    for (int cg = 0; cg < p.kc; ++cg) {
      p.prog[size_t(r) * p.kc + cg] = uint32_t(p.ops.size());
      for (const Op& op : p.pg.ranks[r].ops) {
        if (op.kind == OP_WAIT) {
          std::vector<OpIn> mine;
          for (auto& in : op.ins)
            if (group_of(p, in.chunk) == cg) mine.push_back(in);
          if (!mine.empty()) encode(r, op, mine);
        } else if (group_of(p, op.chunk) == cg) {
          encode(r, op, op.ins);
        }
      }
    }
  p.prog[size_t(P) * p.kc] = uint32_t(p.ops.size());
  // per (rank, chunk group): its contiguous op / in / out descriptor ranges
  // (the simple kernel copies them into shared memory in its prologue)
  p.dtab.assign(size_t(P) * p.kc * 8, 0);
  for (size_t g = 0; g < size_t(P) * p.kc; ++g) {
    const uint32_t b = p.prog[g], e = p.prog[g + 1];
    uint32_t* t = &p.dtab[g * 8];
    t[0] = b, t[1] = e;
    t[2] = b < e ? p.ops[b].in_begin : 0, t[3] = b < e ? p.ops[e - 1].in_begin + p.ops[e - 1].nin : 0;
    t[4] = b < e ? p.ops[b].out_begin : 0, t[5] = b < e ? p.ops[e - 1].out_begin + p.ops[e - 1].nout : 0;
    bool idle = true;  // t[6]: the compute warps have nothing to do (no REDUCE, no unaligned op)
    for (uint32_t o = b; o < e; ++o) idle &= p.ops[o].kind == OP_WAIT || (p.ops[o].kind == OP_COPY && p.ops[o].vec);
    t[6] = idle ? 1 : 0;
  }
}

// Streaming policies (launches over ModePolicy::stream_bytes; loopback table only):
//  * window-major (simple protocol, every op 16-byte aligned, some op
//    re-reads a receipt): a CTA moves one byte window of each op, in
//    program order, before the next window, so relayed and reduced receipts
//    are read back while still in L2.  One tile when a CTA has several ops
//    per step (the other ops of the step cover the hop latency), up to 4
//    tiles when it has one (a ring) (tools/gpu_runs/r01/window_round1r.sh,
//    window2_round1s.sh).  Schedules that never re-read a receipt (one-shot,
//    direct alltoall) stay op-major: the per-window descriptor reloads
//    would only cost.  Below stream_bytes: AR at 16 MiB/rank was 3-5 %
//    slower with windows and hints.
//  * L2 hints: single-use loads and stores evict-first
//    (tools/gpu_runs/r01/l2hint_round1t.sh).  Receipts a later op re-reads are
//    stored with the default policy: evict-last cost 1.5-3 % on relays and
//    reduce chains (AG (7,7,7) 128 MiB 1945 -> 1888 us, AR (56,14,14)
//    663 -> 654, ring AR 616 -> 600; tools/gpu_runs/r01/l2mode2_round1w.sh).
//    Only plans that discard the receipts after use keep evict-last (one-shot
//    AR: 572 vs 578 us).  Demoting a relay to evict_normal with
//    applypriority after its last load cost 7-17 % (the instructions).
//    Discarding chain receipts from the signaler warp once their tile's
//    writes landed (off the compute path) still cost 1-3 % on (56,14,14)
//    and ring AR, and 5 % on (8,2,2) against the compute warps
//    (tools/gpu_runs/r01/discard3_round1w.sh).
//  * discards: streaming reductions drop consumed scratch receipts from L2
//    (discard.global.L2: no write-back of dead bytes): push-lowered (8,2,2)
//    at 64/128 MiB 321 -> 296 / 614 -> 560 us; chains of 2-input reduces
//    lost 10-20 % to the discard instructions in round 1 but gain 4-6 % with
//    the round-2 pipeline (numbers below).
// SCCL_WINDOW=<bytes> (0 = op-major), SCCL_L2HINT and SCCL_DISCARD override.
void choose_streaming(sccl_plan& p, const ProgramStats& st, bool loopback, const ModePolicy& pol) {
  const bool streams = !p.ll && st.bytes > pol.stream_bytes;
  bool all_vec = true;
  for (auto& d : p.ops) all_vec &= d.kind == OP_WAIT || d.vec;
  const double ops_per_step = double(st.nops_rank0) / double(std::max(1, p.kc * st.steps));
  const int m = std::max(1, std::min(4, int(std::ceil(4.0 / std::max(ops_per_step, 1e-9)))));
  p.window = (streams && pol.window_major && all_vec && st.rereads) ? uint32_t(p.tile) * uint32_t(m) : 0u;
  if (const char* env = std::getenv("SCCL_WINDOW")) {
    const long w = std::atol(env);
    p.window = (w > 0 && all_vec && !p.ll) ? uint32_t(std::max<long>(16, w) / 16 * 16) : 0u;
  }
  // pull-lowered reductions with no receipts (the loopback one-shot
  // allreduce) run better without evict-first hints: AR (8,2,2) bf16 at
  // 64 / 128 / 256 MiB per rank 182.7 / 358.5 / 713.1 -> 181.3 / 352.6 /
  // 696.3 us (tools/gpu_runs/r02/s2_verify1.sh); copy-only one-shots keep
  // them (A2A (8,1,1) +3.4 / +2.5 % without, profiles/r02/s2_rule_audit.jsonl)
  const bool pulled_oneshot = p.pg.pull && st.reduces && !st.rereads;
  p.l2hint = streams && pol.l2_hints && !pulled_oneshot ? 1 : 0;
  const char* hint_env = std::getenv("SCCL_L2HINT");  // 0, 1, or 3 (| kL2RelayPlain)
  if (hint_env) p.l2hint = std::atoi(hint_env) & 3;
  if (p.l2hint == kL2RelayPlain) p.l2hint = 0;
  bool any_dead = false;  // scratch receipts with one reader (pull plans of one-shot reductions have none)
  for (auto& x : p.ins) any_dead |= x.dead_after != 0;
  // (round 2: with pull and the current pipeline, chains gain too: AR
  // (56,14,14) 64 / 256 MiB 260 -> 245 / 1040 -> 977 us, ring AR -3.5 %,
  // DRAM 1.49 -> 1.29 GB per 64 MiB launch; tools/gpu_runs/r02/chain_discard.sh)
  p.discard = p.l2hint && pol.discard && any_dead;
  if (const char* env = std::getenv("SCCL_DISCARD")) p.discard = std::atoi(env) != 0 && !p.ll;
  if (p.l2hint && !p.discard && !hint_env) p.l2hint |= kL2RelayPlain;
  p.dcache_min_ops = 4;  // SCCL_DCACHE=<n> overrides (0 = off)
  if (const char* env = std::getenv("SCCL_DCACHE")) p.dcache_min_ops = std::max(0, std::atoi(env));
  // windows of each launched CTA's program
  const int nl = loopback ? p.sched.P : 1;
  p.nwin.assign(size_t(nl) * p.nch, 1u);
  if (!p.window) return;
  for (int lr = 0; lr < nl; ++lr) {
    const int r = loopback ? lr : p.rank;
    for (int ch = 0; ch < p.nch; ++ch) {
      const int cg = ch % p.kc, cb = ch / p.kc;
      int64_t maxq = 0;
      for (uint32_t o = p.prog[size_t(r) * p.kc + cg]; o < p.prog[size_t(r) * p.kc + cg + 1]; ++o)
        if (p.ops[o].kind != OP_WAIT) maxq = std::max(maxq, split16(int64_t(p.ops[o].len), p.kb, cb).len);
      p.nwin[size_t(lr) * p.nch + ch] = uint32_t(std::max<int64_t>(1, (maxq + p.window - 1) / p.window));
    }
  }
}

// Memory layout of one rank's region: [flags | scratch | recv (multi-process)].
void layout_memory(sccl_plan& p, bool loopback) {
  auto up = [](size_t x, size_t a) { return (x + a - 1) / a * a; };
  p.entry_base = p.pg.max_slots * p.nch;
  p.flags_bytes = up(sizeof(uint64_t) * size_t(p.entry_base + p.sched.P * p.nch), 4096);
  p.scratch_off = p.flags_bytes;
  p.scratch_set = up(size_t(p.pg.scratch_bytes), 4096);
  const size_t scratch = p.scratch_set * (p.ll_parity ? 2 : 1);
  p.recv_off = p.scratch_off + scratch;
  p.region_bytes = p.recv_off + (loopback ? 0 : up(size_t(p.pg.recv_bytes), 4096));
  p.region_bytes = up(p.region_bytes, 1 << 21);
}

}  // namespace

void plan_build_host(sccl_plan& p, const std::string& json, int rank, int nranks, int64_t bytes, int dtype,
                     int redop, int device, const ChannelRequest& req, int64_t timeout_ms, bool loopback) {
  if (redop != SCCL_SUM) throw invalid_argument_error("only SCCL_SUM is supported");
  const int es = esize_of(dtype);
  p.sched = parse_schedule(json);
  if (p.sched.P > kMaxRanks) throw invalid_argument_error("P exceeds the executor's 16-rank pointer table");
  if (!loopback) {
    if (nranks != p.sched.P) throw invalid_argument_error("nranks != schedule P");
    if (rank < 0 || rank >= nranks) throw invalid_argument_error("rank out of range");
  }
  int64_t maxlen = 0;  // the largest chunk
  for (auto& g : chunk_geometry(p.sched.kind, p.sched.P, p.sched.flat().back()->G, bytes)) maxlen = std::max(maxlen, g.len);

  // pull (combining sends of untouched inputs read in place by the
  // receiver): loopback only -- every rank's SEND is addressable there and
  // read-only for the whole launch.  Multi-process plans push: peers'
  // sendbufs are not mapped, and over NVLink the bytes per direction are
  // the same either way.
  if (req.pull > 0 && !loopback) throw invalid_argument_error("pull needs a loopback plan (peers' send buffers are not mapped)");
  const bool pull = loopback && req.pull >= 0;
  p.ll = choose_ll(p, bytes, es, req.protocol, loopback, pull);
  // SCCL_LL_PARITY=0: keep the entry handshake (A/B)
  const char* par_env = std::getenv("SCCL_LL_PARITY");
  p.ll_parity = p.ll && !loopback && !(par_env && par_env[0] == '0') && ll_parity_safe(p.sched);
  p.rank = loopback ? 0 : rank;
  p.nranks = p.sched.P;
  p.loopback = loopback;
  p.dtype = dtype;
  p.redop = redop;
  p.device = device;
  p.host_only = device < 0;
  // watchdog default: 10 s in loopback (every rank is in the one launch, so
  // a wait that long is a bug); 600 s for one rank per GPU, where a peer may
  // legitimately enter the collective late (checkpointing, evaluation, a
  // data-loader stall) -- the same order as torch.distributed's default
  // collective timeout.  An expiry aborts cooperatively (status 5, the CUDA
  // context stays usable, the plan is poisoned).
  const int64_t def_ms = loopback ? 10000 : 600000;
  p.timeout_ns = timeout_ms < 0 ? 0 : (timeout_ms == 0 ? def_ms : timeout_ms) * 1000000LL;

  const ProgramStats st = program_stats(p.sched, p.pg, loopback);
  const ModePolicy& pol = mode_policy(loopback);
  p.policy = pol.version;
  choose_stages(p, st, maxlen, req, pol);
  choose_channels(p, st, maxlen, req, loopback, pol);
  assign_groups(p);
  choose_release(p, loopback);
  encode_program(p);
  choose_streaming(p, st, loopback, pol);
  layout_memory(p, loopback);
}

}  // namespace sccl

using namespace sccl;

namespace {

void plan_device_setup(sccl_plan& p) {
  cuda_check(cudaSetDevice(p.device), "cudaSetDevice");
  auto upload = [](auto& vec, auto** dptr) {
    size_t n = std::max<size_t>(1, vec.size()) * sizeof(vec[0]);
    cuda_check(cudaMalloc(reinterpret_cast<void**>(dptr), n), "cudaMalloc(program)");
    if (!vec.empty()) cuda_check(cudaMemcpy(*dptr, vec.data(), vec.size() * sizeof(vec[0]), cudaMemcpyHostToDevice), "upload");
  };
  upload(p.ops, &p.d_ops);
  upload(p.ins, &p.d_ins);
  upload(p.outs, &p.d_outs);
  upload(p.prog, &p.d_prog);
  upload(p.dtab, &p.d_dtab);
  upload(p.nwin, &p.d_nwin);
  int nlaunch = p.loopback ? p.nranks : 1;
  size_t ne = size_t(nlaunch) * p.nch;
  cuda_check(cudaMalloc(&p.d_epochs, ne * sizeof(uint64_t)), "cudaMalloc(epochs)");
  cuda_check(cudaMemset(p.d_epochs, 0, ne * sizeof(uint64_t)), "memset(epochs)");
  size_t total = p.region_bytes * size_t(nlaunch);
  if (p.external) {
    // the caller supplies every rank's region at bind time (e.g. torch
    // symmetric memory, sccl_plan_bind_peers_external)
  } else if (p.vmm) {  // shareable cuMem allocation (POSIX fd)
    const Vmm& v = vmm_api();
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = p.device;
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    cu_check(v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    p.vmm_size = (total + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h = 0;
    cu_check(v.create(&h, p.vmm_size, &prop, 0), "cuMemCreate");
    p.vmm_handle = uint64_t(h);
    p.d_region = vmm_map(v, h, p.vmm_size, p.device);
  } else {
    cuda_check(cudaMalloc(&p.d_region, total), "cudaMalloc(region)");
  }
  if (!p.external) cuda_check(cudaMemset(p.d_region, 0, total), "memset(region)");
  cuda_check(cudaHostAlloc(&p.h_err, 64 * sizeof(int), cudaHostAllocMapped), "cudaHostAlloc(err)");
  std::memset(p.h_err, 0, 64 * sizeof(int));
  cuda_check(cudaHostGetDevicePointer(&p.d_err, p.h_err, 0), "cudaHostGetDevicePointer");
  cuda_check(cudaMalloc(&p.d_abort, 256), "cudaMalloc(abort)");
  cuda_check(cudaMemset(p.d_abort, 0, 256), "memset(abort)");
  cuda_check(cudaDeviceSynchronize(), "plan setup");
  if (!p.loopback) {
    p.peer_region.assign(p.nranks, nullptr);
    p.peer_region[p.rank] = p.d_region;
  }
}

struct OccCtx {
  int dtype;
  bool sys;
};
int occ_fn(void* ctx, int tile, int nstage) {
  auto* c = static_cast<OccCtx*>(ctx);
  int bps = 0;
  cuda_check(exec_occupancy(c->dtype, c->sys, tile, nstage, &bps), "occupancy");
  return bps;
}

// A launch whose watchdog expired leaves the plan's epochs and counters out
// of step with its peers': the plan cannot run again (destroy it).
void refuse_if_poisoned(const sccl_plan& p) {
  if (p.h_err && reinterpret_cast<volatile int*>(p.h_err)[0] != 0)
    throw timeout_error("plan aborted by an earlier peer timeout (watchdog); destroy it and create a new one");
}

void check_aligned(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) % 16) throw invalid_argument_error(std::string(what) + " must be 16-byte aligned");
}


void fill_common(const sccl_plan& p, KParams& k) {
  std::memset(&k, 0, sizeof k);
  k.ops = p.d_ops;
  k.ins = p.d_ins;
  k.outs = p.d_outs;
  k.prog = p.d_prog;
  k.dtab = p.d_dtab;
  k.dcache_min_ops = p.dcache_min_ops;
  k.window = p.window;
  k.l2hint = p.l2hint;
  k.discard = p.discard ? 1 : 0;
  k.nwin = p.d_nwin;
  k.epochs = p.d_epochs;
  k.errinfo = p.d_err;
  k.abort = p.d_abort;
  k.timeout_ns = p.timeout_ns;
  k.P = p.nranks;
  k.nch = p.nch;
  k.kc = p.kc;
  k.kb = p.kb;
  k.kb_magic = p.kb > 1 ? ~uint64_t(0) / uint64_t(p.kb) + 1 : 0;
  // x / d == umulhi(x, floor(2^32 / d) + 1) exactly for x, d < 2^16 (the
  // kernel's fastdiv; d == 1 is passed as 0 and handled there)
  auto magic32 = [](int d) -> uint32_t { return d <= 1 ? 0u : uint32_t((uint64_t(1) << 32) / uint64_t(d) + 1); };
  k.nch_magic = magic32(p.nch);
  k.kc_magic = magic32(p.kc);
  k.tile = p.tile;
  k.nstage = p.nstage;
  k.ll = p.ll ? 1 : 0;
  k.entry_base = p.entry_base;
  k.ll_parity = p.ll_parity ? uint64_t(p.scratch_set) : 0;
  k.trace = p.d_trace;
  k.trace_cap = p.trace_cap;
  k.selfpub = p.selfpub ? 1 : 0;
}

}  // namespace

extern "C" {

void sccl_plan_opts_init(sccl_plan_opts* o) {
  if (!o) return;
  o->device = 0;
  o->nchannels = 0;
  o->chunk_groups = 0;
  o->tile_bytes = 0;
  o->protocol = 0;
  o->timeout_ms = 0;
  o->mem_handles = 0;
  o->pull = 0;
}

const char* sccl_last_error(void) { return g_err.c_str(); }
const char* sccl_version(void) { return "sccl-b200 1.0 (sm_100a)"; }

int sccl_schedule_verify(const char* json, char* report, size_t* len) {
  bool bad = false;
  int rc = guarded([&] {
    if (!json) throw invalid_argument_error("schedule_json is NULL");
    Schedule s = parse_schedule(json);
    auto v = verify(s);
    std::ostringstream o;
    o << "[";
    for (size_t i = 0; i < v.size(); ++i)
      o << (i ? "," : "") << "[" << v[i].kind << "," << v[i].step << "," << v[i].chunk << "," << v[i].src << ","
        << v[i].dst << "]";
    o << "]";
    if (len) put_string(o.str(), report, len);
    bad = !v.empty();
    if (bad) g_err = "schedule has " + std::to_string(v.size()) + " violation(s): " + v[0].str();
  });
  return rc != SCCL_OK ? rc : (bad ? SCCL_INVALID_ARGUMENT : SCCL_OK);
}

int sccl_schedule_canonicalize(const char* json, char* out, size_t* len) {
  return guarded([&] {
    if (!json) throw invalid_argument_error("schedule_json is NULL");
    put_string(serialize(parse_schedule(json)), out, len);
  });
}

int sccl_schedule_invert(const char* json, char* out, size_t* len) {
  return guarded([&] {
    if (!json) throw invalid_argument_error("schedule_json is NULL");
    put_string(serialize(invert_schedule(parse_schedule(json))), out, len);
  });
}

int sccl_schedule_compose_allreduce(const char* rs, const char* ag, char* out, size_t* len) {
  return guarded([&] {
    if (!rs || !ag) throw invalid_argument_error("schedule_json is NULL");
    put_string(serialize(compose_allreduce(parse_schedule(rs), parse_schedule(ag))), out, len);
  });
}

int sccl_schedule_select(const char* const* jsons, int n, size_t bytes, int dtype, int multiprocess, int* index,
                         int* protocol, double* predicted_us) {
  return guarded([&] {
    if (!jsons || n <= 0 || !index || !protocol) throw invalid_argument_error("NULL argument or no candidates");
    const int es = esize_of(dtype);
    double best = 0;
    int bi = -1, bp = 0, P = -1;
    Kind kind{};
    for (int i = 0; i < n; ++i) {
      if (!jsons[i]) throw invalid_argument_error("schedule_json is NULL");
      const Schedule s = parse_schedule(jsons[i]);
      if (i == 0) {
        P = s.P;
        kind = s.kind;
      } else if (s.P != P || s.kind != kind) {
        throw invalid_argument_error("candidates must share the collective and P");
      }
      int steps = 0;
      for (auto* ph : s.flat()) steps += ph->S;
      for (int ll = 0; ll < 2; ++ll) {  // lower() verifies and throws on invalid input
        const bool mp = multiprocess != 0;
        const double t = predict_us(lower(s, int64_t(bytes), es, ll != 0, !mp), steps, ll != 0, signal_policy(!mp));
        if (bi < 0 || t < best) {
          best = t;
          bi = i;
          bp = ll ? 2 : 1;
        }
      }
    }
    *index = bi;
    *protocol = bp;
    if (predicted_us) *predicted_us = best;
  });
}

static int create_common(const char* json, int rank, int nranks, size_t bytes, int dtype, int redop,
                         const sccl_plan_opts* opts, sccl_plan** out, bool loopback) {
  return guarded([&] {
    if (!json || !out) throw invalid_argument_error("NULL argument");
    *out = nullptr;
    sccl_plan_opts o;
    sccl_plan_opts_init(&o);
    if (opts) o = *opts;
    auto* p = new sccl_plan();
    try {
      ChannelRequest req;
      req.nchannels = o.nchannels;
      req.chunk_groups = o.chunk_groups;
      req.tile = o.tile_bytes;
      req.protocol = o.protocol;
      req.pull = o.pull;
      OccCtx occ{dtype, !loopback};
      if (o.device >= 0) {
        cudaDeviceProp prop{};
        cuda_check(cudaGetDeviceProperties(&prop, o.device), "cudaGetDeviceProperties");
        cuda_check(cudaSetDevice(o.device), "cudaSetDevice");
        req.sms = prop.multiProcessorCount;
        req.blocks_per_sm = occ_fn;
        req.ctx = &occ;
      }
      plan_build_host(*p, json, rank, nranks, int64_t(bytes), dtype, redop, o.device, req, o.timeout_ms, loopback);
      if (loopback && p->nch * p->nranks > p->resident_cap)
        throw invalid_argument_error("loopback needs P*nchannels <= resident CTAs (" +
                                     std::to_string(p->resident_cap) + ")");
      if (o.mem_handles < 0 || o.mem_handles > 2)
        throw invalid_argument_error("mem_handles must be 0 (CUDA IPC), 1 (VMM fd) or 2 (caller-provided regions)");
      if (loopback && o.mem_handles == 2) throw invalid_argument_error("loopback plans own their memory");
      p->vmm = !loopback && o.mem_handles == 1;
      p->external = !loopback && o.mem_handles == 2;
      if (!p->host_only) plan_device_setup(*p);
    } catch (...) {
      sccl_plan_destroy(p);
      throw;
    }
    *out = p;
  });
}

int sccl_plan_create(const char* json, int rank, int nranks, size_t bytes, int dtype, int redop,
                     const sccl_plan_opts* opts, sccl_plan** out) {
  return create_common(json, rank, nranks, bytes, dtype, redop, opts, out, false);
}

int sccl_plan_create_loopback(const char* json, size_t bytes, int dtype, int redop, const sccl_plan_opts* opts,
                              sccl_plan** out) {
  return create_common(json, 0, 0, bytes, dtype, redop, opts, out, true);
}

int sccl_plan_export_handles(sccl_plan* p, void* blob, size_t* len) {
  return guarded([&] {
    if (!p || !len) throw invalid_argument_error("NULL argument");
    if (p->loopback) throw invalid_argument_error("loopback plans have no peers");
    if (!blob || *len < sizeof(IpcBlob)) {
      *len = sizeof(IpcBlob);
      if (blob) throw invalid_argument_error("blob buffer too small");
      return;
    }
    IpcBlob b{};
    std::memcpy(b.magic, "SCCLIPC3", 8);
    std::strncpy(b.fingerprint, p->pg.fingerprint.c_str(), sizeof b.fingerprint - 1);
    b.rank = p->rank;
    b.nranks = p->nranks;
    b.nch = p->nch;
    b.kc = p->kc;
    b.kb = p->kb;
    b.tile = p->tile;
    b.dtype = p->dtype;
    b.redop = p->redop;
    b.ll_parity = p->ll_parity ? 1 : 0;
    b.region_bytes = p->region_bytes;
    if (!p->host_only && !p->vmm && !p->external) {
      cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
      cuda_check(cudaIpcGetMemHandle(&b.handle, p->d_region), "cudaIpcGetMemHandle");
    }
    std::memcpy(blob, &b, sizeof b);
    *len = sizeof b;
  });
}

static std::vector<IpcBlob> check_blobs(sccl_plan* p, const void* const* blobs, size_t blob_len) {
  if (!p || !blobs) throw invalid_argument_error("NULL argument");
  if (p->loopback) throw invalid_argument_error("loopback plans have no peers");
  if (p->bound) throw invalid_argument_error("plan already bound");
  if (blob_len < sizeof(IpcBlob)) throw invalid_argument_error("blob too short");
  std::vector<IpcBlob> bs(p->nranks);
  for (int r = 0; r < p->nranks; ++r) {
    if (!blobs[r]) throw invalid_argument_error("missing blob for rank " + std::to_string(r));
    std::memcpy(&bs[r], blobs[r], sizeof(IpcBlob));
    const IpcBlob& b = bs[r];
    if (std::memcmp(b.magic, "SCCLIPC3", 8)) throw invalid_argument_error("bad blob magic from rank " + std::to_string(r));
    if (b.rank != r || b.nranks != p->nranks)
      throw invalid_argument_error("blob " + std::to_string(r) + " has rank/nranks mismatch");
    if (std::strncmp(b.fingerprint, p->pg.fingerprint.c_str(), sizeof b.fingerprint - 1))
      throw invalid_argument_error("rank " + std::to_string(r) + " lowered a different program (fingerprint mismatch)");
    if (b.nch != p->nch || b.kc != p->kc || b.kb != p->kb || b.tile != p->tile || b.region_bytes != p->region_bytes)
      throw invalid_argument_error("rank " + std::to_string(r) + " uses different channels/tile/region size");
    if (b.ll_parity != (p->ll_parity ? 1 : 0))
      throw invalid_argument_error("rank " + std::to_string(r) + " uses a different LL slot protocol (SCCL_LL_PARITY)");
    if (b.dtype != p->dtype || b.redop != p->redop)
      throw invalid_argument_error("rank " + std::to_string(r) + " uses a different dtype/redop (dtype " +
                                   std::to_string(b.dtype) + " vs " + std::to_string(p->dtype) + ")");
  }
  return bs;
}

int sccl_plan_bind_peers(sccl_plan* p, const void* const* blobs, size_t blob_len) {
  return guarded([&] {
    const std::vector<IpcBlob> bs = check_blobs(p, blobs, blob_len);
    if (p->vmm) throw invalid_argument_error("VMM plan: bind with sccl_plan_bind_peers_fd");
    if (p->external) throw invalid_argument_error("external-region plan: bind with sccl_plan_bind_peers_external");
    if (!p->host_only) {
      cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
      for (int r = 0; r < p->nranks; ++r) {
        if (r == p->rank) continue;
        void* ptr = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&ptr, bs[r].handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        p->peer_region[r] = static_cast<char*>(ptr);
      }
    }
    p->bound = true;
  });
}

int sccl_plan_export_fd(sccl_plan* p, int* fd) {
  return guarded([&] {
    if (!p || !fd) throw invalid_argument_error("NULL argument");
    if (!p->vmm) throw invalid_argument_error("plan was not created with mem_handles = 1 (VMM)");
    if (p->host_only) throw invalid_argument_error("host-only plan has no device region");
    const Vmm& v = vmm_api();
    int out = -1;
    cu_check(v.export_handle(&out, CUmemGenericAllocationHandle(p->vmm_handle), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
             "cuMemExportToShareableHandle");
    *fd = out;
  });
}

int sccl_plan_bind_peers_fd(sccl_plan* p, const void* const* blobs, size_t blob_len, const int* fds) {
  return guarded([&] {
    const std::vector<IpcBlob> bs = check_blobs(p, blobs, blob_len);
    if (!p->vmm) throw invalid_argument_error("plan was not created with mem_handles = 1 (VMM)");
    if (!fds) throw invalid_argument_error("NULL fds");
    if (!p->host_only) {
      cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
      const Vmm& v = vmm_api();
      p->peer_vmm.assign(p->nranks, 0);
      for (int r = 0; r < p->nranks; ++r) {
        if (r == p->rank) continue;
        if (fds[r] < 0) throw invalid_argument_error("missing fd for rank " + std::to_string(r));
        CUmemGenericAllocationHandle h = 0;
        cu_check(v.import_handle(&h, reinterpret_cast<void*>(uintptr_t(fds[r])), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 "cuMemImportFromShareableHandle");
        p->peer_vmm[r] = uint64_t(h);
        p->peer_region[r] = vmm_map(v, h, p->vmm_size, p->device);
      }
    }
    p->bound = true;
  });
}

int sccl_plan_register_export(sccl_plan* p, void* buf, size_t bytes, void* blob, size_t* len) {
  return guarded([&] {
    if (!p || !len) throw invalid_argument_error("NULL argument");
    if (p->loopback) throw invalid_argument_error("loopback plans write caller buffers directly (nothing to register)");
    if (!blob || *len < sizeof(RegBlob)) {
      *len = sizeof(RegBlob);
      if (blob) throw invalid_argument_error("blob buffer too small");
      return;
    }
    if (!buf) throw invalid_argument_error("NULL buffer");
    check_aligned(buf, "registered buffer");
    if (bytes < size_t(p->pg.recv_bytes))
      throw invalid_argument_error("registered buffer smaller than the plan's receive size (" +
                                   std::to_string(p->pg.recv_bytes) + " bytes)");
    RegBlob b{};
    std::memcpy(b.magic, "SCCLREG1", 8);
    b.rank = p->rank;
    b.bytes = bytes;
    if (!p->host_only) {
      cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
      CUdeviceptr base = 0;
      size_t sz = 0;
      cu_check(vmm_api().address_range(&base, &sz, CUdeviceptr(buf)), "cuMemGetAddressRange");
      b.offset = uint64_t(CUdeviceptr(buf) - base);
      if (b.offset + bytes > sz) throw invalid_argument_error("registered buffer runs past its allocation");
      cuda_check(cudaIpcGetMemHandle(&b.handle, reinterpret_cast<void*>(base)),
                 "cudaIpcGetMemHandle (registered buffers must come from cudaMalloc / the torch caching allocator)");
    }
    std::memcpy(blob, &b, sizeof b);
    *len = sizeof b;
  });
}

int sccl_plan_register_bind(sccl_plan* p, void* buf, const void* const* blobs, size_t blob_len) {
  return guarded([&] {
    if (!p || !buf || !blobs) throw invalid_argument_error("NULL argument");
    if (p->loopback) throw invalid_argument_error("loopback plans have no peers");
    if (!p->bound) throw invalid_argument_error("bind the plan's peers first (sccl_plan_bind_peers)");
    if (blob_len < sizeof(RegBlob)) throw invalid_argument_error("blob too short");
    for (auto& g : p->regs)
      if (g.local == buf) throw invalid_argument_error("buffer already registered with this plan");
    sccl_plan::RegBuf reg;
    reg.local = static_cast<char*>(buf);
    reg.peer.assign(p->nranks, nullptr);
    reg.peer[p->rank] = reg.local;
    for (int r = 0; r < p->nranks; ++r) {
      if (!blobs[r]) throw invalid_argument_error("missing registration blob for rank " + std::to_string(r));
      RegBlob b;
      std::memcpy(&b, blobs[r], sizeof b);
      if (std::memcmp(b.magic, "SCCLREG1", 8) || b.rank != r)
        throw invalid_argument_error("bad registration blob from rank " + std::to_string(r));
      if (b.bytes < uint64_t(p->pg.recv_bytes))
        throw invalid_argument_error("rank " + std::to_string(r) + " registered a buffer smaller than the receive size");
      if (r == p->rank) {
        reg.bytes = size_t(b.bytes);
        continue;
      }
      if (p->host_only) continue;
      // one mapping per peer allocation (torch's caching allocator carves many
      // tensors out of one cudaMalloc segment; a handle opens once per process)
      const std::string key = std::to_string(r) + "|" + std::string(reinterpret_cast<const char*>(&b.handle), sizeof b.handle);
      char* base = nullptr;
      for (auto& kv : p->ipc_open)
        if (kv.first == key) base = kv.second;
      if (!base) {
        cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
        void* ptr = nullptr;
        cuda_check(cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle (registered buffer)");
        base = static_cast<char*>(ptr);
        p->ipc_open.push_back({key, base});
      }
      reg.peer[r] = base + b.offset;
    }
    p->regs.push_back(std::move(reg));
  });
}

int sccl_plan_deregister(sccl_plan* p, void* buf) {
  return guarded([&] {
    if (!p || !buf) throw invalid_argument_error("NULL argument");
    for (size_t i = 0; i < p->regs.size(); ++i)
      if (p->regs[i].local == buf) {
        p->regs.erase(p->regs.begin() + long(i));
        return;  // peer mappings stay open until the plan is destroyed (other registrations may share them)
      }
    throw invalid_argument_error("buffer is not registered with this plan");
  });
}

int sccl_plan_region_bytes(sccl_plan* p, size_t* bytes) {
  return guarded([&] {
    if (!p || !bytes) throw invalid_argument_error("NULL argument");
    if (p->loopback) throw invalid_argument_error("loopback plans have no shared region");
    *bytes = p->region_bytes;
  });
}

int sccl_plan_bind_peers_external(sccl_plan* p, const void* const* regions) {
  return guarded([&] {
    if (!p || !regions) throw invalid_argument_error("NULL argument");
    if (!p->external) throw invalid_argument_error("plan was not created with mem_handles = 2 (caller-provided regions)");
    if (p->bound) throw invalid_argument_error("plan already bound");
    for (int r = 0; r < p->nranks; ++r) {
      if (!regions[r]) throw invalid_argument_error("missing region for rank " + std::to_string(r));
      check_aligned(regions[r], "region");
    }
    if (!p->host_only) {
      cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
      p->d_region = static_cast<char*>(const_cast<void*>(regions[p->rank]));
      // counters start at zero; peers may write into this region only after
      // this rank's first launch (entry handshake), and the caller's barrier
      // after every bind orders this memset before any peer's first launch
      cuda_check(cudaMemset(p->d_region, 0, p->region_bytes), "memset(external region)");
      cuda_check(cudaDeviceSynchronize(), "bind");
      for (int r = 0; r < p->nranks; ++r) p->peer_region[r] = static_cast<char*>(const_cast<void*>(regions[r]));
    }
    p->bound = true;
  });
}

int sccl_plan_recv_buffer(sccl_plan* p, void** ptr, size_t* bytes) {
  return guarded([&] {
    if (!p || !ptr) throw invalid_argument_error("NULL argument");
    if (p->loopback || p->host_only) throw invalid_argument_error("no registered receive buffer");
    *ptr = p->d_region + p->recv_off;
    if (bytes) *bytes = size_t(p->pg.recv_bytes);
  });
}

int sccl_launch(sccl_plan* p, const void* sendbuf, void* recvbuf, void* stream) {
  return guarded([&] {
    if (!p) throw invalid_argument_error("NULL plan");
    if (p->loopback) throw invalid_argument_error("use sccl_launch_loopback for loopback plans");
    if (p->host_only) throw invalid_argument_error("host-only plan cannot launch (no CUDA device)");
    if (!p->bound) throw invalid_argument_error("plan not bound to peers (sccl_plan_bind_peers)");
    if (p->pg.send_bytes && !sendbuf) throw invalid_argument_error("sendbuf is NULL");
    check_aligned(sendbuf, "sendbuf");
    char* reg = p->d_region + p->recv_off;
    if (recvbuf) check_aligned(recvbuf, "recvbuf");
    refuse_if_poisoned(*p);
    const sccl_plan::RegBuf* target = nullptr;  // a registered caller buffer: peers write it directly
    for (auto& g : p->regs)
      if (recvbuf && g.local == recvbuf) target = &g;
    KParams k;
    fill_common(*p, k);
    for (int r = 0; r < p->nranks; ++r) {
      char* reg_r = p->peer_region[r];
      k.base[r][SP_SEND] = r == p->rank ? const_cast<char*>(static_cast<const char*>(sendbuf)) : nullptr;
      k.base[r][SP_RECV] = target ? target->peer[r] : reg_r + p->recv_off;
      k.base[r][SP_SCRATCH] = reg_r + p->scratch_off;
      k.base[r][SP_FLAGS] = reg_r;
    }
    k.rank0 = p->rank;
    k.nranks_launch = 1;
    k.multiprocess = 1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
    cuda_check(launch_exec(k, p->dtype, true, st), "launch");
    p->launches++;
    if (!target && recvbuf && recvbuf != reg && p->pg.recv_bytes)
      cuda_check(cudaMemcpyAsync(recvbuf, reg, size_t(p->pg.recv_bytes), cudaMemcpyDeviceToDevice, st),
                 "copy-out of the registered receive buffer");
  });
}

int sccl_launch_loopback(sccl_plan* p, const void* const* sendbufs, void* const* recvbufs, void* stream) {
  return guarded([&] {
    if (!p || !sendbufs || !recvbufs) throw invalid_argument_error("NULL argument");
    if (!p->loopback) throw invalid_argument_error("not a loopback plan");
    if (p->host_only) throw invalid_argument_error("host-only plan cannot launch (no CUDA device)");
    refuse_if_poisoned(*p);
    KParams k;
    fill_common(*p, k);
    for (int r = 0; r < p->nranks; ++r) {
      if (p->pg.send_bytes && !sendbufs[r]) throw invalid_argument_error("sendbuf is NULL");
      if (p->pg.recv_bytes && !recvbufs[r]) throw invalid_argument_error("recvbuf is NULL");
      check_aligned(sendbufs[r], "sendbuf");
      check_aligned(recvbufs[r], "recvbuf");
      char* reg = p->d_region + size_t(r) * p->region_bytes;
      k.base[r][SP_SEND] = const_cast<char*>(static_cast<const char*>(sendbufs[r]));
      k.base[r][SP_RECV] = static_cast<char*>(recvbufs[r]);
      k.base[r][SP_SCRATCH] = reg + p->scratch_off;
      k.base[r][SP_FLAGS] = reg;
    }
    k.rank0 = 0;
    k.nranks_launch = p->nranks;
    k.multiprocess = 0;
    cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
    // SCCL_LOOPBACK_SYS=1 (measurement only): system-scope fences and flags,
    // as in multi-process mode, to price that mode's signalling on one GPU
    cuda_check(launch_exec(k, p->dtype, loopback_sys(), static_cast<cudaStream_t>(stream)), "launch");
    p->launches++;
  });
}

int sccl_launch_loopback_copy_engine(sccl_plan* p, const void* const* sendbufs, void* const* recvbufs,
                                     void* stream) {
  return guarded([&] {
    if (!p || !sendbufs || !recvbufs) throw invalid_argument_error("NULL argument");
    if (!p->loopback || p->host_only) throw invalid_argument_error("needs a device loopback plan");
    if (p->ll) throw invalid_argument_error("copy-engine baseline needs the simple protocol's program");
    // the paper's per-step cudaMemcpy lowering:
    // every send of the lowered program becomes one stream-ordered
    // device-to-device copy, steps in order -- a comparison point, not the
    // hot path (no reductions: combining schedules need the kernel)
    std::vector<std::pair<int, std::pair<int, const Op*>>> order;
    for (int r = 0; r < p->nranks; ++r)
      for (const Op& op : p->pg.ranks[r].ops) {
        if (op.kind == OP_REDUCE) throw invalid_argument_error("copy-engine baseline: combining schedules unsupported");
        if (op.kind == OP_COPY) order.push_back({op.key, {r, &op}});
      }
    std::stable_sort(order.begin(), order.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    auto base = [&](int rank, int space) -> char* {
      if (space == SP_SEND) return const_cast<char*>(static_cast<const char*>(sendbufs[rank]));
      if (space == SP_RECV) return static_cast<char*>(recvbufs[rank]);
      return p->d_region + size_t(rank) * p->region_bytes + p->scratch_off;
    };
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_check(cudaSetDevice(p->device), "cudaSetDevice");
    for (auto& e : order) {
      const Op& op = *e.second.second;
      if (op.len == 0) continue;
      const char* src = base(op.ins[0].loc.rank, op.ins[0].loc.space) + op.ins[0].loc.off;
      for (auto& o : op.outs)
        cuda_check(cudaMemcpyAsync(base(o.loc.rank, o.loc.space) + o.loc.off, src, size_t(op.len),
                                   cudaMemcpyDeviceToDevice, st),
                   "cudaMemcpyAsync");
    }
  });
}

int sccl_plan_check(sccl_plan* p) {
  return guarded([&] {
    if (!p) throw invalid_argument_error("NULL plan");
    if (p->h_err && p->h_err[0] != 0) {
      volatile int* e = p->h_err;
      throw timeout_error("peer timeout: rank " + std::to_string(e[1]) + " channel " + std::to_string(e[2]) +
                          " op " + std::to_string(e[3]) + " slot " + std::to_string(e[4]) + " waited for " +
                          std::to_string(e[5]) + ", saw " + std::to_string(e[6]));
    }
  });
}

int sccl_plan_info(sccl_plan* p, char* out, size_t* len) {
  return guarded([&] {
    if (!p) throw invalid_argument_error("NULL plan");
    std::ostringstream o;
    o << "{\"nchannels\":" << p->nch << ",\"chunk_groups\":" << p->kc << ",\"byte_parts\":" << p->kb
      << ",\"storer_warps\":" << kStorerWarps << ",\"selfpub\":" << (p->selfpub ? 1 : 0) << ",\"window\":" << p->window << ",\"l2hint\":" << (p->l2hint & 1) << ",\"relay_evict_last\":" << ((p->l2hint & 1) && !(p->l2hint & kL2RelayPlain) ? 1 : 0) << ",\"discard\":" << (p->discard ? 1 : 0) << ",\"groups_balanced\":" << (p->groups_balanced ? 1 : 0) << ",\"nstage\":" << p->nstage << ",\"protocol\":\"" << (p->ll ? "ll" : "simple") << "\"" << ",\"ll_parity\":" << (p->ll_parity ? 1 : 0) << ",\"pull\":" << (p->pg.pull ? 1 : 0) << ",\"policy\":\"" << p->policy << "\"" << ",\"tile_bytes\":" << p->tile << ",\"threads\":" << exec_threads()
      << ",\"loopback\":" << (p->loopback ? 1 : 0) << ",\"rank\":" << p->rank << ",\"nranks\":" << p->nranks
      << ",\"grid\":" << (p->loopback ? p->nranks : 1) * p->nch << ",\"region_bytes\":" << p->region_bytes
      << ",\"nops\":" << p->ops.size() << ",\"program\":" << p->pg.summary_json() << "}";
    put_string(o.str(), out, len);
  });
}

int64_t sccl_plan_launch_count(sccl_plan* p) { return p ? p->launches : -1; }

int sccl_plan_destroy(sccl_plan* p) {
  if (!p) return SCCL_OK;
  if (!p->host_only && p->device >= 0) {
    cudaSetDevice(p->device);
    if (p->vmm) {
      const Vmm& v = vmm_api();
      for (size_t r = 0; r < p->peer_region.size(); ++r)
        if (int(r) != p->rank && p->peer_region[r]) {
          v.unmap(CUdeviceptr(p->peer_region[r]), p->vmm_size);
          v.addr_free(CUdeviceptr(p->peer_region[r]), p->vmm_size);
          if (r < p->peer_vmm.size() && p->peer_vmm[r]) v.release(CUmemGenericAllocationHandle(p->peer_vmm[r]));
        }
    } else if (!p->external) {  // (caller-provided regions are the caller's to unmap)
      for (size_t r = 0; r < p->peer_region.size(); ++r)
        if (int(r) != p->rank && p->peer_region[r]) cudaIpcCloseMemHandle(p->peer_region[r]);
    }
    for (auto& kv : p->ipc_open) cudaIpcCloseMemHandle(kv.second);
    cudaFree(p->d_ops);
    cudaFree(p->d_ins);
    cudaFree(p->d_outs);
    cudaFree(p->d_prog);
    cudaFree(p->d_dtab);
    cudaFree(p->d_nwin);
    cudaFree(p->d_epochs);
    if (p->external) {
      // caller-owned regions
    } else if (p->vmm) {
      if (p->d_region) {
        const Vmm& v = vmm_api();
        v.unmap(CUdeviceptr(p->d_region), p->vmm_size);
        v.addr_free(CUdeviceptr(p->d_region), p->vmm_size);
        v.release(CUmemGenericAllocationHandle(p->vmm_handle));
      }
    } else {
      cudaFree(p->d_region);
    }
    if (p->h_err) cudaFreeHost(p->h_err);
    cudaFree(p->d_abort);
  }
  delete p;
  return SCCL_OK;
}

}  // extern "C"
