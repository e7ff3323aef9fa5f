// Plan object behind the C-ABI: the lowered program, its device encoding,
// the plan-owned memory (flags, scratch, registered receive buffer) and the
// peer mappings.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "devprog.hpp"
#include "lower.hpp"
#include "schedule.hpp"

struct sccl_plan {
  sccl::Schedule sched;
  sccl::Program pg;
  int rank = 0, nranks = 0;
  bool loopback = false, host_only = false;
  int device = -1, dtype = 0, redop = 0;
  int nch = 1, kc = 1, kb = 1, tile = 32768, nstage = 6;
  int resident_cap = 0;  // loopback: CTAs that fit on the device at once
  bool ll = false;       // low-latency protocol
  bool ll_parity = false;  // LL, one rank per GPU: two scratch slot sets by launch parity, no entry handshake
  bool selfpub = false;  // simple protocol: storer warps release their own counters (latency-bound plans)
  long long timeout_ns = 0;
  std::string policy;    // version of the policy table the plan was built under

  // host copy of the device program (also used by the CPU interpreter)
  std::vector<sccl::DevOp> ops;
  std::vector<sccl::DevIn> ins;
  std::vector<sccl::DevOut> outs;
  std::vector<uint32_t> prog;  // [P*kc+1]: op range per (rank, chunk group)
  int dcache_min_ops = 4;      // simple kernel: descriptors cached in smem from this many ops per CTA
  std::vector<int> group_of;    // chunk id -> chunk group (balanced over the ranks' work)
  bool groups_balanced = false; // group_of is the greedy map, not chunk % kc
  std::vector<uint32_t> dtab;  // [P*kc][8]: op / in / out ranges per (rank, chunk group)
  uint32_t window = 0;         // simple protocol: window-major byte window (0 = op-major)
  int l2hint = 0;              // L2 eviction hints on bulk copies (bit 0; bits 1-2: experiments)
  bool discard = false;        // drop consumed scratch receipts of reduce tiles from L2
  std::vector<uint32_t> nwin;  // [launched CTAs] windows of each CTA's program

  // device program
  sccl::DevOp* d_ops = nullptr;
  sccl::DevIn* d_ins = nullptr;
  sccl::DevOut* d_outs = nullptr;
  uint32_t* d_prog = nullptr;
  uint32_t* d_dtab = nullptr;
  uint32_t* d_nwin = nullptr;
  uint64_t* d_epochs = nullptr;

  // plan memory: per rank region = [flags | scratch | recv (multi-process)]
  char* d_region = nullptr;
  size_t region_bytes = 0, flags_bytes = 0, scratch_off = 0, recv_off = 0;
  size_t scratch_set = 0;  // bytes of one scratch slot set (ll_parity: the scratch holds two)
  int entry_base = 0;
  std::vector<char*> peer_region;  // multi-process: every rank's region (own included)
  // VMM mode (opts.mem_handles = 1): cuMem allocation handles (CUmemGenericAllocationHandle)
  bool vmm = false;
  bool external = false;  // opts.mem_handles = 2: regions supplied by the caller (torch symmetric memory)
  uint64_t vmm_handle = 0;
  size_t vmm_size = 0;
  std::vector<uint64_t> peer_vmm;  // imported handles, 0 = none
  bool bound = false;
  // caller buffers registered as zero-copy receive targets (multi-process):
  // local pointer, size, every rank's mapping of its counterpart
  struct RegBuf {
    char* local = nullptr;
    size_t bytes = 0;
    std::vector<char*> peer;
  };
  std::vector<RegBuf> regs;
  std::vector<std::pair<std::string, char*>> ipc_open;  // opened peer allocations (rank|handle -> base)

  int* h_err = nullptr;  // host-mapped watchdog record
  int* d_err = nullptr;
  int* d_abort = nullptr;  // device abort word (cooperative watchdog abort)
  int64_t launches = 0;
  uint64_t* d_trace = nullptr;  // debug trace buffer (caller-owned), sccl_debug_set_trace
  int trace_cap = 0;
};

namespace sccl {

// host-side construction (no CUDA calls)
// Channel policy inputs: user overrides (0 = auto) and the resident-CTA
// capacity per SM as a function of the tile (shared-memory stage) size.
struct ChannelRequest {
  int nchannels = 0, chunk_groups = 0, tile = 0, protocol = 0, stage_budget = 0;
  int pull = 0;  // 0 auto (loopback: on), 1 on (loopback only), -1 off
  int sms = 148;
  int (*blocks_per_sm)(void* ctx, int tile, int nstage) = nullptr;
  void* ctx = nullptr;
};

void plan_build_host(sccl_plan& p, const std::string& json, int rank, int nranks, int64_t bytes, int dtype,
                     int redop, int device, const ChannelRequest& req, int64_t timeout_ms, bool loopback);

}  // namespace sccl
