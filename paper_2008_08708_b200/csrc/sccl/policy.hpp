// Plan policy tables, one per execution mode.
//
// Loopback plans (every rank on one GPU) were tuned on B200 with all rank
// buffers in one HBM: HBM/L2 behaviour decides there (window-major order, L2
// eviction hints, receipt discards, the chunk-group split of big relays).
// One-rank-per-GPU plans move their bytes over NVLink (900 GB/s per
// direction against 6.5 TB/s of local HBM), so none of those HBM policies is
// inherited: they are off in the multi-process table until an N>1 sweep
// says otherwise.  Each table has a version string (reported by
// sccl_plan_info); SCCL_POLICY=<file.json> replaces either table at run time
// (tools/tune.py --multi writes such a file from N>1 measurements).
#pragma once

#include <string>

namespace sccl {

struct ModePolicy {
  std::string version;
  // protocol cost model t = c + alpha * steps + beta * MB (tools/fit_protocol.py)
  double ll_c, ll_alpha, ll_beta;
  double simple_c, simple_alpha, simple_beta;
  double stream_bytes;      // a launch "streams" past L2 above this many program bytes (this rank's share)
  bool window_major;        // streaming relay schedules walk byte windows of every op
  bool l2_hints;            // streaming bulk copies carry L2 eviction hints
  bool discard;             // streaming wide reductions drop consumed receipts from L2
  bool group_split;         // streaming copy relays with >= 4 ops per step split into two chunk groups
  int max_ctas_per_rank;    // 0 = all resident CTAs / P (loopback); else this cap
  int selfpub_max_tiles;    // storer warps release their own counters up to this many tiles per CTA
};

// the compiled-in tables (or SCCL_POLICY's replacement of them)
const ModePolicy& mode_policy(bool loopback);

// a table from JSON text: {"loopback": {...}, "multiprocess": {...}} (either
// may be omitted); fields as in ModePolicy.  Throws invalid_argument_error.
void parse_policy_tables(const std::string& json, ModePolicy& loopback, ModePolicy& multiprocess);

}  // namespace sccl
