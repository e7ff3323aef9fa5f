#include "policy.hpp"

#include <cstdlib>
#include <fstream>
#include <mutex>
#include <sstream>

#include "error.hpp"
#include "json.hpp"

namespace sccl {

namespace {

// Loopback (all ranks in one HBM): the round-1 B200 measurements.
//  * protocol fit: tools/fit_protocol.py over the loopback crossover sweep
//    (7 schedules x 16 KiB-16 MiB x both protocols), mean regret 0.9 %;
//  * 1 GB streaming threshold, window-major, L2 hints and discards:
//    profiles/r01/window, l2policy, discard;
//  * no chunk-group split: round 1 split the (7,7,7) allgather's chunks into
//    two groups above 4 GB of traffic, but with the round-2 pipeline one
//    group is faster at every size (64 / 128 / 256 / 512 MiB per rank:
//    911 / 1752 / 3518 / 7044 -> 872 / 1730 / 3509 / 6903 us, medians of 3;
//    tools/gpu_runs/r02/s2_ag_split_ab.sh, profiles/r02/s2_ag_split_ab.jsonl);
//  * self-publish up to 16 tiles per CTA (tools/gpu_runs/r01/winsig_round1h.sh).
ModePolicy loopback_default() {
  ModePolicy p;
  p.version = "loopback-b200-r02.1";
  p.ll_c = 4.80, p.ll_alpha = 0.522, p.ll_beta = 0.353;
  p.simple_c = 4.50, p.simple_alpha = 2.72, p.simple_beta = 0.126;
  p.stream_bytes = 1e9;
  p.window_major = p.l2_hints = p.discard = true;
  p.group_split = false;
  p.max_ctas_per_rank = 0;
  p.selfpub_max_tiles = 16;
  return p;
}

// One rank per GPU.  Protocol constants: the system-scope fit (the same
// kernel at sys scope in loopback, SCCL_LOOPBACK_SYS=1, mean regret 0.8 %),
// the only sys-scope data one GPU can give; an N>1 sweep refits them
// (tools/tune.py --multi).  No HBM streaming policies (see policy.hpp);
// 32 CTAs per rank (NCCL's channel count order on NVSwitch boxes);
// self-publish up to 4 tiles (the sys fence on the store path costs ~3x).
ModePolicy multiprocess_default() {
  ModePolicy p;
  p.version = "multiprocess-sysproxy-r02";
  p.ll_c = 4.79, p.ll_alpha = 0.520, p.ll_beta = 0.353;
  p.simple_c = 5.00, p.simple_alpha = 6.33, p.simple_beta = 0.163;
  p.stream_bytes = 1e9;
  p.window_major = p.l2_hints = p.discard = p.group_split = false;
  p.max_ctas_per_rank = 32;
  p.selfpub_max_tiles = 4;
  return p;
}

void apply(const json::Value& v, ModePolicy& p) {
  auto num = [&](const char* k, double& out) {
    if (const json::Value* x = v.find(k)) {
      if (x->type == json::Value::Int) out = double(x->i);
      else if (x->type == json::Value::Real) out = x->d;
      else throw invalid_argument_error(std::string("policy: '") + k + "' must be a number");
    }
  };
  auto flag = [&](const char* k, bool& out) {
    if (const json::Value* x = v.find(k)) {
      if (x->type == json::Value::Bool) out = x->b;
      else if (x->type == json::Value::Int) out = x->i != 0;
      else throw invalid_argument_error(std::string("policy: '") + k + "' must be a boolean");
    }
  };
  auto integer = [&](const char* k, int& out) {
    if (const json::Value* x = v.find(k)) out = int(x->as_int(k));
  };
  if (const json::Value* x = v.find("version")) p.version = x->as_str("version");
  num("ll_c", p.ll_c), num("ll_alpha", p.ll_alpha), num("ll_beta", p.ll_beta);
  num("simple_c", p.simple_c), num("simple_alpha", p.simple_alpha), num("simple_beta", p.simple_beta);
  num("stream_bytes", p.stream_bytes);
  flag("window_major", p.window_major), flag("l2_hints", p.l2_hints), flag("discard", p.discard);
  flag("group_split", p.group_split);
  integer("max_ctas_per_rank", p.max_ctas_per_rank);
  integer("selfpub_max_tiles", p.selfpub_max_tiles);
  if (p.max_ctas_per_rank < 0 || p.selfpub_max_tiles < 0 || p.stream_bytes <= 0)
    throw invalid_argument_error("policy: negative limits");
}

}  // namespace

void parse_policy_tables(const std::string& text, ModePolicy& loopback, ModePolicy& multiprocess) {
  json::Value v = json::Parser(text).parse();
  if (v.type != json::Value::Object) throw invalid_argument_error("policy: top level must be an object");
  if (const json::Value* x = v.find("loopback")) apply(*x, loopback);
  if (const json::Value* x = v.find("multiprocess")) apply(*x, multiprocess);
}

const ModePolicy& mode_policy(bool loopback) {
  static ModePolicy lb, mp;
  static std::once_flag once;
  std::call_once(once, [] {
    lb = loopback_default();
    mp = multiprocess_default();
    if (const char* path = std::getenv("SCCL_POLICY")) {
      std::ifstream f(path);
      if (!f) throw invalid_argument_error(std::string("SCCL_POLICY: cannot read ") + path);
      std::stringstream ss;
      ss << f.rdbuf();
      parse_policy_tables(ss.str(), lb, mp);
    }
  });
  return loopback ? lb : mp;
}

}  // namespace sccl
