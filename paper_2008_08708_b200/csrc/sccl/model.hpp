// Topology and collective model (the reference's L0 layer).
//   topology     SPEC.md:17-109   (builders :36-71, file format :103-104)
//   collectives  SPEC.md:111-200  (relations :129-164, to_global :165-173,
//                                   make_spec :174-182, chunk id i*P+n :191)
// plus the NVSwitch target `switch:P` (per-GPU egress/ingress groups,
// PAPER.md:345), which replaces the DGX-1 hybrid cube-mesh as the synthesis
// target on an 8xB200 box.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace sccl {

struct Constraint {
  std::vector<std::pair<int, int>> edges;  // directed (src, dst)
  int bound = 0;                           // chunks per round
};

struct Topology {
  std::string name;
  int P = 0;
  std::vector<Constraint> constraints;

  // E: pairs covered by >= 1 constraint, all of bound > 0.
  std::vector<uint8_t> links() const;
  // FNV-1a 64 of the canonical constraint text, 16 lowercase hex digits.
  std::string hash() const;
};

Topology build_ring(int P, int bw = 1);
Topology build_fully_connected(int P, int bw = 1);
Topology build_dgx1();
Topology build_amd_z52();
Topology build_switch(int P, int bw = 1);
// "ring:N" | "full:N" | "switch:N" | "dgx1" | "amd-z52"
Topology topology_by_name(const std::string& name);
// flip every edge, keep bounds.
Topology reverse_topology(const Topology& t);

enum class Kind { Gather, Allgather, Alltoall, Broadcast, Scatter, Reduce, Reducescatter, Allreduce };

Kind parse_kind(const std::string& s);
const char* kind_name(Kind k);
bool is_combining(Kind k);
bool is_rooted(Kind k);
int to_global(Kind k, int C, int P);

// G x P relation, [c * P + n]
using Relation = std::vector<uint8_t>;

// Non-combining kinds: (pre, post) of Table 2.
// Combining kinds: (contrib, dest) = (dual post, dual pre), i.e. the
// placement the inverted dual schedule starts from and must reduce into
// (SPEC.md:338-355).  Allreduce has no single relation (it is a composition).
void pre_post(Kind k, int G, int P, int root, Relation& pre, Relation& post);

}  // namespace sccl
