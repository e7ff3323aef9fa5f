// Schedule IR (the reference's L2 layer): the canonical
// schedule file is the drop-in boundary's input.
//   Schedule{S, Q, T}
//   verify
//   verify_combining
//   serialize / deserialize
//   invert_schedule
//   AR composition (RS, AG)
#pragma once

#include <string>
#include <vector>

#include "model.hpp"

namespace sccl {

struct Send {
  int chunk, src, dst, step;
};

struct Schedule {
  Kind kind = Kind::Allgather;
  Topology topo;  // resolved from topology.name (or inline constraints)
  bool inline_topo = false;
  int P = 0, G = 0, C = 0, S = 0, R = 0;
  int root = -1;  // rooted kinds only
  std::vector<int> rounds;  // Q
  std::vector<Send> sends;  // T, canonical order (step, chunk, src, dst)
  std::vector<Schedule> phases;  // Allreduce composition: {RS, AG}

  bool is_composition() const { return !phases.empty(); }
  // the non-composite phases, in execution order
  std::vector<const Schedule*> flat() const;
};

struct Violation {
  enum Kind { Schema = 1, Edge = 2, Unavailable = 3, Bandwidth = 4, Post = 5, Duplicate = 6, Multiplicity = 7 };
  int kind, step, chunk, src, dst;
  std::string str() const;
};

// deserialize: throws invalid_argument_error on schema violations
// (step >= S, ids out of range, G != to_global, topology hash mismatch).
Schedule parse_schedule(const std::string& json_text);
// canonical, byte-stable serialization (sends sorted by (step,chunk,src,dst))
std::string serialize(const Schedule& s);

// Semantic verification of one phase against its topology (run semantics
// PAPER.md:450-461).  Non-combining kinds -> verify, combining -> verify_combining.
std::vector<Violation> verify_phase(const Schedule& s);
// All phases of a schedule or composition.
std::vector<Violation> verify(const Schedule& s);

// T' = {(c, n', n, S-1-t)}, Q reversed, topology reversed.
// Allgather -> Reducescatter, Broadcast -> Reduce.
Schedule invert_schedule(const Schedule& s);
// Allreduce = (RS, AG) back to back; tuple (P*C_AG, 2S, 2R) for RS = invert(AG).
Schedule compose_allreduce(const Schedule& rs, const Schedule& ag);

}  // namespace sccl
