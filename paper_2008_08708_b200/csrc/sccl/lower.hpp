// Lowering: synthesized step schedule -> per-rank channel program.
//
// The reference's GPU lowering exists only as prose (a
// per-GPU program of what/where/when/with-reduce commands, CUDA-IPC push,
// one fused kernel with a flag per (chunk, connection)).  This pass turns a
// verified Schedule (or RS;AG composition) into, for every rank, an ordered
// list of Ops.  Every chunk is split into `nch` channel sub-ranges; CTA
// (rank, ch) executes the rank's op list restricted to sub-range ch, so
// program order inside one CTA replaces all intra-rank synchronisation and
// only cross-rank receipts carry flags.
//
// Memory spaces per rank: SEND (caller input, read only), RECV (caller
// output / registered buffer), SCRATCH (plan-owned: relay copies and
// combining receipt slots), FLAGS (plan-owned counters).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "layout.hpp"
#include "schedule.hpp"

namespace sccl {

enum Space : int { SP_SEND = 0, SP_RECV = 1, SP_SCRATCH = 2, SP_FLAGS = 3, NSPACE = 4 };

struct Loc {
  int rank = -1, space = -1;
  int64_t off = 0;
  int chunk = -1;  // owner chunk: zero-length chunks share offsets, so identity includes it
  bool operator==(const Loc& o) const {
    return rank == o.rank && space == o.space && off == o.off && chunk == o.chunk;
  }
};

struct OpIn {
  Loc loc;
  int flag = -1;  // receipt slot at loc.rank whose counter gates this input, or -1
  int64_t len = 0;
  int chunk = -1;
  bool operator==(const OpIn& o) const { return loc == o.loc && flag == o.flag && len == o.len; }
};

struct OpOut {
  Loc loc;
  int flag = -1;            // receipt slot at loc.rank to signal, or -1
  bool every_tile = false;  // signal per tile (consumer forwards) or only at the end
};

enum OpKind : int { OP_COPY = 0, OP_REDUCE = 1, OP_WAIT = 2 };

struct Op {
  int kind = OP_COPY;
  int key = 0;       // ordering key: 2*step (sends), 2*step+1 (reduces)
  int chunk = -1;
  int64_t len = 0;   // chunk bytes (all ins/outs)
  std::vector<OpIn> ins;    // REDUCE: ins[0] is the base, then receipts by src
  std::vector<OpOut> outs;
};

struct RankProgram {
  std::vector<Op> ops;
  int nslots = 0;           // receipt slots (flags) at this rank
  int64_t scratch_bytes = 0;
};

struct Program {
  Kind kind;
  int P = 0, G = 0;
  int64_t nbytes = 0, send_bytes = 0, recv_bytes = 0;
  int esize = 1;
  std::vector<ChunkGeo> geo;
  std::vector<RankProgram> ranks;
  int max_slots = 0;
  int64_t scratch_bytes = 0;  // symmetric per-rank scratch size
  bool ll = false;            // low-latency protocol: every receipt is an LL slot in scratch
  bool pull = false;          // combining sends of untouched inputs are read in place by the receiver
  std::string fingerprint;    // hash of (canonical schedule, sizes, dtype, protocol)

  std::string summary_json() const;
};

// Throws invalid_argument_error for unverified schedules or
// inconsistent sizes.  ll = low-latency protocol: every receipt lands in a
// scratch slot encoded as (4 data bytes, 4 flag bytes) words (2x the chunk),
// so the receiver polls the data itself; post entries then get a local
// unpacking copy, fused with the forward of the same receipt.
//
// pull = combining sends whose sender still holds its untouched input (the
// one-shot reduce-scatter, the first hop of every reduction chain) become
// reads of the sender's SEND buffer by the receiver's REDUCE: no receipt
// slot in scratch, no copy op, no flag.  Same reduction order and operands,
// so the same bits.  Only where every rank's SEND is addressable and
// unchanged for the whole launch (loopback).
Program lower(const Schedule& s, int64_t nbytes, int esize, bool ll = false, bool pull = false);

// bytes of an LL slot for a chunk of len bytes
inline int64_t ll_bytes(int64_t len) { return 2 * ((len + 15) / 16 * 16); }

}  // namespace sccl
