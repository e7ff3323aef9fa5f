// Chunk-id -> buffer-offset map (derived from
// SPEC.md:147-173, 191) and the 16-byte-aligned chunk split (Appendix A8).
// The CPU oracle (oracle/oracle.py chunk_geometry) restates the same rules
// independently; GPU parity tests compare the two through whole buffers.
#pragma once

#include <cstdint>
#include <vector>

#include "model.hpp"

namespace sccl {

struct Part {
  int64_t off, len;
};

// Part i of K of an L-byte range: starts at multiples of 16, remainder in
// the last part.
inline Part split16(int64_t L, int64_t K, int64_t i) {
  int64_t U = L / 16;
  int64_t lo = (i * U / K) * 16;
  int64_t hi = (i == K - 1) ? L : ((i + 1) * U / K) * 16;
  return {lo, hi - lo};
}

struct ChunkGeo {
  int64_t len;      // bytes
  int64_t in_off;   // offset in the send buffer of every rank that holds it there
  int64_t out_off;  // offset in the recv buffer of every rank that holds it there
};

// (send bytes, recv bytes) per rank for the per-rank size argument
// (NCCL conventions: allgather/gather in = m, out = P*m; reducescatter /
// scatter in = P*m, out = m; others in = out = M).
void buffer_sizes(Kind k, int P, int64_t nbytes, int64_t& send_bytes, int64_t& recv_bytes);

// Geometry of all G chunks for the top-level collective (for an allreduce
// composition: Kind::Allreduce with G = P*C_AG).
std::vector<ChunkGeo> chunk_geometry(Kind k, int P, int G, int64_t nbytes);

}  // namespace sccl
