#include "layout.hpp"

#include "error.hpp"

namespace sccl {

void buffer_sizes(Kind k, int P, int64_t nbytes, int64_t& sb, int64_t& rb) {
  switch (k) {
    case Kind::Allgather:
    case Kind::Gather: sb = nbytes; rb = P * nbytes; break;
    case Kind::Reducescatter:
    case Kind::Scatter: sb = P * nbytes; rb = nbytes; break;
    default: sb = nbytes; rb = nbytes; break;
  }
}

std::vector<ChunkGeo> chunk_geometry(Kind k, int P, int G, int64_t nbytes) {
  std::vector<ChunkGeo> g(G);
  for (int c = 0; c < G; ++c) {
    switch (k) {
      case Kind::Allgather:
      case Kind::Gather: {  // chunk i*P+n = piece i of rank n's m bytes
        int n = c % P, i = c / P;
        Part p = split16(nbytes, G / P, i);
        g[c] = {p.len, p.off, n * nbytes + p.off};
        break;
      }
      case Kind::Reducescatter:
      case Kind::Scatter: {  // chunk i*P+n lands at rank n
        int n = c % P, i = c / P;
        Part p = split16(nbytes, G / P, i);
        g[c] = {p.len, n * nbytes + p.off, p.off};
        break;
      }
      case Kind::Broadcast:
      case Kind::Reduce: {
        Part p = split16(nbytes, G, c);
        g[c] = {p.len, p.off, p.off};
        break;
      }
      case Kind::Allreduce: {  // segment n of M, piece i of that segment
        int n = c % P, i = c / P;
        Part s = split16(nbytes, P, n);
        Part p = split16(s.len, G / P, i);
        g[c] = {p.len, s.off + p.off, s.off + p.off};
        break;
      }
      case Kind::Alltoall: {  // src = c%P, dst = (c/P)%P, j = c/P^2
        if (nbytes % P) throw invalid_argument_error("alltoall needs bytes % P == 0");
        int64_t seg = nbytes / P;
        int src = c % P, dst = (c / P) % P, j = c / (P * P);
        Part p = split16(seg, G / (P * P), j);
        g[c] = {p.len, dst * seg + p.off, src * seg + p.off};
        break;
      }
    }
  }
  return g;
}

}  // namespace sccl
