#include "model.hpp"

#include <algorithm>
#include <cstdio>
#include <map>

#include "error.hpp"

namespace sccl {

std::vector<uint8_t> Topology::links() const {
  std::vector<uint8_t> cov(size_t(P) * P, 0), zero(size_t(P) * P, 0);
  for (auto& c : constraints)
    for (auto& e : c.edges) {
      if (e.first < 0 || e.first >= P || e.second < 0 || e.second >= P) continue;
      cov[e.first * P + e.second] = 1;
      if (c.bound <= 0) zero[e.first * P + e.second] = 1;
    }
  for (size_t i = 0; i < cov.size(); ++i) cov[i] = cov[i] && !zero[i];
  return cov;
}

std::string Topology::hash() const {
  std::vector<std::pair<std::vector<std::pair<int, int>>, int>> cs;
  for (auto& c : constraints) {
    auto e = c.edges;
    std::sort(e.begin(), e.end());
    cs.emplace_back(std::move(e), c.bound);
  }
  std::sort(cs.begin(), cs.end());
  std::string text = std::to_string(P) + "|";
  for (size_t k = 0; k < cs.size(); ++k) {
    if (k) text += ";";
    text += std::to_string(cs[k].second) + ":";
    for (size_t j = 0; j < cs[k].first.size(); ++j) {
      if (j) text += ",";
      text += std::to_string(cs[k].first[j].first) + ">" + std::to_string(cs[k].first[j].second);
    }
  }
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char ch : text) {
    h ^= ch;
    h *= 0x100000001b3ull;
  }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  return buf;
}

static Topology pairs_topology(std::string name, int P, const std::vector<std::pair<std::pair<int, int>, int>>& eb) {
  Topology t;
  t.name = std::move(name);
  t.P = P;
  for (auto& x : eb) {
    Constraint c;
    c.edges.push_back(x.first);
    c.bound = x.second;
    t.constraints.push_back(std::move(c));
  }
  return t;
}

Topology build_ring(int P, int bw) {
  if (P < 2) throw invalid_argument_error("build_ring: P must be >= 2 (SPEC.md:56)");
  std::vector<std::pair<std::pair<int, int>, int>> eb;
  for (int i = 0; i < P; ++i) {
    std::pair<int, int> f{i, (i + 1) % P}, r{(i + 1) % P, i};
    for (auto e : {f, r}) {
      bool dup = false;
      for (auto& x : eb) dup |= x.first == e;
      if (!dup) eb.push_back({e, bw});
    }
  }
  return pairs_topology("ring:" + std::to_string(P), P, eb);
}

Topology build_fully_connected(int P, int bw) {
  if (P < 1) throw invalid_argument_error("build_fully_connected: P must be >= 1");
  std::vector<std::pair<std::pair<int, int>, int>> eb;
  for (int a = 0; a < P; ++a)
    for (int b = 0; b < P; ++b)
      if (a != b) eb.push_back({{a, b}, bw});
  return pairs_topology("full:" + std::to_string(P), P, eb);
}

Topology build_dgx1() {
  // cycle (0,1,4,5,6,7,2,3) with 2 NVLinks per edge and
  // cycle (0,2,1,3,6,4,7,5) with one.
  std::map<std::pair<int, int>, int> bw;
  const int c2[8] = {0, 1, 4, 5, 6, 7, 2, 3}, c1[8] = {0, 2, 1, 3, 6, 4, 7, 5};
  for (int i = 0; i < 8; ++i) {
    int a = c2[i], b = c2[(i + 1) % 8];
    bw[{a, b}] += 2;
    bw[{b, a}] += 2;
    a = c1[i];
    b = c1[(i + 1) % 8];
    bw[{a, b}] += 1;
    bw[{b, a}] += 1;
  }
  std::vector<std::pair<std::pair<int, int>, int>> eb(bw.begin(), bw.end());
  return pairs_topology("dgx1", 8, eb);
}

Topology build_amd_z52() {
  Topology t = build_ring(8, 1);  // SPEC.md:94 design decision: ring order 0..7
  t.name = "amd-z52";
  return t;
}

Topology build_switch(int P, int bw) {
  if (P < 1) throw invalid_argument_error("build_switch: P must be >= 1");
  Topology t;
  t.name = "switch:" + std::to_string(P);
  t.P = P;
  for (int n = 0; n < P; ++n) {  // egress group of GPU n
    Constraint c;
    c.bound = bw;
    for (int d = 0; d < P; ++d)
      if (d != n) c.edges.push_back({n, d});
    t.constraints.push_back(std::move(c));
  }
  for (int n = 0; n < P; ++n) {  // ingress group of GPU n
    Constraint c;
    c.bound = bw;
    for (int s = 0; s < P; ++s)
      if (s != n) c.edges.push_back({s, n});
    t.constraints.push_back(std::move(c));
  }
  return t;
}

Topology topology_by_name(const std::string& name) {
  if (name == "dgx1") return build_dgx1();
  if (name == "amd-z52") return build_amd_z52();
  auto colon = name.find(':');
  if (colon == std::string::npos) throw invalid_argument_error("unknown topology '" + name + "'");
  std::string k = name.substr(0, colon);
  int P = 0;
  try {
    P = std::stoi(name.substr(colon + 1));
  } catch (...) {
    throw invalid_argument_error("bad topology size in '" + name + "'");
  }
  if (P < 1 || P > 64) throw invalid_argument_error("topology size out of range in '" + name + "'");
  if (k == "ring") return build_ring(P);
  if (k == "full") return build_fully_connected(P);
  if (k == "switch") return build_switch(P);
  throw invalid_argument_error("unknown topology '" + name + "'");
}

Topology reverse_topology(const Topology& t) {
  Topology r = t;
  for (auto& c : r.constraints)
    for (auto& e : c.edges) std::swap(e.first, e.second);
  return r;
}

static const char* kNames[] = {"gather", "allgather", "alltoall", "broadcast",
                               "scatter", "reduce", "reducescatter", "allreduce"};

Kind parse_kind(const std::string& s) {
  for (int i = 0; i < 8; ++i)
    if (s == kNames[i]) return Kind(i);
  throw invalid_argument_error("unknown collective '" + s + "'");
}
const char* kind_name(Kind k) { return kNames[int(k)]; }
bool is_combining(Kind k) { return k == Kind::Reduce || k == Kind::Reducescatter || k == Kind::Allreduce; }
bool is_rooted(Kind k) {
  return k == Kind::Gather || k == Kind::Broadcast || k == Kind::Scatter || k == Kind::Reduce;
}

int to_global(Kind k, int C, int P) {
  if (C < 1) throw invalid_argument_error("to_global: C must be >= 1");
  if (k == Kind::Broadcast || k == Kind::Reduce) return C;
  if (k == Kind::Alltoall && C % P) throw invalid_argument_error("to_global: Alltoall needs C mod P == 0");
  return P * C;
}

enum class Rel { All, Root, Scattered, Transpose };

static Relation relation(Rel r, int G, int P, int root) {
  Relation m(size_t(G) * P, 0);
  for (int c = 0; c < G; ++c) switch (r) {
      case Rel::All:
        for (int n = 0; n < P; ++n) m[c * P + n] = 1;
        break;
      case Rel::Root: m[c * P + root] = 1; break;
      case Rel::Scattered:
        if (G % P) throw invalid_argument_error("Scattered relation needs G mod P == 0 (SPEC.md:146)");
        m[c * P + c % P] = 1;
        break;
      case Rel::Transpose:
        if (G % (P * P)) throw invalid_argument_error("Transpose relation needs G mod P^2 == 0 (SPEC.md:156)");
        m[c * P + (c / P) % P] = 1;
        break;
    }
  return m;
}

void pre_post(Kind k, int G, int P, int root, Relation& pre, Relation& post) {
  if (is_rooted(k) && (root < 0 || root >= P)) throw invalid_argument_error("root out of range");
  Rel a = Rel::All, b = Rel::All;
  switch (k) {
    case Kind::Gather: a = Rel::Scattered; b = Rel::Root; break;
    case Kind::Allgather: a = Rel::Scattered; b = Rel::All; break;
    case Kind::Alltoall: a = Rel::Scattered; b = Rel::Transpose; break;
    case Kind::Broadcast: a = Rel::Root; b = Rel::All; break;
    case Kind::Scatter: a = Rel::Root; b = Rel::Scattered; break;
    case Kind::Reduce: a = Rel::All; b = Rel::Root; break;             // dual Broadcast inverted
    case Kind::Reducescatter: a = Rel::All; b = Rel::Scattered; break;  // dual Allgather inverted
    case Kind::Allreduce: throw invalid_argument_error("allreduce is a composition (RS, AG); no single relation");
  }
  pre = relation(a, G, P, root);
  post = relation(b, G, P, root);
}

}  // namespace sccl
