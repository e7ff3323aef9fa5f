#include "schedule.hpp"

#include <algorithm>
#include <sstream>
#include <tuple>

#include "error.hpp"
#include "json.hpp"

namespace sccl {

static const int kVersion = 1;

std::vector<const Schedule*> Schedule::flat() const {
  std::vector<const Schedule*> v;
  if (phases.empty()) v.push_back(this);
  else
    for (auto& p : phases) v.push_back(&p);
  return v;
}

std::string Violation::str() const {
  static const char* names[] = {"?", "schema", "edge", "unavailable", "bandwidth", "post", "duplicate", "multiplicity"};
  std::ostringstream o;
  o << names[(kind >= 1 && kind <= 7) ? kind : 0] << "(step=" << step << ",chunk=" << chunk << ",src=" << src
    << ",dst=" << dst << ")";
  return o.str();
}

static void canonical_sort(std::vector<Send>& v) {
  std::sort(v.begin(), v.end(), [](const Send& a, const Send& b) {
    return std::tie(a.step, a.chunk, a.src, a.dst) < std::tie(b.step, b.chunk, b.src, b.dst);
  });
}

// ---------------------------------------------------------------------------
// deserialize
// ---------------------------------------------------------------------------
static Topology parse_topology(const json::Value& tv, int P) {
  const std::string& name = tv.at("name").as_str("topology.name");
  Topology t;
  if (const json::Value* cons = tv.find("constraints")) {
    if (cons->type != json::Value::Array) throw invalid_argument_error("topology.constraints must be an array");
    t.name = name;
    t.P = P;
    for (auto& cv : cons->arr) {
      Constraint c;
      c.bound = int(cv.at("bound").as_int("bound"));
      if (c.bound < 0) throw invalid_argument_error("constraint bound must be >= 0");
      for (auto& ev : cv.at("edges").arr) {
        if (ev.type != json::Value::Array || ev.arr.size() != 2) throw invalid_argument_error("edge must be [src,dst]");
        int a = int(ev.arr[0].as_int("edge")), b = int(ev.arr[1].as_int("edge"));
        if (a < 0 || a >= P || b < 0 || b >= P) throw invalid_argument_error("edge node id out of range");
        c.edges.push_back({a, b});
      }
      if (c.edges.empty()) throw invalid_argument_error("constraint with empty edge set (SPEC.md:27)");
      t.constraints.push_back(std::move(c));
    }
  } else {
    t = topology_by_name(name);
  }
  if (const json::Value* h = tv.find("hash")) {
    if (h->type == json::Value::String && !h->s.empty() && h->s != t.hash())
      throw invalid_argument_error("topology hash mismatch for '" + name + "': file " + h->s + ", rebuilt " + t.hash());
  }
  return t;
}

static Schedule parse_obj(const json::Value& v, int depth) {
  if (v.type != json::Value::Object) throw invalid_argument_error("schedule must be a JSON object");
  Schedule s;
  s.kind = parse_kind(v.at("collective").as_str("collective"));
  if (const json::Value* ver = v.find("version"))
    if (ver->as_int("version") != kVersion) throw invalid_argument_error("unsupported schedule version");
  s.P = int(v.at("P").as_int("P"));
  if (s.P < 1 || s.P > 64) throw invalid_argument_error("P out of range [1,64]");
  const json::Value& tv = v.at("topology");
  s.inline_topo = tv.find("constraints") != nullptr;
  s.topo = parse_topology(tv, s.P);
  if (s.topo.P != s.P) throw invalid_argument_error("topology node count != P");
  s.G = int(v.at("G").as_int("G"));
  s.C = int(v.at("C").as_int("C"));
  s.S = int(v.at("S").as_int("S"));
  s.R = int(v.at("R").as_int("R"));
  if (const json::Value* r = v.find("root"))
    if (r->type != json::Value::Null) s.root = int(r->as_int("root"));
  if (is_rooted(s.kind)) {
    if (s.root < 0) s.root = 0;  // SPEC.md:190 default root 0
    if (s.root >= s.P) throw invalid_argument_error("root out of range");
  }

  if (const json::Value* ph = v.find("phases")) {
    if (depth > 0 || s.kind != Kind::Allreduce) throw invalid_argument_error("only allreduce may have phases");
    if (ph->type != json::Value::Array || ph->arr.size() != 2)
      throw invalid_argument_error("allreduce needs exactly two phases (RS, AG)");
    Schedule rs = parse_obj(ph->arr[0], depth + 1);
    Schedule ag = parse_obj(ph->arr[1], depth + 1);
    Schedule c = compose_allreduce(rs, ag);
    if (c.G != s.G || c.C != s.C || c.S != s.S || c.R != s.R || c.P != s.P)
      throw invalid_argument_error("allreduce header (G,C,S,R) disagrees with its phases");
    c.topo = s.topo;
    c.inline_topo = s.inline_topo;
    return c;
  }
  if (s.kind == Kind::Allreduce) throw invalid_argument_error("allreduce must be given as phases [RS, AG]");

  if (s.G < 1 || s.S < 1 || s.C < 1) throw invalid_argument_error("G, C, S must be >= 1");
  if (s.G != to_global(s.kind, s.C, s.P)) throw invalid_argument_error("G != to_global(collective, C, P) (SPEC.md:165)");
  const json::Value& rv = v.at("rounds");
  if (rv.type != json::Value::Array || int(rv.arr.size()) != s.S)
    throw invalid_argument_error("rounds must have S entries");
  int sum = 0;
  for (auto& x : rv.arr) {
    int r = int(x.as_int("rounds[]"));
    if (r < 1) throw invalid_argument_error("every step needs >= 1 round (SPEC.md:386)");
    s.rounds.push_back(r);
    sum += r;
  }
  if (sum != s.R) throw invalid_argument_error("sum(rounds) != R");
  const json::Value& sv = v.at("sends");
  if (sv.type != json::Value::Array) throw invalid_argument_error("sends must be an array");
  for (auto& x : sv.arr) {
    if (x.type != json::Value::Array || x.arr.size() != 4)
      throw invalid_argument_error("send must be [chunk,src,dst,step]");
    Send t{int(x.arr[0].as_int("chunk")), int(x.arr[1].as_int("src")), int(x.arr[2].as_int("dst")),
           int(x.arr[3].as_int("step"))};
    if (t.chunk < 0 || t.chunk >= s.G) throw invalid_argument_error("send chunk out of range");
    if (t.src < 0 || t.src >= s.P || t.dst < 0 || t.dst >= s.P) throw invalid_argument_error("send node out of range");
    if (t.src == t.dst) throw invalid_argument_error("send with src == dst");
    if (t.step < 0 || t.step >= s.S) throw invalid_argument_error("send step >= S (SPEC.md:435)");
    s.sends.push_back(t);
  }
  canonical_sort(s.sends);
  return s;
}

Schedule parse_schedule(const std::string& text) { return parse_obj(json::parse(text), 0); }

// ---------------------------------------------------------------------------
// serialize
// ---------------------------------------------------------------------------
static void write_topology(std::ostringstream& o, const Schedule& s) {
  o << "\"topology\":{\"name\":\"" << s.topo.name << "\",\"hash\":\"" << s.topo.hash() << "\"";
  if (s.inline_topo) {
    o << ",\"constraints\":[";
    for (size_t k = 0; k < s.topo.constraints.size(); ++k) {
      auto& c = s.topo.constraints[k];
      o << (k ? "," : "") << "{\"edges\":[";
      for (size_t j = 0; j < c.edges.size(); ++j)
        o << (j ? "," : "") << "[" << c.edges[j].first << "," << c.edges[j].second << "]";
      o << "],\"bound\":" << c.bound << "}";
    }
    o << "]";
  }
  o << "}";
}

static void write_obj(std::ostringstream& o, const Schedule& s) {
  o << "{\"collective\":\"" << kind_name(s.kind) << "\",\"version\":" << kVersion << ",";
  write_topology(o, s);
  o << ",\"P\":" << s.P << ",\"G\":" << s.G << ",\"C\":" << s.C << ",\"S\":" << s.S << ",\"R\":" << s.R;
  if (is_rooted(s.kind)) o << ",\"root\":" << s.root;
  if (s.is_composition()) {
    o << ",\"phases\":[";
    write_obj(o, s.phases[0]);
    o << ",";
    write_obj(o, s.phases[1]);
    o << "]}";
    return;
  }
  o << ",\"rounds\":[";
  for (size_t i = 0; i < s.rounds.size(); ++i) o << (i ? "," : "") << s.rounds[i];
  o << "],\"sends\":[";
  std::vector<Send> v = s.sends;
  canonical_sort(v);
  for (size_t i = 0; i < v.size(); ++i)
    o << (i ? "," : "") << "[" << v[i].chunk << "," << v[i].src << "," << v[i].dst << "," << v[i].step << "]";
  o << "]}";
}

std::string serialize(const Schedule& s) {
  std::ostringstream o;
  write_obj(o, s);
  return o.str();
}

// ---------------------------------------------------------------------------
// verify / verify_combining
// ---------------------------------------------------------------------------
static void check_bandwidth(const Schedule& s, const std::vector<uint8_t>& ok, std::vector<Violation>& out) {
  const int P = s.P;
  std::vector<int> cnt(size_t(P) * P);
  for (int st = 0; st < s.S; ++st) {
    std::fill(cnt.begin(), cnt.end(), 0);
    for (size_t i = 0; i < s.sends.size(); ++i)
      if (ok[i] && s.sends[i].step == st) cnt[s.sends[i].src * P + s.sends[i].dst]++;
    for (auto& c : s.topo.constraints) {
      long tot = 0;
      for (auto& e : c.edges) tot += cnt[e.first * P + e.second];
      if (tot > long(c.bound) * s.rounds[st])
        out.push_back({Violation::Bandwidth, st, -1, c.edges[0].first, c.edges[0].second});
    }
  }
}

static std::vector<uint8_t> check_schema(const Schedule& s, std::vector<Violation>& out) {
  auto links = s.topo.links();
  std::vector<uint8_t> ok(s.sends.size(), 1);
  for (size_t i = 0; i < s.sends.size(); ++i) {
    const Send& t = s.sends[i];
    if (!links[t.src * s.P + t.dst]) {
      out.push_back({Violation::Edge, t.step, t.chunk, t.src, t.dst});
      ok[i] = 0;
    }
  }
  return ok;
}

static std::vector<Violation> verify_plain(const Schedule& s) {
  std::vector<Violation> out;
  auto ok = check_schema(s, out);
  Relation pre, post;
  pre_post(s.kind, s.G, s.P, s.root, pre, post);
  const int P = s.P;
  std::vector<uint8_t> V = pre, Vn;
  for (int st = 0; st < s.S; ++st) {
    Vn = V;
    for (size_t i = 0; i < s.sends.size(); ++i) {
      const Send& t = s.sends[i];
      if (!ok[i] || t.step != st) continue;
      if (!V[t.chunk * P + t.src]) {
        out.push_back({Violation::Unavailable, st, t.chunk, t.src, t.dst});
        continue;
      }
      if (Vn[t.chunk * P + t.dst]) {
        out.push_back({Violation::Duplicate, st, t.chunk, t.src, t.dst});
        continue;
      }
      Vn[t.chunk * P + t.dst] = 1;
    }
    V.swap(Vn);
  }
  for (int c = 0; c < s.G; ++c)
    for (int n = 0; n < P; ++n)
      if (post[c * P + n] && !V[c * P + n]) out.push_back({Violation::Post, s.S, c, -1, n});
  check_bandwidth(s, ok, out);
  return out;
}

static std::vector<Violation> verify_comb(const Schedule& s) {
  std::vector<Violation> out;
  auto ok = check_schema(s, out);
  Relation contrib, dest;
  pre_post(s.kind, s.G, s.P, s.root, contrib, dest);
  const int P = s.P;
  // contribution multisets per (chunk, node): counts[(c*P+n)*P+p]
  std::vector<uint16_t> ms(size_t(s.G) * P * P, 0), mn;
  for (int c = 0; c < s.G; ++c)
    for (int n = 0; n < P; ++n)
      if (contrib[c * P + n]) ms[(size_t(c) * P + n) * P + n] = 1;
  for (int st = 0; st < s.S; ++st) {
    mn = ms;
    for (size_t i = 0; i < s.sends.size(); ++i) {
      const Send& t = s.sends[i];
      if (!ok[i] || t.step != st) continue;
      const uint16_t* from = &ms[(size_t(t.chunk) * P + t.src) * P];
      uint16_t* to = &mn[(size_t(t.chunk) * P + t.dst) * P];
      bool any = false;
      for (int p = 0; p < P; ++p) any |= from[p] != 0;
      if (!any) {
        out.push_back({Violation::Unavailable, st, t.chunk, t.src, t.dst});
        continue;
      }
      for (int p = 0; p < P; ++p) to[p] = uint16_t(std::min(65535, int(to[p]) + from[p]));
    }
    ms.swap(mn);
  }
  for (int c = 0; c < s.G; ++c)
    for (int n = 0; n < P; ++n) {
      if (!dest[c * P + n]) continue;
      const uint16_t* m = &ms[(size_t(c) * P + n) * P];
      for (int p = 0; p < P; ++p)
        if (m[p] != (contrib[c * P + p] ? 1 : 0)) {
          out.push_back({Violation::Multiplicity, s.S, c, p, n});
          break;
        }
    }
  check_bandwidth(s, ok, out);
  return out;
}

std::vector<Violation> verify_phase(const Schedule& s) {
  if (s.is_composition()) throw invalid_argument_error("verify_phase on a composition");
  return is_combining(s.kind) ? verify_comb(s) : verify_plain(s);
}

std::vector<Violation> verify(const Schedule& s) {
  std::vector<Violation> all;
  for (const Schedule* p : s.flat()) {
    auto v = verify_phase(*p);
    all.insert(all.end(), v.begin(), v.end());
  }
  return all;
}

// ---------------------------------------------------------------------------
// inversion and composition
// ---------------------------------------------------------------------------
Schedule invert_schedule(const Schedule& s) {
  if (s.is_composition()) throw invalid_argument_error("cannot invert a composition");
  Schedule r = s;
  if (s.kind == Kind::Allgather) r.kind = Kind::Reducescatter;
  else if (s.kind == Kind::Broadcast) r.kind = Kind::Reduce;
  else if (s.kind == Kind::Reducescatter) r.kind = Kind::Allgather;  // involution
  else if (s.kind == Kind::Reduce) r.kind = Kind::Broadcast;
  else throw invalid_argument_error(std::string("no combining dual for ") + kind_name(s.kind));
  r.topo = reverse_topology(s.topo);
  if (r.topo.hash() == s.topo.hash()) r.topo.name = s.topo.name;
  else if (!s.inline_topo) {
    r.inline_topo = true;
    r.topo.name = s.topo.name + "-reversed";
  }
  std::reverse(r.rounds.begin(), r.rounds.end());
  for (auto& t : r.sends) {
    std::swap(t.src, t.dst);
    t.step = s.S - 1 - t.step;
  }
  canonical_sort(r.sends);
  return r;
}

Schedule compose_allreduce(const Schedule& rs, const Schedule& ag) {
  if (rs.kind != Kind::Reducescatter || ag.kind != Kind::Allgather)
    throw invalid_argument_error("allreduce composition needs (reducescatter, allgather)");
  if (rs.P != ag.P || rs.G != ag.G) throw invalid_argument_error("allreduce phases disagree on P or G");
  Schedule c;
  c.kind = Kind::Allreduce;
  c.topo = ag.topo;
  c.inline_topo = ag.inline_topo;
  c.P = ag.P;
  c.G = ag.G;
  c.C = ag.P * ag.C;  // (P*C, 2S, 2R) for RS = invert(AG)
  c.S = rs.S + ag.S;
  c.R = rs.R + ag.R;
  c.phases = {rs, ag};
  return c;
}

}  // namespace sccl
