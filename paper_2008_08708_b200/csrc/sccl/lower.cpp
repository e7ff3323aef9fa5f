#include "lower.hpp"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <map>
#include <sstream>

#include "error.hpp"

namespace sccl {

namespace {

struct Cur {
  Loc loc;
  int flag = -1;
  bool valid = false;
};

struct Builder {
  const Schedule& s;
  Program& pg;
  std::vector<Cur> cur;  // [c*P+n]

  Builder(const Schedule& sch, Program& p) : s(sch), pg(p) {}

  int64_t scratch_alloc(int rank, int64_t len) {
    int64_t& top = pg.ranks[rank].scratch_bytes;
    int64_t off = top;
    top += (len + 255) / 256 * 256;
    return off;
  }
  int new_slot(int rank) { return pg.ranks[rank].nslots++; }
  Loc out_loc(int c, int n) const { return {n, SP_RECV, pg.geo[c].out_off, c}; }
  Loc in_loc(int c, int n) const { return {n, SP_SEND, pg.geo[c].in_off, c}; }

  void add_copy(int rank, int key, int c, const Cur& src, Loc dst, int slot) {
    Op op;
    op.kind = OP_COPY;
    op.key = key;
    op.chunk = c;
    op.len = pg.geo[c].len;
    op.ins.push_back({src.loc, src.flag, op.len, c});
    op.outs.push_back({dst, slot, false});
    pg.ranks[rank].ops.push_back(std::move(op));
  }
};

bool writes_loc(const Op& op, const Loc& L) {
  for (auto& o : op.outs)
    if (o.loc == L) return true;
  return false;
}

}  // namespace

Program lower(const Schedule& s, int64_t nbytes, int esize, bool ll, bool pull) {
  auto viol = verify(s);
  if (!viol.empty())
    throw invalid_argument_error("executing an unverified schedule is rejected (SPEC.md:420): " + viol[0].str() +
                                 (viol.size() > 1 ? " (+" + std::to_string(viol.size() - 1) + " more)" : ""));
  if (nbytes < 0) throw invalid_argument_error("negative size");
  if (esize < 1 || nbytes % esize) throw invalid_argument_error("bytes_per_rank must be a multiple of the element size");
  const int P = s.P;
  auto phases = s.flat();
  const int G = phases.back()->G;
  for (auto* ph : phases)
    if (ph->G != G || ph->P != P) throw invalid_argument_error("phases disagree on G or P");
  if (s.kind == Kind::Alltoall && (nbytes % P || (nbytes / P) % esize))
    throw invalid_argument_error("alltoall needs bytes_per_rank divisible by P * element size");

  Program pg;
  pg.ll = ll;
  pg.pull = pull;
  pg.kind = s.kind;
  pg.P = P;
  pg.G = G;
  pg.nbytes = nbytes;
  pg.esize = esize;
  buffer_sizes(s.kind, P, nbytes, pg.send_bytes, pg.recv_bytes);
  pg.geo = chunk_geometry(s.kind, P, G, nbytes);
  pg.ranks.resize(P);

  Builder b(s, pg);
  b.cur.assign(size_t(G) * P, Cur{});
  const int root = s.root >= 0 ? s.root : (phases[0]->root >= 0 ? phases[0]->root : 0);
  Relation fpre, fpost;
  pre_post(phases.back()->kind, G, P, root, fpre, fpost);
  std::vector<int64_t> acc_scratch_off(size_t(G) * P, -1);

  int step_base = 0;
  for (size_t k = 0; k < phases.size(); ++k) {
    const Schedule& ph = *phases[k];
    const bool last = k + 1 == phases.size();
    Relation pre, post;
    pre_post(ph.kind, G, P, root, pre, post);
    for (int c = 0; c < G; ++c)
      for (int n = 0; n < P; ++n) {
        Cur& x = b.cur[c * P + n];
        if (k == 0) {
          if (pre[c * P + n]) x = {b.in_loc(c, n), -1, true};
        } else if (!pre[c * P + n]) {
          x.valid = false;  // composition: the next phase starts from its own pre
        }
      }

    if (!is_combining(ph.kind)) {
      for (int st = 0; st < ph.S; ++st) {
        struct Upd {
          int c, n;
          Loc loc;
          int slot;
        };
        std::vector<Upd> upd;
        for (auto& t : ph.sends) {
          if (t.step != st) continue;
          const Cur& src = b.cur[t.chunk * P + t.src];
          if (!src.valid) throw invalid_argument_error("internal: sender lacks chunk after verification");
          Loc dst;
          const int64_t len = pg.geo[t.chunk].len;
          if (!ll && last && fpost[t.chunk * P + t.dst]) dst = b.out_loc(t.chunk, t.dst);
          else dst = {t.dst, SP_SCRATCH, b.scratch_alloc(t.dst, ll ? ll_bytes(len) : len), t.chunk};
          int slot = b.new_slot(t.dst);
          b.add_copy(t.src, 2 * (step_base + st), t.chunk, src, dst, slot);
          upd.push_back({t.chunk, t.dst, dst, slot});
        }
        for (auto& u : upd) b.cur[u.c * P + u.n] = {u.loc, u.slot, true};
      }
    } else {
      // nodes that receive a contribution of chunk c in this phase reduce
      // it into their accumulator (RECV, which an in-place caller aliases
      // with SEND): their input is pulled only if they never do, so no
      // reader can race the owner's own write
      std::vector<uint8_t> receives(size_t(G) * P, 0);
      for (auto& t : ph.sends) receives[size_t(t.chunk) * P + t.dst] = 1;
      for (int st = 0; st < ph.S; ++st) {
        struct Rc {
          int src, slot;
          Loc loc;
        };
        std::map<std::pair<int, int>, std::vector<Rc>> recv;  // (dst, chunk) -> receipts
        for (auto& t : ph.sends) {
          if (t.step != st) continue;
          const Cur& src = b.cur[t.chunk * P + t.src];
          if (!src.valid) throw invalid_argument_error("internal: sender holds no contribution after verification");
          if (pull && src.loc.space == SP_SEND && src.flag < 0 && !receives[size_t(t.chunk) * P + t.src]) {
            // pull: the sender's value at V_s is its untouched input, so the
            // receiver's reduce reads it in place (no receipt slot, no copy)
            recv[{t.dst, t.chunk}].push_back({t.src, -1, src.loc});
            continue;
          }
          const int64_t len = pg.geo[t.chunk].len;
          Loc dst{t.dst, SP_SCRATCH, b.scratch_alloc(t.dst, ll ? ll_bytes(len) : len), t.chunk};
          int slot = b.new_slot(t.dst);
          b.add_copy(t.src, 2 * (step_base + st), t.chunk, src, dst, slot);
          recv[{t.dst, t.chunk}].push_back({t.src, slot, dst});
        }
        for (auto& kv : recv) {
          int n = kv.first.first, c = kv.first.second;
          auto rs = kv.second;
          std::sort(rs.begin(), rs.end(), [](const Rc& a, const Rc& z) { return a.src < z.src; });
          Op op;
          op.kind = OP_REDUCE;
          op.key = 2 * (step_base + st) + 1;
          op.chunk = c;
          op.len = pg.geo[c].len;
          Cur& x = b.cur[c * P + n];
          if (x.valid) op.ins.push_back({x.loc, x.flag, op.len, c});
          for (auto& r : rs) op.ins.push_back({r.loc, r.slot, op.len, c});
          Loc acc;
          if (s.kind == Kind::Allreduce || post[c * P + n]) {
            acc = b.out_loc(c, n);
          } else {
            int64_t& off = acc_scratch_off[c * P + n];
            if (off < 0) off = b.scratch_alloc(n, op.len);
            acc = {n, SP_SCRATCH, off, c};
          }
          op.outs.push_back({acc, -1, false});
          pg.ranks[n].ops.push_back(std::move(op));
          x = {acc, -1, true};
        }
      }
    }
    step_base += ph.S;
  }

  // every post entry must end in its output location (local copy otherwise)
  for (int c = 0; c < G; ++c)
    for (int n = 0; n < P; ++n) {
      if (!fpost[c * P + n]) continue;
      const Cur& x = b.cur[c * P + n];
      if (!x.valid) throw invalid_argument_error("internal: post entry unresolved");
      Loc o = b.out_loc(c, n);
      if (x.loc == o) continue;
      int key = INT_MAX;
      for (auto& op : pg.ranks[n].ops)
        if (op.kind == OP_COPY && op.ins.size() == 1 && op.ins[0].loc == x.loc && op.ins[0].flag == x.flag)
          key = std::min(key, op.key);
      if (key == INT_MAX) key = 2 * step_base;
      b.add_copy(n, key, c, x, o, -1);
    }

  // within a step ops keep the canonical (step, chunk, src, dst) order;
  // SCCL_SEND_ORDER=rotate starts rank r's sends at r+1 (measured on B200:
  // -1 % at 128 MiB allgather, +4..10 % at 1-16 MiB multi-hop; off by default)
  const char* order_env = std::getenv("SCCL_SEND_ORDER");
  const bool canonical_order = !(order_env && std::string(order_env) == "rotate");
  for (int r = 0; r < P; ++r) {
    auto& ops = pg.ranks[r].ops;
    std::stable_sort(ops.begin(), ops.end(), [](const Op& a, const Op& z) { return a.key < z.key; });

    // F1: copies of one input at one key -> one op with several outputs
    std::vector<Op> merged;
    for (auto& op : ops) {
      bool done = false;
      if (op.kind == OP_COPY)
        for (auto& m : merged)
          if (m.kind == OP_COPY && m.key == op.key && m.ins == op.ins) {
            m.outs.insert(m.outs.end(), op.outs.begin(), op.outs.end());
            done = true;
            break;
          }
      if (!done) merged.push_back(std::move(op));
    }
    ops.swap(merged);

    // optional rotation: rank r sends to r+1 first, then r+2, ...
    auto dist = [&](const Op& op) {
      int d = P;
      for (auto& o : op.outs)
        if (o.loc.rank != r) d = std::min(d, (o.loc.rank - r + P) % P);
      return d;
    };
    if (!canonical_order)
      std::stable_sort(ops.begin(), ops.end(),
                       [&](const Op& a, const Op& z) { return a.key != z.key ? a.key < z.key : dist(a) < dist(z); });

    // F2: fold copies that read a reduce's result into the reduce (fused
    // receive-reduce-forward, "reduce on receipt")
    for (size_t i = 0; i < ops.size(); ++i) {
      if (ops[i].kind != OP_REDUCE) continue;
      Loc L = ops[i].outs[0].loc;
      for (size_t j = i + 1; j < ops.size();) {
        Op& y = ops[j];
        if (y.kind == OP_COPY && y.ins.size() == 1 && y.ins[0].loc == L && y.ins[0].flag == -1) {
          bool clean = true;
          for (size_t q = i + 1; q < j; ++q) clean &= !writes_loc(ops[q], L);
          if (clean) {
            ops[i].outs.insert(ops[i].outs.end(), y.outs.begin(), y.outs.end());
            ops.erase(ops.begin() + j);
            continue;
          }
        }
        if (writes_loc(y, L)) break;
        ++j;
      }
    }

    // dead accumulator stores: a reduce result nobody reads locally and
    // that is not the rank's final value (e.g. an allreduce partial that the
    // allgather phase overwrites)
    for (size_t i = 0; i < ops.size(); ++i) {
      if (ops[i].kind != OP_REDUCE || ops[i].outs.size() < 2) continue;
      Loc L = ops[i].outs[0].loc;
      int c = ops[i].chunk;
      bool read = false;
      for (size_t j = i + 1; j < ops.size() && !read; ++j) {
        for (auto& in : ops[j].ins) read |= in.loc == L && in.flag == -1;
        if (writes_loc(ops[j], L)) break;
      }
      const Cur& fin = b.cur[c * P + r];
      bool final_here = fpost[c * P + r] && fin.valid && fin.loc == L && fin.flag == -1;
      if (!read && !final_here) ops[i].outs.erase(ops[i].outs.begin());
    }
  }

  // signal modes and end-of-program waits (every receipt must have landed
  // before the rank's kernel exits)
  for (int d = 0; d < P; ++d) {
    std::vector<uint8_t> consumed(pg.ranks[d].nslots, 0);
    for (auto& op : pg.ranks[d].ops)
      for (auto& in : op.ins)
        if (in.flag >= 0) consumed[in.flag] = 1;
    for (int r = 0; r < P; ++r)
      for (auto& op : pg.ranks[r].ops)
        for (auto& o : op.outs)
          if (o.flag >= 0 && o.loc.rank == d) o.every_tile = consumed[o.flag] != 0;
    Op w;
    w.kind = OP_WAIT;
    w.key = INT_MAX;
    for (int r = 0; r < P; ++r)
      for (auto& op : pg.ranks[r].ops)
        for (auto& o : op.outs)
          if (o.flag >= 0 && o.loc.rank == d && !consumed[o.flag]) w.ins.push_back({o.loc, o.flag, op.len, op.chunk});
    std::sort(w.ins.begin(), w.ins.end(), [](const OpIn& a, const OpIn& z) { return a.flag < z.flag; });
    if (!w.ins.empty()) pg.ranks[d].ops.push_back(std::move(w));
  }

  for (auto& rp : pg.ranks) {
    pg.max_slots = std::max(pg.max_slots, rp.nslots);
    pg.scratch_bytes = std::max(pg.scratch_bytes, rp.scratch_bytes);
  }
  // fingerprint: every rank must lower the identical program
  std::string text = serialize(s) + "|" + std::to_string(nbytes) + "|" + std::to_string(esize) + (ll ? "|ll" : "") +
                     (pull ? "|pull" : "");
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char ch : text) {
    h ^= ch;
    h *= 0x100000001b3ull;
  }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)h);
  pg.fingerprint = buf;
  return pg;
}

std::string Program::summary_json() const {
  std::ostringstream o;
  o << "{\"collective\":\"" << kind_name(kind) << "\",\"P\":" << P << ",\"G\":" << G << ",\"bytes\":" << nbytes
    << ",\"send_bytes\":" << send_bytes << ",\"recv_bytes\":" << recv_bytes << ",\"max_slots\":" << max_slots
    << ",\"scratch_bytes\":" << scratch_bytes << ",\"protocol\":\"" << (ll ? "ll" : "simple") << "\",\"pull\":" << (pull ? 1 : 0)
    << ",\"fingerprint\":\"" << fingerprint << "\",\"ranks\":[";
  static const char* sp[] = {"send", "recv", "scratch", "flags"};
  for (int r = 0; r < P; ++r) {
    o << (r ? "," : "") << "{\"nslots\":" << ranks[r].nslots << ",\"ops\":[";
    const auto& ops = ranks[r].ops;
    for (size_t i = 0; i < ops.size(); ++i) {
      const Op& op = ops[i];
      o << (i ? "," : "") << "{\"kind\":\"" << (op.kind == OP_COPY ? "copy" : op.kind == OP_REDUCE ? "reduce" : "wait")
        << "\",\"key\":" << (op.key == INT_MAX ? -1 : op.key) << ",\"chunk\":" << op.chunk << ",\"len\":" << op.len
        << ",\"ins\":[";
      for (size_t j = 0; j < op.ins.size(); ++j) {
        auto& in = op.ins[j];
        o << (j ? "," : "") << "[" << in.loc.rank << ",\"" << sp[in.loc.space] << "\"," << in.loc.off << "," << in.flag
          << "]";
      }
      o << "],\"outs\":[";
      for (size_t j = 0; j < op.outs.size(); ++j) {
        auto& ou = op.outs[j];
        o << (j ? "," : "") << "[" << ou.loc.rank << ",\"" << sp[ou.loc.space] << "\"," << ou.loc.off << ","
          << ou.flag << "," << (ou.every_tile ? 1 : 0) << "]";
      }
      o << "]}";
    }
    o << "]}";
  }
  o << "]}";
  return o.str();
}

}  // namespace sccl
