// cf_dsl.cpp -- native DSL: algorithm builders and the lowering pipeline.
//
// Replaces the reference's Python builder library (cf/collectives.py:30-270)
// and pass pipeline (cf/lowering.py:295-648) with host C++ inside libcf.  The
// Python ProgramGraph (paper_2504_09014_b200/lowering.py) only records a
// program; `cfDslLower` runs the passes here and returns canonical plan JSON
// (sorted keys, no whitespace, ASCII -- the bytes cf/plan.py:146-162 would
// serialize), so a program lowers to the same plan document as in the
// reference.  `cfDslBuild` emits a library algorithm as a recorded program in
// the same interchange format, so builders and user programs share one path.
//
// Interchange format of a recorded program (JSON object):
//   name, collective, protocol, dtype, num_ranks, elems
//   buffers : [[id, kind, rank | "all", elems], ...]
//   channels: [[id, type, src, dst, protocol | null] | [id, "switch", [ranks], null], ...]
//   instrs  : [[rank, tb, op, chan | null, src, dst, src2, arrives, flag, tb_group], ...]
//             in emission order; ranges are [buffer, offset, size] or null.
//
// Ordering model (cf/lowering.py:11-17): within one thread block channel
// sync ops and port pushes take effect in issue order; data ops are work
// handed to the block's threads, unordered w.r.t. later ops until a tb_sync
// or device_barrier; a port put's source read happens on the proxy and is
// ordered only by a flush of that channel.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "cf.h"
#include "cf_json.h"

namespace cf {
cfStatus fail(cfStatus s, const char* fmt, ...);   // cf_runtime.cu: sets cfLastErrorMessage
namespace dsl {

namespace {

struct Span {
  bool on = false;
  std::string buf;
  long long off = 0, len = 0;
  long long lo() const { return off; }
  long long hi() const { return off + len; }
  bool operator==(const Span& o) const { return on == o.on && buf == o.buf && off == o.off && len == o.len; }
  bool overlaps(const std::string& b, long long l, long long h) const {
    return on && buf == b && off < h && l < off + len;
  }
};

Span span(const std::string& b, long long off, long long len) {
  Span s;
  s.on = true;
  s.buf = b;
  s.off = off;
  s.len = len;
  return s;
}

enum Site { kLocal = 0, kProxy = 1, kArrival = 2 };

struct Ins {
  int id = 0;   // creation number (the reference's instruction index)
  int rank = 0, tb = 0;
  std::string op;
  std::string chan;   // "" = none
  Span src, dst, src2, arrives;
  bool has_flag = false;
  long long flag = 0;
  bool has_group = false;
  std::vector<long long> group;
  bool synthetic = false;                  // tb_sync / flush added by sync insertion
  std::vector<std::pair<int, int>> orders; // dependences an added sync enforces
  std::string ctype = "none";              // channel type of `chan`
};

struct Chan {
  std::string id, type, proto;   // proto "" = null
  int src = 0, dst = 0;
  std::vector<long long> ranks;
};

struct Buf {
  std::string id, kind;
  long long rank = -1;   // -1 = "all"
  long long elems = 0;
};

struct Program {
  std::string name, collective, protocol, dtype;
  int nranks = 1;
  long long elems = 0;
  std::vector<Buf> bufs;
  std::vector<Chan> chans;
  std::vector<Ins> ins;
  // streams in first-use order (the reference iterates a dict)
  std::vector<std::pair<std::pair<int, int>, std::vector<int>>> streams;

  std::vector<int>& stream(int rank, int tb) {
    for (auto& s : streams)
      if (s.first.first == rank && s.first.second == tb) return s.second;
    streams.push_back({{rank, tb}, {}});
    return streams.back().second;
  }
  const Chan* chan(const std::string& id) const {
    for (auto& c : chans)
      if (c.id == id) return &c;
    return nullptr;
  }
  int add(Ins i) {
    i.id = (int)ins.size();
    if (!i.chan.empty()) {
      const Chan* c = chan(i.chan);
      i.ctype = c ? c->type : "none";
    }
    ins.push_back(i);
    return i.id;
  }
  int push(Ins i) {   // record into its (rank, tb) stream
    const int id = add(i);
    stream(ins[id].rank, ins[id].tb).push_back(id);
    return id;
  }
  std::vector<std::pair<int, int>> sorted_keys() const {
    std::vector<std::pair<int, int>> k;
    for (auto& s : streams) k.push_back(s.first);
    std::sort(k.begin(), k.end());
    return k;
  }
  const std::vector<int>* find(std::pair<int, int> key) const {
    for (auto& s : streams)
      if (s.first == key) return &s.second;
    return nullptr;
  }
};

struct DslError {
  cfStatus status;
  std::string msg;
};

[[noreturn]] void raise(cfStatus s, const std::string& m) { throw DslError{s, m}; }

// ---------------------------------------------------------------- effects

struct Touch {
  std::string buf;
  long long lo, hi;
  int site;
};

// Same-rank effects that order an instruction inside its stream
// (cf/lowering.py:68-96).  Remote sides are the channels' business.
void effects(const Ins& x, std::vector<Touch>& rd, std::vector<Touch>& wr) {
  rd.clear();
  wr.clear();
  auto R = [&](const Span& s, int site) { if (s.on) rd.push_back({s.buf, s.lo(), s.hi(), site}); };
  auto W = [&](const Span& s, int site) { if (s.on) wr.push_back({s.buf, s.lo(), s.hi(), site}); };
  const std::string& o = x.op;
  if (o == "reduce") {
    R(x.dst, kLocal);
    if (x.chan.empty()) R(x.src, kLocal);
  } else if (o == "copy") {
    if (x.chan.empty()) R(x.src, kLocal);
  } else if (o == "put" || o == "put_with_signal" || o == "put_packets") {
    R(x.src, x.ctype == "port" ? kProxy : kLocal);
  } else if (o == "reduce_put") {
    R(x.src, kLocal);
    R(x.src2, kLocal);
  } else if (o == "switch_reduce" || o == "switch_broadcast") {
    R(x.src, kLocal);
  }
  if (o == "reduce" || o == "copy" || o == "read_packets" || o == "switch_reduce" || o == "switch_broadcast")
    W(x.dst, kLocal);
  else if (o == "wait")
    W(x.arrives, kArrival);
}

// Every (buffer, rank) instance range an op touches, remote sides included
// (liveness for fusion, cf/lowering.py:438-470).
struct Where {
  std::string buf;
  long long rank, lo, hi;
};
void footprint(const Program& P, const Ins& x, std::vector<Where>& out) {
  out.clear();
  const Chan* c = x.chan.empty() ? nullptr : P.chan(x.chan);
  auto at = [&](const Span& s, long long r) { if (s.on) out.push_back({s.buf, r, s.lo(), s.hi()}); };
  const std::string& o = x.op;
  if (o == "put" || o == "put_with_signal" || o == "put_packets") {
    at(x.src, x.rank);
    at(x.dst, c ? c->dst : 0);
  } else if (o == "reduce_put") {
    at(x.src, x.rank);
    at(x.src2, x.rank);
    at(x.dst, c ? c->dst : 0);
  } else if ((o == "reduce" || o == "copy") && c && c->type != "switch") {
    at(x.dst, x.rank);
    at(x.src, c->dst);
  } else if (o == "switch_reduce" || o == "switch_broadcast") {
    const bool red = o == "switch_reduce";
    if (c)
      for (long long r : c->ranks) at(red ? x.src : x.dst, r);
    at(red ? x.dst : x.src, x.rank);
  } else if (o == "wait") {
    at(x.arrives, x.rank);
  } else {
    at(x.src, x.rank);
    at(x.dst, x.rank);
    at(x.src2, x.rank);
  }
}

// ---------------------------------------------------------------- passes

// dependence edge: (from, to, site of the earlier access); RAW/WAR/WAW are
// not distinguished downstream, only the site matters
using Edge = std::tuple<int, int, int>;

std::set<Edge> dependences(const Program& P) {
  std::set<Edge> edges;
  std::vector<Touch> rd, wr;
  for (auto& s : P.streams) {
    struct Rec { long long lo, hi; int id, site; };
    std::map<std::string, std::pair<std::vector<Rec>, std::vector<Rec>>> live;   // buf -> (writes, reads)
    for (int id : s.second) {
      effects(P.ins[id], rd, wr);
      for (auto& t : rd) {
        auto& st = live[t.buf];
        for (auto& w : st.first)
          if (t.lo < w.hi && w.lo < t.hi && w.id != id) edges.insert({w.id, id, w.site});
        st.second.push_back({t.lo, t.hi, id, t.site});
      }
      for (auto& t : wr) {
        auto& st = live[t.buf];
        for (auto& r : st.second)
          if (t.lo < r.hi && r.lo < t.hi && r.id != id) edges.insert({r.id, id, r.site});
        for (auto& w : st.first)
          if (t.lo < w.hi && w.lo < t.hi && w.id != id) edges.insert({w.id, id, w.site});
        // a record this write fully covers is implied through this write
        auto covered = [&](const Rec& q) { return t.lo <= q.lo && q.hi <= t.hi; };
        st.first.erase(std::remove_if(st.first.begin(), st.first.end(), covered), st.first.end());
        st.first.push_back({t.lo, t.hi, id, t.site});
        st.second.erase(std::remove_if(st.second.begin(), st.second.end(), covered), st.second.end());
      }
    }
  }
  return edges;
}

// Before each instruction, a flush per channel whose proxy read it depends on
// and a tb_sync if it depends on unjoined block work (cf/lowering.py:337-386).
void place_syncs(Program& P, const std::set<Edge>& edges) {
  std::map<int, std::vector<Edge>> into;
  for (auto& e : edges) into[std::get<1>(e)].push_back(e);
  std::vector<Touch> rd, wr;
  for (size_t si = 0; si < P.streams.size(); si++) {
    const int rank = P.streams[si].first.first, tb = P.streams[si].first.second;
    const std::vector<int> in = P.streams[si].second;
    std::vector<int> out;
    std::set<int> open_local;
    std::map<std::string, std::set<int>> open_proxy;
    for (int id : in) {
      std::vector<std::pair<int, int>> joins;
      std::map<std::string, std::vector<std::pair<int, int>>> flushes;   // sorted by channel id
      auto it = into.find(id);
      if (it != into.end())
        for (auto& e : it->second) {
          const int from = std::get<0>(e), site = std::get<2>(e);
          if (site == kLocal && open_local.count(from)) {
            joins.push_back({from, id});
          } else if (site == kProxy) {
            const std::string& ch = P.ins[from].chan;
            auto op = open_proxy.find(ch);
            if (op != open_proxy.end() && op->second.count(from)) flushes[ch].push_back({from, id});
          }
        }
      for (auto& f : flushes) {
        Ins fl;
        fl.rank = rank;
        fl.tb = tb;
        fl.op = "flush";
        fl.chan = f.first;
        fl.synthetic = true;
        fl.orders = f.second;
        const int nid = P.add(fl);
        P.ins[nid].ctype = "port";
        out.push_back(nid);
        open_proxy[f.first].clear();
      }
      if (!joins.empty()) {
        Ins sy;
        sy.rank = rank;
        sy.tb = tb;
        sy.op = "tb_sync";
        sy.synthetic = true;
        sy.orders = joins;
        out.push_back(P.add(sy));
        open_local.clear();
      }
      const Ins& x = P.ins[id];
      if (x.op == "tb_sync" || x.op == "device_barrier") {
        open_local.clear();
      } else if (x.op == "flush") {
        open_proxy[x.chan].clear();
      } else {
        effects(x, rd, wr);
        bool loc = false, prx = false;
        for (auto* v : {&rd, &wr})
          for (auto& t : *v) {
            loc |= t.site == kLocal;
            prx |= t.site == kProxy;
          }
        if (loc) open_local.insert(id);
        if (prx) open_proxy[x.chan].insert(id);
      }
      out.push_back(id);
    }
    P.streams[si].second = out;
  }
}

// Back-to-back tb_syncs collapse into the first (cf/lowering.py:389-400).
void merge_syncs(Program& P) {
  for (auto& s : P.streams) {
    std::vector<int> out;
    for (int id : s.second) {
      if (P.ins[id].op == "tb_sync" && !out.empty() && P.ins[out.back()].op == "tb_sync") {
        auto& keep = P.ins[out.back()].orders;
        keep.insert(keep.end(), P.ins[id].orders.begin(), P.ins[id].orders.end());
        continue;
      }
      out.push_back(id);
    }
    s.second = out;
  }
}

// Is instance (ref, rank) touched after position `pos` of stream `si`, or by
// any other stream at all?
bool touched_later(const Program& P, const Span& ref, long long rank, size_t si, size_t pos) {
  std::vector<Where> fp;
  for (size_t k = 0; k < P.streams.size(); k++) {
    const auto& ids = P.streams[k].second;
    for (size_t q = (k == si ? pos + 1 : 0); q < ids.size(); q++) {
      footprint(P, P.ins[ids[q]], fp);
      for (auto& w : fp)
        if (w.buf == ref.buf && w.rank == rank && ref.lo() < w.hi && w.lo < ref.hi()) return true;
    }
  }
  return false;
}

// {put; signal} -> put_with_signal and {local reduce into scratch; [the tb_sync
// only ordering that pair]; memory put of it} -> reduce_put, to a fixed point
// (cf/lowering.py:473-535).
void fuse_ops(Program& P) {
  auto kind_of = [&](const std::string& b) {
    std::string k;
    for (auto& d : P.bufs)
      if (d.id == b) k = d.kind;   // last declaration wins, as a dict would
    return k;
  };
  for (;;) {
    bool again = false;
    for (size_t si = 0; si < P.streams.size() && !again; si++) {
      std::vector<int>& ids = P.streams[si].second;
      for (size_t pos = 0; pos + 1 < ids.size(); pos++) {
        const Ins& a = P.ins[ids[pos]];
        const Ins& b = P.ins[ids[pos + 1]];
        const Ins* c = pos + 2 < ids.size() ? &P.ins[ids[pos + 2]] : nullptr;
        if (a.op == "put" && b.op == "signal" && a.chan == b.chan) {
          Ins f = a;
          f.op = "put_with_signal";
          f.orders.clear();
          const int nid = P.add(f);
          ids.erase(ids.begin() + pos, ids.begin() + pos + 2);
          ids.insert(ids.begin() + pos, nid);
          again = true;
          break;
        }
        const bool mid = b.op == "tb_sync" && c != nullptr;
        const Ins& put = mid ? *c : b;
        if (!(a.op == "reduce" && a.chan.empty() && put.op == "put" && put.ctype == "memory" &&
              put.src == a.dst && kind_of(a.dst.buf) == "scratch"))
          continue;
        if (touched_later(P, a.dst, a.rank, si, pos + (mid ? 2 : 1))) continue;
        if (mid) {
          bool other = false;
          for (auto& e : b.orders) other |= !(e.first == a.id && e.second == put.id);
          if (!b.synthetic || other) continue;   // that sync orders something else
        }
        Ins f;
        f.rank = a.rank;
        f.tb = a.tb;
        f.op = "reduce_put";
        f.chan = put.chan;
        f.dst = put.dst;
        f.src = a.src;
        f.src2 = a.dst;
        const std::string ctype = put.ctype;
        const int nid = P.add(f);
        P.ins[nid].ctype = ctype;
        ids.erase(ids.begin() + pos, ids.begin() + pos + (mid ? 3 : 2));
        ids.insert(ids.begin() + pos, nid);
        again = true;
        break;
      }
    }
    if (!again) return;
  }
}

// LL flags: a generation per channel starting at 1, bumped when a packet
// range is reused; each read takes the generation of the k-th put of its
// range (cf/lowering.py:538-577).
void ll_flags(Program& P) {
  std::vector<int> puts;
  for (auto& x : P.ins)
    if (x.op == "put_packets") puts.push_back(x.id);   // creation order
  std::map<std::string, long long> gen;
  std::map<std::string, std::vector<Span>> used;
  std::map<std::string, std::vector<std::pair<Span, long long>>> issued;
  for (int id : puts) {
    Ins& x = P.ins[id];
    if (!x.has_flag) {
      long long& g = gen.emplace(x.chan, 1).first->second;
      auto& u = used[x.chan];
      bool reuse = false;
      for (auto& r : u) reuse |= r.overlaps(x.dst.buf, x.dst.lo(), x.dst.hi());
      if (reuse) {
        g += 1;
        u.clear();
      }
      u.push_back(x.dst);
      x.has_flag = true;
      x.flag = g;
    }
    issued[x.chan].push_back({x.dst, x.flag});
  }
  std::map<std::tuple<std::string, std::string, long long, long long>, size_t> taken;
  for (auto key : P.sorted_keys())
    for (int id : *P.find(key)) {
      Ins& x = P.ins[id];
      if (x.op != "read_packets" || x.has_flag) continue;
      std::vector<long long> m;
      for (auto& pf : issued[x.chan])
        if (pf.first.buf == x.src.buf && x.src.lo() < pf.first.hi() && pf.first.lo() < x.src.hi())
          m.push_back(pf.second);
      if (m.empty()) raise(CF_E_SHAPE, "read_packets on " + x.chan + " has no matching put");
      size_t& k = taken[{x.chan, x.src.buf, x.src.lo(), x.src.hi()}];
      x.has_flag = true;
      x.flag = m[std::min(k, m.size() - 1)];
      k++;
    }
}

// `instances` copies of every stream on thread blocks tb*I + i and channel
// sets "<id>.i<i>", instance i taking slice i of every range
// (cf/lowering.py:580-619).
Program replicate(const Program& P, int inst) {
  if (inst == 1) return P;
  for (auto& x : P.ins)
    for (const Span* s : {&x.src, &x.dst, &x.src2, &x.arrives})
      if (s->on && s->len % inst)
        raise(CF_E_SHAPE, "chunk size " + std::to_string(s->len) + " not divisible by " + std::to_string(inst) +
                              " instances");
  Program Q;
  Q.name = P.name;
  Q.collective = P.collective;
  Q.protocol = P.protocol;
  Q.dtype = P.dtype;
  Q.nranks = P.nranks;
  Q.elems = P.elems;
  Q.bufs = P.bufs;
  std::map<std::pair<std::string, int>, std::string> cmap;
  for (auto& c : P.chans)
    for (int i = 0; i < inst; i++) {
      Chan d = c;
      if (i) d.id = c.id + ".i" + std::to_string(i);
      cmap[{c.id, i}] = d.id;
      Q.chans.push_back(d);
    }
  auto cut = [&](const Span& s, int i) {
    if (!s.on) return s;
    const long long share = s.len / inst;
    return span(s.buf, s.off + i * share, share);
  };
  for (auto key : P.sorted_keys())
    for (int i = 0; i < inst; i++)
      for (int id : *P.find(key)) {
        Ins y = P.ins[id];
        y.tb = key.second * inst + i;
        if (!y.chan.empty()) {
          auto it = cmap.find({y.chan, i});
          y.chan = it == cmap.end() ? std::string() : it->second;
        }
        y.src = cut(y.src, i);
        y.dst = cut(y.dst, i);
        y.src2 = cut(y.src2, i);
        y.arrives = cut(y.arrives, i);
        y.orders.clear();
        const std::string ctype = y.ctype;
        const int nid = Q.push(y);
        Q.ins[nid].ctype = ctype;
      }
  return Q;
}

// ---------------------------------------------------------------- canonical JSON

void jstr(std::string& o, const std::string& s) {
  o.push_back('"');
  for (size_t i = 0; i < s.size(); i++) {
    const unsigned char c = (unsigned char)s[i];
    switch (c) {
      case '"': o += "\\\""; continue;
      case '\\': o += "\\\\"; continue;
      case '\n': o += "\\n"; continue;
      case '\r': o += "\\r"; continue;
      case '\t': o += "\\t"; continue;
      case '\b': o += "\\b"; continue;
      case '\f': o += "\\f"; continue;
    }
    char tmp[16];
    if (c < 0x20) {
      snprintf(tmp, sizeof tmp, "\\u%04x", c);
      o += tmp;
    } else if (c < 0x80) {
      o.push_back((char)c);
    } else {   // UTF-8 -> \uXXXX (json.dumps ensure_ascii)
      unsigned cp = 0;
      int extra = c >= 0xf0 ? 3 : c >= 0xe0 ? 2 : 1;
      cp = c & (0x3f >> extra);
      for (int k = 0; k < extra && i + 1 < s.size(); k++) cp = (cp << 6) | ((unsigned char)s[++i] & 0x3f);
      if (cp >= 0x10000) {
        cp -= 0x10000;
        snprintf(tmp, sizeof tmp, "\\u%04x\\u%04x", 0xd800 + (cp >> 10), 0xdc00 + (cp & 0x3ff));
      } else {
        snprintf(tmp, sizeof tmp, "\\u%04x", cp);
      }
      o += tmp;
    }
  }
  o.push_back('"');
}

void jspan(std::string& o, const Span& s) {
  o.push_back('[');
  jstr(o, s.buf);
  o += "," + std::to_string(s.off) + "," + std::to_string(s.len) + "]";
}

void jints(std::string& o, const std::vector<long long>& v) {
  o.push_back('[');
  for (size_t i = 0; i < v.size(); i++) o += (i ? "," : "") + std::to_string(v[i]);
  o.push_back(']');
}

// Keys in sorted order throughout, as json.dumps(sort_keys=True) writes them.
std::string emit(const Program& P) {
  std::string o = "{\"buffers\":[";
  for (size_t i = 0; i < P.bufs.size(); i++) {
    const Buf& b = P.bufs[i];
    o += i ? ",{" : "{";
    o += "\"elems\":" + std::to_string(b.elems) + ",\"id\":";
    jstr(o, b.id);
    o += ",\"kind\":";
    jstr(o, b.kind);
    o += ",\"rank\":";
    o += b.rank < 0 ? std::string("\"all\"") : std::to_string(b.rank);
    o += "}";
  }
  o += "],\"channels\":[";
  for (size_t i = 0; i < P.chans.size(); i++) {
    const Chan& c = P.chans[i];
    o += i ? ",{" : "{";
    const bool sw = c.type == "switch";
    if (!sw) o += "\"dst\":" + std::to_string(c.dst) + ",";
    o += "\"id\":";
    jstr(o, c.id);
    if (!c.proto.empty()) {
      o += ",\"protocol\":";
      jstr(o, c.proto);
    }
    if (sw) {
      o += ",\"ranks\":";
      jints(o, c.ranks);
    } else {
      o += ",\"src\":" + std::to_string(c.src);
    }
    o += ",\"type\":";
    jstr(o, c.type);
    o += "}";
  }
  o += "],\"collective\":";
  jstr(o, P.collective);
  o += ",\"dtype\":";
  jstr(o, P.dtype);
  o += ",\"name\":";
  jstr(o, P.name);
  o += ",\"num_ranks\":" + std::to_string(P.nranks) + ",\"programs\":[";
  bool first = true;
  for (auto key : P.sorted_keys()) {
    o += first ? "{" : ",{";
    first = false;
    o += "\"ops\":[";
    bool f2 = true;
    for (int id : *P.find(key)) {
      const Ins& x = P.ins[id];
      o += f2 ? "{" : ",{";
      f2 = false;
      std::string body;
      auto field = [&](const char* k) {
        if (!body.empty()) body.push_back(',');
        body += "\"";
        body += k;
        body += "\":";
      };
      if (x.arrives.on) { field("arrives"); jspan(body, x.arrives); }
      if (!x.chan.empty()) { field("chan"); jstr(body, x.chan); }
      if (x.dst.on) { field("dst"); jspan(body, x.dst); }
      if (x.has_flag) { field("flag"); body += std::to_string(x.flag); }
      field("op");
      jstr(body, x.op == "switch_reduce" ? "reduce" : x.op == "switch_broadcast" ? "copy" : x.op);
      if (x.src.on) { field("src"); jspan(body, x.src); }
      if (x.src2.on) { field("src2"); jspan(body, x.src2); }
      if (x.has_group) { field("tb_group"); jints(body, x.group); }
      o += body + "}";
    }
    o += "],\"rank\":" + std::to_string(key.first) + ",\"tb\":" + std::to_string(key.second) + "}";
  }
  o += "],\"protocol\":";
  jstr(o, P.protocol);
  o += ",\"version\":1}";
  return o;
}

// Recorded-program interchange (the format documented at the top).
std::string emit_program(const Program& P) {
  std::string o = "{\"buffers\":[";
  for (size_t i = 0; i < P.bufs.size(); i++) {
    const Buf& b = P.bufs[i];
    o += i ? ",[" : "[";
    jstr(o, b.id);
    o += ",";
    jstr(o, b.kind);
    o += ",";
    o += b.rank < 0 ? std::string("\"all\"") : std::to_string(b.rank);
    o += "," + std::to_string(b.elems) + "]";
  }
  o += "],\"channels\":[";
  for (size_t i = 0; i < P.chans.size(); i++) {
    const Chan& c = P.chans[i];
    o += i ? ",[" : "[";
    jstr(o, c.id);
    o += ",";
    jstr(o, c.type);
    if (c.type == "switch") {
      o += ",";
      jints(o, c.ranks);
      o += ",null]";
    } else {
      o += "," + std::to_string(c.src) + "," + std::to_string(c.dst) + ",";
      if (c.proto.empty()) o += "null";
      else jstr(o, c.proto);
      o += "]";
    }
  }
  o += "],\"collective\":";
  jstr(o, P.collective);
  o += ",\"dtype\":";
  jstr(o, P.dtype);
  o += ",\"elems\":" + std::to_string(P.elems) + ",\"instrs\":[";
  // emission order = creation order of recorded instructions
  bool first = true;
  for (auto& x : P.ins) {
    o += first ? "[" : ",[";
    first = false;
    o += std::to_string(x.rank) + "," + std::to_string(x.tb) + ",";
    jstr(o, x.op);
    o += ",";
    if (x.chan.empty()) o += "null";
    else jstr(o, x.chan);
    for (const Span* s : {&x.src, &x.dst, &x.src2, &x.arrives}) {
      o += ",";
      if (s->on) jspan(o, *s);
      else o += "null";
    }
    o += ",";
    o += x.has_flag ? std::to_string(x.flag) : std::string("null");
    o += ",";
    if (x.has_group) jints(o, x.group);
    else o += "null";
    o += "]";
  }
  o += "],\"name\":";
  jstr(o, P.name);
  o += ",\"num_ranks\":" + std::to_string(P.nranks) + ",\"protocol\":";
  jstr(o, P.protocol);
  o += "}";
  return o;
}

// ---------------------------------------------------------------- reading

long long as_int(const json::Value* v, const char* what) {
  if (!v || v->type != json::Value::Int) raise(CF_E_SYNTAX, std::string("program: ") + what + " must be an integer");
  return v->i;
}
std::string as_str(const json::Value* v, const char* what) {
  if (!v || v->type != json::Value::Str) raise(CF_E_SYNTAX, std::string("program: ") + what + " must be a string");
  return v->s;
}
Span as_span(const json::Value& v) {
  if (v.type == json::Value::Null) return Span();
  if (v.type != json::Value::Arr || v.arr.size() != 3 || v.arr[0].type != json::Value::Str || !v.arr[1].is_int() ||
      !v.arr[2].is_int())
    raise(CF_E_SYNTAX, "program: range must be [buffer, offset, size]");
  return span(v.arr[0].s, v.arr[1].i, v.arr[2].i);
}

Program read_program(const char* text, size_t len) {
  json::Value doc;
  std::string err;
  json::Parser ps(text, len);
  if (!ps.parse(doc, err)) raise(CF_E_SYNTAX, "program: " + err);
  if (doc.type != json::Value::Obj) raise(CF_E_SYNTAX, "program: top level must be an object");
  Program P;
  P.name = as_str(doc.get("name"), "name");
  P.collective = as_str(doc.get("collective"), "collective");
  P.protocol = as_str(doc.get("protocol"), "protocol");
  P.dtype = as_str(doc.get("dtype"), "dtype");
  P.nranks = (int)as_int(doc.get("num_ranks"), "num_ranks");
  P.elems = as_int(doc.get("elems"), "elems");
  const json::Value* bufs = doc.get("buffers");
  const json::Value* chans = doc.get("channels");
  const json::Value* ins = doc.get("instrs");
  if (!bufs || !chans || !ins || bufs->type != json::Value::Arr || chans->type != json::Value::Arr ||
      ins->type != json::Value::Arr)
    raise(CF_E_SYNTAX, "program: buffers, channels and instrs must be arrays");
  for (auto& b : bufs->arr) {
    if (b.type != json::Value::Arr || b.arr.size() != 4) raise(CF_E_SYNTAX, "program: buffer entry");
    Buf d;
    d.id = as_str(&b.arr[0], "buffer id");
    d.kind = as_str(&b.arr[1], "buffer kind");
    d.rank = b.arr[2].type == json::Value::Str ? -1 : as_int(&b.arr[2], "buffer rank");
    d.elems = as_int(&b.arr[3], "buffer elems");
    P.bufs.push_back(d);
  }
  for (auto& c : chans->arr) {
    if (c.type != json::Value::Arr || c.arr.size() < 4) raise(CF_E_SYNTAX, "program: channel entry");
    Chan d;
    d.id = as_str(&c.arr[0], "channel id");
    d.type = as_str(&c.arr[1], "channel type");
    if (d.type == "switch") {
      if (c.arr[2].type != json::Value::Arr) raise(CF_E_SYNTAX, "program: switch ranks");
      for (auto& r : c.arr[2].arr) d.ranks.push_back(as_int(&r, "switch rank"));
    } else {
      d.src = (int)as_int(&c.arr[2], "channel src");
      d.dst = (int)as_int(&c.arr[3], "channel dst");
      if (c.arr.size() > 4 && c.arr[4].type == json::Value::Str) d.proto = c.arr[4].s;
    }
    if (d.type == "switch" && c.arr[3].type == json::Value::Str) d.proto = c.arr[3].s;
    P.chans.push_back(d);
  }
  for (auto& e : ins->arr) {
    if (e.type != json::Value::Arr || e.arr.size() != 10) raise(CF_E_SYNTAX, "program: instruction entry");
    Ins x;
    x.rank = (int)as_int(&e.arr[0], "rank");
    x.tb = (int)as_int(&e.arr[1], "tb");
    x.op = as_str(&e.arr[2], "op");
    if (e.arr[3].type == json::Value::Str) x.chan = e.arr[3].s;
    x.src = as_span(e.arr[4]);
    x.dst = as_span(e.arr[5]);
    x.src2 = as_span(e.arr[6]);
    x.arrives = as_span(e.arr[7]);
    if (e.arr[8].type != json::Value::Null) {
      x.has_flag = true;
      x.flag = as_int(&e.arr[8], "flag");
    }
    if (e.arr[9].type == json::Value::Arr) {
      x.has_group = true;
      for (auto& t : e.arr[9].arr) x.group.push_back(as_int(&t, "tb_group"));
    }
    P.push(x);
  }
  return P;
}

// ---------------------------------------------------------------- builders

// Library algorithms (cf/collectives.py:30-270) recorded natively.  Each
// emits the same buffers, channels (same creation order, so the same ids)
// and per-stream instruction sequences as the reference builder, so the
// lowered plans are the reference's plans byte for byte.
struct Builder {
  Program P;
  explicit Builder(const std::string& name, const std::string& coll, int n, long long elems, const std::string& dtype,
                   const std::string& proto) {
    P.name = name;
    P.collective = coll;
    P.nranks = n;
    P.elems = elems;
    P.dtype = dtype;
    P.protocol = proto;
  }
  void buffer(const std::string& id, const std::string& kind, long long elems) {
    if (elems <= 0) raise(CF_E_SHAPE, "buffer '" + id + "' must have positive elems");
    P.bufs.push_back({id, kind, -1, elems});
  }
  std::string channel(const std::string& type, int src, int dst) {
    Chan c;
    c.id = std::string(1, type[0]) + std::to_string(P.chans.size());
    c.type = type;
    c.src = src;
    c.dst = dst;
    if (type == "memory") c.proto = P.protocol;
    P.chans.push_back(c);
    return c.id;
  }
  const Chan& ch(const std::string& id) const { return *P.chan(id); }
  void op(int rank, const std::string& name, const std::string& chan, Span dst, Span src, Span arrives = Span()) {
    Ins x;
    x.rank = rank;
    x.tb = 0;
    x.op = name;
    x.chan = chan;
    x.dst = dst;
    x.src = src;
    x.arrives = arrives;
    P.push(x);
  }
  // channel-side conveniences: the rank an op runs on follows from the op
  void put(const std::string& c, Span dst, Span src) { op(ch(c).src, "put", c, dst, src); }
  void put_packets(const std::string& c, Span dst, Span src) { op(ch(c).src, "put_packets", c, dst, src); }
  void read_packets(const std::string& c, Span dst, Span src) { op(ch(c).dst, "read_packets", c, dst, src); }
  void signal(const std::string& c) { op(ch(c).src, "signal", c, Span(), Span()); }
  void wait(const std::string& c, Span arrives) { op(ch(c).dst, "wait", c, Span(), Span(), arrives); }
  void flush(const std::string& c) { op(ch(c).src, "flush", c, Span(), Span()); }
  void pull_reduce(const std::string& c, Span dst, Span src) { op(ch(c).src, "reduce", c, dst, src); }
  void reduce(int r, Span dst, Span src) { op(r, "reduce", "", dst, src); }
  void copy(int r, Span dst, Span src) { op(r, "copy", "", dst, src); }
};

using Key = std::pair<int, int>;

// ring ReduceScatter with overlapped halves (cf/collectives.py:30-79); with
// `full` the output is the whole vector (the 2PR phase 1) and the output
// buffer was declared by the caller.
void ring_reduce_scatter(Builder& B, bool full) {
  const int n = B.P.nranks;
  const long long e = B.P.elems;
  if (e % (2 * n)) raise(CF_E_SHAPE, "ring ReduceScatter needs elems divisible by " + std::to_string(2 * n));
  const long long cs = e / n, h = cs / 2;
  B.buffer("input", "input", e);
  B.buffer("scratch", "scratch", e);
  if (!full) B.buffer("output", "output", cs);
  if (n == 1) {
    B.copy(0, span("output", 0, cs), span("input", 0, cs));
    return;
  }
  std::vector<std::string> link(n);
  for (int r = 0; r < n; r++) link[r] = B.channel("port", r, (r + 1) % n);
  for (int r = 0; r < n; r++) {
    const std::string& out = link[r];
    const std::string& in = link[(r + n - 1) % n];
    const long long obase = full ? (long long)r * cs : 0;
    for (int step = 0; step < n; step++) {
      const long long mine = (long long)((r - step + n) % n) * cs;        // chunk this step forwards
      const long long got = (long long)((r - step - 1 + 2 * n) % n) * cs; // chunk arriving this step
      B.put(out, span("scratch", mine, h), span("input", mine, h));
      B.signal(out);
      if (step) B.reduce(r, span("input", mine + h, h), span("scratch", mine + h, h));
      B.wait(in, span("scratch", got, h));
      B.flush(out);
      B.put(out, span("scratch", mine + h, h), span("input", mine + h, h));
      B.signal(out);
      if (step + 1 < n) B.reduce(r, span("input", got, h), span("scratch", got, h));
      else B.reduce(r, span("output", obase, h), span("scratch", got, h));
      B.wait(in, span("scratch", got + h, h));
      B.flush(out);
    }
    B.reduce(r, span("output", obase + h, h), span("scratch", (long long)r * cs + h, h));
  }
}

Program build(const std::string& algo, const std::string& variant, int n, long long e, const std::string& dtype,
              const std::string& proto) {
  auto peers_of = [n](int r) {
    std::vector<int> v;
    for (int p = 0; p < n; p++)
      if (p != r) v.push_back(p);
    return v;
  };
  // all-pairs channel table in the reference's creation order (r outer, p inner)
  auto all_pairs = [&](Builder& B, const char* type) {
    std::map<Key, std::string> t;
    for (int r = 0; r < n; r++)
      for (int p : peers_of(r)) t[{r, p}] = B.channel(type, r, p);
    return t;
  };
  if (algo == "ring_rs") {
    Builder B("ring_rs", "reducescatter", n, e, dtype, proto);
    ring_reduce_scatter(B, false);
    return B.P;
  }
  if (algo == "ring_ag") {
    Builder B("ring_ag", "allgather", n, e, dtype, proto);
    const long long cs = e;
    B.buffer("input", "input", cs);
    B.buffer("output", "output", n * cs);
    if (n == 1) {
      B.copy(0, span("output", 0, cs), span("input", 0, cs));
      return B.P;
    }
    std::vector<std::string> link(n);
    for (int r = 0; r < n; r++) link[r] = B.channel("port", r, (r + 1) % n);
    for (int r = 0; r < n; r++) {
      B.copy(r, span("output", (long long)r * cs, cs), span("input", 0, cs));
      for (int t = 0; t + 1 < n; t++) {
        const long long fwd = (long long)((r - t + n) % n) * cs, got = (long long)((r - t - 1 + 2 * n) % n) * cs;
        B.put(link[r], span("output", fwd, cs), span("output", fwd, cs));
        B.signal(link[r]);
        B.wait(link[(r + n - 1) % n], span("output", got, cs));
        B.flush(link[r]);
      }
    }
    return B.P;
  }
  if (algo == "2pr") {
    if (e % (2 * n)) raise(CF_E_SHAPE, "two-phase ring needs elems divisible by " + std::to_string(2 * n));
    Builder B("2pr", "allreduce", n, e, dtype, proto);
    B.buffer("output", "output", e);
    ring_reduce_scatter(B, true);
    if (n == 1) return B.P;
    const long long cs = e / n, h = cs / 2;
    for (int r = 0; r < n; r++) {
      const std::string out = B.P.chans[r].id, in = B.P.chans[(r + n - 1) % n].id;
      for (int t = 0; t + 1 < n; t++) {
        const long long fwd = (long long)((r - t + n) % n) * cs, got = (long long)((r - t - 1 + 2 * n) % n) * cs;
        for (long long half : {0LL, h}) {
          B.put(out, span("output", fwd + half, h), span("output", fwd + half, h));
          B.signal(out);
          B.wait(in, span("output", got + half, h));
          B.flush(out);
        }
      }
    }
    return B.P;
  }
  if (algo == "1pa") {
    if (proto != "LL") raise(CF_E_PROTOCOL, "put_packets requires the LL protocol, plan is " + proto);
    Builder B("1pa", "allreduce", n, e, dtype, proto);
    B.buffer("input", "input", e);
    B.buffer("output", "output", e);
    B.buffer("llscr", "scratch", 2 * n * e);
    B.buffer("tmp", "scratch", n * e);
    auto C = all_pairs(B, "memory");
    for (int r = 0; r < n; r++) {
      for (int p : peers_of(r)) B.put_packets(C[{r, p}], span("llscr", (long long)r * e, e), span("input", 0, e));
      B.copy(r, span("output", 0, e), span("input", 0, e));
      for (int p : peers_of(r))
        B.read_packets(C[{p, r}], span("tmp", (long long)p * e, e), span("llscr", (long long)p * e, e));
      for (int p : peers_of(r)) B.reduce(r, span("output", 0, e), span("tmp", (long long)p * e, e));
    }
    return B.P;
  }
  if (algo == "2pa") {
    const std::string var = variant.empty() ? "memory" : variant;
    if (var != "memory" && var != "ll" && var != "port") raise(CF_E_NO_ALGO, "unknown 2pa variant '" + var + "'");
    if (e % n) raise(CF_E_SHAPE, "two-phase all-pairs needs elems divisible by " + std::to_string(n));
    const long long cs = e / n;
    Builder B("2pa_" + var, "allreduce", n, e, dtype, proto);
    B.buffer("input", "input", e);
    B.buffer("output", "output", e);
    if (var == "ll") {
      if (proto != "LL") raise(CF_E_PROTOCOL, "put_packets requires the LL protocol, plan is " + proto);
      B.buffer("ph1", "scratch", 2 * e);
      B.buffer("ph2", "scratch", 2 * e);
      B.buffer("tmp", "scratch", e);
    } else if (var == "port") {
      B.buffer("slots", "scratch", e);
    } else if (proto != "HB") {
      raise(CF_E_PROTOCOL, "reduce on a memory channel requires HB, plan is " + proto);
    }
    auto C = all_pairs(B, var == "port" ? "port" : "memory");
    auto chunk = [cs](const char* b, int q) { return span(b, (long long)q * cs, cs); };
    for (int r = 0; r < n; r++) {
      const std::vector<int> peers = peers_of(r);
      if (var == "memory") {
        B.copy(r, chunk("output", r), chunk("input", r));
        for (int p : peers) B.pull_reduce(C[{r, p}], chunk("output", r), chunk("input", r));
        for (int p : peers) {
          B.put(C[{r, p}], chunk("output", r), chunk("output", r));
          B.signal(C[{r, p}]);
        }
        for (int p : peers) B.wait(C[{p, r}], chunk("output", p));
      } else if (var == "port") {
        for (int p : peers) {
          B.put(C[{r, p}], chunk("slots", r), chunk("input", p));
          B.signal(C[{r, p}]);
        }
        B.copy(r, chunk("output", r), chunk("input", r));
        for (int p : peers) B.wait(C[{p, r}], chunk("slots", p));
        for (int p : peers) B.reduce(r, chunk("output", r), chunk("slots", p));
        for (int p : peers) {
          B.put(C[{r, p}], chunk("output", r), chunk("output", r));
          B.signal(C[{r, p}]);
        }
        for (int p : peers) B.wait(C[{p, r}], chunk("output", p));
        for (int p : peers) B.flush(C[{r, p}]);
      } else {
        for (int p : peers) B.put_packets(C[{r, p}], chunk("ph1", r), chunk("input", p));
        B.copy(r, chunk("output", r), chunk("input", r));
        for (int p : peers) B.read_packets(C[{p, r}], chunk("tmp", p), chunk("ph1", p));
        for (int p : peers) B.reduce(r, chunk("output", r), chunk("tmp", p));
        for (int p : peers) B.put_packets(C[{r, p}], chunk("ph2", r), chunk("output", r));
        for (int p : peers) B.read_packets(C[{p, r}], chunk("output", p), chunk("ph2", p));
      }
    }
    return B.P;
  }
  if (algo == "switch_2pa") {
    if (e % n) raise(CF_E_SHAPE, "switch all-pairs needs elems divisible by " + std::to_string(n));
    const long long cs = e / n;
    Builder B("switch_2pa", "allreduce", n, e, dtype, proto);
    B.buffer("input", "input", e);
    B.buffer("output", "output", e);
    B.buffer("tmp", "scratch", cs);
    Chan sw;
    sw.id = "s" + std::to_string(B.P.chans.size());
    sw.type = "switch";
    for (int r = 0; r < n; r++) sw.ranks.push_back(r);
    B.P.chans.push_back(sw);
    for (int r = 0; r < n; r++) {
      B.op(r, "switch_reduce", sw.id, span("tmp", 0, cs), span("input", (long long)r * cs, cs));
      B.op(r, "switch_broadcast", sw.id, span("output", (long long)r * cs, cs), span("tmp", 0, cs));
    }
    return B.P;
  }
  if (algo == "allpairs_ag") {
    const long long cs = e;
    Builder B("allpairs_ag", "allgather", n, e, dtype, proto);
    B.buffer("input", "input", cs);
    B.buffer("output", "output", n * cs);
    auto C = all_pairs(B, "memory");
    for (int r = 0; r < n; r++) {
      B.copy(r, span("output", (long long)r * cs, cs), span("input", 0, cs));
      for (int p : peers_of(r)) {
        B.put(C[{r, p}], span("output", (long long)r * cs, cs), span("input", 0, cs));
        B.signal(C[{r, p}]);
      }
      for (int p : peers_of(r)) B.wait(C[{p, r}], span("output", (long long)p * cs, cs));
    }
    return B.P;
  }
  if (algo == "2ph") raise(CF_E_TOPOLOGY, "2ph is the multi-node hierarchical algorithm (out of scope)");
  raise(CF_E_NO_ALGO, "unknown algorithm '" + algo + "'");
}

cfStatus deliver(const std::string& s, char* out, size_t cap, size_t* out_len) {
  if (out_len) *out_len = s.size();
  if (!out || cap < s.size()) return fail(CF_E_BAD_SIZE, "output buffer holds %zu bytes, need %zu", cap, s.size());
  memcpy(out, s.data(), s.size());
  return CF_OK;
}

}  // namespace
}  // namespace dsl
}  // namespace cf

using namespace cf::dsl;

extern "C" cfStatus cfDslLower(const char* program, size_t len, int instances, int passes, char* out, size_t cap,
                               size_t* out_len) {
  if (!program) return cf::fail(CF_E_CONFIG, "null program");
  if (instances < 1) return cf::fail(CF_E_SHAPE, "instances must be >= 1");
  try {
    Program P = replicate(read_program(program, len), instances);
    const std::set<Edge> deps = dependences(P);
    if (passes & CF_DSL_PASS_SYNC) {
      place_syncs(P, deps);
      merge_syncs(P);
    }
    if (passes & CF_DSL_PASS_FUSE) fuse_ops(P);
    if (P.protocol == "LL") ll_flags(P);
    return deliver(emit(P), out, cap, out_len);
  } catch (const DslError& e) {
    return cf::fail(e.status, "%s", e.msg.c_str());
  } catch (const std::exception& e) {
    return cf::fail(CF_E_INTERNAL, "lowering: %s", e.what());
  }
}

extern "C" cfStatus cfDslBuild(const char* algo, const char* variant, int nranks, size_t elems, const char* dtype,
                               const char* protocol, char* out, size_t cap, size_t* out_len) {
  if (!algo || !dtype || !protocol) return cf::fail(CF_E_CONFIG, "null argument");
  if (nranks < 1) return cf::fail(CF_E_BAD_SIZE, "nranks must be >= 1");
  try {
    return deliver(emit_program(build(algo, variant ? variant : "", nranks, (long long)elems, dtype, protocol)), out,
                   cap, out_len);
  } catch (const DslError& e) {
    return cf::fail(e.status, "%s", e.msg.c_str());
  }
}
