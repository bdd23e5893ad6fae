// cf_plan_parse.cu -- plan JSON -> host IR, with the reference's parse errors.
//
// Follows parse_plan / _resolve_refs (cf/plan.py:174-291):
//   exactly the 9 top-level keys (+ optional "lowered")       -> E_SYNTAX
//   version == 1                                              -> E_VERSION
//   collective / protocol / dtype domains, num_ranks >= 1     -> E_SYNTAX
//   buffer kinds, channel types, op names, op keys, ranges    -> E_SYNTAX
//   unknown / duplicate buffer or channel ids                 -> E_REF
// dtype additionally accepts "f16" and "bf16" (B200 extension of cf/plan.py:22).
#include <cstring>
#include <set>
#include "cf_json.h"
#include "cf_plan.h"
#include "cf_runtime.h"

namespace cf {
namespace plan {

static const char* kOpNames[P_NUM_OPS] = {"put", "put_packets", "put_with_signal", "signal",
                                          "wait", "flush", "read_packets", "reduce",
                                          "reduce_put", "copy", "tb_sync", "device_barrier"};

const char* op_name(int k) { return (k >= 0 && k < P_NUM_OPS) ? kOpNames[k] : "?"; }

namespace {

using json::Value;

struct Err {
  cfStatus s;
  std::string msg;
};

[[noreturn]] void syntax(const std::string& m) { throw Err{CF_E_SYNTAX, m}; }

const Value& need(const Value& o, const char* key, const std::string& where) {
  if (o.type != Value::Obj) syntax(where + ": expected an object");
  const Value* v = o.get(key);
  if (!v) syntax(where + ": missing key '" + key + "'");
  return *v;
}

long long as_int(const Value& v, const std::string& where) {
  if (v.type != Value::Int) syntax(where + ": expected an integer");
  return v.i;
}

const std::string& as_str(const Value& v, const std::string& where) {
  if (v.type != Value::Str) syntax(where + ": expected a string");
  return v.s;
}

int index_of(const char* const* names, int n, const std::string& s) {
  for (int i = 0; i < n; i++)
    if (s == names[i]) return i;
  return -1;
}

struct RawRef {
  std::string buf;
  long long off, size;
};

bool as_range(const Value* v, RawRef& out, const std::string& where) {
  if (!v || v->type == Value::Null) return false;
  if (v->type != Value::Arr || v->arr.size() != 3 || v->arr[1].type != Value::Int ||
      v->arr[2].type != Value::Int || v->arr[0].type != Value::Str)
    syntax(where + ": range must be [buffer, offset, size]");
  out.buf = v->arr[0].s;
  out.off = v->arr[1].i;
  out.size = v->arr[2].i;
  return true;
}

}  // namespace

cfStatus parse(const char* text, size_t len, int dtype_override, Plan& P) {
  Value doc;
  std::string err;
  json::Parser parser(text, len);
  if (!parser.parse(doc, err)) return fail(CF_E_SYNTAX, "invalid JSON: %s", err.c_str());
  try {
    if (doc.type != Value::Obj) syntax("top level must be an object");
    static const char* top[] = {"version", "name", "collective", "protocol", "dtype",
                                "num_ranks", "buffers", "channels", "programs"};
    std::set<std::string> keys;
    for (auto& kv : doc.obj) keys.insert(kv.first);
    for (auto& k : keys)
      if (index_of(top, 9, k) < 0 && k != "lowered") syntax("unknown top-level keys ['" + k + "']");
    for (auto* k : top)
      if (!keys.count(k)) syntax(std::string("missing top-level keys ['") + k + "']");
    const Value& ver = *doc.get("version");
    if (ver.type != Value::Int || ver.i != 1) throw Err{CF_E_VERSION, "unsupported plan version"};
    static const char* colls[] = {"allreduce", "allgather", "reducescatter", "custom"};
    static const char* protos[] = {"LL", "HB"};
    static const char* dtypes[] = {"i32", "f32", "f16", "bf16"};
    P.collective = index_of(colls, 4, as_str(*doc.get("collective"), "collective"));
    if (P.collective < 0) syntax("collective must be one of ('allreduce', 'allgather', 'reducescatter', 'custom')");
    P.protocol = index_of(protos, 2, as_str(*doc.get("protocol"), "protocol"));
    if (P.protocol < 0) syntax("protocol must be one of ('LL', 'HB')");
    P.dtype = index_of(dtypes, 4, as_str(*doc.get("dtype"), "dtype"));
    if (P.dtype < 0) syntax("dtype must be one of ('i32', 'f32', 'f16', 'bf16')");
    if (dtype_override >= 0) P.dtype = dtype_override;
    const Value& nr = *doc.get("num_ranks");
    if (nr.type != Value::Int || nr.i < 1) syntax("num_ranks must be a positive integer");
    P.nranks = (int)nr.i;
    P.name = doc.get("name")->type == Value::Str ? doc.get("name")->s : "";
    if (const Value* lw = doc.get("lowered")) P.lowered = lw->type == Value::Bool ? lw->b : true;

    const Value& bufs = *doc.get("buffers");
    if (bufs.type != Value::Arr) syntax("buffers must be a list");
    static const char* kinds[] = {"input", "output", "scratch"};
    for (size_t i = 0; i < bufs.arr.size(); i++) {
      const std::string where = "buffers[" + std::to_string(i) + "]";
      const Value& b = bufs.arr[i];
      Buf B;
      B.id = as_str(need(b, "id", where), where);
      B.kind = index_of(kinds, 3, as_str(need(b, "kind", where), where));
      if (B.kind < 0) syntax(where + ": unknown kind");
      const Value& rk = need(b, "rank", where);
      if (rk.type == Value::Str && rk.s == "all") B.rank = -1;
      else if (rk.type == Value::Int) B.rank = (int)rk.i;
      else syntax(where + ": rank must be an integer or \"all\"");
      B.elems = as_int(need(b, "elems", where), where);
      P.bufs.push_back(B);
    }
    const Value& chans = *doc.get("channels");
    if (chans.type != Value::Arr) syntax("channels must be a list");
    static const char* ctypes[] = {"port", "memory", "switch"};
    for (size_t i = 0; i < chans.arr.size(); i++) {
      const std::string where = "channels[" + std::to_string(i) + "]";
      const Value& c = chans.arr[i];
      Chan C;
      C.type = index_of(ctypes, 3, as_str(need(c, "type", where), where));
      if (C.type < 0) syntax(where + ": unknown channel type");
      C.id = as_str(need(c, "id", where), where);
      if (C.type == C_SWITCH) {
        const Value& rs = need(c, "ranks", where);
        if (rs.type != Value::Arr) syntax(where + ": ranks must be a list");
        for (auto& r : rs.arr) C.ranks.push_back((int)as_int(r, where));
      } else {
        C.src = (int)as_int(need(c, "src", where), where);
        C.dst = (int)as_int(need(c, "dst", where), where);
      }
      if (const Value* pr = c.get("protocol"))
        if (pr->type == Value::Str) C.protocol = index_of(protos, 2, pr->s);
      P.chans.push_back(C);
    }
    // ids: duplicate -> E_REF (cf/plan.py:277-283)
    std::set<std::string> bid, cid;
    for (auto& b : P.bufs) bid.insert(b.id);
    for (auto& c : P.chans) cid.insert(c.id);
    if (bid.size() != P.bufs.size()) throw Err{CF_E_REF, "duplicate buffer ids"};
    if (cid.size() != P.chans.size()) throw Err{CF_E_REF, "duplicate channel ids"};
    auto buf_index = [&](const std::string& id, const std::string& where) {
      for (size_t k = 0; k < P.bufs.size(); k++)
        if (P.bufs[k].id == id) return (int)k;
      throw Err{CF_E_REF, where + ": buffer '" + id + "' not declared"};
    };
    auto chan_index = [&](const std::string& id, const std::string& where) {
      for (size_t k = 0; k < P.chans.size(); k++)
        if (P.chans[k].id == id) return (int)k;
      throw Err{CF_E_REF, where + ": channel '" + id + "' not declared"};
    };

    const Value& progs = *doc.get("programs");
    if (progs.type != Value::Arr) syntax("programs must be a list");
    static const char* allowed[] = {"op", "chan", "src", "dst", "src2", "flag", "arrives", "tb_group"};
    for (size_t i = 0; i < progs.arr.size(); i++) {
      const std::string where = "programs[" + std::to_string(i) + "]";
      const Value& p = progs.arr[i];
      Prog G;
      const Value& ops = need(p, "ops", where);
      G.rank = (int)as_int(need(p, "rank", where), where);
      G.tb = (int)as_int(need(p, "tb", where), where);
      if (ops.type != Value::Arr) syntax(where + ": ops must be a list");
      for (size_t j = 0; j < ops.arr.size(); j++) {
        const std::string ow = where + ".ops[" + std::to_string(j) + "]";
        const Value& o = ops.arr[j];
        if (o.type != Value::Obj || !o.get("op")) syntax(ow + ": op entry must be an object with 'op'");
        Op op;
        op.kind = index_of(kOpNames, P_NUM_OPS, as_str(*o.get("op"), ow));
        if (op.kind < 0) syntax(ow + ": unknown op '" + o.get("op")->s + "'");
        for (auto& kv : o.obj)
          if (index_of(allowed, 8, kv.first) < 0) syntax(ow + ": unknown op keys ['" + kv.first + "']");
        const Value* ch = o.get("chan");
        if (ch && ch->type != Value::Null) op.chan = chan_index(as_str(*ch, ow), ow);
        RawRef r;
        if ((op.has_src = as_range(o.get("src"), r, ow))) op.src = {buf_index(r.buf, ow), r.off, r.size};
        if ((op.has_dst = as_range(o.get("dst"), r, ow))) op.dst = {buf_index(r.buf, ow), r.off, r.size};
        if ((op.has_src2 = as_range(o.get("src2"), r, ow))) op.src2 = {buf_index(r.buf, ow), r.off, r.size};
        if ((op.has_arrives = as_range(o.get("arrives"), r, ow)))
          op.arrives = {buf_index(r.buf, ow), r.off, r.size};
        if (const Value* f = o.get("flag"))
          if (f->type != Value::Null) { op.has_flag = true; op.flag = as_int(*f, ow); }
        if (const Value* g = o.get("tb_group"))
          if (g->type != Value::Null) {
            if (g->type != Value::Arr) syntax(ow + ": tb_group must be a list");
            op.has_group = true;
            for (auto& t : g->arr) op.group.push_back((int)as_int(t, ow));
          }
        G.ops.push_back(op);
      }
      P.progs.push_back(G);
    }
  } catch (const Err& e) {
    return fail(e.s, "%s", e.msg.c_str());
  }
  return CF_OK;
}

}  // namespace plan
}  // namespace cf
