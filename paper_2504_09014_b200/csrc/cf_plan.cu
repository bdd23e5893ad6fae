// cf_plan.cu -- plan loading: validation, lowering of reference plan ops to
// the device op array, fusion, sync classification, buffer binding, and the
// cfPlan* entry points (replaces Runtime, cf/executor.py:73-178).
//
// Op semantics follow the reference executor exactly (cf/executor.py:237-379):
//   put / put_with_signal : chan.src's src range -> chan.dst's dst range (+ signal)
//   put_packets           : chan.src's payload -> LL packets in chan.dst's buffer
//   read_packets          : own packets -> own dst (size taken from src)
//   reduce  memory chan   : own dst += chan.dst's src      switch: own dst = sum_r src@r
//   copy    memory chan   : own dst  = chan.dst's src      switch: src -> dst@r for all r
//   reduce_put            : chan.dst's dst = own src + own src2
//   port put / signal     : a request to the host proxy (copy-engine DMA, then the
//                           signal in stream order); flush waits for its completion
//   memory put / flush    : executed by the CTAs themselves; memory flush is a no-op
// Fusions (same results, fewer passes over memory):
//   reduce chains on one destination -> one n-source reduce, plan order kept
//   copy feeding such a chain         -> first source of the chain
//   puts of the reduced range         -> extra destinations of the reduce
//   (the SURVEY.md Appendix B pattern "pull-reduce then push").
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include "cf_plan.h"
#include "cf_runtime.h"

namespace cf {
namespace plan {
cfStatus parse(const char* text, size_t len, int dtype_override, Plan& P);
const char* op_name(int k);
const void* plan_kernel_for(int dtype, int cls);
const void* plan_single_kernel_for(int dtype);
const void* plan_ll_kernel_for(int dtype);

namespace {

// host-side op under construction
struct R {
  int buf, rank;
  long long off;     // elements
  bool packet;       // packet-space range (2 bytes of packet per payload byte)
};
struct HOp {
  int code = D_NOP;
  int flags = 0;
  long long size = 0;
  uint32_t llflag = 0;
  int chan = -1, peer = -1;
  std::vector<int> members;   // device_barrier tbs
  std::vector<R> src, dst;
  int plan_index = -1;
};

struct Group {
  int dev;
  std::vector<int> progs;     // indices into compiled program list (sorted by rank, tb)
  DevOp* d_ops = nullptr;
  int32_t* d_meta = nullptr;  // begin | end | rank
  char** d_bufptr = nullptr;
  int32_t* d_zero = nullptr;
  uint64_t* d_done = nullptr;  // proxy completion counters [nprog * K]
  int nops = 0;
  std::vector<int32_t> beg, end;  // host copy of the op ranges (parameter-space table)
  // Op arrays resolved on the host for one I/O binding (the n input and n
  // output addresses of a call), uploaded once and reused while the caller
  // keeps its buffers (decode loops, CUDA graphs): the interpreter then skips
  // its per-call resolve pass.  Bounded; further bindings resolve on device.
  std::vector<DevOp> h_ops;       // host copy, plan-owned buffers baked
  struct Bound {
    std::vector<char*> io;        // io_in[0..n) | io_out[0..n)
    DevOp* d_ops = nullptr;
    DevOp* h_pin = nullptr;       // pinned source of the upload (kept: the copy is stream-ordered)
    std::vector<PlanArgs::Prefetch> pf;   // per program of the group (first data op's sources)
  };
  std::vector<Bound> bound;
};
constexpr size_t kMaxBound = 32;

}  // namespace
}  // namespace plan
}  // namespace cf

struct cfPlan {
  cfComm* comm = nullptr;
  cf::plan::Plan ir;
  int dtype = 0, es = 4, K = 1, threads = CF_PLAN_THREADS;
  int in_buf = -1, out_buf = -1;
  bool input_private = false;
  uint32_t flag_stride = 2;
  std::vector<std::vector<cf::plan::DevOp>> prog_ops;  // per compiled program
  std::vector<int> prog_rank, prog_tb;
  std::vector<char*> heap;            // per rank plan heap
  std::vector<size_t> buf_off;        // per buffer: offset in the heap (all ranks alike)
  size_t state_off = 0, lanes_off = 0, bars_off = 0, heap_bytes = 0;
  int nbars = 0;
  std::vector<std::vector<int>> zero_bufs;  // per rank
  std::vector<cf::plan::Group> groups;
  int n_device_ops = 0;
  int window = 1;                     // ops staged per shared-memory window (<= kPlanWindow)
  bool uses_port = false;             // port-channel ops go through the proxy
  int cls = 3;                        // interpreter class: bit 0 LL packet ops, bit 1 port ops
  bool has_prologue = false;          // per-call zeroing / private input copy
  bool single_ok = false;             // every program one plain MULTI / COPY: plan_single_kernel applies
  bool ll_ok = false;                 // every program a short LL16 op sequence: plan_ll_kernel applies
  std::vector<int> ll_stream;         // per program: PUT_PACKETS op streamed with the MULTI after it (-1: none)
  std::vector<int> ll_fuse_put;       // per program: MULTI whose result the PUT_PACKETS two ops on broadcasts (-1: none)
  // one-process-per-GPU: this process runs rank `me`'s programs; the peers'
  // plan heaps are IPC-mapped by cfPlanConnect, which finalizes the plan
  bool mp = false;
  int me = 0;
  bool ready = false;
  std::vector<bool> heap_mapped;      // heap[r] is an IPC mapping (close, not free)
  bool peer_in = false, peer_out = false;  // data ops touch another rank's I/O buffer
};

namespace cf {
namespace plan {
namespace {

struct Fail {
  cfStatus s;
  std::string m;
};
[[noreturn]] void bad(cfStatus s, const std::string& m) { throw Fail{s, m}; }

std::string where(int pi, int oi) {
  return "programs[" + std::to_string(pi) + "].ops[" + std::to_string(oi) + "]";
}

// ------------------------------------------------------------------ validation helpers

void check_ref(const Plan& P, const Ref& r, int rank, bool packet, long long size, const std::string& w) {
  const Buf& b = P.bufs[r.buf];
  if (b.rank != -1 && b.rank != rank)
    bad(CF_E_OOB, w + ": buffer '" + b.id + "' not present on rank " + std::to_string(rank));
  const long long limit = packet ? b.elems / 2 : b.elems;
  if (r.off < 0 || size < 0 || r.off + size > limit)
    bad(CF_E_OOB, w + ": [" + std::to_string(r.off) + "," + std::to_string(r.off + size) + ") exceeds " +
                      (packet ? "packet capacity " : "elems ") + std::to_string(limit) + " of buffer '" + b.id + "'");
}

void check_rank(const Plan& P, int r, const std::string& w) {
  if (r < 0 || r >= P.nranks) bad(CF_E_OOB, w + ": rank " + std::to_string(r) + " out of range");
}

// ------------------------------------------------------------------ lowering to HOps

std::vector<HOp> lower_program(const Plan& P, int pi, int es) {
  const Prog& G = P.progs[pi];
  std::vector<HOp> out;
  const int rank = G.rank;
  for (size_t oi = 0; oi < G.ops.size(); oi++) {
    const Op& op = G.ops[oi];
    const std::string w = where(pi, (int)oi);
    const Chan* ch = op.chan >= 0 ? &P.chans[op.chan] : nullptr;
    auto need_chan = [&](bool allow_switch) {
      if (!ch) bad(CF_E_SHAPE, w + ": " + op_name(op.kind) + " requires a channel");
      if (!allow_switch && ch->type == C_SWITCH)
        bad(CF_E_PROTOCOL, w + ": " + op_name(op.kind) + " needs a port or memory channel");
      if (ch->type != C_SWITCH) { check_rank(P, ch->src, w); check_rank(P, ch->dst, w); }
      else for (int r : ch->ranks) check_rank(P, r, w);
    };
    auto need = [&](bool have, const char* what) {
      if (!have) bad(CF_E_SHAPE, w + ": " + op_name(op.kind) + " needs " + what);
    };
    HOp h;
    h.plan_index = (int)oi;
    switch (op.kind) {
      case P_PUT:
      case P_PUT_WITH_SIGNAL: {
        need_chan(false);
        need(op.has_src && op.has_dst, "src and dst");
        check_ref(P, op.src, ch->src, false, op.src.size, w);
        check_ref(P, op.dst, ch->dst, false, op.src.size, w);
        h.size = op.src.size;
        h.src = {{op.src.buf, ch->src, op.src.off, false}};
        h.dst = {{op.dst.buf, ch->dst, op.dst.off, false}};
        if (ch->type == C_PORT) {
          // PortChannel: the proxy copies with the copy engine, then signals
          h.code = D_PORT_PUT;
          h.chan = op.chan;
          h.peer = ch->dst;
          if (op.kind == P_PUT_WITH_SIGNAL) h.flags |= F_SIGNAL;
          out.push_back(h);
          break;
        }
        h.code = D_COPY;
        if (h.size > 0) out.push_back(h);
        if (op.kind == P_PUT_WITH_SIGNAL) {
          HOp s;
          s.code = D_SIGNAL;
          s.chan = op.chan;
          s.peer = ch->dst;
          s.plan_index = (int)oi;
          out.push_back(s);
        }
        break;
      }
      case P_SIGNAL:
        need_chan(false);
        h.code = ch->type == C_PORT ? D_PORT_SIGNAL : D_SIGNAL;
        h.chan = op.chan;
        h.peer = ch->dst;
        out.push_back(h);
        break;
      case P_WAIT:
        need_chan(false);
        h.code = D_WAIT;
        h.chan = op.chan;
        out.push_back(h);
        break;
      case P_FLUSH:   // memory-channel flush is a no-op (cf/channels.py:239-240)
        need_chan(true);
        if (ch->type == C_PORT) {
          h.code = D_PORT_FLUSH;
          h.chan = op.chan;
          out.push_back(h);
        }
        break;
      case P_PUT_PACKETS: {
        need_chan(false);
        need(op.has_src && op.has_dst, "src and dst");
        if (!op.has_flag || op.flag == 0) bad(CF_E_ZERO_FLAG, w + ": LL flag must be nonzero");
        if (op.flag < 0 || op.flag > 0x7fffffff) bad(CF_E_SHAPE, w + ": LL flag out of range");
        if ((op.src.size * es) % 4) bad(CF_E_BAD_ALIGN, w + ": LL payload must be a multiple of 4 bytes");
        check_ref(P, op.src, ch->src, false, op.src.size, w);
        check_ref(P, op.dst, ch->dst, true, op.src.size, w);
        h.code = D_PUT_PACKETS;
        h.size = op.src.size;
        h.llflag = (uint32_t)op.flag;
        h.src = {{op.src.buf, ch->src, op.src.off, false}};
        h.dst = {{op.dst.buf, ch->dst, op.dst.off, true}};
        if (h.size > 0) out.push_back(h);
        break;
      }
      case P_READ_PACKETS: {
        need(op.has_src && op.has_dst, "src and dst");
        if (!op.has_flag || op.flag == 0) bad(CF_E_ZERO_FLAG, w + ": LL flag must be nonzero");
        if (op.flag < 0 || op.flag > 0x7fffffff) bad(CF_E_SHAPE, w + ": LL flag out of range");
        if ((op.src.size * es) % 4) bad(CF_E_BAD_ALIGN, w + ": LL payload must be a multiple of 4 bytes");
        check_ref(P, op.src, rank, true, op.src.size, w);
        check_ref(P, op.dst, rank, false, op.src.size, w);
        h.code = D_READ_PACKETS;
        h.size = op.src.size;
        h.llflag = (uint32_t)op.flag;
        h.src = {{op.src.buf, rank, op.src.off, true}};
        h.dst = {{op.dst.buf, rank, op.dst.off, false}};
        if (h.size > 0) out.push_back(h);
        break;
      }
      case P_REDUCE: {
        need(op.has_src && op.has_dst, "src and dst");
        h.code = D_MULTI;
        h.size = op.src.size;
        check_ref(P, op.dst, rank, false, h.size, w);
        if (ch && ch->type == C_SWITCH) {
          need_chan(true);
          if ((int)ch->ranks.size() > kMaxSrc) bad(CF_E_SHAPE, w + ": switch channel wider than 16 ranks");
          h.flags = F_ZERO;
          for (int r : ch->ranks) {
            check_ref(P, op.src, r, false, h.size, w);
            h.src.push_back({op.src.buf, r, op.src.off, false});
          }
        } else {
          const int peer = (ch && ch->type == C_MEMORY) ? ch->dst : rank;
          if (ch) need_chan(false);
          check_ref(P, op.src, peer, false, h.size, w);
          h.flags = F_ROUND_EACH;
          h.src = {{op.dst.buf, rank, op.dst.off, false}, {op.src.buf, peer, op.src.off, false}};
        }
        h.dst = {{op.dst.buf, rank, op.dst.off, false}};
        if (h.size > 0) out.push_back(h);
        break;
      }
      case P_COPY: {
        need(op.has_src && op.has_dst, "src and dst");
        h.code = D_COPY;
        h.size = op.src.size;
        if (ch && ch->type == C_SWITCH) {
          need_chan(true);
          if ((int)ch->ranks.size() > kMaxDst) bad(CF_E_SHAPE, w + ": switch broadcast wider than 8 ranks");
          check_ref(P, op.src, rank, false, h.size, w);
          h.src = {{op.src.buf, rank, op.src.off, false}};
          for (int r : ch->ranks) {
            check_ref(P, op.dst, r, false, h.size, w);
            h.dst.push_back({op.dst.buf, r, op.dst.off, false});
          }
        } else {
          const int peer = (ch && ch->type == C_MEMORY) ? ch->dst : rank;
          if (ch) need_chan(false);
          check_ref(P, op.src, peer, false, h.size, w);
          check_ref(P, op.dst, rank, false, h.size, w);
          h.src = {{op.src.buf, peer, op.src.off, false}};
          h.dst = {{op.dst.buf, rank, op.dst.off, false}};
        }
        if (h.size > 0) out.push_back(h);
        break;
      }
      case P_REDUCE_PUT: {
        need_chan(false);
        need(op.has_src && op.has_dst && op.has_src2, "src, src2 and dst");
        h.code = D_MULTI;
        h.size = op.src.size;
        h.flags = F_ROUND_EACH;
        check_ref(P, op.src, rank, false, h.size, w);
        check_ref(P, op.src2, rank, false, h.size, w);
        check_ref(P, op.dst, ch->dst, false, h.size, w);
        h.src = {{op.src.buf, rank, op.src.off, false}, {op.src2.buf, rank, op.src2.off, false}};
        h.dst = {{op.dst.buf, ch->dst, op.dst.off, false}};
        if (h.size > 0) out.push_back(h);
        break;
      }
      case P_TB_SYNC:
        h.code = D_SYNC_CTA;
        out.push_back(h);
        break;
      case P_DEVICE_BARRIER:
        h.code = D_DEV_BARRIER;
        h.members = op.group;
        out.push_back(h);
        break;
      default:
        bad(CF_E_SYNTAX, w + ": unknown op");
    }
  }
  return out;
}

// ------------------------------------------------------------------ fusion

bool same_ref(const R& a, const R& b) {
  return a.buf == b.buf && a.rank == b.rank && a.off == b.off && a.packet == b.packet;
}

// byte interval of a ref
void span(const R& r, long long size, int es, long long& lo, long long& hi) {
  const int mul = r.packet ? 2 : 1;
  lo = r.off * es * mul;
  hi = (r.off + size) * es * mul;
}

bool overlaps(const R& a, long long asz, const R& b, long long bsz, int es) {
  if (a.buf != b.buf || a.rank != b.rank) return false;
  long long alo, ahi, blo, bhi;
  span(a, asz, es, alo, ahi);
  span(b, bsz, es, blo, bhi);
  return alo < bhi && blo < ahi;
}

bool is_data(const HOp& h) {
  return h.code == D_MULTI || h.code == D_COPY || h.code == D_PUT_PACKETS || h.code == D_READ_PACKETS ||
         h.code == D_PORT_PUT;
}

bool port_signals(const HOp& h) {
  return h.code == D_PORT_SIGNAL || (h.code == D_PORT_PUT && (h.flags & F_SIGNAL));
}

bool touches(const HOp& h, const R& r, long long size, int es, bool writes_only) {
  if (!is_data(h)) return false;
  for (auto& d : h.dst)
    if (overlaps(d, h.size, r, size, es)) return true;
  if (!writes_only)
    for (auto& s : h.src)
      if (overlaps(s, h.size, r, size, es)) return true;
  return false;
}

// accumulate form: dst[0] += ...  (srcs[0] is the destination itself)
bool accumulate_form(const HOp& h) {
  return h.code == D_MULTI && h.dst.size() == 1 && !(h.flags & F_ZERO) && !h.src.empty() &&
         same_ref(h.src[0], h.dst[0]);
}

void fuse(std::vector<HOp>& ops, int es) {
  bool changed = true;
  while (changed) {
    changed = false;
    for (size_t i = 0; i < ops.size() && !changed; i++) {
      HOp& a = ops[i];
      // (1) reduce chain: A(dst D, D + ...) [sync]* B(dst D, D + ...)
      if (accumulate_form(a) || (a.code == D_MULTI && a.dst.size() == 1 && !(a.flags & F_ZERO))) {
        size_t k = i + 1;
        while (k < ops.size() && ops[k].code == D_SYNC_CTA) k++;
        if (k < ops.size() && accumulate_form(ops[k]) && same_ref(ops[k].dst[0], a.dst[0]) &&
            ops[k].size == a.size && ops[k].flags == a.flags &&
            a.src.size() + ops[k].src.size() - 1 <= (size_t)kMaxSrc) {
          for (size_t s = 1; s < ops[k].src.size(); s++) a.src.push_back(ops[k].src[s]);
          ops.erase(ops.begin() + i + 1, ops.begin() + k + 1);
          changed = true;
          break;
        }
      }
      // (2) copy S0 -> D feeding a later accumulate chain on D
      if (a.code == D_COPY && a.dst.size() == 1 && a.src.size() == 1) {
        for (size_t k = i + 1; k < ops.size(); k++) {
          HOp& b = ops[k];
          if (accumulate_form(b) && same_ref(b.dst[0], a.dst[0]) && b.size == a.size) {
            b.src[0] = a.src[0];
            ops.erase(ops.begin() + i);
            changed = true;
            break;
          }
          if (b.code == D_WAIT || b.code == D_DEV_BARRIER || b.code == D_SYNC_GROUP) break;
          if (touches(b, a.dst[0], a.size, es, false) || touches(b, a.src[0], a.size, es, true)) break;
        }
        if (changed) break;
      }
      // (3) puts of the reduced range become extra destinations of the reduce
      if (a.code == D_MULTI && a.dst.size() < (size_t)kMaxDst) {
        for (size_t k = i + 1; k < ops.size(); k++) {
          HOp& b = ops[k];
          if (b.code == D_SYNC_CTA || b.code == D_SIGNAL) continue;
          if (b.code == D_COPY && b.src.size() == 1 && b.dst.size() == 1 && same_ref(b.src[0], a.dst[0]) &&
              b.size == a.size) {
            bool clash = false;
            for (auto& d : a.dst) clash |= overlaps(d, a.size, b.dst[0], b.size, es);
            for (auto& s : a.src) clash |= overlaps(s, a.size, b.dst[0], b.size, es);
            if (!clash) {
              a.dst.push_back(b.dst[0]);
              ops.erase(ops.begin() + k);
              changed = true;
            }
          }
          break;
        }
        if (changed) break;
      }
    }
  }
  // collapse runs of syncs
  std::vector<HOp> out;
  for (auto& h : ops) {
    if (h.code == D_SYNC_CTA && !out.empty() && out.back().code == D_SYNC_CTA) continue;
    out.push_back(h);
  }
  ops.swap(out);
}

// ------------------------------------------------------------------ sync classification

// Two data ops touch the same bytes in the same per-element layout, so one
// CTA slice covers the same elements in both.
bool aligned_pair(const HOp& a, const HOp& b, int es) {
  auto refs = [](const HOp& h) {
    std::vector<std::pair<R, bool>> v;
    for (auto& s : h.src) v.push_back({s, false});
    for (auto& d : h.dst) v.push_back({d, true});
    return v;
  };
  for (auto& ra : refs(a))
    for (auto& rb : refs(b)) {
      if (!ra.second && !rb.second) continue;  // read/read
      if (!overlaps(ra.first, a.size, rb.first, b.size, es)) continue;
      if (!(a.size == b.size && ra.first.off == rb.first.off && ra.first.packet == rb.first.packet))
        return false;
    }
  return true;
}

void classify_syncs(std::vector<HOp>& ops, int K, int es) {
  if (K == 1) return;
  int last_group = -1;
  for (int s = 0; s < (int)ops.size(); s++) {
    if (ops[s].code == D_WAIT || ops[s].code == D_DEV_BARRIER) last_group = s;
    if (ops[s].code != D_SYNC_CTA) continue;
    bool group = false;
    for (int i = last_group + 1; i < s && !group; i++) {
      if (!is_data(ops[i])) continue;
      for (int k = s + 1; k < (int)ops.size() && !group; k++)
        if (is_data(ops[k]) && !aligned_pair(ops[i], ops[k], es)) group = true;
    }
    if (group) {
      ops[s].code = D_SYNC_GROUP;
      last_group = s;
    }
  }
}

// ------------------------------------------------------------------ zero / private analysis

struct Interval {
  long long lo, hi;
};
bool covered(const std::vector<Interval>& iv, long long lo, long long hi) {
  // iv sorted/merged on insert
  for (auto& x : iv)
    if (x.lo <= lo && hi <= x.hi) return true;
  return false;
}
void add_interval(std::vector<Interval>& iv, long long lo, long long hi) {
  iv.push_back({lo, hi});
  std::sort(iv.begin(), iv.end(), [](const Interval& a, const Interval& b) { return a.lo < b.lo; });
  std::vector<Interval> m;
  for (auto& x : iv) {
    if (!m.empty() && x.lo <= m.back().hi) m.back().hi = std::max(m.back().hi, x.hi);
    else m.push_back(x);
  }
  iv.swap(m);
}

// ------------------------------------------------------------------ read_packets -> reduce fusion

bool data_code(int code) {
  return code == D_MULTI || code == D_COPY || code == D_PUT_PACKETS || code == D_READ_PACKETS ||
         code == D_PORT_PUT;
}

// byte span of a DRef touched by op d (payload or packet layout)
void dref_span(const DevOp& d, const DRef& r, bool packet, int es, uint64_t& lo, uint64_t& hi) {
  lo = r.off;
  hi = r.off + d.size * es * (packet ? 2 : 1);
}

bool same_loc(const DRef& a, const DRef& b) { return a.buf == b.buf && a.rank == b.rank; }

// Is byte range [lo, hi) of location `loc` touched by any data op other than
// ops (pa, ia) and (pb, ib)?
bool touched_elsewhere(const cfPlan* pl, const DRef& loc, uint64_t lo, uint64_t hi, size_t pa, size_t ia,
                       size_t pb, size_t ib) {
  for (size_t p = 0; p < pl->prog_ops.size(); p++)
    for (size_t i = 0; i < pl->prog_ops[p].size(); i++) {
      if ((p == pa && i == ia) || (p == pb && i == ib)) continue;
      const DevOp& d = pl->prog_ops[p][i];
      if (!data_code(d.code)) continue;
      for (int k = 0; k < d.nsrc + d.ndst; k++) {
        const bool is_src = k < d.nsrc;
        const DRef& r = is_src ? d.src[k] : d.dst[k - d.nsrc];
        if (!same_loc(r, loc)) continue;
        const bool packet = (d.code == D_READ_PACKETS && is_src) || (d.code == D_PUT_PACKETS && !is_src) ||
                            (d.code == D_MULTI && is_src && ((d.pkt_mask >> k) & 1u));
        uint64_t a0, a1;
        dref_span(d, r, packet, pl->es, a0, a1);
        if (a0 < hi && lo < a1) return true;
      }
    }
  return false;
}

// [read_packets P_k -> T_k]* ; tb_sync ; reduce(... T_k ...)  ==>  reduce(... P_k ...)
// when T_k is scratch nobody else touches: the reduction reads the LL16
// packets directly (one pass, no temporary), exactly the one-shot LL kernel.
void fuse_packet_reads(cfPlan* pl) {
  // Always fused: on the compiled LL kernel (one unit per thread, every
  // source in flight) the fused reduce wins at every size (2pa_ll plan b=1
  // 8.9 -> 8.3 us: no sync, no scratch round trip).  (The interpreter, which
  // runs what does not compile, preferred the separate batched read below
  // 8 KiB per range: b=1 12.1 -> 11.4 us.)
  long long min_bytes = 0;
  if (const char* ev = getenv("CF_PLAN_FUSE_READS_MIN")) min_bytes = atoll(ev);   // diagnostic
  if (const char* ev = getenv("CF_PLAN_FUSE_READS"))   // diagnostic: 0 keeps read_packets separate
    if (atoi(ev) == 0) return;
  for (size_t p = 0; p < pl->prog_ops.size(); p++) {
    auto& ops = pl->prog_ops[p];
    for (size_t m = 0; m < ops.size(); m++) {
      DevOp& M = ops[m];
      if (M.code != D_MULTI || !(M.flags & F_VEC)) continue;
      for (size_t r = m; r-- > 0;) {
        DevOp& R = ops[r];
        if (R.code == D_SYNC_CTA) continue;
        if (R.code != D_READ_PACKETS) break;
        if (!(R.flags & F_LL16) || R.size != M.size) break;
        if ((long long)R.size * pl->es < min_bytes) break;
        for (int k = 0; k < R.nsrc; k++) {
          for (int s = 0; s < M.nsrc; s++) {
            if ((M.pkt_mask >> s) & 1u) continue;
            if (!same_loc(M.src[s], R.dst[k]) || M.src[s].off != R.dst[k].off) continue;
            if (R.dst[k].buf != kAbsolute) continue;   // plan-owned scratch only, never user I/O
            uint64_t lo, hi;
            dref_span(R, R.dst[k], false, pl->es, lo, hi);
            if (touched_elsewhere(pl, R.dst[k], lo, hi, p, r, p, m)) continue;
            M.src[s] = R.src[k];
            M.llflag_k[s] = R.llflag_k[k];
            M.pkt_mask |= 1u << s;
            for (int q = k; q + 1 < R.nsrc; q++) {   // drop pair k from the batch
              R.src[q] = R.src[q + 1];
              R.dst[q] = R.dst[q + 1];
              R.llflag_k[q] = R.llflag_k[q + 1];
            }
            R.nsrc--;
            R.ndst--;
            k--;
            break;
          }
        }
        if (R.nsrc == 0) R.code = D_NOP;
        break;
      }
    }
    std::vector<DevOp> keep;
    for (auto& d : ops)
      if (d.code != D_NOP) keep.push_back(d);
    pl->n_device_ops -= (int)(ops.size() - keep.size());
    ops.swap(keep);
  }
}

}  // namespace

// ------------------------------------------------------------------ load

cfStatus finalize(cfPlan* pl);

cfStatus load(cfComm* c, const char* json, size_t len, int dtype_override, cfPlan** out) {
  std::unique_ptr<cfPlan> pl(new cfPlan());
  pl->comm = c;
  CF_TRY(parse(json, len, dtype_override, pl->ir));
  Plan& P = pl->ir;
  try {
    if (!P.lowered) bad(CF_E_SHAPE, "cannot execute a pre-lowering document; lower it first");
    if (P.nranks != c->nranks)
      bad(CF_E_RANK_MISMATCH, "plan wants " + std::to_string(P.nranks) + " ranks, world has " +
                                  std::to_string(c->nranks));
    if ((int)P.bufs.size() > kMaxBufs) bad(CF_E_SHAPE, "plans are limited to 16 buffers");
    for (size_t b = 0; b < P.bufs.size(); b++) {
      if (P.bufs[b].elems <= 0) bad(CF_E_BAD_SIZE, "buffer '" + P.bufs[b].id + "' has non-positive elems");
      if (P.bufs[b].rank < -1 || P.bufs[b].rank >= P.nranks) bad(CF_E_OOB, "buffer '" + P.bufs[b].id + "' rank out of range");
      if (P.bufs[b].kind == B_INPUT) { if (pl->in_buf >= 0) bad(CF_E_SHAPE, "plan must declare exactly one input buffer, found 2"); pl->in_buf = (int)b; }
      if (P.bufs[b].kind == B_OUTPUT) { if (pl->out_buf >= 0) bad(CF_E_SHAPE, "plan must declare exactly one output buffer, found 2"); pl->out_buf = (int)b; }
    }
    if (pl->in_buf < 0) bad(CF_E_SHAPE, "plan must declare exactly one input buffer, found 0");
    if (pl->out_buf < 0) bad(CF_E_SHAPE, "plan must declare exactly one output buffer, found 0");
    if (P.bufs[pl->in_buf].rank != -1 || P.bufs[pl->out_buf].rank != -1)
      bad(CF_E_SHAPE, "input and output buffers must exist on every rank");
    for (auto& g : P.progs) check_rank(P, g.rank, "program");
    for (size_t i = 0; i < P.progs.size(); i++)
      for (size_t k = i + 1; k < P.progs.size(); k++)
        if (P.progs[i].rank == P.progs[k].rank && P.progs[i].tb == P.progs[k].tb)
          bad(CF_E_SHAPE, "duplicate program for rank " + std::to_string(P.progs[i].rank) + " tb " +
                              std::to_string(P.progs[i].tb));
  } catch (const Fail& f) {
    return fail(f.s, "%s", f.m.c_str());
  }
  pl->dtype = P.dtype;
  pl->es = dtype_size(P.dtype);
  const int es = pl->es, n = P.nranks;

  // programs sorted by (rank, tb); ranks without a program get an empty one so
  // the call-bracketing rank barrier always has a participant.
  std::vector<int> order(P.progs.size());
  for (size_t i = 0; i < order.size(); i++) order[i] = (int)i;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return std::make_pair(P.progs[a].rank, P.progs[a].tb) < std::make_pair(P.progs[b].rank, P.progs[b].tb);
  });
  std::vector<std::vector<HOp>> hops;
  std::vector<int> prank, ptb;
  try {
    int next = 0;
    for (int r = 0; r < n; r++) {
      bool any = false;
      while (next < (int)order.size() && P.progs[order[next]].rank == r) {
        hops.push_back(lower_program(P, order[next], es));
        prank.push_back(r);
        ptb.push_back(P.progs[order[next]].tb);
        next++;
        any = true;
      }
      if (!any) { hops.emplace_back(); prank.push_back(r); ptb.push_back(1 << 30); }
    }
  } catch (const Fail& f) {
    return fail(f.s, "%s", f.m.c_str());
  }
  for (auto& h : hops) fuse(h, es);

  // CTAs per program: enough threads for the largest data op, all programs
  // of a device co-resident.
  long long max_bytes = 0;
  bool packets = false;   // LL plans: packet ops run one 8-byte payload unit per thread
  bool port = false;
  for (auto& h : hops) {
    int run = 0;   // consecutive packet ops of one kind and size: they batch into one device op
    for (size_t i = 0; i < h.size(); i++) {
      const HOp& o = h[i];
      const bool pkt = o.code == D_PUT_PACKETS || o.code == D_READ_PACKETS;
      // (paired puts -- different payload ranges -- and packet reads; a
      // payload broadcast to several ranges stays one unit per thread)
      const bool batch = pkt && i && h[i - 1].code == o.code && h[i - 1].size == o.size &&
                         (o.code == D_READ_PACKETS || !(h[i - 1].src.size() && o.src.size() &&
                                                        h[i - 1].src[0].buf == o.src[0].buf && h[i - 1].src[0].rank == o.src[0].rank &&
                                                        h[i - 1].src[0].off == o.src[0].off));
      run = batch ? std::min(run + 1, kMaxDst) : 1;
      // a batched packet op spreads its ranges over the threads (one unit each)
      if (is_data(o)) max_bytes = std::max(max_bytes, o.size * es * (pkt ? run : 1));
      packets |= pkt;
      port |= o.code == D_PORT_PUT || o.code == D_PORT_SIGNAL || o.code == D_PORT_FLUSH;
    }
  }
  // the smallest interpreter class covering every op of the plan (MULTI ops
  // take packet sources only where the plan has packet ops to fuse)
  pl->cls = (packets ? 1 : 0) | (port ? 2 : 0);
  if (const char* ev = getenv("CF_PLAN_CLASS")) pl->cls = atoi(ev);   // diagnostic: force a class
  const void* kernel = plan_kernel_for(pl->dtype, pl->cls);
  int cap = INT32_MAX, progs_per_dev_max = 1;
  pl->mp = c->multiprocess;
  pl->me = c->local[0].rank;
  {
    // programs co-resident per device; one process per GPU: every rank
    // computes the same K from the busiest rank (lanes are indexed by K)
    std::map<int, int> per_dev;
    if (pl->mp) {
      std::map<int, int> per_rank;
      int busiest = 0;
      for (int r : prank) busiest = std::max(busiest, ++per_rank[r]);
      per_dev[c->local[0].dev] = busiest;
    } else {
      for (int r : prank) per_dev[c->local[r].dev]++;
    }
    for (auto& kv : per_dev) {
      progs_per_dev_max = std::max(progs_per_dev_max, kv.second);
      int nb = 0;
      cudaSetDevice(kv.first);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, pl->threads, kPlanWindow * sizeof(DevOp)) !=
          cudaSuccess)
        nb = 1;
      cap = std::min(cap, std::max(nb, 1) * c->sm_count[kv.first] / kv.second);
    }
  }
  if (cap < 1) return fail(CF_E_CONFIG, "plan has more programs per device than co-resident CTAs");
  // a quarter of a 16-byte vector (half an 8-byte packet unit) per thread and
  // CTA: small plans are latency-bound, more CTAs keep more loads in flight
  // (C5 2pa plan b=4 4.8 -> 3.8 us, b=16 5.1 -> 4.1 us; 2pa_ll b=4 9.2 -> 8.6
  // us; b >= 64 unchanged: the 32-CTA cap applies; was one vector / unit per
  // thread, 1pa plan b=1 11.6 -> 9.5 us before that)
  long long per_cta = (long long)pl->threads * 4;
  if (const char* ev = getenv("CF_PLAN_BYTES_PER_CTA")) per_cta = std::max(1LL, atoll(ev));   // diagnostic
  pl->K = (int)std::max(1LL, std::min<long long>({(max_bytes + per_cta - 1) / per_cta, (long long)cap, 32LL}));
  const int K = pl->K;

  try {
    for (auto& h : hops) classify_syncs(h, K, es);
  } catch (const Fail& f) {
    return fail(f.s, "%s", f.m.c_str());
  }

  // One launch holding every rank: a wait after a program's last data op only
  // guards data the call's end publishes anyway (the kernel boundary is a
  // barrier over all ranks), so such tail waits -- and the signals of channels
  // whose every wait is a tail wait -- are dropped.
  if (c->groups.size() == 1 && (int)c->local.size() == n) {
    std::vector<char> all_tail(P.chans.size(), 1);
    std::vector<std::vector<char>> tail(hops.size());
    // a channel with fewer signals than waits deadlocks in the reference
    // (cf/sched.py:93-99); keep its waits so the device reports E_DEADLOCK too
    std::vector<long long> nsig(P.chans.size(), 0), nwait(P.chans.size(), 0);
    for (auto& h : hops)
      for (auto& o : h) {
        if (o.code == D_SIGNAL || port_signals(o)) nsig[o.chan]++;
        if (o.code == D_WAIT) nwait[o.chan]++;
      }
    for (size_t ch = 0; ch < P.chans.size(); ch++)
      if (nsig[ch] < nwait[ch]) all_tail[ch] = 0;
    for (size_t p = 0; p < hops.size(); p++) {
      int last = -1;
      for (int i = 0; i < (int)hops[p].size(); i++)
        if (is_data(hops[p][i])) last = i;
      tail[p].assign(hops[p].size(), 0);
      for (int i = 0; i < (int)hops[p].size(); i++) {
        if (hops[p][i].code != D_WAIT) continue;
        tail[p][i] = i > last;
        if (i < last) all_tail[hops[p][i].chan] = 0;
      }
    }
    for (size_t p = 0; p < hops.size(); p++) {
      std::vector<HOp> keep;
      for (size_t i = 0; i < hops[p].size(); i++) {
        HOp& o = hops[p][i];
        const bool elide = o.chan >= 0 && all_tail[o.chan];
        if (o.code == D_WAIT && tail[p][i] && elide) continue;
        if ((o.code == D_SIGNAL || o.code == D_PORT_SIGNAL) && elide) continue;
        if (o.code == D_PORT_PUT && elide) o.flags &= ~F_SIGNAL;
        keep.push_back(o);
      }
      hops[p].swap(keep);
    }
  }

  // signals per call per channel; waits restricted to one program per channel
  std::vector<long long> sig(P.chans.size(), 0);
  std::vector<int> waiter(P.chans.size(), -1);
  long long max_flag = 1;
  std::vector<int> port_signaler(P.chans.size(), -1);
  for (size_t p = 0; p < hops.size(); p++)
    for (auto& o : hops[p]) {
      if (o.code == D_SIGNAL || port_signals(o)) sig[o.chan]++;
      if (port_signals(o)) {   // the proxy writes absolute counts: one signaling block per channel
        if (port_signaler[o.chan] >= 0 && port_signaler[o.chan] != (int)p)
          return fail(CF_E_PROTOCOL, "port channel '%s' is signalled from more than one thread block",
                      P.chans[o.chan].id.c_str());
        port_signaler[o.chan] = (int)p;
        pl->uses_port = true;
      }
      if (o.code == D_PORT_PUT || o.code == D_PORT_FLUSH) pl->uses_port = true;
      if (o.code == D_WAIT) {
        if (waiter[o.chan] >= 0 && waiter[o.chan] != (int)p)
          return fail(CF_E_PROTOCOL, "channel '%s' is waited on by more than one thread block",
                      P.chans[o.chan].id.c_str());
        waiter[o.chan] = (int)p;
      }
      if (o.code == D_PUT_PACKETS || o.code == D_READ_PACKETS) max_flag = std::max<long long>(max_flag, o.llflag);
    }
  pl->flag_stride = (uint32_t)(max_flag + 1);

  // barrier counters: one per program for group syncs, one per device_barrier key
  int nbar = 0;
  std::map<std::pair<int, std::vector<int>>, int> bar_key;
  std::map<std::pair<int, std::vector<int>>, std::map<int, int>> bar_count;  // key -> program -> count
  std::vector<int> gbar(hops.size(), -1);
  for (size_t p = 0; p < hops.size(); p++) {
    int gsyncs = 0, m = 0;
    for (auto& o : hops[p]) gsyncs += o.code == D_SYNC_GROUP;
    if (gsyncs) gbar[p] = nbar++;
    std::map<std::pair<int, std::vector<int>>, int> occ;
    for (auto& o : hops[p]) {
      if (o.code == D_SYNC_GROUP) {
        o.chan = gbar[p];
        o.peer = ++m;                      // m
        o.members.assign(1, gsyncs);       // per_call stash
      } else if (o.code == D_DEV_BARRIER) {
        std::vector<int> mem = o.members;
        if (mem.empty())
          for (size_t q = 0; q < hops.size(); q++)
            if (prank[q] == prank[p] && ptb[q] != (1 << 30)) mem.push_back(ptb[q]);
        std::sort(mem.begin(), mem.end());
        auto key = std::make_pair(prank[p], mem);
        if (!bar_key.count(key)) bar_key[key] = nbar++;
        o.chan = bar_key[key];
        o.peer = ++occ[key];
        bar_count[key][(int)p] = o.peer;
        o.members = mem;
      }
    }
  }
  for (auto& kv : bar_count) {
    const auto& mem = kv.first.second;
    int per_call = -1;
    for (auto& pc : kv.second) {
      if (per_call >= 0 && pc.second != per_call)
        return fail(CF_E_PROTOCOL, "device_barrier members disagree on the barrier count");
      per_call = pc.second;
    }
    for (int tb : mem) {
      bool found = false;
      for (size_t q = 0; q < hops.size(); q++) found |= prank[q] == kv.first.first && ptb[q] == tb;
      if (!found) return fail(CF_E_OOB, "device_barrier names tb %d, which has no program", tb);
    }
    if ((int)kv.second.size() != (int)mem.size())
      return fail(CF_E_PROTOCOL, "device_barrier member without a matching barrier");
  }
  pl->nbars = nbar;

  // zeroing and private-input analysis
  std::vector<std::set<int>> zero(n);
  for (size_t p = 0; p < hops.size(); p++) {
    std::map<std::pair<int, int>, std::vector<Interval>> written;
    for (auto& o : hops[p]) {
      if (!is_data(o)) continue;
      for (auto& s : o.src) {
        if (s.packet || s.buf == pl->in_buf) continue;
        long long lo, hi;
        span(s, o.size, es, lo, hi);
        auto& iv = written[{s.buf, s.rank}];
        if (s.rank != prank[p] || !covered(iv, lo, hi)) zero[s.rank].insert(s.buf);
      }
      for (auto& d : o.dst) {
        if (d.buf == pl->in_buf) pl->input_private = true;
        if (d.packet) continue;
        long long lo, hi;
        span(d, o.size, es, lo, hi);
        add_interval(written[{d.buf, d.rank}], lo, hi);
      }
    }
  }
  pl->zero_bufs.assign(n, {});
  for (int r = 0; r < n; r++)
    for (int b : zero[r]) {
      if (P.bufs[b].rank != -1 && P.bufs[b].rank != r) continue;
      if ((int)pl->zero_bufs[r].size() < kMaxZero) pl->zero_bufs[r].push_back(b);
    }

  // encode device ops
  for (size_t p = 0; p < hops.size(); p++) {
    std::vector<DevOp> dv;
    std::map<int, int> wm, pm;
    for (auto& o : hops[p]) {
      DevOp d;
      memset(&d, 0, sizeof(d));
      d.code = (uint8_t)o.code;
      d.size = (uint64_t)o.size;
      d.llflag = o.llflag;
      d.flags = (uint8_t)(o.flags & (F_ZERO | F_ROUND_EACH));
      d.nsrc = (uint8_t)o.src.size();
      d.ndst = (uint8_t)o.dst.size();
      bool vec = true;
      for (size_t k = 0; k < o.src.size(); k++) {
        d.src[k] = {o.src[k].buf, o.src[k].rank, (uint64_t)(o.src[k].off * es * (o.src[k].packet ? 2 : 1))};
        vec &= (d.src[k].off % 16) == 0;
      }
      for (size_t k = 0; k < o.dst.size(); k++) {
        d.dst[k] = {o.dst[k].buf, o.dst[k].rank, (uint64_t)(o.dst[k].off * es * (o.dst[k].packet ? 2 : 1))};
        vec &= (d.dst[k].off % 16) == 0;
      }
      if (vec) d.flags |= F_VEC;
      if (o.code == D_PUT_PACKETS || o.code == D_READ_PACKETS) {
        const R& pay = o.code == D_PUT_PACKETS ? o.src[0] : o.dst[0];
        if ((pay.off * es) % 8 == 0 && (o.size * es) % 8 == 0) d.flags |= F_LL16;
      }
      DevOp* prev = dv.empty() ? nullptr : &dv.back();
      switch (o.code) {
        case D_PORT_PUT:
        case D_PORT_SIGNAL:
          d.id = o.chan;
          d.peer = o.peer;
          d.flags |= (uint8_t)(o.flags & F_SIGNAL);
          if (port_signals(o)) {
            d.m = (uint64_t)(++pm[o.chan]);
            d.per_call = (uint64_t)sig[o.chan];
          }
          break;
        case D_SIGNAL:   // consecutive signals batch into one op (one thread per signal)
          if (prev && prev->code == D_SIGNAL && prev->ndst < kMaxDst) {
            prev->dst[prev->ndst++] = {o.chan, o.peer, 0};
            continue;
          }
          d.ndst = 1;
          d.dst[0] = {o.chan, o.peer, 0};
          break;
        case D_WAIT: {   // consecutive waits batch into one op (polled in parallel)
          const DRef w = {o.chan, (int32_t)sig[o.chan], (uint64_t)(++wm[o.chan])};
          if (prev && prev->code == D_WAIT && prev->nsrc < kMaxSrc) {
            prev->src[prev->nsrc++] = w;
            continue;
          }
          d.nsrc = 1;
          d.src[0] = w;
          break;
        }
        case D_PUT_PACKETS: {  // batched: one payload to several peers (one load, ndst packet stores),
                               // or several (payload -> peer) pairs with all loads in flight
          const bool like = prev && prev->code == D_PUT_PACKETS && prev->size == d.size &&
                            prev->llflag == d.llflag && prev->ndst < kMaxDst &&
                            (prev->flags & F_LL16) == (d.flags & F_LL16);
          const bool same_src = like && !(prev->flags & F_PAIRED) && prev->src[0].buf == d.src[0].buf &&
                                prev->src[0].rank == d.src[0].rank && prev->src[0].off == d.src[0].off;
          if (same_src) {
            prev->dst[prev->ndst++] = d.dst[0];
            continue;
          }
          if (like && (prev->flags & F_PAIRED || prev->ndst == 1)) {
            // no packet range of the batch may overlap a payload range of it
            const long long len_pkt = 2 * d.size * es, len_pay = d.size * es;
            auto ovl = [](const DRef& x, long long lx, const DRef& y, long long ly) {
              return x.buf == y.buf && x.rank == y.rank && (long long)x.off < (long long)y.off + ly &&
                     (long long)y.off < (long long)x.off + lx;
            };
            bool ok = true;
            for (int k = 0; k < prev->ndst && ok; k++)
              ok = !ovl(prev->dst[k], len_pkt, d.src[0], len_pay) && !ovl(d.dst[0], len_pkt, prev->src[k], len_pay);
            if (ok) {
              prev->flags |= F_PAIRED;
              prev->src[prev->nsrc++] = d.src[0];
              prev->dst[prev->ndst++] = d.dst[0];
              continue;
            }
          }
          break;
        }
        case D_READ_PACKETS: {  // several packet ranges drained together, loads in flight
          d.llflag_k[0] = d.llflag;
          bool ok = prev && prev->code == D_READ_PACKETS && prev->size == d.size && prev->nsrc < kMaxDst &&
                    (prev->flags & F_LL16) == (d.flags & F_LL16);
          if (ok) {  // no range of the batch may overlap another's (order-free merge)
            const long long len_pkt = 2 * d.size * es, len_pay = d.size * es;
            auto ovl = [](const DRef& x, long long lx, const DRef& y, long long ly) {
              return x.buf == y.buf && x.rank == y.rank && (long long)x.off < (long long)y.off + ly &&
                     (long long)y.off < (long long)x.off + lx;
            };
            for (int k = 0; k < prev->nsrc && ok; k++)
              ok = !ovl(prev->dst[k], len_pay, d.dst[0], len_pay) && !ovl(prev->dst[k], len_pay, d.src[0], len_pkt) &&
                   !ovl(d.dst[0], len_pay, prev->src[k], len_pkt);
          }
          if (ok) {
            prev->llflag_k[prev->nsrc] = d.llflag;
            prev->src[prev->nsrc++] = d.src[0];
            prev->dst[prev->ndst++] = d.dst[0];
            continue;
          }
          break;
        }
        case D_SYNC_GROUP:
          d.id = o.chan;
          d.m = (uint64_t)o.peer;
          d.per_call = (uint64_t)o.members[0];
          d.members = (uint64_t)K;
          break;
        case D_DEV_BARRIER:
          d.id = o.chan;
          d.m = (uint64_t)o.peer;
          d.per_call = (uint64_t)bar_count[{prank[p], o.members}][(int)p];
          d.members = (uint64_t)(o.members.size() * K);
          break;
        default:
          break;
      }
      dv.push_back(d);
    }
    pl->n_device_ops += (int)dv.size();
    pl->prog_ops.push_back(dv);
  }
  pl->prog_rank = prank;
  pl->prog_tb = ptb;
  // shared-memory window: the longest program, up to kPlanWindow ops
  for (auto& prog : pl->prog_ops) pl->window = std::max(pl->window, (int)std::min<size_t>(prog.size(), kPlanWindow));

  // per-rank plan heap: [PlanState | lanes | bars | buffers]
  pl->state_off = 0;
  pl->lanes_off = round_up(sizeof(PlanState), 256);
  pl->bars_off = round_up(pl->lanes_off + P.chans.size() * K * sizeof(uint64_t) + 8, 256);
  size_t off = round_up(pl->bars_off + (size_t)(nbar + 1) * sizeof(uint64_t), 256);
  pl->buf_off.assign(P.bufs.size(), 0);
  for (size_t b = 0; b < P.bufs.size(); b++) {
    if ((int)b == pl->out_buf || ((int)b == pl->in_buf && !pl->input_private)) continue;
    pl->buf_off[b] = off;
    off += round_up((size_t)P.bufs[b].elems * es, 256);
  }
  pl->heap_bytes = round_up(off, 4096);
  int prev_dev = -1;
  cudaGetDevice(&prev_dev);
  pl->heap.assign(n, nullptr);
  pl->heap_mapped.assign(n, false);
  for (int r = 0; r < n; r++) {
    if (pl->mp && r != pl->me) continue;   // peers' heaps arrive through cfPlanConnect
    if (cudaSetDevice(c->local[pl->mp ? 0 : r].dev) != cudaSuccess ||
        cudaMalloc((void**)&pl->heap[r], pl->heap_bytes) != cudaSuccess ||
        cudaMemset(pl->heap[r], 0, pl->heap_bytes) != cudaSuccess) {
      cudaSetDevice(prev_dev);
      cfPlanDestroy(pl.release());
      return fail(CF_E_CUDA, "plan heap allocation failed");
    }
    PlanState st;
    memset(&st, 0, sizeof(st));
    st.base.timeout_ns = c->cfg.spin_timeout_ns;
    cudaMemcpy(pl->heap[r] + pl->state_off, &st, sizeof(st), cudaMemcpyHostToDevice);
  }
  pl->has_prologue = pl->input_private;
  for (auto& z : pl->zero_bufs) pl->has_prologue |= !z.empty();
  cudaSetDevice(prev_dev);
  if (pl->mp) {   // finalized by cfPlanConnect once every heap is mapped
    *out = pl.release();
    return CF_OK;
  }
  const cfStatus fs = finalize(pl.get());
  if (fs != CF_OK) {
    cfPlanDestroy(pl.release());
    return fs;
  }
  *out = pl.release();
  return CF_OK;
}

// Do data ops x and y touch a common byte with at least one of them writing it?
bool ops_conflict(const DevOp& x, const DevOp& y, int es) {
  for (int i = 0; i < x.nsrc + x.ndst; i++)
    for (int k = 0; k < y.nsrc + y.ndst; k++) {
      const bool xw = i >= x.nsrc, yw = k >= y.nsrc;
      if (!xw && !yw) continue;
      const DRef& rx = xw ? x.dst[i - x.nsrc] : x.src[i];
      const DRef& ry = yw ? y.dst[k - y.nsrc] : y.src[k];
      if (!same_loc(rx, ry)) continue;
      auto pkt = [](const DevOp& d, int j, bool w) {
        return (d.code == D_READ_PACKETS && !w) || (d.code == D_PUT_PACKETS && w) ||
               (d.code == D_MULTI && !w && ((d.pkt_mask >> j) & 1u));
      };
      uint64_t a0, a1, b0, b1;
      dref_span(x, rx, pkt(x, i, xw), es, a0, a1);
      dref_span(y, ry, pkt(y, k, yw), es, b0, b1);
      if (a0 < b1 && b0 < a1) return true;
    }
  return false;
}

// CTA-local syncs that another barrier already provides: first / last op of a
// program (the staging barrier / the end-of-call barrier), next to an op that
// starts with a block barrier (signal, port ops, group / device barriers,
// another sync) or after one that ends with one (wait, port flush, group /
// device barriers).  Fusion leaves such syncs behind (the hoisted copy's).
void drop_redundant_syncs(cfPlan* pl) {
  auto starts_bar = [](uint8_t c) {
    return c == D_SIGNAL || c == D_SYNC_GROUP || c == D_DEV_BARRIER || c == D_PORT_PUT || c == D_PORT_SIGNAL ||
           c == D_SYNC_CTA || c == D_WAIT;
  };
  auto ends_bar = [](uint8_t c) {
    return c == D_WAIT || c == D_SYNC_GROUP || c == D_DEV_BARRIER || c == D_PORT_FLUSH || c == D_SYNC_CTA;
  };
  for (auto& ops : pl->prog_ops) {
    std::vector<DevOp> keep;
    for (size_t i = 0; i < ops.size(); i++) {
      if (ops[i].code == D_SYNC_CTA) {
        const bool first = keep.empty(), last = i + 1 == ops.size();
        if (first || last || ends_bar(keep.back().code) || starts_bar(ops[i + 1].code)) continue;
      }
      keep.push_back(ops[i]);
    }
    pl->n_device_ops -= (int)(ops.size() - keep.size());
    ops.swap(keep);
  }
  // A CTA-local sync whose two sides (the data ops back to the previous and
  // on to the next non-data op) share no location with a write on either
  // side orders nothing (e.g. the 1pa plan's packet scatter vs its fused
  // read-reduce: packets written by peers are ordered by their flags).
  const int es = pl->es;
  auto refs_conflict = [&](const DevOp& x, const DevOp& y) { return ops_conflict(x, y, es); };
  auto is_data = [](uint8_t c) { return c == D_MULTI || c == D_COPY || c == D_PUT_PACKETS || c == D_READ_PACKETS; };
  for (auto& ops : pl->prog_ops) {
    for (size_t i = 0; i < ops.size(); i++) {
      if (ops[i].code != D_SYNC_CTA) continue;
      size_t a = i, b = i + 1;
      while (a > 0 && is_data(ops[a - 1].code)) a--;
      while (b < ops.size() && is_data(ops[b].code)) b++;
      bool hazard = a == i || b == i + 1;   // a non-data neighbour: keep
      for (size_t x = a; x < i && !hazard; x++)
        for (size_t y = i + 1; y < b && !hazard; y++) hazard = refs_conflict(ops[x], ops[y]);
      if (!hazard) {
        ops.erase(ops.begin() + i);
        pl->n_device_ops--;
        i--;
      }
    }
  }
}

// Streamed packet pairs of the compiled LL kernel.  A program's unpaired
// PUT_PACKETS followed by a MULTI of the same size that reduces LL16 packets
// may run interleaved (a thread reduces unit u one iteration after putting
// it) when the pairs form a closed, symmetric exchange:
//  - every pair has the same size (same CTA slices, same unit -> thread map);
//  - each packet source of a pair's MULTI is exactly the range one pair's
//    PUT writes (same location and base, same plan flag);
//  - nothing else in the plan touches the ranges the pair PUTs write;
//  - the PUT's source and the MULTI's I/O destinations start at the same
//    offset (a thread only overwrites units it already put when in place).
// Then the thread that puts unit u on every rank has the same index and
// iteration, and the thread waiting for unit u at iteration k depends only on
// puts of iteration k - 1 (the hand one-shot's argument); without these
// conditions the plan runs op by op.
void compute_ll_stream(cfPlan* pl) {
  const size_t np = pl->prog_ops.size();
  pl->ll_stream.assign(np, -1);
  if (!pl->ll_ok) return;
  if (const char* ev = getenv("CF_PLAN_LL_STREAM"))   // diagnostic: 0 runs op by op
    if (atoi(ev) == 0) return;
  const int es = pl->es;
  std::vector<int> cand(np, -1);
  uint64_t size = 0;
  bool any = false;
  for (size_t p = 0; p < np; p++) {
    const auto& ops = pl->prog_ops[p];
    for (size_t i = 0; i + 1 < ops.size(); i++) {
      const DevOp &u = ops[i], &m = ops[i + 1];
      if (u.code != D_PUT_PACKETS || (u.flags & F_PAIRED) || !(u.flags & F_LL16)) continue;
      if (m.code != D_MULTI || !(m.flags & F_VEC) || !m.pkt_mask || m.size != u.size) continue;
      if (any && u.size != size) return;
      bool io_ok = true;
      for (int d = 0; d < m.ndst; d++)
        if (m.dst[d].buf != kAbsolute && u.src[0].buf != kAbsolute && m.dst[d].off != u.src[0].off) io_ok = false;
      if (!io_ok) return;
      cand[p] = (int)i;
      size = u.size;
      any = true;
      break;
    }
  }
  if (!any) return;
  struct Range {
    size_t p;
    int k;
    DRef loc;
    uint64_t lo, hi;
    uint32_t flag;
  };
  std::vector<Range> put_ranges;
  for (size_t p = 0; p < np; p++) {
    if (cand[p] < 0) continue;
    const DevOp& u = pl->prog_ops[p][cand[p]];
    for (int k = 0; k < u.ndst; k++) {
      uint64_t lo, hi;
      dref_span(u, u.dst[k], true, es, lo, hi);
      put_ranges.push_back({p, k, u.dst[k], lo, hi, u.llflag});
    }
  }
  for (size_t p = 0; p < np; p++)
    for (size_t i = 0; i < pl->prog_ops[p].size(); i++) {
      const DevOp& d = pl->prog_ops[p][i];
      if (!data_code(d.code)) continue;
      const bool pair_put = cand[p] == (int)i, pair_multi = cand[p] >= 0 && cand[p] + 1 == (int)i;
      for (int k = 0; k < d.nsrc + d.ndst; k++) {
        const bool is_src = k < d.nsrc;
        const DRef& r = is_src ? d.src[k] : d.dst[k - d.nsrc];
        const bool packet = (d.code == D_READ_PACKETS && is_src) || (d.code == D_PUT_PACKETS && !is_src) ||
                            (d.code == D_MULTI && is_src && ((d.pkt_mask >> k) & 1u));
        uint64_t lo, hi;
        dref_span(d, r, packet, es, lo, hi);
        bool matched = false;
        for (const Range& R : put_ranges) {
          if (!same_loc(r, R.loc) || !(lo < R.hi && R.lo < hi)) continue;
          if (pair_put && !is_src && R.p == p && R.k == k - d.nsrc) continue;   // the range itself
          if (pair_multi && packet && lo == R.lo && hi == R.hi && d.llflag_k[k] == R.flag) {
            matched = true;
            continue;
          }
          return;   // touched by something outside the exchange
        }
        if (pair_multi && packet && !matched) return;   // a packet source no pair writes
      }
    }
  for (size_t p = 0; p < np; p++) pl->ll_stream[p] = cand[p];
}

// Reduce-then-broadcast of the compiled LL kernel: MULTI m ; sync ; an
// unpaired PUT_PACKETS whose source is m's destination (same location, base
// and size) -- the two-shot LL plan's phase-2 scatter of the reduced chunk.
// Both ops map unit u to the same thread, so the thread broadcasts the value
// it just reduced (no sync, no reload) when m and the PUT are the only
// conflicting pair across that sync.
void compute_ll_fuse_put(cfPlan* pl) {
  const size_t np = pl->prog_ops.size();
  pl->ll_fuse_put.assign(np, -1);
  if (!pl->ll_ok) return;
  if (const char* ev = getenv("CF_PLAN_LL_FUSE_PUT"))   // diagnostic: 0 keeps the sync and the reload
    if (atoi(ev) == 0) return;
  const int es = pl->es;
  auto is_data = [](uint8_t c) { return c == D_MULTI || c == D_COPY || c == D_PUT_PACKETS || c == D_READ_PACKETS; };
  for (size_t p = 0; p < np; p++) {
    const auto& ops = pl->prog_ops[p];
    for (size_t i = 0; i + 2 < ops.size(); i++) {
      const DevOp &m = ops[i], &u = ops[i + 2];
      if ((m.code != D_MULTI && m.code != D_COPY) || !(m.flags & F_VEC) || ops[i + 1].code != D_SYNC_CTA) continue;
      if (u.code != D_PUT_PACKETS || (u.flags & F_PAIRED) || !(u.flags & F_LL16) || u.size != m.size) continue;
      bool src_is_dst = false, misaligned = false;
      for (int d = 0; d < m.ndst; d++) {
        const bool same = same_loc(m.dst[d], u.src[0]) && m.dst[d].off == u.src[0].off;
        src_is_dst |= same;
        uint64_t a0, a1, b0, b1;
        dref_span(m, m.dst[d], false, es, a0, a1);
        dref_span(u, u.src[0], false, es, b0, b1);
        misaligned |= !same && same_loc(m.dst[d], u.src[0]) && a0 < b1 && b0 < a1;
      }
      if (!src_is_dst || misaligned) continue;
      DevOp writes = u;   // the PUT's packet stores against everything m touches
      writes.nsrc = 0;
      if (ops_conflict(m, writes, es)) continue;
      size_t a = i, b = i + 2;
      while (a > 0 && is_data(ops[a - 1].code)) a--;
      while (b < ops.size() && is_data(ops[b].code)) b++;
      bool other = false;
      for (size_t x = a; x <= i && !other; x++)
        for (size_t y = i + 2; y < b && !other; y++)
          if (!(x == i && y == i + 2)) other = ops_conflict(ops[x], ops[y], es);
      if (other) continue;
      pl->ll_fuse_put[p] = (int)i;
      break;
    }
  }
}

// Bake plan-owned buffer addresses into the device ops, fuse packet reads,
// upload the per-device tables, start the proxy (port channels).
cfStatus finalize(cfPlan* pl) {
  cfComm* c = pl->comm;
  Plan& P = pl->ir;
  const int n = P.nranks, K = pl->K;
  int prev_dev = -1;
  cudaGetDevice(&prev_dev);
  // plan-owned buffers live at fixed addresses: bake them into the data ops so
  // the interpreter resolves them without a table load
  for (size_t p = 0; p < pl->prog_ops.size(); p++)
    for (auto& d : pl->prog_ops[p]) {
      if (d.code != D_MULTI && d.code != D_COPY && d.code != D_PUT_PACKETS && d.code != D_READ_PACKETS &&
          d.code != D_PORT_PUT)
        continue;
      auto bake = [&](DRef& r) {
        const bool io = r.buf == pl->out_buf || (r.buf == pl->in_buf && !pl->input_private);
        if (io && r.rank != pl->prog_rank[p]) (r.buf == pl->out_buf ? pl->peer_out : pl->peer_in) = true;
        if (io || r.buf == kAbsolute) return;
        r.off = (uint64_t)(pl->heap[r.rank] + pl->buf_off[r.buf]) + r.off;
        r.buf = kAbsolute;
      };
      for (int k = 0; k < d.nsrc; k++) bake(d.src[k]);
      for (int k = 0; k < d.ndst; k++) bake(d.dst[k]);
    }
  fuse_packet_reads(pl);
  drop_redundant_syncs(pl);
  // each data op's CTA slice: ceil(size / K) elements rounded up to whole
  // 16-byte vectors (the interpreter multiplies, never divides)
  {
    const uint64_t V = 16 / (uint64_t)pl->es, Kk = (uint64_t)K;
    for (auto& prog : pl->prog_ops)
      for (auto& d : prog)
        if (d.code == D_MULTI || d.code == D_COPY || d.code == D_PUT_PACKETS || d.code == D_READ_PACKETS ||
            d.code == D_PORT_PUT)
          d.per = ((d.size + Kk - 1) / Kk + V - 1) / V * V;
    // compiled LL plans: put / read packets (LL16), MULTI / COPY on whole
    // 8-byte units (plain or LL16 packet sources), CTA-local syncs
    const uint64_t H = 8 / (uint64_t)pl->es;
    pl->ll_ok = pl->cls == 1 && !pl->prog_ops.empty() && (int)pl->prog_ops.size() <= kLLProgs;
    for (auto& prog : pl->prog_ops) {
      if (!pl->ll_ok) break;
      pl->ll_ok = !prog.empty() && (int)prog.size() <= kLLOps;
      for (auto& d : prog) {
        if (!pl->ll_ok) break;
        if (d.code == D_SYNC_CTA) continue;
        const bool pk = d.code == D_PUT_PACKETS || d.code == D_READ_PACKETS;
        const bool dm = d.code == D_MULTI || d.code == D_COPY;
        pl->ll_ok = (pk && (d.flags & F_LL16)) || (dm && (d.flags & F_VEC) && d.nsrc >= 1);
        pl->ll_ok = pl->ll_ok && d.nsrc <= 8 && d.ndst <= 8 && d.size % H == 0;
        // latency regime only: from 64 KiB per op the interpreter's vector
        // path (two units per thread in flight) wins (1pa plan b=16: 17.0 vs
        // 18.5 us compiled; 2pa_ll b=64: 23.0 vs 26.2 us)
        static const uint64_t ll_max = [] {
          const char* v = getenv("CF_PLAN_LL_MAX");   // diagnostic: largest op (bytes) compiled
          return v ? (uint64_t)atoll(v) : ~(uint64_t)0;
        }();
        pl->ll_ok = pl->ll_ok && d.size * (uint64_t)pl->es <= ll_max;
      }
    }
    compute_ll_stream(pl);
    compute_ll_fuse_put(pl);
    pl->single_ok = pl->cls == 0 && !pl->prog_ops.empty() && (int)pl->prog_ops.size() <= kSingleProgs;
    for (auto& prog : pl->prog_ops) {
      if (!pl->single_ok) break;
      const bool one = prog.size() == 1;
      const DevOp* d = one ? &prog[0] : nullptr;
      pl->single_ok = one && (d->code == D_MULTI || d->code == D_COPY) && (d->flags & F_VEC) && !d->pkt_mask &&
                      d->nsrc >= 1 && d->nsrc <= 8 && d->ndst <= 8 && d->size % V == 0;
    }
  }
  // device tables per device group
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    Group G;
    G.dev = c->local[c->groups[gi][0]].dev;
    std::set<int> ranks;
    for (int li : c->groups[gi]) ranks.insert(c->local[li].rank);
    const auto& prank = pl->prog_rank;
    std::vector<DevOp> all;
    std::vector<int32_t> meta;
    std::vector<int32_t> beg, end, rk;
    for (size_t p = 0; p < pl->prog_ops.size(); p++) {
      if (!ranks.count(prank[p])) continue;
      G.progs.push_back((int)p);
      beg.push_back((int32_t)all.size());
      all.insert(all.end(), pl->prog_ops[p].begin(), pl->prog_ops[p].end());
      end.push_back((int32_t)all.size());
      rk.push_back(prank[p]);
    }
    G.beg = beg;
    G.end = end;
    G.h_ops = all;
    meta = beg;
    meta.insert(meta.end(), end.begin(), end.end());
    meta.insert(meta.end(), rk.begin(), rk.end());
    std::vector<char*> bp((size_t)P.bufs.size() * n, nullptr);
    for (size_t b = 0; b < P.bufs.size(); b++)
      for (int r = 0; r < n; r++) bp[b * n + r] = pl->heap[r] + pl->buf_off[b];
    std::vector<int32_t> zl((size_t)n * kMaxZero, -1);
    for (int r = 0; r < n; r++)
      for (size_t z = 0; z < pl->zero_bufs[r].size(); z++) zl[(size_t)r * kMaxZero + z] = pl->zero_bufs[r][z];
    cudaSetDevice(G.dev);
    bool ok = cudaMalloc((void**)&G.d_ops, std::max<size_t>(1, all.size()) * sizeof(DevOp)) == cudaSuccess &&
              cudaMalloc((void**)&G.d_meta, std::max<size_t>(1, meta.size()) * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc((void**)&G.d_bufptr, bp.size() * sizeof(char*) + 8) == cudaSuccess &&
              cudaMalloc((void**)&G.d_zero, zl.size() * sizeof(int32_t)) == cudaSuccess;
    if (ok && !all.empty()) ok = cudaMemcpy(G.d_ops, all.data(), all.size() * sizeof(DevOp), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && !meta.empty()) ok = cudaMemcpy(G.d_meta, meta.data(), meta.size() * sizeof(int32_t), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) ok = cudaMemcpy(G.d_bufptr, bp.data(), bp.size() * sizeof(char*), cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok) ok = cudaMemcpy(G.d_zero, zl.data(), zl.size() * sizeof(int32_t), cudaMemcpyHostToDevice) == cudaSuccess;
    G.nops = (int)all.size();
    if (ok) ok = cudaMalloc((void**)&G.d_done, std::max<size_t>(1, G.progs.size() * K) * sizeof(uint64_t)) == cudaSuccess &&
                 cudaMemset(G.d_done, 0, std::max<size_t>(1, G.progs.size() * K) * sizeof(uint64_t)) == cudaSuccess;
    pl->groups.push_back(G);
    if (!ok) {
      cudaSetDevice(prev_dev);
      return fail(CF_E_CUDA, "plan table upload failed");
    }
  }
  cudaSetDevice(prev_dev);
  if (pl->uses_port) CF_TRY(proxy_start(c));
  if (getenv("CF_PLAN_DUMP")) {   // "explain": the compiled device program of each (rank, tb)
    static const char* names[] = {"nop", "sync_cta", "sync_group", "dev_barrier", "signal", "wait", "multi",
                                  "copy", "put_packets", "read_packets", "port_put", "port_signal",
                                  "port_flush"};
    fprintf(stderr, "plan '%s': K=%d CTAs/program, entry=%d prologue=%d\n", pl->ir.name.c_str(), pl->K,
            (int)pl->has_prologue, (int)pl->input_private);
    for (size_t p = 0; p < pl->prog_ops.size(); p++) {
      fprintf(stderr, "  r%d.tb%d:", pl->prog_rank[p], pl->prog_tb[p]);
      for (auto& d : pl->prog_ops[p])
        fprintf(stderr, " %s[n=%llu s%d d%d f%x p%x]", names[d.code], (unsigned long long)d.size, d.nsrc, d.ndst,
                d.flags, d.pkt_mask);
      fprintf(stderr, "\n");
    }
  }
  pl->ready = true;
  return CF_OK;
}

}  // namespace plan
}  // namespace cf

using namespace cf;
using namespace cf::plan;

extern "C" cfStatus cfPlanLoad(cfComm_t comm, const char* json, size_t len, int dtype_override, cfPlan_t* plan) {
  if (!comm || !json || !plan) return fail(CF_E_CONFIG, "null argument");
  if (!comm->connected) return fail(CF_E_CONFIG, "communicator not connected");
  if (dtype_override < -1 || dtype_override > 3) return fail(CF_E_SHAPE, "unknown dtype %d", dtype_override);
  return cf::plan::load(comm, json, len, dtype_override, plan);
}

namespace cf {
namespace plan {
namespace {
// The group's op array with every I/O reference of this call's binding
// resolved (see Group::bound), or nullptr: binding table full, or a stream
// capture is in progress (the first upload of a binding happens outside
// capture; a captured launch then reuses it).
bool single_enabled() {
  static const bool on = [] {
    const char* v = getenv("CF_PLAN_SINGLE");   // diagnostic: 0 keeps every plan on the interpreter
    return !(v && atoi(v) == 0);
  }();
  return on;
}

DevOp* bound_ops(const cfPlan* pl, Group& G, const PlanArgs& a, cudaStream_t st) {
  const int n = pl->ir.nranks;
  std::vector<char*> key(a.io_in, a.io_in + n);
  key.insert(key.end(), a.io_out, a.io_out + n);
  for (auto& b : G.bound)
    if (b.io == key) return b.d_ops;
  if (G.bound.size() >= kMaxBound || G.h_ops.empty()) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  Group::Bound b;
  b.io = key;
  const size_t bytes = G.h_ops.size() * sizeof(DevOp);
  if (cudaMalloc((void**)&b.d_ops, bytes) != cudaSuccess) return nullptr;
  if (cudaMallocHost((void**)&b.h_pin, bytes) != cudaSuccess) {
    cudaFree(b.d_ops);
    return nullptr;
  }
  memcpy(b.h_pin, G.h_ops.data(), bytes);
  for (size_t i = 0; i < G.h_ops.size(); i++) {
    DevOp& d = b.h_pin[i];
    if (d.code != D_MULTI && d.code != D_COPY && d.code != D_PUT_PACKETS && d.code != D_READ_PACKETS &&
        d.code != D_PORT_PUT)
      continue;
    auto fix = [&](DRef& r) {   // the device resolve pass, done once on the host
      if (r.buf == kAbsolute) return;
      char* base;
      if (r.buf == pl->in_buf && !pl->input_private) base = a.io_in[r.rank];
      else if (r.buf == pl->out_buf) base = a.io_out[r.rank];
      else base = pl->heap[r.rank] + pl->buf_off[r.buf];
      r.off = reinterpret_cast<uint64_t>(base + r.off);
      r.buf = kAbsolute;
    };
    for (int k = 0; k < d.nsrc; k++) fix(d.src[k]);
    for (int k = 0; k < d.ndst; k++) fix(d.dst[k]);
  }
  // prefetch hints: a program whose first data op is a packet put with more
  // than one payload unit per thread in its CTA slice (its threads then loop,
  // one dependent HBM read per round): the payload lines are requested while
  // the op window is staged (2pa_ll plan b=64 27.2 -> 24.5 us, 1pa plan b=16
  // 19.2 -> 17.2 us).  Not for reduce-first plans (HB): there the hint's own
  // parameter read delays the staging more than it saves (2pa plan b=1
  // 4.9 -> 5.3 us).
  for (size_t p = 0; p < G.progs.size() && (int)p < kPfProgs; p++) {
    PlanArgs::Prefetch h;
    memset(&h, 0, sizeof(h));
    for (int i = G.beg[p]; i < G.end[p]; i++) {
      const DevOp& d = b.h_pin[i];
      const bool data = d.code == D_PUT_PACKETS &&
                        (uint64_t)d.size * pl->es / (uint64_t)pl->K > (uint64_t)pl->threads * 8;
      if (!data && (d.code == D_SYNC_CTA || d.code == D_NOP)) continue;
      if (data) {
        const int ns = (d.code == D_PUT_PACKETS && !(d.flags & F_PAIRED)) ? 1 : std::min<int>(d.nsrc, 8);
        h.size = d.size;
        h.per = d.per;
        h.es = (uint32_t)pl->es;
        for (int k = 0; k < ns; k++)
          if (!((d.pkt_mask >> k) & 1u) && d.src[k].buf == kAbsolute) h.src[h.nsrc++] = (const char*)d.src[k].off;
      }
      break;   // only the program's first data op (before any wait / barrier)
    }
    b.pf.push_back(h);
  }
  bool any = false;
  for (auto& h : b.pf) any |= h.nsrc > 0;
  if (!any) b.pf.clear();   // no hint: the kernel skips the parameter read
  if (cudaMemcpyAsync(b.d_ops, b.h_pin, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaFree(b.d_ops);
    cudaFreeHost(b.h_pin);
    return nullptr;
  }
  G.bound.push_back(std::move(b));
  return G.bound.back().d_ops;
}
}  // namespace
}  // namespace plan
}  // namespace cf

extern "C" cfStatus cfPlanExecute(cfPlan_t pl, const void* const* inputs, void* const* outputs,
                                  const cudaStream_t* streams) {
  if (!pl || !inputs || !outputs || !streams) return fail(CF_E_CONFIG, "null argument");
  if (!pl->ready) return fail(CF_E_CONFIG, "plan not connected (cfPlanGetHandle / cfPlanConnect)");
  cfComm* c = pl->comm;
  const int n = pl->ir.nranks;
  // one process per GPU: peers' I/O buffers come from the registration table,
  // or from the symmetric heap (cfMemAlloc buffers: base[p] + offset)
  const Registration* reg_in = nullptr;
  const Registration* reg_out = nullptr;
  long long sym_in = -1, sym_out = -1;
  if (pl->mp) {
    bool mapped = c->sym.on();
    for (int p = 0; mapped && p < c->nranks; p++) mapped = c->sym.peer[0][p] != nullptr;
    if (mapped) {
      sym_in = c->sym.offset(0, inputs[0]);
      sym_out = c->sym.offset(0, outputs[0]);
    }
    if (pl->peer_in && sym_in < 0 && !(reg_in = c->find_reg(inputs[0])))
      return fail(CF_E_TOPOLOGY, "plan reads the peers' input: register input %p (cfBufferExport/Import) or "
                                 "allocate it with cfMemAlloc", inputs[0]);
    if (pl->peer_out && sym_out < 0 && !(reg_out = c->find_reg(outputs[0])))
      return fail(CF_E_TOPOLOGY, "plan writes the peers' output: register output %p (cfBufferExport/Import) or "
                                 "allocate it with cfMemAlloc", outputs[0]);
  }
  for (size_t li = 0; li < c->local.size(); li++) {
    if (!inputs[li] || !outputs[li]) return fail(CF_E_OOB, "local rank %zu: null buffer", li);
    if (((uintptr_t)inputs[li] | (uintptr_t)outputs[li]) & 15)
      return fail(CF_E_BAD_ALIGN, "local rank %zu: buffers must be 16-byte aligned", li);
  }
  int prev = -1;
  cudaGetDevice(&prev);
  const void* kernel = plan_kernel_for(pl->dtype, pl->cls);
  for (size_t gi = 0; gi < pl->groups.size(); gi++) {
    Group& G = pl->groups[gi];
    PlanArgs a;
    memset(&a, 0, sizeof(a));
    const int np = (int)G.progs.size();
    a.ops = G.d_ops;
    a.prog_begin = G.d_meta;
    a.prog_end = G.d_meta + np;
    a.prog_rank = G.d_meta + 2 * np;
    a.bufptr = G.d_bufptr;
    a.zero_list = G.d_zero;
    a.n = n;
    a.K = pl->K;
    a.nprog = np;
    a.nbuf = (int)pl->ir.bufs.size();
    a.in_buf = pl->in_buf;
    a.out_buf = pl->out_buf;
    a.input_private = pl->input_private ? 1 : 0;
    a.gpu_scope = (pl->groups.size() == 1 && !pl->mp) ? 1 : 0;
    // One launch holding every rank: the kernel boundary already separates
    // calls, so only a prologue that zeroes / copies buffers peers touch needs
    // the entry barrier, and no exit barrier is needed.
    const bool single = !pl->mp && pl->groups.size() == 1 && (int)c->local.size() == n;
    bool prologue = pl->input_private;
    for (auto& z : pl->zero_bufs) prologue |= !z.empty();
    a.entry_barrier = (!single || prologue) ? 1 : 0;
    a.exit_barrier = single ? 0 : 1;
    a.flag_stride = pl->flag_stride;
    for (size_t b = 0; b < pl->ir.bufs.size(); b++) a.buf_bytes[b] = (uint64_t)pl->ir.bufs[b].elems * pl->es;
    for (int r = 0; r < n; r++) {
      if (pl->mp) {
        a.io_in[r] = r == pl->me ? (char*)inputs[0]
                   : sym_in >= 0 ? c->sym.peer[0][r] + sym_in
                   : reg_in ? reg_in->peer[r] + ((const char*)inputs[0] - reg_in->ptr) : nullptr;
        a.io_out[r] = r == pl->me ? (char*)outputs[0]
                    : sym_out >= 0 ? c->sym.peer[0][r] + sym_out
                    : reg_out ? reg_out->peer[r] + ((char*)outputs[0] - reg_out->ptr) : nullptr;
      } else {
        a.io_in[r] = (char*)inputs[r];     // one-process world: local index == rank
        a.io_out[r] = (char*)outputs[r];
      }
      a.st[r] = (PlanState*)(pl->heap[r] + pl->state_off);
      a.lanes[r] = (uint64_t*)(pl->heap[r] + pl->lanes_off);
      a.bars[r] = (uint64_t*)(pl->heap[r] + pl->bars_off);
      a.rank_ctas[r] = 0;
      a.rank_leader[r] = -1;
    }
    for (int p = 0; p < np; p++) {
      const int r = pl->prog_rank[G.progs[p]];
      if (a.rank_leader[r] < 0) a.rank_leader[r] = p * pl->K;
      a.rank_ctas[r] += pl->K;
    }
    cudaSetDevice(G.dev);
    cfStatus s = join_streams(c, (int)gi, streams, false);
    if (s != CF_OK) { cudaSetDevice(prev); return s; }
    if (np <= kParamProgs) {
      a.prog_in_param = 1;
      for (int p = 0; p < np; p++) {
        a.prog_tab[p] = make_int4(pl->prog_rank[G.progs[p]], G.beg[p], G.end[p], 0);
      }
    }
    DevOp* rops = bound_ops(pl, G, a, streams[c->groups[gi][0]]);
    // rank barriers of the compiled launches: the interpreter's (same CTAs per
    // rank, same numbering), so calls may alternate between the two paths
    PlanBarriers pb;
    memset(&pb, 0, sizeof(pb));
    for (int r = 0; r < n; r++) {
      pb.pst[r] = a.st[r];
      pb.leader[r] = a.rank_leader[r];
    }
    pb.n = n;
    pb.gpu_scope = a.gpu_scope;
    pb.entry = a.entry_barrier;
    pb.exit = a.exit_barrier;
    const bool compiled_ok = rops && !pl->has_prologue && !pl->uses_port && single_enabled();
    if (compiled_ok && pl->single_ok) {
      // the plan compiled to a kernel: each program's resolved op in the parameter space
      const Group::Bound* bb = nullptr;
      for (auto& x : G.bound)
        if (x.d_ops == rops) bb = &x;
      SingleArgs sa;
      memset(&sa, 0, sizeof(sa));
      sa.K = pl->K;
      sa.nprog = np;
      for (int p = 0; p < np; p++) {
        const DevOp& d = bb->h_pin[G.beg[p]];
        auto& P = sa.p[p];
        for (int k = 0; k < d.nsrc; k++) P.src[k] = (const char*)d.src[k].off;
        for (int k = 0; k < d.ndst; k++) P.dst[k] = (char*)d.dst[k].off;
        P.size = d.size;
        P.per = d.per;
        P.nsrc = d.nsrc;
        P.ndst = d.ndst;
        P.flags = d.flags | (d.code == D_MULTI ? 0x100 : 0);
        P.rank = pl->prog_rank[G.progs[p]];
        sa.rank_ctas[P.rank] += pl->K;
      }
      for (int r = 0; r < n; r++) sa.st[r] = &a.st[r]->base;
      sa.bar = pb;
      void* sargs[] = {&sa};
      cudaError_t e = cudaLaunchKernel(plan_single_kernel_for(pl->dtype), dim3(np * pl->K), dim3(pl->threads),
                                       sargs, 0, streams[c->groups[gi][0]]);
      if (e != cudaSuccess) {
        cudaSetDevice(prev);
        return fail(CF_E_CUDA, "plan kernel launch: %s", cudaGetErrorString(e));
      }
      s = join_streams(c, (int)gi, streams, true);
      if (s != CF_OK) { cudaSetDevice(prev); return s; }
      continue;
    }
    if (compiled_ok && pl->ll_ok) {
      const Group::Bound* bb = nullptr;
      for (auto& x : G.bound)
        if (x.d_ops == rops) bb = &x;
      LLArgs la;
      memset(&la, 0, sizeof(la));
      // the compiled kernel runs 2 CTAs per SM: up to twice the interpreter's
      // CTAs per program (slices recomputed for that count)
      // (only as many as the largest op keeps busy: small plans keep K, their
      // extra CTAs would only add launch and barrier cost)
      uint64_t busiest = 0;   // largest op's items: 8-byte units x flattened ranges
      for (int p = 0; p < np; p++)
        for (int i = G.beg[p]; i < G.end[p]; i++) {
          const DevOp& d = bb->h_pin[i];
          const uint64_t units = d.size * (uint64_t)pl->es / 8;
          const bool flat = d.code == D_READ_PACKETS || (d.code == D_PUT_PACKETS && (d.flags & F_PAIRED));
          busiest = std::max(busiest, units * (flat ? (uint64_t)std::max<int>(d.nsrc, d.ndst) : 1));
        }
      const int K2 = (pb.entry || pb.exit) ? pl->K   // barrier counts assume the interpreter's CTAs per rank
                   : (int)std::min<uint64_t>(2ull * pl->K, std::max<uint64_t>(
                         pl->K, (busiest + pl->threads - 1) / pl->threads));
      const uint64_t V2 = 16 / (uint64_t)pl->es;
      la.K = K2;
      la.nprog = np;
      la.flag_stride = pl->flag_stride;
      for (int p = 0; p < np; p++) {
        auto& P = la.p[p];
        P.rank = pl->prog_rank[G.progs[p]];
        P.nops = G.end[p] - G.beg[p];
        // streamed pairs need the same CTAs per program on every rank
        P.stream = (K2 == pl->K || np == (int)pl->prog_ops.size()) ? pl->ll_stream[G.progs[p]] : -1;
        P.fuse_put = pl->ll_fuse_put[G.progs[p]];
        for (int i = 0; i < P.nops; i++) {
          const DevOp& d = bb->h_pin[G.beg[p] + i];
          auto& o = P.op[i];
          for (int k = 0; k < d.nsrc && k < 8; k++) {
            o.src[k] = (const char*)d.src[k].off;
            o.llflag_k[k] = d.llflag_k[k];
          }
          for (int k = 0; k < d.ndst && k < 8; k++) o.dst[k] = (char*)d.dst[k].off;
          o.size = d.size;
          o.per = ((d.size + K2 - 1) / K2 + V2 - 1) / V2 * V2;
          o.llflag = d.llflag;
          o.code = d.code;
          o.nsrc = d.nsrc;
          o.ndst = d.ndst;
          o.flags = d.flags;
          o.pkt_mask = d.pkt_mask;
        }
        // streaming pays from a few units per thread (one or two: op by op
        // is as fast; 1pa plan b=4 7.7 vs 8.8 us, b=64 57.8 vs 49.1 us)
        if (P.stream >= 0 && P.op[P.stream].per * pl->es / 8 <= 2ull * pl->threads) P.stream = -1;
        la.rank_ctas[P.rank] += K2;
      }
      for (int r = 0; r < n; r++) la.st[r] = &a.st[r]->base;
      la.bar = pb;
      for (int r = 0; r < n; r++)   // the leader CTA of each rank at this launch's CTAs per program
        if (pb.leader[r] >= 0) la.bar.leader[r] = pb.leader[r] / pl->K * K2;
      void* largs[] = {&la};
      cudaError_t e = cudaLaunchKernel(plan_ll_kernel_for(pl->dtype), dim3(np * K2), dim3(pl->threads), largs,
                                       0, streams[c->groups[gi][0]]);
      if (e != cudaSuccess) {
        cudaSetDevice(prev);
        return fail(CF_E_CUDA, "plan kernel launch: %s", cudaGetErrorString(e));
      }
      s = join_streams(c, (int)gi, streams, true);
      if (s != CF_OK) { cudaSetDevice(prev); return s; }
      continue;
    }
    if (rops) {
      a.ops = rops;
      a.resolved = 1;
      for (auto& bb : G.bound)
        if (bb.d_ops == rops && !getenv("CF_PLAN_NO_PREFETCH")) {
          a.npf = (int)bb.pf.size();
          for (int p = 0; p < a.npf; p++) a.pf[p] = bb.pf[p];
        }
    }
    void* args[] = {&a};
    a.window = pl->window;
    a.has_prologue = pl->has_prologue ? 1 : 0;
    if (pl->uses_port) {
      if (!proxy_alive(c)) { cudaSetDevice(prev); return fail(CF_E_PROXY_DOWN, "port-channel proxy is not running"); }
      for (int li : c->groups[gi]) a.port[c->local[li].rank] = proxy_queue(c, li);
      a.port_done = G.d_done;
    }
    cudaError_t e = cudaLaunchKernel(kernel, dim3(np * pl->K), dim3(pl->threads), args,
                                     pl->window * sizeof(DevOp), streams[c->groups[gi][0]]);
    if (e != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(CF_E_CUDA, "plan kernel launch: %s", cudaGetErrorString(e));
    }
    s = join_streams(c, (int)gi, streams, true);
    if (s != CF_OK) { cudaSetDevice(prev); return s; }
  }
  cudaSetDevice(prev);
  return CF_OK;
}

extern "C" cfStatus cfPlanInfo(cfPlan_t pl, size_t* in_elems, size_t* out_elems, int* dtype, int* n_programs,
                               int* n_device_ops) {
  if (!pl) return fail(CF_E_CONFIG, "null plan");
  if (in_elems) *in_elems = (size_t)pl->ir.bufs[pl->in_buf].elems;
  if (out_elems) *out_elems = (size_t)pl->ir.bufs[pl->out_buf].elems;
  if (dtype) *dtype = pl->dtype;
  if (n_programs) *n_programs = (int)pl->prog_ops.size();
  if (n_device_ops) *n_device_ops = pl->n_device_ops;
  return CF_OK;
}

// Reset after a reported device timeout: a timed-out execution leaves
// semaphore lanes, barrier counters and LL scratch in a state later calls
// cannot reason about, so every heap this process owns returns to its load-
// time state (zeroed, fresh PlanState).  One process per GPU: every rank calls
// it at a quiescent point (no execution of the plan in flight anywhere).
extern "C" cfStatus cfPlanClearDeviceError(cfPlan_t pl) {
  if (!pl) return fail(CF_E_CONFIG, "null plan");
  int prev = -1;
  cudaGetDevice(&prev);
  for (size_t r = 0; r < pl->heap.size(); r++) {
    if (!pl->heap[r] || pl->heap_mapped[r]) continue;   // own heaps only
    cudaSetDevice(pl->comm->local[pl->mp ? 0 : r].dev);
    PlanState st;
    memset(&st, 0, sizeof(st));
    st.base.timeout_ns = pl->comm->cfg.spin_timeout_ns;
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemset(pl->heap[r], 0, pl->heap_bytes) != cudaSuccess ||
        cudaMemcpy(pl->heap[r] + pl->state_off, &st, sizeof(st), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(CF_E_CUDA, "plan state reset failed");
    }
  }
  cudaSetDevice(prev);
  return CF_OK;
}

extern "C" cfStatus cfPlanLastDeviceError(cfPlan_t pl, int* code) {
  if (!pl || !code) return fail(CF_E_CONFIG, "null argument");
  int prev = -1;
  cudaGetDevice(&prev);
  uint32_t worst = 0;
  for (size_t r = 0; r < pl->heap.size(); r++) {
    if (!pl->heap[r] || pl->heap_mapped[r]) continue;   // own heaps only
    cudaSetDevice(pl->comm->local[pl->mp ? 0 : r].dev);
    // synchronous legacy-stream copy: waits for the caller's (blocking)
    // streams, not for unrelated non-blocking ones
    PlanState st;
    if (cudaMemcpy(&st, pl->heap[r] + pl->state_off, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(CF_E_CUDA, "plan state read failed");
    }
    worst = std::max(worst, st.base.error);
  }
  cudaSetDevice(prev);
  *code = (int)worst;
  return CF_OK;
}

extern "C" cfStatus cfPlanDestroy(cfPlan_t pl) {
  if (!pl) return CF_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& G : pl->groups) {
    cudaSetDevice(G.dev);
    cudaFree(G.d_ops);
    for (auto& b : G.bound) {
      cudaFree(b.d_ops);
      cudaFreeHost(b.h_pin);
    }
    cudaFree(G.d_meta);
    cudaFree(G.d_bufptr);
    cudaFree(G.d_zero);
    cudaFree(G.d_done);
  }
  for (size_t r = 0; r < pl->heap.size(); r++)
    if (pl->heap[r]) {
      cudaSetDevice(pl->comm->local[pl->mp ? 0 : r].dev);
      if (pl->heap_mapped[r]) cudaIpcCloseMemHandle(pl->heap[r]);
      else cudaFree(pl->heap[r]);
    }
  cudaSetDevice(prev);
  delete pl;
  return CF_OK;
}

// ------------------------------------------------------------------ one process per GPU

namespace {
struct PlanBlob {
  uint32_t magic;
  int32_t rank;
  uint64_t heap_bytes;
  cudaIpcMemHandle_t ipc;
};
constexpr uint32_t kPlanMagic = 0x43465031;  // "CFP1"
}  // namespace

extern "C" cfStatus cfPlanGetHandle(cfPlan_t pl, void* handle, size_t* bytes) {
  if (!pl || !bytes) return fail(CF_E_CONFIG, "null argument");
  if (!pl->mp) return fail(CF_E_CONFIG, "cfPlanGetHandle is for one-process-per-GPU communicators");
  if (*bytes < CF_PLAN_HANDLE_BYTES || !handle) {
    *bytes = CF_PLAN_HANDLE_BYTES;
    return fail(CF_E_CONFIG, "plan handle buffer needs %d bytes", CF_PLAN_HANDLE_BYTES);
  }
  static_assert(sizeof(PlanBlob) <= CF_PLAN_HANDLE_BYTES, "plan handle too large");
  PlanBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kPlanMagic;
  b.rank = pl->me;
  b.heap_bytes = pl->heap_bytes;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->comm->local[0].dev);
  const cudaError_t e = cudaIpcGetMemHandle(&b.ipc, pl->heap[pl->me]);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(CF_E_CUDA, "cudaIpcGetMemHandle(plan heap): %s", cudaGetErrorString(e));
  memset(handle, 0, CF_PLAN_HANDLE_BYTES);
  memcpy(handle, &b, sizeof(b));
  *bytes = CF_PLAN_HANDLE_BYTES;
  return CF_OK;
}

extern "C" cfStatus cfPlanConnect(cfPlan_t pl, const void* handles, size_t bytes_per_handle) {
  if (!pl || !handles) return fail(CF_E_CONFIG, "null argument");
  if (!pl->mp) return fail(CF_E_CONFIG, "cfPlanConnect is for one-process-per-GPU communicators");
  if (pl->ready) return CF_OK;
  if (bytes_per_handle < sizeof(PlanBlob)) return fail(CF_E_CONFIG, "plan handle too small");
  const int n = pl->ir.nranks;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->comm->local[0].dev);
  for (int r = 0; r < n; r++) {
    PlanBlob b;
    memcpy(&b, (const char*)handles + (size_t)r * bytes_per_handle, sizeof(b));
    if (b.magic != kPlanMagic || b.rank != r || b.heap_bytes != pl->heap_bytes) {
      cudaSetDevice(prev);
      return fail(CF_E_RANK_MISMATCH, "plan handle %d is not rank %d's handle of this plan", r, r);
    }
    if (r == pl->me) continue;
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(CF_E_CUDA, "cudaIpcOpenMemHandle(plan heap of rank %d): %s", r, cudaGetErrorString(e));
    }
    pl->heap[r] = (char*)p;
    pl->heap_mapped[r] = true;
  }
  cudaSetDevice(prev);
  return finalize(pl);
}
