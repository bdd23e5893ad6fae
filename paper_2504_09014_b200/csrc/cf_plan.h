// cf_plan.h -- execution-plan IR, device op array and launch arguments of the
// GPU plan interpreter (K10).  Internal to libcf.
//
// Reference: plan wire format and IR   cf/plan.py:20-101, 136-291
//            plan interpreter           cf/executor.py:73-379
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include "cf_proxy.h"
#include "device/cf_device.cuh"

// threads per CTA of the plan interpreter (one launch-bounds for the kernel)
#ifndef CF_PLAN_THREADS
#define CF_PLAN_THREADS 512
#endif

namespace cf {
namespace plan {

// ---------------------------------------------------------------- host IR (cf/plan.py:38-86)

enum OpKind { P_PUT, P_PUT_PACKETS, P_PUT_WITH_SIGNAL, P_SIGNAL, P_WAIT, P_FLUSH, P_READ_PACKETS,
              P_REDUCE, P_REDUCE_PUT, P_COPY, P_TB_SYNC, P_DEVICE_BARRIER, P_NUM_OPS };
enum BufKind { B_INPUT, B_OUTPUT, B_SCRATCH };
enum ChanType { C_PORT, C_MEMORY, C_SWITCH };

struct Ref {
  int buf = -1;
  long long off = 0, size = 0;
};

struct Op {
  int kind = -1;
  int chan = -1;
  bool has_src = false, has_dst = false, has_src2 = false, has_arrives = false;
  Ref src, dst, src2, arrives;
  bool has_flag = false;
  long long flag = 0;
  bool has_group = false;
  std::vector<int> group;
};

struct Buf {
  std::string id;
  int kind = B_SCRATCH;
  int rank = -1;          // -1 = "all"
  long long elems = 0;
};

struct Chan {
  std::string id;
  int type = C_MEMORY;
  int src = -1, dst = -1;
  std::vector<int> ranks;
  int protocol = -1;      // -1 = plan protocol
};

struct Prog {
  int rank = 0, tb = 0;
  std::vector<Op> ops;
};

struct Plan {
  std::string name;
  int collective = 0, protocol = 0, dtype = 0, nranks = 0;
  bool lowered = true;
  std::vector<Buf> bufs;
  std::vector<Chan> chans;
  std::vector<Prog> progs;
};

// ---------------------------------------------------------------- device op array

constexpr int kMaxSrc = 16;
constexpr int kMaxDst = 8;

enum DevCode : uint8_t {
  D_NOP = 0,
  D_SYNC_CTA,      // tb_sync whose dependences stay inside each CTA's slice
  D_SYNC_GROUP,    // tb_sync across the CTAs of one program
  D_DEV_BARRIER,   // device_barrier over member programs        cf/executor.py:208-226
  D_SIGNAL,        // +1 on each CTA lane of the receiver         cf/channels.py:227-232
  D_WAIT,          // every lane >= target                        cf/channels.py:234-237
  D_MULTI,         // dst[*] = [0 +] src0 + src1 + ...            reduce / reduce_put / switch reduce
  D_COPY,          // dst[*] = src0                               put / copy / switch broadcast
  D_PUT_PACKETS,   // payload -> LL packets                       cf/channels.py:244-280
  D_READ_PACKETS,  // LL packets -> payload                       cf/channels.py:303-330
  D_PORT_PUT,      // port put (+signal): request to the proxy    cf/channels.py:80-108
  D_PORT_SIGNAL,   // port signal, ordered after earlier puts     cf/channels.py:98-103
  D_PORT_FLUSH,    // wait until the proxy completed every request  cf/channels.py:110-114
};
enum DevFlags : uint8_t { F_ZERO = 1, F_ROUND_EACH = 2, F_VEC = 4, F_LL16 = 8, F_SIGNAL = 16,
                          F_PAIRED = 32 /* D_PUT_PACKETS batch: src[k] -> dst[k] */ };

struct DRef {
  int32_t buf;         // plan buffer index, or kAbsolute: `off` is the device address
  int32_t rank;
  uint64_t off;        // bytes
};
constexpr int32_t kAbsolute = -1;

struct DevOp {
  uint8_t code, nsrc, ndst, flags;
  uint32_t llflag;     // plan flag (the runtime flag also folds in the call epoch)
  uint64_t size;       // elements (payload elements for LL ops)
  int32_t id;          // channel index (signal/wait) or counter index (barriers)
  int32_t peer;        // signal: receiving rank
  uint64_t m;          // wait / barrier: 1-based occurrence within the call
  uint64_t per_call;   // wait: signals per call on the channel; barrier: occurrences per call
  uint64_t members;    // barrier: participating CTAs
  // data ops: buffer references.  Batched sync ops reuse the slots:
  //   D_SIGNAL  dst[k] = {channel, receiving rank, -}     (ndst signals)
  //   D_WAIT    src[k] = {channel, signals per call, m}   (nsrc waits)
  DRef src[kMaxSrc];
  DRef dst[kMaxDst];
  uint32_t llflag_k[kMaxSrc];  // plan flag of packet source k (READ_PACKETS batch, MULTI pkt_mask)
  uint32_t pkt_mask;           // D_MULTI: sources read straight from LL16 packet areas
  uint32_t pad_;
  uint64_t per;                // data ops: elements per CTA slice, whole 16-byte vectors (set at
                               // load time from K, so the interpreter never divides)
};

// Per-rank execution state of one loaded plan (in the plan heap of the rank).
struct PlanState {
  RankState base;            // epoch / done counter / error word / timeout
  uint64_t bar_arrive;       // rank barrier: local CTA arrivals (monotonic)
  uint64_t bar_release;      // rank barrier: leader's release value
  uint64_t rankbar[CF_MAX_RANKS];  // rank barrier: value written by each peer
};

struct PlanArgs {
  const DevOp* ops;
  const int32_t* prog_begin;   // per launched program
  const int32_t* prog_end;
  const int32_t* prog_rank;
  char* const* bufptr;         // [nbuf * n] (plan-owned buffers; io buffers from io_in/io_out)
  const int32_t* zero_list;    // per rank: buffers to zero each call, packed [rank][kMaxZero]
  int n, K, nprog, nbuf;
  int in_buf, out_buf;
  int input_private;           // 1: plan writes its input -> copy user input into the plan buffer
  int gpu_scope;               // every rank on this device: .gpu-scope release/acquire
  int window;                  // ops staged into shared memory at a time
  int resolved;                // 1: `ops` already holds this call's I/O addresses (host-resolved)
  int has_prologue;            // any zeroing / private-input copy this call
  int entry_barrier;           // rank barrier after the prologue (zeroing / private input)
  int exit_barrier;            // rank barrier at the end (not needed when one launch holds every rank)
  uint32_t flag_stride;
  uint64_t buf_bytes[16];      // byte size of each buffer (<= 16 buffers)
  char* io_in[CF_MAX_RANKS];
  char* io_out[CF_MAX_RANKS];
  PlanState* st[CF_MAX_RANKS];
  uint64_t* lanes[CF_MAX_RANKS];
  uint64_t* bars[CF_MAX_RANKS];
  int rank_ctas[CF_MAX_RANKS];
  int rank_leader[CF_MAX_RANKS];
  PortQueue port[CF_MAX_RANKS];  // proxy request rings (plans with port channels)
  uint64_t* port_done;           // [nprog * K] completion counters of this launch's CTAs
  // Program table {rank, begin, end, -} in the parameter space when it fits,
  // so a CTA knows its op range without a dependent global load.
  int prog_in_param;
  int4 prog_tab[128];
  // L2 prefetch hints (host-resolved bindings only): the source ranges of
  // each program's first data op, so their HBM reads overlap the dependent
  // load that stages the op window (npf = 0: none)
  int npf;
  struct Prefetch {
    const char* src[8];
    uint64_t size, per;  // the op's elements and its CTA slice (DevOp::per)
    uint32_t nsrc, es;   // sources; bytes per element of the ranges (packet ranges: 2 x)
  } pf[32];
};
constexpr int kParamProgs = 128;
constexpr int kPfProgs = 32;

// Plans whose every program is one plain-vector MULTI / COPY (the fused C5
// two-shot plan: an n-source pull-reduce pushed to n destinations) run, when
// one launch holds every rank and the I/O binding is host-resolved, on a
// specialized kernel that takes each program's resolved op in its parameter
// space: no op staging, no interpreter -- the plan compiled to a kernel.
constexpr int kSingleProgs = 16;
// Rank barriers of a compiled plan launch (one process per GPU: entry = the
// peers' inputs are produced and outputs free, exit = nobody still reads this
// rank's buffers), numbered like the interpreter's.
struct PlanBarriers {
  PlanState* pst[CF_MAX_RANKS];
  int leader[CF_MAX_RANKS];
  int n, gpu_scope, entry, exit;
};
struct SingleArgs {
  int K, nprog;
  struct Prog {
    const char* src[8];
    char* dst[8];
    uint64_t size, per;    // elements; CTA slice (DevOp::per)
    int nsrc, ndst, flags, rank;
  } p[kSingleProgs];
  RankState* st[CF_MAX_RANKS];   // &PlanState::base of each rank (the call epoch)
  int rank_ctas[CF_MAX_RANKS];
  PlanBarriers bar;
};

// LL plans compiled to a kernel: every program a short sequence of LL16
// packet puts / reads, plain-vector or packet-source MULTI / COPY and
// CTA-local syncs (the C5 1pa and 2pa_ll plans), one launch holding every
// rank, binding host-resolved: the resolved ops travel in the parameter
// space and run on a lean kernel (no staging, no general interpreter, two
// CTAs per SM) -- packet ops spread their (range, unit) items over the
// threads, reduces run one 8-byte unit per thread.
constexpr int kLLProgs = 8;
constexpr int kLLOps = 7;
struct LLArgs {
  int K, nprog;
  uint32_t flag_stride;
  struct Op {
    const char* src[8];
    char* dst[8];
    uint32_t llflag_k[8];  // plan flags of packet sources (READ / MULTI)
    uint64_t size, per;
    uint32_t llflag;       // PUT
    uint8_t code, nsrc, ndst, flags;
    uint32_t pkt_mask;
  };
  struct Prog {
    Op op[kLLOps];
    int nops, rank;
    int stream;            // op index of a PUT_PACKETS run streamed with the MULTI after it (-1: none)
    int fuse_put;          // op index of a MULTI whose units the PUT_PACKETS at +2 broadcasts (-1: none)
  } p[kLLProgs];
  RankState* st[CF_MAX_RANKS];
  int rank_ctas[CF_MAX_RANKS];
  PlanBarriers bar;
};
static_assert(sizeof(LLArgs) <= 32764, "kernel parameter space");
static_assert(sizeof(PlanArgs) <= 32764, "kernel parameter space");
constexpr int kMaxBufs = 16;
constexpr int kMaxZero = 16;
constexpr int kPlanWindow = 32;   // DevOps staged in shared memory at a time
static_assert(sizeof(DevOp) % 16 == 0, "DevOp is copied as 16-byte vectors");

}  // namespace plan
}  // namespace cf
