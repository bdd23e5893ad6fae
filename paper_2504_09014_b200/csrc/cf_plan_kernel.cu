// cf_plan_kernel.cu -- K10: the GPU plan interpreter (cf/executor.py:197-379).
//
// One launch per device runs every (rank, tb) program of the ranks on that
// device.  Program p is executed by K CTAs: data ops are sliced contiguously
// across them (element slice j of K); sync ops keep the reference's
// per-thread-block ordering model (cf/lowering.py:11-17):
//   tb_sync        -> __syncthreads when every dependence across it stays in
//                     one CTA's slice (decided at load time), else a counter
//                     barrier over the program's K CTAs
//   signal         -> each CTA adds 1 to its own lane of the receiver's
//                     semaphore after its own slice (release at .sys scope)
//   wait           -> every lane of the channel >= (call-1)*signals_per_call + m
//   device_barrier -> counter barrier over the member programs' CTAs
// Calls are bracketed by rank-level barriers (entry: inputs produced, outputs
// zeroed where the plan reads them before writing -- the reference zeroes
// every region per execute, cf/executor.py:153-154; exit: nobody touches a
// rank's buffers after it returns), so plan buffers are reused across calls
// without host work, and LL flags are re-stamped with the call epoch.
#include "cf_plan.h"
#define TS_CTA_COND (blockIdx.x % a.K == 0)
#include "cf_ts.cuh"

namespace cf {
namespace plan {

__device__ __forceinline__ void red_add_release(uint64_t* p, uint64_t v, bool gpu) {
  if (gpu) asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}


// Data-op references are resolved to absolute addresses when their window is
// staged (see resolve_window), so the op bodies read one shared-memory word per
// pointer instead of a chain of dependent parameter/table loads.
__device__ __forceinline__ char* ptr(const DRef& r) { return reinterpret_cast<char*>(r.off); }

__device__ __forceinline__ bool is_data_code(uint8_t c) {
  return c == D_MULTI || c == D_COPY || c == D_PUT_PACKETS || c == D_READ_PACKETS || c == D_PORT_PUT;
}

// ((e - 1) * stride + f) mod (2^32 - 1) + 1 without a 64-bit division
// (2^32 = 1 mod 2^32 - 1: fold the high word into the low word twice)
__device__ __forceinline__ uint32_t runtime_flag(uint64_t e, uint32_t stride, uint32_t f) {
  const uint64_t x = (e - 1) * (uint64_t)stride + f;
  uint64_t y = (x >> 32) + (x & 0xffffffffull);
  y = (y >> 32) + (y & 0xffffffffull);
  if (y >= 0xffffffffull) y -= 0xffffffffull;
  return (uint32_t)y + 1u;
}

// counter barrier: every participant adds 1, then waits for the call's total
// (every thread fences its own writes before the block barrier: one thread's
// fence after bar.sync is not relied on to cover the other warps' stores)
__device__ __forceinline__ void counter_barrier(uint64_t* ctr, uint64_t target, RankState* rs) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd((unsigned long long*)ctr, 1ull);
    wait_geq(ctr, target, rs, true);
  }
  __syncthreads();
}

// All CTAs of `rank` meet; the rank's leader CTA exchanges `k` with every
// other rank's leader, then releases its rank.
// (`st`: every rank's PlanState as this device addresses it; the rank's CTAs
// count `rank_ctas` arrivals per barrier, so every launch path of a plan --
// interpreter or compiled -- must run the same CTAs per rank)
__device__ __noinline__ void rank_barrier_raw(PlanState* const* st, int n, int rank, int leader, int rank_ctas,
                                              uint64_t k, bool gpu) {
  PlanState* ps = st[rank];
  fence_publish(gpu);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)&ps->bar_arrive, 1ull);
  if ((int)blockIdx.x == leader) {
    if (threadIdx.x == 0) wait_geq(&ps->bar_arrive, k * (uint64_t)rank_ctas, &ps->base, true);
    __syncthreads();
    const int t = threadIdx.x;
    if (t < n && t != rank) {
      fence_publish(gpu);
      st_release(&st[t]->rankbar[rank], k, gpu);
      wait_geq(&ps->rankbar[t], k, &ps->base, gpu);
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(&ps->bar_release, k);
  } else if (threadIdx.x == 0) {
    wait_geq(&ps->bar_release, k, &ps->base, true);
  }
  __syncthreads();
}
__device__ __forceinline__ void rank_barrier(const PlanArgs& a, int rank, uint64_t k) {
  rank_barrier_raw(a.st, a.n, rank, a.rank_leader[rank], a.rank_ctas[rank], k, a.gpu_scope);
}

// ---------------------------------------------------------------- element helpers

template <typename T>
__device__ __forceinline__ uint4 load_part(const char* p, int nval) {
  constexpr int V = 16 / sizeof(T);
  if (nval >= V) return ld16(p);
  return ld_partial16<sizeof(T)>(p, nval * (int)sizeof(T));
}
template <typename T>
__device__ __forceinline__ void store_part(char* p, uint4 v, int nval) {
  constexpr int V = 16 / sizeof(T);
  if (nval >= V) { st16(p, v); return; }
  st_masked16<sizeof(T)>(p, v, 0, nval);
}

template <typename T>
__device__ __forceinline__ void acc_vec(typename Vec<T>::Acc* acc, uint4 x, bool round_each) {
  constexpr int V = Vec<T>::N;
  typename Vec<T>::Acc t[V];
  Vec<T>::load(x, t);
#pragma unroll
  for (int j = 0; j < V; j++) {
    acc[j] = acc_add(acc[j], t[j]);
    if (round_each) acc[j] = Vec<T>::round(acc[j]);
  }
}

// Issue the 16-byte payload load of source k at vector v: a plain vector, or
// the two LL16 packets carrying it (flags checked later, see finish_src).
template <typename T>
__device__ __forceinline__ void issue_src(const char* p, size_t v, int nval, bool pkt, uint4& r0, uint4& r1) {
  if (!pkt) {
    r0 = load_part<T>(p + v * 16, nval);
    return;
  }
  r0 = ld16_volatile(p + v * 32);
  r1 = nval * (int)sizeof(T) > 8 ? ld16_volatile(p + v * 32 + 16) : make_uint4(0, 0, 0, 0);
}
template <typename T>
__device__ __forceinline__ uint4 finish_src(const char* p, size_t v, int nval, bool pkt, uint32_t flag, uint4 r0,
                                            uint4 r1, RankState* rs) {
  if (!pkt) return r0;
  uint2 d0 = make_uint2(r0.x, r0.z), d1 = make_uint2(r1.x, r1.z);
  if (r0.y != flag || r0.w != flag) d0 = ll16_get(p + v * 32, flag, rs);
  if (nval * (int)sizeof(T) > 8) {
    if (r1.y != flag || r1.w != flag) d1 = ll16_get(p + v * 32 + 16, flag, rs);
  } else {
    d1 = make_uint2(0, 0);
  }
  return make_uint4(d0.x, d0.y, d1.x, d1.y);
}

// D_MULTI / D_COPY on this CTA's slice [lo, hi) of the op's elements.  MULTI
// sources flagged in pkt_mask are read straight from LL16 packet areas (a
// read_packets fused into the reduce).
template <typename T>
__device__ __noinline__ void data_op_general(const DevOp& op, uint64_t lo, uint64_t hi, uint32_t fstride, uint64_t e,
                                             RankState* rs);

// The common fused shape -- an n-source (n <= 8) pull-reduce pushed to up to 8
// destinations, plain (non-packet) 16-byte vectors -- with every pointer in a
// register and all sources in flight; anything else goes to the general path
// (kept out of line so its register pressure does not spill this loop).
template <typename T>
__device__ __noinline__ void multi_fast(const DevOp& op, uint64_t lo, uint64_t hi);

// This CTA's slice [lo, hi) of an op's elements: contiguous, whole vectors.
// (`per` = DevOp::per, computed at load time: no division on the device)
__device__ __forceinline__ void slice(uint64_t size, uint64_t per, int j, uint64_t& lo, uint64_t& hi) {
  lo = min((uint64_t)j * per, size);
  hi = min(lo + per, size);
}

template <typename T>
__device__ __forceinline__ void data_op(const PlanArgs& a, const DevOp& op, int j, uint64_t e, RankState* rs) {
  uint64_t lo, hi;
  slice(op.size, op.per, j, lo, hi);
  if (lo >= hi) return;
  if ((op.flags & F_VEC) && op.code == D_MULTI && op.nsrc <= 8 && !op.pkt_mask) {
    constexpr int V = 16 / sizeof(T);
    const uint64_t full = lo + (hi - lo) / V * V;
    if (full > lo) multi_fast<T>(op, lo, full);
    if (full < hi) data_op_general<T>(op, full, hi, a.flag_stride, e, rs);   // ragged last vector
  } else {
    data_op_general<T>(op, lo, hi, a.flag_stride, e, rs);
  }
}

// Out of line so the interpreter's live state does not share its registers.
template <typename T>
__device__ __noinline__ void multi_fast(const DevOp& op, uint64_t lo, uint64_t hi) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  constexpr int B = 8;
  const int nsrc = op.nsrc, ndst = op.ndst;
  const bool zero = op.flags & F_ZERO, round_each = op.flags & F_ROUND_EACH;
  // whole vectors only (the caller hands the ragged tail to the general path),
  // so every load is a plain 16-byte load and x[] stays in registers
  for (uint64_t v = lo / V + threadIdx.x; v * V < hi; v += blockDim.x) {
    const size_t boff = (size_t)v * 16;
    uint4 x[B];
#pragma unroll
    for (int i = 0; i < B; i++) x[i] = i < nsrc ? ld16(ptr(op.src[i]) + boff) : make_uint4(0, 0, 0, 0);
    A acc[V];
    if (zero) {
#pragma unroll
      for (int i = 0; i < V; i++) acc[i] = A(0);
      acc_vec<T>(acc, x[0], round_each);
    } else {
      Vec<T>::load(x[0], acc);
    }
#pragma unroll
    for (int i = 1; i < B; i++)
      if (i < nsrc) acc_vec<T>(acc, x[i], round_each);
    const uint4 res = Vec<T>::store(acc);
#pragma unroll
    for (int d = 0; d < kMaxDst; d++)
      if (d < ndst) st16(ptr(op.dst[d]) + boff, res);
  }
}

template <typename T>
__device__ __noinline__ void data_op_general(const DevOp& op, uint64_t lo, uint64_t hi, uint32_t fstride, uint64_t e,
                                             RankState* rs) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  constexpr int B = 8;   // sources in flight per round
  const int nsrc = op.nsrc, ndst = op.ndst;
  const bool zero = op.flags & F_ZERO, round_each = op.flags & F_ROUND_EACH;
  const bool multi = op.code == D_MULTI;
  const uint32_t pkt = op.pkt_mask;
  // pointers and (runtime) packet flags are read from the staged op in shared
  // memory at each use: no per-thread arrays (they would live in local memory)
  auto src = [&](int k) -> const char* { return ptr(op.src[k]); };
  auto dst = [&](int k) -> char* { return ptr(op.dst[k]); };
  if (op.flags & F_VEC) {
    for (uint64_t v = lo / V + threadIdx.x; v * V < hi; v += blockDim.x) {
      const int nval = (int)min((uint64_t)V, hi - v * V);
      const size_t boff = (size_t)v * 16;
      uint4 res;
      if (!multi) {
        res = load_part<T>(src(0) + boff, nval);
      } else {
        A acc[V];
        if (zero) {
#pragma unroll
          for (int i = 0; i < V; i++) acc[i] = A(0);
        }
        for (int k0 = 0; k0 < nsrc; k0 += B) {   // B sources' loads in flight per round
          uint4 r0[B], r1[B];
#pragma unroll
          for (int i = 0; i < B; i++)
            if (k0 + i < nsrc) issue_src<T>(src(k0 + i), v, nval, (pkt >> (k0 + i)) & 1u, r0[i], r1[i]);
#pragma unroll
          for (int i = 0; i < B; i++) {
            const int k = k0 + i;
            if (k >= nsrc) break;
            const uint32_t fl = ((pkt >> k) & 1u) ? runtime_flag(e, fstride, op.llflag_k[k]) : 0u;
            const uint4 x = finish_src<T>(src(k), v, nval, (pkt >> k) & 1u, fl, r0[i], r1[i], rs);
            if (k == 0 && !zero) Vec<T>::load(x, acc);
            else acc_vec<T>(acc, x, round_each);
          }
        }
        res = Vec<T>::store(acc);
      }
      for (int d = 0; d < ndst; d++) store_part<T>(dst(d) + boff, res, nval);
    }
  } else {
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const size_t boff = (size_t)i * sizeof(T);
      T res;
      if (!multi) {
        res = *reinterpret_cast<const T*>(src(0) + boff);
      } else {
        A acc = zero ? A(0) : to_acc<T>(*reinterpret_cast<const T*>(src(0) + boff));
        for (int k = zero ? 0 : 1; k < nsrc; k++) {
          acc = acc_add(acc, to_acc<T>(*reinterpret_cast<const T*>(src(k) + boff)));
          if (round_each) acc = Vec<T>::round(acc);
        }
        res = from_acc<T>(acc);
      }
      for (int d = 0; d < ndst; d++) *reinterpret_cast<T*>(dst(d) + boff) = res;
    }
  }
}

// One 8-byte unit per thread, every range of the batch: payload / packet
// loads of all nb ranges in flight first (the large-slice path).
template <typename T>
__device__ __noinline__ void packet_units(const DevOp& op, uint64_t u0, uint64_t u1, bool put, bool paired, int nb,
                                             uint32_t pflag, uint32_t fstride, uint64_t e, RankState* rs) {
  if (put && paired) {   // src[k] -> dst[k]
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      uint2 d[kMaxDst];
#pragma unroll
      for (int k = 0; k < kMaxDst; k++)
        if (k < nb) d[k] = *reinterpret_cast<const uint2*>(ptr(op.src[k]) + u * 8);
#pragma unroll
      for (int k = 0; k < kMaxDst; k++)
        if (k < nb) ll16_put(ptr(op.dst[k]) + u * 16, d[k], pflag);
    }
  } else if (put) {      // one payload -> nb ranges
    const char* src = ptr(op.src[0]);
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      const uint2 d = *reinterpret_cast<const uint2*>(src + u * 8);
      for (int k = 0; k < nb; k++) ll16_put(ptr(op.dst[k]) + u * 16, d, pflag);
    }
  } else {
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      uint4 raw[kMaxDst];
#pragma unroll
      for (int k = 0; k < kMaxDst; k++)   // all packets in flight first
        if (k < nb) raw[k] = ld16_volatile(ptr(op.src[k]) + u * 16);
#pragma unroll
      for (int k = 0; k < kMaxDst; k++) {
        if (k < nb) {
          const uint32_t flag = runtime_flag(e, fstride, op.llflag_k[k]);
          uint2 d = make_uint2(raw[k].x, raw[k].z);
          if (raw[k].y != flag || raw[k].w != flag) d = ll16_get(ptr(op.src[k]) + u * 16, flag, rs);
          *reinterpret_cast<uint2*>(ptr(op.dst[k]) + u * 8) = d;
        }
      }
    }
  }
}

#ifndef CF_PLAN_PKT_U
#define CF_PLAN_PKT_U 2
#endif
constexpr int kPktU = CF_PLAN_PKT_U;

// LL packets (cf/channels.py:244-330).  LL16: 8 payload bytes per 16-byte
// packet {d0, f, d1, f}; LL8: one reference packet {d, f} per 4 payload bytes.
template <typename T>
__device__ __noinline__ void packet_op(const DevOp& op, int K, int j, uint32_t fstride, uint64_t e, RankState* rs) {
  uint64_t lo, hi;
  slice(op.size, op.per, j, lo, hi);
  if (lo >= hi) return;
  const bool put = op.code == D_PUT_PACKETS;
  // batched ops: a put sends one payload to ndst packet ranges (one plan op
  // each); a read drains nsrc packet ranges into nsrc payload ranges
  const int nb = put ? op.ndst : op.nsrc;
  // plan flags -> this call's runtime flags (fold in the epoch)
  const uint32_t pflag = put ? runtime_flag(e, fstride, op.llflag) : 0;
  if (op.flags & F_LL16) {
    // (range k, unit u) items flattened over the CTA's threads -- consecutive
    // threads take consecutive units of one range -- so a batch of nb ranges
    // spreads over nb times the threads instead of looping in each one;
    // kPktU items per thread per round, their loads in flight together
    const uint64_t u0 = lo * sizeof(T) / 8, u1 = (hi * sizeof(T) + 7) / 8;
    const uint32_t nu = (uint32_t)(u1 - u0), items = nu * (uint32_t)nb;
    const bool paired = op.flags & F_PAIRED;
    constexpr int U = kPktU;
    const float rnu = 1.0f / (float)nu;   // item w -> range w / nu without an integer division
    if (nu >= 4 * blockDim.x || (put && !paired)) {
      // enough units to keep every thread busy (or one payload to many
      // ranges): one unit per thread, all nb ranges' accesses in flight
      packet_units<T>(op, u0, u1, put, paired, nb, pflag, fstride, e, rs);
      return;
    }
    for (uint32_t w0 = threadIdx.x; w0 < items; w0 += U * blockDim.x) {
      uint32_t kk[U];
      uint64_t uu[U];
#pragma unroll
      for (int i = 0; i < U; i++) {
        const uint32_t w = w0 + (uint32_t)i * blockDim.x;
        uint32_t q = (uint32_t)((float)w * rnu);   // exact after one correction (w < 2^24)
        q -= q * nu > w;
        q += (q + 1) * nu <= w;
        kk[i] = w < items ? q : (uint32_t)kMaxDst;
        uu[i] = u0 + (w - kk[i] * nu);
      }
      if (put) {
        uint2 d[U];
#pragma unroll
        for (int i = 0; i < U; i++)
          if (kk[i] < (uint32_t)nb)
            d[i] = *reinterpret_cast<const uint2*>(ptr(op.src[paired ? kk[i] : 0]) + uu[i] * 8);
#pragma unroll
        for (int i = 0; i < U; i++)
          if (kk[i] < (uint32_t)nb) ll16_put(ptr(op.dst[kk[i]]) + uu[i] * 16, d[i], pflag);
      } else {
        uint4 raw[U];
#pragma unroll
        for (int i = 0; i < U; i++)   // all packets in flight first
          if (kk[i] < (uint32_t)nb) raw[i] = ld16_volatile(ptr(op.src[kk[i]]) + uu[i] * 16);
#pragma unroll
        for (int i = 0; i < U; i++)
          if (kk[i] < (uint32_t)nb) {
            const uint32_t flag = runtime_flag(e, fstride, op.llflag_k[kk[i]]);
            uint2 d = make_uint2(raw[i].x, raw[i].z);
            if (raw[i].y != flag || raw[i].w != flag) d = ll16_get(ptr(op.src[kk[i]]) + uu[i] * 16, flag, rs);
            *reinterpret_cast<uint2*>(ptr(op.dst[kk[i]]) + uu[i] * 8) = d;
          }
      }
    }
  } else {
    const uint64_t u0 = lo * sizeof(T) / 4, u1 = (hi * sizeof(T) + 3) / 4;
    for (int k = 0; k < nb; k++) {
      const char* src = ptr(op.src[put && !(op.flags & F_PAIRED) ? 0 : k]);
      char* dst = ptr(op.dst[k]);
      const uint32_t flag = put ? pflag : runtime_flag(e, fstride, op.llflag_k[k]);
      for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
        if (put) {
          const uint32_t d = *reinterpret_cast<const uint32_t*>(src + u * 4);
          st8_volatile(dst + u * 8, make_uint2(d, flag));
        } else {
          uint2 v = ld8_volatile(src + u * 8);
          if (v.y != flag) {
            const uint64_t t0 = globaltimer();
            for (uint32_t it = 1; v.y != flag; ++it) {
              v = ld8_volatile(src + u * 8);
              if ((it & 255u) == 0) {
                if (*(volatile uint32_t*)&rs->error != kDevOk) break;
                if (globaltimer() - t0 > rs->timeout_ns) { atomicExch(&rs->error, (uint32_t)kDevTimeout); break; }
              }
            }
          }
          *reinterpret_cast<uint32_t*>(dst + u * 4) = v.x;
        }
      }
    }
  }
}

// Port channel ops: thread 0 posts one proxy request for this CTA's slice
// (copy-engine DMA), the signal (if any) targeting this CTA's lane of the
// receiver with the absolute count (call-1)*signals_per_call + m.  The CTA's
// prior writes to the source are published before the post.
template <typename T>
__device__ __noinline__ void port_op(const PlanArgs& a, const DevOp& op, int rank, int pid, int j, uint64_t e, RankState* rs,
                        uint64_t& last) {
  __threadfence_system();   // every thread's writes to the source, before the copy engine reads it
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t src = 0, dst = 0, bytes = 0;
  if (op.code == D_PORT_PUT) {
    uint64_t lo, hi;
    slice(op.size, op.per, j, lo, hi);
    if (hi > lo) {
      src = (uint64_t)(ptr(op.src[0]) + lo * sizeof(T));
      dst = (uint64_t)(ptr(op.dst[0]) + lo * sizeof(T));
      bytes = (hi - lo) * sizeof(T);
    }
  }
  const bool sig = op.code == D_PORT_SIGNAL || (op.flags & F_SIGNAL);
  if (!bytes && !sig) return;
  const uint64_t sem = sig ? (uint64_t)(a.lanes[op.peer] + (size_t)op.id * a.K + j) : 0;
  const uint64_t val = sig ? (e - 1) * op.per_call + op.m : 0;
  last = port_post(a.port[rank], src, dst, bytes, sem, val, (uint64_t)(a.port_done + (size_t)pid * a.K + j), rs);
}

// Prologue of a call, split over the rank's CTAs: copy the user input into the
// private input buffer (plans that write their input, e.g. ring RS) and zero
// the buffers the plan reads before writing (cf/executor.py:153-154).
__device__ __noinline__ void prologue(const PlanArgs& a, int rank) {
  const int cta = (int)blockIdx.x - a.rank_leader[rank];
  const int nct = a.rank_ctas[rank];
  const size_t stride = (size_t)nct * blockDim.x;
  const size_t t0 = (size_t)cta * blockDim.x + threadIdx.x;
  if (a.input_private) {
    const char* s = a.io_in[rank];
    char* d = a.bufptr[a.in_buf * a.n + rank];
    const size_t nb = a.buf_bytes[a.in_buf];
    for (size_t i = t0; i < nb / 16; i += stride) st16(d + i * 16, ld16(s + i * 16));
    for (size_t i = nb / 16 * 16 + t0; i < nb; i += stride) d[i] = s[i];
  }
  for (int z = 0; z < kMaxZero; z++) {
    const int b = a.zero_list[rank * kMaxZero + z];
    if (b < 0) break;
    char* d = b == a.out_buf ? a.io_out[rank] : a.bufptr[b * a.n + rank];
    const size_t nb = a.buf_bytes[b];
    for (size_t i = t0; i < nb / 16; i += stride) st16(d + i * 16, make_uint4(0, 0, 0, 0));
    for (size_t i = nb / 16 * 16 + t0; i < nb; i += stride) d[i] = 0;
  }
}

// Rewrite the staged window's I/O references as absolute addresses (the io
// buffers change per call).  Only when the host did not hand over an op array
// already resolved for this call's I/O binding (PlanArgs.resolved).
__device__ __forceinline__ void resolve_window(const PlanArgs& a, DevOp* ops, int nops, char* const* io) {
  constexpr int kSlots = kMaxSrc + kMaxDst;
  for (int t = threadIdx.x; t < nops * kSlots; t += blockDim.x) {
    DevOp& op = ops[t / kSlots];
    if (!is_data_code(op.code)) continue;
    const int k = t % kSlots;
    if (k < kMaxSrc ? k >= op.nsrc : k - kMaxSrc >= op.ndst) continue;
    DRef& r = k < kMaxSrc ? op.src[k] : op.dst[k - kMaxSrc];
    if (r.buf == kAbsolute) continue;
    char* base;
    if (r.buf == a.in_buf && !a.input_private) base = io[r.rank];
    else if (r.buf == a.out_buf) base = io[CF_MAX_RANKS + r.rank];
    else base = a.bufptr[r.buf * a.n + r.rank];
    r.off = reinterpret_cast<uint64_t>(base + r.off);
    r.buf = kAbsolute;
  }
}

// Op classes: one interpreter per class, so a plan runs the smallest body
// that covers its ops (less register pressure and a smaller instruction
// footprint on the latency path than one switch over every op kind).
//   kClsHB   sync ops, MULTI / COPY on plain vectors (memory-channel plans)
//   kClsLL   + LL packet ops and packet sources of MULTI
//   kClsAll  + port-channel requests through the proxy
enum PlanClass { kClsHB = 0, kClsLL = 1, kClsAll = 3 };

template <typename T, int CLS>
__global__ void __launch_bounds__(CF_PLAN_THREADS) plan_kernel(const __grid_constant__ PlanArgs a) {
  const int pid = blockIdx.x / a.K, j = blockIdx.x % a.K;
  TS_DECL
  TS_MARK();
  int rank, pb, pe;
  if (a.prog_in_param) {
    const int4 t = a.prog_tab[pid];
    rank = t.x, pb = t.y, pe = t.z;
  } else {
    rank = a.prog_rank[pid], pb = a.prog_begin[pid], pe = a.prog_end[pid];
  }
  PlanState* ps = a.st[rank];
  RankState* rs = &ps->base;
  // Ops are staged into shared memory in windows of a.window ops: every field
  // read of the interpreter then hits shared memory (the acquire loads of the
  // waits invalidate L1, which would otherwise send each field load to L2).
  // The first window's copy is in flight together with the epoch load.
  extern __shared__ uint4 s_raw[];
  DevOp* s_ops = reinterpret_cast<DevOp*>(s_raw);
  auto stage = [&](int w0, int w1) {
    const uint4* src = reinterpret_cast<const uint4*>(a.ops + w0);
    const int nvec = (w1 - w0) * (int)(sizeof(DevOp) / 16);
    for (int t = threadIdx.x; t < nvec; t += blockDim.x) s_raw[t] = src[t];
  };
  // the ranks' I/O bases in shared memory: the resolve pass indexes them per
  // thread, which on the parameter space would serialize the warp
  __shared__ char* s_io[2 * CF_MAX_RANKS];
  if (!a.resolved && threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < CF_MAX_RANKS; r++) {
      s_io[r] = a.io_in[r];
      s_io[CF_MAX_RANKS + r] = a.io_out[r];
    }
  }
  __shared__ uint64_t s_e;
  if (threadIdx.x == 0) s_e = *(volatile uint64_t*)&rs->epoch + 1;
  if (pb < pe) stage(pb, min(pb + a.window, pe));
  if (pid < a.npf) {   // the first data op's source lines, requested while its op is staged
    const PlanArgs::Prefetch& h = a.pf[pid];
    uint64_t lo, hi;
    slice(h.size, h.per, j, lo, hi);
    for (uint32_t k = 0; k < h.nsrc; k++)
      for (uint64_t b = lo * h.es + threadIdx.x * 128ull; b < hi * h.es; b += blockDim.x * 128ull)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(h.src[k] + b));
  }
  __syncthreads();
  const uint64_t e = s_e;
  TS_MARK();
  if (a.has_prologue) prologue(a, rank);
  // rank barriers are numbered consecutively across calls (monotonic counters)
  const uint64_t per_call = (uint64_t)(a.entry_barrier + a.exit_barrier);
  if (a.entry_barrier) rank_barrier(a, rank, (e - 1) * per_call + 1);
  [[maybe_unused]] uint64_t port_last = ~0ull;   // thread 0: this CTA's most recent proxy ticket
  const int end = pe;
  for (int w0 = pb; w0 < end; w0 += a.window) {
    const int w1 = min(w0 + a.window, end);
    if (w0 != pb) {
      __syncthreads();
      stage(w0, w1);
      __syncthreads();
    }
    if (!a.resolved) {
      resolve_window(a, s_ops, w1 - w0, s_io);
      __syncthreads();
    }
    TS_MARK();
  for (int i = w0; i < w1; i++) {
    const DevOp& op = s_ops[i - w0];
    TS_MARK();
    switch (op.code) {
      case D_SYNC_CTA:
        __syncthreads();
        break;
      case D_SYNC_GROUP:
      case D_DEV_BARRIER:
        counter_barrier(a.bars[rank] + op.id, ((e - 1) * op.per_call + op.m) * op.members, rs);
        break;
      case D_SIGNAL:   // ndst consecutive signals, one thread each, after every thread's fence
        fence_publish(a.gpu_scope);
        __syncthreads();
        if ((int)threadIdx.x < op.ndst) {
          const DRef& s = op.dst[threadIdx.x];
          red_add_release(a.lanes[s.rank] + (size_t)s.buf * a.K + j, 1, a.gpu_scope);
        }
        break;
      case D_WAIT:     // nsrc consecutive waits x K lanes, polled in parallel
        for (int t = threadIdx.x; t < op.nsrc * a.K; t += blockDim.x) {
          const DRef& w = op.src[t / a.K];
          wait_geq(a.lanes[rank] + (size_t)w.buf * a.K + (t % a.K), (e - 1) * (uint64_t)w.rank + w.off, rs,
                   a.gpu_scope);
        }
        __syncthreads();
        break;
      case D_MULTI:
      case D_COPY:
        if constexpr (CLS == kClsHB) {
          // plain vectors only in this class: no packet sources
          uint64_t lo, hi;
          slice(op.size, op.per, j, lo, hi);
          constexpr int V = 16 / sizeof(T);
          const uint64_t full = lo + (hi > lo ? (hi - lo) / V * V : 0);
          if ((op.flags & F_VEC) && op.code == D_MULTI && op.nsrc <= 8) {
            if (full > lo) multi_fast<T>(op, lo, full);
            if (full < hi) data_op_general<T>(op, full, hi, a.flag_stride, e, rs);
          } else if (lo < hi) {
            data_op_general<T>(op, lo, hi, a.flag_stride, e, rs);
          }
        } else {
          data_op<T>(a, op, j, e, rs);
        }
        break;
      case D_PUT_PACKETS:
      case D_READ_PACKETS:
        if constexpr ((CLS & kClsLL) != 0) packet_op<T>(op, a.K, j, a.flag_stride, e, rs);
        break;
      case D_PORT_PUT:
      case D_PORT_SIGNAL:
        if constexpr (CLS == kClsAll) port_op<T>(a, op, rank, pid, j, e, rs, port_last);
        break;
      case D_PORT_FLUSH:
        if constexpr (CLS == kClsAll) {
          if (threadIdx.x == 0 && port_last != ~0ull)
            port_flush(a.port_done + (size_t)pid * a.K + j, port_last, rs);
          __syncthreads();
        }
        break;
      default:
        break;
    }
    TS_MARK();
  }
  }
  // requests still in flight complete before the call ends (their data and
  // signals are part of this call)
  if constexpr (CLS == kClsAll)
    if (threadIdx.x == 0 && port_last != ~0ull) port_flush(a.port_done + (size_t)pid * a.K + j, port_last, rs);
  if (a.exit_barrier) rank_barrier(a, rank, e * per_call);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&rs->arrive, 1u);
    if (prev == (uint32_t)a.rank_ctas[rank] - 1) {   // no fence needed: see end_call
      *(volatile uint32_t*)&rs->arrive = 0;
      *(volatile uint64_t*)&rs->epoch = e;
    }
  }
  TS_MARK();
  TS_DUMP("plan", rank);
}

// The single-op plan kernel (see SingleArgs): CTA j of program p reduces its
// slice of the program's op with every source's load in flight, stores it to
// every destination, and the rank's last CTA publishes the call epoch.
template <typename T>
__global__ void __launch_bounds__(512) plan_single_kernel(const __grid_constant__ SingleArgs a) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  const int pid = blockIdx.x / a.K, j = blockIdx.x % a.K;
  const SingleArgs::Prog& P = a.p[pid];
  RankState* rs = a.st[P.rank];
  const bool bars = a.bar.entry | a.bar.exit;
  const uint64_t e = (threadIdx.x == 0 || bars) ? *(volatile uint64_t*)&rs->epoch + 1 : 0;
  const uint64_t per_call = (uint64_t)(a.bar.entry + a.bar.exit);
  if (a.bar.entry)   // one process per GPU: the peers' inputs are produced, their outputs free
    rank_barrier_raw(a.bar.pst, a.bar.n, P.rank, a.bar.leader[P.rank], a.rank_ctas[P.rank], (e - 1) * per_call + 1,
                     a.bar.gpu_scope);
  uint64_t lo, hi;
  slice(P.size, P.per, j, lo, hi);
  const int nsrc = P.nsrc, ndst = P.ndst;
  const bool multi = P.flags & 0x100, zero = P.flags & F_ZERO, round_each = P.flags & F_ROUND_EACH;
  const char* src[8];
  char* dst[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    src[i] = P.src[i];
    dst[i] = P.dst[i];
  }
  for (uint64_t v = lo / V + threadIdx.x; v * V < hi; v += blockDim.x) {
    const size_t boff = (size_t)v * 16;
    uint4 x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = i < nsrc ? ld16(src[i] + boff) : make_uint4(0, 0, 0, 0);
    uint4 res = x[0];
    if (multi) {
      A acc[V];
      if (zero) {
#pragma unroll
        for (int i = 0; i < V; i++) acc[i] = A(0);
        acc_vec<T>(acc, x[0], round_each);
      } else {
        Vec<T>::load(x[0], acc);
      }
#pragma unroll
      for (int i = 1; i < 8; i++)
        if (i < nsrc) acc_vec<T>(acc, x[i], round_each);
      res = Vec<T>::store(acc);
    }
#pragma unroll
    for (int d = 0; d < 8; d++)
      if (d < ndst) st16(dst[d] + boff, res);
  }
  if (a.bar.exit)    // nobody reads this rank's buffers once it returns
    rank_barrier_raw(a.bar.pst, a.bar.n, P.rank, a.bar.leader[P.rank], a.rank_ctas[P.rank], e * per_call,
                     a.bar.gpu_scope);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&rs->arrive, 1u);
    if (prev == (uint32_t)a.rank_ctas[P.rank] - 1) {
      *(volatile uint32_t*)&rs->arrive = 0;
      *(volatile uint64_t*)&rs->epoch = e;
    }
  }
}

// One payload unit of an unpaired PUT_PACKETS: one load, every range's packet.
// (`gpu`: every rank on this GPU, plain stores meet in its L2)
__device__ __forceinline__ void ll_bcast_unit(const LLArgs::Op& op, uint64_t u, uint32_t pflag, int nb, bool gpu) {
  const uint2 d = *reinterpret_cast<const uint2*>(op.src[0] + u * 8);
#pragma unroll
  for (int k = 0; k < 8; k++)
    if (k < nb) ll16_put_scoped(op.dst[k] + u * 16, d, pflag, gpu);
}

// One 8-byte unit of a MULTI / COPY: every source (plain unit or LL16
// packet) in flight, then the plan's order and rounding.
template <typename T>
__device__ __forceinline__ uint2 ll_multi_unit(const LLArgs::Op& op, uint64_t u, uint64_t e, uint32_t fs,
                                               RankState* rs) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  const int nsrc = op.nsrc, ndst = op.ndst;
  const uint32_t pkt = op.pkt_mask;
  uint4 x[8];
#pragma unroll
  for (int i = 0; i < 8; i++)
    if (i < nsrc) {
      if ((pkt >> i) & 1u) {
        x[i] = ld16_volatile(op.src[i] + u * 16);
      } else {
        const uint2 d = *reinterpret_cast<const uint2*>(op.src[i] + u * 8);
        x[i] = make_uint4(d.x, 0u, d.y, 0u);
      }
    }
  // unstamped packets are re-polled together, one round trip per round for
  // all of them (not one per late source)
  uint32_t pend = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
    if (i < nsrc && ((pkt >> i) & 1u)) {
      const uint32_t f = runtime_flag(e, fs, op.llflag_k[i]);
      if (x[i].y != f || x[i].w != f) pend |= 1u << i;
    }
  if (pend) {
    const uint64_t t0 = globaltimer();
    for (uint32_t it = 1; pend; ++it) {
#pragma unroll
      for (int i = 0; i < 8; i++)
        if ((pend >> i) & 1u) x[i] = ld16_volatile(op.src[i] + u * 16);
#pragma unroll
      for (int i = 0; i < 8; i++)
        if ((pend >> i) & 1u) {
          const uint32_t f = runtime_flag(e, fs, op.llflag_k[i]);
          if (x[i].y == f && x[i].w == f) pend &= ~(1u << i);
        }
      if ((it & 255u) == 0 && pend) {
        if (*(volatile uint32_t*)&rs->error != kDevOk) break;
        if (globaltimer() - t0 > rs->timeout_ns) {
          atomicExch(&rs->error, (uint32_t)kDevTimeout);
          break;
        }
      }
    }
  }
  uint2 res = make_uint2(x[0].x, x[0].z);
  if (op.code == D_MULTI) {
    const bool round_each = op.flags & F_ROUND_EACH;
    A acc[V];
    if (op.flags & F_ZERO) {
#pragma unroll
      for (int i = 0; i < V; i++) acc[i] = A(0);
      acc_vec<T>(acc, make_uint4(x[0].x, x[0].z, 0u, 0u), round_each);
    } else {
      Vec<T>::load(make_uint4(x[0].x, x[0].z, 0u, 0u), acc);
    }
#pragma unroll
    for (int i = 1; i < 8; i++)
      if (i < nsrc) acc_vec<T>(acc, make_uint4(x[i].x, x[i].z, 0u, 0u), round_each);
    const uint4 r4 = Vec<T>::store(acc);
    res = make_uint2(r4.x, r4.y);
  }
#pragma unroll
  for (int d = 0; d < 8; d++)
    if (d < ndst) *reinterpret_cast<uint2*>(op.dst[d] + u * 8) = res;
  return res;
}

// Streamed packet pairs: a thread reduces unit u this many of its iterations
// after putting it (the peers' packets for u then had as long to land).
#ifndef CF_PLL_LAG
#define CF_PLL_LAG 2
#endif
constexpr int kStreamLag = CF_PLL_LAG;
static_assert(kStreamLag == 1 || kStreamLag == 2, "stream lag of 1 or 2 iterations");

// The compiled LL plan kernel (see LLArgs).  Op fields are read from the
// parameter space (uniform per CTA); every thread reads the call epoch itself.
template <typename T>
__global__ void __launch_bounds__(512, 2) plan_ll_kernel(const __grid_constant__ LLArgs a) {
  constexpr int H = 8 / sizeof(T);   // elements per 8-byte payload unit
  TS_DECL
  TS_MARK();
  const int pid = blockIdx.x / a.K, j = blockIdx.x % a.K;
  const LLArgs::Prog& P = a.p[pid];
  RankState* rs = a.st[P.rank];
  const uint64_t e = *(volatile uint64_t*)&rs->epoch + 1;
  const uint32_t fs = a.flag_stride;
  const uint64_t per_call = (uint64_t)(a.bar.entry + a.bar.exit);
  if (a.bar.entry)
    rank_barrier_raw(a.bar.pst, a.bar.n, P.rank, a.bar.leader[P.rank], a.rank_ctas[P.rank], (e - 1) * per_call + 1,
                     a.bar.gpu_scope);
  TS_MARK();
  for (int oi = 0; oi < P.nops; oi++) {
    const LLArgs::Op& op = P.op[oi];
    TS_MARK();
    if (op.code == D_SYNC_CTA) {
      __syncthreads();
      continue;
    }
    uint64_t lo, hi;
    slice(op.size, op.per, j, lo, hi);
    if (lo >= hi) continue;
    const uint64_t u0 = lo / H, u1 = (hi + H - 1) / H;
    const uint32_t nu = (uint32_t)(u1 - u0);
    const bool streamed = oi == P.stream;   // host-checked pair: this PUT, then the MULTI after it
    if (op.code == D_PUT_PACKETS && !(op.flags & F_PAIRED) && !streamed) {
      // one payload to ndst ranges: one load per unit, every range's packet
      const uint32_t pflag = runtime_flag(e, fs, op.llflag);
      const int nb = op.ndst;
      for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) ll_bcast_unit(op, u, pflag, nb, a.bar.gpu_scope);
      continue;
    }
    if ((op.code == D_PUT_PACKETS || op.code == D_READ_PACKETS) && !streamed) {
      const bool put = op.code == D_PUT_PACKETS;
      const int nb = put ? op.ndst : op.nsrc;
      const bool paired = op.flags & F_PAIRED;
      const uint32_t pflag = put ? runtime_flag(e, fs, op.llflag) : 0u;
      const uint32_t items = nu * (uint32_t)nb;
      const float rnu = 1.0f / (float)nu;
      for (uint32_t w = threadIdx.x; w < items; w += blockDim.x) {
        uint32_t k = (uint32_t)((float)w * rnu);
        k -= k * nu > w;
        k += (k + 1) * nu <= w;
        const uint64_t u = u0 + (w - k * nu);
        if (put) {
          const uint2 d = *reinterpret_cast<const uint2*>(op.src[paired ? k : 0] + u * 8);
          ll16_put_scoped(op.dst[k] + u * 16, d, pflag, a.bar.gpu_scope);
        } else {
          const uint32_t f = runtime_flag(e, fs, op.llflag_k[k]);
          const uint4 raw = ld16_volatile(op.src[k] + u * 16);
          uint2 d = make_uint2(raw.x, raw.z);
          if (raw.y != f || raw.w != f) d = ll16_get(op.src[k] + u * 16, f, rs);
          *reinterpret_cast<uint2*>(op.dst[k] + u * 8) = d;
        }
      }
      continue;
    }
    // MULTI / COPY, one 8-byte payload unit per thread.  A streamed pair
    // (PUT_PACKETS + the MULTI reducing the packets the peers' puts land)
    // runs interleaved: a thread reduces unit u kStreamLag iterations after
    // putting it, and the peers' threads with the same index put it at about the same
    // time, so packets are read while still in L2 (the hand one-shot's
    // schedule; the host checked the pair's symmetry).  One call site of the
    // unit body keeps its in-flight sources in registers.
    // A fused broadcast (host-checked: the PUT_PACKETS two ops on sends this
    // MULTI's destination, the sync between them orders only that) takes the
    // reduced unit straight from registers.
    const bool fput = oi == P.fuse_put;
    const LLArgs::Op& m = P.op[oi + streamed];
    const LLArgs::Op& bp = P.op[oi + 2 * fput];
    const uint32_t pflag = streamed ? runtime_flag(e, fs, op.llflag) : fput ? runtime_flag(e, fs, bp.llflag) : 0u;
    constexpr uint64_t kNone = ~(uint64_t)0;
    uint64_t q0 = kNone, q1 = kNone;   // units put and not yet reduced (streamed)
    for (uint64_t u = u0 + threadIdx.x;; u += blockDim.x) {
      const bool has = u < u1;
      if (streamed && has) ll_bcast_unit(op, u, pflag, op.ndst, a.bar.gpu_scope);
      const uint64_t mu = streamed ? (kStreamLag == 2 ? q1 : q0) : (has ? u : kNone);
      if (mu != kNone) {
        const uint2 r = ll_multi_unit<T>(m, mu, e, fs, rs);
        if (fput) {
#pragma unroll
          for (int k = 0; k < 8; k++)
            if (k < bp.ndst) ll16_put_scoped(bp.dst[k] + mu * 16, r, pflag, a.bar.gpu_scope);
        }
      }
      if (kStreamLag == 2) q1 = q0;
      q0 = has ? u : kNone;
      if (!has && (!streamed || (q0 == kNone && q1 == kNone))) break;
    }
    oi += streamed + 2 * fput;
  }
  TS_MARK();
  if (a.bar.exit)
    rank_barrier_raw(a.bar.pst, a.bar.n, P.rank, a.bar.leader[P.rank], a.rank_ctas[P.rank], e * per_call,
                     a.bar.gpu_scope);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&rs->arrive, 1u);
    if (prev == (uint32_t)a.rank_ctas[P.rank] - 1) {
      *(volatile uint32_t*)&rs->arrive = 0;
      *(volatile uint64_t*)&rs->epoch = e;
    }
  }
  TS_MARK();
  TS_DUMP("planll", P.rank);
}

const void* plan_ll_kernel_for(int dtype) {
  switch (dtype) {
    case 0: return (const void*)plan_ll_kernel<int32_t>;
    case 1: return (const void*)plan_ll_kernel<float>;
    case 2: return (const void*)plan_ll_kernel<__half>;
    case 3: return (const void*)plan_ll_kernel<__nv_bfloat16>;
  }
  return nullptr;
}

const void* plan_single_kernel_for(int dtype) {
  switch (dtype) {
    case 0: return (const void*)plan_single_kernel<int32_t>;
    case 1: return (const void*)plan_single_kernel<float>;
    case 2: return (const void*)plan_single_kernel<__half>;
    case 3: return (const void*)plan_single_kernel<__nv_bfloat16>;
  }
  return nullptr;
}

template <int CLS>
static const void* by_dtype(int dtype) {
  switch (dtype) {
    case 0: return (const void*)plan_kernel<int32_t, CLS>;
    case 1: return (const void*)plan_kernel<float, CLS>;
    case 2: return (const void*)plan_kernel<__half, CLS>;
    case 3: return (const void*)plan_kernel<__nv_bfloat16, CLS>;
  }
  return nullptr;
}

// cls: bit 0 = the plan has LL packet ops, bit 1 = port-channel ops
const void* plan_kernel_for(int dtype, int cls) {
  if (cls & 2) return by_dtype<kClsAll>(dtype);
  if (cls & 1) return by_dtype<kClsLL>(dtype);
  return by_dtype<kClsHB>(dtype);
}

}  // namespace plan
}  // namespace cf
