// cf_collectives.cu -- hand-written sm_100a collective kernels.
//
//   K1 ll_oneshot      AllReduce, one-shot LL16 packets      build_1pa            cf/collectives.py:139-162
//   K2 pull_reduce     AllReduce, one-shot HB pull (whole)   MemoryChannel.reduce cf/channels.py:202-225
//   K3 pull_reduce     AllReduce, two-shot HB (push=1)       build_2pa memory     cf/collectives.py:187-197
//   K4 ll_twoshot      AllReduce, two-shot LL16 packets      build_2pa ll         cf/collectives.py:216-231
//   K6 push_gather     AllGather, direct peer stores         build_allpairs_ag    cf/collectives.py:253-270
//   K8 pull_reduce     ReduceScatter, all-pairs (rs_shift=1) 2PA RS phase         cf/collectives.py:188-191
//
// One launch serves every rank co-resident on a device: blockIdx.y selects the
// rank (CollArgs.rk), blockIdx.x the CTA within the rank.  CTA b of rank r
// only synchronizes with CTA b of its peers, through its own semaphore slot,
// so no kernel needs a grid-wide barrier.  All peer traffic is 16-byte
// vectors; element ranges that do not start/end on a vector boundary are
// handled with guarded element-wise loads and masked stores.
#include <cstdio>
#include "cf_kernels.cuh"
#include "cf_ts.cuh"

namespace cf {


// ---------------------------------------------------------------- call bracket

// Semaphore values are epoch * kPhases + phase (phase in [1, kPhases)) for every
// kernel, so a slot's value only grows no matter which kernels run in between.
constexpr uint64_t kPhases = 1ull << 20;

// Every CTA reads the rank's call counter once; the last CTA of the rank to
// finish publishes epoch+1 (last-CTA-done, no grid barrier).  Keeping the
// counter on the device makes the kernels CUDA-graph replayable.
__device__ __forceinline__ uint64_t begin_call(const RankCtx& rk) {
  __shared__ uint64_t s_e;
  if (threadIdx.x == 0) s_e = *(volatile uint64_t*)&rk.st->epoch + 1;
  __syncthreads();
  return s_e;
}

// No fences: every CTA of this launch read the epoch before its arrival was
// counted (the last arriver sees all of them), and the next launch on the
// stream sees these stores through the kernel boundary.  Data visibility to
// peers is the handshakes' / LL flags' business, not the epoch's.
// Single-launch HB kernels need the epoch only in thread 0 at the very end:
// load it without the block barrier so the data loads start right away.
__device__ __forceinline__ uint64_t begin_call_lazy(const RankCtx& rk, bool single) {
  if (!single) return begin_call(rk);
  return threadIdx.x == 0 ? *(volatile uint64_t*)&rk.st->epoch + 1 : 0;
}

__device__ __forceinline__ void end_call(const RankCtx& rk, uint64_t e) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&rk.st->arrive, 1u);
    if (prev == gridDim.x - 1) {
      *(volatile uint32_t*)&rk.st->arrive = 0;
      *(volatile uint64_t*)&rk.st->epoch = e;
    }
  }
}

// CTA-pair handshake with every peer: signal value `v` to CTA b of each peer,
// then wait until each peer's CTA b signalled >= v.  `publish` makes this
// CTA's prior global writes visible system-wide first (fence before signal,
// cf/channels.py:227-232).
// `publish`: EVERY thread fences its own prior writes before the barrier --
// one thread's fence after bar.sync is not relied on to cover the other
// warps' stores still in flight (a rare stale read of the emulated NVLS
// kernel pointed at exactly that).
__device__ __forceinline__ void handshake(const RankCtx& rk, int n, uint64_t v, bool publish, bool gpu) {
  const int t = threadIdx.x, r = rk.rank, b = blockIdx.x;
  if (publish) {
#if CF_DROP_FENCE != 1
    fence_publish(gpu);
#endif
    __syncthreads();
  }
  if (t < n && t != r) {
    CF_STRESS_AT(10);
#if CF_DROP_FENCE == 1
    st_relaxed(rk.sem[t] + sem_index(r, b), v, gpu);
#else
    st_release(rk.sem[t] + sem_index(r, b), v, gpu);
#endif
#if CF_DROP_FENCE == 5
    if (!publish)
#endif
      wait_geq(rk.sem[r] + sem_index(t, b), v, rk.st, gpu);
  }
  __syncthreads();
}

// Barrier over every CTA of every rank, in two halves: cta_arrive publishes
// this CTA's writes and marks slot (r, b) on every rank; all_wait returns
// once all n x G slots of this rank carry `v` (every thread of the CTA calls
// both, each with the call's epoch in `v`).  The whole grid of every rank
// must be resident (the CTA budget / co-residency cap guarantees it).
__device__ __forceinline__ void cta_arrive(const RankCtx& rk, int n, uint64_t v, bool gpu) {
  const int t = threadIdx.x, r = rk.rank, b = blockIdx.x;
#if CF_DROP_FENCE != 1
  fence_publish(gpu);
#endif
  __syncthreads();
  if (t < n) {
    CF_STRESS_AT(10);
#if CF_DROP_FENCE == 1
    st_relaxed(rk.sem[t] + sem_index(r, b), v, gpu);
#else
    st_release(rk.sem[t] + sem_index(r, b), v, gpu);
#endif
  }
}
// ... or once every CTA of every rank has: one thread per slot, all n x G
// slots polled in parallel (measured: one warp polling every slot with
// relaxed loads and one acquire fence is slower, C5 K13 b=256 37.5 vs 36.9 us)
__device__ __forceinline__ void all_wait(const RankCtx& rk, int n, uint64_t v, bool gpu) {
  const int G = gridDim.x;
  for (int i = threadIdx.x; i < n * G; i += blockDim.x) wait_geq(rk.sem[rk.rank] + sem_index(i / G, i % G), v, rk.st, gpu);
  __syncthreads();
}

// ---------------------------------------------------------------- vector helpers

// Ragged-edge paths stay out of line: the small-message kernels execute each
// instruction about once per launch on a cold instruction cache, so code size
// on the latency path is latency (one copy of the edge code, not one per
// unrolled peer).
template <int ES>
__device__ __noinline__ uint4 ld_partial16_ool(const char* p, int nbytes) {
  return ld_partial16<ES>(p, nbytes);
}
template <int ES>
__device__ __noinline__ void st_masked16_ool(char* p, uint4 v, int jlo, int jhi) {
  st_masked16<ES>(p, v, jlo, jhi);
}

// Load 16-byte vector `v` of a T array of `count` elements; lanes past the end
// read as zero.
template <typename T>
__device__ __forceinline__ uint4 load_vec(const char* base, size_t v, size_t count) {
  constexpr int V = 16 / sizeof(T);
  const size_t e0 = v * V;
  if (e0 + V <= count) return ld16(base + v * 16);
  const int nb = e0 < count ? (int)((count - e0) * sizeof(T)) : 0;
  return ld_partial16_ool<sizeof(T)>(base + v * 16, nb);
}

// Store the lanes of vector `v` whose element index lies in [lo, hi) at
// element position (index - shift) of `base`.
template <typename T>
__device__ __forceinline__ void store_vec(char* base, size_t v, uint4 val, size_t lo, size_t hi,
                                          size_t shift) {
  constexpr int V = 16 / sizeof(T);
  const size_t e0 = v * V;
  char* p = base + (e0 - shift) * sizeof(T);
  if (e0 >= lo && e0 + V <= hi && ((uintptr_t)p & 15) == 0) {
    st16(p, val);
    return;
  }
  const int jlo = lo > e0 ? (int)min(lo - e0, (size_t)V) : 0;
  const int jhi = hi > e0 ? (int)min(hi - e0, (size_t)V) : 0;
  st_masked16_ool<sizeof(T)>(p, val, jlo, jhi);
}

// 8-byte payload units (one LL16 packet each): unit u of a T array of
// `count` elements; ragged last unit out of line.
template <typename T>
__device__ __forceinline__ uint2 load_unit(const char* base, size_t u, size_t count) {
  constexpr int H = 8 / sizeof(T);
  const size_t e0 = u * H;
  if (e0 + H <= count) return ld8(base + u * 8);
  const int nb = e0 < count ? (int)((count - e0) * sizeof(T)) : 0;
  const uint4 w = ld_partial16_ool<sizeof(T)>(base + u * 8, nb);
  return make_uint2(w.x, w.y);
}
template <typename T>
__device__ __forceinline__ void store_unit(char* base, size_t u, uint2 val, size_t count) {
  constexpr int H = 8 / sizeof(T);
  const size_t e0 = u * H;
  if (e0 + H <= count) {
    st8(base + u * 8, val);
    return;
  }
  const int jhi = e0 < count ? (int)(count - e0) : 0;
  st_masked16_ool<sizeof(T)>(base + u * 8, make_uint4(val.x, val.y, 0u, 0u), 0, jhi);
}

// Accumulate NR (runtime n <= NR) 16-byte vectors in order: x[0] first (or a
// zero accumulator when `zero`), then x[1], x[2], ...  f16/bf16 accumulate in
// f32 and round once; i32 wraps; f32 is one RNE add per source.
template <typename T, int NR>
__device__ __forceinline__ uint4 reduce_vecs(const uint4 (&x)[NR], int n, bool zero) {
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  A acc[V];
  if (zero) {
#pragma unroll
    for (int j = 0; j < V; j++) acc[j] = A(0);
  } else {
    Vec<T>::load(x[0], acc);
  }
#pragma unroll
  for (int k = 0; k < NR; k++) {
    if (k < n && (zero || k > 0)) {
      A t[V];
      Vec<T>::load(x[k], t);
#pragma unroll
      for (int j = 0; j < V; j++) acc[j] = acc_add(acc[j], t[j]);
    }
  }
  return Vec<T>::store(acc);
}

// reduce_vecs on 8-byte units (the upper half of each vector is zero and its
// lanes are dead code).
template <typename T, int NR>
__device__ __forceinline__ uint2 reduce_units(const uint2 (&x)[NR], int n) {
  uint4 w[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) w[k] = make_uint4(x[k].x, x[k].y, 0u, 0u);
  const uint4 res = reduce_vecs<T, NR>(w, n, false);
  return make_uint2(res.x, res.y);
}

// ---------------------------------------------------------------- K2 / K3 / K8

// Pull-reduce: after an entry handshake (peers' send buffers are produced and
// their recv buffers free), rank r reads its range from all n send buffers in
// the reference order, reduces, and stores to its own recv buffer (K2, K8) or
// to every rank's recv buffer (K3, `push`).  An exit handshake guarantees no
// peer still reads r's send buffer when r's kernel retires.
template <typename T, int NR>
__global__ void __launch_bounds__(512) pull_reduce_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int V = Vec<T>::N;
  const int n = a.n, r = rk.rank;
  const uint64_t e = begin_call_lazy(rk, a.single_launch);
  if (!a.single_launch) handshake(rk, n, e * kPhases + 1, false, a.gpu_scope);

  size_t lo = 0, hi = a.count;
  if (!a.whole) {
    const size_t c0 = (size_t)r * a.cs;
    lo = min(c0 + a.win_lo, a.count);
    hi = min(c0 + min(a.cs, a.win_hi), a.count);
    lo = min(lo, hi);
  }
  const bool zero = a.order != kLead;
  const char* src[NR];
#pragma unroll
  for (int k = 0; k < NR; k++) src[k] = k < n ? rk.in[order_src(a.order, k, r, n)] : nullptr;
  const size_t shift = a.rs_shift ? lo : 0;
  const size_t vlo = lo / V, vhi = (hi + V - 1) / V;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t v = vlo + (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < vhi; v += stride) {
    uint4 x[NR];
#pragma unroll
    for (int k = 0; k < NR; k++)
      if (k < n) x[k] = load_vec<T>(src[k], v, a.count);
    const uint4 res = reduce_vecs<T, NR>(x, n, zero);
    if (a.push) {
#pragma unroll
      for (int p = 0; p < NR; p++)
        if (p < n) store_vec<T>(rk.out[p], v, res, lo, hi, 0);
    } else {
      store_vec<T>(rk.out[r], v, res, lo, hi, shift);
    }
  }
  if (!a.single_launch) handshake(rk, n, e * kPhases + 2, true, a.gpu_scope);
  end_call(rk, e);
}

// ---------------------------------------------------------------- K1

// One-shot LL: every rank writes its whole send buffer as LL16 packets into
// slot r of each peer's scratch (parity half e&1), then polls its own n-1
// slots and reduces in the 1pa order (own input first, peers ascending,
// cf/collectives.py:156-161).  No semaphores, no fences: the flag travels in
// the same 16-byte store as the data.  One thread per 8-byte payload unit
// (= one packet), so a warp's packet stores to a peer cover 512 contiguous
// bytes.  Latency structure: the first input load is issued before the epoch
// read; the read phase keeps every peer's packet in flight and re-polls all
// unstamped ones per round (ll16_poll): waiting for n-1 peers costs one round
// trip per round, not one per peer.
// Packet units per thread per round in K4's scatter / gather phases.
#ifndef CF_LL2U
#define CF_LL2U 4
#endif
constexpr int kLL2U = CF_LL2U;

#ifndef CF_LL1_STREAM
#define CF_LL1_STREAM 1
#endif
#ifndef CF_LL1_LAG
#define CF_LL1_LAG 2
#endif
template <typename T, int NR>
__global__ void __launch_bounds__(512, 2) ll_oneshot_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int P = NR - 1;
  constexpr int H = 8 / sizeof(T);
  const int n = a.n, r = rk.rank;
  TS_DECL
  TS_MARK();
  const size_t nunit = (a.count + H - 1) / H;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint2 first = t0 < nunit ? load_unit<T>(rk.in[r], t0, a.count) : make_uint2(0u, 0u);
  const uint64_t e = begin_call(rk);
  TS_MARK();
  const uint32_t flag = ll_flag(e);
  const size_t par = (e & 1) * a.half;

  const uint32_t all = (1u << (n - 1)) - 1u;
  auto put = [&](size_t u, uint2 x) {
#pragma unroll
    for (int p = 0; p < NR; p++)
      if (p < n && p != r) ll16_put_scoped(rk.scr[p] + par + (size_t)r * a.slot + u * 16, x, flag, a.gpu_scope);
  };
  auto read = [&](size_t u, uint2 own) {
    const char* base = rk.scr[r] + par + u * 16;
    uint4 pk[P];
#pragma unroll
    for (int i = 0; i < P; i++)
      if (i < n - 1) pk[i] = ld16_volatile(ll_unit(base, a.slot, r, i));
    ll16_poll<P>(base, a.slot, r, pk, all, flag, rk.st);
    uint2 x[NR];
    x[0] = own;
#pragma unroll
    for (int i = 0; i < P; i++) x[i + 1] = make_uint2(pk[i].x, pk[i].z);
    store_unit<T>(rk.out[r], u, reduce_units<T, NR>(x, n), a.count);
  };
#if CF_LL1_STREAM
  // Streamed: every thread reads unit u CF_LL1_LAG iterations after putting
  // it (the peers' threads with the same index put it at about the same
  // time), so packets are consumed while they are still in L2 instead of after
  // the whole message was scattered.  Every rank launches the same grid (same
  // count, same occupancy on a homogeneous box), so the unit a thread waits
  // for was put, iterations earlier, by a thread that is itself never waiting
  // on a later unit.  Lag 2 (default) vs 1: the peers' packets had two put
  // rounds to land, fewer re-polls (1 MiB 42.0 -> 37.2 us, 4 MiB 166 -> 162 us,
  // 16 KiB 5.1 -> 4.9 us; 8 co-resident ranks, bf16).
#if CF_LL1_LAG == 2
  uint2 prev = first, prev2 = make_uint2(0u, 0u);
  for (size_t u = t0; u < nunit; u += stride) {
    const uint2 x = u == t0 ? first : load_unit<T>(rk.in[r], u, a.count);
    put(u, x);
    if (u >= t0 + 2 * stride) read(u - 2 * stride, prev2);
    prev2 = prev;
    prev = x;
  }
  if (t0 < nunit) {
    const size_t last = t0 + (nunit - 1 - t0) / stride * stride;
    if (last >= t0 + stride) read(last - stride, prev2);
    read(last, prev);
  }
#else
  uint2 prev = first;
  for (size_t u = t0; u < nunit; u += stride) {
    const uint2 x = u == t0 ? first : load_unit<T>(rk.in[r], u, a.count);
    put(u, x);
    if (u != t0) read(u - stride, prev);
    prev = x;
  }
  if (t0 < nunit) read(t0 + (nunit - 1 - t0) / stride * stride, prev);
#endif
#else
  for (size_t u = t0; u < nunit; u += stride) put(u, u == t0 ? first : load_unit<T>(rk.in[r], u, a.count));
  TS_MARK();
  for (size_t u = t0; u < nunit; u += stride) read(u, u == t0 ? first : load_unit<T>(rk.in[r], u, a.count));
#endif
  TS_MARK();
  end_call(rk, e);
  TS_MARK();
  TS_DUMP("1pa", rk.rank);
}

// ---------------------------------------------------------------- K4

// Two-shot LL (cf/collectives.py:216-231): phase 1 sends chunk p of the send
// buffer as packets into peer p's ph1 slot r; rank r reduces chunk r (owner
// first, peers ascending), stores it, and sends the result as packets into
// every peer's ph2 slot r; phase 2 decodes the peers' chunks into recv.
// Chunks follow the reference chunking (cs elements); packets carry the
// 16-byte vectors covering a chunk, and stores are masked to the chunk.
// Each phase issues all of its loads (inputs, every peer's packets) before
// the first store / poll check, so a phase costs one round trip, not n-1.
template <typename T, int NR>
__global__ void __launch_bounds__(512) ll_twoshot_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int V = Vec<T>::N;
  constexpr int P = NR - 1;
  const int n = a.n, r = rk.rank;
  TS_DECL
  TS_MARK();
  const uint64_t e = begin_call(rk);
  TS_MARK();
  const uint32_t flag = ll_flag(e);
  const size_t ph1 = (e & 1) * a.half, ph2 = ph1 + (size_t)n * a.slot;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  auto clo = [&](int c) { return min((size_t)c * a.cs, a.count); };
  auto chi = [&](int c) { return min((size_t)c * a.cs + a.cs, a.count); };
  auto vlo = [&](int c) { return clo(c) / V; };
  auto vhi = [&](int c) { return (chi(c) + V - 1) / V; };
  const size_t nvmax = (a.cs + V - 1) / V + 1;   // vectors covering any chunk
  // Chunk bounds min(c * cs, count) on the 8-byte unit grid (cs and count
  // multiples of H, the common case): every unit belongs to exactly one
  // chunk, so each phase runs one 8-byte unit (= one packet) per thread over
  // the whole buffer (peer = u / cu) -- all threads busy, contiguous packet
  // stores, one short code path.  Otherwise the per-chunk vector loops below
  // handle 16-byte vectors that straddle two chunks.
  constexpr int H = 8 / sizeof(T);
  const bool grid = a.cs % H == 0 && a.count % H == 0;
  const uint32_t cu = (uint32_t)(a.cs / H);
  const size_t nunit = a.count / H;

  // phase 1: scatter my chunks as packets
  if (grid) {   // kLL2U units per thread per round: their loads in flight together
    for (size_t ub = t0; ub < nunit; ub += (size_t)kLL2U * stride) {
      uint2 x[kLL2U];
#pragma unroll
      for (int j = 0; j < kLL2U; j++) {
        const size_t u = ub + (size_t)j * stride;
        if (u < nunit && (int)((uint32_t)u / cu) != r) x[j] = ld8(rk.in[r] + u * 8);
      }
#pragma unroll
      for (int j = 0; j < kLL2U; j++) {
        const size_t u = ub + (size_t)j * stride;
        if (u >= nunit) break;
        const uint32_t p = (uint32_t)u / cu, i = (uint32_t)u - p * cu;
        if ((int)p != r)
          ll16_put_scoped(rk.scr[p] + ph1 + (size_t)r * a.slot + (size_t)i * 16, x[j], flag, a.gpu_scope);
      }
    }
  } else for (size_t i = t0; i < nvmax; i += stride) {   // every peer's input vector loaded first
    uint4 x[NR];
#pragma unroll
    for (int p = 0; p < NR; p++)
      if (p < n && p != r && vlo(p) + i < vhi(p)) x[p] = load_vec<T>(rk.in[r], vlo(p) + i, a.count);
#pragma unroll
    for (int p = 0; p < NR; p++) {
      if (p < n && p != r && vlo(p) + i < vhi(p)) {
        char* d = rk.scr[p] + ph1 + (size_t)r * a.slot + i * 32;
        ll16_put_scoped(d, make_uint2(x[p].x, x[p].y), flag, a.gpu_scope);
        ll16_put_scoped(d + 16, make_uint2(x[p].z, x[p].w), flag, a.gpu_scope);
      }
    }
  }
  TS_MARK();
  // reduce my chunk (owner first, peers ascending), store, broadcast as packets
  const uint32_t all = (1u << (n - 1)) - 1u;
  if (grid) {
    const size_t u0 = min((size_t)r * cu, nunit), nu = min(u0 + cu, nunit) - u0;
    for (size_t i = t0; i < nu; i += stride) {
      const uint2 own = ld8(rk.in[r] + (u0 + i) * 8);
      const char* base = rk.scr[r] + ph1 + i * 16;
      uint4 pk[P];
#pragma unroll
      for (int k = 0; k < P; k++)
        if (k < n - 1) pk[k] = ld16_volatile(ll_unit(base, a.slot, r, k));
      ll16_poll<P>(base, a.slot, r, pk, all, flag, rk.st);
      uint2 x[NR];
      x[0] = own;
#pragma unroll
      for (int k = 0; k < P; k++) x[k + 1] = make_uint2(pk[k].x, pk[k].z);
      const uint2 res = reduce_units<T, NR>(x, n);
      st8(rk.out[r] + (u0 + i) * 8, res);
#pragma unroll
      for (int p = 0; p < NR; p++)
        if (p < n && p != r) ll16_put_scoped(rk.scr[p] + ph2 + (size_t)r * a.slot + i * 16, res, flag, a.gpu_scope);
    }
  } else {
    const size_t b = vlo(r), nv = vhi(r) > b ? vhi(r) - b : 0;
    for (size_t i = t0; i < nv; i += stride) {
      const uint4 own = load_vec<T>(rk.in[r], b + i, a.count);
      const char* base = rk.scr[r] + ph1 + i * 32;
      uint4 r0[P], r1[P];
#pragma unroll
      for (int k = 0; k < P; k++) {
        if (k < n - 1) {
          const char* u = ll_unit(base, a.slot, r, k);
          r0[k] = ld16_volatile(u);
          r1[k] = ld16_volatile(u + 16);
        }
      }
      ll16x2_poll<P>(base, a.slot, r, r0, r1, all, flag, rk.st);
      uint4 x[NR];
      x[0] = own;
#pragma unroll
      for (int k = 0; k < P; k++)
        if (k < n - 1) x[k + 1] = ll16x2_payload(r0[k], r1[k]);
      const uint4 res = reduce_vecs<T, NR>(x, n, false);
      store_vec<T>(rk.out[r], b + i, res, clo(r), chi(r), 0);
#pragma unroll
      for (int p = 0; p < NR; p++) {
        if (p < n && p != r) {
          char* d = rk.scr[p] + ph2 + (size_t)r * a.slot + i * 32;
          ll16_put_scoped(d, make_uint2(res.x, res.y), flag, a.gpu_scope);
          ll16_put_scoped(d + 16, make_uint2(res.z, res.w), flag, a.gpu_scope);
        }
      }
    }
  }
  TS_MARK();
  // phase 2: decode the peers' reduced chunks
  if (grid) {   // kLL2U packets per thread in flight, unstamped ones re-polled together
    for (size_t ub = t0; ub < nunit; ub += (size_t)kLL2U * stride) {
      const char* src[kLL2U];
      uint4 pk[kLL2U];
      uint32_t pend = 0;
#pragma unroll
      for (int j = 0; j < kLL2U; j++) {
        const size_t u = ub + (size_t)j * stride;
        if (u >= nunit) break;
        const uint32_t p = (uint32_t)u / cu, i = (uint32_t)u - p * cu;
        if ((int)p == r) continue;
        src[j] = rk.scr[r] + ph2 + (size_t)p * a.slot + (size_t)i * 16;
        pk[j] = ld16_volatile(src[j]);
        pend |= 1u << j;
      }
      const uint32_t todo = pend;
#pragma unroll
      for (int j = 0; j < kLL2U; j++)
        if (((pend >> j) & 1u) && pk[j].y == flag && pk[j].w == flag) pend &= ~(1u << j);
      if (pend) {
        const uint64_t tw = globaltimer();
        for (uint32_t it = 1; pend; ++it) {
#pragma unroll
          for (int j = 0; j < kLL2U; j++)
            if ((pend >> j) & 1u) pk[j] = ld16_volatile(src[j]);
#pragma unroll
          for (int j = 0; j < kLL2U; j++)
            if (((pend >> j) & 1u) && pk[j].y == flag && pk[j].w == flag) pend &= ~(1u << j);
          if ((it & 255u) == 0 && pend) {
            if (*(volatile uint32_t*)&rk.st->error != kDevOk) break;
            if (globaltimer() - tw > rk.st->timeout_ns) { atomicExch(&rk.st->error, (uint32_t)kDevTimeout); break; }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kLL2U; j++)
        if ((todo >> j) & 1u) st8(rk.out[r] + (ub + (size_t)j * stride) * 8, make_uint2(pk[j].x, pk[j].z));
    }
  } else for (size_t i = t0; i < nvmax; i += stride) {   // all peers' packets of vector i in flight
    const char* base = rk.scr[r] + ph2 + i * 32;
    uint4 r0[NR], r1[NR];
    uint32_t pend = 0;
#pragma unroll
    for (int p = 0; p < NR; p++) {
      if (p < n && p != r && vlo(p) + i < vhi(p)) {
        const char* u = base + (size_t)p * a.slot;
        r0[p] = ld16_volatile(u);
        r1[p] = ld16_volatile(u + 16);
        pend |= 1u << p;
      }
    }
    ll16x2_poll<NR>(base, a.slot, NR, r0, r1, pend, flag, rk.st);
#pragma unroll
    for (int p = 0; p < NR; p++)
      if ((pend >> p) & 1u) store_vec<T>(rk.out[r], vlo(p) + i, ll16x2_payload(r0[p], r1[p]), clo(p), chi(p), 0);
  }
  TS_MARK();
  end_call(rk, e);
  TS_MARK();
  TS_DUMP("2pa_ll", rk.rank);
}

// ---------------------------------------------------------------- K6

// Direct AllGather: entry handshake (peer recv buffers free), then each rank
// stores its shard into slot r of every rank's recv buffer, then an exit
// handshake publishes the data (put + signal, wait; cf/collectives.py:262-269).
template <typename T>
__global__ void __launch_bounds__(512) push_gather_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int V = 16 / sizeof(T);
  const int n = a.n, r = rk.rank;
  const uint64_t e = begin_call_lazy(rk, a.single_launch);
  if (!a.single_launch) handshake(rk, n, e * kPhases + 1, false, a.gpu_scope);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t sb = a.count * sizeof(T);
  if ((sb & 15) == 0) {
    const size_t nvec = sb / 16;
    for (size_t v = t0; v < nvec; v += stride) {
      const uint4 x = ld16(rk.in[r] + v * 16);
#pragma unroll 8
      for (int p = 0; p < CF_MAX_RANKS; p++)
        if (p < n) st16(rk.out[p] + (size_t)r * sb + v * 16, x);
    }
  } else {
    // ragged shard: slot r starts off the 16-byte grid; vector loads, element stores
    const size_t nvec = (a.count + V - 1) / V;
    for (size_t v = t0; v < nvec; v += stride) {
      const uint4 x = load_vec<T>(rk.in[r], v, a.count);
      for (int p = 0; p < n; p++)
        store_vec<T>(rk.out[p] + (size_t)r * sb, v, x, 0, a.count, 0);
    }
  }
  if (!a.single_launch) handshake(rk, n, e * kPhases + 2, true, a.gpu_scope);
  end_call(rk, e);
}

// K6 bulk: the same direct AllGather on the TMA bulk-copy engine.  One warp
// per CTA; lane 0 streams the shard through two 32 KiB shared-memory stages
// -- cp.async.bulk global -> shared (mbarrier complete_tx), then one
// cp.async.bulk shared -> global store per rank from the same stage -- so a
// tile is read from HBM once and written n times by the copy engine, with
// no register staging and one instruction per 32 KiB per destination.
// Needs a 16-byte-multiple shard and 16-byte-aligned buffers.
#ifndef CF_BULK_TILE_KB
#define CF_BULK_TILE_KB 32
#endif
constexpr int kBulkTile = CF_BULK_TILE_KB * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(32) push_gather_bulk_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  const int n = a.n, r = rk.rank;
  extern __shared__ __align__(128) char sbuf[];   // 2 stages of kBulkTile
  __shared__ __align__(8) uint64_t mbar[2];
  const uint64_t e = begin_call(rk);
  if (!a.single_launch) handshake(rk, n, e * kPhases + 1, false, a.gpu_scope);
  const size_t sb = a.count * sizeof(T);
  const size_t ntiles = (sb + kBulkTile - 1) / kBulkTile;
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const char* src = rk.in[r];
    auto tile_bytes = [&](size_t t) { return (uint32_t)min((size_t)kBulkTile, sb - t * kBulkTile); };
    size_t t = blockIdx.x;
    if (t < ntiles) {
      mbar_expect_tx(&mbar[0], tile_bytes(t));
      bulk_load(sbuf, src + t * kBulkTile, tile_bytes(t), &mbar[0]);
    }
    for (uint32_t k = 0; t < ntiles; k++, t += gridDim.x) {
      const int st = k & 1;
      const size_t tn = t + gridDim.x;
      if (tn < ntiles) {
        // the other stage still feeds the stores of tile k-1: wait until they read it
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_expect_tx(&mbar[st ^ 1], tile_bytes(tn));
        bulk_load(sbuf + (st ^ 1) * kBulkTile, src + tn * kBulkTile, tile_bytes(tn), &mbar[st ^ 1]);
      }
      mbar_wait(&mbar[st], (k >> 1) & 1);
      for (int p = 0; p < n; p++)
        bulk_store(rk.out[p] + (size_t)r * sb + t * kBulkTile, sbuf + st * kBulkTile, tile_bytes(t));
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // every store performed
    asm volatile("fence.proxy.async.global;" ::: "memory");      // ... and ordered before generic accesses
  }
  __syncwarp();
  if (!a.single_launch) handshake(rk, n, e * kPhases + 2, true, a.gpu_scope);
  end_call(rk, e);
}

// ---------------------------------------------------------------- K5

// NVLS switch primitives (multimem_ld_reduce / multimem_st16) live in
// device/cf_device.cuh with the SwitchChannelDevice they back.

// Switch reductions each thread keeps in flight in the NVLS kernels: one
// multimem.ld_reduce is a round trip through NVSwitch, so a single one per
// thread caps a rank far below its NVLink rate.
#ifndef CF_NVLS_U
#define CF_NVLS_U 4
#endif
constexpr int kNvlsU = CF_NVLS_U;

// K5 NVLS AllReduce (build_switch_2pa, cf/collectives.py:235-250; switch_reduce /
// switch_broadcast, cf/channels.py:367-409), one launch per call.  The message
// runs in pieces of the staging half; per piece:
//   A  copy the send buffer into the own multicast-bound input half,
//   B  (after the entry handshake) multimem.ld_reduce the slice of chunk r and
//      multimem.st it into every member's output half,
//   C  (after the exit handshake) copy the own output half into recv.
// Vector v of a piece belongs to chunk v / cv and, within it, to CTA
// (v mod cv) / per on EVERY rank, in all three phases and in every piece, so
// the CTA-pair handshakes (CTA b of each rank) order exactly the accesses
// that meet.
// `emul` replaces the two multimem instructions by per-rank loads / stores
// (0 + x_0 + x_1 + ..., the reference switch order) on unicast staging, so the
// co-resident world exercises this control path on one GPU.
template <typename T>
__global__ void __launch_bounds__(512) nvls_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int V = 16 / sizeof(T);
  const int n = a.n, r = rk.rank, b = blockIdx.x, B = gridDim.x;
  const uint64_t e = begin_call(rk);
  const size_t total = (a.count + V - 1) / V;      // 16-byte vectors of the message
  const size_t piece = a.half / 16;                // vectors per staging half
  char* my_in = rk.nv[r];
  char* my_out = rk.nv[r] + a.half;
  // The chunk / CTA owning staging vector v must be the same in EVERY piece:
  // the handshakes order CTA b with the CTAs b of the other ranks only, so a
  // CTA that moves on to the next piece must never touch an offset another
  // CTA of its rank may still read.  cv / per therefore come from the first
  // (largest) piece; a shorter last piece just ends early (v < pv).
  const size_t cv = (min(piece, total) + n - 1) / n;
  const size_t per = (cv + B - 1) / B;
  const size_t w0 = min((size_t)b * per, cv), w1 = min(w0 + per, cv);
  int ph = 1;
  for (size_t p0 = 0; p0 < total; p0 += piece, ph += 2) {
    const size_t pv = min(piece, total - p0);
    // A: this CTA's share of every chunk, send buffer -> own input half
    for (int o = 0; o < n; o++)
      for (size_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
        const size_t v = (size_t)o * cv + w;
        if (v < pv) st16(my_in + v * 16, load_vec<T>(rk.in[r], p0 + v, a.count));
      }
    handshake(rk, n, e * kPhases + ph, true, a.gpu_scope);
    // B: reduce chunk r across the members, broadcast the result
    const size_t base = (size_t)r * cv;
    const size_t we = pv > base ? min(w1, pv - base) : 0;
    size_t w = w0 + threadIdx.x;
    if (!a.emul)   // kNvlsU switch reductions in flight per thread
      for (; w + (kNvlsU - 1) * blockDim.x < we; w += kNvlsU * blockDim.x) {
        uint4 x[kNvlsU];
#pragma unroll
        for (int u = 0; u < kNvlsU; u++) x[u] = multimem_ld_reduce<T>(rk.nv_mc + (base + w + u * blockDim.x) * 16);
#pragma unroll
        for (int u = 0; u < kNvlsU; u++) multimem_st16(rk.nv_mc + a.half + (base + w + u * blockDim.x) * 16, x[u]);
      }
    for (; w < we; w += blockDim.x) {
      const size_t v = base + w;
      if (!a.emul) {
        multimem_st16(rk.nv_mc + a.half + v * 16, multimem_ld_reduce<T>(rk.nv_mc + v * 16));
      } else {
        uint4 x[CF_MAX_RANKS];
#pragma unroll
        for (int q = 0; q < CF_MAX_RANKS; q++)
          if (q < n) x[q] = ld16_cg(rk.nv[q] + v * 16);
        const uint4 res = reduce_vecs<T, CF_MAX_RANKS>(x, n, true);
#pragma unroll
        for (int q = 0; q < CF_MAX_RANKS; q++)
          if (q < n) st16(rk.nv[q] + a.half + v * 16, res);
      }
    }
    handshake(rk, n, e * kPhases + ph + 1, true, a.gpu_scope);
    // C: this CTA's share of every chunk, own output half -> recv
    for (int o = 0; o < n; o++)
      for (size_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
        const size_t v = (size_t)o * cv + w;
        if (v < pv) store_vec<T>(rk.out[r], p0 + v, ld16_cg(my_out + v * 16), 0, a.count, 0);
      }
  }
  end_call(rk, e);
}

// K5 direct: NVLS AllReduce in place on SYMMETRIC buffers (cfMemAlloc), the
// copy-free form of build_switch_2pa (cf/collectives.py:235-250): rank r's
// CTAs multimem.ld_reduce chunk r of the send buffer across every member and
// multimem.st the sums into every member's recv buffer -- S of NVLink traffic
// per rank per direction and no staging copies.  `emul` (boxes without
// multicast) runs the same schedule with per-member unicast loads / stores in
// the reference switch order (0 + x_0 + x_1 + ...).  A ragged last vector
// (count * sizeof(T) not a multiple of 16) is reduced through the unicast
// mappings by one thread of the last rank.  Entry handshake: every member's
// send buffer is produced; exit handshake: every member stored its chunk
// into this rank's recv buffer.  A single co-resident launch (emulated) needs
// neither.
template <typename T>
__global__ void __launch_bounds__(512) nvls_direct_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  constexpr int V = 16 / sizeof(T);
  const int n = a.n, r = rk.rank;
  const uint64_t e = begin_call_lazy(rk, a.single_launch);
  if (!a.single_launch) handshake(rk, n, e * kPhases + 1, false, a.gpu_scope);
  const size_t full = a.count / V;
  const size_t cv = (full + n - 1) / n;
  const size_t v0 = min((size_t)r * cv, full), v1 = min(v0 + cv, full);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  if (!a.emul) {
    // kNvlsU switch reductions in flight per thread: one multimem.ld_reduce
    // is a round trip through the switch, so a thread issuing one at a time
    // would move 16 bytes per round trip
    size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (kNvlsU - 1) * stride < v1; v += kNvlsU * stride) {
      uint4 x[kNvlsU];
#pragma unroll
      for (int u = 0; u < kNvlsU; u++) x[u] = multimem_ld_reduce<T>(rk.mc_in + (v + u * stride) * 16);
#pragma unroll
      for (int u = 0; u < kNvlsU; u++) multimem_st16(rk.mc_out + (v + u * stride) * 16, x[u]);
    }
    for (; v < v1; v += stride) multimem_st16(rk.mc_out + v * 16, multimem_ld_reduce<T>(rk.mc_in + v * 16));
  } else {
    for (size_t v = v0 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; v < v1; v += stride) {
      const uint4 s = switch_sum_unicast<T>((char* const*)rk.in, n, v * 16);
#pragma unroll
      for (int q = 0; q < CF_MAX_RANKS; q++)
        if (q < n) st16(rk.out[q] + v * 16, s);
    }
  }
  if (full * V < a.count && r == n - 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    const int nb = (int)((a.count - full * V) * sizeof(T));
    uint4 x[CF_MAX_RANKS];
#pragma unroll
    for (int q = 0; q < CF_MAX_RANKS; q++)
      if (q < n) x[q] = ld_partial16_ool<sizeof(T)>(rk.in[q] + full * 16, nb);
    const uint4 s = reduce_vecs<T, CF_MAX_RANKS>(x, n, true);
    for (int q = 0; q < n; q++) st_masked16_ool<sizeof(T)>(rk.out[q] + full * 16, s, 0, nb / (int)sizeof(T));
  }
  if (!a.single_launch) handshake(rk, n, e * kPhases + 2, true, a.gpu_scope);
  end_call(rk, e);
}

// ---------------------------------------------------------------- K9 / K12 / K7 ring

// CTA b's contiguous share of element range [lo, hi) (multiple of V elements).
__device__ __forceinline__ void cta_slice(size_t lo, size_t hi, int b, int B, size_t V, size_t& s0,
                                          size_t& s1) {
  const size_t len = hi > lo ? hi - lo : 0;
  const size_t per = ((len + B - 1) / B + V - 1) / V * V;
  s0 = min(lo + (size_t)b * per, hi);
  s1 = min(s0 + per, hi);
}

// Point-to-point stream of fixed-size units from rank r's CTA b to the next
// rank's CTA b: kRingSlots slots in the receiver's ring region, data signals
// on the receiver's semaphore slab, credits (acks) on the sender's ack slab.
// Values are epoch * kPhases + sequence; the value epoch * kPhases itself is
// the receiver's "entered this call" ready mark, so slots are never
// overwritten while the previous call still reads them.
// Thread 0's fence before a ring link's data release: across GPUs the full
// system fence; at .gpu scope the per-thread fences below already ordered the
// slot stores.
__device__ __forceinline__ void ring_publish(bool gpu) {
  if (!gpu) __threadfence_system();
}
// Every thread fences its own slot stores before the barrier that precedes
// thread 0's release (not relying on bar.sync making one thread's fence
// cumulative over the other warps' in-flight stores; costs ~5% of ring RS).
#ifndef CF_RING_THREAD_FENCE
#define CF_RING_THREAD_FENCE 1
#endif
// Discard consumed ring slots from L2 (no write-back).  Measured (256 MiB
// ring RS, 8 co-resident ranks, ncu): DRAM writes 1.25 -> 0.32 GB (1.19x the
// output) but 1.53 -> 1.72 ms -- the discards sit on the credit's critical
// path of a latency-bound chain -- so it is off by default.
#ifndef CF_RING_DISCARD
#define CF_RING_DISCARD 0
#endif
// Evict-first L2 policy on the streamed inputs, so they do not push the ring
// slots out of L2 (256 MiB ring RS: DRAM writes 1.85 -> 1.25 GB, 1.56 ->
// 1.53 ms).
#ifndef CF_RING_EVICT_FIRST
#define CF_RING_EVICT_FIRST 1
#endif

struct RingLink {
  char* my_slots;         // slots I receive into (from prev)
  char* nx_slots;         // slots I send into (next's)
  const uint64_t* data_in;
  uint64_t* data_out;
  const uint64_t* ack_in;
  uint64_t* ack_out;
  uint64_t base;
  uint64_t qs, qr;
  RankState* st;
  bool gpu;

  __device__ char* recv_slot() const { return my_slots + (qr % kRingSlots) * kRingSlot; }
  __device__ char* send_slot() const { return nx_slots + (qs % kRingSlots) * kRingSlot; }
  __device__ void recv_wait() {
    if (threadIdx.x == 0) wait_geq(data_in, base + qr + 1, st, gpu);
    __syncthreads();
  }
  // The consumed slot's lines are discarded from L2 (no write-back: the next
  // unit overwrites them), so slot traffic stays on chip instead of being
  // evicted to HBM by the streaming inputs.  The fence orders every thread's
  // discards before the credit release (a discard is a weak write).
  __device__ void discard_recv(size_t bytes) {
#if CF_RING_DISCARD
    char* sl = recv_slot();
    for (size_t o = (size_t)threadIdx.x * 128; o < bytes; o += (size_t)blockDim.x * 128)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(sl + o) : "memory");
#else
    (void)bytes;
#endif
  }
  __device__ void recv_done(size_t bytes) {
    discard_recv(bytes);
    if (CF_RING_DISCARD) fence_publish(gpu);
    __syncthreads();
    if (threadIdx.x == 0) st_release(ack_out, base + qr + 1, gpu);
    qr++;
  }
  __device__ void credit_wait() {
#if CF_DROP_FENCE != 6
    wait_geq(ack_in, base + (qs >= kRingSlots ? qs - kRingSlots + 1 : 0), st, gpu);
#endif
  }
  __device__ void publish_data() {
    CF_STRESS_AT(20);
#if CF_DROP_FENCE == 3
    st_relaxed(data_out, base + qs + 1, gpu);
#else
    ring_publish(gpu);
    st_release(data_out, base + qs + 1, gpu);
#endif
  }
  __device__ void send_wait() {
    if (threadIdx.x == 0) credit_wait();
    __syncthreads();
  }
  __device__ void send_done() {
    if (CF_RING_THREAD_FENCE && CF_DROP_FENCE != 3) fence_publish(gpu);
    __syncthreads();
    if (threadIdx.x == 0) publish_data();
    qs++;
  }
  // One barrier for both waits of a step: thread 0 polls the incoming data,
  // thread 32 (another warp) the send credit, concurrently.
  __device__ void wait_both(bool rcv, bool snd) {
    if (rcv && threadIdx.x == 0) wait_geq(data_in, base + qr + 1, st, gpu);
    if (snd && threadIdx.x == 32) credit_wait();
    __syncthreads();
  }
  // One barrier for both completions of a step: free the received slot, then
  // publish the sent one.
  __device__ void done_both(bool rcv, bool snd, size_t rbytes) {
    if (rcv) discard_recv(rbytes);
    if ((CF_RING_THREAD_FENCE && CF_DROP_FENCE != 3 && snd) || (CF_RING_DISCARD && rcv)) fence_publish(gpu);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (rcv) {
        CF_STRESS_AT(21);
        st_release(ack_out, base + qr + 1, gpu);
      }
      if (snd) publish_data();
    }
    if (rcv) qr++;
    if (snd) qs++;
  }
};

__device__ __forceinline__ RingLink make_link(const CollArgs& a, const RankCtx& rk, uint64_t e) {
  const int n = a.n, r = rk.rank, b = blockIdx.x;
  const int prev = (r + n - 1) % n, next = (r + 1) % n;
  RingLink L;
  L.my_slots = rk.ring[r] + (size_t)b * kRingSlots * kRingSlot;
  L.nx_slots = rk.ring[next] + (size_t)b * kRingSlots * kRingSlot;
  L.data_in = rk.sem[r] + sem_index(prev, b);
  L.data_out = rk.sem[next] + sem_index(r, b);
  L.ack_in = rk.ack[r] + sem_index(next, b);
  L.ack_out = rk.ack[prev] + sem_index(r, b);
  L.base = e * kPhases;
  L.qs = L.qr = 0;
  L.st = rk.st;
  L.gpu = a.gpu_scope;
  // ready mark: my slots are free for this call (I finished the previous one)
  if (threadIdx.x == 0) st_release(L.ack_out, L.base, L.gpu);
  return L;
}

// V accumulator values (f32 / i32) <-> NQ 16-byte words of a ring slot.
template <typename T>
struct AccVec {
  using A = typename Vec<T>::Acc;
  static constexpr int V = Vec<T>::N;
  static constexpr int NQ = V * (int)sizeof(A) / 16;
  __device__ static void load(const void* p, A* a) {
#pragma unroll
    for (int q = 0; q < NQ; q++) {
      const uint4 w = ld16(reinterpret_cast<const char*>(p) + q * 16);
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; k++) a[q * 4 + k] = bits_to<A>(u[k]);
    }
  }
  __device__ static void store(void* p, const A* a) {
#pragma unroll
    for (int q = 0; q < NQ; q++)
      st16(reinterpret_cast<char*>(p) + q * 16,
           make_uint4(to_bits(a[q * 4]), to_bits(a[q * 4 + 1]), to_bits(a[q * 4 + 2]), to_bits(a[q * 4 + 3])));
  }
  template <typename X> __device__ static X bits_to(uint32_t u);
  __device__ static uint32_t to_bits(float x) { return __float_as_uint(x); }
  __device__ static uint32_t to_bits(int32_t x) { return (uint32_t)x; }
};
template <typename T> template <typename X>
__device__ X AccVec<T>::bits_to(uint32_t u) {
  if constexpr (sizeof(X) == 4 && X(0.5f) != X(0)) return __uint_as_float(u);
  else return (X)u;
}

// Passes (16-byte vectors of T per thread) of a ring unit's own contribution
// prefetched into registers before a step's waits.
#ifndef CF_RING_PRE
#define CF_RING_PRE 4
#endif
constexpr int kRingPre = CF_RING_PRE;

// Ring ReduceScatter (build_ring_rs, cf/collectives.py:30-79) and, with
// `push`, the two-phase ring AllReduce (build_2pr, :107-136).  Step s sends
// the partial of chunk (r - s) mod n to the next rank; the partial that
// arrives is added to the own contribution (partials travel in the
// accumulator type, f32 for f16/bf16, so rounding happens once), and after n
// steps chunk r holds 0 + x_r + x_{r+1} + ... + x_{r-1}: the reference's
// ring order.  The AllGather phase then forwards the finished chunks.
// 256-thread ring CTAs, 3 resident per SM (<= 85 registers): 55 independent
// links per rank at 8 co-resident ranks (256 MiB ring RS: 2/SM 1.69 ms,
// 3/SM 1.48 ms, 4/SM 1.52 ms).
#ifndef CF_RING_MINB
#define CF_RING_MINB 3
#endif
template <typename T>
__global__ void __launch_bounds__(256, CF_RING_MINB) ring_kernel(const __grid_constant__ CollArgs a) {
  using A = typename Vec<T>::Acc;
  const RankCtx& rk = a.rk[blockIdx.y];
  const int n = a.n, r = rk.rank, b = blockIdx.x, B = gridDim.x;
  constexpr size_t V = 16 / sizeof(T);
  const uint64_t e = begin_call(rk);
  RingLink L = make_link(a, rk, e);
  const T* x = reinterpret_cast<const T*>(rk.in[r]);
  T* y = reinterpret_cast<T*>(rk.out[r]);
  constexpr size_t UA = kRingSlot / sizeof(A);   // elements per unit, RS phase
  auto chunk = [&](int c, size_t& s0, size_t& s1) {
    const size_t lo = min((size_t)c * a.cs, a.count), hi = min(lo + a.cs, a.count);
    cta_slice(lo, hi, b, B, V, s0, s1);
  };
  // Unit-major schedule (unit k walks through every step before unit k+1):
  // each send after the first step is preceded by the receive that feeds it,
  // so with kRingSlots credits the ring never stalls on a full slot ring.
  // Sender and receiver skip the same (chunk, unit) pairs, so the per-link
  // sequence numbers stay aligned.
  size_t ka = 0;
  for (int c = 0; c < n; c++) {
    size_t s0, s1;
    chunk(c, s0, s1);
    ka = max(ka, (s1 - s0 + UA - 1) / UA);
  }
  const size_t shift = a.rs_shift ? min((size_t)r * a.cs, a.count) : 0;
  // every chunk starts on the 16-byte grid: whole-vector loops (chunk ends,
  // CTA slices and units are then multiples of V as well)
  const bool vec = a.cs % V == 0 && a.count % V == 0 && (((uintptr_t)x | (uintptr_t)y) & 15) == 0;
  // inputs are read once: evict-first, so the slots stay L2-resident
  const uint64_t pol = l2_policy_evict_first();
  auto ldx = [&](const T* p) { return CF_RING_EVICT_FIRST ? ld16_hint(p, pol) : ld16(p); };
  TS_DECL
  TS_MARK();
  for (size_t k = 0; k < ka; k++) {
    // ReduceScatter: step s adds the own contribution to chunk (r - s)
    for (int s = 0; s < n; s++) {
      size_t s0, s1;
      chunk((r - s + n) % n, s0, s1);
      const size_t u0 = s0 + k * UA;
      if (u0 >= s1) continue;
      const size_t u1 = min(u0 + UA, s1);
      if (vec) {
        // whole 16-byte vectors of T; the first kRingPre passes of the own
        // contribution are prefetched into registers before the waits (their
        // HBM latency overlaps the flag round trip), later passes load after;
        // the slots carry V accumulators per vector
        const size_t pass = (size_t)blockDim.x * V;
        uint4 xv[kRingPre];
#pragma unroll
        for (int m = 0; m < kRingPre; m++) {
          const size_t i = u0 + m * pass + threadIdx.x * V;
          if (i < u1) xv[m] = ldx(x + i);
        }
        L.wait_both(s > 0, true);
        const A* in_slot = reinterpret_cast<const A*>(L.recv_slot());
        A* out_slot = reinterpret_cast<A*>(L.send_slot());
        auto step = [&](size_t i, uint4 xi) {
          A v[V];
          Vec<T>::load(xi, v);
          if (s > 0) {
            A p[V];
            AccVec<T>::load(in_slot + (i - u0), p);
#pragma unroll
            for (int j = 0; j < (int)V; j++) v[j] = acc_add(p[j], v[j]);
          }
          AccVec<T>::store(out_slot + (i - u0), v);
        };
#pragma unroll
        for (int m = 0; m < kRingPre; m++) {
          const size_t i = u0 + m * pass + threadIdx.x * V;
          if (i < u1) step(i, xv[m]);
        }
        for (size_t i = u0 + kRingPre * pass + threadIdx.x * V; i < u1; i += pass) step(i, ldx(x + i));
        L.done_both(s > 0, true, (u1 - u0) * sizeof(A));
        continue;
      }
      if (s > 0) L.recv_wait();
      L.send_wait();
      const A* in_slot = reinterpret_cast<const A*>(L.recv_slot());
      A* out_slot = reinterpret_cast<A*>(L.send_slot());
      if (vec) {   // whole 16-byte vectors of T; the slots carry V accumulators per vector
        for (size_t i = u0 + threadIdx.x * V; i < u1; i += (size_t)blockDim.x * V) {
          A v[V];
          Vec<T>::load(ld16(x + i), v);
          if (s > 0) {
            A p[V];
            AccVec<T>::load(in_slot + (i - u0), p);
#pragma unroll
            for (int j = 0; j < (int)V; j++) v[j] = acc_add(p[j], v[j]);
          }
          AccVec<T>::store(out_slot + (i - u0), v);
        }
      } else {
        for (size_t i = u0 + threadIdx.x; i < u1; i += blockDim.x) {
          A v = to_acc<T>(x[i]);
          if (s > 0) v = acc_add(in_slot[i - u0], v);
          out_slot[i - u0] = v;
        }
      }
      if (s > 0) L.recv_done((u1 - u0) * sizeof(A));
      L.send_done();
    }
    // own chunk r completed the circle: materialize 0 + P (cf/collectives.py:74-79)
    size_t s0, s1;
    chunk(r, s0, s1);
    const size_t u0 = s0 + k * UA;
    if (u0 < s1) {
      const size_t u1 = min(u0 + UA, s1);
      L.recv_wait();
      const A* in_slot = reinterpret_cast<const A*>(L.recv_slot());
      if (vec) {
        for (size_t i = u0 + threadIdx.x * V; i < u1; i += (size_t)blockDim.x * V) {
          A p[V];
          AccVec<T>::load(in_slot + (i - u0), p);
#pragma unroll
          for (int j = 0; j < (int)V; j++) p[j] = acc_add(A(0), p[j]);
          st16(y + (i - shift), Vec<T>::store(p));
        }
      } else {
        for (size_t i = u0 + threadIdx.x; i < u1; i += blockDim.x)
          y[i - shift] = from_acc<T>(acc_add(A(0), in_slot[i - u0]));
      }
      L.recv_done((u1 - u0) * sizeof(A));
    }
  }
  if (a.push) {
    // AllGather (build_ring_ag's forwarding, cf/collectives.py:82-104): step t
    // stores this CTA's slice of chunk (r - t) straight into the next rank's
    // output and signals; chunk (r - 1 - t) lands in mine from the previous
    // rank.  Each output range is written once per call, so no slots or
    // credits -- but the next rank must have consumed every ReduceScatter
    // unit I sent it: then it no longer reads its input, which its output may
    // alias (in place), and it entered this call.
    const int next = (r + 1) % n;
    T* yn = reinterpret_cast<T*>(rk.out[next]);
    if (threadIdx.x == 0) wait_geq(L.ack_in, L.base + L.qs, rk.st, L.gpu);
    for (int t = 0; t < n - 1; t++) {
      size_t s0, s1;
      chunk((r - t + n) % n, s0, s1);
      __syncthreads();
      if (vec) {   // 4 vectors in flight per thread
        const size_t step = (size_t)blockDim.x * V;
        size_t i = s0 + threadIdx.x * V;
        for (; i + 3 * step < s1; i += 4 * step) {
          const uint4 w0 = ld16(y + i), w1 = ld16(y + i + step), w2 = ld16(y + i + 2 * step),
                      w3 = ld16(y + i + 3 * step);
          st16(yn + i, w0);
          st16(yn + i + step, w1);
          st16(yn + i + 2 * step, w2);
          st16(yn + i + 3 * step, w3);
        }
        for (; i < s1; i += step) st16(yn + i, ld16(y + i));
      } else {
        for (size_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) yn[i] = y[i];
      }
      L.send_done();
      L.recv_wait();   // chunk (r - 1 - t) landed in my output
      L.qr++;
    }
  }
  TS_MARK();
  TS_DUMP("ring", rk.rank);
  end_call(rk, e);
}

// Ring AllGather (build_ring_ag, cf/collectives.py:82-104): each rank copies
// its shard into its own output slot, then n-1 times forwards the shard it
// holds most recently straight into the next rank's output and signals.
template <typename T>
__global__ void __launch_bounds__(512) ring_gather_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  const int n = a.n, r = rk.rank, b = blockIdx.x, B = gridDim.x;
  const int next = (r + 1) % n;
  constexpr size_t V = 16 / sizeof(T);
  const uint64_t e = begin_call(rk);
  RingLink L = make_link(a, rk, e);
  // the next rank's output is free once it entered this call
  if (threadIdx.x == 0) wait_geq(L.ack_in, L.base, rk.st, L.gpu);
  __syncthreads();
  const T* x = reinterpret_cast<const T*>(rk.in[r]);
  T* y = reinterpret_cast<T*>(rk.out[r]);
  T* yn = reinterpret_cast<T*>(rk.out[next]);
  const size_t cnt = a.count;
  size_t s0, s1;
  cta_slice(0, cnt, b, B, V, s0, s1);
  const bool vec = cnt % V == 0 && (((uintptr_t)x | (uintptr_t)y | (uintptr_t)yn) & 15) == 0;
  auto copy = [&](T* d, const T* src) {   // this CTA's slice [s0, s1)
    if (vec) {
      for (size_t i = s0 + threadIdx.x * V; i < s1; i += (size_t)blockDim.x * V) st16(d + i, ld16(src + i));
    } else {
      for (size_t i = s0 + threadIdx.x; i < s1; i += blockDim.x) d[i] = src[i];
    }
  };
  copy(y + (size_t)r * cnt, x);
  for (int t = 0; t < n - 1; t++) {
    const size_t off = (size_t)((r - t + n) % n) * cnt;
    __syncthreads();
    copy(yn + off, y + off);
    L.send_done();
    L.recv_wait();   // shard (r - 1 - t) landed in my output
    L.qr++;
  }
  end_call(rk, e);
}

// ---------------------------------------------------------------- launchers

// ---------------------------------------------------------------- K13

// AllReduce + residual add + RMSNorm (the epilogue of the C5
// consumer fused into the collective; the reference composes it from a
// `collective("allreduce")` and host-side arithmetic).  Per row of `hidden`
// elements, with h = x_0 + x_1 + ... + x_{n-1} (f32 accumulate, rounded to T
// once -- the same bits on every rank):
//   resid_out = T(h + resid[r])                       (written to out2)
//   norm_out  = T(resid_out * rsqrt(mean(resid_out^2) + eps) * weight[r])   (out)
// One CTA per row (G CTAs per rank, row R on CTA R mod G).  One-shot: every
// rank reduces every row itself.  Two-shot (`push`): rank r owns rows
// [r*per, (r+1)*per); phase 1 reduces the owned rows -- spread over all G
// CTAs of the rank by vector -- and stores h into every rank's norm_out (rows
// are disjoint per owner, so this is safe in place); after a barrier over
// every CTA of every rank, every rank finishes ALL rows with its OWN residual
// and weight (phase 2 touches only local buffers), so per-rank residuals /
// weights are honoured.  No exit handshake is needed: after the barrier no
// peer reads or writes this rank's buffers.  The first
// kCache vectors of a thread's share of the row stay in registers between
// the two passes; the rest are re-read from this rank's own resid_out
// (written by the same thread).
template <typename T, int NR>
__global__ void __launch_bounds__(512) ar_rmsnorm_kernel(const __grid_constant__ CollArgs a) {
  const RankCtx& rk = a.rk[blockIdx.y];
  TS_DECL
  TS_MARK();
  using A = typename Vec<T>::Acc;
  constexpr int V = Vec<T>::N;
  constexpr int kCache = (NR >= 8 || sizeof(T) >= 4) ? 2 : 4;   // vectors of a thread's share held in registers between the passes
  const int n = a.n, r = rk.rank;
  const bool push = a.push;
  // Single launch: the epoch is needed by thread 0 at the end and, two-shot,
  // by every thread that arrives or waits on the owners' CTAs (t < max(n, G)):
  // each thread loads it itself (before its CTA's arrival is counted in
  // end_call), nobody waits for a block barrier.
  uint64_t e;
  if (!a.single_launch) e = begin_call(rk);
  else if (push) e = *(volatile uint64_t*)&rk.st->epoch + 1;
  else e = begin_call_lazy(rk, true);
  if (!a.single_launch) handshake(rk, n, e * kPhases + 1, false, a.gpu_scope);
  const size_t nv = a.hidden / V;
  const size_t T0 = threadIdx.x, NT = blockDim.x;
  const size_t per = push ? (a.rows + n - 1) / n : a.rows;
  __shared__ float s_red[32];
  if (push) {
    // phase 1: the owned rows as one contiguous range of vectors spread over
    // every CTA of the rank, h pushed into every rank's norm_out; two vectors
    // per thread per round (both vectors' n loads in flight together).
    const size_t G = gridDim.x, stride = G * NT;
    const size_t r0 = min((size_t)r * per, a.rows), r1 = min(r0 + per, a.rows);
    const size_t v1 = r1 * nv;
    CF_STRESS_AT(11);   // late pushes: phase 2 must wait for the owners' arrivals
    for (size_t v = r0 * nv + blockIdx.x * NT + T0; v < v1; v += 2 * stride) {
      const bool two = v + stride < v1;
      uint4 x0[NR], x1[NR];
#pragma unroll
      for (int k = 0; k < NR; k++)
        if (k < n) {
          x0[k] = ld16(rk.in[k] + v * 16);
          if (two) x1[k] = ld16(rk.in[k] + (v + stride) * 16);
        }
      const uint4 h0 = reduce_vecs<T, NR>(x0, n, false);
#pragma unroll
      for (int p = 0; p < NR; p++)
        if (p < n) st16(rk.out[p] + v * 16, h0);
      if (two) {
        const uint4 h1 = reduce_vecs<T, NR>(x1, n, false);
#pragma unroll
        for (int p = 0; p < NR; p++)
          if (p < n) st16(rk.out[p] + (v + stride) * 16, h1);
      }
    }
    TS_MARK();
    // every CTA of every rank pushed: any row may now be finished anywhere
    // (measured: waiting per row for the CTAs of the row's owner only is
    // slower, C5 b=256 39.5 vs 36.9 us -- one wait per owner change stalls the
    // software pipeline of phase 2)
    cta_arrive(rk, n, e * kPhases + 2, a.gpu_scope);
#if CF_DROP_FENCE != 7
    all_wait(rk, n, e * kPhases + 2, a.gpu_scope);
#endif
    TS_MARK();
  }
  // finish a row on this rank: h (reduced here, or pushed by its owner) +
  // own residual, sum of squares, then the normalised row with own weight.
  // The first kCache vectors of the thread's share: every load (h or the n
  // sources, residual, weight) is issued before the first store, and ro stays
  // in registers for the second pass; the rest re-read resid_out.
  auto h_of = [&](size_t b) -> uint4 {
    if (push) return ld16(rk.out[r] + b);
    uint4 x[NR];
#pragma unroll
    for (int k = 0; k < NR; k++)
      if (k < n) x[k] = ld16(rk.in[k] + b);
    return reduce_vecs<T, NR>(x, n, false);
  };
  auto resid_add = [&](uint4 hv4, uint4 rv4, float& ss) -> uint4 {
    A hv[V], rv[V];
    Vec<T>::load(hv4, hv);
    Vec<T>::load(rv4, rv);
#pragma unroll
    for (int j = 0; j < V; j++) hv[j] = hv[j] + rv[j];
    const uint4 ro = Vec<T>::store(hv);
    A q[V];
    Vec<T>::load(ro, q);
#pragma unroll
    for (int j = 0; j < V; j++) ss = fmaf(q[j], q[j], ss);
    return ro;
  };
  auto normed = [&](uint4 ro, uint4 w4, float inv) -> uint4 {
    A q[V], w[V];
    Vec<T>::load(ro, q);
    Vec<T>::load(w4, w);
#pragma unroll
    for (int j = 0; j < V; j++) q[j] = q[j] * inv * w[j];
    return Vec<T>::store(q);
  };
  auto finish_row = [&](size_t row) {
    const size_t off = row * a.hidden * sizeof(T);
    float ss = 0.f;
    uint4 hc[kCache], rc[kCache], wc[kCache];
#pragma unroll
    for (int i = 0; i < kCache; i++)
      if (T0 + i * NT < nv) {
        const size_t v = T0 + i * NT;
        if (push) hc[i] = ld16(rk.out[r] + off + v * 16);
        rc[i] = ld16(rk.resid + off + v * 16);
        wc[i] = ld16(rk.weight + v * 16);
      }
#pragma unroll
    for (int i = 0; i < kCache; i++)
      if (T0 + i * NT < nv) {
        // one-shot: the n sources of one vector in flight at a time (all
        // kCache x n would not fit the registers)
        if (!push) hc[i] = h_of(off + (T0 + i * NT) * 16);
        hc[i] = resid_add(hc[i], rc[i], ss);   // hc[i] now holds ro
        st16(rk.out2[r] + off + (T0 + i * NT) * 16, hc[i]);
      }
    for (size_t v = T0 + kCache * NT; v < nv; v += NT) {
      const uint4 ro = resid_add(h_of(off + v * 16), ld16(rk.resid + off + v * 16), ss);
      st16(rk.out2[r] + off + v * 16, ro);
    }
    // block sum of squares
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((T0 & 31) == 0) s_red[T0 >> 5] = ss;
    __syncthreads();
    if (T0 < 32) {
      float t = T0 < (NT + 31) / 32 ? s_red[T0] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (T0 == 0) s_red[0] = t;
    }
    __syncthreads();
    const float inv = rsqrtf(s_red[0] / (float)a.hidden + a.eps);
    __syncthreads();   // s_red is reused by the next row
#pragma unroll
    for (int i = 0; i < kCache; i++)
      if (T0 + i * NT < nv) st16(rk.out[r] + off + (T0 + i * NT) * 16, normed(hc[i], wc[i], inv));
    for (size_t v = T0 + kCache * NT; v < nv; v += NT)
      st16(rk.out[r] + off + v * 16, normed(ld16(rk.out2[r] + off + v * 16), ld16(rk.weight + v * 16), inv));
  };
  if (!push) {
    for (size_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
      finish_row(row);
      TS_MARK();
    }
  } else {
    // two-shot phase 2 touches local buffers only: software-pipelined over
    // the CTA's rows -- the next row's h and residual loads are in flight
    // while this row is reduced and stored; the weight is loaded once
    uint4 hn[kCache], rn[kCache], wc[kCache];
    auto issue = [&](size_t row) {
      const size_t off = row * a.hidden * sizeof(T);
#pragma unroll
      for (int i = 0; i < kCache; i++)
        if (T0 + i * NT < nv) {
          hn[i] = ld16(rk.out[r] + off + (T0 + i * NT) * 16);
          rn[i] = ld16(rk.resid + off + (T0 + i * NT) * 16);
        }
    };
#pragma unroll
    for (int i = 0; i < kCache; i++)
      if (T0 + i * NT < nv) wc[i] = ld16(rk.weight + (T0 + i * NT) * 16);
    if (blockIdx.x < a.rows) issue(blockIdx.x);
    for (size_t row = blockIdx.x; row < a.rows; row += gridDim.x) {
      const size_t off = row * a.hidden * sizeof(T);
      uint4 hc[kCache], rc[kCache];
#pragma unroll
      for (int i = 0; i < kCache; i++) hc[i] = hn[i], rc[i] = rn[i];
      if (row + gridDim.x < a.rows) issue(row + gridDim.x);
      float ss = 0.f;
#pragma unroll
      for (int i = 0; i < kCache; i++)
        if (T0 + i * NT < nv) {
          hc[i] = resid_add(hc[i], rc[i], ss);   // hc[i] now holds ro
          st16(rk.out2[r] + off + (T0 + i * NT) * 16, hc[i]);
        }
      for (size_t v = T0 + kCache * NT; v < nv; v += NT) {
        const uint4 ro = resid_add(ld16(rk.out[r] + off + v * 16), ld16(rk.resid + off + v * 16), ss);
        st16(rk.out2[r] + off + v * 16, ro);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if ((T0 & 31) == 0) s_red[T0 >> 5] = ss;
      __syncthreads();
      if (T0 < 32) {
        float t = T0 < (NT + 31) / 32 ? s_red[T0] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (T0 == 0) s_red[0] = t;
      }
      __syncthreads();
      const float inv = rsqrtf(s_red[0] / (float)a.hidden + a.eps);
      __syncthreads();   // s_red is reused by the next row
#pragma unroll
      for (int i = 0; i < kCache; i++)
        if (T0 + i * NT < nv) st16(rk.out[r] + off + (T0 + i * NT) * 16, normed(hc[i], wc[i], inv));
      for (size_t v = T0 + kCache * NT; v < nv; v += NT)
        st16(rk.out[r] + off + v * 16, normed(ld16(rk.out2[r] + off + v * 16), ld16(rk.weight + v * 16), inv));
      TS_MARK();
    }
  }
  if (!push && !a.single_launch) handshake(rk, n, e * kPhases + 2, true, a.gpu_scope);
  end_call(rk, e);
  TS_MARK();
  TS_DUMP("k13", rk.rank);
}

template <typename T>
static const void* pick_norm(int nr) {
  if (nr <= 2) return (const void*)ar_rmsnorm_kernel<T, 2>;
  if (nr <= 4) return (const void*)ar_rmsnorm_kernel<T, 4>;
  return (const void*)ar_rmsnorm_kernel<T, 8>;
}

template <template <typename, int> class K> struct KernelTable;

template <typename T>
static const void* pick_pull(int nr) {
  if (nr <= 2) return (const void*)pull_reduce_kernel<T, 2>;
  if (nr <= 4) return (const void*)pull_reduce_kernel<T, 4>;
  return (const void*)pull_reduce_kernel<T, 8>;
}
template <typename T>
static const void* pick_ll1(int nr) {
  if (nr <= 2) return (const void*)ll_oneshot_kernel<T, 2>;
  if (nr <= 4) return (const void*)ll_oneshot_kernel<T, 4>;
  return (const void*)ll_oneshot_kernel<T, 8>;
}
template <typename T>
static const void* pick_ll2(int nr) {
  if (nr <= 2) return (const void*)ll_twoshot_kernel<T, 2>;
  if (nr <= 4) return (const void*)ll_twoshot_kernel<T, 4>;
  return (const void*)ll_twoshot_kernel<T, 8>;
}

template <const void* (*F32)(int), const void* (*I32)(int), const void* (*F16)(int),
          const void* (*BF16)(int)>
static const void* by_dtype(int dtype, int n) {
  switch (dtype) {
    case 0: return I32(n);
    case 1: return F32(n);
    case 2: return F16(n);
    case 3: return BF16(n);
  }
  return nullptr;
}

// Kernel entry point for (kind, dtype, n).  kind: 0 pull-reduce, 1 LL one-shot,
// 2 LL two-shot, 3 push-gather, 4 NVLS multimem, 5 ring RS(+AG), 6 ring AG,
// 7 AllReduce + residual + RMSNorm, 8 NVLS in place on symmetric buffers.
const void* collective_kernel(int kind, int dtype, int n) {
  switch (kind) {
    case 0: return by_dtype<pick_pull<float>, pick_pull<int32_t>, pick_pull<__half>,
                            pick_pull<__nv_bfloat16>>(dtype, n);
    case 1: return by_dtype<pick_ll1<float>, pick_ll1<int32_t>, pick_ll1<__half>,
                            pick_ll1<__nv_bfloat16>>(dtype, n);
    case 2: return by_dtype<pick_ll2<float>, pick_ll2<int32_t>, pick_ll2<__half>,
                            pick_ll2<__nv_bfloat16>>(dtype, n);
    case 3:
      switch (dtype) {
        case 0: return (const void*)push_gather_kernel<int32_t>;
        case 1: return (const void*)push_gather_kernel<float>;
        case 2: return (const void*)push_gather_kernel<__half>;
        case 3: return (const void*)push_gather_kernel<__nv_bfloat16>;
      }
      break;
    case 4:
      switch (dtype) {
        case 0: return (const void*)nvls_kernel<int32_t>;
        case 1: return (const void*)nvls_kernel<float>;
        case 2: return (const void*)nvls_kernel<__half>;
        case 3: return (const void*)nvls_kernel<__nv_bfloat16>;
      }
      break;
    case 5:
      switch (dtype) {
        case 0: return (const void*)ring_kernel<int32_t>;
        case 1: return (const void*)ring_kernel<float>;
        case 2: return (const void*)ring_kernel<__half>;
        case 3: return (const void*)ring_kernel<__nv_bfloat16>;
      }
      break;
    case 7:   // K13 (floating point only)
      switch (dtype) {
        case 1: return pick_norm<float>(n);
        case 2: return pick_norm<__half>(n);
        case 3: return pick_norm<__nv_bfloat16>(n);
      }
      break;
    case 9:   // K6 bulk (TMA bulk copies)
      switch (dtype) {
        case 0: return (const void*)push_gather_bulk_kernel<int32_t>;
        case 1: return (const void*)push_gather_bulk_kernel<float>;
        case 2: return (const void*)push_gather_bulk_kernel<__half>;
        case 3: return (const void*)push_gather_bulk_kernel<__nv_bfloat16>;
      }
      break;
    case 8:   // K5 direct (symmetric buffers)
      switch (dtype) {
        case 0: return (const void*)nvls_direct_kernel<int32_t>;
        case 1: return (const void*)nvls_direct_kernel<float>;
        case 2: return (const void*)nvls_direct_kernel<__half>;
        case 3: return (const void*)nvls_direct_kernel<__nv_bfloat16>;
      }
      break;
    case 6:
      switch (dtype) {
        case 0: return (const void*)ring_gather_kernel<int32_t>;
        case 1: return (const void*)ring_gather_kernel<float>;
        case 2: return (const void*)ring_gather_kernel<__half>;
        case 3: return (const void*)ring_gather_kernel<__nv_bfloat16>;
      }
      break;
  }
  return nullptr;
}

}  // namespace cf
