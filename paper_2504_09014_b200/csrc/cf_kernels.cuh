// cf_kernels.cuh -- launch-argument layout shared by the host runtime and the
// collective kernels.  Internal to libcf (not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include "device/cf_device.cuh"

namespace cf {

// Everything one rank's CTAs need, as addressable from that rank's device.
struct RankCtx {
  int rank;
  int pad_;
  const char* in[CF_MAX_RANKS];   // every rank's send buffer (pull kernels)
  char* out[CF_MAX_RANKS];        // every rank's recv buffer (push kernels)
  char* scr[CF_MAX_RANKS];        // every rank's LL scratch base
  uint64_t* sem[CF_MAX_RANKS];    // every rank's semaphore slab (data / handshake signals)
  uint64_t* ack[CF_MAX_RANKS];    // every rank's ack slab (ring credits, ring "ready")
  char* ring[CF_MAX_RANKS];       // every rank's ring slot region
  char* out2[CF_MAX_RANKS];       // K13: every rank's residual-out buffer (push)
  char* nv[CF_MAX_RANKS];         // K5: NVLS staging [input half | output half], unicast: own rank's
                                  // (emulated switch: every rank's)
  char* nv_mc;                    // K5: own staging's multicast mapping (null when emulated)
  const char* mc_in;              // K5 direct: multicast mapping of the (symmetric) send buffer
  char* mc_out;                   // K5 direct: multicast mapping of the (symmetric) recv buffer
  const char* resid;              // K13: this rank's residual input
  const char* weight;             // K13: this rank's RMSNorm weight [hidden]
  RankState* st;                  // this rank's state
};

// Ring slots: per receiving rank and CTA, kRingSlots slots of kRingSlot bytes.
// Two 64 KiB slots (double buffering): every ring step pays a flag round trip
// plus a release, so larger units amortize it, while the active slots of 8
// ranks x 37 links stay L2-resident (measured, 256 MiB ring RS: 4 x 32 KiB
// 2.14 ms, 2 x 64 KiB 1.57 ms, 3 x 64 KiB 1.84 ms, 2 x 128 KiB 1.94 ms).
#ifndef CF_RING_SLOTS
#define CF_RING_SLOTS 2
#endif
#ifndef CF_RING_SLOT_KB
#define CF_RING_SLOT_KB 64
#endif
constexpr int kRingCtas = 64;
constexpr int kRingSlots = CF_RING_SLOTS;
constexpr size_t kRingSlot = (size_t)CF_RING_SLOT_KB * 1024;
constexpr size_t kRingBytes = (size_t)kRingCtas * kRingSlots * kRingSlot;

// Semaphore slab of a receiving rank: slot [src_rank][cta].
__host__ __device__ inline size_t sem_index(int src, int cta) {
  return (size_t)src * CF_MAX_BLOCKS + (size_t)cta;
}

struct CollArgs {
  int n;            // ranks in the communicator
  int nlocal;       // ranks served by this launch (gridDim.y)
  int order;        // cf::Order
  int push;         // pull-reduce: store the result into every rank's recv buffer
  int whole;        // pull-reduce: each rank reduces [0,count) instead of its chunk
  int rs_shift;     // pull-reduce: recv is the shard (offset by -chunk start)
  int gpu_scope;    // every rank on this device: .gpu-scope release/acquire suffice
  int single_launch;// every rank runs in this one launch: stream order already provides the
                    // entry (inputs produced, outputs free) and exit (no peer still reading)
                    // guarantees, so the HB kernels skip their handshakes
  size_t count;     // elements per rank (AR/RS: send elements; AG: shard elements)
  size_t cs;        // reference chunk size in elements (cf/collectives.py:170-172)
  size_t slot;      // LL slot stride in bytes
  size_t half;      // LL parity-half stride in bytes
  size_t rows;      // K13: rows of `hidden` elements (count = rows * hidden)
  size_t hidden;
  float eps;        // K13: RMSNorm epsilon
  int emul;         // K5: emulated switch (per-rank loads/stores in place of multimem)
  size_t win_lo;    // pull-reduce (not whole): element window [win_lo, win_hi) inside each
  size_t win_hi;    // rank's chunk (pipelined host calls); 0 / SIZE_MAX = the whole chunk
  RankCtx rk[CF_MAX_RANKS];
};

}  // namespace cf
