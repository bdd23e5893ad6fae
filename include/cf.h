/*
 * cf.h -- C ABI of the B200-native collective library (libcf.so).
 *
 * Plain pointers, sizes and cudaStream_t handles only; no torch types.  Every
 * entry point returns a cfStatus whose code string (cfStatusCode) is the
 * reference's stable error code (commforge 0.1.0, cf/errors.py:6-93).
 *
 * Each declaration cites the reference interface it replaces.  The reference
 * is a Python package with no FFI of its own; the binding a maintainer would
 * add on the reference side (a ctypes stub) is shown in INTEGRATION.md.
 *
 * Rank model.  A communicator drives `nlocal` local ranks out of `nranks`.
 *   - cfCommInitAll: one process drives every rank (the reference's in-process
 *     SimWorld, cf/world.py:80-185).  Ranks may share a device: co-resident
 *     ranks on one GPU run in ONE launch whose CTAs are split by rank.
 *   - cfCommCreateRank + cfCommGetHandle + cfCommConnect: one process per
 *     GPU; the opaque handles are exchanged by the caller's bootstrap
 *     (torch.distributed store / gloo in the Python package).
 * Collective calls take arrays with one entry per LOCAL rank (length 1 in the
 * one-process-per-GPU mode), in local-rank order.  Calls are asynchronous and
 * stream-ordered; calls on one communicator must be issued in the same order
 * on every rank (NCCL rules).
 */
#ifndef CF_H_
#define CF_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#if defined(__GNUC__)
#define CF_API __attribute__((visibility("default")))
#else
#define CF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CF_VERSION 1
#define CF_MAX_RANKS 8        /* one 8-GPU NVSwitch domain */
#define CF_MAX_BLOCKS 1024    /* CTAs per rank per launch (semaphore slab width) */
#define CF_HANDLE_BYTES 256   /* cfCommGetHandle blob size */

/* cf/errors.py:6-93 -- one status per reference error class. */
typedef enum {
  CF_OK = 0,
  CF_E_GENERIC = 1,        /* CommforgeError        E_GENERIC        */
  CF_E_BAD_SIZE = 2,       /* BadSizeError          E_BAD_SIZE       */
  CF_E_NO_SEM = 3,         /* NoSemError            E_NO_SEM         */
  CF_E_BAD_DELTA = 4,      /* BadDeltaError         E_BAD_DELTA      */
  CF_E_OOB = 5,            /* OutOfBoundsError      E_OOB            */
  CF_E_DEADLOCK = 6,       /* DeadlockError         E_DEADLOCK  (device spin timeout) */
  CF_E_PROXY_DOWN = 7,     /* ProxyDownError        E_PROXY_DOWN     */
  CF_E_ZERO_FLAG = 8,      /* ZeroFlagError         E_ZERO_FLAG      */
  CF_E_WRONG_PROTOCOL = 9, /* WrongProtocolError    E_WRONG_PROTOCOL */
  CF_E_BAD_ALIGN = 10,     /* BadAlignError         E_BAD_ALIGN      */
  CF_E_SYNTAX = 11,        /* PlanSyntaxError       E_SYNTAX         */
  CF_E_VERSION = 12,       /* PlanVersionError      E_VERSION        */
  CF_E_REF = 13,           /* PlanRefError          E_REF            */
  CF_E_SHAPE = 14,         /* ShapeError            E_SHAPE          */
  CF_E_PROTOCOL = 15,      /* ProtocolError         E_PROTOCOL       */
  CF_E_RANK_MISMATCH = 16, /* RankMismatchError     E_RANK_MISMATCH  */
  CF_E_TOPOLOGY = 17,      /* TopologyError         E_TOPOLOGY (e.g. no multicast) */
  CF_E_NO_ALGO = 18,       /* NoAlgoError           E_NO_ALGO        */
  CF_E_BAD_TIME = 19,      /* BadTimeError          E_BAD_TIME       */
  CF_E_CONFIG = 20,        /* ConfigError           E_CONFIG         */
  CF_E_CUDA = 21,          /* (new) CUDA runtime/driver failure      */
  CF_E_INTERNAL = 22       /* (new) invariant violated inside libcf  */
} cfStatus;

/* cf/dtypes.py:7-8 (i32, f32) extended with the 2-byte types. */
typedef enum { CF_I32 = 0, CF_F32 = 1, CF_F16 = 2, CF_BF16 = 3 } cfDtype;

/*
 * Algorithms (cf/collectives.py:23-24 ALGO_NAMES, single-node subset).
 * Each GPU algorithm reproduces the reference algorithm's accumulation order,
 * so f32 results are bit-identical to the reference `collective()` output.
 */
typedef enum {
  CF_ALGO_AUTO = -1,        /* measured selector (cf/collectives.py:464-491) */
  CF_ALGO_1PA = 0,          /* one-shot LL packets        build_1pa        :139-162 */
  CF_ALGO_1PA_HB = 1,       /* one-shot HB pull (K2)      channels.py:202-225      */
  CF_ALGO_2PA = 2,          /* two-shot HB pull/push      build_2pa memory :187-197 */
  CF_ALGO_2PA_LL = 3,       /* two-shot LL packets        build_2pa ll     :216-231 */
  CF_ALGO_SWITCH_2PA = 4,   /* NVLS multimem              build_switch_2pa :235-250 */
  CF_ALGO_2PR = 5,          /* two-phase (ring order)     build_2pr        :107-136 */
  CF_ALGO_ALLPAIRS_AG = 6,  /* direct AllGather           build_allpairs_ag:253-270 */
  CF_ALGO_RING_AG = 7,      /* ring AllGather             build_ring_ag    :82-104  */
  CF_ALGO_RING_RS = 8,      /* ReduceScatter, ring order  build_ring_rs    :30-79   */
  CF_ALGO_RS_DIRECT = 9,    /* ReduceScatter, all-pairs (2PA RS phase)  :188-191  */
  CF_ALGO_COUNT = 10
} cfAlgo;

/*
 * Transport of the ring algorithms (CF_ALGO_2PR, CF_ALGO_RING_RS,
 * CF_ALGO_RING_AG).  The reference moves their data around a ring of
 * PortChannels (cf/collectives.py:30-136).  What a caller observes is the
 * padding (2n for ring_rs / 2pr, cf/collectives.py:497-504) and the
 * accumulation order (0 + x[c] + x[c+1] + ... for chunk c); on one NVSwitch
 * domain every GPU reaches every peer at full bandwidth, so by default these
 * algorithms run all-pairs -- rank r pulls chunk r from every peer and adds it
 * in ring order (K3/K8 with the ring order), AllGather stores direct (K6) --
 * with bit-identical results and no per-step ring chain.  OR this flag into
 * the algorithm to run the literal ring over point-to-point links instead
 * (K9 / K12 ring_kernel, K7 ring_gather_kernel).
 */
#define CF_ALGO_RING_LINKS 0x100

typedef struct cfComm* cfComm_t;
typedef struct cfPlan* cfPlan_t;

typedef struct {
  size_t ll_max_bytes;      /* largest per-rank message the LL algorithms accept (0 = default 4 MiB) */
  int max_blocks;           /* CTA cap per rank (0 = derived from occupancy and co-residency) */
  int threads;              /* threads per CTA (0 = 512; multiple of 32 in [64, 512]) */
  uint64_t spin_timeout_ns; /* device spin-wait timeout -> CF_E_DEADLOCK (0 = 10 s) */
  int use_multicast;        /* 1 = build NVLS multicast objects when supported; 2 = emulated switch:
                               switch_2pa runs the NVLS kernel (K5) on unicast staging with per-rank
                               loads / stores in place of multimem (in-process communicators; tests) */
  size_t nvls_bytes;        /* per-rank NVLS staging region (input and output halves each; 0 = 64 MiB) */
} cfConfig;

/* cf/errors.py: the `.code` string of each class ("E_SHAPE", ...). */
CF_API const char* cfStatusCode(cfStatus status);
/* Detail message of the last failing call on this host thread. */
CF_API const char* cfLastErrorMessage(void);
CF_API int cfVersion(void);

/* Replaces make_world(num_nodes=1, gpus_per_node=n) (cf/world.py:184-185):
 * one process, `nranks` ranks on devices devs[0..nranks) (entries may repeat). */
CF_API cfStatus cfCommInitAll(cfComm_t* comm, int nranks, const int* devs, const cfConfig* cfg);

/* One-process-per-GPU bootstrap (replaces make_world for real multi-process
 * runs).  Create, export the opaque handle, let the caller
 * all-gather the handles, then connect with all nranks handles (rank order). */
CF_API cfStatus cfCommCreateRank(cfComm_t* comm, int nranks, int rank, int cuda_dev, const cfConfig* cfg);
CF_API cfStatus cfCommGetHandle(cfComm_t comm, void* handle, size_t* bytes);
CF_API cfStatus cfCommConnect(cfComm_t comm, const void* handles, size_t bytes_per_handle);
CF_API cfStatus cfCommDestroy(cfComm_t comm);

/* Buffer registration for the one-process-per-GPU mode (the B200 counterpart
 * of binding plan buffers to world regions, cf/executor.py:97-105): export the
 * IPC handle of a device buffer (any cudaMalloc'd range, e.g. a torch tensor),
 * all-gather the handles with the bootstrap, then import them so HB
 * algorithms can read/write the peers' corresponding buffers zero-copy.
 * Collective calls on pointers inside a registered range use the peers'
 * ranges at the same offset.  No-ops for cfCommInitAll communicators. */
#define CF_BUFFER_HANDLE_BYTES 128
CF_API cfStatus cfBufferExport(cfComm_t comm, const void* ptr, size_t bytes, void* handle);
CF_API cfStatus cfBufferImport(cfComm_t comm, const void* ptr, const void* handles, size_t bytes_per_handle);
CF_API cfStatus cfBufferRelease(cfComm_t comm, const void* ptr);

/* NVLS (SwitchChannel multimem, cf/channels.py:333-409) for the one-process-
 * per-GPU mode, in phases the caller separates with bootstrap barriers:
 *   rank 0: cfNvlsCreate -> POSIX fd of the multicast object, sent to every
 *           other rank over a Unix socket (SCM_RIGHTS);
 *   others: cfNvlsImport(fd);
 *   all   : barrier, cfNvlsBind (binds and maps this rank's memory), barrier.
 * cfCommInitAll communicators over distinct devices set NVLS up internally
 * when cfConfig.use_multicast is set and every device supports multicast. */
CF_API cfStatus cfDeviceMulticastSupported(int cuda_dev, int* supported);
CF_API cfStatus cfNvlsCreate(cfComm_t comm, int* fd);
CF_API cfStatus cfNvlsImport(cfComm_t comm, int fd);
CF_API cfStatus cfNvlsBind(cfComm_t comm);
/* Emulated switch for one-process-per-GPU communicators (tests, boxes without
 * multicast): `staging` (>= 32 B, 16-byte aligned, registered with
 * cfBufferExport/cfBufferImport on every rank) is split into the input and
 * output halves; switch_2pa then runs the NVLS kernel with per-rank loads /
 * stores over the mapped peers' staging in place of multimem (the in-process
 * twin is cfConfig.use_multicast = 2).  Replaces SwitchChannel
 * (cf/channels.py:333-409) in emulation only. */
CF_API cfStatus cfNvlsEmulate(cfComm_t comm, void* staging, size_t bytes);

/* Symmetric heap and allocator (SURVEY §8(b) cfMemAlloc; the reference's
 * per-rank regions, cf/world.py:113-138, and SwitchChannel, cf/channels.py:
 * 333-409).  One cuMem allocation per rank, mapped into every rank; mode 1
 * binds the heaps to an NVLS multicast object, mode 2 emulates the switch
 * with unicast loads / stores (boxes without multicast), mode 0 is a plain
 * symmetric heap.  Buffers from cfMemAlloc sit at the same offset of every
 * rank's heap, so collectives on them need no registration and switch_2pa
 * runs IN PLACE on them (multimem.ld_reduce from send, multimem.st into recv:
 * no staging copies); AUTO picks it for symmetric buffers >= 1 MiB per rank
 * when the heap is multicast-bound.
 *   cfCommInitAll communicators: cfSymHeapCreate does everything (fd unused).
 *   cfCommCreateRank communicators, phases separated by bootstrap barriers:
 *     cfSymHeapCreate -> *fd of this rank's heap; send it to every peer
 *     (Unix socket SCM_RIGHTS); cfSymHeapMapPeer for every peer; mode 1 then
 *     cfSymHeapMulticast phase 0 (rank 0: *fd out), 1 (others: *fd in), 2 (all);
 *     phase 3 on every rank when any rank failed a phase (switch off, heap kept).
 * cfMemAlloc is collective (same sizes, same order on every rank); ptrs gets
 * one pointer per local rank.  cfMemFree takes any local rank's pointer. */
CF_API cfStatus cfSymHeapCreate(cfComm_t comm, size_t bytes, int mode, int* fd);
CF_API cfStatus cfSymHeapMapPeer(cfComm_t comm, int peer, int fd);
CF_API cfStatus cfSymHeapMulticast(cfComm_t comm, int phase, int* fd);
CF_API cfStatus cfSymHeapInfo(cfComm_t comm, int local_rank, void** bases, size_t* bytes, int* mode);
CF_API cfStatus cfMemAlloc(cfComm_t comm, size_t bytes, void** ptrs);
CF_API cfStatus cfMemFree(cfComm_t comm, const void* ptr);
/* SwitchChannel handle for local rank `local_rank`'s kernels: a
 * cf::SwitchChannelDevice (csrc/device/cf_device.cuh) with reduce /
 * broadcast / reduce_broadcast over heap offsets. */
CF_API cfStatus cfSwitchChannelCreate(cfComm_t comm, int local_rank, void* handle, size_t* handle_bytes);

/* Channels for user kernels (the Primitive API; reference
 * MemoryChannel / PortChannel, cf/channels.py:54-330).  Fills `handle` with a
 * device struct (cf::MemoryChannelDevice / cf::PortChannelDevice from
 * csrc/device/cf_device.cuh and csrc/cf_proxy.h) that kernels of both
 * endpoints take by value.  `tag` (< CF_MAX_CHANNEL_TAGS) names the channel's
 * semaphore slot for the (src, dst) pair; one-process communicators. */
#define CF_CHANNEL_HANDLE_BYTES 256
#define CF_MAX_CHANNEL_TAGS 64
CF_API cfStatus cfMemoryChannelCreate(cfComm_t comm, int src_rank, int dst_rank, int tag, void* src_buf,
                                      void* dst_buf, void* handle, size_t* handle_bytes);
CF_API cfStatus cfPortChannelCreate(cfComm_t comm, int src_rank, int dst_rank, int tag, void* src_buf,
                                    void* dst_buf, void* handle, size_t* handle_bytes);

CF_API cfStatus cfCommNumRanks(cfComm_t comm, int* nranks);
CF_API cfStatus cfCommLocalRanks(cfComm_t comm, int* nlocal, int* ranks /* nullable, nlocal entries */);
CF_API cfStatus cfCommMulticastSupported(cfComm_t comm, int* supported);

/* Device-side spin timeout word (SURVEY.md §5 failure detection): 0 if clean,
 * CF_E_DEADLOCK if any wait of any local rank timed out.  Reads the word
 * with a synchronous legacy-stream copy: it waits for work on blocking
 * streams, not for the whole device (a compute kernel on a non-blocking
 * stream beside the collectives is not waited for) -- synchronize the
 * streams the collectives ran on first. */
CF_API cfStatus cfCommLastDeviceError(cfComm_t comm, int* code);
CF_API cfStatus cfCommClearDeviceError(cfComm_t comm);

/* Collective API (cf/collectives.py:532-573 `collective`).  `send`/`recv`/
 * `streams` hold one entry per local rank.  Counts are in elements:
 *   AllReduce      count     = elements per rank (in and out)
 *   AllGather      sendcount = shard elements; recv holds nranks*sendcount
 *   ReduceScatter  recvcount = shard elements; send holds nranks*recvcount
 * In the one-process mode the buffers of every rank must be device memory
 * reachable from every rank's device (same device, or peer access).  In the
 * one-process-per-GPU mode the LL algorithms take any buffers (they touch no
 * peer user buffer); HB algorithms need buffers registered with
 * cfBufferExport/cfBufferImport (CF_E_TOPOLOGY otherwise). */
CF_API cfStatus cfAllReduce(cfComm_t comm, const void* const* send, void* const* recv, size_t count,
                     cfDtype dtype, int algo, const cudaStream_t* streams);
CF_API cfStatus cfAllGather(cfComm_t comm, const void* const* send, void* const* recv, size_t sendcount,
                     cfDtype dtype, int algo, const cudaStream_t* streams);
CF_API cfStatus cfReduceScatter(cfComm_t comm, const void* const* send, void* const* recv, size_t recvcount,
                         cfDtype dtype, int algo, const cudaStream_t* streams);

/* AllReduce of HOST buffers (the reference's calling convention: collective()
 * takes host arrays and returns host arrays, cf/collectives.py:532-573 with
 * the copies of cf/executor.py:160-175).  One-process worlds only
 * (CF_E_TOPOLOGY otherwise).  The comm keeps device staging buffers (grown on
 * demand); two-shot messages >= 32 MiB per rank run as a pipeline of windows
 * per chunk so H2D copies, the kernel and D2H copies overlap -- results are
 * bit-identical to cfAllReduce.  Pinned host memory makes the copies
 * asynchronous; completion is ordered on streams[] (synchronize them before
 * reading recv). */
CF_API cfStatus cfAllReduceHost(cfComm_t comm, const void* const* host_send, void* const* host_recv, size_t count,
                                cfDtype dtype, int algo, const cudaStream_t* streams);
/* cfAllReduceHost with caller-provided device staging buffers (count elements
 * each, send != recv) -- the form the one-process-per-GPU mode uses, with the
 * staging buffers registered through cfBufferExport/cfBufferImport. */
CF_API cfStatus cfAllReduceHostStaged(cfComm_t comm, const void* const* host_send, void* const* host_recv,
                                      const void* const* dev_send, void* const* dev_recv, size_t count,
                                      cfDtype dtype, int algo, const cudaStream_t* streams);

/* Fused AllReduce + residual add + RMSNorm (the reference
 * composes it as `collective("allreduce", ...)` (cf/collectives.py:532-573)
 * followed by host arithmetic).  Per local rank, on rows x hidden elements
 * (f32/f16/bf16; hidden * elem_size a multiple of 16 bytes):
 *   h         = send_0 + send_1 + ... + send_{n-1}  (f32 accumulate, rounded
 *               to dtype once; identical bits on every rank)
 *   resid_out = dtype(h + resid_in)
 *   norm_out  = dtype(resid_out * rsqrt(mean_row(resid_out^2) + eps) * weight)
 * weight holds `hidden` elements.  resid_out may alias resid_in.  algo:
 * CF_ALGO_1PA_HB (one-shot: every rank reduces every row; not in place),
 * CF_ALGO_2PA (two-shot: rank r owns rows [r*ceil(rows/n), ...), reduces them
 * and stores h into every rank's norm_out; every rank then finishes all rows
 * with its own resid_in and weight; in the one-process-per-GPU mode send and
 * norm_out must be registered), or CF_ALGO_AUTO (picked from rows, hidden,
 * dtype and n only; in place it needs CF_ALGO_2PA, which it takes itself in
 * one-process communicators and reports as CF_E_SHAPE one process per GPU). */
CF_API cfStatus cfAllReduceAddRMSNorm(cfComm_t comm, const void* const* send, const void* const* resid_in,
                                      void* const* resid_out, void* const* norm_out, const void* const* weight,
                                      size_t rows, size_t hidden, float eps, cfDtype dtype, int algo,
                                      const cudaStream_t* streams);

/* CTA budget per rank for `algo` (CF_ALGO_COUNT = the fused K13 kernel; -1 =
 * every algorithm without its own budget; ctas = 0 restores the default).
 * Default: no cap beyond co-residency when ranks share a GPU (the HBM-proxy
 * world needs every SM); 64 CTAs per rank when every rank has its own GPU --
 * NVLink-bound collectives saturate the link with far fewer than 148 CTAs,
 * and a grid under half the SMs stays fully resident next to a compute
 * kernel holding the other half, so the CTA-pair handshakes cannot wait on
 * a partner that is not scheduled. */
CF_API cfStatus cfCommSetCtaBudget(cfComm_t comm, int algo, int ctas);

/* Measured selection table ("measured crossover table per
 * (collective, dtype, n) from the sweep"; the Python Communicator.tune /
 * World.tune measure it on the live GPUs and install the same table on every
 * rank).  CF_ALGO_AUTO then picks algos[i] for the first i with
 * nbytes <= max_bytes[i] (the last entry also covers every larger size); LL
 * picks beyond cfConfig.ll_max_bytes fall back to CF_ALGO_2PA.  coll: 0
 * AllReduce (per-rank bytes), 1 AllGather (output bytes), 2 ReduceScatter
 * (input bytes).  nentries = 0 restores the built-in table.  The table must be
 * the same on every rank (AUTO is then rank-uniform). */
CF_API cfStatus cfCommSetSelection(cfComm_t comm, int coll, cfDtype dtype, int nentries, const size_t* max_bytes,
                                   const int* algos);
/* Smallest per-rank AllReduce that AUTO runs in place on the NVLS switch when
 * the buffers are symmetric and multicast-bound (default 1 MiB; SIZE_MAX =
 * never).  Same on every rank. */
CF_API cfStatus cfCommSetNvlsMinBytes(cfComm_t comm, size_t bytes);

/* The algorithm the measured selector picks (cf/collectives.py:473-491).
 * collective: 0 = allreduce, 1 = allgather, 2 = reducescatter; nbytes as the
 * reference counts them (AG: output bytes). */
CF_API cfStatus cfSelectAlgorithm(cfComm_t comm, int collective, size_t nbytes, cfDtype dtype, int* algo);

/* Plan executor (cf/executor.py:73-379 Runtime; wire format cf/plan.py:1-36).
 * cfPlanLoad parses canonical plan JSON (dtype i32/f32/f16/bf16, or forced by
 * dtype_override >= 0), validates it, compiles it to a device op array and
 * allocates the plan's buffers per rank.  cfPlanExecute runs every (rank, tb)
 * program on the GPU with the caller's per-local-rank input/output buffers
 * bound zero-copy as the plan's input/output buffers (sizes: the declared
 * elems).  One-process communicators run every rank's programs; one process
 * per GPU runs this rank's programs after cfPlanGetHandle / cfPlanConnect
 * (below). */
CF_API cfStatus cfPlanLoad(cfComm_t comm, const char* json, size_t len, int dtype_override, cfPlan_t* plan);
CF_API cfStatus cfPlanExecute(cfPlan_t plan, const void* const* inputs, void* const* outputs,
                              const cudaStream_t* streams);
CF_API cfStatus cfPlanInfo(cfPlan_t plan, size_t* in_elems, size_t* out_elems, int* dtype, int* n_programs,
                           int* n_device_ops);
/* Device spin-timeout word of the plan's ranks (0 or CF_E_DEADLOCK); read like
 * cfCommLastDeviceError (synchronize the plan's streams first). */
CF_API cfStatus cfPlanLastDeviceError(cfPlan_t plan, int* code);
/* After a reported timeout: return every plan heap this process owns to its
 * load-time state (error word, semaphore lanes, barriers, LL scratch), so the
 * plan runs again (the reference Runtime rebuilds its channels per execute,
 * cf/executor.py:159).  One process per GPU: every rank calls it while no
 * execution of the plan is in flight.  Synchronizes. */
CF_API cfStatus cfPlanClearDeviceError(cfPlan_t plan);
/* One process per GPU: every rank loads the same plan with cfPlanLoad, exports
 * its plan heap (semaphore lanes, barrier counters, scratch buffers) with
 * cfPlanGetHandle, all-gathers the handles through the caller's bootstrap and
 * connects with all nranks handles (rank order); then cfPlanExecute runs this
 * rank's programs (inputs/outputs: one entry; plans that touch the peers'
 * input/output need those buffers registered, CF_E_TOPOLOGY otherwise). */
#define CF_PLAN_HANDLE_BYTES 128
CF_API cfStatus cfPlanGetHandle(cfPlan_t plan, void* handle, size_t* bytes);
CF_API cfStatus cfPlanConnect(cfPlan_t plan, const void* handles, size_t bytes_per_handle);
CF_API cfStatus cfPlanDestroy(cfPlan_t plan);

/* Native DSL (replaces the reference's Python builder library
 * cf/collectives.py:30-270 and pass pipeline cf/lowering.py:295-648).
 * Programs travel as the recorded-program JSON documented in csrc/cf_dsl.cpp
 * (buffers, channels, instructions in emission order).  Output goes to
 * `out` (capacity `cap`); `*out_len` receives the length, and a too-small
 * buffer returns CF_E_BAD_SIZE with `*out_len` set so the caller can retry.
 *   cfDslBuild: a library algorithm ("1pa", "2pa" + variant memory|ll|port,
 *     "switch_2pa", "allpairs_ag", "ring_ag", "ring_rs", "2pr") recorded for
 *     nranks x elems (cf/collectives.py:510-525 build_algo).
 *   cfDslLower: replicate `instances` -> dependence analysis -> sync insertion
 *     + redundant-sync elimination (CF_DSL_PASS_SYNC) -> fusion
 *     (CF_DSL_PASS_FUSE) -> LL flag assignment -> canonical plan JSON, the
 *     bytes cf/plan.py:146-162 serializes for the reference's lower(). */
#define CF_DSL_PASS_SYNC 1
#define CF_DSL_PASS_FUSE 2
CF_API cfStatus cfDslBuild(const char* algo, const char* variant, int nranks, size_t elems, const char* dtype,
                           const char* protocol, char* out, size_t cap, size_t* out_len);
CF_API cfStatus cfDslLower(const char* program, size_t len, int instances, int passes, char* out, size_t cap,
                           size_t* out_len);

#ifdef __cplusplus
}
#endif
#endif /* CF_H_ */
