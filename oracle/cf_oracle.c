/*
 * cf_oracle.c -- CPU restatement of the reference's reduction and LL-packet
 * arithmetic.  TEST INFRASTRUCTURE ONLY: imported by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * `--impl reference` legs.  The product (paper_2504_09014_b200/) never links it.
 *
 * What is restated (reference = commforge 0.1.0 under /root/reference/pkg):
 *   - numpy element-wise accumulation `acc += src` in a fixed source order
 *       MemoryChannel.reduce         channels.py:202-225
 *       switch_reduce (zero-init)    channels.py:367-389
 *       Runtime._local_reduce        executor.py:338-350
 *       Runtime._reduce_put          executor.py:362-379
 *       brute-force oracle           cli.py:22-31  (np.sum(np.stack(x), 0))
 *     i32 wraps (numpy int32), f32 is one IEEE RNE add per step.
 *   - fp16/bf16 (absent from the reference, dtypes.py:8): accumulate in f32 in
 *     the same order, round-to-nearest-even once (or after every step when
 *     `round_each` is set, which is the plan-op semantics).  Parity for these
 *     two dtypes is pinned only through the f32 order.
 *   - LL packets: payload word i + flag word at packet byte 8*i
 *       MemoryChannel.put_ll         channels.py:244-280
 *       ll_read_range                channels.py:303-330
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

enum { CFO_I32 = 0, CFO_F32 = 1, CFO_F16 = 2, CFO_BF16 = 3 };

/* ---- scalar conversions (RNE), independent of any compiler half type ---- */

static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

float cfo_bf16_to_f32(uint16_t h) { return u2f((uint32_t)h << 16); }

uint16_t cfo_f32_to_bf16(float f) {
    uint32_t u = f2u(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float cfo_f16_to_f32(uint16_t h) {
    uint32_t s = (uint32_t)(h & 0x8000u) << 16, e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
    if (e == 0) {
        if (m == 0) return u2f(s);
        /* subnormal: value = m * 2^-24 exactly representable in f32 */
        float v = (float)m * 5.9604644775390625e-08f;
        return s ? -v : v;
    }
    if (e == 31) return u2f(s | 0x7f800000u | (m << 13));
    return u2f(s | ((e + 112u) << 23) | (m << 13));
}

uint16_t cfo_f32_to_f16(float f) {
    uint32_t u = f2u(f);
    uint16_t s = (uint16_t)((u >> 16) & 0x8000u);
    uint32_t a = u & 0x7fffffffu;
    if (a > 0x7f800000u) return (uint16_t)(s | 0x7e00u | ((a >> 13) & 0x3ffu));  /* NaN */
    if (a >= 0x477ff000u) return (uint16_t)(s | 0x7c00u);  /* rounds to inf (>= 65520) */
    if (a < 0x38800000u) {                                  /* below f16 min normal */
        /* subnormal result: round a * 2^24 to integer (RNE) */
        if (a < 0x33000000u) return s;                      /* < 2^-25: rounds to 0 */
        uint32_t e = a >> 23, m = (a & 0x7fffffu) | 0x800000u;
        uint32_t shift = 126u - e;                           /* 14..24 */
        uint32_t q = m >> shift, rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1u);
        if (rem > half || (rem == half && (q & 1u))) q++;
        return (uint16_t)(s | q);
    }
    uint32_t r = a + 0xfffu + ((a >> 13) & 1u) - (112u << 23);
    return (uint16_t)(s | (r >> 13));
}

static inline float load_f(int dt, const void* p, size_t i) {
    switch (dt) {
    case CFO_F32: return ((const float*)p)[i];
    case CFO_F16: return cfo_f16_to_f32(((const uint16_t*)p)[i]);
    default: return cfo_bf16_to_f32(((const uint16_t*)p)[i]);
    }
}

static inline float round_to(int dt, float v) {
    if (dt == CFO_F16) return cfo_f16_to_f32(cfo_f32_to_f16(v));
    if (dt == CFO_BF16) return cfo_bf16_to_f32(cfo_f32_to_bf16(v));
    return v;
}

static inline void store_f(int dt, void* p, size_t i, float v) {
    switch (dt) {
    case CFO_F32: ((float*)p)[i] = v; break;
    case CFO_F16: ((uint16_t*)p)[i] = cfo_f32_to_f16(v); break;
    default: ((uint16_t*)p)[i] = cfo_f32_to_bf16(v); break;
    }
}

typedef struct {
    int dt, nord, zero_init, round_each;
    const void* const* srcs;
    const int* order;
    size_t lo, hi;
    void* out;
} reduce_job;

static void reduce_range(const reduce_job* j) {
    int dt = j->dt;
    if (dt == CFO_I32) {
        for (size_t i = j->lo; i < j->hi; i++) {
            uint32_t acc = j->zero_init ? 0u : ((const uint32_t*)j->srcs[j->order[0]])[i];
            for (int k = j->zero_init ? 0 : 1; k < j->nord; k++)
                acc += ((const uint32_t*)j->srcs[j->order[k]])[i];   /* two's-complement wrap */
            ((uint32_t*)j->out)[i] = acc;
        }
        return;
    }
    for (size_t i = j->lo; i < j->hi; i++) {
        float acc = j->zero_init ? 0.0f : load_f(dt, j->srcs[j->order[0]], i);
        for (int k = j->zero_init ? 0 : 1; k < j->nord; k++) {
            acc = acc + load_f(dt, j->srcs[j->order[k]], i);
            if (j->round_each) acc = round_to(dt, acc);
        }
        store_f(dt, j->out, i, acc);
    }
}

static void* reduce_thread(void* arg) { reduce_range((const reduce_job*)arg); return NULL; }

int cfo_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/*
 * out[i] = (zero_init ? 0 : src[order[0]][i]) (+) src[order[k]][i] ... in order.
 * `srcs` holds nsrc base pointers; `order` lists nord indices into it.
 * round_each: f16/bf16 result rounded after every add (one plan op per add).
 * nthreads <= 0 uses one thread per online core.  Returns 0, or -1 on bad args.
 */
int cfo_reduce(int dt, int nsrc, const void* const* srcs, const int* order, int nord,
               size_t count, int zero_init, int round_each, void* out, int nthreads) {
    if (dt < CFO_I32 || dt > CFO_BF16 || nord < 1) return -1;
    for (int k = 0; k < nord; k++) if (order[k] < 0 || order[k] >= nsrc) return -1;
    int nt = nthreads > 0 ? nthreads : cfo_max_threads();
    if (nt > 256) nt = 256;
    if ((size_t)nt > count / 4096 + 1) nt = (int)(count / 4096 + 1);
    reduce_job jobs[256];
    pthread_t tids[256];
    size_t per = (count + nt - 1) / nt;
    for (int t = 0; t < nt; t++) {
        reduce_job j = {dt, nord, zero_init, round_each, srcs, order, 0, 0, out};
        j.lo = (size_t)t * per < count ? (size_t)t * per : count;
        j.hi = j.lo + per < count ? j.lo + per : count;
        jobs[t] = j;
    }
    int spawned = 0;
    for (int t = 1; t < nt; t++) {
        if (pthread_create(&tids[t], NULL, reduce_thread, &jobs[t]) != 0) break;
        spawned = t;
    }
    for (int t = spawned + 1; t < nt; t++) reduce_range(&jobs[t]);   /* spawn failures run inline */
    reduce_range(&jobs[0]);
    for (int t = 1; t <= spawned; t++) pthread_join(tids[t], NULL);
    return 0;
}

/* LL encode: payload of nbytes (multiple of 4) -> nbytes/4 packets of [word|flag]. */
int cfo_ll_pack(const void* payload, size_t nbytes, uint32_t flag, void* packets) {
    if (flag == 0) return -2;               /* E_ZERO_FLAG, channels.py:254-255 */
    if (nbytes % 4) return -3;              /* E_BAD_ALIGN, channels.py:256-257 */
    const uint32_t* w = (const uint32_t*)payload;
    uint32_t* p = (uint32_t*)packets;
    for (size_t i = 0; i < nbytes / 4; i++) { p[2 * i] = w[i]; p[2 * i + 1] = flag; }
    return 0;
}

/* LL decode: returns the number of packets whose flag != `flag` (0 = all ready). */
size_t cfo_ll_unpack(const void* packets, size_t npackets, uint32_t flag, void* payload) {
    const uint32_t* p = (const uint32_t*)packets;
    uint32_t* w = (uint32_t*)payload;
    size_t bad = 0;
    for (size_t i = 0; i < npackets; i++) {
        if (p[2 * i + 1] != flag) bad++;
        w[i] = p[2 * i];
    }
    return bad;
}

/* Gather (AllGather restatement, collectives.py:82-104, 253-270): byte copy. */
void cfo_concat(int n, const void* const* shards, size_t shard_bytes, void* out) {
    for (int r = 0; r < n; r++)
        memcpy((char*)out + (size_t)r * shard_bytes, shards[r], shard_bytes);
}

