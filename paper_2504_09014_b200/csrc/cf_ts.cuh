// cf_ts.cuh -- optional per-phase device timestamps for latency diagnosis.
// Build with `make EXTRA=-DCF_TS`: thread 0 of CTA 0 of each rank records
// %globaltimer at every TS_MARK and prints the offsets at TS_DUMP
// (scripts/ts_probe.py).  Without CF_TS the macros compile to nothing.
#pragma once
#include <cstdio>
#include "device/cf_device.cuh"

#ifdef CF_TS
#ifndef TS_CTA_COND
#define TS_CTA_COND (blockIdx.x == 0)
#endif
#define TS_DECL \
  uint64_t ts_[24];  \
  int tsn_ = 0;      \
  const bool ts_on_ = threadIdx.x == 0 && (TS_CTA_COND);
#define TS_MARK()                                                             \
  do {                                                                        \
    if (ts_on_ && tsn_ < 24) ts_[tsn_] = cf::globaltimer(); \
    tsn_++;                                                                   \
  } while (0)
#define TS_D_(q) (unsigned)((q) < tsn_ ? ts_[q] - ts_[0] : 0)
#define TS_DUMP(nm, rank)                                                                        \
  do {                                                                                           \
    if (ts_on_)                                                                                  \
      printf("TS %s rank %d t0 %llu : %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u %u\n", \
             nm, (int)(rank), (unsigned long long)ts_[0], TS_D_(1), TS_D_(2), TS_D_(3), TS_D_(4),       \
             TS_D_(5), TS_D_(6), TS_D_(7), TS_D_(8), TS_D_(9), TS_D_(10), TS_D_(11), TS_D_(12),         \
             TS_D_(13), TS_D_(14), TS_D_(15), TS_D_(16), TS_D_(17), TS_D_(18), TS_D_(19), TS_D_(20));   \
  } while (0)
#else
#define TS_DECL
#define TS_MARK()
#define TS_DUMP(nm, rank)
#endif
