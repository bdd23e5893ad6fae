"""Message-passing litmus on one B200 (tests/kernels/channels_test.cu
mp_litmus): stale payload words seen by a consumer CTA after the producer's
flag, with the collective kernels' ordering (fence + release / acquire) and
with relaxed accesses only (the CF_DROP_FENCE 1-3 mutations)."""
import ctypes
import os
import sys

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "tests", "kernels", "libcf_channels_test.so"))
lib.cftest_mp_litmus.restype = ctypes.c_longlong
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for consumer in (1, 74, 147):
    for ordered in (1, 0):
        print(f"consumer CTA {consumer:3d} ordered={ordered}: stale words = "
              f"{lib.cftest_mp_litmus(rounds, ordered, consumer)} over {rounds} rounds x 16384 words")
