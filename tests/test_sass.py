"""The committed SASS listings (profiles/sass/, north_star: "each kernel
evidenced by ... a committed SASS listing") are the SASS of the libcf.so built
from HEAD: a kernel change without a re-dump (`python scripts/dump_sass.py`)
fails here.  CPU only (cuobjdump on the cross-compiled library)."""

import os
import re
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
LIB = os.path.join(ROOT, "paper_2504_09014_b200", "libcf.so")

pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and shutil.which("cuobjdump")),
                                reason="libcf.so not built or cuobjdump missing")


def test_committed_sass_matches_fresh_build():
    import dump_sass
    fresh = dump_sass.listings(LIB)
    assert set(fresh) == {t for t, _ in dump_sass.KERNELS}, "kernel instantiation missing from libcf.so"
    for tag, (dem, body) in fresh.items():
        path = os.path.join(ROOT, "profiles", "sass", tag + ".sass")
        assert os.path.exists(path), f"{tag}: no committed listing (run scripts/dump_sass.py)"
        committed = open(path).read()
        assert committed.splitlines()[0] == f"// {dem}", tag
        got, want = dump_sass.n_instructions(body), dump_sass.n_instructions(committed)
        assert got == want, f"{tag}: fresh build has {got} SASS instructions, committed listing {want} " \
                            "(re-run scripts/dump_sass.py)"


def test_sass_index_counts_match_listings():
    import dump_sass
    index = open(os.path.join(ROOT, "profiles", "sass", "README.md")).read()
    for tag, _ in dump_sass.KERNELS:
        body = open(os.path.join(ROOT, "profiles", "sass", tag + ".sass")).read()
        row = re.search(rf"^\| `{tag}` \|.*\| (\d+) \|$", index, re.M)
        assert row and int(row.group(1)) == dump_sass.n_instructions(body), tag


def test_tma_and_multimem_instructions_present():
    """The bulk AllGather runs on the TMA bulk-copy engine (UBLKCP + mbarrier
    SYNCS); the NVLS kernels assemble multimem.ld_reduce to LDGMC."""
    d = os.path.join(ROOT, "profiles", "sass")
    bulk = open(os.path.join(d, "k6_push_gather_bulk_bf16.sass")).read()
    assert re.search(r"\bUBLKCP\.S\.G\b", bulk) and re.search(r"\bUBLKCP\.G\.S\b", bulk)
    assert re.search(r"\bSYNCS\.", bulk)
    for tag in ("k5_nvls_bf16", "k5_nvls_direct_bf16"):
        assert re.search(r"\bLDGMC\.", open(os.path.join(d, tag + ".sass")).read()), tag
