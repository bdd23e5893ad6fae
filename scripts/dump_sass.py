"""Commit the SASS of libcf's main kernel instantiations (north_star: each
kernel evidenced by a committed SASS listing) into profiles/sass/, with an
index of the instructions that matter for these kernels: 16-byte global
loads/stores, strong (volatile / release / acquire) accesses, multimem
(NVLS) ops, local-memory spills, barriers."""

import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_09014_b200", "libcf.so")
OUT = os.path.join(ROOT, "profiles", "sass")
KERNELS = [   # (file tag, substring of the demangled name)
    ("k3_pull_reduce_bf16_8", "pull_reduce_kernel<__nv_bfloat16, 8>"),
    ("k1_ll_oneshot_f32_8", "ll_oneshot_kernel<float, 8>"),
    ("k4_ll_twoshot_bf16_8", "ll_twoshot_kernel<__nv_bfloat16, 8>"),
    ("k6_push_gather_bf16", "push_gather_kernel<__nv_bfloat16>"),
    ("k5_nvls_bf16", "nvls_kernel<__nv_bfloat16>"),
    ("k9_ring_bf16", "ring_kernel<__nv_bfloat16>"),
    ("k7_ring_gather_bf16", "ring_gather_kernel<__nv_bfloat16>"),
    ("k13_ar_rmsnorm_bf16_8", "ar_rmsnorm_kernel<__nv_bfloat16, 8>"),
    ("k5_nvls_direct_bf16", "nvls_direct_kernel<__nv_bfloat16>"),
    ("k6_push_gather_bulk_bf16", "push_gather_bulk_kernel<__nv_bfloat16>"),
    ("k10_plan_hb_bf16", "plan_kernel<__nv_bfloat16, 0>"),
    ("k10_plan_ll_bf16", "plan_kernel<__nv_bfloat16, 1>"),
    ("k10_plan_all_bf16", "plan_kernel<__nv_bfloat16, 3>"),
    ("k10_plan_single_bf16", "plan_single_kernel<__nv_bfloat16>"),
    ("k10_plan_ll_compiled_bf16", "plan_ll_kernel<__nv_bfloat16>"),
]
PATTERNS = {
    "LDG.128": r"LDG\.E\.128\b(?!\.STRONG)", "STG.128": r"STG\.E\.128\b(?!\.STRONG)",
    "LDG.128.STRONG": r"LDG\.E\.128\.STRONG", "STG.128.STRONG": r"STG\.E\.128\.STRONG",
    "LDG.STRONG(any)": r"LDG\.E[^ ]*\.STRONG", "RED/ATOM": r"\b(RED|ATOMG)\.",
    "LDGMC (multimem.ld_reduce)": r"\bLDGMC\.",
    "UBLKCP (TMA bulk copy)": r"\bUBLKCP\.", "SYNCS (mbarrier)": r"\bSYNCS\.",
    "LDL/STL (local)": r"\b(LDL|STL)\b", "BAR.SYNC": r"BAR\.SYNC", "MEMBAR": r"MEMBAR",
    "FENCE/ERRBAR": r"\b(FENCE|ERRBAR|CCTL)\b",
}


def n_instructions(body: str) -> int:
    """SASS instructions in a listing (lines carrying an /*addr*/ prefix)."""
    return len(re.findall(r"^\s+/\*[0-9a-f]{4,}\*/\s+\S", body, re.M))


def listings(lib: str = LIB) -> dict:
    """{tag: (demangled name, SASS body)} of the KERNELS instantiations in `lib`."""
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)
    names = [b.split("\n", 1)[0].strip() for b in blocks[1:]]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    out = {}
    for tag, want in KERNELS:
        for d, b in zip(dem, blocks[1:]):
            if want in d:
                out[tag] = (d.strip(), "Function : " + b)
                break
    return out


def main():
    found = listings()
    os.makedirs(OUT, exist_ok=True)
    index = ["# SASS listings (sm_100a, from libcf.so; `scripts/dump_sass.py`)", "",
             "Instruction counts per kernel (static):", "",
             "| kernel | " + " | ".join(PATTERNS) + " | instructions |",
             "|---|" + "---|" * (len(PATTERNS) + 1)]
    for tag, _ in KERNELS:
        if tag not in found:
            index.append(f"| `{tag}` | (not found) |")
            continue
        dem, body = found[tag]
        with open(os.path.join(OUT, tag + ".sass"), "w") as f:
            f.write(f"// {dem}\n" + body)
        counts = [str(len(re.findall(p, body))) for p in PATTERNS.values()]
        index.append(f"| `{tag}` | " + " | ".join(counts) + f" | {n_instructions(body)} |")
    index += ["", "`multimem.st` assembles to `STG.E.128.STRONG.SYS` on the multicast address; "
              "`multimem.ld_reduce` to `LDGMC.E.<op>.<type>`.  LL packet reads/writes are the "
              "`.STRONG` 16-byte accesses; the plan interpreter's LDL/STL are the saved "
              "interpreter state around its out-of-line op bodies, not the data path."]
    with open(os.path.join(OUT, "README.md"), "w") as f:
        f.write("\n".join(index) + "\n")
    print("\n".join(index))


if __name__ == "__main__":
    sys.exit(main())
