"""Summarise ncu reports from gpurun_out/ into profiles/<tag>/ (tracked).

For every prof_*.ncu-rep: duration, DRAM bytes read/written, throughput
percentages, registers, occupancy and the top stall locations (SASS source
page); the headline kernel's per-launch DRAM traffic also goes to
profiles/headline_traffic.json, which bench.py reports as roofline.traffic.
"""

import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else "ncu"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                d[m] = f"{v[h.index(m)]} {units[h.index(m)]}".strip()
        res.append(d)
    return res


def hot(rep, top=12):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_hot.py"), rep, str(top)],
                         capture_output=True, text=True).stdout
    return out.strip().splitlines()


def to_bytes(s):
    val, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(val) * mul


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "round1"
    src = os.path.join(ROOT, "gpurun_out")
    # optional 2nd argument: output directory (on the GPU box: under gpurun_out/
    # so the summary travels back while the large .ncu-rep files are dropped)
    dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    md = [f"# ncu summaries ({tag})", "",
          "Captured with `scripts/profile.sh` (ncu --set full --clock-control none, 1 GPU, "
          "8 co-resident ranks, one launch per collective).", ""]
    for f in sorted(os.listdir(src)):
        if f.endswith(".ncu-rep"):
            rep = os.path.join(src, f)
            info = raw(rep)
            stalls = hot(rep)
            md.append(f"## {f[:-8]}")
            for d in info:
                md.append("")
                for k, v in d.items():
                    md.append(f"- `{k}`: {v}")
            md.append("")
            md.append("Top stall locations (share of warp-stall samples, SASS):")
            md.append("```")
            md.extend(stalls)
            md.append("```")
            md.append("")
            if f.startswith("prof_2pa_256m") and info:
                d = info[0]
                traffic = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
                with open(os.path.join(dst, "headline_traffic.json"), "w") as fh:
                    json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": traffic,
                               "source": f"profiles/{tag}/summary.md ({f})"}, fh, indent=1)
        elif f.startswith("launches") and f.endswith(".csv"):
            shutil.copyfile(os.path.join(src, f), os.path.join(dst, f))
    with open(os.path.join(dst, "summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
