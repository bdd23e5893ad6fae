"""Summarise an ncu --csv launch list: per kernel name, count and mean/min/max
of gpu__time_duration.sum (diagnostic)."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    d = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = (r["Kernel Name"][:70], r["Grid Size"], r["Block Size"])
        d.setdefault(k, []).append(float(r["Metric Value"]))
    for (name, grid, block), v in d.items():
        print(f"{name:70s} grid={grid:>14s} block={block:>12s} n={len(v):4d} "
              f"mean={sum(v) / len(v):9.0f} min={min(v):9.0f} max={max(v):9.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
