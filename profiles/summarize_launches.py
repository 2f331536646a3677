"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`)
into per-kernel launch counts, mean and total durations, and the step kernel's share of GPU time.

usage: python profiles/summarize_launches.py launches.csv "<command that was profiled>" > profiles/rN_launches.txt
"""
import collections
import csv
import sys


def main(path, command):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    head = rows[0]
    ki, vi, ui = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    total = sum(sum(v) for v in agg.values())
    ours = {k: sum(v) for k, v in agg.items() if "nsdi::" in k or "nsd::" in k or k.startswith("void k_")}
    step = sum(ours.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400: {command}")
    print("# per-launch times are cold-cache and serialised; the shares, not the absolutes, compare with bench.py")
    print("launches  mean_us  total_us  kernel")
    for k, v in agg.items():
        print(f"{len(v):8d} {sum(v) / len(v):8.1f} {sum(v):9.1f}  {k[:70]}")
    for k, t in ours.items():
        print(f"# {k.split('(')[0][5:]}: {100 * t / step:.1f}% of the step's kernel time")
    print(f"# share of GPU time in the library's kernels: {100 * step / total:.1f}% "
          "(the rest: the 256 MiB L2-flush memsets between timed steps, outside the timed events)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
