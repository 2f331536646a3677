#!/usr/bin/env python3
"""Summarise an ncu --set full report of the batch kernel into profiles/:
key raw metrics (duration, DRAM bytes, L1/L2 traffic, occupancy, issue, stall
reasons) and the source-line hotspots (warp-stall samples, instructions).

    python profiles/summarize_ncu.py <report.ncu-rep> <out_prefix> [--traffic KEY TU.cu]

--traffic also records the capture's dram__bytes_read.sum + dram__bytes_write.sum as
profiles/dram_traffic.json[KEY], with the sha256 of the TU and every header it
includes: bench.py reports it as roofline.traffic only while those sources are
unchanged (a stale capture reads as null).
"""
import hashlib
import os
import re
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "sm__maximum_warps_per_active_cycle_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    lines = [f"kernel: {d.get('Kernel Name', '?')}", ""]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k]:>20s} {u.get(k, '')}")
    stalls = sorted(((k, float(v.replace(',', '') or 0)) for k, v in d.items()
                     if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")),
                    key=lambda x: -x[1])[:10]
    lines += ["", "stall reasons (warps per issue-active cycle):"]
    lines += [f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:8.3f}"
              for k, v in stalls]
    open(out + "_raw.txt", "w").write("\n".join(lines) + "\n")
    dur_ns = float(d["gpu__time_duration.sum"].replace(',', '')) * (1e6 if u.get("gpu__time_duration.sum") == "ms" else 1e3 if u.get("gpu__time_duration.sum") == "us" else 1)
    def mbytes(k):
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[u.get(k, "Mbyte")]
        return float(d[k].replace(',', '')) * scale
    traffic_mb = mbytes("dram__bytes_read.sum") + mbytes("dram__bytes_write.sum")
    # source hotspots
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    agg = collections.defaultdict(lambda: [0, 0])
    cur, hdr, last = None, None, None
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0].isdigit():
            last = (cur, int(r[0]), r[1].strip()[:100])
            if len(r) > 7 and r[4].isdigit():
                agg[last][0] += int(r[4]); agg[last][1] += int(r[7] or 0)
        elif last and len(r) > 7 and r[4].isdigit():
            agg[last][0] += int(r[4]); agg[last][1] += int(r[7] or 0)
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    hs = [f"warp-stall samples {tot}, instructions {toti}", "samples% instr%  file:line  source"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
        hs.append(f"{100 * v[0] / tot:6.1f} {100 * v[1] / toti:6.1f}  {k[0]}:{k[1]}  {k[2]}")
    open(out + "_source_hotspots.txt", "w").write("\n".join(hs) + "\n")
    if "--sass" in sys.argv:  # the 60 SASS instructions with the most warp-stall samples
        sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
        head = next((r for r in sass if r and r[0] == "Address"), None) or (sass[0] if sass else [])
        rows = [r for r in sass if r and r is not head and len(r) == len(head)]
        si = next((i for i, c in enumerate(head) if c.startswith("Warp Stall Sampling (All")), None)
        if si is not None:
            rows.sort(key=lambda r: -float((r[si] or "0").replace(",", "")) if (r[si] or "0").replace(",", "").replace(".", "").isdigit() else 0)
            with open(out + "_sass_top.txt", "w") as f:
                f.write(" | ".join(head) + "\n")
                for r in rows[:60]:
                    f.write(" | ".join(c.strip()[:90] for c in r) + "\n")
    print(json.dumps({"duration_ms": dur_ns / 1e6, "dram_traffic_bytes": traffic_mb * 1e6}))
    if "--traffic" in sys.argv:
        i = sys.argv.index("--traffic")
        record_traffic(sys.argv[i + 1], sys.argv[i + 2], int(round(traffic_mb * 1e6)), rep)


def tu_sources(tu):
    """The TU and its transitive quoted includes, in first-visit order, repo-relative."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    seen, todo = [], [os.path.relpath(os.path.abspath(tu), root)]
    while todo:
        f = todo.pop(0)
        if f in seen:
            continue
        seen.append(f)
        for inc in re.findall(r'#include "([^"]+)"', open(os.path.join(root, f)).read()):
            todo.append(os.path.join(os.path.dirname(f), inc))
    return root, seen


def record_traffic(key, tu, nbytes, rep):
    root, srcs = tu_sources(tu)
    h = hashlib.sha256()
    for f in srcs:
        h.update(open(os.path.join(root, f), "rb").read())
    path = os.path.join(root, "profiles", "dram_traffic.json")
    try:
        d = json.load(open(path))
    except Exception:
        d = {}
    d[key] = {"bytes": nbytes, "sources": srcs, "sha256": h.hexdigest(),
              "capture": os.path.basename(rep) + " (ncu --set full, cache control all: cold L2)"}
    json.dump(d, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
