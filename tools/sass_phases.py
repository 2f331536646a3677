#!/usr/bin/env python3
"""Attribute an ncu SASS-level capture of one kernel to source lines of a chosen
function via nvdisasm -gi line info (anchors: instructions whose innermost or
direct-caller line falls in [lo, hi] of FILE; unanchored instructions inherit
the preceding anchor, which follows code layout).

    python tools/sass_phases.py <report.ncu-rep> <cubin> <mangled-kernel> <file-substr> <lo> <hi>
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, cubin, kern, fsub, lo, hi):
    lo, hi = int(lo), int(hi)
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    start = dis.find(f".text.{kern}:")
    dis = dis[start:]
    end = dis.find("\n.L_x_", 0)
    line_of = {}
    cur = None
    for ln in dis.splitlines():
        m = re.search(r'## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:
            cands = [(m.group(1), int(m.group(2)))]
            if m.group(3):
                cands.append((m.group(3), int(m.group(4))))
            cur = next((l for f, l in cands if fsub in f and lo <= l <= hi), None)
            continue
        a = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if a:
            line_of[int(a.group(1), 16)] = cur
        if ".text." in ln and kern not in ln and line_of:
            break
    rows = list(csv.reader(io.StringIO(subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
    head = next(r for r in rows if r and r[0] == "Address")
    ia, isamp, iins = head.index("Address"), head.index("Warp Stall Sampling (All Samples)"), head.index("Instructions Executed")
    body = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(head)]
    base = int(body[0][ia], 16)
    agg = collections.defaultdict(lambda: [0, 0])
    last = None
    for r in body:
        off = int(r[ia], 16) - base
        ln = line_of.get(off)
        if ln is not None:
            last = ln
        key = ln if ln is not None else last
        agg[key][0] += int(r[isamp] or 0)
        agg[key][1] += int(r[iins] or 0)
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"samples {ts}, instructions {ti}; by {fsub} line in [{lo}, {hi}]")
    src = open(fsub).read().splitlines() if fsub.endswith((".cuh", ".cu")) else None
    for k, v in sorted(agg.items(), key=lambda kv: (kv[0] is None, kv[0] or 0)):
        if v[0] * 500 < ts and v[1] * 500 < ti:
            continue
        txt = src[k - 1].strip()[:70] if (src and k) else ""
        print(f"{k!s:>5} {100 * v[0] / ts:6.2f}% smp {100 * v[1] / ti:6.2f}% ins  {txt}")


if __name__ == "__main__":
    main(*sys.argv[1:])
