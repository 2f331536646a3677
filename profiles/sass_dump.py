#!/usr/bin/env python3
"""cuobjdump -sass of the hot kernels into profiles/ (xz-compressed, one file per
kernel) plus an opcode-class summary. Run from the repo root after a build:

    python profiles/sass_dump.py r2
"""
import collections
import lzma
import re
import subprocess
import sys

OBJS = {"paper_1907_04587_b200/_build/nsd_k_warp.o": ["k_batch_warpIdd", "k_batch_warpIdf", "k_batch_collideId"],
        "paper_1907_04587_b200/_build/nsd_k_single.o": ["k_single_blockIdLb0", "k_single_gridIdLb1ELi2"]}
CLASSES = [("fp64 math", r"^(DFMA|DMUL|DADD|DSETP|DMNMX)"), ("fp32 math", r"^(FFMA|FMUL|FADD|FSETP|FMNMX|FSEL)"),
           ("MUFU", r"^MUFU"), ("shared ld/st", r"^(LDS|STS)"), ("global ld/st", r"^(LDG|STG)"),
           ("generic ld/st", r"^(LD|ST)\b|^(LD|ST)\."), ("local ld/st (spills, stack)", r"^(LDL|STL)"),
           ("shuffle", r"^SHFL"), ("barrier/warpsync", r"^(BAR|WARPSYNC|BSYNC|BSSY)"), ("atomics", r"^(ATOM|RED)"),
           ("TMA / tcgen05 (none: not a GEMM)", r"^(UTMA|UBLKCP|UTC|LDTM|STTM)"), ("branch", r"^(BRA|BRX|JMP|CALL|RET|EXIT)")]


def main(tag):
    out = [f"# SASS of the hot kernels (cuobjdump -sass, sm_100a), opcode classes per kernel ({tag})", ""]
    for obj, keys in OBJS.items():
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        funcs = re.split(r"\n\s*Function : ", sass)
        for f in funcs[1:]:
            name = f.split("\n", 1)[0].strip()
            key = next((k for k in keys if k in name), None)
            if not key:
                continue
            ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f)
            cnt = collections.Counter()
            for op in ops:
                base = op.split(".")[0]
                cls = next((c for c, rx in CLASSES if re.match(rx, base)), "other")
                cnt[cls] += 1
            out.append(f"{name}: {len(ops)} instructions")
            for c, _ in CLASSES + [("other", "")]:
                if cnt[c]:
                    out.append(f"  {c:34s} {cnt[c]:7d}  {100.0 * cnt[c] / len(ops):5.1f}%")
            out.append("")
            with lzma.open(f"profiles/{tag}_sass_{key}.txt.xz", "wt") as fh:
                fh.write("Function : " + f)
    open(f"profiles/{tag}_sass_summary.txt", "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2")
