# Per-phase / per-CTA cycle diagnostics (NSD_PHASE_TIMING) of the partitioned grid PCR
# for the default build and every tools/_var*/ variant, C2 and C4.
set -u
L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/default.so
for v in default $(ls -d tools/_var*/ 2>/dev/null); do
  [ "$v" = default ] && cp /tmp/default.so $L || cp $v/libnsdyn_b200.so $L
  for wl in c2 c4; do
    echo "== $v $wl"
    NSD_PHASE_TIMING=1 python bench.py --workload $wl --steps 10 --warmup 2 --no-cpu-baseline 2>&1 | grep -E "nsd_step|^\{" |
      python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); print("  ms/step", round(d["ms_per_step"],3))
    else: print(" ", l.strip())'
  done
done
cp /tmp/default.so $L
