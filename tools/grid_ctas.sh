# Grid size sweep of the single-scene cooperative kernel (C2, C4): CTAs per launch
# (NSD_GRID_CTAS; default one per SM) vs ms/step, fp64 and the fp32 mode.
# usage: bash tools/grid_ctas.sh [ctas...]
set -u
for n in ${@:-148 120 96 74}; do
  for prec in fp64 fp32; do
    for wl in c2 c4; do
      NSD_GRID_CTAS=$n python bench.py --workload $wl --precision $prec --steps 10 --warmup 2 --no-cpu-baseline 2>/dev/null |
        python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); print(sys.argv[1], d["config"]["workload"], d["dtype"], round(d["ms_per_step"],3), "ms", round(d["us_per_cr_iter_budget"],2), "us/CR")' $n
    done
  done
done
