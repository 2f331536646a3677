# A/B of the single-scene grid kernel (C2, C4) between the default build and the
# variants in tools/_var*/ (each run twice, interleaved), then the FEM/C4 GPU
# parity tests on each variant.  usage: bash tools/ab_grid.sh
set -u
L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/default.so
run() {
  for wl in ${AB_WORKLOADS:-c2 c4}; do
    python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c '
import sys,json
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); print(d["config"]["workload"], round(d["ms_per_step"],3), "ms", round(d["us_per_cr_iter_budget"],2), "us/CR")' | tr '\n' ' '
  done
}
for pass in 1 2; do
  cp /tmp/default.so $L; echo "default $(run)"
  for v in $(ls -d tools/_var*/ 2>/dev/null); do cp $v/libnsdyn_b200.so $L; echo "$v $(run)"; done
done
[ "${AB_TESTS:-1}" = 1 ] && for v in $(ls -d tools/_var*/ 2>/dev/null); do
  cp $v/libnsdyn_b200.so $L
  echo "$v tests: $(timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_world.py -m gpu -q -x 2>&1 | tail -1)"
done
cp /tmp/default.so $L
