# The GPU parity suites and a short C5/C2 bench on the checked build (make -C
# paper_1907_04587_b200 checks: NSD_CHECK bounds/invariant traps in the kernels and
# host code) — the stand-in for compute-sanitizer, which is closed on the GPU pool.
# usage: bash tools/run_checked.sh   (restores the product library afterwards)
set -u
L=paper_1907_04587_b200/_build/libnsdyn_b200.so
cp $L /tmp/product.so
cp paper_1907_04587_b200/_build_checks/libnsdyn_b200.so $L
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decisions.py tests/test_gpu_batch.py \
  tests/test_world.py tests/test_gpu_spec.py -m gpu -q 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-alt --no-scenes --no-cpu-baseline 2>&1 | grep -E "^\{|NSD_CHECK|error" | cut -c1-200
python bench.py --workload c2 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "^\{|NSD_CHECK|error" | cut -c1-200
cp /tmp/product.so $L
