"""Profiling driver: one c2 newton_step through the C ABI (fp64)."""
import sys
sys.path.insert(0, ".")
from tests.helpers import oracle_case, run_gpu
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
case = oracle_case(name, 0, 0)
for _ in range(2):
    g = run_gpu(case, prec)
print(name, prec, g["ms"])
