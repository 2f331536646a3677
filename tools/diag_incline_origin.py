# Diagnostic (GPU): incline step-0 divergence at the Fischer-Burmeister origin (see tests/test_world.py).
import numpy as np, sys
sys.path.insert(0, '/root/repo')
from tests.helpers import oracle_case, run_gpu, run_oracle, rel_err, decision_mismatches
for warm in [0, 1, 2]:
    case = oracle_case("incline:35:0.5", 0, warm)
    g = run_gpu(case, "fp64"); o = run_oracle(case)
    print("warm", warm, "q", rel_err(g["q"], o["q"]), "u", rel_err(g["u"], o["u"], floor=1e-6))
    print(" pcr g", g["stats"][:, 5], "o", o["stats"][:, 5])
    print(" linres g", g["stats"][:, 6], "o", o["stats"][:, 6])
    print(" hist0 g", g["hist"][:, 0], "o", o["hist"][:, 0])
    print(" mism", decision_mismatches(g, o, case["cfg"]["linear_tolerance"]))
