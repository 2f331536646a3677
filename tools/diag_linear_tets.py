# Diagnostic (GPU): linear co-rotational tets vs the oracle, one Newton x one PCR iteration.
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from tests.helpers import oracle_case, run_gpu, run_oracle, rel_err
for warm in [0, 2]:
    case = oracle_case("stretch_sheet_linear", 0, warm, overrides=dict(newton_iterations=1, linear_max_iterations=1))
    g = run_gpu(case, "fp64"); o = run_oracle(case)
    rj = case["dims"]["rows_joint"]
    lg, lo = g["lam"], o["lam"]
    ratio = np.where(np.abs(lo) > 1e-14, lg / np.where(lo == 0, 1, lo), np.nan)
    print("warm", warm, "hist g", g["hist"][0, :2], "o", o["hist"][0, :2])
    print("  joint rows ratio", np.round(ratio[:rj][:8], 4))
    print("  tet rows ratio  ", np.round(ratio[rj:rj + 12], 4))
    print("  lam g", lg[rj:rj + 6], "\n  lam o", lo[rj:rj + 6])
