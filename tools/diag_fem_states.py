# Diagnostic (GPU): single-step FEM parity from oracle states at several warm steps.
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from tests.helpers import oracle_case, run_gpu, run_oracle, rel_err, decision_mismatches
for name in sys.argv[1:] or ["c4:6", "c2:6"]:
    for warm in [0, 1, 2, 3]:
        case = oracle_case(name, 0, warm)
        g = run_gpu(case, "fp64"); o = run_oracle(case)
        dq = np.abs(g["q"] - o["q"]); i = int(np.argmax(dq))
        print(name, "warm", warm, "q", f"{rel_err(g['q'], o['q']):.2e}", "u", f"{rel_err(g['u'], o['u'], floor=1e-6):.2e}",
              "lam", f"{rel_err(g['lam'], o['lam'], floor=1e-9):.2e}", "argmax", i, "nc", len(case["contacts"][0]))
        print("  pcr g", g["stats"][:, 5].astype(int), "o", o["stats"][:, 5].astype(int))
        print("  res g", np.array2string(g["stats"][:, 0], precision=3), "o", np.array2string(o["stats"][:, 0], precision=3))
        print("  linres g", np.array2string(g["stats"][:, 6], precision=2), "o", np.array2string(o["stats"][:, 6], precision=2))
