"""Diagnostic: fp32 and fp64 vs oracle at fixed budgets (linear tolerance 0) on every config."""
import sys
sys.path.insert(0, ".")
from tests.helpers import oracle_case, rel_err, run_gpu, run_oracle

CASES = [("c1", 0, 0), ("c1", 0, 20), ("c3", 0, 0), ("c3", 0, 15), ("c5", 0, 0), ("c5", 3, 12), ("c2:6", 0, 0),
         ("c4:6", 0, 0), ("heavy_stack", 0, 0), ("box_pile", 1, 30), ("stretch_sheet", 0, 3), ("incline:35:0.5", 0, 5),
         ("arch", 0, 0), ("c2", 0, 0), ("c4", 0, 0)]
for name, seed, warm in CASES:
    for tol in (1e-10, 0.0):
        for prec in ("fp64", "fp32"):
            case = oracle_case(name, seed, warm, overrides=dict(linear_tolerance=tol))
            g = run_gpu(case, prec)
            o = run_oracle(case)
            print(f"{name:15s} w{warm:2d} tol={tol:g} {prec} q {rel_err(g['q'], o['q']):.2e} u {rel_err(g['u'], o['u'], 1e-6):.2e} "
                  f"lam {rel_err(g['lam'], o['lam'], 1e-9):.2e} lin_eq {int((g['stats'][:,5]==o['stats'][:,5]).all())} ms {g['ms']:.2f}", flush=True)
