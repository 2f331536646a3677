import sys; sys.path.insert(0, '.')
from tests.helpers import oracle_case, run_gpu, run_oracle, rel_err
for name, warm in [("c2:6", 0), ("c2", 0), ("c4", 0), ("c4:6", 0)]:
    case = oracle_case(name, 0, warm)
    o = run_oracle(case)
    for prec in ("fp64", "fp32"):
        g = run_gpu(case, prec)
        print(name, warm, prec, "q %.2e u %.2e lam %.2e" % (rel_err(g["q"], o["q"]), rel_err(g["u"], o["u"], floor=1e-6), rel_err(g["lam"], o["lam"], floor=1e-9)), flush=True)
