"""Diagnostic: single-scene kernel time per config (fp64/fp32) and us per CR iteration."""
import sys
sys.path.insert(0, ".")
from tests.helpers import oracle_case, rel_err, run_gpu, run_oracle
for name in ["c1", "c3", "c5", "c2:6", "c4:6", "c2", "c4"]:
    for prec in ("fp64", "fp32"):
        case = oracle_case(name, 0, 0)
        ms = []
        for _ in range(3):
            g = run_gpu(case, prec)
            ms.append(g["ms"])
        o = run_oracle(case)
        its = int(g["stats"][:, 5].sum())
        print(f"{name:6s} {prec} kernel {min(ms):8.3f} ms  CR iters {its:4d}  us/CR {1000*min(ms)/max(its,1):7.2f}  q err {rel_err(g['q'], o['q']):.1e} rows {g['n_rows']}", flush=True)
