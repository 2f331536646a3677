"""Diagnostic (not collected by pytest): prints GPU-vs-oracle errors for every
config so a single gpurun call shows the whole picture."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from tests.helpers import oracle_case, rel_err, run_gpu, run_oracle  # noqa: E402

cases = sys.argv[1:] or ["c1", "c3", "c5", "c2:6", "c4:6", "heavy_stack", "stretch_sheet", "c2", "c4"]
for name in cases:
    for prec in ("fp64", "fp32"):
        try:
            case = oracle_case(name, 0, 0)
            t0 = time.time()
            g = run_gpu(case, prec)
            t1 = time.time()
            o = run_oracle(case)
            t2 = time.time()
            print(f"{name:14s} {prec} q {rel_err(g['q'], o['q']):.2e} u {rel_err(g['u'], o['u'], 1e-6):.2e} "
                  f"lam {rel_err(g['lam'], o['lam'], 1e-9):.2e} lin g {g['stats'][:, 5].astype(int).tolist()} "
                  f"o {o['stats'][:, 5].astype(int).tolist()} res g {g['stats'][-1, 0]:.3e} o {o['stats'][-1, 0]:.3e} "
                  f"kernel {g['ms']:.3f} ms gpu-call {t1 - t0:.2f}s oracle {t2 - t1:.2f}s", flush=True)
        except Exception:
            traceback.print_exc()
