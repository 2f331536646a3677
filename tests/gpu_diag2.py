"""Diagnostic: error growth vs Newton/PCR budget on FEM cases (fp64), and
per-step divergence of the batched fp32 path."""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests.helpers import oracle_case, rel_err, run_gpu, run_oracle
from oracle import oracle_py as O

for name in ["c2:6", "stretch_sheet", "c4:6"]:
    for (ni, nl, tol) in [(1, 1, 1e-10), (1, 5, 1e-10), (1, 20, 1e-10), (1, 60, 1e-10), (2, 60, 1e-10), (10, 60, 1e-10), (1, 60, 0.0)]:
        for prec in ("fp64", "fp32"):
            case = oracle_case(name, 0, 0, overrides=dict(newton_iterations=ni, linear_max_iterations=nl, linear_tolerance=tol))
            g = run_gpu(case, prec)
            o = run_oracle(case)
            print(f"{name:13s} N={ni:2d} L={nl:2d} tol={tol:g} {prec} q {rel_err(g['q'], o['q']):.2e} u {rel_err(g['u'], o['u'], 1e-6):.2e} lam {rel_err(g['lam'], o['lam'], 1e-9):.2e} lin {g['stats'][:,5].astype(int).tolist()} vs {o['stats'][:,5].astype(int).tolist()} hist0 g {g['hist'][0,0]:.6e} o {o['hist'][0,0]:.6e}", flush=True)

from paper_1907_04587_b200 import BatchSolver, Scene
for prec in ("fp32", "fp64"):
    n_env = 16
    s0 = Scene("c5", 0)
    qs = np.concatenate([Scene("c5", e).q for e in range(n_env)])
    us = np.concatenate([Scene("c5", e).u for e in range(n_env)])
    cfg = s0.config; cfg.precision = prec
    b = BatchSolver(s0.topology, s0.shapes, s0.n_shapes, s0.margin, s0.mu_default, cfg, n_env, 48)
    b.set_state(qs, us)
    ws = [O.OracleWorld("c5", e) for e in range(n_env)]
    for st in range(30):
        for w in ws: w.step(1)
        b.step(s0.h, s0.gravity)
        r = b.results()
        q, u = b.get_state()
        eq = max(rel_err(q[e], ws[e].state()[0]) for e in range(n_env))
        eu = max(rel_err(u[e], ws[e].state()[1], 1e-3) for e in range(n_env))
        mism = sum(int(r["n_contacts"][e] != ws[e].dims()["n_contacts"]) for e in range(n_env))
        print(f"batch {prec} step {st:2d} max q err {eq:.2e} u err {eu:.2e} contact-count mismatches {mism} ncontacts {r['n_contacts'][:6].tolist()}", flush=True)
