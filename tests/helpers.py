"""Shared helpers for parity tests: build a case with the CPU oracle, run the
same newton_step through the C ABI on the GPU, compare."""
import numpy as np

from oracle import oracle_py as O


def oracle_case(name, seed=0, warm_steps=0, overrides=None):
    w = O.OracleWorld(name, seed)
    if overrides:
        w.set_config(**overrides)
    if warm_steps:
        w.step(warm_steps)
    w.prepare()
    q, u = w.state()
    ib, db = w.contacts()
    return dict(world=w, topo=w.topology(), q=q, u=u, contacts=(ib, db), h=w.h, gravity=w.gravity(),
                joint_frame=w.joint_frames(), cfg=w.get_config(), dims=w.dims())


def newton_config(cfg, precision):
    from paper_1907_04587_b200 import NewtonConfig

    return NewtonConfig(newton_iterations=cfg["newton_iterations"], step_fraction=cfg["step_fraction"],
                        epsilon_reg=cfg["epsilon_reg"], geometric_stiffness=bool(cfg["geometric_stiffness"]),
                        r_strategy=cfg["r_strategy"], ncp_kind=cfg["ncp_kind"], linear_method=cfg["linear_method"],
                        linear_max_iterations=cfg["linear_max_iterations"], linear_tolerance=cfg["linear_tolerance"],
                        preconditioner=cfg["preconditioner"], newton_tolerance=cfg["newton_tolerance"],
                        line_search=bool(cfg["line_search"]), precision=precision)


def run_gpu(case, precision, f_extra=None):
    from paper_1907_04587_b200 import NewtonSolver, Topology

    topo = Topology(**case["topo"])
    s = NewtonSolver(topo, newton_config(case["cfg"], precision))
    out = s.newton_step(case["q"], case["u"], case["contacts"], h=case["h"], gravity=tuple(case["gravity"]),
                        f_extra=f_extra, joint_frame=case["joint_frame"])
    s.close()
    return out


def run_oracle(case):
    w = case["world"]
    rc = w.newton()
    q, u = w.state()
    rep = w.report()
    return dict(q=q, u=u, rc=rc, decisions=w.decisions(), **rep)


def rel_err(a, b, floor=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), floor))


def decision_mismatches(g, o, tol, floor_ratio=1e-9):
    """PCR iteration counts per Newton iteration: returns (n_mismatch, n_non_borderline).
    A count differs legitimately only where the run ended at a rounding-level
    boundary: residual within 10x of the absolute tolerance, or at the numerical
    floor (<= floor_ratio of the initial residual) where the monotone guard fires."""
    bad = 0
    mism = 0
    for i in range(min(g["n_iterations"], o["n_iterations"])):
        if g["stats"][i, 5] == o["stats"][i, 5]:
            continue
        mism += 1
        h0 = max(g["hist"][i, 0], o["hist"][i, 0])
        ends = [g["stats"][i, 6], o["stats"][i, 6]]
        borderline = any(tol > 0 and tol / 10 <= e <= tol * 10 for e in ends) or \
            any(e <= floor_ratio * h0 for e in ends)
        if not borderline:
            bad += 1
    return mism, bad


def oracle_self_divergence(name, seed=0, warm_steps=0, eps=1e-15, trials=3, overrides=None):
    """Rounding sensitivity of one newton_step at a state: the largest relative
    change of the ORACLE's own (q, u) when its input q is perturbed by eps
    (relative, a few ulp). Where the PCR stops far from convergence (stiff FEM
    with the 1e12 friction-W cap, or a Fischer-Burmeister decision taken at the
    origin) two correct implementations that associate sums differently can
    differ by this much; GPU-vs-oracle tolerances there are stated as a
    multiple of it."""
    ref = run_oracle(oracle_case(name, seed, warm_steps, overrides))
    worst_q = worst_u = 0.0
    for t in range(trials):
        c = oracle_case(name, seed, warm_steps, overrides)
        w = c["world"]
        q, u = w.state()
        rng = np.random.default_rng(1000 + t)
        w.set_state(q * (1.0 + eps * rng.standard_normal(q.size)), u)
        w.prepare()
        p = run_oracle(c)
        worst_q = max(worst_q, rel_err(p["q"], ref["q"]))
        worst_u = max(worst_u, rel_err(p["u"], ref["u"], floor=1e-6))
    return worst_q, worst_u


def oracle_trajectory(name, seed, steps, perturb=0.0, perturb_seed=0):
    """q, u after each of `steps` oracle step_world calls (optionally from a
    relatively perturbed initial q), plus the per-step contact index arrays."""
    w = O.OracleWorld(name, seed)
    if perturb:
        q, u = w.state()
        rng = np.random.default_rng(perturb_seed)
        w.set_state(q * (1.0 + perturb * rng.standard_normal(q.size)), u)
    out = []
    for _ in range(steps):
        rc = w.step(1)
        q, u = w.state()
        out.append((q, u, w.contacts()[0], rc))
    return out
