"""GPU parity: the sm_100a Newton step (through the C ABI) against the CPU
oracle on identical inputs (state, contact set, joint frames) at the
reference's fixed Newton/PCR budgets.

Tolerances (stated per precision, relative to the max magnitude of the
oracle quantity):
  fp64 parity mode: q, u 1e-9; lambda 1e-6; decisions (PCR iterations used,
                    breakdown, abort) identical.
  fp32 performance mode: q, u 1e-4 (BASELINE north_star); lambda 1e-2 (the
                    multipliers of stiff FEM rows are ill-conditioned in fp32).
"""
import numpy as np
import pytest

from tests.helpers import oracle_case, rel_err, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = [("c1", 0, 0), ("c1", 0, 20), ("c3", 0, 0), ("c3", 0, 15), ("c5", 0, 0), ("c5", 3, 12), ("c2:6", 0, 0),
         ("c4:6", 0, 0), ("heavy_stack", 0, 0), ("box_pile", 1, 30), ("stretch_sheet", 0, 3), ("incline:35:0.5", 0, 5),
         ("arch", 0, 0)]


def _compare(case_name, prec, seed, warm):
    case = oracle_case(case_name, seed, warm)
    g = run_gpu(case, prec)
    o = run_oracle(case)
    tol_q = 1e-9 if prec == "fp64" else 1e-4
    tol_l = 1e-6 if prec == "fp64" else 1e-2
    assert g["aborted"] == (o["rc"] == 2)
    eq = rel_err(g["q"], o["q"])
    eu = rel_err(g["u"], o["u"], floor=1e-6)
    el = rel_err(g["lam"], o["lam"], floor=1e-9)
    msg = f"{case_name} {prec}: q {eq:.2e} u {eu:.2e} lam {el:.2e}"
    assert eq <= tol_q, msg
    assert eu <= tol_q * 10, msg
    assert el <= tol_l, msg
    if prec == "fp64":
        assert np.array_equal(g["stats"][:, 5], o["stats"][:, 5]), (msg, g["stats"][:, 5], o["stats"][:, 5])
        assert np.array_equal(g["stats"][:, 7], o["stats"][:, 7]), msg
    return g, o


@pytest.mark.parametrize("name,seed,warm", CASES)
def test_newton_step_fp64(name, seed, warm):
    _compare(name, "fp64", seed, warm)


@pytest.mark.parametrize("name,seed,warm", CASES)
def test_newton_step_fp32(name, seed, warm):
    _compare(name, "fp32", seed, warm)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c4"])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_newton_step_full_fem(name, prec):
    _compare(name, prec, 0, 0)


def test_report_fields_fp64():
    case = oracle_case("c1", 0, 10)
    g = run_gpu(case, "fp64")
    o = run_oracle(case)
    # per-iteration statistics (newton.h:45-54) and final classification
    for k in (0, 1, 2, 3, 4, 6):
        assert rel_err(g["stats"][:, k], o["stats"][:, k], floor=1e-12) < 1e-6, k
    assert rel_err(g["final"][:4], o["final"][:4], floor=1e-12) < 1e-6
    assert g["final"][6] == o["final"][6]
    # linear residual histories
    for i in range(g["n_iterations"]):
        n = g["hist_len"][i]
        assert n == o["hist_len"][i]
        assert rel_err(g["hist"][i, :n], o["hist"][i, :n], floor=1e-14) < 1e-6
    # contact telemetry and multiplier write-back
    assert rel_err(g["tel"], o["tel"], floor=1e-9) < 1e-6
    gib, gdb = g["contacts"]
    oib, odb = case["world"].contacts()
    assert np.array_equal(gib, oib)
    assert rel_err(gdb[:, 17:20], odb[:, 17:20], floor=1e-9) < 1e-6


def test_extra_force_hook_fp64():
    case = oracle_case("c5", 5, 3)
    w = case["world"]
    tau = np.linspace(-1, 1, case["dims"]["n_joints"])
    w.set_joint_torques(tau)
    fx = w.f_extra()
    w.prepare()  # recompute contacts with the hook active
    case["contacts"] = w.contacts()
    q, u = w.state()
    case["q"], case["u"] = q, u
    case["joint_frame"] = w.joint_frames()
    g = run_gpu(case, "fp64", f_extra=fx)
    o = run_oracle(case)
    assert rel_err(g["q"], o["q"]) < 1e-9
    assert rel_err(g["u"], o["u"], floor=1e-6) < 1e-8


def test_line_search_frictionless_fp64():
    case = oracle_case("c3:30", 0, 2, overrides=dict(line_search=1))
    g = run_gpu(case, "fp64")
    o = run_oracle(case)
    assert rel_err(g["q"], o["q"]) < 1e-9
    assert np.allclose(g["stats"][:, 4], o["stats"][:, 4], rtol=1e-6, atol=1e-12)


def test_invalid_h_rejected():
    from paper_1907_04587_b200 import NsdError

    case = oracle_case("c1", 0, 0)
    case["h"] = 0.0
    with pytest.raises(NsdError) as e:
        run_gpu(case, "fp64")
    assert e.value.code == 1


def test_determinism_bitwise():
    case = oracle_case("c2:6", 0, 0)
    a = run_gpu(case, "fp32")
    b = run_gpu(case, "fp32")
    assert np.array_equal(a["q"], b["q"]) and np.array_equal(a["lam"], b["lam"])
