"""SPEC acceptance criteria (and the newton_step
examples at :505-507) as goldens for the PRODUCT path: World.step (host caller
work + the GPU newton_step through the C ABI) in fp64, with the CPU oracle's
step_world run beside it on the same scene. Each criterion is asserted on the
product; the oracle must satisfy it too, and the two runs must agree to the
stated tolerance where the scene is well conditioned."""
import math

import numpy as np
import pytest

from oracle import oracle_py as O
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

G = 9.81


def _world(name, **cfg):
    from paper_1907_04587_b200 import World

    w = World(name, 0, precision="fp64")
    for k, v in cfg.items():
        setattr(w.config, k, v)
    ow = O.OracleWorld(name, 0)
    if cfg:
        ow.set_config(**cfg)
    return w, ow


def _speed(u):
    return float(np.linalg.norm(u[:3]))


def test_spec5_incline_20deg_sticks():  # SPEC.md:703 (tan 20 deg = 0.364 < mu = 0.5)
    w, ow = _world("incline:20:0.5")
    for _ in range(200):
        w.step()
    assert ow.step(200) == 0
    oq, ou = ow.state()
    assert _speed(w.u) < 1e-3 and _speed(ou) < 1e-3
    assert rel_err(w.q, oq) < 1e-9


def test_spec5_incline_35deg_slides_at_g_sin_minus_mu_cos():
    w, ow = _world("incline:35:0.5")
    th = math.radians(35.0)
    expect = G * (math.sin(th) - 0.5 * math.cos(th))
    v = []
    for _ in range(120):
        w.step()
        v.append(_speed(w.u))
    ov = []
    for _ in range(120):
        assert ow.step(1) == 0
        ov.append(_speed(ow.state()[1]))
    acc = []
    for series in (v, ov):
        a = (series[119] - series[19]) / (100 * w.h)
        assert abs(a - expect) <= 0.05 * expect, (a, expect)
        acc.append(a)
    # the box starts touching (gap 0, lambda 0), the Fischer-Burmeister origin: the same
    # branch on both sides (the device's uncontracted gap), so the runs agree throughout
    assert rel_err(v, ov) < 1e-9


def test_spec6_friction_cone_and_dissipation():  # SPEC.md:704, box pile + incline
    # with the scenes' own budgets no step meets newton_tolerance (1e-6), which leaves the
    # criterion vacuous; a 30 x 100 budget makes the steps converge
    converged = 0
    for name, steps in (("box_pile", 40), ("incline:35:0.5", 40)):
        w, ow = _world(name, newton_iterations=30, linear_max_iterations=100)
        for _ in range(steps):
            rep = w.step()
            orc = ow.step(1)
            assert orc == 0 and not rep["aborted"]
            for tel, conv in ((rep["tel"], rep["final"][6]), (ow.report()["tel"], ow.report()["final"][6])):
                if not conv or len(tel) == 0:
                    continue
                converged += 1
                h = w.h
                # |lambda_f| <= mu lambda_n + 1e-6 (impulses = force x h)
                assert np.all(tel[:, 2] * h <= tel[:, 3] * tel[:, 1] * h + 1e-6), name
                sliding = tel[:, 4] > 1e-6
                assert np.all(tel[sliding, 5] <= 1e-9), name  # friction opposes the tangential velocity
    assert converged > 0


def _max_penetration(w, steps):
    worst = 0.0
    for _ in range(steps):
        rep = w.step()
        assert not rep["aborted"]
        worst = max(worst, -rep["final"][3])  # min_gap of the final state
    return worst


def _oracle_max_penetration(ow, steps):
    worst = 0.0
    for _ in range(steps):
        assert ow.step(1) == 0
        worst = max(worst, -ow.report()["final"][3])
    return worst


def test_spec7_heavy_stack_pcr_penetration_below_5mm():  # SPEC.md:705, PCR 25 x Newton 5, 500 steps
    w, ow = _world("heavy_stack", newton_iterations=5, linear_max_iterations=25)
    pen = _max_penetration(w, 500)
    opn = _oracle_max_penetration(ow, 500)
    assert pen < 5e-3 and opn < 5e-3, (pen, opn)


def test_spec7_heavy_stack_jacobi_exceeds_5mm():  # SPEC.md:705, the comparative half (Fig. 8)
    w, ow = _world("heavy_stack", newton_iterations=5, linear_max_iterations=25, linear_method=0)
    pen = _max_penetration(w, 500)
    opn = _oracle_max_penetration(ow, 500)
    assert pen > 5e-3 and opn > 5e-3, (pen, opn)


def test_spec8_effective_mass_beats_identity_10x():  # SPEC.md:706, one step, 100 Newton iterations
    errs = {}
    for strat in (0, 2):  # identity, effective mass
        w, ow = _world("heavy_stack", newton_iterations=100, r_strategy=strat)
        rep = w.step()
        assert ow.step(1) == 0
        errs[strat] = (rep["final"][1], ow.report()["final"][1])
    assert errs[0][0] >= 10.0 * errs[2][0], errs
    assert errs[0][1] >= 10.0 * errs[2][1], errs


def test_spec11_epsilon_halving_changes_impulses_below_1e4():  # SPEC.md:709, box_on_plane
    lam = {}
    for eps in (1e-6, 5e-7):
        w, ow = _world("box_on_plane", epsilon_reg=eps)
        for _ in range(30):
            rep = w.step()
        assert ow.step(30) == 0
        lam[eps] = (rep["lam"].copy(), ow.report()["lam"].copy())
    for i in range(2):  # product, oracle
        a, b = lam[1e-6][i], lam[5e-7][i]
        assert np.max(np.abs(a - b)) <= 1e-4 * np.max(np.abs(a)), i


def test_spec12_determinism_bitwise():  # SPEC.md:710, two identical product runs
    runs = []
    for _ in range(2):
        w, _ = _world("box_pile")
        traj = []
        for _ in range(40):
            rep = w.step()
            traj.append(np.concatenate([rep["q"], rep["u"], rep["lam"]]))
        runs.append(np.concatenate(traj))
    assert np.array_equal(runs[0], runs[1])


def test_spec_free_fall_one_iteration_is_u_tilde():  # SPEC.md:505, through World
    from paper_1907_04587_b200 import World

    w = World("box_on_plane", 0, precision="fp64")
    w.config.newton_iterations = 1
    w.config.step_fraction = 1.0  # the undamped update of the SPEC example
    w.q = w.q.copy()
    w.q[2] += 10.0  # lifted far above the margin: no contacts
    u0 = w.u.copy()
    rep = w.step()
    assert len(rep["tel"]) == 0
    ut = u0.copy()
    ut[2] += w.h * (-G)
    assert np.array_equal(w.u, ut)  # unit mass, zero spin: M^-1 (M u~) is exact here
