"""World / step_world through the product (scene.cpp:709-732): host-side caller
work (driven anchors, u~, contact detection) + the GPU Newton step, against
the oracle's step_world.

CPU: the product's host detection (nsd_scene_detect) returns the oracle's
contact set bit for bit (count, order, bodies, features, geometry) on rigid,
FEM-particle and driven-anchor scenes.
GPU: multi-step trajectories in fp64 track the oracle (stated tolerances as in
test_gpu_parity.py) with identical contact sets every step.
"""
import numpy as np
import pytest

from oracle import oracle_py as O
from tests.helpers import oracle_trajectory, rel_err

DETECT_CASES = [("c1", 0, 0), ("c1", 0, 20), ("c5", 3, 12), ("c2:6", 0, 3), ("c4:6", 0, 4), ("box_pile", 1, 30),
                ("arch", 0, 2), ("c3", 0, 5), ("heavy_stack", 0, 10), ("incline:35:0.5", 0, 5),
                ("c4", 0, 3)]


@pytest.mark.parametrize("name,seed,warm", DETECT_CASES)
def test_host_detect_matches_oracle_bitwise(name, seed, warm):
    from paper_1907_04587_b200 import World

    w = O.OracleWorld(name, seed)
    if warm:
        w.step(warm)
    w.prepare()
    q, u = w.state()
    ib, db = w.contacts()
    pw = World(name, seed)
    pw.q, pw.u = q.copy(), u.copy()
    gib, gdb = pw.detect()
    pw.close()
    assert len(gib) == len(ib)
    assert np.array_equal(gib[:, :3], ib[:, :3])
    assert np.array_equal(gdb[:, :17], db[:, :17])


def test_host_detect_with_extra_force():
    """u~ includes the extension force (step_world f_extra), so the predicted-gap filter sees it."""
    from paper_1907_04587_b200 import World

    w = O.OracleWorld("c5", 2)
    w.step(6)
    tau = np.linspace(-2.0, 2.0, w.dims()["n_joints"])
    w.set_joint_torques(tau)
    fx = w.f_extra()
    w.prepare()
    q, u = w.state()
    ib, db = w.contacts()
    pw = World("c5", 2)
    pw.q, pw.u, pw.f_extra = q.copy(), u.copy(), fx.copy()
    gib, gdb = pw.detect()
    assert np.array_equal(gib[:, :3], ib[:, :3]) and np.array_equal(gdb[:, :17], db[:, :17])


def test_driven_anchor_frames_advance():
    from paper_1907_04587_b200 import World, _lib

    pw = World("c4:6", 0)
    f0 = pw.joint_frames()
    _lib.check(_lib.lib().nsd_scene_advance_anchors(pw._h))
    f1 = pw.joint_frames()
    moved = np.nonzero(np.any(f0.reshape(-1, 21) != f1.reshape(-1, 21), axis=1))[0]
    assert len(moved) == 4  # the four fingertip drives (anchor_velocity 0.02 m/s inward)
    d = (f1 - f0).reshape(-1, 21)[moved]
    assert np.allclose(np.linalg.norm(d[:, 3:6], axis=1), 0.02 * pw.h)


# Rigid scenes: fixed stated tolerances. FEM scenes and the incline: the
# tolerance is 10x the oracle's own trajectory change under a 1e-15 relative
# perturbation of the initial q (tests/helpers.py:oracle_self_divergence) —
# stiff FEM with the 1e12 friction-W cap stops the PCR far from convergence,
# and the incline box starts at gap 0 / lambda 0, the Fischer-Burmeister origin
# where dphi switches branch (ncp.cpp:22-31) on a rounding-level gap.
STEP_CASES = [("c1", 0, 12, 1e-9), ("c3:30", 0, 6, 1e-9), ("c5", 1, 15, 1e-8), ("box_pile", 2, 10, 1e-8),
              ("incline:35:0.5", 0, 10, 1e-9), ("bend_chain", 0, 30, 1e-9), ("bend_chain:6:5", 0, 30, 1e-9),
              ("c4:6", 0, 4, None), ("c2:6", 0, 3, None)]

_TRAJ = {}


def _traj(name, seed, steps, perturb=0.0, k=0):
    """oracle_trajectory, memoised across test cases and precisions."""
    key = (name, seed, steps, perturb, k)
    if key not in _TRAJ:
        _TRAJ[key] = oracle_trajectory(name, seed, steps, perturb=perturb, perturb_seed=k)
    return _TRAJ[key]


def _reference(name, seed, steps, perturb, trials=2):
    """The oracle trajectory and, for the self-divergence bound, `trials` trajectories
    from a relatively perturbed initial q."""
    per = [_traj(name, seed, steps, perturb, k) for k in range(trials)] if perturb else None
    return _traj(name, seed, steps), per


# self-divergence perturbation: a few fp64 ulp; for the fp32 mode the fp32 unit roundoff
# (its J/C coefficients carry that relative rounding)
EPS = {"fp64": 1e-15, "fp32": 2.0 ** -24}


def _track(name, seed, steps, prec, tol, floor=0.0, trials=2):
    """World.step against the oracle's step_world, step by step. tol: fixed bound on q
    (u: 100x) with bit-exact contact sets; None: max(floor, 10x the oracle's
    self-divergence under a relative perturbation EPS[prec] of its initial q) on q and u."""
    from paper_1907_04587_b200 import World

    ref, per = _reference(name, seed, steps, EPS[prec] if tol is None else 0.0, trials)
    pw = World(name, seed, precision=prec)
    worst = 0.0
    for s in range(steps):
        rep = pw.step(1)
        oq, ou, oib, orc = ref[s]
        assert bool(rep["aborted"]) == (orc == 2), (name, s)
        eq, eu = rel_err(pw.q, oq), rel_err(pw.u, ou, floor=1e-3)
        worst = max(worst, eq)
        if tol is None:
            sq = max(rel_err(p[s][0], oq) for p in per)
            su = max(rel_err(p[s][1], ou, floor=1e-3) for p in per)
            assert eq <= max(floor, 10 * sq + 1e-9), (name, prec, s, eq, sq)
            assert eu <= max(100 * floor, 10 * su + 1e-7), (name, prec, s, eu, su)
        else:
            gib, _ = pw.contacts
            assert np.array_equal(gib[:, :3], oib[:, :3]), (name, prec, s)
            assert eq < tol, (name, prec, s, eq)
            assert eu < 100 * tol, (name, prec, s, eu)
    pw.close()
    print(f"{name} {prec} {steps} steps: max q rel err {worst:.2e}")


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed,steps,tol", STEP_CASES)
def test_world_steps_match_oracle_fp64(name, seed, steps, tol):
    _track(name, seed, steps, "fp64", tol)


# fp32 mode (fp64 state and arithmetic, fp32 J/C coefficient storage): the north_star
# tolerance 1e-4 on q (u 1e-2) after >= 25 steps through ground impacts, contact sets
# bit-exact (measured: c1 5e-14, c3 3e-10, c5 2e-8, box_pile 6e-7). Stiff FEM and the
# incline's Fischer-Burmeister origin: 1e-4, or 10x the oracle's own change when its
# initial q carries fp32-sized (2^-24) relative rounding, where that is larger — on
# full-size C2 at step 0 the oracle amplifies a 1e-15 input perturbation ~3e7-fold,
# so fp32-rounded coefficients cannot stay within 1e-4 of it.
FP32_CASES = [("c1", 0, 25, 1e-4), ("c3", 0, 25, 1e-4), ("c5", 1, 25, 1e-4), ("box_pile", 2, 25, 1e-4),
              ("bend_chain", 0, 25, 1e-4), ("incline:35:0.5", 0, 25, None), ("c2:6", 0, 6, None), ("c4:6", 0, 6, None)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed,steps,tol", FP32_CASES)
def test_world_steps_match_oracle_fp32(name, seed, steps, tol):
    _track(name, seed, steps, "fp32", tol, floor=1e-4)


# Full-size FEM configs (C2: 12^3 block, 10,368 tets; C4: hand + 5,520-tet ball) over 6
# steps, both precisions, against the oracle's explicit-S step_world.
@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
@pytest.mark.parametrize("name", ["c2", "c4"])
def test_world_full_fem_six_steps(name, prec):
    _track(name, 0, 6, prec, None, floor=1e-9 if prec == "fp64" else 1e-4, trials=1 if name == "c2" else 2)
