"""Batched many-environment path (C5 ants) against the oracle's step_world run
per environment: bit-exact contact set (count, order, bodies, features) every
step, states within the stated tolerance, with and without the joint-torque
extension hook, and env results independent of how environments are grouped
(the property that makes GPU sharding safe)."""
import numpy as np
import pytest

from oracle import oracle_py as O
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _batch(n_env, prec, env0=0, max_contacts=48, team=None, env=None):
    import os

    from paper_1907_04587_b200 import BatchSolver, Scene

    env = dict(env or {})
    if team:
        env["NSD_BATCH_TEAM"] = str(team)
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    s0 = Scene("c5", 0)
    qs, us = [], []
    for e in range(env0, env0 + n_env):
        s = Scene("c5", e)
        qs.append(s.q)
        us.append(s.u)
    cfg = s0.config
    cfg.precision = prec
    try:
        b = BatchSolver(s0.topology, s0.shapes, s0.n_shapes, s0.margin, s0.mu_default, cfg, n_env, max_contacts)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    b.set_state(np.concatenate(qs), np.concatenate(us))
    return b, s0


def _torques(env, step, nj):
    rng = np.random.default_rng(env * 1000003 + step)
    return rng.uniform(-1.0, 1.0, nj)


# fp64: tracked to 1e-11 over 25 steps (measured ~1e-14). fp32 is the mixed mode
# (fp64 state, assembly, Newton update and reductions; fp32 PCR operator): the
# north_star's 1e-4 over the same 25 steps, contact sets bit-exact.
@pytest.mark.parametrize("prec,steps,tol", [("fp64", 25, 1e-11), ("fp32", 25, 1e-4)])
@pytest.mark.parametrize("actuated", [False, True])
def test_batch_matches_oracle(prec, steps, tol, actuated):
    n_env = 24
    b, s0 = _batch(n_env, prec)
    nj = s0.topology.n_joints
    worlds = [O.OracleWorld("c5", e) for e in range(n_env)]
    for st in range(steps):
        tau = np.stack([_torques(e, st, nj) for e in range(n_env)]) if actuated else None
        for e, w in enumerate(worlds):
            w.set_joint_torques(tau[e] if actuated else None)
            assert w.step(1) == 0
        b.step(s0.h, s0.gravity, torque=tau.reshape(-1) if actuated else None)
        res = b.results()
        assert not res["aborted"].any()
        q, u = b.get_state()
        for e, w in enumerate(worlds):
            ib, db = w.contacts()
            gib, gdb = b.contacts(e)
            assert res["n_contacts"][e] == len(ib), (st, e)
            assert np.array_equal(gib[:, :3], ib[:, :3]), (st, e)
            oq, ou = w.state()
            assert rel_err(q[e], oq) < tol, (st, e, rel_err(q[e], oq))
            assert rel_err(u[e], ou, floor=1e-3) < tol * 100, (st, e)


def test_batch_team_shapes_agree_fp64():
    """Warp-per-env and CTA-per-env teams give the same states (fixed-order reductions differ
    only in association; fp64 agreement to 1e-12)."""
    teams = [_batch(16, "fp64", team=t) for t in (8, 16, 32, 64)]  # 8/16/32: object solver, 64: CTA engine
    s0 = teams[0][1]
    for _ in range(5):
        for b, _ in teams:
            b.step(s0.h, s0.gravity)
    q0, _ = teams[0][0].get_state()
    for b, _ in teams[1:]:
        q, _ = b.get_state()
        assert rel_err(q, q0) < 1e-11


def test_batch_env_offset_independent():
    """Env i gives the same bits whether it runs in a batch starting at env 0 or env 8
    (what the GPU sharding relies on)."""
    a, s0 = _batch(16, "fp32", env0=0)
    b, _ = _batch(8, "fp32", env0=8)
    for _ in range(6):
        a.step(s0.h, s0.gravity)
        b.step(s0.h, s0.gravity)
    qa, _ = a.get_state()
    qb, _ = b.get_state()
    assert np.array_equal(qa[8:], qb)


def test_batch_overflow_reported():
    from paper_1907_04587_b200 import NsdError

    b, s0 = _batch(4, "fp32", max_contacts=4)
    b.step(s0.h, s0.gravity)
    with pytest.raises(NsdError):
        b.results()


def test_batch_odd_env_count_partial_block_fp64():
    """n_env not a multiple of the envs per block: the last block's second team has no
    env (fixed region split there, no pool exchange); every env still tracks the oracle."""
    n_env = 5
    b, s0 = _batch(n_env, "fp64")
    worlds = [O.OracleWorld("c5", e) for e in range(n_env)]
    for st in range(6):
        for w in worlds:
            assert w.step(1) == 0
        b.step(s0.h, s0.gravity)
    q, _ = b.get_state()
    for e, w in enumerate(worlds):
        assert rel_err(q[e], w.state()[0]) < 1e-8, e


def test_batch_nan_env_aborts_alone():
    """One env with a NaN velocity aborts (rolled back, flagged); its neighbours in
    the same warp/block are unaffected and keep tracking the oracle."""
    b, s0 = _batch(4, "fp64")
    q, u = b.get_state()
    u = u.copy()
    u[1, 2] = np.nan
    b.set_state(q.reshape(-1), u.reshape(-1))
    b.step(s0.h, s0.gravity)
    res = b.results()
    assert res["aborted"].tolist() == [False, True, False, False]
    q1, _ = b.get_state()
    assert np.array_equal(q1[1], q[1])
    w = O.OracleWorld("c5", 2)
    assert w.step(1) == 0
    assert rel_err(q1[2], w.state()[0]) < 1e-12


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_batch_step_mapped_matches_device_step(prec):
    """nsd_batch_step_mapped (the step kernel reads the torques from, and writes (q, u)
    to, pinned host memory) gives the same bits as step_device + get_state, every step,
    in both precisions and for float and double torques."""
    import torch

    n_env = 20
    a, s0 = _batch(n_env, prec)
    b, _ = _batch(n_env, prec)
    nj, nq, nu = s0.topology.n_joints, s0.topology.num_coord, s0.topology.num_dof
    dt = torch.float64  # the batch state is fp64 in both modes (fp32 = mixed precision)
    h_q = torch.zeros(n_env * nq, dtype=dt, pin_memory=True)
    h_u = torch.zeros(n_env * nu, dtype=dt, pin_memory=True)
    for st in range(6):
        tdt = torch.float64 if st % 2 else torch.float32
        tau = np.stack([_torques(e, st, nj) for e in range(n_env)])
        h_tq = torch.tensor(tau, dtype=tdt).pin_memory()
        d_tq = h_tq.cuda()
        code = 1 if tdt == torch.float64 else 0
        torch.cuda.synchronize()
        a.step_device(s0.h, s0.gravity, d_tq.data_ptr(), code)
        b.step_mapped(s0.h, s0.gravity, h_tq.data_ptr(), code, h_q.data_ptr(), h_u.data_ptr())
        a.sync()
        b.sync()
        qa, ua = a.get_state()
        qb, ub = b.get_state()
        assert np.array_equal(qa, qb) and np.array_equal(ua, ub), st
        assert np.array_equal(h_q.numpy().astype(np.float64), qb.reshape(-1)), st
        assert np.array_equal(h_u.numpy().astype(np.float64), ub.reshape(-1)), st


def test_batch_step_mapped_rejects_pageable_memory():
    from paper_1907_04587_b200 import NsdError

    b, s0 = _batch(4, "fp64")
    q = np.zeros(4 * s0.topology.num_coord)
    with pytest.raises(NsdError):
        b.step_mapped(s0.h, s0.gravity, None, 1, q.ctypes.data, None)


# The default C5 path is the warp-per-env solver (nsd_warp.cuh) between the
# narrow-phase launch and the large-env launch; NSD_BATCH_FAST=0 runs the
# sub-warp object solver for every env, NSD_WARP_MAX_OBJ=k routes envs with more
# than k constraint objects (8 joints + contacts) to it.
@pytest.mark.parametrize("routing", [{"NSD_BATCH_FAST": "0"}, {"NSD_WARP_MAX_OBJ": "20"}, {"NSD_WARP_MAX_OBJ": "0"}])
def test_batch_warp_solver_matches_object_solver_fp64(routing):
    n_env = 48
    a, s0 = _batch(n_env, "fp64")
    b, _ = _batch(n_env, "fp64", env=routing)
    nj = s0.topology.n_joints
    for st in range(20):
        tau = np.stack([_torques(e, st, nj) for e in range(n_env)]).reshape(-1)
        a.step(s0.h, s0.gravity, torque=tau)
        b.step(s0.h, s0.gravity, torque=tau)
        ra, rb = a.results(with_iters=True), b.results(with_iters=True)
        assert np.array_equal(ra["n_contacts"], rb["n_contacts"]), st
        assert not ra["aborted"].any() and not rb["aborted"].any()
        # PCR iteration counts per Newton iteration agree (rounding-level operator differences)
        assert np.mean(ra["stats"][:, :, 5] == rb["stats"][:, :, 5]) > 0.98, st
    qa, ua = a.get_state()
    qb, ub = b.get_state()
    assert rel_err(qa, qb) < 1e-10
    assert rel_err(ua, ub, floor=1e-3) < 1e-8
    for e in (0, 7, 31, 47):
        ia, da = a.contacts(e)
        ib, db = b.contacts(e)
        assert np.array_equal(ia, ib)
        assert rel_err(da, db, floor=1e-6) < 1e-6  # geometry + multipliers


def test_batch_large_envs_track_oracle_fp64():
    """Envs routed to the large-env launch (more than 10 contacts: NSD_WARP_MAX_OBJ=18)
    and envs solved by the warp solver side by side in one actuated batch, both against
    the oracle every step. Half the ants start 0.3 m higher, so they land later and the
    batch holds both contact counts."""
    n_env, steps = 16, 25
    b, s0 = _batch(n_env, "fp64", env={"NSD_WARP_MAX_OBJ": "18"})
    nj = s0.topology.n_joints
    q, u = b.get_state()
    q = q.copy()
    bt = s0.topology.a["body_type"]
    zc = [7 * i + 2 for i in range(len(bt))]  # z of every (rigid) body
    q[: n_env // 2, zc] += 0.3
    b.set_state(q.reshape(-1), u.reshape(-1))
    worlds = [O.OracleWorld("c5", e) for e in range(n_env)]
    for e, w in enumerate(worlds):
        w.set_state(q[e], u[e])
    mixed = 0
    for st in range(steps):
        tau = np.stack([_torques(e, st, nj) for e in range(n_env)])
        for e, w in enumerate(worlds):
            w.set_joint_torques(tau[e])
            assert w.step(1) == 0
        b.step(s0.h, s0.gravity, torque=tau.reshape(-1))
        res = b.results()
        routed = int((res["n_contacts"] > 10).sum())
        mixed += 0 < routed < n_env
        qg, _ = b.get_state()
        for e, w in enumerate(worlds):
            assert res["n_contacts"][e] == len(w.contacts()[0]), (st, e)
            assert rel_err(qg[e], w.state()[0]) < 1e-8, (st, e)
    assert mixed > 0


def test_batch_counters_count_pcr_iterations():
    """nsd_batch_counters()[0] is the sum of linear_iterations over envs and Newton
    iterations (what bench.py's roofline numerator uses)."""
    b, s0 = _batch(12, "fp64")
    b.counters()
    b.step(s0.h, s0.gravity)
    res = b.results(with_iters=True)
    c = b.counters()
    its = res["stats"][:, :, 5].sum(axis=1)
    assert c["cr_iterations"] == int(its.sum())
    assert c["cr_iterations_x_contacts"] == int((its * res["n_contacts"]).sum())
    assert c["env_steps"] == 12
    b.profile(cycles=True, launch_timing=True)
    for _ in range(3):
        b.step(s0.h, s0.gravity)
    c = b.counters()
    assert 0 < c["cr_cycles"] < c["env_cycles"]
    assert c["timed_steps"] == 3 and c["warp_solver_ms"] > 0 and c["narrow_phase_ms"] > 0


def test_batch_flags_sticky_until_results():
    """An abort in an earlier step stays reported until nsd_batch_results clears it."""
    b, s0 = _batch(4, "fp64")
    q, u = b.get_state()
    u = u.copy()
    u[2, 0] = np.nan
    b.set_state(q.reshape(-1), u.reshape(-1))
    b.step(s0.h, s0.gravity)
    q1, u1 = b.get_state()
    u1 = u1.copy()
    u1[2, 0] = 0.0
    b.set_state(q1.reshape(-1), u1.reshape(-1))
    b.step(s0.h, s0.gravity)  # env 2 steps normally now
    assert b.results()["aborted"].tolist() == [False, False, True, False]
    b.step(s0.h, s0.gravity)
    assert not b.results()["aborted"].any()
