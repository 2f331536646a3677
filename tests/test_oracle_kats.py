"""Pins the CPU oracle (oracle/, the restatement of /root/reference/proj/src)
against the reference's own doctest cases, ported one-for-one where the case
exercises the Newton hot path. Each test names the reference case it ports.
Eigen-dependent test scaffolding (random SPD construction, LDLT oracle) is
replaced by numpy equivalents.
"""
import math

import numpy as np
import pytest

from oracle import oracle_py as O

MINMAP, FB = 0, 1


# ---------------------------------------------------------------- ncp (tests/test_ncp.cpp)
def test_fb_pythagorean_triple():  # test_ncp.cpp:11-14
    assert O.phi_n(3.0, 4.0, 1.0, FB)[0] == pytest.approx(2.0)


def test_fb_boundary():  # :16-19
    assert O.phi_n(0.0, 5.0, 1.0, FB)[0] == pytest.approx(0.0)


def test_minmap_branches():  # :21-30
    p = O.phi_n(2.0, 3.0, 1.0, MINMAP)
    assert p[0] == pytest.approx(2.0) and p[1] == 1.0 and p[2] == 0.0
    q = O.phi_n(5.0, 3.0, 1.0, MINMAP)
    assert q[0] == pytest.approx(3.0) and q[1] == 0.0 and q[2] == 1.0


@pytest.mark.parametrize("r", [0.1, 1.0, 10.0])
def test_fb_origin_subgradient(r):  # :32-39
    p = O.phi_n(0.0, 0.0, r, FB)
    assert p[0] == 0.0 and p[1] == 0.0 and p[2] == r


@pytest.mark.parametrize("kind", [MINMAP, FB])
@pytest.mark.parametrize("r", [0.1, 1.0, 10.0])
def test_ncp_root_set_grid(kind, r):  # :41-57
    n = 81
    for i in range(n):
        a = -2.0 + 4.0 * i / (n - 1)
        for j in range(n):
            b = -2.0 + 4.0 * j / (n - 1)
            root = abs(O.phi_n(a, b, r, kind)[0]) <= 1e-9
            comp = a >= -1e-9 and b >= -1e-9 and abs(a * b) <= 1e-9
            assert root == comp, (a, b, r, kind)


def test_fb_derivatives_fd():  # :59-81 (seeded numpy stream instead of mt19937(29))
    rng = np.random.default_rng(29)
    eps, tested = 1e-7, 0
    while tested < 1000:
        a, b = rng.uniform(-2, 2, 2)
        r = rng.uniform(0.1, 10.0)
        if a * a + b * b <= 1e-4:
            continue
        tested += 1
        p = O.phi_n(a, b, r, FB)
        fa = (O.phi_n(a + eps, b, r, FB)[0] - O.phi_n(a - eps, b, r, FB)[0]) / (2 * eps)
        fb = (O.phi_n(a, b + eps, r, FB)[0] - O.phi_n(a, b - eps, r, FB)[0]) / (2 * eps)
        assert p[1] == pytest.approx(fa, rel=1e-6, abs=1e-6)
        assert p[2] == pytest.approx(fb, rel=1e-6, abs=1e-6)


def test_friction_W_stick_minmap():  # :83-87
    assert O.friction_W(0.0, 2.0, 5.0, 1.0, MINMAP) == 0.0
    assert O.friction_W(1.0, 0.0, 5.0, 1.0, MINMAP) == 0.0
    assert O.friction_W(0.0, 0.0, 3.0, 0.5, MINMAP) == 0.0


def test_friction_W_cone_limit():  # :89-96
    assert O.friction_W(0.5, 5.0, 5.0, 1.0, MINMAP) == pytest.approx(0.1)
    assert O.friction_W(0.5, 5.0, 5.0, 1.0, FB) == pytest.approx(0.1)


def test_friction_W_fb_stick():  # :98-101
    assert O.friction_W(0.0, 2.0, 5.0, 1.0, FB) == pytest.approx(0.0, abs=1e-12)


def test_friction_W_caps():  # :103-109
    assert O.friction_W(0.0, 0.0, 0.0, 1.0, MINMAP) == 0.0
    assert O.friction_W(1e-6, 0.0, 0.0, 1.0, MINMAP) == 1e12
    assert O.friction_W(0.0, 0.0, 0.0, 1.0, FB) == 1e12
    assert O.friction_W(0.0, 11.0, 5.0, 1.0, FB) == 1e12


def test_friction_W_nonnegative():  # :111-121
    rng = np.random.default_rng(31)
    for _ in range(5000):
        v, l = rng.uniform(0, 5, 2)
        m = rng.uniform(0, 5) + 1e-6
        r = rng.uniform(0.01, 10.0)
        for kind in (MINMAP, FB):
            assert O.friction_W(v, l, m, r, kind) >= 0.0


# ---------------------------------------------------------------- solvers (tests/test_solvers.cpp)
def _random_spd(n, rng):
    a = rng.standard_normal((n, n))
    return a @ a.T + 0.1 * np.eye(n)


@pytest.mark.parametrize("method", [0, 1, 2, 3])
def test_identity_one_iteration(method):  # test_solvers.cpp:38-49
    b = np.array([1, -2, 3, 0.5])
    r = O.solve_linear(np.eye(4), b, method=method, max_it=10, tol=1e-12)
    assert np.linalg.norm(r["x"] - b) < 1e-12
    assert r["iters"] == 1
    assert len(r["hist"]) == r["iters"] + 1


def test_pcr_2x2():  # :51-59
    r = O.solve_linear([[4, 1], [1, 3]], [1, 2], method=3, max_it=10, tol=1e-14)
    assert r["x"][0] == pytest.approx(1 / 11, rel=1e-8)
    assert r["x"][1] == pytest.approx(7 / 11, rel=1e-8)


def test_pcr_singular_diagonal():  # :61-70
    r = O.solve_linear([[1, 0], [0, 0]], [1, 0], method=3, max_it=20, tol=1e-14)
    assert np.all(np.isfinite(r["x"]))
    assert r["x"][0] == pytest.approx(1.0, rel=1e-10)
    assert r["hist"][-1] < 1e-12


def test_pcr_precond_norm_monotone():  # :84-103
    rng = np.random.default_rng(5)
    for trial in range(50):
        n = 5 + trial
        m = _random_spd(n, rng)
        if trial % 3 == 0:
            w, v = np.linalg.eigh(m)
            w[0] = 0.0
            m = (v * w) @ v.T
        b = rng.uniform(-1, 1, n)
        r = O.solve_linear(m, b, method=3, max_it=2 * n, tol=0.0)
        ph = r["phist"]
        assert np.all(ph[1:] <= ph[:-1] + 1e-12)


@pytest.mark.parametrize("method", [2, 3])
def test_krylov_bound(method):  # :105-119
    rng = np.random.default_rng(9)
    for trial in range(10):
        n = 10 + 4 * trial
        m = _random_spd(n, rng)
        b = rng.uniform(-1, 1, n)
        direct = np.linalg.solve(m, b)
        r = O.solve_linear(m, b, method=method, max_it=2 * n, tol=1e-12)
        assert np.linalg.norm(r["x"] - direct) < 1e-8 * max(1.0, np.linalg.norm(direct))


@pytest.mark.parametrize("method", [0, 1])
def test_relaxation_contracts(method):  # :121-144
    rng = np.random.default_rng(13)
    n = 20
    m = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(m, 0.0)
    np.fill_diagonal(m, np.abs(m).sum(axis=1) + 1.0)
    sym = 0.5 * (m + m.T) + n * np.eye(n)
    b = rng.uniform(-1, 1, n)
    r = O.solve_linear(sym, b, method=method, max_it=200, tol=1e-10)
    assert r["hist"][-1] <= 1e-10
    assert np.all(r["hist"][1:] <= r["hist"][:-1] + 1e-12)


@pytest.mark.parametrize("method", [0, 1, 2, 3])
def test_consistent_start(method):  # :146-158
    rng = np.random.default_rng(17)
    m = _random_spd(6, rng)
    x0 = rng.uniform(-1, 1, 6)
    r = O.solve_linear(m, m @ x0, x0=x0, method=method, max_it=50, tol=1e-9)
    assert np.linalg.norm(r["x"] - x0) < 1e-12
    assert r["iters"] == 0


# ---------------------------------------------------------------- linalg (tests/test_linalg.cpp)
def test_svd3_identity_scale():  # test_linalg.cpp:96-101
    _, s, _ = O.svd3(np.eye(3))
    assert np.linalg.norm(s - 1) < 1e-12
    _, s, _ = O.svd3(2 * np.eye(3))
    assert np.linalg.norm(s - 2) < 1e-12


def test_svd3_inversion_on_s3():  # :103-113
    f = np.diag([1.0, 1.0, -1.0])
    u, s, v = O.svd3(f)
    assert np.linalg.det(u) == pytest.approx(1.0)
    assert np.linalg.det(v) == pytest.approx(1.0)
    assert s[2] == pytest.approx(-1.0)
    assert s[0] >= s[1]
    assert np.linalg.norm(u @ np.diag(s) @ v.T - f) < 1e-10


def test_svd3_random_reconstruction():  # :115-131
    rng = np.random.default_rng(3)
    for trial in range(1000):
        f = rng.standard_normal((3, 3))
        if trial % 5 == 0:
            f[:, 1] = f[:, 0] * 1e-7
        u, s, v = O.svd3(f)
        assert np.linalg.det(u) == pytest.approx(1.0, rel=1e-9)
        assert np.linalg.det(v) == pytest.approx(1.0, rel=1e-9)
        scale = max(1.0, np.linalg.norm(f))
        assert np.linalg.norm(u @ np.diag(s) @ v.T - f) / scale < 1e-10
        assert s[0] >= s[1] >= abs(s[2])


def test_project_psd3_pd_unchanged():  # :133-137
    m = np.array([[4, 1, 0], [1, 3, 0.5], [0, 0.5, 2]], float)
    assert np.linalg.norm(O.project_psd3(m) - m) < 1e-12


def test_project_psd3_clamps():  # :139-145
    p = O.project_psd3(np.diag([1.0, -2.0, 3.0]))
    ev = np.linalg.eigvalsh(p)
    assert ev.min() == pytest.approx(3e-10, rel=1e-5)
    assert ev.max() == pytest.approx(3.0)


def test_project_psd3_rank1():  # :147-159
    rng = np.random.default_rng(11)
    for _ in range(100):
        v = rng.standard_normal(3)
        m = np.outer(v, v)
        p = O.project_psd3(m)
        ev = np.linalg.eigvalsh(p)
        assert ev.min() >= -1e-18
        assert ev.min() == pytest.approx(1e-10 * v @ v, rel=1e-5)
        assert np.linalg.norm(p - m) <= 1e-9 * max(1.0, np.linalg.norm(m))


def test_sym_eig3_matches_numpy():  # restated SelfAdjointEigenSolver (Appendix B)
    rng = np.random.default_rng(19)
    for _ in range(2000):
        a = rng.standard_normal((3, 3))
        m = a + a.T
        vals, vecs, rc = O.sym_eig3(m)
        assert rc == 0
        assert np.allclose(vals, np.linalg.eigvalsh(m), rtol=1e-12, atol=1e-12)
        assert np.linalg.norm(vecs @ np.diag(vals) @ vecs.T - m) < 1e-12 * max(1, np.linalg.norm(m))
        assert np.all(np.diff(vals) >= 0)


def test_inverse3_and_det3():
    rng = np.random.default_rng(23)
    for _ in range(200):
        m = rng.standard_normal((3, 3))
        assert O.det3(m) == pytest.approx(np.linalg.det(m), rel=1e-10, abs=1e-12)
        assert np.allclose(O.inverse3(m) @ m, np.eye(3), atol=1e-8)


# ---------------------------------------------------------------- constraints (tests/test_constraints.cpp)
def test_tangent_basis_axis_aligned():  # test_constraints.cpp:83-93
    d1, d2 = O.tangent_basis([0, 0, 1.0])
    assert np.linalg.norm(d1 - [1, 0, 0]) < 1e-15 and np.linalg.norm(d2 - [0, 1, 0]) < 1e-15
    d1, d2 = O.tangent_basis([1.0, 0, 0])
    assert abs(d1[0]) < 1e-15 and abs(d2[0]) < 1e-15 and abs(np.linalg.norm(d1) - 1) < 1e-15


def test_tangent_basis_random():  # :95-109
    rng = np.random.default_rng(37)
    for _ in range(20000):
        n = rng.standard_normal(3)
        if np.linalg.norm(n) < 1e-6:
            continue
        n /= np.linalg.norm(n)
        d1, d2 = O.tangent_basis(n)
        e1, e2 = O.tangent_basis(n)
        assert np.array_equal(d1, e1) and np.array_equal(d2, e2)
        assert abs(np.cross(d1, d2) @ n - 1.0) < 1e-12


def test_r_factor():  # :111-125
    m, h = 2.0, 0.01
    assert O.r_factor(1 / m, h, 0, 2) == pytest.approx(h * h / m)
    assert O.r_factor(1 / m, h, 0, 2) == pytest.approx(5e-5)
    assert O.r_factor(1 / m, h, 1, 2) == pytest.approx(5e-3)
    assert O.r_factor(0.7, h, 0, 0) == 1.0
    assert O.r_factor(0.7, h, 0, 1) == h * h
    assert O.r_factor(0.7, h, 1, 1) == h
    assert O.r_factor(0.0, h, 0, 2) == h * h


# ---------------------------------------------------------------- materials (tests/test_materials.cpp)
REST = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def test_nh_gradient_special():  # test_materials.cpp:65-74
    assert np.linalg.norm(O.nh_gradient([2, 1, 1], [1, 0, 1]) - [4, 2, 2]) < 1e-14
    assert np.linalg.norm(O.nh_gradient([1, 1, 1], [3, 0, 1]) - [6, 6, 6]) < 1e-14


def test_lame_rest_stress_free():  # :76-86
    c1, d1, alpha = O.lame(1e5, 0.45)
    mu, lam = 1e5 / 2.9, 1e5 * 0.45 / (1.45 * 0.1)
    assert mu == pytest.approx(3.448e4, rel=1e-3) and lam == pytest.approx(3.103e5, rel=1e-3)
    assert c1 == pytest.approx(0.5 * mu) and d1 == pytest.approx(0.5 * lam) and alpha == pytest.approx(1 + mu / lam)
    assert np.linalg.norm(O.nh_gradient([1, 1, 1], [c1, d1, alpha])) < 1e-10


def test_lame_edges():  # :88-95
    c1, d1, alpha = O.lame(1e5, 0.0)
    assert d1 == 0.0 and alpha == 1.0
    for y, nu in ((1e5, 0.4999), (1e5, 0.5), (-1.0, 0.3)):
        with pytest.raises(ValueError):
            O.lame(y, nu)


def test_nh_hessian_rest():  # :97-112
    h = O.nh_hessian([1, 1, 1], [2, 3, 1])
    expect = np.array([[5, 3, 3], [3, 5, 3], [3, 3, 5]], float)
    assert np.linalg.norm(h - 2 * expect) < 1e-14
    assert np.linalg.norm(O.nh_hessian([1.3, 0.8, 1.1], [2, 0, 1]) - 4 * np.eye(3)) < 1e-14


def test_nh_derivatives_fd():  # :114-133
    rng = np.random.default_rng(47)
    mat = O.lame(2e4, 0.3)
    eps = 1e-6
    for _ in range(300):
        s = rng.uniform(0.4, 1.8, 3)
        g, hh = O.nh_gradient(s, mat), O.nh_hessian(s, mat)
        for i in range(3):
            sp, sm = s.copy(), s.copy()
            sp[i] += eps
            sm[i] -= eps
            fd = (O.nh_energy(sp, mat) - O.nh_energy(sm, mat)) / (2 * eps)
            assert g[i] == pytest.approx(fd, rel=1e-5, abs=1e-5)
            row = (O.nh_gradient(sp, mat) - O.nh_gradient(sm, mat)) / (2 * eps)
            assert np.allclose(hh[i], row, rtol=1e-5, atol=1e-4)


def test_compliance_identities():  # :135-154
    mat = O.lame(1e5, 0.45)
    ve = 1.0 / 6.0
    h = O.nh_hessian([1, 1, 1], mat)
    eb = O.compliance_block(ve, h)
    assert np.linalg.norm(eb @ (ve * h) - np.eye(3)) < 1e-8
    ep = O.compliance_block(1.0, np.diag([1.0, -2.0, 3.0]))
    assert np.linalg.eigvalsh(ep).min() > 0.0


def test_strain_jacobian_fd():  # :156-180
    rng = np.random.default_rng(53)
    dm_inv = np.linalg.inv((REST[1:] - REST[0]).T)
    eps = 1e-6

    def stretches(p):
        ds = (p[1:] - p[0]).T
        return O.strain_jacobian(dm_inv, ds @ dm_inv)[1]

    for _ in range(60):
        p = REST + rng.normal(0, 0.05, (4, 3))
        jac, _ = O.strain_jacobian(dm_inv, (p[1:] - p[0]).T @ dm_inv)
        for k in range(4):
            for d in range(3):
                pp, pm = p.copy(), p.copy()
                pp[k, d] += eps
                pm[k, d] -= eps
                fd = (stretches(pp) - stretches(pm)) / (2 * eps)
                assert np.allclose(jac[:, 3 * k + d], fd, rtol=2e-5, atol=2e-5)


def test_strain_jacobian_rotation_annihilation():  # :182-195
    p = REST * np.array([1.2, 0.9, 1.05])
    dm_inv = np.linalg.inv((REST[1:] - REST[0]).T)
    jac, _ = O.strain_jacobian(dm_inv, (p[1:] - p[0]).T @ dm_inv)
    axis = np.array([0.3, -0.5, 0.8])
    axis /= np.linalg.norm(axis)
    dq = np.concatenate([np.cross(axis, p[k]) for k in range(4)])
    assert np.linalg.norm(jac @ dq) < 1e-10


@pytest.mark.parametrize("model", [1, 0])
def test_force_matches_energy_gradient(model):  # :246-276
    rng = np.random.default_rng(61)
    eps = 1e-6
    for _ in range(20):
        p = REST + rng.normal(0, 0.02, (4, 3))
        dim, c, jac, _, _ = O.material_rows(model, 1e5, 0.45, REST, p)
        force = -jac[:dim].T @ c[:dim]
        for k in range(4):
            for d in range(3):
                pp, pm = p.copy(), p.copy()
                pp[k, d] += eps
                pm[k, d] -= eps
                up = O.material_rows(model, 1e5, 0.45, REST, pp)[4]
                um = O.material_rows(model, 1e5, 0.45, REST, pm)[4]
                assert force[3 * k + d] == pytest.approx(-(up - um) / (2 * eps), rel=1e-5, abs=1e-3)


def test_linear_strain_rest_and_stretch():  # :197-208
    dim, c, _, _, _ = O.material_rows(0, 1e5, 0.45, REST, REST)
    assert dim == 6 and np.linalg.norm(c) < 1e-12


# ---------------------------------------------------------------- bodies (tests/test_bodies.cpp)
def test_integrate_particle():  # test_bodies.cpp:116-122
    q, _, _ = O.body_step_kat(0, 1.0, np.eye(3), [0, 0, 0], [1, 0, 0], [0, 0, 0], 0.1)
    assert q[0] == pytest.approx(0.1)


def test_integrate_rigid_spin():  # :131-140
    q, _, _ = O.body_step_kat(1, 1.0, np.eye(3), [0, 0, 0, 1, 0, 0, 0], [0, 0, 0, 0, 0, math.pi], [0, 0, 0], 0.5)
    t = q[3:]
    assert abs(np.linalg.norm(t) - 1) < 1e-12
    assert t[0] == pytest.approx(0.786, rel=1e-3) and t[3] == pytest.approx(0.618, rel=1e-3)


def test_gravity_force():  # :149-155
    _, f, ut = O.body_step_kat(0, 2.0, np.eye(3), [0, 0, 0], [0, 0, 0], [0, 0, -9.8], 0.1)
    assert f[2] == pytest.approx(-19.6) and ut[2] == pytest.approx(-0.98)


def test_gyroscopic_torque():  # :157-170
    _, f, ut = O.body_step_kat(1, 1.0, np.diag([1.0, 2.0, 3.0]), [0, 0, 0, 1, 0, 0, 0], [0, 0, 0, 1, 1, 0],
                               [0, 0, 0], 0.1)
    assert f[3] == pytest.approx(0.0) and f[4] == pytest.approx(0.0) and f[5] == pytest.approx(-1.0)
    assert ut[5] == pytest.approx(-0.1 / 3.0)


# ---------------------------------------------------------------- SPEC newton examples
def test_spec_zero_rows_free_fall():
    """no constraints, 1 Newton iteration (undamped, t = 1): u equals u~ exactly."""
    w = O.OracleWorld("box_on_plane", 0)
    w.set_config(newton_iterations=1, step_fraction=1.0)
    q, u = w.state()
    q = q.copy()
    q[2] += 10.0  # far above the margin: no contacts, no rows
    w.set_state(q, u)
    assert w.step(1) == 0
    r = w.report()
    assert r["n_iterations"] == 1 and len(r["tel"]) == 0
    ut = u.copy()
    ut[2] += w.h * w.gravity()[2]  # unit mass, zero spin: u~ = u- + h g
    assert np.array_equal(w.state()[1], ut)