"""Known-answer tests of the reference that need a body state: collision
(tests/test_collision.cpp, all 9 cases), constraint rows and their
finite-difference gradients (tests/test_constraints.cpp:56-81,127-234), the body
layer (tests/test_bodies.cpp:37-110,124-129,142-147,172-203), CSR / spmv
(tests/test_linalg.cpp:10-94), solver diagonal preconditioner
(tests/test_solvers.cpp:72-82) and materials (tests/test_materials.cpp:47-63,
210-244, 278-320). Each test ports one reference TEST_CASE (file:line) against
the CPU oracle; the collision cases also run through the product's narrow phase
(nsd_scene_detect: the host/device code of csrc/nsd_collide.cuh that the batched
GPU step runs) and require the same contact list bit for bit.

Random inputs come from seeded numpy streams instead of std::mt19937 (the
reference checks properties, not particular draws).
"""
import json

import numpy as np
import pytest

from oracle import oracle_py as O

EYE9 = np.eye(3).ravel()
RIGID = 1


# ---------------------------------------------------------------- collision fixtures
class Fixture:
    """tests/test_collision.cpp:10-43: rigid unit-inertia bodies + attached shapes."""

    def __init__(self):
        self.pos, self.shapes, self.json_bodies = [], [], []

    def add_rigid(self, pos, shape, mass=1.0):
        b = len(self.pos)
        self.pos.append(np.asarray(pos, float))
        self.shapes.append(dict(shape, body=b))
        js = {"type": "rigid", "mass": mass, "inertia": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "position": list(pos)}
        if shape["kind"] == 1:
            js["shape"] = {"kind": "sphere", "radius": shape["radius"]}
        else:
            js["shape"] = {"kind": "box", "half_extents": list(shape["half_extents"])}
        self.json_bodies.append(js)
        return b

    def add_ground(self):
        self.shapes.append(dict(body=-1, kind=0, normal=(0, 0, 1), offset=0.0))
        self.json_bodies.append({"type": "static", "shape": {"kind": "halfspace", "normal": [0, 0, 1], "offset": 0}})

    def q(self):
        return np.concatenate([np.r_[p, 1.0, 0.0, 0.0, 0.0] for p in self.pos])

    def detect(self, u=None):
        n = len(self.pos)
        return O.detect([RIGID] * n, [1.0] * n, np.tile(EYE9, n), self.q(), self.shapes, u_predict=u)

    def gap(self, ib, db, i):
        n = len(self.pos)
        g, _ = O.contact_gap_row([RIGID] * n, self.q(), int(ib[i, 0]), db[i, 0:3], int(ib[i, 1]), db[i, 3:6],
                                 db[i, 6:9], db[i, 15])
        return g

    def product_detect(self):
        """The product's narrow phase on the same fixture (zero gravity, so the predicted
        velocity is zero as in the reference fixture's detect(state, shapes, 0, h))."""
        from paper_1907_04587_b200 import World

        doc = {"timestep": 0.0083, "gravity": [0, 0, 0], "bodies": self.json_bodies}
        w = World(json_text=json.dumps(doc))
        try:
            return w.detect()
        finally:
            w.close()


def sphere(r):
    return dict(kind=1, radius=r)


def box(he):
    return dict(kind=2, half_extents=tuple(he))


def _same_as_product(f, ib, db):
    """Product narrow phase: same count, order, bodies (static shapes are world, -1),
    features, and bit-identical geometry, thickness and mu."""
    pib, pdb = f.product_detect()
    assert np.array_equal(pib[:, :3], ib[:, :3])
    assert np.array_equal(pdb[:, :17], db[:, :17])


def test_sphere_above_margin_no_contact():  # test_collision.cpp:60-65
    f = Fixture()
    f.add_ground()
    f.add_rigid((0, 0, 0.6), sphere(0.5))
    ib, db = f.detect()
    assert len(ib) == 0
    _same_as_product(f, ib, db)


def test_sphere_within_margin_one_contact():  # test_collision.cpp:67-75
    f = Fixture()
    f.add_ground()
    f.add_rigid((0, 0, 0.505), sphere(0.5))
    ib, db = f.detect()
    assert len(ib) == 1
    assert np.linalg.norm(db[0, 6:9] - (0, 0, 1)) < 1e-12
    assert f.gap(ib, db, 0) == pytest.approx(0.005)
    _same_as_product(f, ib, db)


def test_resting_box_four_equal_gap_corners():  # test_collision.cpp:77-87
    f = Fixture()
    f.add_ground()
    f.add_rigid((0, 0, 0.2), box([0.2] * 3))
    ib, db = f.detect()
    assert len(ib) == 4
    for i in range(4):
        assert abs(f.gap(ib, db, i)) <= 1e-12
        assert np.linalg.norm(db[i, 6:9] - (0, 0, 1)) < 1e-12
    _same_as_product(f, ib, db)


def test_stacked_boxes_eight_contacts():  # test_collision.cpp:89-105
    f = Fixture()
    f.add_ground()
    f.add_rigid((0, 0, 0.5), box([0.5] * 3))
    f.add_rigid((0, 0, 1.5), box([0.5] * 3))
    ib, db = f.detect()
    assert len(ib) == 8  # 4 ground corners + 4 between the boxes
    between = [i for i in range(8) if ib[i, 0] >= 0 and ib[i, 1] >= 0]
    assert len(between) == 4
    for i in between:
        assert abs(db[i, 8]) == pytest.approx(1.0)
        assert abs(f.gap(ib, db, i)) <= 1e-12
    _same_as_product(f, ib, db)


def test_sphere_sphere_and_sphere_box():  # test_collision.cpp:107-122
    f = Fixture()
    f.add_rigid((0, 0, 0), sphere(0.5))
    f.add_rigid((1.005, 0, 0), sphere(0.5))
    ib, db = f.detect()
    assert len(ib) == 1
    assert f.gap(ib, db, 0) == pytest.approx(0.005)
    _same_as_product(f, ib, db)
    g = Fixture()
    g.add_rigid((0, 0, 0), box([0.5] * 3))
    g.add_rigid((1.004, 0, 0), sphere(0.5))
    ib, db = g.detect()
    assert len(ib) == 1
    assert g.gap(ib, db, 0) == pytest.approx(0.004)
    _same_as_product(g, ib, db)


def test_emitted_gaps_within_margin_unit_normals():  # test_collision.cpp:124-137
    f = Fixture()
    f.add_ground()
    f.add_rigid((0.1, 0, 0.199), box([0.2] * 3))
    f.add_rigid((0.35, 0.1, 0.6), box([0.2] * 3))
    f.add_rigid((-0.3, 0, 0.3), sphere(0.3))
    ib, db = f.detect()
    assert len(ib) > 0
    for i in range(len(ib)):
        n, d1, d2 = db[i, 6:9], db[i, 9:12], db[i, 12:15]
        assert f.gap(ib, db, i) <= 0.01 + 1e-12
        assert abs(np.linalg.norm(n) - 1.0) < 1e-12
        assert abs(np.dot(np.cross(d1, d2), n) - 1.0) < 1e-12
    _same_as_product(f, ib, db)


def _exchange_fixtures():
    f = Fixture()
    f.add_rigid((0, 0, 0.5), box([0.5] * 3))
    f.add_rigid((0.2, 0.1, 1.5), box([0.5] * 3))
    g = Fixture()
    g.add_rigid((0.2, 0.1, 1.5), box([0.5] * 3))
    g.add_rigid((0, 0, 0.5), box([0.5] * 3))
    return f, g


def test_detection_under_pair_exchange_same_count():  # test_collision.cpp:139-163 (REQUIRE part)
    f, g = _exchange_fixtures()
    fi, fd = f.detect()
    gi, gd = g.detect()
    assert len(fi) == len(gi) > 0
    _same_as_product(f, fi, fd)
    _same_as_product(g, gi, gd)


@pytest.mark.xfail(strict=True, reason=(
    "reference inconsistency: the two boxes touch exactly, so the face axes of both boxes tie at separation 0 and "
    "box_box keeps the first (collision.cpp:180-190, 'sep > best_sep + 1e-12'): exchanging the pair swaps the "
    "reference face, and the emitted incident corner differs ((-0.3,-0.4,1) with +z vs (0.5,0.5,1) with -z). "
    "collision.cpp as written fails this reference case; the reference does not build here (SURVEY §0), so its "
    "suite never ran. The oracle and the product agree with each other bit for bit in both orders."))
def test_detection_symmetric_under_pair_exchange():  # test_collision.cpp:139-163 (CHECK(found) part)
    f, g = _exchange_fixtures()
    fi, fd = f.detect()
    gi, gd = g.detect()

    def world_a(fx, ib, db, i):  # attach_world_point of the a side (identity orientations)
        return fx.pos[ib[i, 0]] + db[i, 0:3]

    for i in range(len(fi)):
        assert any(np.linalg.norm(world_a(f, fi, fd, i) - world_a(g, gi, gd, j)) < 1e-12
                   and np.linalg.norm(fd[i, 6:9] - gd[j, 6:9]) < 1e-12 for j in range(len(gi)))


def test_identical_state_identical_ordered_list():  # test_collision.cpp:165-182
    f = Fixture()
    f.add_ground()
    f.add_rigid((0, 0, 0.2), box([0.2] * 3))
    f.add_rigid((0.15, 0.21, 0.6), box([0.2] * 3))
    a_i, a_d = f.detect()
    b_i, b_d = f.detect(u=np.zeros(12))
    assert np.array_equal(a_i, b_i) and np.array_equal(a_d, b_d)
    _same_as_product(f, a_i, a_d)


def test_approaching_bodies_predictive_contact():  # test_collision.cpp:184-195
    f = Fixture()
    f.add_ground()
    b = f.add_rigid((0, 0, 0.55), sphere(0.5))
    u = np.zeros(6)
    u[6 * b + 2] = -10.0  # gap 0.05 > margin, closing at 10 m/s covers it within one step
    ib, _ = f.detect(u=u)
    assert len(ib) == 1
    assert len(f.detect()[0]) == 0


# ---------------------------------------------------------------- constraint rows
def _q2(p0, p1, t0=(1, 0, 0, 0), t1=(1, 0, 0, 0)):
    return np.r_[p0, t0, p1, t1].astype(float)


def _unit_quat(rng):
    q = rng.normal(size=4)
    return q / np.linalg.norm(q)


def test_contact_gap_sign_convention():  # test_constraints.cpp:56-81
    q = np.r_[0, 0, 1, 1, 0, 0, 0.0]
    g, _ = O.contact_gap_row([RIGID], q, 0, (0, 0, 0), -1, (0, 0, 0), (0, 0, 1), 0.1)
    assert g == pytest.approx(0.9)
    g, _ = O.contact_gap_row([RIGID], np.r_[0, 0, 0, 1, 0, 0, 0.0], 0, (0, 0, 0), -1, (0, 0, 0), (0, 0, 1), 0.0)
    assert g == pytest.approx(0.0)
    g, _ = O.contact_gap_row([RIGID], np.r_[0, 0, 0.05, 1, 0, 0, 0.0], 0, (0, 0, 0), -1, (0, 0, 0), (0, 0, 1), 0.1)
    assert g == pytest.approx(-0.05)


def test_fixed_point_rows_vanish_at_shared_point():  # test_constraints.cpp:127-139
    q = _q2((0, 0, 0), (1, 0, 0))
    vals, _, _ = O.joint_rows(0, [RIGID, RIGID], 0, 1, q, (0.5, 0, 0), (0, 0, 1), q)
    assert len(vals) == 3
    assert np.all(np.abs(vals) < 1e-15)


def test_fixed_point_sees_separation_along_x():  # test_constraints.cpp:141-155
    q = _q2((0, 0, 0), (1, 0, 0))
    delta = 0.03
    vals, _, _ = O.joint_rows(0, [RIGID, RIGID], 0, 1, q, (0.5, 0, 0), (0, 0, 1), _q2((0, 0, 0), (1 + delta, 0, 0)))
    assert vals[0] == pytest.approx(-delta)
    assert abs(vals[1]) < 1e-15


def test_bend_spring_stiffness_maps_to_compliance():  # test_constraints.cpp:157-169
    q = _q2((0, 0, 0), (1, 0, 0))
    vals, comp, _ = O.joint_rows(3, [RIGID, RIGID], 0, 1, q, (0.5, 0, 0), (1, 0, 0), q, stiffness=250.0)
    assert len(vals) == 2
    assert np.allclose(comp, 0.004, rtol=1e-12)


def _fd_rows(rows_at, q, types, eps=1e-6):
    """Central differences of row values along each generalized velocity direction
    integrated into the coordinates (test_constraints.cpp:31-53)."""
    _, _, ndof, _ = O.layout(types)
    cols = []
    for dof in range(ndof):
        du = np.zeros(ndof)
        du[dof] = 1.0
        qp = O.integrate_state(types, q, du, eps)
        qm = O.integrate_state(types, q, -du, eps)
        cols.append((rows_at(qp) - rows_at(qm)) / (2 * eps))
    return np.array(cols).T


_PRISMATIC_FD = pytest.mark.xfail(strict=True, reason=(
    "reference inconsistency: the prismatic translation rows use t1, t2 = tangent_basis(axis) "
    "(constraints.cpp:183-185), which is rebuilt from a world axis and so does not rotate rigidly with body a, "
    "but their Jacobian adds t x d on body a's angular dofs as if it did (:195-196). The row values match; the "
    "angular-a columns of the two translation rows differ from central differences by O(1). The oracle follows "
    "constraints.cpp (and the device the oracle); the reference does not build here, so its suite never ran."))


@pytest.mark.parametrize("trial", [t if t % 4 != 2 else pytest.param(t, marks=_PRISMATIC_FD) for t in range(12)])
def test_joint_row_gradients_match_fd(trial):  # test_constraints.cpp:171-199
    rng = np.random.default_rng(41 + trial)
    kind = trial % 4  # FixedPoint, Revolute, Prismatic, BendSpring
    types = [RIGID, RIGID]
    qb = _q2((0, 0, 0), (1, 0, 0))
    axis = np.array([0.3, 0.5, 1.0]) / np.linalg.norm([0.3, 0.5, 1.0])
    stiff = 100.0 if kind == 3 else 0.0
    up = lambda: rng.uniform(-0.3, 0.3, 3)
    q = _q2(up(), np.r_[1.0, 0, 0] + up(), _unit_quat(rng), _unit_quat(rng))
    vals, _, jac = O.joint_rows(kind, types, 0, 1, qb, (0.5, 0, 0.1), axis, q, stiffness=stiff)
    fd = _fd_rows(lambda qq: O.joint_rows(kind, types, 0, 1, qb, (0.5, 0, 0.1), axis, qq, stiffness=stiff)[0], q,
                  types)
    assert np.allclose(jac, fd, rtol=1e-5, atol=1e-7)


def test_prismatic_rows_fd_except_body_a_angular():  # test_constraints.cpp:171-199, prismatic trials
    """The prismatic rows match central differences everywhere except the translation rows'
    angular-a block (see _PRISMATIC_FD): values, linear dofs, body b and the three axis rows."""
    for trial in (2, 6, 10):
        rng = np.random.default_rng(41 + trial)
        types = [RIGID, RIGID]
        qb = _q2((0, 0, 0), (1, 0, 0))
        axis = np.array([0.3, 0.5, 1.0]) / np.linalg.norm([0.3, 0.5, 1.0])
        up = lambda: rng.uniform(-0.3, 0.3, 3)
        q = _q2(up(), np.r_[1.0, 0, 0] + up(), _unit_quat(rng), _unit_quat(rng))
        _, _, jac = O.joint_rows(2, types, 0, 1, qb, (0.5, 0, 0.1), axis, q)
        fd = _fd_rows(lambda qq: O.joint_rows(2, types, 0, 1, qb, (0.5, 0, 0.1), axis, qq)[0], q, types)
        mask = np.ones_like(jac, bool)
        mask[:2, 3:6] = False
        assert np.allclose(jac[mask], fd[mask], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("trial", range(20))
def test_contact_rows_match_fd_of_gap(trial):  # test_constraints.cpp:201-234
    rng = np.random.default_rng(43 + trial)
    types = [RIGID, RIGID]
    up = lambda: rng.uniform(-0.2, 0.2, 3)
    q = _q2(up() + (0, 0, 1.0), up() - (0, 0, 1.0), _unit_quat(rng), _unit_quat(rng))
    n = rng.normal(size=3)
    n /= np.linalg.norm(n)
    la, lb = up(), up()
    _, row = O.contact_gap_row(types, q, 0, la, 1, lb, n)
    fd = _fd_rows(lambda qq: np.array([O.contact_gap_row(types, qq, 0, la, 1, lb, n)[0]]), q, types)[0]
    assert np.allclose(row, fd, rtol=1e-5, atol=1e-7)


# ---------------------------------------------------------------- bodies
def test_layout_offsets_sum_to_totals():  # test_bodies.cpp:37-48
    do, co, ndof, ncoord = O.layout([0, 1, 0, 1])
    assert ndof == 3 + 6 + 3 + 6 and ncoord == 3 + 7 + 3 + 7
    assert do.tolist() == [0, 3, 9, 12] and co.tolist() == [0, 3, 10, 13]


def test_quat_rate_identity_half_omega():  # test_bodies.cpp:50-59
    w = np.array([0.3, -0.2, 0.9])
    r = O.quat_rate([1, 0, 0, 0], w)
    assert r[0] == pytest.approx(0.0) and np.allclose(r[1:], 0.5 * w)


def _qmul(a, b):
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def test_quat_rate_matches_quaternion_product():  # test_bodies.cpp:61-84
    r = O.quat_rate([0, 1, 0, 0], [0, 0, 1])
    assert np.allclose(r, [0, 0, 0.5, 0])
    rng = np.random.default_rng(1)
    for _ in range(100):
        t = rng.normal(size=4)
        t /= np.linalg.norm(t)
        w = rng.normal(size=3)
        r2 = 0.5 * _qmul(np.r_[0.0, w], t)
        assert np.linalg.norm(O.quat_rate(t, w) - r2) < 1e-12


def test_quat_rate_columns_orthogonal_to_theta():  # test_bodies.cpp:86-95
    rng = np.random.default_rng(23)
    for _ in range(200):
        t = rng.normal(size=4)
        t /= np.linalg.norm(t)
        for c in range(3):  # column c of Q(t) = 2 * rate(t, e_c)
            col = 2.0 * O.quat_rate(t, np.eye(3)[c])
            assert abs(np.dot(col, t)) < 1e-12


def test_integrate_rigid_at_rest_stays_put():  # test_bodies.cpp:124-129
    q0 = np.r_[0, 0, 0, 1, 0, 0, 0.0]
    assert np.array_equal(O.integrate_state([RIGID], q0, np.zeros(6), 0.1), q0)


def test_integrate_rejects_nonpositive_h():  # bodies.cpp:80 (the invalid_argument of integrate_coordinates)
    with pytest.raises(ValueError):
        O.integrate_state([RIGID], np.r_[0, 0, 0, 1, 0, 0, 0.0], np.zeros(6), 0.0)


def test_unconstrained_velocity_zero_force_unchanged():  # test_bodies.cpp:142-147
    q, u = np.zeros(3), np.array([1.0, 2.0, 3.0])
    _, _, ut = O.body_step_kat(0, 2.0, np.eye(3), q, u, (0, 0, 0), 0.1)
    assert np.array_equal(ut, u)


def test_free_rigid_body_preserves_momentum():  # test_bodies.cpp:172-181
    q = np.r_[0, 0, 0, 1, 0, 0, 0.0]
    u = np.array([1.0, -2.0, 0.5, 4.0, -1.0, 2.0])
    q1, _, ut = O.body_step_kat(1, 3.0, np.diag([0.2, 0.3, 0.4]), q, u, (0, 0, 0), 0.01, integrate_with_ut=True)
    assert np.array_equal(ut[:3], u[:3])
    assert abs(np.linalg.norm(q1[3:7]) - 1.0) < 1e-12


def test_block_mass_round_trip_and_inverse_quadratic():  # test_bodies.cpp:183-203
    types, masses = [0, 1], [2.0, 3.0]
    inert = np.r_[np.eye(3).ravel(), np.diag([1.0, 2.0, 3.0]).ravel()]
    q = np.r_[0, 0, 0, 0, 0, 0, 1, 0, 0, 0.0]
    v = np.random.default_rng(3).uniform(-1, 1, 9)
    mv, mi, quad = O.mass_kat(types, masses, inert, q, v, idx=[0, 6, 7, 8], val=[2.0, 1.0, 0.0, 1.0])
    assert np.linalg.norm(mi - v) < 1e-12
    assert quad == pytest.approx(4.0 / 2.0 + 1.0 / 1.0 + 0.0 + 1.0 / 3.0)


# ---------------------------------------------------------------- linalg (CSR / spmv)
def test_csr_sums_duplicates_orders_columns():  # test_linalg.cpp:10-19
    off, idx, val, valid = O.csr(2, 3, [(0, 2, 1.0), (0, 0, 2.0), (0, 2, 3.0), (1, 1, -1.0)])
    assert valid and len(val) == 3
    assert off.tolist() == [0, 2, 3] and idx.tolist() == [0, 2, 1]
    assert val[0] == 2.0 and val[1] == 4.0


def test_spmv_identity_and_zero():  # test_linalg.cpp:21-29
    x = np.array([1.0, 2.0, 3.0])
    ident = [(i, i, 1.0) for i in range(3)]
    assert np.array_equal(O.spmv(3, 3, ident, x), x)
    assert np.linalg.norm(O.spmv(3, 3, [], x)) == 0.0


def test_spmv_2x2_hand_and_symmetric_transpose():  # test_linalg.cpp:31-43
    a = [(0, 0, 4.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 3.0)]
    x = np.array([1.0, 2.0])
    y = O.spmv(2, 2, a, x)
    assert y.tolist() == pytest.approx([6.0, 7.0])
    assert np.array_equal(O.spmv(2, 2, a, x, mode=2), y)


def test_spmv_transpose_examples():  # test_linalg.cpp:45-58
    x = np.array([4.0, 5.0, 6.0])
    assert np.array_equal(O.spmv(3, 3, [(i, i, 1.0) for i in range(3)], x, mode=2), x)
    assert O.spmv(1, 3, [(0, 0, 1.0)], [5.0], mode=2).tolist() == [5.0, 0.0, 0.0]


def test_spmv_dimension_mismatch_throws():  # test_linalg.cpp:60-64
    ident = [(i, i, 1.0) for i in range(3)]
    with pytest.raises(ValueError):
        O.spmv(3, 3, ident, np.zeros(4))
    with pytest.raises(ValueError):
        O.spmv(3, 3, ident, np.zeros(2), mode=2)


def test_adjoint_identity_random_sparse():  # test_linalg.cpp:66-80
    rng = np.random.default_rng(42)
    for _ in range(50):
        rows, cols = rng.integers(1, 41, 2)
        t = [(int(rng.integers(rows)), int(rng.integers(cols)), float(rng.uniform(-2, 2))) for _ in range(2 * rows)]
        x, y = rng.uniform(-1, 1, cols), rng.uniform(-1, 1, rows)
        lhs = y @ O.spmv(rows, cols, t, x)
        rhs = O.spmv(rows, cols, t, y, mode=2) @ x
        assert lhs == pytest.approx(rhs, rel=1e-10, abs=1e-12)


def test_omp_spmv_matches_serial_bitwise():  # test_linalg.cpp:82-94
    rng = np.random.default_rng(7)
    n = 200
    t = [(int(rng.integers(n)), int(rng.integers(n)), float(rng.uniform(-1, 1))) for _ in range(3000)]
    x = rng.uniform(-1, 1, n)
    assert np.array_equal(O.spmv(n, n, t, x, mode=0), O.spmv(n, n, t, x, mode=1))


# ---------------------------------------------------------------- solvers
def test_diagonal_preconditioner_entries():  # test_solvers.cpp:72-82
    assert np.array_equal(O.diag_precond(np.eye(3)), np.ones(3))
    inv = O.diag_precond(np.diag([4.0, 2.0]))
    assert inv[0] == 0.25 and inv[1] == 0.5
    assert O.diag_precond(np.diag([1.0, 0.0]))[1] == 1.0


# ---------------------------------------------------------------- materials
REST = np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], float)


def test_deformation_gradient_identities():  # test_materials.cpp:47-63
    assert np.linalg.norm(O.deformation_gradient(REST, REST) - np.eye(3)) < 1e-14
    f2 = O.deformation_gradient(REST, 2 * REST)
    assert np.linalg.norm(f2 - 2 * np.eye(3)) < 1e-14
    assert O.det3(f2) == pytest.approx(8.0)
    p = REST.reshape(4, 3).copy()
    p[:, 0] += 0.3 * p[:, 2]
    expect = np.eye(3)
    expect[0, 2] = 0.3
    assert np.linalg.norm(O.deformation_gradient(REST, p) - expect) < 1e-14


def _rotation(axis, angle):
    a = np.asarray(axis, float) / np.linalg.norm(axis)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(angle) * k + (1 - np.cos(angle)) * k @ k


def test_linear_strain_invariant_under_rotation():  # test_materials.cpp:210-217
    r = _rotation((1, 2, 3), 0.7)
    p = (REST.reshape(4, 3) @ r.T).ravel()
    _, c, _, _, _ = O.material_rows(0, 1e5, 0.45, REST, p)
    assert np.linalg.norm(c[:6]) < 1e-10


def test_linear_strain_jacobian_matches_fd():  # test_materials.cpp:219-244
    rng = np.random.default_rng(59)
    eps = 1e-6
    for _ in range(60):
        p = REST + rng.normal(0, 0.04, 12)
        _, _, jac, comp, _ = O.material_rows(0, 1e5, 0.45, REST, p)
        for j in range(12):
            pp, pm = p.copy(), p.copy()
            pp[j] += eps
            pm[j] -= eps
            cp, cm = O.material_rows(0, 1e5, 0.45, REST, pp)[1][:6], O.material_rows(0, 1e5, 0.45, REST, pm)[1][:6]
            # strain = K^-1 c / V_e = comp c (comp = K^-1 / V_e, materials.cpp:153); J = d strain / dq
            fd = comp @ (cp - cm) / (2 * eps)
            assert np.allclose(jac[:6, j], fd, rtol=2e-5, atol=1e-9)


def test_compliance_identity_for_assembled_blocks():  # test_materials.cpp:278-293
    rng = np.random.default_rng(67)
    checked = 0
    for _ in range(50):
        p = REST + rng.normal(0, 0.03, 12)
        f = O.deformation_gradient(REST, p)
        _, s, _ = O.svd3(f)
        h = O.nh_hessian(s, O.lame(1e5, 0.45))
        if np.linalg.eigvalsh(h).min() <= 0.0:
            continue  # the identity applies in the PD case
        vol = 1.0 / 6.0
        e = O.compliance_block(vol, h)
        assert np.linalg.norm(e @ (vol * h) - np.eye(3)) < 1e-8
        checked += 1
    assert checked > 0


def test_parallel_material_rows_equal_serial_bitwise():  # test_materials.cpp:295-320
    rng = np.random.default_rng(71)
    rest = np.concatenate([REST + np.tile([1.5 * i, 0, 0], 4) for i in range(64)])
    pos = rest + rng.normal(0, 0.05, rest.size)
    s = O.material_rows_many(1e5, 0.45, rest, pos, parallel=False)
    p = O.material_rows_many(1e5, 0.45, rest, pos, parallel=True)
    for a, b in zip(s, p):
        assert np.array_equal(a, b)
