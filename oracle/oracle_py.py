"""ORACLE — test infrastructure only.

ctypes wrapper over oracle/_build/liboracle.so, the CPU double-precision
restatement of the reference nsdyn solver (/root/reference/proj/src). Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
arm may import this module; the product path (paper_1907_04587_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_friction_W.restype = C.c_double
        _lib.orc_det3.restype = C.c_double
        _lib.orc_r_factor.restype = C.c_double
        _lib.orc_nh_energy.restype = C.c_double
        _lib.orc_world_create.restype = C.c_void_p
        _lib.orc_world_create.argtypes = [C.c_char_p, C.c_uint]
        for n in ("orc_world_destroy", "orc_world_dims", "orc_world_get_state", "orc_world_set_state",
                  "orc_world_topology", "orc_world_shapes", "orc_world_n_contacts", "orc_world_contacts",
                  "orc_world_prepare", "orc_world_newton", "orc_world_step", "orc_world_report",
                  "orc_world_get_config", "orc_world_set_config", "orc_world_h", "orc_world_gravity",
                  "orc_world_set_joint_torques", "orc_world_get_f_extra", "orc_world_joint_frames"):
            getattr(_lib, n).argtypes = None
        _lib.orc_world_h.restype = C.c_double
        _lib.orc_c5_bench.restype = C.c_double
        _lib.orc_action_torque.restype = C.c_double
        _lib.orc_contact_gap_row.restype = C.c_double
    return _lib


def dp(a):
    return a.ctypes.data_as(D)


def ip(a):
    return a.ctypes.data_as(I)


def m3(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(3, 3))


def _f64(a, n=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    assert n is None or a.size == n
    return a


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


# ---------------------------------------------------------------- state-level KAT helpers
def layout(types):
    t = _i32(types)
    do, co, tot = np.zeros(len(t), np.int32), np.zeros(len(t), np.int32), np.zeros(2, np.int32)
    lib().orc_layout(C.c_int(len(t)), ip(t), ip(do), ip(co), ip(tot))
    return do, co, int(tot[0]), int(tot[1])


def quat_rate(theta, omega):
    out = np.zeros(4)
    lib().orc_quat_rate(dp(_f64(theta, 4)), dp(_f64(omega, 3)), dp(out))
    return out


def integrate_state(types, q, u, h):
    """integrate_coordinates (bodies.cpp:78-86); raises ValueError on invalid input."""
    t, q = _i32(types), _f64(q).copy()
    if lib().orc_integrate_state(C.c_int(len(t)), ip(t), dp(q), dp(_f64(u)), C.c_double(h)):
        raise ValueError(lib().orc_last_error().decode())
    return q


def mass_kat(types, masses, inertias, q, v, idx=(), val=()):
    t = _i32(types)
    v = _f64(v)
    mv, mi = np.zeros(v.size), np.zeros(v.size)
    quad = C.c_double()
    ii, vv = _i32(idx), _f64(val)
    lib().orc_mass_kat(C.c_int(len(t)), ip(t), dp(_f64(masses)), dp(_f64(inertias)), dp(_f64(q)), dp(v), dp(mv),
                       dp(mi), C.c_int(ii.size), ip(ii), dp(vv), C.byref(quad))
    return mv, mi, quad.value


def detect(types, masses, inertias, q, shapes, u_predict=None, h=0.0083, margin=0.01, mu_default=0.5, cap=256):
    """detect (collision.cpp:239-297) on a fixture. shapes: list of dicts with body,
    kind (0 half-space, 1 sphere, 2 box), normal, offset, radius, half_extents,
    thickness, mu. Returns (ib, db) in orc_world_contacts' layout."""
    t = _i32(types)
    ns = len(shapes)
    sb = _i32([sh["body"] for sh in shapes])
    sk = _i32([sh["kind"] for sh in shapes])
    sp = _f64([list(sh.get("normal", (0, 0, 1))) + [sh.get("offset", 0.0), sh.get("radius", 0.5)]
               + list(sh.get("half_extents", (0.5, 0.5, 0.5))) + [sh.get("thickness", 0.0), sh.get("mu", -1.0), 0.0]
               for sh in shapes])
    ib, db = np.zeros((cap, 4), np.int32), np.zeros((cap, 22))
    up = _f64(u_predict) if u_predict is not None else None
    n = lib().orc_detect(C.c_int(len(t)), ip(t), dp(_f64(masses)), dp(_f64(inertias)), dp(_f64(q)),
                         dp(up) if up is not None else None, C.c_int(ns), ip(sb), ip(sk), dp(sp), C.c_double(h),
                         C.c_double(margin), C.c_double(mu_default), C.c_int(cap), ip(ib), dp(db))
    if n < 0:
        raise ValueError(lib().orc_last_error().decode())
    return ib[:n], db[:n]


def contact_gap_row(types, q, a_body, a_local, b_body, b_local, normal, thickness=0.0):
    t = _i32(types)
    _, _, ndof, _ = layout(t)
    row = np.zeros(ndof)
    g = lib().orc_contact_gap_row(C.c_int(len(t)), ip(t), dp(_f64(q)), C.c_int(a_body), dp(_f64(a_local, 3)),
                                  C.c_int(b_body), dp(_f64(b_local, 3)), dp(_f64(normal, 3)), C.c_double(thickness),
                                  dp(row))
    return g, row


def joint_rows(kind, types, body_a, body_b, q_bind, anchor, axis, q_eval, compliance=0.0, stiffness=0.0):
    """bind_joint at q_bind, joint_rows at q_eval: (values, compliances, dense Jacobian)."""
    t = _i32(types)
    _, _, ndof, _ = layout(t)
    vals, comp, jac = np.zeros(5), np.zeros(5), np.zeros(5 * ndof)
    n = lib().orc_joint_rows(C.c_int(kind), C.c_double(compliance), C.c_double(stiffness), C.c_int(len(t)), ip(t),
                             C.c_int(body_a), C.c_int(body_b), dp(_f64(q_bind)), dp(_f64(anchor, 3)),
                             dp(_f64(axis, 3)), dp(_f64(q_eval)), dp(vals), dp(comp), dp(jac))
    if n < 0:
        raise ValueError(lib().orc_last_error().decode())
    return vals[:n], comp[:n], jac[:n * ndof].reshape(n, ndof)


def csr(rows, cols, trips):
    r = _i32([x[0] for x in trips])
    c = _i32([x[1] for x in trips])
    v = _f64([x[2] for x in trips])
    off, idx, val, valid = np.zeros(rows + 1, np.int32), np.zeros(max(len(trips), 1), np.int32), \
        np.zeros(max(len(trips), 1)), C.c_int()
    n = lib().orc_csr(C.c_int(rows), C.c_int(cols), C.c_int(len(trips)), ip(r), ip(c), dp(v), ip(off), ip(idx),
                      dp(val), C.byref(valid))
    if n < 0:
        raise ValueError(lib().orc_last_error().decode())
    return off, idx[:n], val[:n], bool(valid.value)


def spmv(rows, cols, trips, x, mode=0):
    """mode 0 spmv (OpenMP rows), 1 spmv_serial, 2 spmv_transpose; ValueError on a dimension mismatch."""
    r = _i32([t[0] for t in trips]) if trips else np.zeros(1, np.int32)
    c = _i32([t[1] for t in trips]) if trips else np.zeros(1, np.int32)
    v = _f64([t[2] for t in trips]) if trips else np.zeros(1)
    x = _f64(x)
    y = np.zeros(cols if mode == 2 else rows)
    if lib().orc_spmv(C.c_int(rows), C.c_int(cols), C.c_int(len(trips)), ip(r), ip(c), dp(v), C.c_int(mode), dp(x),
                      C.c_int(x.size), dp(y)):
        raise ValueError(lib().orc_last_error().decode())
    return y


def diag_precond(dense):
    a = np.asarray(dense, dtype=np.float64)
    n = a.shape[0]
    ii, jj = np.nonzero(a)
    out = np.zeros(n)
    lib().orc_diag_precond(C.c_int(n), C.c_int(len(ii)), ip(_i32(ii)), ip(_i32(jj)), dp(_f64(a[ii, jj])), dp(out))
    return out


def deformation_gradient(rest, pos):
    f = np.zeros(9)
    lib().orc_deformation_gradient(dp(_f64(rest, 12)), dp(_f64(pos, 12)), dp(f))
    return f.reshape(3, 3)


def material_rows_many(young, poisson, rest, pos, parallel):
    rest, pos = _f64(rest), _f64(pos)
    ne = rest.size // 12
    c, jac, comp = np.zeros(3 * ne), np.zeros(36 * ne), np.zeros(9 * ne)
    lib().orc_material_rows_many(C.c_int(ne), C.c_double(young), C.c_double(poisson), dp(rest), dp(pos),
                                 C.c_int(1 if parallel else 0), dp(c), dp(jac), dp(comp))
    return c.reshape(ne, 3), jac.reshape(ne, 3, 12), comp.reshape(ne, 3, 3)


# ---------------------------------------------------------------- KAT helpers
def phi_n(c, lam, r, kind):
    out = np.zeros(3)
    lib().orc_phi_n(C.c_double(c), C.c_double(lam), C.c_double(r), C.c_int(kind), dp(out))
    return out


def friction_W(vt, lf, mln, r, kind):
    return lib().orc_friction_W(C.c_double(vt), C.c_double(lf), C.c_double(mln), C.c_double(r), C.c_int(kind))


def svd3(f):
    f = m3(f)
    u, v, s = np.zeros((3, 3)), np.zeros((3, 3)), np.zeros(3)
    lib().orc_svd3(dp(f), dp(u), dp(s), dp(v))
    return u, s, v


def project_psd3(m):
    m = m3(m)
    out = np.zeros((3, 3))
    lib().orc_project_psd3(dp(m), dp(out))
    return out


def sym_eig3(m):
    m = m3(m)
    vals, vecs = np.zeros(3), np.zeros((3, 3))
    rc = lib().orc_sym_eig3(dp(m), dp(vals), dp(vecs))
    return vals, vecs, rc


def inverse3(m):
    m = m3(m)
    out = np.zeros((3, 3))
    lib().orc_inverse3(dp(m), dp(out))
    return out


def det3(m):
    return lib().orc_det3(dp(m3(m)))


def tangent_basis(n):
    n = np.ascontiguousarray(n, dtype=np.float64)
    d1, d2 = np.zeros(3), np.zeros(3)
    lib().orc_tangent_basis(dp(n), dp(d1), dp(d2))
    return d1, d2


def r_factor(emd, h, row_class, strat):
    return lib().orc_r_factor(C.c_double(emd), C.c_double(h), C.c_int(row_class), C.c_int(strat))


def lame(young, poisson):
    out = np.zeros(3)
    rc = lib().orc_lame(C.c_double(young), C.c_double(poisson), dp(out))
    if rc:
        raise ValueError(lib().orc_last_error().decode())
    return out


def nh_gradient(s, mat):
    s, mat, out = np.ascontiguousarray(s, float), np.ascontiguousarray(mat, float), np.zeros(3)
    lib().orc_nh_gradient(dp(s), dp(mat), dp(out))
    return out


def nh_hessian(s, mat):
    s, mat, out = np.ascontiguousarray(s, float), np.ascontiguousarray(mat, float), np.zeros((3, 3))
    lib().orc_nh_hessian(dp(s), dp(mat), dp(out))
    return out


def nh_energy(s, mat):
    s, mat = np.ascontiguousarray(s, float), np.ascontiguousarray(mat, float)
    return lib().orc_nh_energy(dp(s), dp(mat))


def compliance_block(vol, h, project=True, diag=False):
    h, out = m3(h), np.zeros((3, 3))
    lib().orc_compliance_block(C.c_double(vol), dp(h), C.c_int(int(project)), C.c_int(int(diag)), dp(out))
    return out


def material_rows(model, young, poisson, rest, pos):
    rest = np.ascontiguousarray(rest, float).reshape(12)
    pos = np.ascontiguousarray(pos, float).reshape(12)
    c, jac, comp, e = np.zeros(6), np.zeros((6, 12)), np.zeros((6, 6)), np.zeros(1)
    dim = lib().orc_material_rows(C.c_int(model), C.c_double(young), C.c_double(poisson), dp(rest), dp(pos),
                                  dp(c), dp(jac), dp(comp), dp(e))
    if dim < 0:
        raise ValueError(lib().orc_last_error().decode())
    return dim, c, jac, comp, float(e[0])


def strain_jacobian(dm_inv, f):
    dm_inv, f = m3(dm_inv), m3(f)
    out, s = np.zeros((3, 12)), np.zeros(3)
    lib().orc_strain_jacobian(dp(dm_inv), dp(f), dp(out), dp(s))
    return out, s


def solve_linear(dense, b, x0=None, method=3, max_it=40, tol=1e-10, precond=1):
    a = np.asarray(dense, float)
    n = a.shape[0]
    r, c = np.nonzero(a)
    rows, cols = np.ascontiguousarray(r, np.int32), np.ascontiguousarray(c, np.int32)
    vals = np.ascontiguousarray(a[r, c])
    b = np.ascontiguousarray(b, float)
    x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, float)
    x = np.zeros(n)
    hist, phist = np.zeros(max_it + 2), np.zeros(max_it + 2)
    hl, pl, it, bd = (C.c_int() for _ in range(4))
    rc = lib().orc_solve_linear(C.c_int(n), C.c_int(len(vals)), ip(rows), ip(cols), dp(vals), dp(b), dp(x0),
                                C.c_int(method), C.c_int(max_it), C.c_double(tol), C.c_int(precond), dp(x),
                                dp(hist), C.byref(hl), dp(phist), C.byref(pl), C.byref(it), C.byref(bd))
    if rc:
        raise ValueError(lib().orc_last_error().decode())
    return dict(x=x, hist=hist[:hl.value].copy(), phist=phist[:pl.value].copy(), iters=it.value,
                breakdown=bool(bd.value))


def body_step_kat(kind, mass, inertia, q, u, gravity, h, integrate_with_ut=False):
    q = np.ascontiguousarray(q, float).copy()
    u = np.ascontiguousarray(u, float).copy()
    inertia = m3(inertia)
    g = np.ascontiguousarray(gravity, float)
    n = 3 if kind == 0 else 6
    f, ut = np.zeros(n), np.zeros(n)
    lib().orc_body_step_kat(C.c_int(kind), C.c_double(mass), dp(inertia), dp(q), dp(u), dp(g), C.c_double(h),
                            dp(f), dp(ut), C.c_int(int(integrate_with_ut)))
    return q, f, ut


# ---------------------------------------------------------------- world level
class OracleWorld:
    """One reference-semantics world (build_world + step_world), CPU double."""

    def __init__(self, name: str, seed: int = 0):
        self._h = lib().orc_world_create(name.encode(), C.c_uint(seed))
        if not self._h:
            raise ValueError(lib().orc_last_error().decode())
        self._hp = C.c_void_p(self._h)
        self.name = name

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_world_destroy(C.c_void_p(h))
            self._h = None

    def dims(self):
        d = np.zeros(12, np.int32)
        lib().orc_world_dims(self._hp, ip(d))
        keys = ["n_bodies", "num_dof", "num_coord", "n_joints", "n_tets", "n_shapes", "n_contacts",
                "rows_joint", "rows_mesh", "newton_iterations", "linear_iterations", "n_meshes"]
        return dict(zip(keys, (int(x) for x in d)))

    @property
    def h(self):
        return lib().orc_world_h(self._hp)

    def gravity(self):
        g = np.zeros(3)
        lib().orc_world_gravity(self._hp, dp(g))
        return g

    def get_config(self):
        ic, dc = np.zeros(8, np.int32), np.zeros(4)
        lib().orc_world_get_config(self._hp, ip(ic), dp(dc))
        return dict(newton_iterations=int(ic[0]), linear_max_iterations=int(ic[1]), line_search=int(ic[2]),
                    geometric_stiffness=int(ic[3]), r_strategy=int(ic[4]), ncp_kind=int(ic[5]),
                    preconditioner=int(ic[6]), linear_method=int(ic[7]), step_fraction=float(dc[0]),
                    epsilon_reg=float(dc[1]), linear_tolerance=float(dc[2]), newton_tolerance=float(dc[3]))

    def set_config(self, **kw):
        c = self.get_config()
        c.update(kw)
        ic = np.array([c["newton_iterations"], c["linear_max_iterations"], c["line_search"],
                       c["geometric_stiffness"], c["r_strategy"], c["ncp_kind"], c["preconditioner"],
                       c["linear_method"]], np.int32)
        dc = np.array([c["step_fraction"], c["epsilon_reg"], c["linear_tolerance"], c["newton_tolerance"]])
        lib().orc_world_set_config(self._hp, ip(ic), dp(dc))

    def state(self):
        d = self.dims()
        q, u = np.zeros(d["num_coord"]), np.zeros(d["num_dof"])
        lib().orc_world_get_state(self._hp, dp(q), dp(u))
        return q, u

    def set_state(self, q, u):
        q, u = np.ascontiguousarray(q, float), np.ascontiguousarray(u, float)
        lib().orc_world_set_state(self._hp, dp(q), dp(u))

    def topology(self):
        d = self.dims()
        nb, nj, nt = d["n_bodies"], d["n_joints"], d["n_tets"]
        t = dict(body_type=np.zeros(nb, np.int32), body_mass=np.zeros(nb), body_inertia=np.zeros(9 * nb),
                 joint_kind=np.zeros(nj, np.int32), joint_body=np.zeros(2 * nj, np.int32),
                 joint_frame=np.zeros(21 * nj), joint_param=np.zeros(2 * nj), tet_body=np.zeros(4 * nt, np.int32),
                 tet_dm_inv=np.zeros(9 * nt), tet_volume=np.zeros(nt), tet_material=np.zeros(4 * nt))
        lib().orc_world_topology(self._hp, ip(t["body_type"]), dp(t["body_mass"]), dp(t["body_inertia"]),
                                 ip(t["joint_kind"]), ip(t["joint_body"]), dp(t["joint_frame"]),
                                 dp(t["joint_param"]), ip(t["tet_body"]), dp(t["tet_dm_inv"]),
                                 dp(t["tet_volume"]), dp(t["tet_material"]))
        return t

    def joint_frames(self):
        f = np.zeros(21 * self.dims()["n_joints"])
        lib().orc_world_joint_frames(self._hp, dp(f))
        return f

    def shapes(self):
        ns = self.dims()["n_shapes"]
        body, kind, dpar, cp = np.zeros(ns, np.int32), np.zeros(ns, np.int32), np.zeros(10 * ns), np.zeros(2)
        lib().orc_world_shapes(self._hp, ip(body), ip(kind), dp(dpar), dp(cp))
        return dict(body=body, kind=kind, dparam=dpar, margin=float(cp[0]), mu_default=float(cp[1]))

    def contacts(self):
        n = lib().orc_world_n_contacts(self._hp)
        ib, db = np.zeros(4 * n, np.int32), np.zeros(22 * n)
        lib().orc_world_contacts(self._hp, ip(ib), dp(db))
        return ib.reshape(n, 4), db.reshape(n, 22)

    def set_joint_torques(self, tau):
        if tau is None:
            lib().orc_world_set_joint_torques(self._hp, None)
        else:
            tau = np.ascontiguousarray(tau, float)
            lib().orc_world_set_joint_torques(self._hp, dp(tau))

    def f_extra(self):
        f = np.zeros(self.dims()["num_dof"])
        lib().orc_world_get_f_extra(self._hp, dp(f))
        return f

    def prepare(self):
        if lib().orc_world_prepare(self._hp):
            raise RuntimeError(lib().orc_last_error().decode())

    def newton(self):
        rc = lib().orc_world_newton(self._hp)
        if rc == 1:
            raise RuntimeError(lib().orc_last_error().decode())
        return rc

    def step(self, n=1):
        rc = lib().orc_world_step(self._hp, C.c_int(n))
        if rc == 1:
            raise RuntimeError(lib().orc_last_error().decode())
        return rc

    def decisions(self):
        """Decision vectors of the last newton step (N x (nc + nt + ndof + 1) bytes, the
        layout of nsd_step_out::decisions)."""
        d = self.dims()
        cfg = self.get_config()
        stride = d["n_contacts"] + d["n_tets"] + d["num_dof"] + 1
        out = np.zeros(cfg["newton_iterations"] * stride, np.uint8)
        n = lib().orc_world_decisions(self._hp, out.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_int(stride),
                                      C.c_int(cfg["newton_iterations"]))
        return out.reshape(-1, stride)[:n]

    def report(self, n_rows=None):
        d = self.dims()
        cfg = self.get_config()
        ni, stride = cfg["newton_iterations"], cfg["linear_max_iterations"] + 1
        nc = d["n_contacts"]
        rows = n_rows if n_rows is not None else d["rows_joint"] + d["rows_mesh"] + 3 * nc
        stats, fin = np.zeros(8 * ni), np.zeros(7)
        hist, hl = np.zeros(ni * stride), np.zeros(ni, np.int32)
        lam, tel = np.zeros(max(rows, 1)), np.zeros(6 * max(nc, 1))
        n = lib().orc_world_report(self._hp, dp(stats), dp(fin), dp(hist), ip(hl), C.c_int(stride), dp(lam), dp(tel))
        stats = stats.reshape(ni, 8)[:n]
        return dict(n_iterations=n, stats=stats, final=fin, hist=hist.reshape(ni, stride), hist_len=hl[:n],
                    lam=lam[:rows], tel=tel.reshape(-1, 6)[:nc])


def run(name, seed, steps, out_dir):
    """Runner CSVs (trajectory.csv, convergence.csv) of the oracle's step_world; returns the exit code."""
    return lib().orc_run(name.encode(), C.c_uint(seed), C.c_int(steps), str(out_dir).encode())


def action_torque(env, step, joint):
    return lib().orc_action_torque(C.c_int(env), C.c_int(step), C.c_int(joint))


def c5_states(env0, n_env, n_steps, ncoord, ndof, actuated=True, threads=0, perturb=0.0, pseed=0):
    """Final (q, u, n_contacts) of C5 ants env0.. after n_steps oracle step_world calls
    (perturb > 0: initial q scaled by 1 + perturb * N(0, 1), seeded by pseed)."""
    q = np.zeros((n_env, ncoord))
    u = np.zeros((n_env, ndof))
    nc = np.zeros(n_env, dtype=np.int32)
    lib().orc_c5_states(C.c_int(env0), C.c_int(n_env), C.c_int(n_steps), C.c_int(int(actuated)), C.c_int(threads),
                        dp(q), dp(u), ip(nc), C.c_double(perturb), C.c_uint(pseed))
    return q, u, nc


def c5_bench(env0, n_env, n_steps, actuated=False, threads=0, warm=0):
    """Times steps [warm, warm + n_steps) of n_env C5 ants (OpenMP over envs)."""
    used, cs = C.c_int(), C.c_double()
    secs = lib().orc_c5_bench(C.c_int(env0), C.c_int(n_env), C.c_int(warm), C.c_int(n_steps), C.c_int(int(actuated)),
                              C.c_int(threads), C.byref(used), C.byref(cs))
    return secs, used.value, cs.value
