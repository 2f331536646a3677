"""B200-native non-smooth Newton step (Macklin et al. 2019, arXiv 1907.04587).

Host-side Python mirror of the reference's solver interface
(/root/reference/proj/include/nsdyn/newton.h) over the C ABI in
include/nsdyn_gpu.h. Names follow the reference: NewtonConfig, newton_step,
count_rows, SolveReport fields, NewtonIterationStats fields.

    solver = NewtonSolver(topology, NewtonConfig(precision="fp64"))
    report = solver.newton_step(q, u, contacts, h=0.0083, gravity=(0, 0, -9.81))

The compute runs in hand-written sm_100a kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (NSD_ABORTED, NSD_FP32, NSD_FP64, NSD_INVALID, NSD_OK, NsdError, check, lib, nsd_config, nsd_contact,
                   nsd_iter_stats, nsd_shape, nsd_step_in, nsd_step_out, nsd_topology)

__all__ = ["NewtonConfig", "NewtonSolver", "BatchSolver", "Scene", "World", "contacts_from_arrays", "contacts_to_arrays",
           "count_rows", "NsdError"]

_R_STRAT = {"identity": 0, "h2": 1, "effmass": 2}
_NCP = {"minmap": 0, "fb": 1}


@dataclass
class NewtonConfig:
    """NewtonConfig + LinearSolverConfig (newton.h:12-23, solvers.h:11-16)."""
    newton_iterations: int = 8
    step_fraction: float = 0.75
    epsilon_reg: float = 1e-6
    geometric_stiffness: bool = True
    r_strategy: int = 2
    ncp_kind: int = 1
    linear_method: int = 3
    linear_max_iterations: int = 40
    linear_tolerance: float = 1e-10
    preconditioner: int = 1
    newton_tolerance: float = 1e-6
    line_search: bool = False
    precision: str = "fp32"

    def to_c(self) -> nsd_config:
        c = nsd_config()
        c.newton_iterations = self.newton_iterations
        c.step_fraction = self.step_fraction
        c.epsilon_reg = self.epsilon_reg
        c.geometric_stiffness = int(bool(self.geometric_stiffness))
        c.r_strategy = _R_STRAT.get(self.r_strategy, self.r_strategy) if isinstance(self.r_strategy, str) else self.r_strategy
        c.ncp_kind = _NCP.get(self.ncp_kind, self.ncp_kind) if isinstance(self.ncp_kind, str) else self.ncp_kind
        c.linear_method = self.linear_method
        c.linear_max_iterations = self.linear_max_iterations
        c.linear_tolerance = self.linear_tolerance
        c.preconditioner = self.preconditioner
        c.newton_tolerance = self.newton_tolerance
        c.line_search = int(bool(self.line_search))
        c.precision = NSD_FP64 if self.precision == "fp64" else NSD_FP32
        return c

    @staticmethod
    def from_c(c: nsd_config, precision=None) -> "NewtonConfig":
        return NewtonConfig(c.newton_iterations, c.step_fraction, c.epsilon_reg, bool(c.geometric_stiffness),
                            c.r_strategy, c.ncp_kind, c.linear_method, c.linear_max_iterations, c.linear_tolerance,
                            c.preconditioner, c.newton_tolerance, bool(c.line_search),
                            precision or ("fp64" if c.precision == NSD_FP64 else "fp32"))


def _dp(a):
    return a.ctypes.data_as(_lib.D)


def _ip(a):
    return a.ctypes.data_as(_lib.I32)


class Topology:
    """Static scene arrays in the C-ABI layout (owns the numpy buffers)."""

    KEYS_I = ("body_type", "joint_kind", "joint_body", "tet_body")
    KEYS_D = ("body_mass", "body_inertia", "joint_frame", "joint_param", "tet_dm_inv", "tet_volume", "tet_material")

    def __init__(self, **arrays):
        self.a = {}
        for k in self.KEYS_I:
            self.a[k] = np.ascontiguousarray(arrays.get(k, np.zeros(0)), dtype=np.int32)
        for k in self.KEYS_D:
            self.a[k] = np.ascontiguousarray(arrays.get(k, np.zeros(0)), dtype=np.float64)
        bt = self.a["body_type"]
        self.n_bodies = len(bt)
        self.num_dof = int(np.sum(np.where(bt == 1, 6, 3)))
        self.num_coord = int(np.sum(np.where(bt == 1, 7, 3)))
        self.n_joints = len(self.a["joint_kind"])
        self.n_tets = len(self.a["tet_volume"])
        self._c = nsd_topology(self.n_bodies, _ip(self.a["body_type"]), _dp(self.a["body_mass"]),
                               _dp(self.a["body_inertia"]), self.n_joints, _ip(self.a["joint_kind"]),
                               _ip(self.a["joint_body"]), _dp(self.a["joint_frame"]), _dp(self.a["joint_param"]),
                               self.n_tets, _ip(self.a["tet_body"]), _dp(self.a["tet_dm_inv"]),
                               _dp(self.a["tet_volume"]), _dp(self.a["tet_material"]))

    @property
    def c(self):
        return self._c


def count_rows(topology: Topology, n_contacts: int) -> int:
    """count_rows (newton.h:114)."""
    return lib().nsd_count_rows(C.byref(topology.c), n_contacts)


def _contact_views(arr, n):
    """(n,4) int32 and (n,22) float64 views of an nsd_contact array: the C struct is
    4 int32 (body_a, body_b, feature, pad) followed by 22 doubles in exactly the
    array layout (local_a, local_b, normal, d1, d2, thickness, mu, lambda_n,
    lambda_f[2], pad[2])."""
    raw = np.frombuffer(arr, dtype=np.uint8)[: n * C.sizeof(nsd_contact)].reshape(n, C.sizeof(nsd_contact))
    return raw[:, :16].view(np.int32), raw[:, 16:].view(np.float64)


def contacts_from_arrays(ib, db):
    """(n,4) int [body_a, body_b, feature, 0] + (n,22) doubles -> nsd_contact array."""
    n = len(ib)
    arr = (nsd_contact * max(n, 1))()
    if n:
        vi, vd = _contact_views(arr, n)
        vi[:, :3] = np.asarray(ib)[:, :3]
        vd[:, :20] = np.asarray(db, np.float64)[:, :20]
    return arr, n


def contacts_to_arrays(arr, n):
    ib = np.zeros((n, 4), np.int32)
    db = np.zeros((n, 22))
    if n:
        vi, vd = _contact_views(arr, n)
        ib[:, :3] = vi[:, :3]
        db[:, :20] = vd[:, :20]
    return ib, db


class NewtonSolver:
    """One scene on one GPU: nsd_create / nsd_step (the newton_step boundary)."""

    def __init__(self, topology: Topology, config: NewtonConfig, device: int = 0):
        self.topology = topology
        self.config = config
        h = C.c_void_p()
        check(lib().nsd_create(C.byref(topology.c), C.byref(config.to_c()), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().nsd_destroy(self._h)
            self._h = None

    __del__ = close

    def set_config(self, config: NewtonConfig):
        check(lib().nsd_set_config(self._h, C.byref(config.to_c())))
        self.config = config

    @property
    def last_step_ms(self):
        return lib().nsd_last_step_ms(self._h)

    def newton_step(self, q, u, contacts=None, h=0.0083, gravity=(0.0, 0.0, -9.81), f_extra=None,
                    joint_frame=None, decisions=True):
        """newton_step (newton.cpp:321-418). contacts: (ib, db) arrays or (nsd_contact array, n).
        decisions: also return the per-iteration decision vectors (a diagnostic; World.step
        skips them)."""
        T, cfg = self.topology, self.config
        q = np.ascontiguousarray(q, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        if contacts is None:
            carr, nc = (nsd_contact * 1)(), 0
        elif isinstance(contacts, tuple) and isinstance(contacts[0], np.ndarray):
            carr, nc = contacts_from_arrays(*contacts)
        else:
            carr, nc = contacts
        fx = None if f_extra is None else np.ascontiguousarray(f_extra, np.float64)
        jf = None if joint_frame is None else np.ascontiguousarray(joint_frame, np.float64)
        sin = nsd_step_in()
        sin.q, sin.u = _dp(q), _dp(u)
        sin.n_contacts, sin.contacts = nc, C.cast(carr, C.POINTER(nsd_contact))
        sin.h = h
        for k in range(3):
            sin.gravity[k] = gravity[k]
        sin.f_extra = _dp(fx) if fx is not None else None
        sin.joint_frame = _dp(jf) if jf is not None else None
        nrows = count_rows(T, nc)
        N, ml = cfg.newton_iterations, cfg.linear_max_iterations
        qo, uo = np.zeros(T.num_coord), np.zeros(T.num_dof)
        lam = np.zeros(max(nrows, 1))
        iters = (nsd_iter_stats * max(N, 1))()
        hist = np.zeros(max(N, 1) * (ml + 1))
        hlen = np.zeros(max(N, 1), np.int32)
        tel = np.zeros(6 * max(nc, 1))
        dec_stride = nc + T.n_tets + T.num_dof + 1
        dec = np.zeros(max(N, 1) * dec_stride if decisions else 1, np.uint8)
        cout = (nsd_contact * max(nc, 1))()
        so = nsd_step_out()
        so.q, so.u, so.lambda_ = _dp(qo), _dp(uo), _dp(lam)
        so.contacts = C.cast(cout, C.POINTER(nsd_contact))
        so.iters = C.cast(iters, C.POINTER(nsd_iter_stats))
        so.linear_history, so.linear_history_len, so.contact_telemetry = _dp(hist), _ip(hlen), _dp(tel)
        so.decisions = dec.ctypes.data_as(C.POINTER(C.c_uint8)) if decisions else None
        rc = lib().nsd_step(self._h, C.byref(sin), C.byref(so))
        check(rc, allow_abort=True)
        n = so.n_iterations
        stats = np.array([[it.residual_inf, it.merit_l2, it.comp_error_max, it.cone_violation_max, it.step_size,
                           it.linear_iterations, it.linear_residual, it.linear_breakdown] for it in iters[:n]])
        return dict(q=qo, u=uo, lam=lam[:nrows], stats=stats.reshape(n, 8), n_iterations=n,
                    hist=hist.reshape(max(N, 1), ml + 1), hist_len=hlen[:n].copy(), tel=tel.reshape(-1, 6)[:nc],
                    final=np.array([so.final_residual_inf, so.final_comp_error, so.final_cone_violation,
                                    so.min_gap, so.min_diag_shift, so.aborted, so.converged]),
                    contacts=contacts_to_arrays(cout, nc), n_rows=so.n_rows, aborted=bool(so.aborted),
                    ms=self.last_step_ms,
                    decisions=dec.reshape(max(N, 1), dec_stride)[:n].copy() if decisions else None)


def _open_scene(name, seed, json_text):
    """nsd_scene_build(name, seed), or nsd_scene_parse(json_text) (the reference's JSON
    scene format, scene.cpp:293-470) with its validation message on failure."""
    h = C.c_void_p()
    if json_text is None:
        check(lib().nsd_scene_build(name.encode(), seed, C.byref(h)))
        return h
    if isinstance(json_text, str):
        json_text = json_text.encode()
    err = C.create_string_buffer(1024)
    if lib().nsd_scene_parse(json_text, C.byref(h), err, len(err)) != NSD_OK:
        raise NsdError(NSD_INVALID, err.value.decode(errors="replace"))
    return h


def serialize_scene(handle) -> str:
    n = C.c_int64()
    check(lib().nsd_scene_serialize(handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().nsd_scene_serialize(handle, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class Scene:
    """Product-side scenes: a builder (nsd_scene_build) or a document in the reference's
    JSON scene format (Scene.from_json, nsd_scene_parse): topology, shapes, state,
    config; to_json() is serialize_scene (scene.cpp:472-556)."""

    def __init__(self, name: str = "", seed: int = 0, json_text=None):
        h = _open_scene(name, seed, json_text)
        self._h = h
        d = np.zeros(8, np.int32)
        check(lib().nsd_scene_dims(h, _ip(d)))
        self.dims = dict(zip(["n_bodies", "num_dof", "num_coord", "n_joints", "n_tets", "n_shapes",
                              "newton_iterations", "linear_max_iterations"], (int(x) for x in d)))
        t = nsd_topology()
        check(lib().nsd_scene_topology(h, C.byref(t)))
        nb, nj, nt = t.n_bodies, t.n_joints, t.n_tets

        def arr(p, n, dt):
            return np.ctypeslib.as_array(p, shape=(max(n, 0),)).astype(dt).copy() if n > 0 else np.zeros(0, dt)

        self.topology = Topology(body_type=arr(t.body_type, nb, np.int32), body_mass=arr(t.body_mass, nb, float),
                                 body_inertia=arr(t.body_inertia, 9 * nb, float),
                                 joint_kind=arr(t.joint_kind, nj, np.int32), joint_body=arr(t.joint_body, 2 * nj, np.int32),
                                 joint_frame=arr(t.joint_frame, 21 * nj, float),
                                 joint_param=arr(t.joint_param, 2 * nj, float), tet_body=arr(t.tet_body, 4 * nt, np.int32),
                                 tet_dm_inv=arr(t.tet_dm_inv, 9 * nt, float), tet_volume=arr(t.tet_volume, nt, float),
                                 tet_material=arr(t.tet_material, 4 * nt, float))
        ns = self.dims["n_shapes"]
        self.shapes = (nsd_shape * max(ns, 1))()
        mg, mud = C.c_double(), C.c_double()
        check(lib().nsd_scene_shapes(h, C.cast(self.shapes, C.POINTER(nsd_shape)), C.byref(mg), C.byref(mud)))
        self.n_shapes, self.margin, self.mu_default = ns, mg.value, mud.value
        self.q, self.u = np.zeros(self.dims["num_coord"]), np.zeros(self.dims["num_dof"])
        check(lib().nsd_scene_state(h, _dp(self.q), _dp(self.u)))
        cfg, hh, g = nsd_config(), C.c_double(), np.zeros(3)
        check(lib().nsd_scene_config(h, C.byref(cfg), C.byref(hh), _dp(g)))
        self.config, self.h, self.gravity = NewtonConfig.from_c(cfg), hh.value, g

    @classmethod
    def from_json(cls, text):
        return cls(json_text=text)

    def to_json(self) -> str:
        return serialize_scene(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().nsd_scene_destroy(h)
            except Exception:
                pass
            self._h = None


class World:
    """World + step_world (scene.h:83-110, scene.cpp:709-732): a built scene whose
    step() moves driven anchors, runs the caller-side contact detection on the
    host at (q, u~) — as the reference does — and then the Newton step on the
    GPU through nsd_step. `contacts` holds the step's contact arrays with the
    multipliers written back; `report` the SolveReport of the last step."""

    def __init__(self, name: str = "", seed: int = 0, precision: str | None = None, contact_capacity: int = 4096,
                 json_text=None):
        self.scene = Scene(name, seed, json_text=json_text)
        self._h = _open_scene(name, seed, json_text)
        self.topology = self.scene.topology
        self.config = self.scene.config
        if precision is not None:
            self.config.precision = precision
        self.h, self.gravity = self.scene.h, self.scene.gravity
        self.q, self.u = self.scene.q.copy(), self.scene.u.copy()
        self.f_extra = None
        self.cap = contact_capacity
        self._buf = (nsd_contact * contact_capacity)()
        self.solver = None  # created at the first step (device memory)
        self.contacts = None
        self.report = None
        self.time = 0.0

    def joint_frames(self):
        fr = np.zeros(21 * self.topology.n_joints)
        if fr.size:
            check(lib().nsd_scene_joint_frames(self._h, _dp(fr)))
        return fr

    def detect(self):
        n = C.c_int32()
        fx = _dp(self.f_extra) if self.f_extra is not None else None
        rc = lib().nsd_scene_detect(self._h, _dp(self.q), _dp(self.u), fx, self.cap,
                                    C.cast(self._buf, C.POINTER(nsd_contact)), C.byref(n))
        if rc != NSD_OK and n.value > self.cap:
            self.cap = 2 * n.value
            self._buf = (nsd_contact * self.cap)()
            return self.detect()
        check(rc)
        return contacts_to_arrays(self._buf, n.value)

    def step(self, n: int = 1):
        """n x step_world; returns the last SolveReport (dict) — aborted steps roll back and are reported."""
        for _ in range(n):
            if self.solver is None:
                self.solver = NewtonSolver(self.topology, self.config)
            check(lib().nsd_scene_advance_anchors(self._h))
            self.contacts = self.detect()
            self.report = self.solver.newton_step(self.q, self.u, self.contacts, h=self.h,
                                                  gravity=tuple(self.gravity), f_extra=self.f_extra,
                                                  joint_frame=self.joint_frames(), decisions=False)
            self.q, self.u = self.report["q"], self.report["u"]
            self.contacts = self.report.get("contacts", self.contacts)
            self.time += self.h
        return self.report

    def close(self):
        if self._h:
            lib().nsd_scene_destroy(self._h)
            self._h = None
        if self.solver is not None:
            self.solver.close()
            self.solver = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def batch_states(name: str, seed0: int, n: int, num_coord: int, num_dof: int):
    """Initial states of n seeded copies of a builder (one C call)."""
    q, u = np.zeros(n * num_coord), np.zeros(n * num_dof)
    check(lib().nsd_scene_batch_state(name.encode(), seed0, n, _dp(q), _dp(u)))
    return q, u


class BatchSolver:
    """Many environments sharing one topology (nsd_batch_*): device narrow phase
    + Newton step per env, one team (warp or CTA) per environment."""

    def __init__(self, topology: Topology, shapes, n_shapes, margin, mu_default, config: NewtonConfig, n_env: int,
                 max_contacts: int = 48, device: int = 0):
        self.topology, self.config, self.n_env = topology, config, n_env
        h = C.c_void_p()
        check(lib().nsd_batch_create(C.byref(topology.c), n_shapes, C.cast(shapes, C.POINTER(nsd_shape)), margin,
                                     mu_default, C.byref(config.to_c()), n_env, max_contacts, device, C.byref(h)))
        self._h = h
        info = np.zeros(6, np.int32)
        check(lib().nsd_batch_info(h, _ip(info)))
        self.info = info

    def close(self):
        if getattr(self, "_h", None):
            lib().nsd_batch_destroy(self._h)
            self._h = None

    __del__ = close

    def set_stream(self, stream_ptr):
        check(lib().nsd_batch_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def set_state(self, q, u):
        q = np.ascontiguousarray(q, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        check(lib().nsd_batch_set_state(self._h, _dp(q), _dp(u)))

    def get_state(self):
        T = self.topology
        q, u = np.zeros(self.n_env * T.num_coord), np.zeros(self.n_env * T.num_dof)
        check(lib().nsd_batch_get_state(self._h, _dp(q), _dp(u)))
        return q.reshape(self.n_env, -1), u.reshape(self.n_env, -1)

    def step(self, h, gravity, torque=None):
        g = np.ascontiguousarray(gravity, np.float64)
        t = None if torque is None else np.ascontiguousarray(torque, np.float64)
        check(lib().nsd_batch_step(self._h, _dp(t) if t is not None else None, 0, h, _dp(g)))

    def step_device(self, h, gravity, torque_ptr=None, dtype=0):
        g = np.ascontiguousarray(gravity, np.float64)
        check(lib().nsd_batch_step_device(self._h, C.c_void_p(torque_ptr) if torque_ptr else None, dtype, h, _dp(g)))

    def step_mapped(self, h, gravity, torque_ptr=None, dtype=0, q_out_ptr=None, u_out_ptr=None):
        """step_device with the transfers fused into the step kernel: torques read
        from, and the final (q, u) written to, pinned host memory (or device memory)
        by the kernel itself (nsd_batch_step_mapped)."""
        g = np.ascontiguousarray(gravity, np.float64)
        vp = lambda p: C.c_void_p(p) if p else None
        check(lib().nsd_batch_step_mapped(self._h, vp(torque_ptr), dtype, vp(q_out_ptr), vp(u_out_ptr), h, _dp(g)))

    def sync(self):
        check(lib().nsd_batch_sync(self._h))

    def results(self, with_iters=False):
        n = self.n_env
        nc, ab, fr = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n)
        N = self.config.newton_iterations
        its = (nsd_iter_stats * (n * N))() if with_iters else None
        check(lib().nsd_batch_results(self._h, _ip(nc), _ip(ab), _dp(fr),
                                      C.cast(its, C.POINTER(nsd_iter_stats)) if its is not None else None))
        out = dict(n_contacts=nc, aborted=ab, final_residual_inf=fr)
        if its is not None:
            out["stats"] = np.array([[it.residual_inf, it.merit_l2, it.comp_error_max, it.cone_violation_max,
                                      it.step_size, it.linear_iterations, it.linear_residual, it.linear_breakdown]
                                     for it in its]).reshape(n, N, 8)
        return out

    def contacts(self, env):
        n = C.c_int32()
        check(lib().nsd_batch_contacts(self._h, env, None, C.byref(n)))
        arr = (nsd_contact * max(n.value, 1))()
        check(lib().nsd_batch_contacts(self._h, env, C.cast(arr, C.POINTER(nsd_contact)), C.byref(n)))
        return contacts_to_arrays(arr, n.value)

    def copy_state_async(self, q_ptr, u_ptr):
        check(lib().nsd_batch_copy_state_async(self._h, C.c_void_p(q_ptr) if q_ptr else None,
                                               C.c_void_p(u_ptr) if u_ptr else None))

    def counters(self):
        """Counters since the previous call (nsd_batch_counters): PCR iterations run
        (summed over envs, Newton iterations and steps), cycles inside the PCR loops
        and per env step (cycles on), env-steps, and the CUDA-event time of each
        launch of the step (launch timing on)."""
        v = (C.c_uint64 * 9)()
        check(lib().nsd_batch_counters(self._h, v))
        return dict(cr_iterations=int(v[0]), cr_cycles=int(v[1]), env_cycles=int(v[2]), env_steps=int(v[3]),
                    narrow_phase_ms=v[4] * 1e-6, warp_solver_ms=v[5] * 1e-6, large_env_ms=v[6] * 1e-6,
                    timed_steps=int(v[7]), cr_iterations_x_contacts=int(v[8]))

    def profile(self, cycles=True, launch_timing=False):
        check(lib().nsd_batch_profile(self._h, (1 if cycles else 0) | (2 if launch_timing else 0)))

    def device_state(self):
        q, u, dt = C.c_void_p(), C.c_void_p(), C.c_int32()
        check(lib().nsd_batch_device_state(self._h, C.byref(q), C.byref(u), C.byref(dt)))
        return q.value, u.value, dt.value
