"""ctypes binding of include/nsdyn_gpu.h (the C ABI of libnsdyn_b200.so).

The product path has no CPU fallback: if the sm_100a library is missing this
module raises at import-time use, and every entry point reports CUDA errors
as exceptions (status NSD_CUDA_ERROR).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "libnsdyn_b200.so")

NSD_OK, NSD_INVALID, NSD_ABORTED, NSD_CUDA_ERROR, NSD_UNSUPPORTED = 0, 1, 2, 3, 4
NSD_FP32, NSD_FP64 = 0, 1

D = C.POINTER(C.c_double)
I32 = C.POINTER(C.c_int32)


class nsd_config(C.Structure):
    _fields_ = [("newton_iterations", C.c_int32), ("step_fraction", C.c_double), ("epsilon_reg", C.c_double),
                ("geometric_stiffness", C.c_int32), ("r_strategy", C.c_int32), ("ncp_kind", C.c_int32),
                ("linear_method", C.c_int32), ("linear_max_iterations", C.c_int32),
                ("linear_tolerance", C.c_double), ("preconditioner", C.c_int32), ("newton_tolerance", C.c_double),
                ("line_search", C.c_int32), ("precision", C.c_int32)]


class nsd_topology(C.Structure):
    _fields_ = [("n_bodies", C.c_int32), ("body_type", I32), ("body_mass", D), ("body_inertia", D),
                ("n_joints", C.c_int32), ("joint_kind", I32), ("joint_body", I32), ("joint_frame", D),
                ("joint_param", D), ("n_tets", C.c_int32), ("tet_body", I32), ("tet_dm_inv", D),
                ("tet_volume", D), ("tet_material", D)]


class nsd_contact(C.Structure):
    _fields_ = [("body_a", C.c_int32), ("body_b", C.c_int32), ("feature", C.c_int32), ("pad", C.c_int32),
                ("local_a", C.c_double * 3), ("local_b", C.c_double * 3), ("normal", C.c_double * 3),
                ("d1", C.c_double * 3), ("d2", C.c_double * 3), ("thickness", C.c_double), ("mu", C.c_double),
                ("lambda_n", C.c_double), ("lambda_f", C.c_double * 2), ("pad2", C.c_double * 2)]


class nsd_iter_stats(C.Structure):
    _fields_ = [("residual_inf", C.c_double), ("merit_l2", C.c_double), ("comp_error_max", C.c_double),
                ("cone_violation_max", C.c_double), ("step_size", C.c_double), ("linear_residual", C.c_double),
                ("linear_iterations", C.c_int32), ("linear_breakdown", C.c_int32)]


class nsd_step_in(C.Structure):
    _fields_ = [("q", D), ("u", D), ("n_contacts", C.c_int32), ("contacts", C.POINTER(nsd_contact)),
                ("h", C.c_double), ("gravity", C.c_double * 3), ("f_extra", D), ("joint_frame", D)]


class nsd_step_out(C.Structure):
    _fields_ = [("q", D), ("u", D), ("lambda_", D), ("contacts", C.POINTER(nsd_contact)),
                ("iters", C.POINTER(nsd_iter_stats)), ("linear_history", D), ("linear_history_len", I32),
                ("contact_telemetry", D), ("n_iterations", C.c_int32), ("n_rows", C.c_int32),
                ("final_residual_inf", C.c_double), ("final_comp_error", C.c_double),
                ("final_cone_violation", C.c_double), ("min_gap", C.c_double), ("min_diag_shift", C.c_double),
                ("aborted", C.c_int32), ("converged", C.c_int32), ("decisions", C.POINTER(C.c_uint8))]


class nsd_shape(C.Structure):
    _fields_ = [("body", C.c_int32), ("kind", C.c_int32), ("normal", C.c_double * 3), ("offset", C.c_double),
                ("radius", C.c_double), ("half_extents", C.c_double * 3), ("thickness", C.c_double),
                ("mu", C.c_double)]


# Every symbol include/nsdyn_gpu.h declares (checked by tests/test_cabi.py).
EXPORTS = [
    "nsd_config_default", "nsd_last_error", "nsd_count_rows", "nsd_create", "nsd_set_config", "nsd_step",
    "nsd_last_step_ms", "nsd_destroy", "nsd_batch_create", "nsd_batch_set_state", "nsd_batch_get_state",
    "nsd_batch_set_stream", "nsd_batch_step", "nsd_batch_step_device", "nsd_batch_step_mapped", "nsd_batch_sync", "nsd_batch_results",
    "nsd_batch_contacts", "nsd_batch_device_state", "nsd_batch_copy_state_async", "nsd_batch_info", "nsd_batch_counters", "nsd_batch_profile", "nsd_batch_destroy", "nsd_scene_build", "nsd_scene_parse", "nsd_scene_serialize",
    "nsd_scene_dims", "nsd_scene_topology", "nsd_scene_shapes", "nsd_scene_state", "nsd_scene_config",
    "nsd_scene_destroy", "nsd_scene_batch_state", "nsd_scene_joint_frames", "nsd_scene_advance_anchors",
    "nsd_scene_detect",
]

_lib = None


class NsdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"nsd error {code}: {msg}")
        self.code = code


def lib():
    """Loads the sm_100a library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    L.nsd_last_error.restype = C.c_char_p
    L.nsd_last_step_ms.restype = C.c_double
    L.nsd_last_step_ms.argtypes = [C.c_void_p]
    L.nsd_config_default.argtypes = [C.POINTER(nsd_config), C.c_int32]
    L.nsd_count_rows.argtypes = [C.POINTER(nsd_topology), C.c_int32]
    L.nsd_create.argtypes = [C.POINTER(nsd_topology), C.POINTER(nsd_config), C.c_int32, C.POINTER(C.c_void_p)]
    L.nsd_set_config.argtypes = [C.c_void_p, C.POINTER(nsd_config)]
    L.nsd_step.argtypes = [C.c_void_p, C.POINTER(nsd_step_in), C.POINTER(nsd_step_out)]
    L.nsd_destroy.argtypes = [C.c_void_p]
    L.nsd_batch_create.argtypes = [C.POINTER(nsd_topology), C.c_int32, C.POINTER(nsd_shape), C.c_double,
                                   C.c_double, C.POINTER(nsd_config), C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(C.c_void_p)]
    L.nsd_batch_set_state.argtypes = [C.c_void_p, D, D]
    L.nsd_batch_get_state.argtypes = [C.c_void_p, D, D]
    L.nsd_batch_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.nsd_batch_step.argtypes = [C.c_void_p, D, C.c_int32, C.c_double, D]
    L.nsd_batch_step_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, D]
    L.nsd_batch_step_mapped.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_double, D]
    L.nsd_batch_sync.argtypes = [C.c_void_p]
    L.nsd_batch_results.argtypes = [C.c_void_p, I32, I32, D, C.POINTER(nsd_iter_stats)]
    L.nsd_batch_contacts.argtypes = [C.c_void_p, C.c_int32, C.POINTER(nsd_contact), I32]
    L.nsd_batch_device_state.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), I32]
    L.nsd_batch_info.argtypes = [C.c_void_p, I32]
    L.nsd_batch_counters.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    L.nsd_batch_profile.argtypes = [C.c_void_p, C.c_int32]
    L.nsd_batch_copy_state_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.nsd_scene_batch_state.argtypes = [C.c_char_p, C.c_uint32, C.c_int32, D, D]
    L.nsd_batch_destroy.argtypes = [C.c_void_p]
    L.nsd_scene_build.argtypes = [C.c_char_p, C.c_uint32, C.POINTER(C.c_void_p)]
    L.nsd_scene_parse.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32]
    L.nsd_scene_serialize.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
    L.nsd_scene_dims.argtypes = [C.c_void_p, I32]
    L.nsd_scene_topology.argtypes = [C.c_void_p, C.POINTER(nsd_topology)]
    L.nsd_scene_shapes.argtypes = [C.c_void_p, C.POINTER(nsd_shape), D, D]
    L.nsd_scene_state.argtypes = [C.c_void_p, D, D]
    L.nsd_scene_config.argtypes = [C.c_void_p, C.POINTER(nsd_config), D, D]
    L.nsd_scene_destroy.argtypes = [C.c_void_p]
    L.nsd_scene_joint_frames.argtypes = [C.c_void_p, D]
    L.nsd_scene_advance_anchors.argtypes = [C.c_void_p]
    L.nsd_scene_detect.argtypes = [C.c_void_p, D, D, D, C.c_int32, C.POINTER(nsd_contact), I32]
    _lib = L
    return L


def check(rc, allow_abort=False):
    if rc == NSD_OK or (allow_abort and rc == NSD_ABORTED):
        return rc
    raise NsdError(rc, lib().nsd_last_error().decode())
