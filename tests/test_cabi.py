"""CPU-side checks of the product boundary: the sm_100a library loads, exports
every symbol include/nsdyn_gpu.h declares, and the product's scene builders
reproduce the oracle's build_world bit for bit (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle_py as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1907_04587_b200 import _lib as L

    return L


def test_library_exports_every_header_symbol():
    L = _lib()
    hdr = open(os.path.join(ROOT, "include", "nsdyn_gpu.h")).read()
    declared = set(re.findall(r"\b(nsd_[a-z_]+)\s*\(", hdr))
    assert declared == set(L.EXPORTS), declared ^ set(L.EXPORTS)
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_config_defaults_match_reference():
    from paper_1907_04587_b200 import NewtonConfig

    L = _lib()
    c = L.nsd_config()
    L.lib().nsd_config_default(C.byref(c), 1)
    ref = NewtonConfig()
    assert (c.newton_iterations, c.step_fraction, c.epsilon_reg, c.geometric_stiffness) == (8, 0.75, 1e-6, 1)
    assert (c.r_strategy, c.ncp_kind, c.linear_method, c.linear_max_iterations) == (2, 1, 3, 40)
    assert (c.linear_tolerance, c.preconditioner, c.newton_tolerance, c.line_search) == (1e-10, 1, 1e-6, 0)
    assert ref.to_c().linear_max_iterations == 40


@pytest.mark.parametrize("name,seed", [("c1", 0), ("c2:4", 0), ("c3:20", 0), ("c4:6", 0), ("c5", 0), ("c5", 17),
                                       ("c5", 4095), ("heavy_stack", 0), ("arch", 0), ("stretch_sheet", 0), ("stretch_sheet_linear", 0),
                                       ("incline:35:0.5", 0), ("box_on_plane", 0), ("bend_chain", 0), ("bend_chain:6:5", 0)])
def test_product_builders_match_oracle_bitwise(name, seed):
    from paper_1907_04587_b200 import Scene

    s = Scene(name, seed)
    w = O.OracleWorld(name, seed)
    t = w.topology()
    for k, v in t.items():
        assert np.array_equal(s.topology.a[k], v), k
    q, u = w.state()
    assert np.array_equal(s.q, q)
    assert np.array_equal(s.u, u)
    sh = w.shapes()
    assert s.n_shapes == len(sh["body"])
    for i in range(s.n_shapes):
        assert s.shapes[i].body == sh["body"][i] and s.shapes[i].kind == sh["kind"][i]
        d = sh["dparam"][10 * i:10 * i + 10]
        mine = list(s.shapes[i].normal) + [s.shapes[i].offset, s.shapes[i].radius] + list(s.shapes[i].half_extents) + \
            [s.shapes[i].thickness, s.shapes[i].mu]
        assert np.array_equal(np.array(mine), d)
    assert (s.margin, s.mu_default) == (sh["margin"], sh["mu_default"])
    cfg = w.get_config()
    assert s.config.newton_iterations == cfg["newton_iterations"]
    assert s.config.linear_max_iterations == cfg["linear_max_iterations"]
    assert s.h == w.h and np.array_equal(s.gravity, w.gravity())


def test_count_rows_layout():
    from paper_1907_04587_b200 import Scene, count_rows

    s = Scene("c3:20", 0)
    # 20 joints: 18 revolute (5 rows) + 2 prismatic (5 rows); no tets
    assert count_rows(s.topology, 0) == 100
    assert count_rows(s.topology, 4) == 112
    s2 = Scene("c2:2", 0)
    assert count_rows(s2.topology, 3) == 3 * 48 + 9


def test_unknown_scene_rejected():
    from paper_1907_04587_b200 import NsdError, Scene

    with pytest.raises(NsdError):
        Scene("no_such_scene", 0)
