"""Runner output formats (runner.cpp:13-27, 80-126, 148-218):
trajectory.csv / convergence.csv / sweep.csv written by the C++ host API
(include/nsdyn_b200.hpp: run, sweep) and by the oracle, diffed file to file.
"""
import csv
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle_py as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "world_demo")
TRAJ_HDR = "step,body,qx,qy,qz,q0,q1,q2,q3,ux,uy,uz,wx,wy,wz"
CONV_HDR = ("step,newton_iter,residual_inf,comp_error_n_max,cone_violation_max,step_size,linear_iters,"
            "linear_residual_final")


def _read(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    return rows[0], np.array(rows[1:], dtype=float)


def test_oracle_runner_csv_format(tmp_path):
    assert O.run("c3:5", 0, 3, tmp_path) == 0
    h, t = _read(tmp_path / "trajectory.csv")
    assert ",".join(h) == TRAJ_HDR and t.shape == (3 * 5, 15)
    h, c = _read(tmp_path / "convergence.csv")
    assert ",".join(h) == CONV_HDR and c.shape == (3 * 8, 8)
    assert O.run("nope", 0, 3, tmp_path) == 1  # validation error exit code


def _cpp(*args):
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("name,steps", [("c1", 10), ("c5", 8), ("c3:30", 6)])
def test_cpp_runner_matches_oracle_files(tmp_path, name, steps):
    g, o = tmp_path / "gpu", tmp_path / "oracle"
    os.makedirs(g)
    os.makedirs(o)
    r = _cpp("--run", name, steps, g)
    assert r.returncode == 0, r.stdout + r.stderr
    assert O.run(name, 0, steps, o) == 0
    hg, tg = _read(g / "trajectory.csv")
    ho, to = _read(o / "trajectory.csv")
    assert hg == ho and tg.shape == to.shape
    assert np.array_equal(tg[:, :2], to[:, :2])
    q = slice(2, 9)
    assert np.max(np.abs(tg[:, q] - to[:, q])) <= 1e-8 * max(1.0, np.max(np.abs(to[:, q])))
    assert np.max(np.abs(tg[:, 9:] - to[:, 9:])) <= 1e-6 * max(1.0, np.max(np.abs(to[:, 9:])))
    hg, cg = _read(g / "convergence.csv")
    ho, co = _read(o / "convergence.csv")
    assert hg == ho and cg.shape == co.shape
    assert np.array_equal(cg[:, :2], co[:, :2])
    # step_size and the complementarity error are well conditioned: compare them.
    # Not compared: linear_iters and residual_inf. Both runs stop the PCR on the
    # monotone guard at their rounding floor (explicit S ~1e-11, matrix-free
    # ~1e-16), so iteration counts legitimately differ there; and residual_inf
    # contains W lambda_f with the friction W capped at 1e12 for sticking
    # contacts (ncp.cpp:34-49), amplifying 1e-12 multiplier differences to O(1).
    for k in (3, 5):
        assert np.allclose(cg[:, k], co[:, k], rtol=1e-5, atol=1e-9 * max(1.0, np.max(np.abs(co[:, k])))), k


@pytest.mark.gpu
def test_cpp_sweep_and_validation(tmp_path):
    r = _cpp("--sweep", "c1", "ncp", 3, tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    with open(tmp_path / "sweep.csv") as f:
        rows = list(csv.reader(f))
    assert ",".join(rows[0]) == "axis_value," + CONV_HDR
    assert {row[0] for row in rows[1:]} == {"minmap", "fb"}
    bad = _cpp("--run", "c1", 0, tmp_path)  # --steps must be >= 1 -> validation exit code 1
    assert bad.returncode == 1 and "--steps" in bad.stdout
