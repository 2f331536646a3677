"""The C++ host API (include/nsdyn_b200.hpp) — the reference's
build_scene_by_name / step_world / newton_step / SolveReport surface over the C
ABI — exercised by a C++ program (tests/cpp/world_demo.cpp).

CPU: the program compiles with -Wall -Wextra and links against the product
library. GPU: free fall through a hand-built StepContext (u = u~ exactly,
SPEC.md:505), std::invalid_argument for h <= 0, and step_world trajectories in
fp64 against the oracle's step_world.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle_py as O
from tests.helpers import oracle_trajectory, rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
EXE = os.path.join(CPP, "_build", "world_demo")


def _build():
    r = subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return EXE


def test_cpp_api_compiles_and_links():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr  # argument check runs without a GPU


def _run(*args):
    r = subprocess.run([_build(), *map(str, args)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def _trajectory(out):
    lines = out.strip().splitlines()
    q = np.array([float(x) for x in lines[-2].split()[1:]])
    u = np.array([float(x) for x in lines[-1].split()[1:]])
    steps = [ln.split() for ln in lines if ln.startswith("step ")]
    return q, u, steps


@pytest.mark.gpu
def test_cpp_free_fall():
    assert "free_fall ok" in _run("--free-fall")


@pytest.mark.gpu
def test_cpp_invalid_h_throws_invalid_argument():
    assert "invalid_argument ok" in _run("--invalid-h")


@pytest.mark.gpu
@pytest.mark.parametrize("name,seed,steps,tol", [("c1", 0, 12, 1e-9), ("c5", 2, 10, 1e-8), ("box_pile", 3, 8, 1e-8),
                                                  ("c4:6", 0, 3, None)])
def test_cpp_step_world_matches_oracle(name, seed, steps, tol):
    """Same stated tolerances as tests/test_world.py (None = 10x the oracle's
    self-divergence under a 1e-15 input perturbation)."""
    q, u, lines = _trajectory(_run(name, seed, steps, "fp64"))
    ref = oracle_trajectory(name, seed, steps)
    oq, ou = ref[-1][0], ref[-1][1]
    if tol is None:
        per = [oracle_trajectory(name, seed, steps, perturb=1e-15, perturb_seed=k)[-1] for k in range(2)]
        assert rel_err(q, oq) <= 10 * max(rel_err(p[0], oq) for p in per) + 1e-9
        return
    for s in range(steps):
        assert int(lines[s][3]) == len(ref[s][2]), (name, s)
    assert rel_err(q, oq) < tol, rel_err(q, oq)
    assert rel_err(u, ou, floor=1e-3) < 100 * tol
