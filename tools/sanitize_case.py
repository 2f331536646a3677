#!/usr/bin/env python3
"""Small invocation of every hot kernel for compute-sanitizer (racecheck /
synccheck / memcheck, one tool per run): the batched C5 path (k_batch_collide,
k_batch_warp fp64 and mixed, k_batch_sub's large-env launch forced for half the
envs), one C1 step (k_single_block) and one c2:6 step (k_single_grid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    from paper_1907_04587_b200 import BatchSolver, Scene, batch_states
    from tests.helpers import oracle_case, run_gpu

    for prec, env in (("fp64", {}), ("fp32", {}), ("fp64", {"NSD_WARP_MAX_OBJ": "20"})):
        os.environ.update(env)
        t = Scene("c5", 0)
        cfg = t.config
        cfg.precision = prec
        n = 16
        q0, u0 = batch_states("c5", 0, n, t.topology.num_coord, t.topology.num_dof)
        b = BatchSolver(t.topology, t.shapes, t.n_shapes, t.margin, t.mu_default, cfg, n, 48)
        b.set_state(q0, u0)
        for _ in range(3):
            b.step(t.h, t.gravity, torque=np.linspace(-1, 1, n * t.topology.n_joints))
        b.results()
        b.close()
        for k in env:
            del os.environ[k]
    for name in ("c1", "c2:6"):
        run_gpu(oracle_case(name, 0, 0), "fp64")
    print("sanitize case ok")


if __name__ == "__main__":
    main()
