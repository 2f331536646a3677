"""Env sharding across ranks on CPU: world_size-2 gloo.

Each rank builds ITS shard's initial states through the product builders
(C ABI, no GPU needed) and advances its envs with the CPU oracle; rank 0
gathers and checks that the result is bitwise identical to one process
owning all envs. This is what makes the GPU run's "env i is independent of N"
claim hold on the host side; the device side is tested by
test_gpu_batch.py::test_batch_env_offset_independent.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

E = 3  # envs per rank
STEPS = 2


def _advance(env0, n, steps, actuated):
    from oracle import oracle_py as O
    from paper_1907_04587_b200.shard import action_torques

    qs = []
    for e in range(env0, env0 + n):
        w = O.OracleWorld("c5", e)
        for s in range(steps):
            if actuated:
                w.set_joint_torques(action_torques([e], s, w.dims()["n_joints"])[0])
            assert w.step(1) == 0
        qs.append(w.state()[0])
    return np.concatenate(qs)


def _worker(rank, world, port, out_dir, actuated):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1907_04587_b200 import Scene
    from paper_1907_04587_b200.shard import env_range, shard_states

    T = Scene("c5", 0).topology
    env0, n = env_range(rank, world, E)
    q0, u0 = shard_states("c5", rank, world, E, T.num_coord, T.num_dof)
    q = _advance(env0, n, STEPS, actuated)
    parts = [torch.zeros(2 * n * T.num_coord + n * T.num_dof, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.concatenate([q0, q, u0])))
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("actuated", [False, True])
def test_two_rank_shards_match_single_process(actuated):
    from paper_1907_04587_b200 import Scene, batch_states

    world = 2
    port = 29500 + (os.getpid() % 2000) + (7 if actuated else 0)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, d, actuated), nprocs=world, join=True)
        g = np.load(os.path.join(d, "gathered.npy"))
    T = Scene("c5", 0).topology
    nc, nd = T.num_coord, T.num_dof
    q0_all, u0_all = batch_states("c5", 0, world * E, nc, nd)
    q_all = _advance(0, world * E, STEPS, actuated)
    per = 2 * E * nc + E * nd
    for r in range(world):
        blk = g[r * per:(r + 1) * per]
        sl_c = slice(r * E * nc, (r + 1) * E * nc)
        assert np.array_equal(blk[:E * nc], q0_all[sl_c])
        assert np.array_equal(blk[E * nc:2 * E * nc], q_all[sl_c])
        assert np.array_equal(blk[2 * E * nc:], u0_all[r * E * nd:(r + 1) * E * nd])


def test_env_range_validation():
    from paper_1907_04587_b200.shard import env_range

    assert env_range(3, 8, 512) == (1536, 512)
    with pytest.raises(ValueError):
        env_range(2, 2, 4)


def test_action_torques_pure_function_of_env_and_step():
    from paper_1907_04587_b200.shard import action_torques

    a = action_torques(range(0, 8), [0, 1, 2], 8)
    b = action_torques(range(4, 8), [1], 8)
    assert a.shape == (3, 8, 8) and np.array_equal(a[1, 4:], b[0])
    assert np.all(a >= -1.0) and np.all(a < 1.0) and abs(a.mean()) < 0.2


def test_oracle_action_stream_matches_host():
    """bench.py's CPU arm (oracle c5_bench) and GPU arm use the same actions."""
    from oracle import oracle_py as O
    from paper_1907_04587_b200.shard import action_torques

    a = action_torques([0, 5, 4095, 70000], [0, 3, 199], 8)
    for si, s in enumerate([0, 3, 199]):
        for ei, e in enumerate([0, 5, 4095, 70000]):
            for j in range(8):
                assert O.action_torque(e, s, j) == a[si, ei, j]
