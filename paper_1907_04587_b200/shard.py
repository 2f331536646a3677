"""Environment sharding for the batched path.

The C5 workload partitions by environment: rank r of N owns the contiguous
global env range [r*E, (r+1)*E). Every per-env input derives from the GLOBAL
env id — the builder seed (`build_c5_ant(env_id)`, initial joint rates from
mt19937(env_id)) and the action stream — so env i's trajectory is the same for
every N and no data-path collective exists (weak scaling). Single scenes
(C1–C4) are not sharded: N ranks are N independent replicas.
"""
from __future__ import annotations

import numpy as np

__all__ = ["env_range", "shard_states", "action_torques"]


def env_range(rank: int, world_size: int, envs_per_rank: int) -> tuple[int, int]:
    """(first global env id, env count) owned by `rank`."""
    if not (0 <= rank < world_size) or envs_per_rank < 0:
        raise ValueError(f"bad shard: rank {rank} of {world_size}, {envs_per_rank} envs per rank")
    return rank * envs_per_rank, envs_per_rank


def shard_states(name: str, rank: int, world_size: int, envs_per_rank: int, num_coord: int, num_dof: int):
    """Initial (q, u) of the rank's envs, seeded by global env id (one C call)."""
    from . import batch_states

    env0, n = env_range(rank, world_size, envs_per_rank)
    return batch_states(name, env0, n, num_coord, num_dof)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def action_torques(env_ids, steps, n_joints: int) -> np.ndarray:
    """Joint torques U(-1, 1), shape (len(steps), len(env_ids), n_joints): a
    counter-based hash of (global env id, step, joint), so an env's actions are
    the same whichever rank owns it. `steps` may be an int or a sequence."""
    e = np.asarray(env_ids, dtype=np.uint64).reshape(1, -1, 1)
    s = np.atleast_1d(np.asarray(steps, dtype=np.uint64)).reshape(-1, 1, 1)
    j = np.arange(n_joints, dtype=np.uint64).reshape(1, 1, -1)
    with np.errstate(over="ignore"):
        key = (e << np.uint64(32)) ^ (s << np.uint64(8)) ^ j
        bits = _splitmix64(key) >> np.uint64(11)  # 53 random bits
    out = bits.astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0
    return out[0] if np.ndim(steps) == 0 else out
