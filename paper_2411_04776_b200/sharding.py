"""Env sharding across GPUs (one process per GPU) and the optional summary
all-gather (BASELINE.json configs[4]).

Environments are independent: the reference's ``VectorEnv`` shares nothing
between envs (REF/envs.py:1305-1334) and serial equals threaded bit-for-bit
(REF/tests/test_envs.py:250-268).  So the hot path has NO collective: rank r
owns the contiguous env block ``env_block(r, world, n_total)``.  The only
exchange is the once-per-step all-gather of the per-env [N, 8] contact
summaries for a centralised learner, done with
``torch.distributed.all_gather_into_tensor`` (NCCL over NVLink on the GPU box,
gloo in the CPU tests).
"""

import torch
import torch.distributed as dist


def env_block(rank: int, world: int, n_total: int):
    """[start, stop) of the envs owned by ``rank`` (balanced, contiguous)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(int(n_total), world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gather_summaries(local: torch.Tensor, out: torch.Tensor = None, group=None, async_op=False):
    """All-gather equal-size [n_local, 8] summary blocks into [world*n_local, 8].

    Equal block sizes are required by ``all_gather_into_tensor``; callers
    with a ragged split pad to ``ceil(n_total/world)`` rows.
    """
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
    work = dist.all_gather_into_tensor(out, local.contiguous(), group=group, async_op=async_op)
    return (out, work) if async_op else out


def gather_env_summaries(local: torch.Tensor, n_total: int, group=None):
    """All-gather per-env [n_local, 8] summaries of contiguous ``env_block``
    shards into the global [n_total, 8] in env order.  Ragged splits are
    padded to ``ceil(n_total / world)`` rows for ``all_gather_into_tensor``
    and stripped afterwards (bench.py keeps padded buffers resident instead)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    blk = -(-int(n_total) // world)
    s, e = env_block(rank, world, n_total)
    if local.shape[0] != e - s:
        raise ValueError(f"rank {rank} holds {local.shape[0]} envs, env_block says {e - s}")
    pad = torch.zeros((blk,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: e - s] = local
    full = gather_summaries(pad, group=group)
    parts = [full[r * blk: r * blk + (env_block(r, world, n_total)[1] - env_block(r, world, n_total)[0])]
             for r in range(world)]
    return torch.cat(parts, 0)
