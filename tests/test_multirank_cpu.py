"""World-size-2 gloo test of the N>1 path on CPU: contiguous env blocks, no
collective on the data path, one all-gather of per-env summaries.

The per-rank compute here is the CPU oracle (the GPU kernels are covered by
the -m gpu tests); what is under test is the sharding and exchange logic the
bench uses on the GPU box with NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_04776_b200.sharding import env_block, gather_env_summaries, gather_summaries


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _summaries(depth, pitch, rest):
    from oracle import marker, tactile

    out = []
    for d in depth:
        c = marker.contact_center(tactile.indentation_from(d, rest), pitch)
        out.append(marker.contact_summary(c, pitch))
    return np.array(out, dtype=np.float32)


def _worker(rank, world, port, n_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _helpers import depth_batch
        from paper_2411_04776_b200 import synthetic

        depth = depth_batch(n_total, 24, 32, seed=5).numpy().astype(np.float64)
        s, e = env_block(rank, world, n_total)
        local = torch.as_tensor(_summaries(depth[s:e], synthetic.PITCH, synthetic.REST))
        full = gather_env_summaries(local, n_total) if n_total % world else gather_summaries(local)
        q.put((rank, full.numpy()))
    finally:
        dist.destroy_process_group()


def test_env_block_partition():
    for n in (0, 1, 7, 32768):
        for world in (1, 2, 4, 8):
            blocks = [env_block(r, world, n) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, d) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n_total", [8, 7])
def test_gloo_world2_gather_matches_single_process(n_total):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    env = dict(os.environ)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), env.get("PYTHONPATH", "")])
    try:
        for p in procs:
            p.start()
        res = dict(q.get(timeout=240) for _ in procs)
        for p in procs:
            p.join(timeout=60)
    finally:
        os.environ.clear()
        os.environ.update(env)
    assert all(p.exitcode == 0 for p in procs)
    from _helpers import depth_batch
    from paper_2411_04776_b200 import synthetic

    depth = depth_batch(n_total, 24, 32, seed=5).numpy().astype(np.float64)
    ref = _summaries(depth, synthetic.PITCH, synthetic.REST)
    for r in (0, 1):
        assert np.array_equal(res[r], ref)
    assert ref[:, 0].any()  # the workload has contacts
