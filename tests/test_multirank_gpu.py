"""World-size-2 run of the product path with both ranks on cuda:0 (gloo for
the exchange): each rank pushes its ``env_block`` half of a configs[2]-shaped
batch through ``TactilePipeline`` and the summaries are all-gathered.  The
gathered summaries and every rank's RGB / displacement block must equal one
full-batch call (envs are independent, REF/envs.py:1305-1334).

The ranks never wait on each other inside a kernel (no collective on the data
path), so sharing one GPU is a faithful stand-in for the host logic of
bench.py --gpus 2."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_TOTAL = 13  # ragged split: 7 + 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_04776_b200 import TactilePipeline, synthetic
        from paper_2411_04776_b200.sharding import env_block, gather_env_summaries

        cfg, n, params, shear, twist = synthetic.workload(2, 3, n_total=N_TOTAL)
        s, e = env_block(rank, world, n)
        dev = torch.device("cuda", 0)
        depth = synthetic.height_maps(params.subset(slice(s, e)), 240, 320, device=dev, dtype=torch.float32)
        pipe = TactilePipeline(cfg, dev)
        obs = pipe.simulate(depth, torch.as_tensor(shear[s:e], device=dev), torch.as_tensor(twist[s:e], device=dev))
        torch.cuda.synchronize()
        full = gather_env_summaries(obs.summary.cpu(), n)
        q.put((rank, full.numpy(), obs.rgb.cpu().numpy(), obs.disp.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_full_batch():
    import torch.multiprocessing as mp

    from paper_2411_04776_b200 import TactilePipeline, synthetic
    from paper_2411_04776_b200.sharding import env_block

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, summ, rgb, disp = q.get(timeout=600)
        res[r] = (summ, rgb, disp)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)

    cfg, n, params, shear, twist = synthetic.workload(2, 3, n_total=N_TOTAL)
    dev = torch.device("cuda", 0)
    depth = synthetic.height_maps(params, 240, 320, device=dev, dtype=torch.float32)
    pipe = TactilePipeline(cfg, dev)
    ref = pipe.simulate(depth, torch.as_tensor(shear, device=dev), torch.as_tensor(twist, device=dev))
    torch.cuda.synchronize()
    for r in (0, 1):
        s, e = env_block(r, 2, n)
        summ, rgb, disp = res[r]
        assert np.array_equal(summ, ref.summary.cpu().numpy())
        assert np.array_equal(rgb, ref.rgb[s:e].cpu().numpy())
        assert np.array_equal(disp, ref.disp[s:e].cpu().numpy())
    assert ref.summary[:, 0].sum() > 0  # the batch has contacts
