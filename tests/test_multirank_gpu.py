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


def _nccl_worker(port, q):
    """bench.py's N>1 step loop on a one-rank NCCL communicator: the pipeline
    on the main stream, the [blk, 8] summary all-gather (device tensors,
    ``all_gather_into_tensor``) on a side stream, summaries double-buffered."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        from paper_2411_04776_b200 import TactilePipeline, synthetic
        from paper_2411_04776_b200.sharding import gather_summaries

        cfg, n, params, shear, twist = synthetic.workload(2, 5, n_total=N_TOTAL)
        depth = synthetic.height_maps(params, 240, 320, device=dev, dtype=torch.float32)
        sh, tw = torch.as_tensor(shear, device=dev), torch.as_tensor(twist, device=dev)
        pipe = TactilePipeline(cfg, dev)
        ref = pipe.simulate(depth, sh, tw).summary.clone()
        blk = n + 3  # padded block, as a ragged split pads to ceil(n_total / world)
        gathered = torch.full((blk, 8), -1.0, dtype=torch.float32, device=dev)
        summ = [torch.zeros((blk, 8), dtype=torch.float32, device=dev) for _ in range(2)]
        outs = [pipe.allocate(n), pipe.allocate(n)]
        for k in range(2):
            outs[k].summary = summ[k][:n]
        args = [pipe.launch_args(depth, sh, tw, outs[k]) for k in range(2)]
        side = torch.cuda.Stream(dev)
        main = torch.cuda.current_stream(dev)
        done = [torch.cuda.Event(), torch.cuda.Event()]
        freed = [torch.cuda.Event(), torch.cuda.Event()]
        for step in range(5):
            k = step & 1
            if step >= 2:
                main.wait_event(freed[k])
            pipe.launch(args[k])
            done[k].record(main)
            side.wait_event(done[k])
            with torch.cuda.stream(side):
                gather_summaries(summ[k], gathered)
                freed[k].record(side)
        main.wait_stream(side)
        torch.cuda.synchronize()
        q.put((dist.get_backend(), gathered[:n].cpu().numpy(), ref.cpu().numpy(), gathered[n:].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_nccl_summary_all_gather_on_a_side_stream():
    """The NCCL leg of bench.py --gpus N (all_gather_into_tensor of the
    per-env summaries on a side stream, double-buffered against the next
    step's kernels) on a one-rank communicator: this run has one GPU, so the
    collective's N>1 exchange itself stays unmeasured."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    backend, got, ref, pad = q.get(timeout=300)
    p.join(60)
    assert p.exitcode == 0
    assert backend == "nccl"
    assert np.array_equal(got, ref)
    assert not pad.any()
