#!/usr/bin/env python
"""Throughput bench of the B200 tactile path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]
    torchrun --nproc-per-node N bench.py --gpus N ...   (bench.py --gpus N > 1 launches this itself)

Workload (default): BASELINE configs[4] -- 32768 envs of 240x320 synthetic
height maps (sphere / cylinder / cube edge / Perlin plate, penetration
U(0, 1.2 mm)), sigma (1,2,4) pyramid, 125x180 random LUT, U[80,160]
background, 7x9 markers with random shear/twist, dots r=3, split evenly over
the N GPUs by ``sharding.env_block`` (strong scaling: N=1 runs all 32768 envs
on one GPU).  One step = one ``tac_pipeline`` call over the rank's env block
and, for N>1, the NCCL all-gather of the [32768, 8] contact summaries (on a
side stream, inside the timed region).  ``--config 1|2|3`` runs the other
BASELINE configs the same way (their global env counts).

Prints ONE JSON line (rank 0).
"""

import argparse
import json
import math
import multiprocessing as mproc
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tactile frames/s (RGB+markers)"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json configs[i] (1..4)")
    ap.add_argument("--envs", type=int, default=0, help="override the global env count")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline sample (wall s)")
    ap.add_argument("--ref-seconds", type=float, default=90.0, help="--impl reference total budget (wall s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shadows", action="store_true", help="add_shadows on (REF/optical.py:261-300)")
    ap.add_argument("--lut-dtype", default="f32", choices=["f32", "f16"])
    ap.add_argument("--kernel-path", default="auto", choices=["auto", "stream", "band", "fused"])
    ap.add_argument("--chunk-envs", type=int, default=0, help="envs per blur/shade launch pair (0 = library default)")
    ap.add_argument("--seed", type=int, default=0)
    return ap.parse_args()


def bench_config(a):
    """(PipelineConfig, n_total, params, shear, twist) of the run's workload."""
    import dataclasses

    from paper_2411_04776_b200 import synthetic

    cfg, n, params, shear, twist = synthetic.workload(a.config, a.seed, a.envs or None)
    over = dict(lut_dtype=a.lut_dtype, kernel_path=a.kernel_path, chunk_envs=a.chunk_envs)
    if a.shadows:
        over.update(light_dirs=default_light_dirs(), shadow_factor=0.6)
    return dataclasses.replace(cfg, **over), n, params, shear, twist


def default_light_dirs():
    """tacsim default_lighting() directions (REF/optical.py:68-79): three lights
    120 degrees apart in azimuth at 35 degrees elevation, unit length."""
    el = math.radians(35.0)
    d = np.array([[math.cos(el) * math.cos(t), math.cos(el) * math.sin(t), math.sin(el)]
                  for t in np.deg2rad([0.0, 120.0, 240.0])])
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def workload_name(a):
    return f"configs[{a.config}]" + (" + shadows" if a.shadows else "")


# --------------------------------------------------------------------------- CPU arm
_W = {}


def _cpu_init(a, env_ids):
    """Pool initializer: one single-threaded process holding a few frames of
    the GPU run's own workload (env indices ``env_ids``, same seeds)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    import torch

    torch.set_num_threads(1)
    from oracle.fast import FastOracle
    from paper_2411_04776_b200 import synthetic

    cfg, n, params, shear, twist = bench_config(a)
    h, w = cfg.sensor.image_size
    # each worker takes its own share of the sample (by process start order)
    ident = mproc.current_process()._identity
    k = (ident[0] - 1) if ident else 0
    mine = env_ids[k % len(env_ids)]
    _W["depth"] = synthetic.height_maps(params.subset(mine), h, w, dtype=torch.float64).numpy()
    _W["shear"], _W["twist"] = shear[mine], twist[mine]
    _W["orc"] = FastOracle(cfg)
    _W["orc"].run(_W["depth"][0], _W["shear"][0], _W["twist"][0])  # warm


def _cpu_job(count):
    """Run `count` frames of the oracle port; returns (frames, seconds)."""
    d, sh, tw, orc = _W["depth"], _W["shear"], _W["twist"], _W["orc"]
    t0 = time.perf_counter()
    for i in range(count):
        k = i % len(d)
        orc.run(d[k], sh[k], tw[k])
    return count, time.perf_counter() - t0


class CpuArm:
    """A process pool (one single-threaded worker per host core) timing the
    oracle port of the reference CPU path on frames of the bench workload:
    worker k holds envs sample[k::cores] (an evenly strided sample of all
    envs, so every indenter kind and pose mix is represented)."""

    def __init__(self, a, cores, worker_frames=8):
        cfg, n, *_ = bench_config(a)
        self.cores = cores
        k = min(n, cores * worker_frames)
        sample = np.unique(np.linspace(0, n - 1, k).round().astype(np.int64))
        self.env_ids = [sample[c::cores] for c in range(cores) if len(sample[c::cores])]
        self.n_sample = len(sample)
        ctx = mproc.get_context("spawn")
        self.pool = ctx.Pool(cores, initializer=_cpu_init, initargs=(a, self.env_ids))
        self.per_frame = max(r[1] / r[0] for r in self.pool.map(_cpu_job, [2] * cores))

    def step(self, frames_per_core):
        """Aggregate frames/s over all cores for one bounded sample."""
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_job, [frames_per_core] * self.cores)
        wall = time.perf_counter() - t0
        frames = sum(r[0] for r in res)
        return frames / wall, statistics.mean(r[0] / r[1] for r in res), wall, frames

    def describe(self, a, fpc):
        return (f"{self.cores}x{fpc} frames per step, cycling {self.n_sample} distinct envs (an even stride "
                f"over the {workload_name(a)} workload, same seeds as the GPU run); oracle port "
                "(scipy.ndimage.gaussian_filter as REF/tactile.py:219, numpy gradient/LUT/markers as "
                "REF/optical.py:160-250, REF/marker.py:103-234" + (", add_shadows REF/optical.py:261-300" if a.shadows
                                                                  else "") + "), f64")

    def close(self):
        self.pool.close()
        self.pool.join()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- helpers
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.02):
        self.samples, self.reasons, self.stop_evt = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.period = period
        self.th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_evt.set()
        if self.nv:
            self.th.join()

    def result(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fma_per_frame(cfg):
    """Dense FMA count per frame of the separable pyramid: per level a
    vertical and a horizontal pass of (2r+1) taps over every pixel (zero
    columns the kernels skip exactly are counted: "dense equivalent")."""
    h, w = cfg.sensor.image_size
    return sum(2 * (2 * r + 1) * h * w for _, r in cfg.levels if r)


def algorithmic_bytes(cfg):
    """Whole path, per frame: depth in (fp32) + RGB out (u8) + marker field + summary."""
    h, w = cfg.sensor.image_size
    r, c = cfg.sensor.marker_grid
    return 4 * h * w + 3 * h * w + 8 * r * c + 32


def kernel_bytes(cfg, pipe):
    """Algorithmic HBM bytes per frame of each kernel kind of the pipeline
    call, in the order tac_timing_end reports them [blur, shade, epilogue]
    (DESIGN.md §5): blur = depth in + blurred out + band partials; shade =
    blurred in + RGB out (the LUT and background are shared, L2-resident);
    epilogue = partials in + marker field + summary out + dot pixels RMW."""
    h, w = cfg.sensor.image_size
    r, c = cfg.sensor.marker_grid
    bands = -(-h // 16)
    rr = cfg.dot_radius
    dot_px = sum(1 for dy in range(-rr, rr + 1) for dx in range(-rr, rr + 1) if dx * dx + dy * dy <= rr * rr)
    names = pipe.kernel_names()
    shadows = bool(cfg.shadows)
    per = {"stream_blur_kernel": 4 * h * w + 4 * h * w + 64,
           "band_blur_kernel": 4 * h * w + 4 * h * w + 64 * bands,
           "band_shade_kernel": 4 * h * w + 3 * h * w + (4 * h * w if shadows else 0),
           "env_epilogue_kernel": 64 * bands + 8 * r * c + 32 + 3 * dot_px * r * c,
           "shadow_kernel": 4 * h * w + 4 * h * w,  # depth in, factor out
           "frame_kernel (fused)": algorithmic_bytes(cfg)}
    per["band_shade_kernel<f16 LUT>"] = per["band_shade_kernel"]
    return {n: per[n] for n in names if n}


# --------------------------------------------------------------------------- arms
def base_line(a, world, n_total):
    """Keys shared by both arms' JSON lines."""
    from paper_2411_04776_b200.sharding import env_block

    cfg = bench_config(a)[0]
    h, w = cfg.sensor.image_size
    return {
        "metric": METRIC,
        "unit": UNIT,
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "data": "synthetic (seeded indenter height maps; BASELINE names no dataset)",
        "config": {
            "workload": workload_name(a),
            "global_envs": n_total,
            "envs_per_gpu": env_block(0, world, n_total)[1],
            "H": h, "W": w,
            "sigmas": [s for s, _ in cfg.levels],
            "lut_bins": list(cfg.lut.shape[:2]),
            "lut_dtype": cfg.lut_dtype,
            "markers": list(cfg.sensor.marker_grid),
            "dot_radius": cfg.dot_radius,
            "shadows": bool(cfg.shadows),
        },
    }


# --------------------------------------------------------------------------- arms
def run_reference(a, rank, world):
    """--impl reference: the oracle port of the reference CPU path on all host
    cores, each step a bounded sample of the same workload so the whole run
    stays within minutes.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    cfg, n_total, *_ = bench_config(a)
    cores = host_cores()
    arm = CpuArm(a, cores)
    budget = max(0.5, a.ref_seconds / max(1, a.steps + a.warmup))  # wall seconds per step
    fpc = max(1, int(budget / arm.per_frame))
    for _ in range(a.warmup):
        arm.step(fpc)
    vals, walls = [], []
    for _ in range(a.steps):
        v, _, wall, _ = arm.step(fpc)
        vals.append(v)
        walls.append(wall)
    arm.close()
    v = statistics.median(vals)
    line = {"impl": "reference", **base_line(a, world, n_total)}
    line.update(value=v, ms_per_step=1e3 * statistics.median(walls), dtype="f64")
    line["config"]["parallelism"] = f"cpu x{cores} processes"
    line["config"]["frames_per_step"] = cores * fpc
    line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": arm.describe(a, fpc)}
    line["e2e"] = {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2411_04776_b200 import TactilePipeline, synthetic
    from paper_2411_04776_b200.hostio import HostStreamer, host_observation
    from paper_2411_04776_b200.sharding import env_block, gather_summaries

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg, n_total, params, shear_np, twist_np = bench_config(a)
    h, w = cfg.sensor.image_size
    e0, e1 = env_block(rank, world, n_total)
    n_env = e1 - e0
    blk = -(-n_total // world)  # all-gather block (ragged splits are padded)
    pipe = TactilePipeline(cfg, dev)

    # this rank's env block of the global workload, resident in HBM before the
    # timed region (> L2, see config.l2)
    depth = synthetic.height_maps(params.subset(slice(e0, e1)), h, w, device=dev, dtype=torch.float32, chunk=512)
    shear = torch.as_tensor(shear_np[e0:e1], device=dev)
    twist = torch.as_tensor(twist_np[e0:e1], device=dev)
    out = pipe.allocate(n_env)
    args = pipe.launch_args(depth, shear, twist, out)
    if world > 1:
        # the once-per-step NCCL all-gather of the [N, 8] summaries runs on a side
        # stream, overlapping the next step's kernels; summaries are double-buffered
        gathered = torch.empty((world * blk, 8), dtype=torch.float32, device=dev)
        summ_ab = [torch.zeros((blk, 8), dtype=torch.float32, device=dev) for _ in range(2)]
        out2 = pipe.allocate(n_env)
        out.summary, out2.summary = summ_ab[0][:n_env], summ_ab[1][:n_env]
        args_ab = [pipe.launch_args(depth, shear, twist, out), pipe.launch_args(depth, shear, twist, out2)]
        args = args_ab[0]
        side = torch.cuda.Stream(dev)
        done = [torch.cuda.Event(), torch.cuda.Event()]   # pipeline k finished (side waits)
        freed = [torch.cuda.Event(), torch.cuda.Event()]  # gather k finished (main waits before k+2)
        k_step = [0]
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)  # communicator up before anything is timed
        if rank == 0:
            print(f"nccl communicator: nranks={dist.get_world_size()} backend={dist.get_backend()}",
                  file=sys.stderr, flush=True)

    def step():
        if world == 1:
            pipe.launch(args)
            return
        k = k_step[0] & 1
        main = torch.cuda.current_stream(dev)
        if k_step[0] >= 2:
            main.wait_event(freed[k])
        pipe.launch(args_ab[k])
        done[k].record(main)
        side.wait_event(done[k])
        with torch.cuda.stream(side):
            gather_summaries(summ_ab[k], gathered)
            freed[k].record(side)
        k_step[0] += 1

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize()
    contact_frac = float((depth < cfg.sensor.gelpad_thickness - cfg.contact_threshold).float().mean())

    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # per-kernel CUDA events at the kernel boundaries of every timed call (in
    # stream, no synchronisation: the timed loop is unchanged)
    pipe.timing_begin(a.steps)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        if world > 1:
            stream.wait_stream(side)  # the last all-gather is inside the timed region
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    region_ms, region_calls = pipe.timing_end()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / a.steps
    value = n_total * a.steps / (ms / 1e3)

    # one tac_pipeline call (all its launches) bracketed by events on the launch stream
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for k0, k1 in kev:
        k0.record(stream)
        pipe.launch(args)
        k1.record(stream)
    torch.cuda.synchronize()
    k_ms = statistics.mean(k0.elapsed_time(k1) for k0, k1 in kev)
    # per-kernel durations: the in-region boundary events (summed per call over
    # its env chunks); the fused path falls back to tac_pipeline_profile
    if region_calls == a.steps:
        kern_ms, kern_src = region_ms, f"CUDA events at the kernel boundaries of the {a.steps} timed calls"
    else:
        kern_ms, kern_src = pipe.profile(args, iters=5), "tac_pipeline_profile (5 calls, in-stream events)"
    launches = pipe.launches_per_call(n_env)

    # e2e: host buffers through the public host API, copies inside the timed region
    e2e = None
    if not a.no_e2e:
        pin = dict(pin_memory=True)
        depth_h = torch.empty(tuple(depth.shape), dtype=depth.dtype, **pin)
        depth_h.copy_(depth)
        shear_h = torch.empty(tuple(shear.shape), dtype=shear.dtype, **pin)
        shear_h.copy_(shear)
        twist_h = torch.empty(tuple(twist.shape), dtype=twist.dtype, **pin)
        twist_h.copy_(twist)
        out_h = host_observation(pipe, n_env)
        streamer = HostStreamer(pipe, chunk=min(256, n_env))  # tools/e2e_sweep.py: best measured
        e_steps = max(3, min(10, a.steps // 10))
        for _ in range(2):
            streamer.run(depth_h, shear_h, twist_h, out_h)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(e_steps):
            streamer.run(depth_h, shear_h, twist_h, out_h)
        x1.record(stream)
        torch.cuda.synchronize()
        ems = x0.elapsed_time(x1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        r, c = cfg.sensor.marker_grid
        e2e = {
            "value": n_total * e_steps / (ems / 1e3),
            "unit": UNIT,
            "h2d_bytes_per_step": n_total * (4 * h * w + 16 + 8),
            "d2h_bytes_per_step": n_total * (3 * h * w + 8 * r * c + 32),
            "steps": e_steps,
            "path": "hostio.HostStreamer -> TactilePipeline.simulate (tac_pipeline C ABI), pinned host buffers",
            "h2d_gbs_per_gpu": n_env * (4 * h * w + 16 + 8) * e_steps / (ems / 1e3) / 1e9,
        }
        del depth_h, out_h

    if rank != 0:
        return
    peak, peak_kind = measured_peak()
    per_launch = algorithmic_bytes(cfg) * n_env
    step_gbs = per_launch / (k_ms / 1e3) / 1e9
    kb = kernel_bytes(cfg, pipe)
    kernels = {}
    for name, kms in zip(pipe.kernel_names(), kern_ms):
        if name and kms > 0:
            gbs = kb[name] * n_env / (kms / 1e3) / 1e9
            kernels[name] = {"ms": kms, "bytes_per_frame": kb[name], "achieved_gbs": gbs, "frac": gbs / peak}
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    achieved = kernels[dom]["achieved_gbs"]
    props = torch.cuda.get_device_properties(dev)
    clocks = clk.result()
    fma = fma_per_frame(cfg)
    sm_ghz = (clocks["sm_mhz"] or 1965) / 1e3
    fma_peak = props.multi_processor_count * 128 * sm_ghz * 1e9
    traffic = None  # dram read+write bytes per launch of the dominant kernel (ncu --set full)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath)).get(workload_name(a))
            traffic = t.get(dom) if isinstance(t, dict) else None
            if traffic is not None:
                traffic = traffic * n_env / t.get("envs", n_env)  # scale to this launch size
        except Exception:
            traffic = None
    line = base_line(a, world, n_total)
    line.update(value=value, ms_per_step=ms_step, dtype="f32")
    line["config"].update({
        "kernel_path": pipe.path_name(),
        "parallelism": f"env-sharded x{world} (sharding.env_block)" +
                       (" + NCCL all_gather(summary) on a side stream" if world > 1 else ""),
        "l2": f"inputs {n_env * h * w * 4 / 2**30:.2f} GiB per GPU > 126 MB L2 (no flush needed)",
        "contact_pixel_fraction": round(contact_frac, 4),
    })
    line["roofline"] = {
        "bound": "hbm",
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "traffic": traffic,
        "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, burst copy)",
        "kernel": dom,
        "kernel_timing": kern_src,
        "kernel_ms": kernels[dom]["ms"],
        "algorithmic_bytes_per_launch": kernels[dom]["bytes_per_frame"] * n_env,
        "kernels": kernels,
        "step": {"ms": k_ms, "algorithmic_bytes_per_frame": algorithmic_bytes(cfg),
                 "achieved_gbs": step_gbs, "frac": step_gbs / peak},
        # pyramid FMAs of a dense frame (zero columns are skipped, so "dense
        # equivalent"): over the whole step and over the blur kernel alone
        "fp32_fma": {"per_frame_dense": fma,
                     "achieved_tflops_dense_equiv": 2 * fma * n_env / (k_ms / 1e3) / 1e12,
                     "blur_kernel_tflops_dense_equiv": 2 * fma * n_env / (kern_ms[0] / 1e3) / 1e12
                     if len(kernels) > 1 else None,
                     "peak_tflops": 2 * fma_peak / 1e12},
    }
    line["gpu_launches"] = a.steps * launches
    line["clocks"] = clocks
    line["device"] = props.name
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not a.no_cpu_baseline:
        cores = host_cores()
        arm = CpuArm(a, cores)
        fpc = max(2, int(a.cpu_seconds / arm.per_frame))
        agg, per_core, wall, frames = arm.step(fpc)
        arm.close()
        line["cpu_baseline"] = {
            "value": agg, "unit": UNIT, "cores": cores, "kind": "port", "per_core": per_core,
            "sample": arm.describe(a, fpc) + f"; {frames} frames in {wall:.1f} s wall",
        }
    print(json.dumps(line), flush=True)


def relaunch(a):
    """bench.py --gpus N outside torchrun: start N ranks of this script."""
    import socket
    import subprocess

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(relaunch(a))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
