"""Run one fused step on a seeded batch (debug / sanitizer helper)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from _helpers import depth_batch  # noqa: E402
from paper_2411_04776_b200 import TactilePipeline, synthetic  # noqa: E402

cfg_i = int(os.environ.get("CFG", 2))
n = int(os.environ.get("N", 12))
kind = os.environ.get("KIND") or None
cfg, _ = synthetic.baseline_config(cfg_i)
h, w = cfg.sensor.image_size
depth = depth_batch(n, h, w, seed=21, fixed_kind=kind)
shear, twist = synthetic.loads(n, 22)
pipe = TactilePipeline(cfg, "cuda:0")
obs = pipe.simulate(depth.cuda(), torch.as_tensor(shear, device="cuda"), torch.as_tensor(twist, device="cuda"),
                    blurred=True, contact=True)
torch.cuda.synchronize()
print("ok", obs.summary[:, 0].tolist())
