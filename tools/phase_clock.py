"""Per-row-block phase timing of the fused slot-ring kernel (diagnostics).

    python tools/phase_clock.py [--envs N] [--config 2]

Runs one configs[i] batch through TactilePipeline with tac_set_profile_buffer
on the first 64 envs and prints mean SM cycles per phase:
  blur  V      = stamp1 - stamp0   (vertical passes, incl. the post-V barrier)
        EMPTY  = stamp2 - stamp1   (refill issue + wait for a free blurred slot)
        H      = stamp3 - stamp2   (thread 0's horizontal items)
        conv   = stamp4 - stamp3   (TMA wait + conversion + barrier)
        block  = next stamp0 - stamp0
  shade wait   = stamp5 - prev stamp6 (FULL wait), work = stamp6 - stamp5
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_04776_b200 import TactilePipeline, synthetic  # noqa: E402
from paper_2411_04776_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--envs", type=int, default=1024)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--kind", default=None)
a = ap.parse_args()
cfg, _ = synthetic.baseline_config(a.config, 0)
h, w = cfg.sensor.image_size
p = synthetic.indenters(a.envs, h, w, 3, fixed_kind=a.kind)
depth = synthetic.height_maps(p, h, w, device="cuda", dtype=torch.float32)
shear, twist = synthetic.loads(a.envs, 4)
pipe = TactilePipeline(cfg, "cuda")
nb = (h + 15) // 16
npe = 64
buf = torch.zeros(npe * nb * 8, dtype=torch.int64, device="cuda")
sh = torch.as_tensor(shear, device="cuda")
tw = torch.as_tensor(twist, device="cuda")
for _ in range(3):
    pipe.simulate(depth, sh, tw)
_lib.check(_lib.load().tac_set_profile_buffer(pipe.ctx.handle, buf.data_ptr(), npe))
pipe.simulate(depth, sh, tw)
torch.cuda.synchronize()
_lib.check(_lib.load().tac_set_profile_buffer(pipe.ctx.handle, None, 0))
t = buf.view(npe, nb, 8).cpu().numpy().astype(np.float64)
blk = np.diff(t[:, :, 0], axis=1)
print(f"envs={a.envs} config={a.config} kind={a.kind} blocks/frame={nb}")
print(f"frame cycles (stamp0 first->last block + last block): {np.mean(t[:, -1, 4] - t[:, 0, 0]):.0f}")
for name, (i, j) in {"V": (0, 1), "EMPTY": (1, 2), "H": (2, 3), "conv": (3, 4), "shade work": (5, 6)}.items():
    d = t[:, :, j] - t[:, :, i]
    print(f"  {name:10s} mean {d.mean():8.0f}  median {np.median(d):8.0f}  per-block-idx {np.round(d.mean(0)).astype(int).tolist()}")
fw = t[:, 1:, 5] - t[:, :-1, 6]
print(f"  {'shade wait':10s} mean {fw.mean():8.0f}")
print(f"  {'block':10s} mean {blk.mean():8.0f}")
