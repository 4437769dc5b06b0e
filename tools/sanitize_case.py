"""Small end-to-end run of every kernel family (pipeline in both load modes,
z-buffer) for checkers such as compute-sanitizer (one tool per invocation;
closed on the round-1 GPU pool).

    python tools/sanitize_case.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _helpers import depth_batch, small_config  # noqa: E402
from paper_2411_04776_b200 import (DEFAULT_PYRAMID, TactilePipeline, levels_from_kernel_sizes,  # noqa: E402
                                   render_heightmaps, synthetic)

import dataclasses  # noqa: E402

cases = [(synthetic.baseline_config(2, 0)[0], 3),            # stream blur, sigma 1,2,4
         (small_config(48, 64), 2),
         (small_config(37, 480, grid=(3, 5)), 2),             # column strips, padded shade rows
         (small_config(48, 64, shadows=True), 2),             # tiled shadow march, stream path
         (dataclasses.replace(small_config(48, 64), lut_dtype="f16"), 2),
         (small_config(40, 56, shadows=True), 2),             # L1 shadow march + fused-path fallback
         (synthetic.baseline_config(3, 0)[0], 2),            # 480x640 sigma 1,2,4,8: wide strips, R4 = 24
         (small_config(50, 640, grid=(4, 6),                  # REF DEFAULT_PYRAMID, strips, ragged rows
                       levels=levels_from_kernel_sizes(DEFAULT_PYRAMID)), 2),
         (dataclasses.replace(small_config(48, 64), kernel_path="band"), 2)]  # band blur kernel
for cfg, n in cases:
    h, w = cfg.sensor.image_size
    pipe = TactilePipeline(cfg, "cuda")
    d = depth_batch(n, h, w, seed=3).cuda()
    sh, tw = synthetic.loads(n, 4)
    obs = pipe.simulate(d, torch.as_tensor(sh, device="cuda"), torch.as_tensor(tw, device="cuda"), blurred=True)
    state = pipe.new_state(n)
    obs = pipe.simulate(d, state=state, pose_delta=torch.zeros((n, 3), dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
# z-buffer
v = torch.rand((2, 30, 3), dtype=torch.float64, device="cuda") * 1e-3
v[..., 2] += 3.5e-3
t = torch.randint(0, 30, (40, 3), device="cuda")
render_heightmaps(v, t, small_config(48, 64))
torch.cuda.synchronize()
print("sanitize case ok")
