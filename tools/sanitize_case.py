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
from paper_2411_04776_b200 import TactilePipeline, render_heightmaps, synthetic  # noqa: E402

for (h, w, n) in ((240, 320, 3), (48, 64, 2)):
    cfg = synthetic.baseline_config(2, 0)[0] if (h, w) == (240, 320) else small_config(h, w)
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
