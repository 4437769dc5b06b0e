import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from _helpers import depth_batch, oracle_env, small_config
from paper_2411_04776_b200 import TactilePipeline, synthetic
cfg = small_config(48, 64)
n = 6
depth = depth_batch(n, 48, 64, seed=3, fixed_kind="sphere", pitch=synthetic.PITCH)
shear, twist = synthetic.loads(n, 5)
pipe = TactilePipeline(cfg, "cuda")
obs = pipe.simulate(depth.cuda(), torch.as_tensor(shear, device="cuda"), torch.as_tensor(twist, device="cuda"), blurred=True, contact=True)
torch.cuda.synchronize()
for i in range(n):
    ref = oracle_env(cfg, depth[i].numpy(), shear[i], twist[i])
    got = obs.rgb[i].cpu().numpy().astype(int)
    d = np.abs(got - ref["rgb"].astype(int)).max(-1)
    ys, xs = np.nonzero(d > 1)
    print(i, "bad px", len(ys), "rows", sorted(set(ys.tolist()))[:20], "cols", sorted(set(xs.tolist()))[:20])
    print("  summary", obs.summary[i].cpu().numpy(), "ref", ref["summary"])
    print("  disp diff", np.abs(obs.disp[i].cpu().numpy() - ref["disp"]).max())
