import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from _helpers import oracle_env, small_config, normwise
from paper_2411_04776_b200 import render_heightmaps, TactilePipeline, synthetic
g = dict(np.load('/root/repo/tests/golden/raster.npz'))
cfg = small_config(48, 64)
v = torch.as_tensor(np.stack([g[f"verts_cam_{k}"] for k in (0, 1, 2)]), device="cuda")
depth = render_heightmaps(v, torch.as_tensor(g["tris_0"], device="cuda"), cfg)
shear, twist = synthetic.loads(3, 77)
pipe = TactilePipeline(cfg, "cuda")
obs = pipe.simulate(depth, torch.as_tensor(shear, device="cuda"), torch.as_tensor(twist, device="cuda"), blurred=True, contact=True)
torch.cuda.synchronize()
for i, k in enumerate((0, 1, 2)):
    ref = oracle_env(cfg, g[f"depth_{k}"].astype(np.float32), shear[i], twist[i])
    got = obs.rgb[i].cpu().numpy().astype(int)
    d = np.abs(got - ref["rgb"].astype(int)).max(-1)
    print(k, "depth equal", np.array_equal(depth[i].cpu().numpy(), g[f"depth_{k}"].astype(np.float32)),
          "bad", int((d > 1).sum()), "blur nw", normwise(obs.blurred[i].cpu().numpy(), ref["blurred"]),
          "disp nw", normwise(obs.disp[i].cpu().numpy(), ref["disp"]))
    print("   sum", obs.summary[i].cpu().numpy(), "\n   ref", ref["summary"])
    ys, xs = np.nonzero(d > 1)
    print("   rows", sorted(set(ys.tolist()))[:12], "cols", sorted(set(xs.tolist()))[:12])
