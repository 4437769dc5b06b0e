"""Blurred-map parity for single / multi-strip plans (debug helper)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from _helpers import depth_batch, normwise, oracle_env, small_config  # noqa
from paper_2411_04776_b200 import TactilePipeline, synthetic  # noqa

h, w = int(os.environ.get("H", 48)), int(os.environ.get("W", 64))
sig = tuple(float(s) for s in os.environ.get("SIG", "1,2,4").split(","))
cfg = small_config(h, w, sigmas=sig)
n = 3
depth = depth_batch(n, h, w, seed=4)
pipe = TactilePipeline(cfg, "cuda:0")
obs = pipe.simulate(depth.cuda(), torch.zeros((n, 2), dtype=torch.float64, device="cuda"),
                    torch.zeros(n, dtype=torch.float64, device="cuda"), blurred=True)
torch.cuda.synchronize()
print("strips", pipe.ctx.tiles_per_frame, "H W", h, w, "sig", sig, "maxstrip", os.environ.get("TAC_MAX_STRIP"))
for i in range(n):
    ref = oracle_env(cfg, depth[i].numpy(), (0.0, 0.0), 0.0)
    b = obs.blurred[i].cpu().numpy()
    d = np.abs(b - ref["blurred"])
    y, x = np.unravel_index(d.argmax(), d.shape)
    rgb = np.abs(obs.rgb[i].cpu().numpy().astype(int) - ref["rgb"].astype(int))
    print(i, "blur normwise", normwise(b, ref["blurred"]), "worst at", (y, x), "rgb>1 frac", (rgb > 1).mean())
if os.environ.get("DUMP"):
    b = obs.blurred[0].cpu().numpy(); ref = oracle_env(cfg, depth[0].numpy(), (0.0, 0.0), 0.0)["blurred"]
    d = np.abs(b - ref) > 1e-4 * np.abs(ref).max()
    print("bad columns", np.where(d.any(0))[0])
    print("bad rows", np.where(d.any(1))[0])
    ind = np.clip(4e-3 - depth[0].numpy().astype(np.float64), 0, 4e-3)
    if not d.any(): sys.exit(0)
    r, c = np.argwhere(d)[0]
    print("first bad", r, c, "got", b[r, c], "ref", ref[r, c], "ind", ind[r, c])
    print("got row", b[r, :8]); print("ref row", ref[r, :8])
