"""smooth_pyramid (blur-only kernel mode) vs oracle for a given strip plan."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from _helpers import depth_batch, normwise  # noqa
from oracle import tactile as otac  # noqa
from paper_2411_04776_b200 import IndentationMap, smooth_pyramid  # noqa
h, w = int(os.environ.get("H", 32)), int(os.environ.get("W", 64))
sig = tuple(float(s) for s in os.environ.get("SIG", "4").split(","))
ind = np.clip(4e-3 - depth_batch(2, h, w, seed=4).numpy().astype(np.float64), 0, 4e-3)
out = smooth_pyramid(IndentationMap(torch.as_tensor(ind, dtype=torch.float32, device="cuda"), 2.66e-5), sigmas=sig)
ref = otac.smooth_pyramid(ind.astype(np.float32).astype(np.float64), otac.levels_from_sigmas(sig))
for i in range(2):
    b = out.values[i].cpu().numpy()
    d = np.abs(b - ref[i]) > 1e-4 * np.abs(ref[i]).max()
    print("blur-mode", sig, "tma", os.environ.get("TAC_NO_TMA"), "nw", normwise(b, ref[i]), "bad rows", np.where(d.any(1))[0][:5], "bad cols", np.where(d.any(0))[0][:40])
