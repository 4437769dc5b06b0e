"""Sweep HostStreamer (streams, chunk) for the e2e host-buffer path (diagnostics)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_04776_b200 import TactilePipeline, synthetic  # noqa: E402
from paper_2411_04776_b200.hostio import HostStreamer, host_observation  # noqa: E402

cfg, n = synthetic.baseline_config(2, 0)
h, w = cfg.sensor.image_size
pipe = TactilePipeline(cfg, "cuda")
p = synthetic.indenters(n, h, w, 10)
depth = synthetic.height_maps(p, h, w, device="cuda", dtype=torch.float32, chunk=512)
sh, tw = synthetic.loads(n, 20)
dh = depth.cpu().pin_memory()
shh = torch.as_tensor(sh).pin_memory()
twh = torch.as_tensor(tw).pin_memory()
out = host_observation(pipe, n)
for ns in (2, 3, 4):
    for chunk in (256, 512, 1024):
        st = HostStreamer(pipe, chunk, n_streams=ns)
        for _ in range(2):
            st.run(dh, shh, twh, out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            st.run(dh, shh, twh, out)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"streams {ns} chunk {chunk}: {n / dt:.0f} frames/s  ({dt * 1e3:.1f} ms/step)", flush=True)
        del st
        torch.cuda.empty_cache()
