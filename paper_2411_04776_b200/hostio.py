"""Host-buffer entry point: the reference-facing call with host arrays.

The reference returns host-owned observations (REF/envs.py:654-665) and its
offline driver reads maps from files (REF/cli.py:274-301), so a drop-in
caller holds HOST buffers.  ``simulate_host`` streams env chunks through the
GPU on two CUDA streams: H2D of chunk i+1 and D2H of chunk i-1 overlap the
kernels of chunk i.
"""

import torch

from .pipeline import Observation, TactilePipeline


class HostStreamer:
    """Reusable device staging for ``simulate_host`` on one pipeline."""

    def __init__(self, pipe: TactilePipeline, chunk: int, n_streams: int = 2):
        self.pipe = pipe
        self.chunk = int(chunk)
        d = pipe.device
        self.streams = [torch.cuda.Stream(d) for _ in range(n_streams)]
        self.bufs = []
        for _ in range(n_streams):
            self.bufs.append(
                dict(
                    depth=torch.empty((chunk, pipe.H, pipe.W), dtype=torch.float32, device=d),
                    shear=torch.empty((chunk, 2), dtype=torch.float64, device=d),
                    twist=torch.empty((chunk,), dtype=torch.float64, device=d),
                    out=pipe.allocate(chunk),
                )
            )

    def run(self, depth_h, shear_h, twist_h, out_h: Observation):
        """depth_h [N,H,W] f32, shear_h [N,2] f64, twist_h [N] f64 (pinned host);
        out_h: host Observation (pinned).  Returns out_h after a full sync."""
        n = depth_h.shape[0]
        cur = torch.cuda.current_stream(self.pipe.device)
        for s in self.streams:
            s.wait_stream(cur)
        for k, start in enumerate(range(0, n, self.chunk)):
            stop = min(n, start + self.chunk)
            m = stop - start
            s = self.streams[k % len(self.streams)]
            b = self.bufs[k % len(self.streams)]
            with torch.cuda.stream(s):
                dd = b["depth"][:m]
                dd.copy_(depth_h[start:stop], non_blocking=True)
                b["shear"][:m].copy_(shear_h[start:stop], non_blocking=True)
                b["twist"][:m].copy_(twist_h[start:stop], non_blocking=True)
                o = b["out"]
                view = Observation(rgb=o.rgb[:m], disp=o.disp[:m], summary=o.summary[:m])
                self.pipe.simulate(dd, b["shear"][:m], b["twist"][:m], out=view)
                out_h.rgb[start:stop].copy_(view.rgb, non_blocking=True)
                out_h.disp[start:stop].copy_(view.disp, non_blocking=True)
                out_h.summary[start:stop].copy_(view.summary, non_blocking=True)
        for s in self.streams:
            cur.wait_stream(s)
        return out_h


def host_observation(pipe: TactilePipeline, n: int) -> Observation:
    pin = dict(pin_memory=True)
    return Observation(
        rgb=torch.empty((n, pipe.H, pipe.W, 3), dtype=torch.uint8, **pin),
        disp=torch.empty((n, pipe.rows, pipe.cols, 2), dtype=torch.float32, **pin),
        summary=torch.empty((n, 8), dtype=torch.float32, **pin),
    )


def simulate_host(pipe: TactilePipeline, depth_h, shear_h, twist_h, chunk=512) -> Observation:
    """One-shot convenience wrapper (allocates staging; use HostStreamer in loops)."""
    out = host_observation(pipe, depth_h.shape[0])
    HostStreamer(pipe, min(chunk, max(1, depth_h.shape[0]))).run(depth_h, shear_h, twist_h, out)
    torch.cuda.current_stream(pipe.device).synchronize()
    return out
