"""The batched hot path: depth maps -> RGB tactile images + marker fields.

``TactilePipeline.simulate`` is one ``tac_pipeline`` call for all envs: the
batched equivalent of the per-sensor loop of ``Environment._observe``
(REF/envs.py:1156-1209) -- including the ``add_shadows`` march when the
config turns shadows on -- followed by the marker-dot splat of
``render_markers`` (REF/marker.py:203-234).
"""

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from .config import PipelineConfig
from .context import _ptr, context_for, require
from .errors import InvalidArgumentError

SUMMARY_FIELDS = ("in_contact", "area", "cx", "cy", "dmax", "force", "nonfinite", "pad")


@dataclass
class Observation:
    """Per-env outputs of one step (device tensors, caller-owned)."""

    rgb: torch.Tensor  # [N, H, W, 3] uint8
    disp: Optional[torch.Tensor]  # [N, rows, cols, 2] float32, metres
    summary: Optional[torch.Tensor]  # [N, 8] float32 (SUMMARY_FIELDS)
    contact: Optional[torch.Tensor] = None  # [N, 8] float64 LoadState of contact_center
    blurred: Optional[torch.Tensor] = None  # [N, H, W] float32 smoothed indentation
    saturated: Optional[torch.Tensor] = None  # [N] int32 channel values the [0, 255] clip changed


class TactilePipeline:
    """One sensor model on one GPU; call ``simulate`` once per control step."""

    def __init__(self, cfg: PipelineConfig, device=None):
        self.cfg = cfg
        self.ctx = context_for(cfg, device)
        self.device = self.ctx.device
        self.H, self.W = self.ctx.H, self.ctx.W
        self.rows, self.cols = self.ctx.rows, self.ctx.cols

    # -- buffers ---------------------------------------------------------------
    def allocate(self, n_env, *, blurred=False, contact=False, saturation=False):
        d = self.device
        return Observation(
            rgb=torch.empty((n_env, self.H, self.W, 3), dtype=torch.uint8, device=d),
            disp=torch.empty((n_env, self.rows, self.cols, 2), dtype=torch.float32, device=d),
            summary=torch.empty((n_env, 8), dtype=torch.float32, device=d),
            contact=torch.empty((n_env, 8), dtype=torch.float64, device=d) if contact else None,
            blurred=torch.empty((n_env, self.H, self.W), dtype=torch.float32, device=d) if blurred else None,
            saturated=torch.empty((n_env,), dtype=torch.int32, device=d) if saturation else None,
        )

    def new_state(self, n_env):
        """Zero LoadState per env (REF/marker.py:68-70), fp64 [N, 8]."""
        return torch.zeros((n_env, 8), dtype=torch.float64, device=self.device)

    # -- the fused step ----------------------------------------------------------
    def simulate(
        self,
        depth,
        shear=None,
        twist=None,
        *,
        state=None,
        pose_delta=None,
        input_kind="depth",
        out: Optional[Observation] = None,
        blurred=False,
        contact=False,
        splat=True,
        saturation=False,
    ) -> Observation:
        """Run the whole path for every env in one ``tac_pipeline`` call
        (band blur + band shade kernels and a per-env epilogue).

        depth: [N, H, W] float32 on the pipeline's device (a HeightMap batch
        when input_kind == "depth", an IndentationMap batch when
        "indentation").  Loads: either ``shear`` [N, 2] (m) + ``twist`` [N]
        (rad) given directly (BASELINE configs[2]), or ``state`` [N, 8] fp64
        LoadState advanced in place by ``pose_delta`` [N, 3] = (dx, dy,
        rotvec_z) through ``track_load`` (REF/marker.py:124-140).
        ``saturation=True`` also counts, per env, the channel values the
        [0, 255] clip changed (``out.saturated`` and summary field 7: the
        count behind the reference's >1 % warning, REF/optical.py:246-249).
        """
        d = self.device
        n = int(depth.shape[0]) if isinstance(depth, torch.Tensor) and depth.dim() == 3 else -1
        require(depth, "depth", torch.float32, (n, self.H, self.W), d)
        if input_kind not in ("depth", "indentation"):
            raise InvalidArgumentError("input_kind must be 'depth' or 'indentation'")
        if out is None:
            out = self.allocate(n, blurred=blurred, contact=contact, saturation=saturation)
        require(out.rgb, "rgb", torch.uint8, (n, self.H, self.W, 3), d)
        if out.disp is not None:
            require(out.disp, "disp", torch.float32, (n, self.rows, self.cols, 2), d)
        if out.summary is not None:
            require(out.summary, "summary", torch.float32, (n, 8), d)
        if out.contact is not None:
            require(out.contact, "contact", torch.float64, (n, 8), d)
        if out.blurred is not None:
            require(out.blurred, "blurred", torch.float32, (n, self.H, self.W), d)
        if out.saturated is not None:
            require(out.saturated, "saturated", torch.int32, (n,), d)
        a = _lib.TacPipelineArgs()
        a.in_ = depth.data_ptr()
        a.input_kind = _lib.TAC_INPUT_DEPTH if input_kind == "depth" else _lib.TAC_INPUT_INDENTATION
        if state is not None:
            require(state, "state", torch.float64, (n, 8), d)
            require(pose_delta, "pose_delta", torch.float64, (n, 3), d)
            a.load_mode = _lib.TAC_LOAD_TRACK
            a.state = state.data_ptr()
            a.pose_delta = pose_delta.data_ptr()
        else:
            if shear is None or twist is None:
                raise InvalidArgumentError("give shear and twist, or state and pose_delta")
            require(shear, "shear", torch.float64, (n, 2), d)
            require(twist, "twist", torch.float64, (n,), d)
            a.load_mode = _lib.TAC_LOAD_GIVEN
            a.shear = shear.data_ptr()
            a.twist = twist.data_ptr()
        a.rgb = out.rgb.data_ptr()
        a.disp = out.disp.data_ptr() if out.disp is not None else None
        a.summary = out.summary.data_ptr() if out.summary is not None else None
        a.contact = out.contact.data_ptr() if out.contact is not None else None
        a.blurred = out.blurred.data_ptr() if out.blurred is not None else None
        a.saturated = out.saturated.data_ptr() if out.saturated is not None else None
        a.splat = 1 if splat else 0
        a.workspace = self.ctx.workspace(n).data_ptr()
        a.n_env = n
        _lib.check(self.ctx.lib.tac_pipeline(self.ctx.handle, ctypes.byref(a), self.ctx.stream()),
                   "tac_pipeline")
        return out

    def launch_args(self, depth, shear, twist, out):
        """Prebuilt argument block for tight loops / CUDA-graph capture."""
        a = _lib.TacPipelineArgs()
        a.in_ = depth.data_ptr()
        a.input_kind = _lib.TAC_INPUT_DEPTH
        a.load_mode = _lib.TAC_LOAD_GIVEN
        a.shear = shear.data_ptr()
        a.twist = twist.data_ptr()
        a.rgb = out.rgb.data_ptr()
        a.disp = out.disp.data_ptr() if out.disp is not None else None
        a.summary = out.summary.data_ptr() if out.summary is not None else None
        a.splat = 1
        a.workspace = self.ctx.workspace(depth.shape[0]).data_ptr()
        a.n_env = int(depth.shape[0])
        return a

    def launch(self, args):
        _lib.check(self.ctx.lib.tac_pipeline(self.ctx.handle, ctypes.byref(args), self.ctx.stream()),
                   "tac_pipeline")

    def path(self):
        """TAC_PATH_* tac_pipeline takes for aligned input (diagnostics)."""
        return int(self.ctx.lib.tac_pipeline_path(self.ctx.handle))

    def path_name(self):
        return {_lib.TAC_PATH_BAND: "band", _lib.TAC_PATH_FUSED: "fused",
                _lib.TAC_PATH_STREAM: "stream"}.get(self.path(), "?")

    def kernel_names(self):
        """Kernel of each timing slot [blur, shade, epilogue] of this path."""
        path = self.path()
        if path == _lib.TAC_PATH_FUSED:
            return ["frame_kernel (fused)"] + (["", "", "shadow_kernel"] if self.cfg.shadows else [])
        blur = "stream_blur_kernel" if path == _lib.TAC_PATH_STREAM else "band_blur_kernel"
        shade = "band_shade_kernel<f16 LUT>" if self.cfg.lut_dtype == "f16" else "band_shade_kernel"
        names = [blur, shade, "env_epilogue_kernel"]
        return names + ["shadow_kernel"] if self.cfg.shadows else names

    def launches_per_call(self, n_env):
        """Kernel launches one tac_pipeline call makes (diagnostics)."""
        return int(self.ctx.lib.tac_pipeline_launches(self.ctx.handle, int(n_env)))

    def profile(self, args, iters=10):
        """Mean per-call CUDA-event milliseconds of each kernel kind
        [blur (or the fused frame kernel), shade, per-env epilogue, shadow]."""
        ms = (ctypes.c_float * _lib.TAC_TIMING_KINDS)()
        _lib.check(self.ctx.lib.tac_pipeline_profile(self.ctx.handle, ctypes.byref(args), self.ctx.stream(),
                                                     int(iters), ms), "tac_pipeline_profile")
        return [float(v) for v in ms]

    def timing_begin(self, max_calls):
        """Record kernel-boundary CUDA events in the next ``max_calls`` pipeline
        calls (diagnostics; no synchronisation inside the calls)."""
        _lib.check(self.ctx.lib.tac_timing_begin(self.ctx.handle, int(max_calls)), "tac_timing_begin")

    def timing_end(self):
        """(mean per-call ms of [blur, shade, epilogue, shadow], calls recorded)."""
        ms = (ctypes.c_float * _lib.TAC_TIMING_KINDS)()
        calls = ctypes.c_int32(0)
        _lib.check(self.ctx.lib.tac_timing_end(self.ctx.handle, ms, ctypes.byref(calls)), "tac_timing_end")
        return [float(v) for v in ms], int(calls.value)


__all__ = ["TactilePipeline", "Observation", "SUMMARY_FIELDS", "_ptr"]
