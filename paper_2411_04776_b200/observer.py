"""Batched mirror of the reference's per-sensor observation step (row f3).

``Environment._observe`` (REF/envs.py:1156-1209) runs, per sensor and per
control step: ``render_heightmap`` -> ``indentation_from`` ->
``smooth_pyramid`` -> ``normals_from`` -> ``shade`` -> ``add_shadows`` ->
``contact_center`` -> ``track_load`` with the case-pose delta
``prev_cam.inverse().compose(cam)`` -> ``marker_displacements``.
``SensorObserver`` does the same for N sensors at once on one GPU: the mesh
z-buffer (``render_heightmaps``, row f2), then one ``tac_pipeline`` call in
``TAC_LOAD_TRACK`` mode that advances the per-env LoadState in place.  The
only state is the LoadState [N, 8] and the previous camera pose [N, 4, 4]
(REF/envs.py:717-734); ``reset`` zeroes them (optionally for a subset).
"""

from dataclasses import dataclass
from typing import Optional

import torch

from .config import PipelineConfig
from .errors import InvalidArgumentError
from .pipeline import Observation, TactilePipeline
from .tactile import render_heightmaps


def _rotvec_z(r: torch.Tensor) -> torch.Tensor:
    """z component of the rotation vector of rotation matrices r [N, 3, 3]
    (the yaw of REF/marker.py:137, ``rot().as_rotvec()[2]``), via the unit
    quaternion (Shepperd's branch on the largest component)."""
    t = r[:, 0, 0] + r[:, 1, 1] + r[:, 2, 2]
    d = torch.stack([r[:, 0, 0], r[:, 1, 1], r[:, 2, 2], t], dim=1)
    k = torch.argmax(d, dim=1)
    # candidate quaternions (x, y, z, w) for each largest component
    s = torch.sqrt(torch.clamp(1.0 + t, min=1e-300)) * 2.0
    qw = torch.stack([(r[:, 2, 1] - r[:, 1, 2]) / s, (r[:, 0, 2] - r[:, 2, 0]) / s,
                      (r[:, 1, 0] - r[:, 0, 1]) / s, 0.25 * s], dim=1)
    sx = torch.sqrt(torch.clamp(1.0 + r[:, 0, 0] - r[:, 1, 1] - r[:, 2, 2], min=1e-300)) * 2.0
    qx = torch.stack([0.25 * sx, (r[:, 0, 1] + r[:, 1, 0]) / sx, (r[:, 0, 2] + r[:, 2, 0]) / sx,
                      (r[:, 2, 1] - r[:, 1, 2]) / sx], dim=1)
    sy = torch.sqrt(torch.clamp(1.0 + r[:, 1, 1] - r[:, 0, 0] - r[:, 2, 2], min=1e-300)) * 2.0
    qy = torch.stack([(r[:, 0, 1] + r[:, 1, 0]) / sy, 0.25 * sy, (r[:, 1, 2] + r[:, 2, 1]) / sy,
                      (r[:, 0, 2] - r[:, 2, 0]) / sy], dim=1)
    sz = torch.sqrt(torch.clamp(1.0 + r[:, 2, 2] - r[:, 0, 0] - r[:, 1, 1], min=1e-300)) * 2.0
    qz = torch.stack([(r[:, 0, 2] + r[:, 2, 0]) / sz, (r[:, 1, 2] + r[:, 2, 1]) / sz, 0.25 * sz,
                      (r[:, 1, 0] - r[:, 0, 1]) / sz], dim=1)
    q = torch.where((k == 3)[:, None], qw, torch.where((k == 0)[:, None], qx,
                                                       torch.where((k == 1)[:, None], qy, qz)))
    q = torch.where(q[:, 3:4] < 0, -q, q)  # w >= 0: rotation angle in [0, pi]
    v = q[:, :3]
    nv = torch.linalg.norm(v, dim=1)
    angle = 2.0 * torch.atan2(nv, q[:, 3])
    scale = torch.where(nv > 0, angle / torch.clamp(nv, min=1e-300), torch.full_like(nv, 2.0))
    return v[:, 2] * scale


def pose_delta(prev: torch.Tensor, cam: torch.Tensor) -> torch.Tensor:
    """(dx, dy, rotvec_z) of prev^-1 @ cam for camera-to-world poses [N, 4, 4]
    (REF/envs.py:1178: ``prev_cam.inverse().compose(cam)``)."""
    r0, t0 = prev[:, :3, :3], prev[:, :3, 3]
    r1, t1 = cam[:, :3, :3], cam[:, :3, 3]
    r0t = r0.transpose(1, 2)
    dr = r0t @ r1
    dt = (r0t @ (t1 - t0)[..., None])[..., 0]
    return torch.stack([dt[:, 0], dt[:, 1], _rotvec_z(dr)], dim=1).contiguous()


@dataclass
class SensorObservation:
    """One step of N sensors (device tensors)."""

    outputs: Observation  # rgb, disp, summary (+ contact)
    loads: torch.Tensor  # [N, 8] fp64 LoadState after track_load
    heightmap: Optional[torch.Tensor]  # [N, H, W] fp32 depth when requested


class SensorObserver:
    """N sensors of one model on one GPU, stepped like ``Environment._observe``."""

    def __init__(self, cfg: PipelineConfig, n_env: int, device=None, *, keep_heightmap=False):
        self.pipe = TactilePipeline(cfg, device)
        self.cfg = cfg
        self.n = int(n_env)
        self.device = self.pipe.device
        self.state = self.pipe.new_state(self.n)
        self.prev_cam: Optional[torch.Tensor] = None
        self.keep_heightmap = keep_heightmap

    def reset(self, cam: torch.Tensor, mask: Optional[torch.Tensor] = None):
        """Zero LoadState (REF/marker.py:68-70) and set the previous camera
        pose, for every env or the envs where ``mask`` is true."""
        cam = self._poses(cam)
        if mask is None or self.prev_cam is None:
            self.state.zero_()
            self.prev_cam = cam.clone()
        else:
            m = mask.to(self.device, torch.bool)
            self.state[m] = 0.0
            self.prev_cam[m] = cam[m]

    def camera_poses(self, case_poses):
        """Camera-to-world poses of the sensors from their case poses [N, 4, 4]:
        ``case_pose.compose(cfg.camera_pose_in_case)`` (REF/envs.py:733-734)."""
        case = torch.as_tensor(case_poses, dtype=torch.float64, device=self.device)
        t = torch.as_tensor(self.cfg.sensor.camera_pose_matrix, device=self.device)
        return case @ t

    def _poses(self, cam):
        cam = torch.as_tensor(cam, dtype=torch.float64, device=self.device)
        if cam.shape != (self.n, 4, 4):
            raise InvalidArgumentError(f"camera poses must be [{self.n}, 4, 4]")
        return cam

    def observe(self, cam, *, depth: Optional[torch.Tensor] = None, verts_world: Optional[torch.Tensor] = None,
                tris: Optional[torch.Tensor] = None) -> SensorObservation:
        """One control step: depth maps [N, H, W] (or world-frame meshes:
        ``verts_world`` [N, V, 3] + ``tris`` [T, 3], rendered here) seen from
        camera-to-world poses ``cam`` [N, 4, 4]."""
        cam = self._poses(cam)
        if self.prev_cam is None:
            self.reset(cam)
        if depth is None:
            if verts_world is None or tris is None:
                raise InvalidArgumentError("give depth, or verts_world and tris")
            v = torch.as_tensor(verts_world, dtype=torch.float64, device=self.device)
            # world -> camera: (p - t) R, the inverse pose of REF/tactile.py:141-146
            vc = (v - cam[:, None, :3, 3]) @ cam[:, :3, :3]
            depth = render_heightmaps(vc, torch.as_tensor(tris, device=self.device), self.cfg)
        delta = pose_delta(self.prev_cam, cam)
        out = self.pipe.simulate(depth, state=self.state, pose_delta=delta)
        self.prev_cam = cam.clone()
        return SensorObservation(out, self.state.clone(), depth if self.keep_heightmap else None)
