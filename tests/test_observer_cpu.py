"""Row f3 host logic: camera-pose deltas (REF/envs.py:1178) and the yaw of
REF/marker.py:137, checked against scipy's Rotation (what the reference's
Pose.rot() uses)."""

import numpy as np
import torch
from scipy.spatial.transform import Rotation

from paper_2411_04776_b200.observer import pose_delta


def _pose(rv, t):
    m = np.eye(4)
    m[:3, :3] = Rotation.from_rotvec(rv).as_matrix()
    m[:3, 3] = t
    return m


def test_pose_delta_matches_scipy():
    rng = np.random.default_rng(3)
    rvs = [rng.normal(size=3) * s for s in (1e-4, 1e-2, 0.5, 2.0)] + [np.array([0.0, 0.0, np.pi - 1e-3]),
                                                                     np.array([np.pi - 1e-6, 0.0, 0.0])]
    prev, cam, want = [], [], []
    for rv in rvs:
        a = _pose(rng.normal(size=3) * 0.3, rng.normal(size=3))
        b = a @ _pose(rv, rng.normal(size=3) * 1e-3)
        prev.append(a)
        cam.append(b)
        d = np.linalg.inv(a) @ b
        want.append([d[0, 3], d[1, 3], Rotation.from_matrix(d[:3, :3]).as_rotvec()[2]])
    got = pose_delta(torch.tensor(np.array(prev)), torch.tensor(np.array(cam))).numpy()
    assert np.allclose(got, np.array(want), rtol=1e-9, atol=1e-12)


def test_identity_delta_is_zero():
    e = torch.eye(4, dtype=torch.float64).repeat(3, 1, 1)
    assert torch.equal(pose_delta(e, e), torch.zeros(3, 3, dtype=torch.float64))
