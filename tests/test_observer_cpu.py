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


class TestDigestAndCaseFrame:
    """observation_digest (REF/envs.py:668-694) and camera_pose_in_case
    (REF/tactile.py:47, REF/envs.py:733-734): host logic, no GPU."""

    def _obs(self, n=3, seed=0):
        import torch

        from paper_2411_04776_b200.pipeline import Observation

        g = torch.Generator().manual_seed(seed)
        return Observation(rgb=torch.randint(0, 256, (n, 6, 8, 3), generator=g, dtype=torch.uint8),
                           disp=torch.randn(n, 2, 3, 2, generator=g),
                           summary=torch.randn(n, 8, generator=g),
                           contact=torch.randn(n, 8, generator=g, dtype=torch.float64))

    def test_digest_is_content_exact(self):
        from paper_2411_04776_b200 import observation_digest

        a, b = self._obs(), self._obs()
        assert observation_digest(a, 3) == observation_digest(b, 3)
        assert observation_digest(a, 3) != observation_digest(a, 4)
        b.rgb[1, 2, 3, 0] ^= 1
        assert observation_digest(a, 3) != observation_digest(b, 3)

    def test_per_env_digest_equals_single_env_digest(self):
        from paper_2411_04776_b200 import observation_digest
        from paper_2411_04776_b200.pipeline import Observation

        a = self._obs(4)
        per = observation_digest(a, 7, per_env=True)
        for i in range(4):
            one = Observation(rgb=a.rgb[i:i + 1], disp=a.disp[i:i + 1], summary=a.summary[i:i + 1],
                              contact=a.contact[i:i + 1])
            assert per[i] == observation_digest(one, 7)
        assert len(set(per)) == 4

    def test_camera_pose_in_case_validated_and_composed(self):
        import numpy as np
        import pytest

        from paper_2411_04776_b200.config import SensorConfig
        from paper_2411_04776_b200.errors import InvalidArgumentError

        assert np.array_equal(SensorConfig().camera_pose_matrix, np.eye(4))
        t = np.eye(4)
        t[:3, 3] = (0.001, -0.002, 0.003)
        c, s = np.cos(0.3), np.sin(0.3)
        t[:2, :2] = [[c, -s], [s, c]]
        cfg = SensorConfig(camera_pose_in_case=t)
        assert np.allclose(cfg.camera_pose_matrix, t)
        hash(cfg)  # still a frozen, hashable config
        with pytest.raises(InvalidArgumentError):
            SensorConfig(camera_pose_in_case=np.eye(3))
        bad = np.eye(4)
        bad[0, 0] = 2.0
        with pytest.raises(InvalidArgumentError):
            SensorConfig(camera_pose_in_case=bad)
