"""The timed CPU baseline port (oracle.fast) computes what the oracle computes."""

import numpy as np

from oracle.fast import FastOracle
from paper_2411_04776_b200 import synthetic

from _helpers import depth_batch, normwise, oracle_env, small_config


def test_fast_port_matches_oracle():
    cfg = small_config(40, 56)
    depth = depth_batch(4, 40, 56, seed=2).numpy().astype(np.float64)
    shear, twist = synthetic.loads(4, 3)
    fast = FastOracle(cfg)
    for i in range(4):
        rgb, disp, summ, blurred = fast.run(depth[i], shear[i], twist[i])
        ref = oracle_env(cfg, depth[i].astype(np.float32), shear[i], twist[i])
        assert normwise(blurred, ref["blurred"]) < 1e-12
        d = np.abs(rgb.astype(int) - ref["rgb"].astype(int))
        assert (d == 0).mean() >= 0.999
        assert normwise(disp, ref["disp"]) < 1e-12
        assert np.allclose(summ, ref["summary"], rtol=1e-12, atol=0)


def test_fast_port_with_shadows_matches_oracle():
    """The shadows-on CPU line (bench.py --shadows) times the same arithmetic
    as the oracle's add_shadows chain (REF/optical.py:261-300)."""
    cfg = small_config(40, 56, shadows=True)
    depth = depth_batch(3, 40, 56, seed=4).numpy().astype(np.float64)
    shear, twist = synthetic.loads(3, 5)
    fast = FastOracle(cfg)
    for i in range(3):
        rgb, disp, summ, blurred = fast.run(depth[i], shear[i], twist[i])
        ref = oracle_env(cfg, depth[i].astype(np.float32), shear[i], twist[i])
        d = np.abs(rgb.astype(int) - ref["rgb"].astype(int))
        assert (d == 0).mean() >= 0.999
