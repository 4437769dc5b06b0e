"""Observation digest for replay determinism (row f4).

Batched counterpart of ``observation_digest`` (REF/envs.py:668-694): a
SHA-256 over the step index and every output field -- shape, dtype and raw
bytes, in a fixed order -- so equal digests mean bit-identical content.  The
reference hashes one Environment observation (markers, load states, rgb,
height maps, poses); here the fields are the batched ``Observation`` of
``TactilePipeline.simulate`` / ``SensorObserver.observe`` (marker
displacements, LoadState, RGB, optional height map, contact summary), either
for the whole batch or per env (``per_env=True`` -> one digest per env, equal
to the digest of that env observed alone).
"""

import hashlib
from typing import List, Optional, Sequence, Union

import numpy as np


def _host(a):
    if a is None:
        return None
    if hasattr(a, "detach"):  # torch tensor (device or host)
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(a)


def _update(h, a: Optional[np.ndarray]) -> None:
    # same encoding as REF/envs.py:673-679
    if a is None:
        h.update(b"\x00none")
        return
    h.update(str(a.shape).encode())
    h.update(str(a.dtype).encode())
    h.update(np.ascontiguousarray(a).tobytes())


def observation_digest(obs, step_index: int = 0, *, loads=None, heightmap=None,
                       per_env: bool = False) -> Union[str, List[str]]:
    """SHA-256 hex digest of one step's outputs.

    obs: an ``Observation`` (rgb [N,H,W,3] u8, disp [N,R,C,2] f32, summary
    [N,8] f32) or a ``SensorObservation`` (its outputs, loads and height map
    are used).  loads: LoadState [N,8] fp64 (defaults to ``obs.contact``).
    """
    if hasattr(obs, "outputs"):  # SensorObservation
        loads = obs.loads if loads is None else loads
        heightmap = obs.heightmap if heightmap is None else heightmap
        obs = obs.outputs
    if loads is None:
        loads = obs.contact
    fields: Sequence = (obs.disp, loads, obs.rgb, heightmap, obs.summary)
    arrays = [_host(f) for f in fields]
    if not per_env:
        h = hashlib.sha256()
        h.update(str(int(step_index)).encode())
        for a in arrays:
            _update(h, a)
        return h.hexdigest()
    n = arrays[2].shape[0]
    out = []
    for i in range(n):
        h = hashlib.sha256()
        h.update(str(int(step_index)).encode())
        for a in arrays:
            _update(h, None if a is None else a[i:i + 1])
        out.append(h.hexdigest())
    return out


__all__ = ["observation_digest"]
