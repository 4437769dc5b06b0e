"""Oracle: the whole per-sensor path for one env (TEST INFRASTRUCTURE).

Composes the restated stages in the order ``Environment._observe`` runs them
(envs.py:1156-1209) with shadows off (add_shadows factor=1.0 is the identity,
optical.py:281-282) and the marker-dot splat of marker.py:203-234 drawn on the
quantised frame:

  depth -> indentation_from -> smooth_pyramid -> gradient/normals -> binned
  LUT shade (-> add_shadows when a shadow factor < 1 is given) -> uint8 ; contact_center (raw indentation, envs.py:1177) ->
  load (given shear/twist, or track_load) -> marker_displacements ->
  render_markers.
"""

import numpy as np

from . import marker, optical, tactile


def simulate_env(
    depth,
    *,
    pitch,
    rest,
    levels,
    lut,
    background,
    g_max,
    rest_grid,
    shear=(0.0, 0.0),
    twist=0.0,
    params=marker.DEFAULT_PARAMS,
    threshold=marker.DEFAULT_CONTACT_THRESHOLD,
    dot_radius=3,
    dot_color=(25, 25, 25),
    splat=True,
    light_dirs=None,
    shadow_factor=1.0,
    shadow_steps=80,
    shadow_softness=5e-5,
):
    """Returns dict(rgb u8 (H,W,3), disp (R,C,2), summary (8,), blurred (H,W))."""
    ind = tactile.indentation_from(depth, rest)
    blurred = tactile.smooth_pyramid(ind, levels)
    shadow = None
    if light_dirs is not None and len(light_dirs) and shadow_factor != 1.0:
        # add_shadows on the height map (elevation = -depth), REF/envs.py:1173
        shadow = optical.shadow_factor(-np.asarray(depth, dtype=np.float64), pitch, light_dirs,
                                       shadow_factor, shadow_steps, shadow_softness)
    rgb, _ = optical.shade_lut(blurred, pitch, lut, background, g_max, shadow)
    c = marker.contact_center(ind, pitch, threshold)
    load = dict(c)
    if c["in_contact"]:
        load.update(sx=float(shear[0]), sy=float(shear[1]), twist=float(twist))
    else:
        load.update(sx=0.0, sy=0.0, twist=0.0)
    disp = marker.marker_displacements(load, rest_grid, params)
    if splat:
        rgb = marker.render_markers(rgb, np.asarray(rest_grid) + disp, pitch, dot_radius, dot_color)
    return dict(
        rgb=rgb,
        disp=disp,
        summary=marker.contact_summary(c, pitch),
        blurred=blurred,
        ind=ind,
    )
