"""On-disk formats of the reference, host side.

* TAC1 raw maps: 16-byte header ``b"TAC1" + <u32 H, u32 W, f32 pitch>`` then
  little-endian float32 rows (REF/tactile.py:225-256).
* Marker CSV: ``row,col,rest_x,rest_y,u_x,u_y`` with ``%.17g`` floats
  (REF/marker.py:168-200).
* Tactile PNG: 8-bit RGB written through cv2 (BGR order), the uint8 rule of
  REF/cli.py:134-139 already applied by the GPU path.
* Polynomial table: JSON coefficients + 16-bit background PNG
  (REF/optical.py:303-339).

These are file I/O only; no tactile computation happens here.
"""

import csv
import json
import os
import struct

import numpy as np

from .errors import InvalidArgumentError, TacsimError

_RAW_MAGIC = b"TAC1"


class MeshFormatError(TacsimError):
    """A file could not be parsed (mirrors REF/errors.py:14-25)."""

    def __init__(self, path, line, reason):
        self.path = str(path)
        self.line = int(line)
        self.reason = reason
        super().__init__(f"{path}:{line}: {reason}")


def save_map_raw(path, values, pixel_pitch):
    """REF/tactile.py:225-233."""
    v = np.ascontiguousarray(np.asarray(values), dtype="<f4")
    if v.ndim != 2:
        raise InvalidArgumentError("raw map must be 2-D")
    header = _RAW_MAGIC + struct.pack("<IIf", v.shape[0], v.shape[1], pixel_pitch)
    with open(path, "wb") as f:
        f.write(header)
        f.write(v.tobytes())


def load_map_raw(path, dtype=np.float32):
    """REF/tactile.py:236-247; returns (values (H, W), pixel_pitch).  The
    values are returned as float32 (the file's precision; the reference widens
    them to float64 without changing any value)."""
    with open(path, "rb") as f:
        header = f.read(16)
        if len(header) != 16 or header[:4] != _RAW_MAGIC:
            raise MeshFormatError(path, 0, "not a raw tactile map")
        h, w, pitch = struct.unpack("<IIf", header[4:])
        body = f.read(h * w * 4)
    if len(body) != h * w * 4:
        raise MeshFormatError(path, 0, "truncated raw tactile map")
    return np.frombuffer(body, dtype="<f4").reshape(h, w).astype(dtype), float(pitch)


def save_markers_csv(path, rest, disp):
    """REF/marker.py:168-180 (one row per marker, %.17g)."""
    rest = np.asarray(rest, dtype=np.float64)
    disp = np.asarray(disp, dtype=np.float64)
    rows, cols = rest.shape[:2]
    with open(path, "w", newline="") as f:
        wr = csv.writer(f)
        wr.writerow(["row", "col", "rest_x", "rest_y", "u_x", "u_y"])
        for i in range(rows):
            for j in range(cols):
                rx, ry = rest[i, j]
                ux, uy = disp[i, j]
                wr.writerow([i, j, f"{rx:.17g}", f"{ry:.17g}", f"{ux:.17g}", f"{uy:.17g}"])


def load_markers_csv(path):
    """REF/marker.py:183-200; returns (rest (R, C, 2), disp (R, C, 2))."""
    with open(path, newline="") as f:
        rd = csv.reader(f)
        header = next(rd)
        if header != ["row", "col", "rest_x", "rest_y", "u_x", "u_y"]:
            raise InvalidArgumentError(f"unexpected marker CSV header in {path}")
        recs = [(int(r[0]), int(r[1]), *map(float, r[2:])) for r in rd]
    if not recs:
        raise InvalidArgumentError(f"empty marker CSV: {path}")
    rows = max(r[0] for r in recs) + 1
    cols = max(r[1] for r in recs) + 1
    rest = np.zeros((rows, cols, 2))
    disp = np.zeros((rows, cols, 2))
    for i, j, rx, ry, ux, uy in recs:
        rest[i, j] = (rx, ry)
        disp[i, j] = (ux, uy)
    return rest, disp


def write_rgb_png(path, rgb_u8):
    """REF/cli.py:134-139 for an already-quantised frame (atomic replace)."""
    import cv2

    img = np.ascontiguousarray(np.asarray(rgb_u8, dtype=np.uint8)[:, :, ::-1])
    tmp = f"{path}.tmp.{os.getpid()}.png"
    if not cv2.imwrite(tmp, img):
        raise MeshFormatError(path, 0, "failed to encode PNG")
    os.replace(tmp, path)


def read_rgb_png(path):
    import cv2

    img = cv2.imread(path, cv2.IMREAD_UNCHANGED)
    if img is None:
        raise MeshFormatError(path, 0, "failed to read PNG")
    return img[:, :, ::-1]


def load_polytable(json_path, png_path):
    """REF/optical.py:318-339: returns (coeffs (3, n_terms), background (H, W, 3)
    in [0, 1]); c0 is re-anchored to the background mean as the reference does
    (it cancels in shading anyway)."""
    import cv2

    with open(json_path) as f:
        doc = json.load(f)
    img = cv2.imread(png_path, cv2.IMREAD_UNCHANGED)
    if img is None:
        raise MeshFormatError(png_path, 0, "failed to read PNG")
    if img.ndim != 3 or img.shape[2] != 3 or img.dtype != np.uint16:
        raise MeshFormatError(png_path, 0, "background must be 16-bit RGB")
    background = img[:, :, ::-1].astype(np.float64) / 65535.0
    coeffs = np.asarray(doc["coeffs"], dtype=np.float64)
    coeffs[:, 0] = background.reshape(-1, 3).mean(axis=0)
    if int(doc.get("degree", 2)) != 2:
        raise InvalidArgumentError("only degree-2 tables map onto the binned LUT")
    return coeffs, background
