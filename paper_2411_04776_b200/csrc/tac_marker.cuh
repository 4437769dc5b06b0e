// Marker-stage device functions (kernel (c)), shared by the fused frame
// kernel's per-env epilogue and the stand-alone per-env kernels.
// All per-marker arithmetic is fp64: a handful of values per env, and the dot
// centres must reproduce Python's half-to-even round exactly.
#pragma once

#include "tac_internal.cuh"

namespace tac {

// LoadState (REF/marker.py:43-70) in registers.
struct Load {
  double cx, cy, dmax, sx, sy, twist;
  bool in_contact;
};

__device__ __forceinline__ Load load_from(const double* s) {
  Load l;
  l.cx = s[0];
  l.cy = s[1];
  l.dmax = s[2];
  l.sx = s[3];
  l.sy = s[4];
  l.twist = s[5];
  l.in_contact = s[6] != 0.0;
  return l;
}

__device__ __forceinline__ void load_store(double* s, const Load& l) {
  s[0] = l.cx;
  s[1] = l.cy;
  s[2] = l.dmax;
  s[3] = l.sx;
  s[4] = l.sy;
  s[5] = l.twist;
  s[6] = l.in_contact ? 1.0 : 0.0;
  s[7] = 0.0;
}

__device__ __forceinline__ Load load_zero() {
  Load l;
  l.cx = l.cy = l.dmax = l.sx = l.sy = l.twist = 0.0;
  l.in_contact = false;
  return l;
}

// track_load, REF/marker.py:124-140.  `contact` carries (c, d_c, in_contact).
__device__ __forceinline__ Load track_load(const Load& prev, double dtx, double dty, double rz,
                                           const Load& contact) {
  if (!contact.in_contact) return load_zero();
  Load out = contact;
  if (!prev.in_contact) {
    out.sx = out.sy = out.twist = 0.0;
    return out;
  }
  out.sx = prev.sx + dtx;
  out.sy = prev.sy + dty;
  out.twist = prev.twist - rz;
  return out;
}

// marker_displacements for one marker, REF/marker.py:150-165 (same operation
// order as the reference, in fp64).
__device__ __forceinline__ void marker_disp(const MarkerGeom& g, const Load& l, double mx,
                                            double my, double& ux, double& uy) {
  if (!l.in_contact) {
    ux = 0.0;
    uy = 0.0;
    return;
  }
  const double rx = mx - l.cx;
  const double ry = my - l.cy;
  const double dist = sqrt(rx * rx + ry * ry);
  const double safe = dist > 0.0 ? dist : 1.0;
  const double en = g.k_n * l.dmax * exp(-dist / g.lambda_n);
  double unx = en * (rx / safe);
  double uny = en * (ry / safe);
  if (dist == 0.0) {
    unx = 0.0;
    uny = 0.0;
  }
  const double es = exp(-(dist * dist) / (2.0 * (g.lambda_s * g.lambda_s)));
  const double et = l.twist * g.k_t * exp(-dist / g.lambda_t);
  ux = unx + es * l.sx + et * (-ry);
  uy = uny + es * l.sy + et * rx;
}

// Dot centre, REF/marker.py:221-225: int(round(p / pitch + 0.5*w - 0.5)),
// Python round = half-to-even = rint.
__device__ __forceinline__ int dot_col(const MarkerGeom& g, double px) {
  return (int)rint(px / g.pitch + 0.5 * (double)g.W - 0.5);
}
__device__ __forceinline__ int dot_row(const MarkerGeom& g, double py) {
  return (int)rint(py / g.pitch + 0.5 * (double)g.H - 0.5);
}

// Block-cooperative: displacements of every marker of one env (written to
// disp if non-null) and, if `rgb` is non-null, the filled-dot splat
// (cv2.circle(..., -1) == {dx^2+dy^2 <= r^2}, clipped, REF/marker.py:233).
// `s_cols` / `s_rows` are shared scratch of rows*cols ints each.
__device__ inline void markers_block(const MarkerGeom& g, const Load& l, float* disp,
                                     uint8_t* rgb, const float* disp_in, int* s_cols,
                                     int* s_rows) {
  const int nm = g.rows * g.cols;
  for (int m = threadIdx.x; m < nm; m += blockDim.x) {
    const double rx = g.rest_grid[2 * m];
    const double ry = g.rest_grid[2 * m + 1];
    double ux, uy;
    if (disp_in != nullptr) {
      ux = (double)disp_in[2 * m];
      uy = (double)disp_in[2 * m + 1];
    } else {
      marker_disp(g, l, rx, ry, ux, uy);
      if (disp != nullptr) {
        disp[2 * m] = (float)ux;
        disp[2 * m + 1] = (float)uy;
      }
    }
    if (rgb != nullptr) {
      s_cols[m] = dot_col(g, rx + ux);
      s_rows[m] = dot_row(g, ry + uy);
    }
  }
  if (rgb == nullptr) return;
  __syncthreads();
  const int r = g.dot_radius;
  const int side = 2 * r + 1;
  const int per = side * side;
  const long long total = (long long)nm * per;
  for (long long i = threadIdx.x; i < total; i += blockDim.x) {
    const int m = (int)(i / per);
    const int o = (int)(i - (long long)m * per);
    const int dy = o / side - r;
    const int dx = o % side - r;
    if (dx * dx + dy * dy > r * r) continue;
    const int y = s_rows[m] + dy;
    const int x = s_cols[m] + dx;
    if (y < 0 || y >= g.H || x < 0 || x >= g.W) continue;
    TAC_CHECK(y >= 0 && y < g.H && x >= 0 && x < g.W);
    uint8_t* px = rgb + ((long long)y * g.W + x) * 3;
    px[0] = g.dot_r;
    px[1] = g.dot_g;
    px[2] = g.dot_b;
  }
}

}  // namespace tac
