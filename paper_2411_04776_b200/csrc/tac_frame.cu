// Frame kernels: kernel (a) gel clamp + multi-scale Gaussian pyramid, fused
// with kernel (b) gradient -> binned LUT -> background -> uint8, and the
// per-tile contact reductions of kernel (c); the last CTA of every env runs
// the marker epilogue (centroid, load, displacements, dot splat).
//
// One CTA = one (env, output tile).  Per CTA:
//   1. load the clamped indentation window (tile + 1-px gradient ring + R halo,
//      replicate borders = scipy mode="nearest", REF/tactile.py:219-221) into
//      shared memory with 128-bit loads;
//   2. per-tile contact partials on the raw indentation (REF/marker.py:109-121);
//   3. if the window is all zero the blur is exactly 0 and the shaded pixel is
//      exactly rint(bg): copy the quantised background (exact skip);
//   4. else, per pyramid level: vertical pass (window -> vbuf) and horizontal
//      pass (vbuf -> acc, += across levels, 1/L folded into the taps);
//   5. shading from acc (np.gradient semantics incl. one-sided borders,
//      REF/optical.py:160) -> LUT bins -> c1..c5 x basis -> + bg -> rint ->
//      clamp -> staged uint8 tile -> 128-bit stores;
//   6. publish the tile partial; the last tile of the env (atomic ticket)
//      reduces the partials in fp64 and runs the marker stage.
#include <cstdio>

#include "tac_internal.cuh"
#include "tac_marker.cuh"

namespace tac {

namespace {

constexpr float kPi = 3.14159265358979323846f;

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
  return fminf(fmaxf(v, lo), hi);
}

// ---------------------------------------------------------------------------
// Separable passes.  RL is the level radius (compile time, so the tap loop is
// fully unrolled and every tap weight lives in a register).

// First pass (vertical, along rows of the window):
//   vbuf[r][c] = sum_{t=-RL..RL} wv[|t|] * win[r + R + t][c]
// for ext rows r in [0, EH) and window columns c in [c_lo, c_hi).
template <int RL>
__device__ __forceinline__ void vpass(const FrameParams& p, int lvl, const float* __restrict__ win,
                                      float* __restrict__ vbuf, int EH, int c_lo, int c_hi) {
  float w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = p.wv[lvl][i];
  const int ncols = c_hi - c_lo;
  const int nchunks = (EH + K - 1) / K;
  const int items = ncols * nchunks;
  const int pitch = p.win_pitch;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int chunk = it / ncols;
    const int c = c_lo + (it - chunk * ncols);
    const int r0 = chunk * K;
    const float* src = win + (r0 + p.R - RL) * pitch + c;
    float acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.f;
#pragma unroll
    for (int j = 0; j < K + 2 * RL; ++j) {
      const float v = src[j * pitch];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = j - k - RL;
        if (t >= -RL && t <= RL) acc[k] = fmaf(w[t < 0 ? -t : t], v, acc[k]);
      }
    }
    float* dst = vbuf + r0 * pitch + c;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (r0 + k < EH) dst[k * pitch] = acc[k];
  }
}

// Second pass (horizontal):
//   acc[r][c] (+)= sum_{t=-RL..RL} wh[|t|] * src[r][c + off + t]
// for ext rows r in [0, EH), ext cols c in [0, EW).
template <int RL>
__device__ __forceinline__ void hpass(const FrameParams& p, int lvl, const float* __restrict__ src_base,
                                      int src_pitch, int off, float* __restrict__ accb, int EH,
                                      int EW, bool first) {
  float w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = p.wh[lvl][i];
  const int nchunks = (EW + K - 1) / K;
  const int items = EH * nchunks;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int chunk = it / EH;
    const int r = it - chunk * EH;
    const int c0 = chunk * K;
    const float* src = src_base + r * src_pitch + c0 + off - RL;
    float acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.f;
#pragma unroll
    for (int j = 0; j < K + 2 * RL; ++j) {
      const float v = src[j];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int t = j - k - RL;
        if (t >= -RL && t <= RL) acc[k] = fmaf(w[t < 0 ? -t : t], v, acc[k]);
      }
    }
    float* dst = accb + r * p.acc_pitch + c0;
    if (first) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (c0 + k < EW) dst[k] = acc[k];
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (c0 + k < EW) dst[k] += acc[k];
    }
  }
}

#define TAC_RADIUS_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24)

// One pyramid level into acc.  Identity levels (radius 0) read the window.
__device__ __forceinline__ void blur_level(const FrameParams& p, int lvl, const float* win,
                                           float* vbuf, float* accb, int EH, int EW, bool first) {
  const int RL = p.radius[lvl];
  if (RL == 0) {
    hpass<0>(p, lvl, win + p.R * p.win_pitch, p.win_pitch, p.R, accb, EH, EW, first);
    __syncthreads();
    return;
  }
  // the horizontal pass reads window columns [R - RL, R + EW + RL)
  const int c_lo = p.R - RL;
  const int c_hi = p.R + EW + RL;
  switch (RL) {
#define X(r)                                        \
  case r:                                           \
    vpass<r>(p, lvl, win, vbuf, EH, c_lo, c_hi);    \
    break;
    TAC_RADIUS_CASES(X)
#undef X
    default:
      break;
  }
  __syncthreads();
  switch (RL) {
#define X(r)                                                                  \
  case r:                                                                     \
    hpass<r>(p, lvl, vbuf, p.win_pitch, p.R, accb, EH, EW, first);            \
    break;
    TAC_RADIUS_CASES(X)
#undef X
    default:
      break;
  }
  __syncthreads();
}

// Copy `nbytes` from shared to global, 16 B at a time when both ends allow.
__device__ __forceinline__ void store_row_bytes(uint8_t* dst, const uint8_t* src, int nbytes,
                                                int lane, int nlanes) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes) & 15) == 0) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = lane; i < nbytes / 16; i += nlanes) d[i] = s[i];
  } else if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes) & 3) == 0) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int i = lane; i < nbytes / 4; i += nlanes) d[i] = s[i];
  } else {
    for (int i = lane; i < nbytes; i += nlanes) dst[i] = src[i];
  }
}

// Shade one pixel from the blurred ext tile (acc).  Returns packed RGB.
// `b` points at the pixel's blurred value inside a tile of row pitch `bp`.
__device__ __forceinline__ void shade_px(const FrameParams& p, const float* __restrict__ b, int bp,
                                         int y, int x, const float* __restrict__ bgp,
                                         uint8_t* out3) {
  float gx, gy;
  // np.gradient: central inside, one-sided first order on the borders
  if (x == 0)
    gx = (b[1] - b[0]) * p.inv_p;
  else if (x == p.W - 1)
    gx = (b[0] - b[-1]) * p.inv_p;
  else
    gx = (b[1] - b[-1]) * p.inv_2p;
  if (y == 0)
    gy = (b[bp] - b[0]) * p.inv_p;
  else if (y == p.H - 1)
    gy = (b[0] - b[-bp]) * p.inv_p;
  else
    gy = (b[bp] - b[-bp]) * p.inv_2p;
  const float g2 = fmaf(gx, gx, gy * gy);
  float r = bgp[0], g = bgp[1], bl = bgp[2];
  if (g2 > 0.f) {
    const float inv = rsqrtf(1.f + g2);
    const float nx = -gx * inv, ny = -gy * inv;
    const float gm = sqrtf(g2);
    const int mb = min((int)(gm * p.mag_scale), p.mag_bins - 1);
    int db = (int)((atan2f(gy, gx) + kPi) * p.dir_scale);
    if (db >= p.dir_bins) db -= p.dir_bins;
    if (db < 0) db = 0;
    const float4* L = p.lut + ((long long)mb * p.dir_bins + db) * 4;
    const float4 a = __ldg(L + 0), c = __ldg(L + 1), d = __ldg(L + 2), e = __ldg(L + 3);
    const float nxx = nx * nx, nxy = nx * ny, nyy = ny * ny;
    // layout: a = R(c1..c4), c = R c5, G c1..c3, d = G c4..c5, B c1..c2, e = B c3..c5, pad
    const float dR = a.x * nx + a.y * ny + a.z * nxx + a.w * nxy + c.x * nyy;
    const float dG = c.y * nx + c.z * ny + c.w * nxx + d.x * nxy + d.y * nyy;
    const float dB = d.z * nx + d.w * ny + e.x * nxx + e.y * nxy + e.z * nyy;
    r += dR;
    g += dG;
    bl += dB;
  }
  out3[0] = (uint8_t)min(max(__float2int_rn(r), 0), 255);
  out3[1] = (uint8_t)min(max(__float2int_rn(g), 0), 255);
  out3[2] = (uint8_t)min(max(__float2int_rn(bl), 0), 255);
}

// Deterministic block reduction of kSumFields values (fields 0..3, 5..7 sum;
// field 4 max).  Result valid in thread 0.
__device__ __forceinline__ void block_reduce_partial(float v[kSumFields], float* s_red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int f = 0; f < kSumFields; ++f) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, v[f], o);
      v[f] = (f == 4) ? fmaxf(v[f], u) : v[f] + u;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int f = 0; f < kSumFields; ++f) s_red[wid * kSumFields + f] = v[f];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
#pragma unroll
      for (int f = 0; f < kSumFields; ++f) {
        const float u = s_red[w * kSumFields + f];
        v[f] = (f == 4) ? fmaxf(v[f], u) : v[f] + u;
      }
    }
  }
}

// Last CTA of an env: fp64 reduction of the tile partials, contact outputs,
// load (given or tracked), marker displacements and dot splat.
__device__ void env_epilogue(const FrameParams& p, long long env, int T, int* s_int,
                             double* s_dbl) {
  const float* part = p.partials + env * (long long)T * kSumFields;
  if (threadIdx.x < 32) {
    double cnt = 0.0, sw = 0.0, swx = 0.0, swy = 0.0, nf = 0.0;
    float mx = 0.f;
    for (int t = threadIdx.x; t < T; t += 32) {
      const float* q = part + t * kSumFields;
      cnt += (double)__ldcg(q + 0);
      sw += (double)__ldcg(q + 1);
      swx += (double)__ldcg(q + 2);
      swy += (double)__ldcg(q + 3);
      mx = fmaxf(mx, __ldcg(q + 4));
      nf += (double)__ldcg(q + 5);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      sw += __shfl_xor_sync(0xffffffffu, sw, o);
      swx += __shfl_xor_sync(0xffffffffu, swx, o);
      swy += __shfl_xor_sync(0xffffffffu, swy, o);
      nf += __shfl_xor_sync(0xffffffffu, nf, o);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (threadIdx.x == 0) {
      const double pitch = p.mg.pitch;
      Load c = load_zero();
      if (cnt > 0.0) {
        c.in_contact = true;
        c.cx = swx / sw * pitch;
        c.cy = swy / sw * pitch;
        c.dmax = (double)mx;
      }
      if (p.summary != nullptr) {
        float* s = p.summary + env * kSumFields;
        s[0] = c.in_contact ? 1.f : 0.f;
        s[1] = (float)(cnt * pitch * pitch);
        s[2] = (float)c.cx;
        s[3] = (float)c.cy;
        s[4] = (float)c.dmax;
        s[5] = c.in_contact ? (float)(sw * pitch * pitch) : 0.f;
        s[6] = (float)nf;
        s[7] = 0.f;
      }
      if (p.contact != nullptr) load_store(p.contact + env * 8, c);
      Load l = c;
      if (p.finalize == 2) {
        if (p.load_mode == TAC_LOAD_TRACK) {
          const Load prev = load_from(p.state + env * 8);
          const double* dl = p.pose_delta + env * 3;
          l = track_load(prev, dl[0], dl[1], dl[2], c);
          load_store(p.state + env * 8, l);
        } else if (c.in_contact) {
          l.sx = p.shear[2 * env];
          l.sy = p.shear[2 * env + 1];
          l.twist = p.twist[env];
        }
      }
      s_dbl[0] = l.cx;
      s_dbl[1] = l.cy;
      s_dbl[2] = l.dmax;
      s_dbl[3] = l.sx;
      s_dbl[4] = l.sy;
      s_dbl[5] = l.twist;
      s_dbl[6] = l.in_contact ? 1.0 : 0.0;
      // leave the ticket counter zeroed for the next launch
      p.counters[env] = 0u;
    }
  }
  __syncthreads();
  if (p.finalize == 2) {
    const Load l = load_from(s_dbl);
    const long long HW = (long long)p.H * p.W;
    const int nm = p.mg.rows * p.mg.cols;
    markers_block(p.mg, l, p.disp ? p.disp + env * (long long)nm * 2 : nullptr,
                  p.splat ? p.rgb + env * HW * 3 : nullptr, nullptr, s_int, s_int + nm);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads) frame_kernel(const __grid_constant__ FrameParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int T = p.tiles_x * p.tiles_y;
  const long long env = blockIdx.x / T;
  const int tile = blockIdx.x - (int)(env * T);
  const int ty = tile / p.tiles_x, tx = tile - ty * p.tiles_x;
  const int x0 = tx * p.TX, y0 = ty * p.TY;
  const int x1 = min(x0 + p.TX, p.W), y1 = min(y0 + p.TY, p.H);
  const int ring = (MODE == kModeFused) ? 1 : 0;
  const int ex0 = max(x0 - ring, 0), ex1 = min(x1 + ring, p.W);
  const int ey0 = max(y0 - ring, 0), ey1 = min(y1 + ring, p.H);
  const int EW = ex1 - ex0, EH = ey1 - ey0;
  const int R = (MODE == kModeContact) ? 0 : p.R;
  const int WW = EW + 2 * R, WH = EH + 2 * R;
  const long long HW = (long long)p.H * p.W;

  float* win = reinterpret_cast<float*>(smem_raw);
  float* vbuf = win + p.win_rows * p.win_pitch;
  float* accb = vbuf + p.win_rows * p.win_pitch;
  float* s_red = accb + p.acc_rows * p.acc_pitch;  // 8 warps x 8
  int* s_int = reinterpret_cast<int*>(s_red + (kThreads / 32) * kSumFields);
  __shared__ int s_flag;
  __shared__ double s_dbl[8];

  // ---- 1. clamped indentation window (replicate borders) -------------------
  const float* src = p.in + env * HW;
  const int gx0 = ex0 - R;  // global col of window col 0
  const int gy0 = ey0 - R;  // global row of window row 0
  // in-frame column span of the window
  const int cx_lo = max(gx0, 0), cx_hi = min(gx0 + WW, p.W);
  float nonfinite = 0.f;
  const bool vec = ((p.W & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (vec) {
    const int a_lo = cx_lo & ~3;             // aligned start
    const int a_hi = (cx_hi + 3) & ~3;       // aligned end (<= W since W % 4 == 0)
    const int nv = (a_hi - a_lo) >> 2;
    const int items = WH * nv;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int wr = it / nv;
      const int v4 = it - wr * nv;
      const int gy = min(max(gy0 + wr, 0), p.H - 1);
      const int gc = a_lo + 4 * v4;
      const float4 d = __ldg(reinterpret_cast<const float4*>(src + (long long)gy * p.W + gc));
      const float dv[4] = {d.x, d.y, d.z, d.w};
      const bool own_row = (gy0 + wr >= y0) && (gy0 + wr < y1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int g = gc + q;
        if (g < cx_lo || g >= cx_hi) continue;
        float v = dv[q];
        if (own_row && g >= x0 && g < x1 && !isfinite(v)) nonfinite += 1.f;
        if (p.input_depth) v = clampf((p.rest - v) + p.rest_lo, 0.f, p.rest);
        win[wr * p.win_pitch + (g - gx0)] = v;
      }
    }
  } else {
    const int nc = cx_hi - cx_lo;
    const int items = WH * nc;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int wr = it / nc;
      const int g = cx_lo + (it - wr * nc);
      const int gy = min(max(gy0 + wr, 0), p.H - 1);
      float v = src[(long long)gy * p.W + g];
      const bool own = (gy0 + wr >= y0) && (gy0 + wr < y1) && g >= x0 && g < x1;
      if (own && !isfinite(v)) nonfinite += 1.f;
      if (p.input_depth) v = clampf((p.rest - v) + p.rest_lo, 0.f, p.rest);
      win[wr * p.win_pitch + (g - gx0)] = v;
    }
  }
  __syncthreads();
  // replicate columns that fall outside the frame
  if (gx0 < 0 || gx0 + WW > p.W) {
    const int left = cx_lo - gx0;            // window cols [0, left) copy col `left`
    const int right = cx_hi - gx0;           // window cols [right, WW) copy col right-1
    const int npad = left + (WW - right);
    for (int it = threadIdx.x; it < WH * npad; it += blockDim.x) {
      const int wr = it / npad;
      const int k = it - wr * npad;
      float* row = win + wr * p.win_pitch;
      if (k < left)
        row[k] = row[left];
      else
        row[right + (k - left)] = row[right - 1];
    }
    __syncthreads();
  }

  // ---- 2. per-tile contact partials on the raw indentation -----------------
  float part[kSumFields];
#pragma unroll
  for (int f = 0; f < kSumFields; ++f) part[f] = 0.f;
  part[5] = nonfinite;
  int any = 0;
  {
    const int tw = x1 - x0, th = y1 - y0;
    for (int it = threadIdx.x; it < tw * th; it += blockDim.x) {
      const int yy = it / tw;
      const int xx = it - yy * tw;
      const float v = win[(y0 + yy - gy0) * p.win_pitch + (x0 + xx - gx0)];
      part[4] = fmaxf(part[4], v);
      if (v > p.threshold) {
        const float xc = (float)(x0 + xx) + 0.5f - p.half_w;
        const float yc = (float)(y0 + yy) + 0.5f - p.half_h;
        part[0] += 1.f;
        part[1] += v;
        part[2] = fmaf(v, xc, part[2]);
        part[3] = fmaf(v, yc, part[3]);
      }
    }
    if (MODE != kModeContact) {
      for (int it = threadIdx.x; it < WH * WW; it += blockDim.x) {
        const int wr = it / WW;
        const int wc = it - wr * WW;
        if (win[wr * p.win_pitch + wc] != 0.f) {
          any = 1;
          break;
        }
      }
    }
  }
  if (MODE != kModeContact) any = __syncthreads_or(any);

  // ---- 3/4. blur ------------------------------------------------------------
  if (MODE != kModeContact && any) {
    for (int l = 0; l < p.n_levels; ++l) blur_level(p, l, win, vbuf, accb, EH, EW, l == 0);
  }

  if (MODE == kModeBlur && p.blurred != nullptr) {
    float* dst = p.blurred + env * HW;
    const int tw = x1 - x0, th = y1 - y0;
    for (int it = threadIdx.x; it < tw * th; it += blockDim.x) {
      const int yy = it / tw;
      const int xx = it - yy * tw;
      dst[(long long)(y0 + yy) * p.W + x0 + xx] =
          any ? accb[(y0 + yy - ey0) * p.acc_pitch + (x0 + xx - ex0)] : 0.f;
    }
  }

  // ---- 5. shading -------------------------------------------------------------
  if (MODE == kModeFused) {
    const int tw = x1 - x0, th = y1 - y0;
    uint8_t* stage = reinterpret_cast<uint8_t*>(vbuf);  // vbuf is dead now
    uint8_t* out = p.rgb + env * HW * 3;
    if (any) {
      if (p.blurred != nullptr) {
        float* dst = p.blurred + env * HW;
        for (int it = threadIdx.x; it < tw * th; it += blockDim.x) {
          const int yy = it / tw;
          const int xx = it - yy * tw;
          dst[(long long)(y0 + yy) * p.W + x0 + xx] =
              accb[(y0 + yy - ey0) * p.acc_pitch + (x0 + xx - ex0)];
        }
      }
      for (int it = threadIdx.x; it < tw * th; it += blockDim.x) {
        const int yy = it / tw;
        const int xx = it - yy * tw;
        const int y = y0 + yy, x = x0 + xx;
        shade_px(p, accb + (y - ey0) * p.acc_pitch + (x - ex0), p.acc_pitch, y, x,
                 p.bg + ((long long)y * p.W + x) * 3, stage + (yy * tw + xx) * 3);
      }
      __syncthreads();
      // rows of 3*tw bytes -> global, one warp per row
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int yy = wid; yy < th; yy += nw)
        store_row_bytes(out + ((long long)(y0 + yy) * p.W + x0) * 3, stage + yy * tw * 3, tw * 3,
                        lane, 32);
    } else {
      if (p.blurred != nullptr) {
        float* dst = p.blurred + env * HW;
        for (int it = threadIdx.x; it < tw * th; it += blockDim.x) {
          const int yy = it / tw;
          dst[(long long)(y0 + yy) * p.W + x0 + (it - yy * tw)] = 0.f;
        }
      }
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      for (int yy = wid; yy < th; yy += nw) {
        const long long o = ((long long)(y0 + yy) * p.W + x0) * 3;
        uint8_t* d = out + o;
        const uint8_t* s = p.bg_u8 + o;
        if (((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s) | (tw * 3)) & 15) == 0) {
          for (int i = lane; i < tw * 3 / 16; i += 32)
            reinterpret_cast<uint4*>(d)[i] = __ldg(reinterpret_cast<const uint4*>(s) + i);
        } else {
          for (int i = lane; i < tw * 3; i += 32) d[i] = s[i];
        }
      }
    }
  }

  // ---- 6. publish partial, last tile of the env runs the epilogue ------------
  if (p.finalize == 0) return;
  block_reduce_partial(part, s_red);
  if (threadIdx.x == 0) {
    float* q = p.partials + (env * T + tile) * kSumFields;
#pragma unroll
    for (int f = 0; f < kSumFields; ++f) q[f] = part[f];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int ticket = atomicAdd(p.counters + env, 1u);
    s_flag = (ticket == (unsigned int)(T - 1));
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  env_epilogue(p, env, T, s_int, s_dbl);
}

size_t frame_smem_bytes(const FrameParams& p, int mode) {
  size_t floats = 2 * (size_t)p.win_rows * p.win_pitch + (size_t)p.acc_rows * p.acc_pitch +
                  (kThreads / 32) * kSumFields;
  size_t bytes = floats * sizeof(float);
  bytes += 2 * sizeof(int) * (size_t)p.mg.rows * p.mg.cols;
  (void)mode;
  return (bytes + 15) & ~size_t(15);
}

template <int MODE>
static cudaError_t launch_mode(const FrameParams& p, cudaStream_t s) {
  const size_t smem = frame_smem_bytes(p, MODE);
  cudaError_t e = cudaFuncSetAttribute(frame_kernel<MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = p.n_env * (long long)(p.tiles_x * p.tiles_y);
  if (blocks == 0) return cudaSuccess;
  frame_kernel<MODE><<<(unsigned)blocks, kThreads, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_frame(const FrameParams& p, int mode, cudaStream_t s) {
  switch (mode) {
    case kModeBlur:
      return launch_mode<kModeBlur>(p, s);
    case kModeFused:
      return launch_mode<kModeFused>(p, s);
    case kModeContact:
      return launch_mode<kModeContact>(p, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Stand-alone shade (kernel (b) from a blurred map in HBM).
__global__ void __launch_bounds__(256) shade_kernel(const __grid_constant__ FrameParams p,
                                                    const float* __restrict__ blurred,
                                                    uint8_t* __restrict__ rgb) {
  const long long HW = (long long)p.H * p.W;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n_env * HW) return;
  const long long env = i / HW;
  const int pix = (int)(i - env * HW);
  const int y = pix / p.W, x = pix - y * p.W;
  // gather the 3x3 neighbourhood into a tiny local tile so shade_px applies
  float loc[9];
  const float* b = blurred + env * HW;
#pragma unroll
  for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
      const int yy = min(max(y + dy, 0), p.H - 1), xx = min(max(x + dx, 0), p.W - 1);
      loc[(dy + 1) * 3 + (dx + 1)] = __ldg(b + (long long)yy * p.W + xx);
    }
  uint8_t o[3];
  shade_px(p, loc + 4, 3, y, x, p.bg + (long long)pix * 3, o);
  uint8_t* d = rgb + i * 3;
  d[0] = o[0];
  d[1] = o[1];
  d[2] = o[2];
}

cudaError_t launch_shade(const FrameParams& p, const float* blurred, uint8_t* rgb, long long n_env,
                         cudaStream_t s) {
  const long long n = n_env * (long long)p.H * p.W;
  if (n == 0) return cudaSuccess;
  shade_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, blurred, rgb);
  return cudaGetLastError();
}

}  // namespace tac
