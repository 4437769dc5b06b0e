// Strip-streaming frame kernel: kernel (a) gel clamp + multi-scale Gaussian
// pyramid, fused with kernel (b) gradient -> binned LUT -> background ->
// uint8, plus the contact reductions and marker epilogue of kernel (c).
//
// One CTA (320 threads) owns one column strip of one env's frame (a whole
// 320-wide frame is one strip) and walks it top to bottom in row blocks of
// RB = 16 rows:
//
//   TMA   cp.async.bulk copies the block's new depth rows (clamped row index =
//         replicate borders, scipy mode="nearest", REF/tactile.py:219-221)
//         into the input buffer, issued one block ahead so the copy overlaps
//         the previous block's horizontal pass and shading;
//   conv  clamp depth -> indentation in place (REF/tactile.py:193-197), fold
//         the contact partials of REF/marker.py:109-121 and per-row non-zero
//         flags into the same pass;
//   V     per level, one thread per column: 16 outputs x (2r+1) taps from
//         registers (each smem load feeds up to 16 FFMAs);
//   H     per level, one thread per (row, 16-column chunk), accumulated over
//         levels into the blurred ring (1/L folded into the taps);
//   shade four pixels per thread: np.gradient differences (one-sided on the
//         borders, REF/optical.py:160), normals, magnitude/direction bins,
//         c1..c5 x basis (REF/optical.py:82-88, :244), + background,
//         round-half-even with saturation -> staged uint8 -> 16-B stores.
//
// A block whose input window is entirely zero blurs to exactly 0 and shades
// to exactly rint(background): it skips V/H/shade and copies the quantised
// background (exact, not an approximation).
//
// After the last block the CTA reduces its partials; the env epilogue
// (centroid, load, displacements, dot splat) runs in the same CTA when the
// frame is one strip, else in the last strip CTA of the env (atomic ticket).
#include <cstdio>

#include "tac_frame_common.cuh"

namespace tac {

namespace {


// ---- named barriers (warp-specialised fused kernel) -------------------------
// id 0: whole CTA; 1: blur group; 2: shade group; 3..5: ring slot FULL[s];
// 6..8: ring slot EMPTY[s].  Groups are 320 threads (10 warps) each.
enum : int { kBarBlur = 1, kBarShade = 2, kBarFull = 3, kBarEmpty = 3 + kSlots };

// ring row of global row r (r >= -1); slots are RB-row aligned
__device__ __forceinline__ int ring_row(int r) { return (r + kRing) % kRing; }

__device__ __forceinline__ void bsync() { bar_sync(kBarBlur, kThreads); }


// Vertical: vb[k][c - vb_base] = sum_t wv[|t|] * in[R + k + t][c - lx0], k < RB,
// for in-frame columns c of [bx0 - RL, bx1 + RL).  One item = a column pair x
// 8 rows (FFMA2 over the pair, LDS.64 loads); consecutive lanes take
// consecutive pairs, so loads are conflict-free and every load feeds 8 FFMA2.
template <int RL>
__device__ __forceinline__ void vpass(const FrameParams& p, const Geo& g, int lvl,
                                      const float* __restrict__ inb, float* __restrict__ vb) {
  float2 w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = make_float2(p.wv[lvl][i], p.wv[lvl][i]);
  const int c_lo = max(g.bx0 - RL, 0) & ~1;
  const int c_hi = (min(g.bx1 + RL, p.W) + 1) & ~1;
  const int npairs = (c_hi - c_lo) >> 1;
  const int vb_base = g.bx0 - p.R;
  const int ip = p.in_pitch, vp = p.v_pitch;
  for (int it = threadIdx.x; it < 2 * npairs; it += kThreads) {
    const int h = it >= npairs ? 1 : 0;
    const int c = c_lo + 2 * (it - h * npairs);
    const float* src = inb + (p.R - RL + 8 * h) * ip + (c - g.lx0);
    float2 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8 + 2 * RL; ++j) {
      const float2 v = *reinterpret_cast<const float2*>(src + j * ip);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = j - k - RL;
        if (t >= -RL && t <= RL) acc[k] = ffma2(w[t < 0 ? -t : t], v, acc[k]);
      }
    }
    float* dst = vb + 8 * h * vp + (c - vb_base);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dst[k * vp] = acc[k].x;
      dst[k * vp + 1] = acc[k].y;
    }
  }
}

// Replicate the vertical-pass result into columns outside the frame (H-pass pads).
__device__ __forceinline__ void vpad(const FrameParams& p, const Geo& g, int RL, float* vb) {
  const int left = max(0, RL - g.bx0);         // columns bx0-RL .. -1
  const int right = max(0, g.bx1 + RL - p.W);  // columns W .. bx1+RL-1
  const int n = left + right;
  if (n == 0) return;
  const int vb_base = g.bx0 - p.R;
  for (int it = threadIdx.x; it < n * RB; it += kThreads) {
    const int k = it & (RB - 1);
    const int q = it / RB;
    float* row = vb + k * p.v_pitch;
    if (q < left)
      row[(-1 - q) - vb_base] = row[0 - vb_base];
    else
      row[(p.W + (q - left)) - vb_base] = row[(p.W - 1) - vb_base];
  }
}

// Horizontal: bb[2 + r][c - bbase] (+)= sum_t wh[|t|] * vb[r][c + t - vb_base]
// for r < RB, c in [bx0, bx1).  One item = rows (r, r + 8) x 8 columns: FFMA2
// pairs the two rows.  A warp covers 8 row pairs x 4 chunks, conflict-free
// with the odd v_pitch; results go out as float4 (b_pitch = 4 x odd).
template <int RL>
__device__ __forceinline__ void hpass(const FrameParams& p, const Geo& g, int lvl,
                                      const float* __restrict__ vb, float* __restrict__ bb,
                                      bool first, int r0) {
  float2 w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = make_float2(p.wh[lvl][i], p.wh[lvl][i]);
  const int EW = g.bx1 - g.bx0;
  const int nch = (EW + 7) >> 3;
  const int vb_base = g.bx0 - p.R;
  const int vp = p.v_pitch;
  for (int it = threadIdx.x; it < 8 * nch; it += kThreads) {
    const int rp = it & 7;
    const int c0 = (it >> 3) * 8;
    const float* s0 = vb + rp * vp + (g.bx0 + c0 - RL - vb_base);
    const float* s1 = s0 + 8 * vp;
    float2 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8 + 2 * RL; ++j) {
      const float2 v = make_float2(s0[j], s1[j]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int t = j - k - RL;
        if (t >= -RL && t <= RL) acc[k] = ffma2(w[t < 0 ? -t : t], v, acc[k]);
      }
    }
    float* d0 = bb + ring_row(r0 + rp) * p.b_pitch + (g.bx0 + c0 - g.bbase);
    float* d1 = bb + ring_row(r0 + rp + 8) * p.b_pitch + (g.bx0 + c0 - g.bbase);
    if (c0 + 8 <= EW) {
      float4* a4 = reinterpret_cast<float4*>(d0);
      float4* b4 = reinterpret_cast<float4*>(d1);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float4 o0 = make_float4(acc[4 * q].x, acc[4 * q + 1].x, acc[4 * q + 2].x, acc[4 * q + 3].x);
        float4 o1 = make_float4(acc[4 * q].y, acc[4 * q + 1].y, acc[4 * q + 2].y, acc[4 * q + 3].y);
        if (!first) {
          const float4 x0 = a4[q], x1 = b4[q];
          o0.x += x0.x; o0.y += x0.y; o0.z += x0.z; o0.w += x0.w;
          o1.x += x1.x; o1.y += x1.y; o1.z += x1.z; o1.w += x1.w;
        }
        a4[q] = o0;
        b4[q] = o1;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (c0 + k < EW) {
          d0[k] = first ? acc[k].x : d0[k] + acc[k].x;
          d1[k] = first ? acc[k].y : d1[k] + acc[k].y;
        }
    }
  }
}

// Identity level (k == 1): bb (+)= in / L, straight from the input buffer.
__device__ __forceinline__ void ident_level(const FrameParams& p, const Geo& g, int lvl,
                                            const float* inb, float* bb, bool first, int r0) {
  const float w = p.wh[lvl][0];
  const int EW = g.bx1 - g.bx0;
  for (int it = threadIdx.x; it < EW * RB; it += kThreads) {
    const int r = it / EW;
    const int c = g.bx0 + (it - r * EW);
    const float v = w * inb[(p.R + r) * p.in_pitch + (c - g.lx0)];
    float* d = bb + ring_row(r0 + r) * p.b_pitch + (c - g.bbase);
    *d = first ? v : *d + v;
  }
}

#define TAC_RADIUS_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
  X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24)


// Shade rows [y_lo, y_hi) of the strip into the staging buffer (rows relative
// to y_lo).  Four consecutive pixels per thread: float4 reads of the blurred
// ring (conflict-free), x-neighbours by warp shuffle, 16-B background loads,
// LUT gathers issued two pixels at a time, 12-B staged stores.
__device__ __forceinline__ void shade_rows(const FrameParams& p, const Geo& g, int y_lo, int y_hi,
                                           const float* __restrict__ bb, uint8_t* __restrict__ stage,
                                           int gtid) {
  const int OW = g.x1 - g.x0;
  const int ng = (OW + 3) >> 2;
  const int sw3 = OW * 3;
  const int rows = y_hi - y_lo;
  const int step = kShadeThreads / ng;  // rows per sweep (>= 1: strips are <= 4 * kShadeThreads wide)
  const int gi = gtid % ng;
  const int ro = gtid / ng;
  const int lane = gtid & 31;
  const int xg = g.x0 + 4 * gi;
  const bool full = xg + 4 <= g.x1;
  const bool vec_bg = ((p.W & 3) == 0) && full;
  const bool need_l = (lane == 0) || (gi == 0);
  const bool need_r = (lane == 31) || (gi == ng - 1);
  const int x_last = p.W - 1;
  for (int y0 = 0; y0 < rows; y0 += step) {
    const int yy = y0 + ro;
    const bool act = (ro < step) && (yy < rows);
    const int y = y_lo + (act ? yy : 0);
    // blurred ring: global row r lives in ring row (r mod kRing)
    const float* rc = bb + ring_row(y) * p.b_pitch + (xg - g.bbase);
    const float* rm = bb + ring_row(y - 1) * p.b_pitch + (xg - g.bbase);
    const float* rp = bb + ring_row(y + 1) * p.b_pitch + (xg - g.bbase);
    const float4 cc = *reinterpret_cast<const float4*>(rc);
    const float4 mm = *reinterpret_cast<const float4*>(rm);
    const float4 nn = *reinterpret_cast<const float4*>(rp);
    float left = __shfl_up_sync(0xffffffffu, cc.w, 1);
    float right = __shfl_down_sync(0xffffffffu, cc.x, 1);
    if (!act) continue;
    if (need_l) left = rc[-1];
    if (need_r) right = rc[4];
    float bgv[12];
    const float* bgp = p.bg + ((long long)y * p.W + xg) * 3;
    if (vec_bg) {
      const float4 b0 = __ldg(reinterpret_cast<const float4*>(bgp));
      const float4 b1 = __ldg(reinterpret_cast<const float4*>(bgp) + 1);
      const float4 b2 = __ldg(reinterpret_cast<const float4*>(bgp) + 2);
      bgv[0] = b0.x; bgv[1] = b0.y; bgv[2] = b0.z; bgv[3] = b0.w;
      bgv[4] = b1.x; bgv[5] = b1.y; bgv[6] = b1.z; bgv[7] = b1.w;
      bgv[8] = b2.x; bgv[9] = b2.y; bgv[10] = b2.z; bgv[11] = b2.w;
    } else {
#pragma unroll
      for (int k = 0; k < 12; ++k) bgv[k] = (xg + k / 3 < g.x1) ? __ldg(bgp + k) : 0.f;
    }
    const float c[6] = {left, cc.x, cc.y, cc.z, cc.w, right};
    const float m[4] = {mm.x, mm.y, mm.z, mm.w};
    const float n[4] = {nn.x, nn.y, nn.z, nn.w};
    const bool top = (y == 0), bot = (y == p.H - 1);
    float gxs[4], gys[4];
    if (!__any_sync(__activemask(), top || bot || xg == 0 || xg + 4 >= p.W)) {
      // interior: central differences only
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        gxs[k] = (c[k + 2] - c[k]) * p.inv_2p;
        gys[k] = (n[k] - m[k]) * p.inv_2p;
      }
    } else {
      const float sy = (top || bot) ? p.inv_p : p.inv_2p;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int x = xg + k;
        const bool lft = (x == 0), rgt = (x == x_last);
        const float xr = rgt ? c[k + 1] : c[k + 2];
        const float xl = lft ? c[k + 1] : c[k];
        gxs[k] = (xr - xl) * ((lft || rgt) ? p.inv_p : p.inv_2p);
        const float yb = bot ? c[k + 1] : n[k];
        const float yt = top ? c[k + 1] : m[k];
        gys[k] = (yb - yt) * sy;
      }
    }
    float sf[4] = {1.f, 1.f, 1.f, 1.f};
    const float* shadow = p.shadow;
    if (shadow) {
      const float* sp = shadow + g.env * (long long)p.H * p.W + (long long)y * p.W + xg;
      if (vec_bg) {
        const float4 f4 = __ldg(reinterpret_cast<const float4*>(sp));
        sf[0] = f4.x; sf[1] = f4.y; sf[2] = f4.z; sf[3] = f4.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) sf[k] = (xg + k < g.x1) ? __ldg(sp + k) : 1.f;
      }
    }
    uint32_t q[12];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const Px p0 = bin_px(p, gxs[2 * h], gys[2 * h]);
      const Px p1 = bin_px(p, gxs[2 * h + 1], gys[2 * h + 1]);
      const float4 a0 = __ldg(p0.lut), c0 = __ldg(p0.lut + 1), d0 = __ldg(p0.lut + 2), e0 = __ldg(p0.lut + 3);
      const float4 a1 = __ldg(p1.lut), c1 = __ldg(p1.lut + 1), d1 = __ldg(p1.lut + 2), e1 = __ldg(p1.lut + 3);
      float r = bgv[6 * h], gg = bgv[6 * h + 1], b = bgv[6 * h + 2];
      add_lut(a0, c0, d0, e0, p0.nx, p0.ny, r, gg, b);
      if (shadow) {  // clip, then the multiplicative shadow (REF/optical.py:246, :299)
        r = clampf(r, 0.f, 255.f) * sf[2 * h];
        gg = clampf(gg, 0.f, 255.f) * sf[2 * h];
        b = clampf(b, 0.f, 255.f) * sf[2 * h];
      }
      q[6 * h] = u8sat(r);
      q[6 * h + 1] = u8sat(gg);
      q[6 * h + 2] = u8sat(b);
      r = bgv[6 * h + 3];
      gg = bgv[6 * h + 4];
      b = bgv[6 * h + 5];
      add_lut(a1, c1, d1, e1, p1.nx, p1.ny, r, gg, b);
      if (shadow) {
        r = clampf(r, 0.f, 255.f) * sf[2 * h + 1];
        gg = clampf(gg, 0.f, 255.f) * sf[2 * h + 1];
        b = clampf(b, 0.f, 255.f) * sf[2 * h + 1];
      }
      q[6 * h + 3] = u8sat(r);
      q[6 * h + 4] = u8sat(gg);
      q[6 * h + 5] = u8sat(b);
    }
    uint8_t* dst = stage + yy * sw3 + 4 * gi * 3;
    if (full && ((reinterpret_cast<uintptr_t>(dst) & 3) == 0)) {
      uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
      d32[0] = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      d32[1] = q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24);
      d32[2] = q[8] | (q[9] << 8) | (q[10] << 16) | (q[11] << 24);
    } else {
      for (int k = 0; k < 12 && xg + k / 3 < g.x1; ++k) dst[k] = (uint8_t)q[k];
    }
  }
}

// staged rows -> global, one warp per row, 16 B per lane when aligned.
__device__ __forceinline__ void store_rows(uint8_t* out_rows, long long row_stride,
                                           const uint8_t* stage, int rows, int nbytes, int gtid) {
  const int lane = gtid & 31, wid = gtid >> 5, nw = kShadeThreads / 32;
  for (int rr = wid; rr < rows; rr += nw) {
    uint8_t* dst = out_rows + rr * row_stride;
    const uint8_t* src = stage + rr * nbytes;
    const uintptr_t al = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes;
    if ((al & 15) == 0) {
      for (int i = lane; i < nbytes / 16; i += 32)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else if ((al & 3) == 0) {
      for (int i = lane; i < nbytes / 4; i += 32)
        reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
    } else {
      for (int i = lane; i < nbytes; i += 32) dst[i] = src[i];
    }
  }
}

// Copy quantised-background rows (blocks whose blur is exactly zero).
__device__ __forceinline__ void bg_rows(const FrameParams& p, const Geo& g, uint8_t* out, int y_lo,
                                        int y_hi, int gtid) {
  const int lane = gtid & 31, wid = gtid >> 5, nw = kShadeThreads / 32;
  const int nbytes = (g.x1 - g.x0) * 3;
  for (int y = y_lo + wid; y < y_hi; y += nw) {
    const long long o = ((long long)y * p.W + g.x0) * 3;
    uint8_t* d = out + o;
    const uint8_t* s = p.bg_u8 + o;
    if (((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s) | nbytes) & 15) == 0) {
      for (int i = lane; i < nbytes / 16; i += 32)
        reinterpret_cast<uint4*>(d)[i] = __ldg(reinterpret_cast<const uint4*>(s) + i);
    } else {
      for (int i = lane; i < nbytes; i += 32) d[i] = s[i];
    }
  }
}


__device__ __forceinline__ void shift_halo(const FrameParams& p, float* inb, int LW, int R, bool vec,
                                           int cg, int cro, int cstep) {
  // rows [RB, RB + 2R) -> [0, 2R).  Phases of RB destination rows never read
  // what they write; a barrier separates the phases.
  for (int m = 0; m < 2 * R; m += RB) {
    const int rows = min(RB, 2 * R - m);
    if (vec) {
      for (int rr = cro; cro < cstep && rr < rows; rr += cstep) {
        float4* d = reinterpret_cast<float4*>(inb + (m + rr) * p.in_pitch) + cg;
        *d = *(reinterpret_cast<const float4*>(inb + (m + rr + RB) * p.in_pitch) + cg);
      }
    } else {
      for (int c = threadIdx.x; c < LW; c += kThreads)
        for (int k = 0; k < rows; ++k) inb[(m + k) * p.in_pitch + c] = inb[(m + k + RB) * p.in_pitch + c];
    }
    if (m + RB < 2 * R) bsync();
  }
}

// Depth -> indentation in place for one float4 group of one row, folding the
// contact partials (own pixels only) and the row non-zero flag.  The thread's
// columns are fixed, so Sum w*xc is kept as per-column fp32 sums (same row
// order for mirrored columns -> bitwise-equal sums) and multiplied by xc in
// fp64 once at the end; Sum w*yc per row in fp64.
__device__ __forceinline__ void convert4(const FrameParams& p, float* row, int gr, int cg,
                                         const bool cown[4], const bool cvr[4], unsigned char* rownz,
                                         Red& red, float colsum[4]) {
  float4* e = reinterpret_cast<float4*>(row) + cg;
  float4 v4 = *e;
  float v[4] = {v4.x, v4.y, v4.z, v4.w};
  const bool rown = gr >= 0 && gr < p.H;
  bool nz = false;
  float rowsum = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool own = rown && cown[q];
    if (own && !(fabsf(v[q]) < INFINITY)) red.nf += 1.f;
    if (p.input_depth) v[q] = clampf((p.rest - v[q]) + p.rest_lo, 0.f, p.rest);
    if (own) {
      red.mx = fmaxf(red.mx, v[q]);
      const bool in = v[q] > p.threshold;
      const float m = in ? v[q] : 0.f;
      red.cnt += in ? 1.f : 0.f;
      rowsum += m;
      colsum[q] += m;
    }
    nz |= (v[q] != 0.f) && cvr[q];
  }
  if (rown) {
    red.sw += (double)rowsum;
    red.swy = fma((double)rowsum, (double)gr + 0.5 - (double)p.half_h, red.swy);
  }
  *e = make_float4(v[0], v[1], v[2], v[3]);
  if (nz) rownz[gr + p.R] = 1;
}

// Scalar fallback (rows not 16-B aligned).
__device__ __forceinline__ void convert1(const FrameParams& p, const Geo& g, float* e, int gr, int gx,
                                         unsigned char* rownz, Red& red) {
  float v = *e;
  const bool own = gr >= 0 && gr < p.H && gx >= g.x0 && gx < g.x1;
  if (own && !(fabsf(v) < INFINITY)) red.nf += 1.f;
  if (p.input_depth) v = clampf((p.rest - v) + p.rest_lo, 0.f, p.rest);
  *e = v;
  if (own) {
    red.mx = fmaxf(red.mx, v);
    if (v > p.threshold) {
      red.cnt += 1.f;
      red.sw += (double)v;
      red.swx = fma((double)v, (double)gx + 0.5 - (double)p.half_w, red.swx);
      red.swy = fma((double)v, (double)gr + 0.5 - (double)p.half_h, red.swy);
    }
  }
  if (v != 0.f && gx >= g.vx0 && gx < g.vx1) rownz[gr + p.R] = 1;
}

}  // namespace

// ---------------------------------------------------------------------------
// Fused mode is warp-specialised: threads [0, 320) are the blur group (TMA,
// conversion, V/H passes), threads [320, 640) the shade group (shading and
// RGB stores).  They hand row blocks over through a 2-slot blurred ring with
// FULL/EMPTY named barriers, so the shade group's LUT-gather latency overlaps
// the blur group's FFMA2 work.  Blur-only and contact modes run the blur group
// alone (320 threads).
template <int MODE>
__global__ void __launch_bounds__(MODE == kModeFused ? kThreads + kShadeThreads : kThreads,
                                  MODE == kModeFused ? 1 : 2)
    frame_kernel(const __grid_constant__ FrameParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Geo g = make_geo(p, MODE);
  const int R = MODE == kModeContact ? 0 : p.R;
  const long long HW = (long long)p.H * p.W;
  const int tid = threadIdx.x;
  const bool blur_group = tid < kThreads;

  float* inb = reinterpret_cast<float*>(smem_raw);
  float* vb = inb + p.in_rows * p.in_pitch;
  float* bb = vb + RB * p.v_pitch;                                       // kRing rows
  uint8_t* stage = reinterpret_cast<uint8_t*>(bb + kRing * p.b_pitch);  // shade group
  double* s_red = reinterpret_cast<double*>(stage + ((p.stage_bytes + 15) & ~15));  // <= 20 warps x 8
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_red + 2 * (kThreads / 32) * 8);
  unsigned char* rownz = reinterpret_cast<unsigned char*>(bar + 1);  // index: global row + R
  int* s_int = reinterpret_cast<int*>(rownz + ((p.H + 2 * p.R + RB + 15) & ~15));
  __shared__ double s_dbl[8];
  __shared__ int s_flag;
  __shared__ int s_nz[kSlots];  // per ring slot: the shaded rows may be non-zero

  const float* src = p.in + g.env * HW;
  const int LW = g.lx1 - g.lx0;
  const unsigned row_bytes = (unsigned)LW * 4u;

  // rows [ga, gb) (global, unclamped) -> buffer rows starting at `slot` (blur group)
  auto issue_rows = [&](int ga, int gb, int slot) {
    if (p.use_tma) {
      if (tid == 0) {
        mbar_expect_tx(bar, row_bytes * (unsigned)(gb - ga));
        for (int gr = ga; gr < gb; ++gr) {
          const int cr = min(max(gr, 0), p.H - 1);
          bulk_g2s(inb + (slot + gr - ga) * p.in_pitch, src + (long long)cr * p.W + g.lx0, row_bytes,
                   bar);
        }
      }
    } else {
      for (int it = tid; it < (gb - ga) * LW; it += kThreads) {
        const int rr = it / LW;
        const int cc = it - rr * LW;
        const int cr = min(max(ga + rr, 0), p.H - 1);
        inb[(slot + rr) * p.in_pitch + cc] = src[(long long)cr * p.W + g.lx0 + cc];
      }
    }
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < p.H + 2 * p.R + RB; i += blockDim.x) rownz[i] = 0;
  __syncthreads();

  Red red = red_zero();
  float colsum[4] = {0.f, 0.f, 0.f, 0.f};

  if (blur_group) {
    // ======================= blur group ========================================
    unsigned phase = 0;
    issue_rows(-R, RB + R, 0);  // block 0 window
    // conversion mapping: thread -> fixed float4 column group, rows strided
    const int ng4 = LW >> 2;
    const bool vec_conv = ((LW & 3) == 0) && ng4 > 0 && ng4 <= kThreads;
    const int cg = vec_conv ? tid % ng4 : 0;
    const int cro = vec_conv ? tid / ng4 : 0;
    const int cstep = vec_conv ? kThreads / ng4 : 1;
    bool cown[4], cvr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gx = g.lx0 + 4 * cg + q;
      cown[q] = gx >= g.x0 && gx < g.x1;
      cvr[q] = gx >= g.vx0 && gx < g.vx1;
    }

    for (int b = 0; b < g.nblocks; ++b) {
      const int r0 = b * RB;
      const bool last = (b == g.nblocks - 1);
      // ---- wait for this block's rows, convert the new ones -----------------
      if (p.use_tma) {
        mbar_wait(bar, phase);
        phase ^= 1u;
      } else {
        bsync();
      }
      {
        const int ga = (b == 0) ? r0 - R : r0 + R;  // first new global row
        const int slot = (b == 0) ? 0 : 2 * R;
        const int nrows = (b == 0) ? RB + 2 * R : RB;
        if (vec_conv) {
          // threads past the last full sweep (cro >= cstep) would duplicate rows
          for (int rr = cro; cro < cstep && rr < nrows; rr += cstep)
            convert4(p, inb + (slot + rr) * p.in_pitch, ga + rr, cg, cown, cvr, rownz, red, colsum);
        } else {
          for (int it = tid; it < nrows * LW; it += kThreads) {
            const int rr = it / LW;
            const int cc = it - rr * LW;
            convert1(p, g, inb + (slot + rr) * p.in_pitch + cc, ga + rr, g.lx0 + cc, rownz, red);
          }
        }
      }
      bsync();

      if (MODE == kModeContact) {
        if (!last) {
          fence_proxy_async();
          bsync();
          issue_rows(r0 + RB, r0 + 2 * RB, 0);
        }
        continue;
      }

      // ---- blur into ring slot b & 1 --------------------------------------------
      bool any = false;
      for (int i = tid; i < RB + 2 * R; i += kThreads) any |= rownz[r0 + i] != 0;  // rows r0-R..r0+RB+R-1
      any = bar_or(kBarBlur, kThreads, any);
      // slot b % kSlots still holds block b-kSlots, whose last rows the shade
      // group reads until it has finished block b-kSlots+1
      if (MODE == kModeFused && b >= kSlots) bar_sync(kBarEmpty + b % kSlots, kThreads + kShadeThreads);
      if (any) {
        for (int l = 0; l < p.n_levels; ++l) {
          const int RL = p.radius[l];
          const bool lastl = (l == p.n_levels - 1);
          if (RL == 0) {
            ident_level(p, g, l, inb, bb, l == 0, r0);
          } else {
            switch (RL) {
#define X(r)                    \
  case r:                       \
    vpass<r>(p, g, l, inb, vb); \
    break;
              TAC_RADIUS_CASES(X)
#undef X
              default:
                break;
            }
          }
          bsync();
          if (lastl && !last) {
            // this block's input rows are consumed: shift the halo, then start
            // the next block's copy (overlaps the H pass)
            shift_halo(p, inb, LW, R, vec_conv, cg, cro, cstep);
            fence_proxy_async();
          }
          if (RL > 0) vpad(p, g, RL, vb);
          bsync();
          if (lastl && !last) issue_rows(r0 + RB + R, r0 + 2 * RB + R, 2 * R);
          if (RL > 0) {
            switch (RL) {
#define X(r)                                   \
  case r:                                      \
    hpass<r>(p, g, l, vb, bb, l == 0, r0);     \
    break;
              TAC_RADIUS_CASES(X)
#undef X
              default:
                break;
            }
          }
          bsync();
        }
      } else {
        // exact zero: the blurred rows are 0
        for (int it = tid; it < RB * p.b_pitch; it += kThreads)
          bb[ring_row(r0) * p.b_pitch + it] = 0.f;
        if (!last) {
          shift_halo(p, inb, LW, R, vec_conv, cg, cro, cstep);
          fence_proxy_async();
        }
        bsync();
        if (!last) issue_rows(r0 + RB + R, r0 + 2 * RB + R, 2 * R);
      }

      // ---- outputs ----------------------------------------------------------------
      if (p.blurred != nullptr) {
        float* dst = p.blurred + g.env * HW;
        const int OW = g.x1 - g.x0;
        const int nr = min(RB, p.H - r0);
        for (int it = tid; it < nr * OW; it += kThreads) {
          const int rr = it / OW;
          const int x = g.x0 + (it - rr * OW);
          dst[(long long)(r0 + rr) * p.W + x] = bb[ring_row(r0 + rr) * p.b_pitch + (x - g.bbase)];
        }
      }
      if (MODE == kModeFused) {
        // may the rows the shade group shades for this block be non-zero?
        // (rows y-1..y+1 of y in [y_lo, y_hi) read input rows [y_lo-1-R, y_hi+R])
        if (tid == 0) {
          const int y_lo = max(r0 - 1, 0);
          const int y_hi = last ? p.H : r0 + RB - 1;
          int nz = 0;
          for (int gr = max(y_lo - 1 - p.R, -p.R); gr <= min(y_hi + p.R, p.H + p.R - 1); ++gr)
            nz |= rownz[gr + p.R];
          s_nz[b % kSlots] = nz || p.shadow != nullptr;  // shadows reach flat regions
        }
        bar_arrive(kBarFull + b % kSlots, kThreads + kShadeThreads);
      } else {
        bsync();
      }
    }
  } else if (MODE == kModeFused) {
    // ======================= shade group =======================================
    const int gtid = tid - kThreads;
    uint8_t* out = p.rgb + g.env * HW * 3;
    for (int b = 0; b < g.nblocks; ++b) {
      const int r0 = b * RB;
      const bool last = (b == g.nblocks - 1);
      bar_sync(kBarFull + b % kSlots, kThreads + kShadeThreads);
      const int y_lo = max(r0 - 1, 0);
      const int y_hi = last ? p.H : r0 + RB - 1;
      if (s_nz[b % kSlots]) {
        shade_rows(p, g, y_lo, y_hi, bb, stage, gtid);
        bar_sync(kBarShade, kShadeThreads);
        store_rows(out + ((long long)y_lo * p.W + g.x0) * 3, (long long)p.W * 3, stage, y_hi - y_lo,
                   (g.x1 - g.x0) * 3, gtid);
        bar_sync(kBarShade, kShadeThreads);  // stage is reused by the next block
      } else {
        bg_rows(p, g, out, y_lo, y_hi, gtid);
      }
      // block b-1's slot (= block b+kSlots-1's) is no longer read
      if (b >= 1 && b + kSlots - 1 < g.nblocks) bar_arrive(kBarEmpty + (b + kSlots - 1) % kSlots, kThreads + kShadeThreads);
    }
  }

  // ---- reduction + env epilogue -------------------------------------------------
  if (p.finalize == 0) return;
  if (blur_group) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cgq = ((LW & 3) == 0 && (LW >> 2) > 0 && (LW >> 2) <= kThreads) ? tid % (LW >> 2) : 0;
      red.swx = fma((double)colsum[q], (double)(g.lx0 + 4 * cgq + q) + 0.5 - (double)p.half_w, red.swx);
    }
  }
  __syncthreads();  // all RGB rows written, s_red free
  block_reduce(red, s_red);
  if (p.strips == 1) {
    if (tid == 0) finalize_load(p, g.env, red.cnt, red.sw, red.swx, red.swy, red.mx, red.nf, s_dbl);
  } else {
    if (tid == 0) {
      double* q = p.partials + (g.env * p.strips + g.strip) * kSumFields;
      q[0] = red.cnt;
      q[1] = red.sw;
      q[2] = red.swx;
      q[3] = red.swy;
      q[4] = red.mx;
      q[5] = red.nf;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned ticket = atomicAdd(p.counters + g.env, 1u);
      s_flag = ticket == (unsigned)(p.strips - 1);
    }
    __syncthreads();
    if (!s_flag) return;
    __threadfence();
    if (tid == 0) {
      double cnt = 0, sw = 0, swx = 0, swy = 0, nf = 0;
      float mx = 0.f;
      const double* q = p.partials + g.env * p.strips * kSumFields;
      for (int s = 0; s < p.strips; ++s) {  // fixed order: deterministic
        cnt += __ldcg(q + s * 8 + 0);
        sw += __ldcg(q + s * 8 + 1);
        swx += __ldcg(q + s * 8 + 2);
        swy += __ldcg(q + s * 8 + 3);
        mx = fmaxf(mx, (float)__ldcg(q + s * 8 + 4));
        nf += __ldcg(q + s * 8 + 5);
      }
      finalize_load(p, g.env, cnt, sw, swx, swy, mx, nf, s_dbl);
      p.counters[g.env] = 0u;
    }
  }
  __syncthreads();
  if (p.finalize == 2) {
    const Load l = load_from(s_dbl);
    const int nm = p.mg.rows * p.mg.cols;
    markers_block(p.mg, l, p.disp ? p.disp + g.env * (long long)nm * 2 : nullptr,
                  p.splat ? p.rgb + g.env * HW * 3 : nullptr, nullptr, s_int, s_int + nm);
  }
}

size_t frame_smem_bytes(const FrameParams& p) {
  size_t bytes = sizeof(float) * ((size_t)p.in_rows * p.in_pitch + (size_t)RB * p.v_pitch +
                                  (size_t)kRing * p.b_pitch);
  bytes += (p.stage_bytes + 15) & ~15;
  bytes += sizeof(double) * 2 * (kThreads / 32) * 8;
  bytes += sizeof(uint64_t);
  bytes += (p.H + 2 * p.R + RB + 15) & ~15;
  bytes += 2 * sizeof(int) * (size_t)p.mg.rows * p.mg.cols;
  return (bytes + 127) & ~size_t(127);
}

template <int MODE>
static cudaError_t launch_mode(const FrameParams& p, cudaStream_t s) {
  const size_t smem = frame_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(frame_kernel<MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = p.n_env * (long long)p.strips;
  if (blocks == 0) return cudaSuccess;
  frame_kernel<MODE><<<(unsigned)blocks, MODE == kModeFused ? kThreads + kShadeThreads : kThreads, smem, s>>>(p);
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
// Stand-alone shade (kernel (b) from a blurred map in HBM), one pixel per thread.
__global__ void __launch_bounds__(256) shade_kernel(const __grid_constant__ FrameParams p,
                                                    const float* __restrict__ blurred,
                                                    uint8_t* __restrict__ rgb,
                                                    unsigned int* __restrict__ saturated) {
  const long long HW = (long long)p.H * p.W;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= p.n_env * HW) return;
  const long long env = i / HW;
  const int pix = (int)(i - env * HW);
  const int y = pix / p.W, x = pix - y * p.W;
  const float* b = blurred + env * HW;
  const int xl = x > 0 ? x - 1 : x, xr = x < p.W - 1 ? x + 1 : x;
  const int yt = y > 0 ? y - 1 : y, yb = y < p.H - 1 ? y + 1 : y;
  const float gx = (__ldg(b + y * p.W + xr) - __ldg(b + y * p.W + xl)) *
                   ((xr - xl == 2) ? p.inv_2p : p.inv_p);
  const float gy = (__ldg(b + yb * p.W + x) - __ldg(b + yt * p.W + x)) *
                   ((yb - yt == 2) ? p.inv_2p : p.inv_p);
  const float* bgp = p.bg + (long long)pix * 3;
  float r = bgp[0], g = bgp[1], bl = bgp[2];
  shade_one(p, gx, gy, r, g, bl);
  if (saturated) {  // channel values the clip changes: REF/optical.py:246-247 (raw != out)
    const unsigned c = (r < 0.f || r > 255.f) + (g < 0.f || g > 255.f) + (bl < 0.f || bl > 255.f);
    if (c) atomicAdd(saturated + env, c);
  }
  uint8_t* d = rgb + i * 3;
  d[0] = (uint8_t)u8sat(r);
  d[1] = (uint8_t)u8sat(g);
  d[2] = (uint8_t)u8sat(bl);
}

cudaError_t launch_shade(const FrameParams& p, const float* blurred, uint8_t* rgb, unsigned int* saturated,
                         long long n_env, cudaStream_t s) {
  const long long n = n_env * (long long)p.H * p.W;
  if (n == 0) return cudaSuccess;
  if (saturated) {
    cudaError_t e = cudaMemsetAsync(saturated, 0, sizeof(unsigned int) * n_env, s);
    if (e != cudaSuccess) return e;
  }
  shade_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, blurred, rgb, saturated);
  return cudaGetLastError();
}

}  // namespace tac
