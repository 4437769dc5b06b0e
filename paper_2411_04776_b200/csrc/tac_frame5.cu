// Band-tiled two-kernel path (v5), the default tac_pipeline path for frames of
// one strip (W <= 320, W % 16 == 0) with pyramid radii <= 16.
//
// Why two kernels: in the fused warp-specialised kernel (tac_frame.cu, and a
// slot-ring variant tried in round 1) both the blur and the shade group run
// ~2.5 warps per SMSP and every row block waits on the slower group;
// per-block clock64 stamps showed both groups latency-bound at ~0.3 IPC.  Here
// each stage gets the occupancy it needs:
//
//  band_blur_kernel   kernel (a): one CTA per (env, 16-row band), 3 CTAs/SM.
//     TMA (cp.async.bulk, clamped row index = replicate border,
//     REF/tactile.py:219-221) loads the band's 16 + 2R depth rows; the
//     conversion pass clamps them (REF/tactile.py:193-197), folds the contact
//     partials of REF/marker.py:109-121 (own rows only) and the band's
//     non-zero column extent; then per level a vertical pass (column pair x 8
//     rows per thread, writing a row-pair-interleaved intermediate) and a
//     horizontal pass (row pair x 8 columns per thread: every FFMA2 operand is
//     one aligned float2, summed over levels in registers) write the blurred
//     band to HBM/L2 with 16-B stores.  Columns farther than R from any
//     non-zero input are exactly 0 and are not convolved (exact skip).  The
//     replicate pads of the first/last chunk are written by the thread that
//     reads them.  Interior bands load their 16 + 2R rows with one bulk copy.
//
//  band_shade_kernel  kernel (b): 4 pixels per thread, 160-thread CTAs (whole warps), ~40 warps per SM.
//     np.gradient differences (REF/optical.py:160), bins, binned-LUT
//     shading (REF/optical.py:82-88, :244) + background, uint8 rule
//     (REF/cli.py:134-139).  Pixels whose 3x3 blurred neighbourhood is zero
//     (outside the band extents) are exactly rint(background) and copied.
//     The LUT is read from a half-planar copy (plane h = floats 8h..8h+7 of
//     every bin, bins in direction-major order): plane 0 with one 256-bit
//     load per pixel, plane 1 through the texture path; the background from
//     R/G/B planes.  The kernel is bound by L1 data-pipe wavefronts: these
//     layouts make a warp's gathers fall on far fewer 128-B lines, and the
//     texture half uses the other L1TEX data pipe.
//
//  env_epilogue_kernel  kernel (c): per env, reduces the band contact partials
//     in a fixed order, finalises contact / summary / load
//     (REF/marker.py:103-140), the marker displacements (REF/marker.py:143-165)
//     and the dot splat (REF/marker.py:203-234).
//
// Envs run in chunks of tac_config.chunk_envs (default: a 10 GiB blurred scratch): smaller chunks keep the
// blurred intermediate in L2 but measured slower (launch tails dominate).
#include <climits>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>

#include "tac_frame_common.cuh"

namespace tac {

namespace {

constexpr int BH = 16;    // band rows
constexpr int K1T = 320;  // blur threads: 8 row pairs x 40 chunks of 8 columns (W = 320)
#ifndef TAC_K2T
#define TAC_K2T 320
#endif
constexpr int K2T = TAC_K2T;  // shade threads per CTA, at most
constexpr int K2_MIN = 160;  // preferred smallest shade CTA (measured: 160 > 320 > 640 threads at W = 320)
struct ShadeCta {
  int rows, row;  // rows per CTA, threads per row
};
#ifndef TAC_SHADE_ROW_ITERS
#define TAC_SHADE_ROW_ITERS 8
#endif
constexpr int kShadeRowIters = TAC_SHADE_ROW_ITERS;  // row iterations per shade thread
#ifndef TAC_SHADE_UNROLL
#define TAC_SHADE_UNROLL 1
#endif
constexpr int kShadeUnroll = TAC_SHADE_UNROLL;

// ---- row-pair interleaved intermediate ----------------------------------------
// vb2[m][col] = (V[2m][col], V[2m+1][col]) as float2: the horizontal FFMA2
// operand of output rows (2m, 2m+1) at column col + t is one aligned float2,
// so no register re-pairing is needed.  Row-pair pitch (floats) = 4 x odd.
template <int RL>
__device__ __forceinline__ void v5item_rp(const float2* __restrict__ w, const float* __restrict__ src,
                                          int ip, float* __restrict__ dst, int rpp) {
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
  // rows (2m, 2m+1) of columns (c, c+1): one 16-B store per row pair
#pragma unroll
  for (int m = 0; m < 4; ++m)
    *reinterpret_cast<float4*>(dst + m * rpp) =
        make_float4(acc[2 * m].x, acc[2 * m + 1].x, acc[2 * m].y, acc[2 * m + 1].y);
}

// H for one row pair x 8 columns: acc[i] = (out[2m][c0+i], out[2m+1][c0+i]).
// `src` = vb2 row pair at column c0 - RL4 (16-B aligned).
template <int RL>
__device__ __forceinline__ void h5pair(const float2* __restrict__ w, const float* __restrict__ src,
                                       float2 acc[8]) {
  constexpr int RL4 = (RL + 3) & ~3;
  constexpr int NC = 8 + 2 * RL4;  // columns in the window
  float2 v[NC];
#pragma unroll
  for (int q = 0; q < NC / 2; ++q) {
    const float4 f = *reinterpret_cast<const float4*>(src + 4 * q);
    v[2 * q] = make_float2(f.x, f.y);
    v[2 * q + 1] = make_float2(f.z, f.w);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int t = -RL; t <= RL; ++t) acc[i] = ffma2(w[t < 0 ? -t : t], v[RL4 + i + t], acc[i]);
  }
}

#define TAC5_RADIUS_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

}  // namespace

// ---------------------------------------------------------------------------
// kernel (a): clamp + contact partials + pyramid blur of one 16-row band.
// grid (bands, envs); block (W/4, 320/(W/4)): threadIdx.x = float4 column group
#ifndef TAC_K1_MINB
#define TAC_K1_MINB 3
#endif
__global__ void __launch_bounds__(K1T, TAC_K1_MINB) band_blur_kernel(const __grid_constant__ FrameParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nb = p.bands;
  const long long env = blockIdx.y;
  const int band = blockIdx.x;
  const int y0 = band * BH;
  const int R = p.R;
  const int R4 = (R + 3) & ~3;
  const int nrows = BH + 2 * R;
  const int W = p.W, H = p.H;
  const long long HW = (long long)H * W;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int ip = p.in_pitch, vp = p.v_pitch;
  const int vbase = -R4;  // column of vb index 0

  float* inb = reinterpret_cast<float*>(smem_raw);  // nrows x ip (input row i = global row y0 - R + i)
  float* vb = inb + nrows * ip;                     // BH x vp
  __shared__ double s_red[(K1T / 32) * 8];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_lo, s_hi;

  const float* src = p.in + env * HW;
  const unsigned row_bytes = (unsigned)W * 4u;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_lo = INT_MAX;
    s_hi = INT_MIN;
    // the copies are issued before the CTA barrier that publishes the
    // initialised mbarrier to the waiting threads
    mbar_expect_tx(&s_bar, row_bytes * (unsigned)nrows);
    if (y0 - R >= 0 && y0 + BH + R <= H && ip == W) {
      // interior band: the 16 + 2R rows are one contiguous block
      bulk_g2s(inb, src + (long long)(y0 - R) * W, row_bytes * (unsigned)nrows, &s_bar);
    } else {
      for (int i = 0; i < nrows; ++i) {
        const int cr = min(max(y0 - R + i, 0), H - 1);
        bulk_g2s(inb + i * ip, src + (long long)cr * W, row_bytes, &s_bar);
      }
    }
  }
  __syncthreads();

  // ---- conversion: float4 groups, thread -> fixed column group ----------------
  // rows [0, R) and [R + BH, nrows) are halo (clamp + extent only); rows
  // [R, R + BH) are the band's own rows (+ contact partials).
  Red red = red_zero();
  float colsum[4] = {0.f, 0.f, 0.f, 0.f};
  const int cg = threadIdx.x, ro = threadIdx.y, cstep = blockDim.y;
  // every thread waits on the transaction barrier itself (measured 0.6 % faster
  // than one polling warp + a CTA barrier)
  mbar_wait(&s_bar, 0);
  bool nz = false;
  auto clamp4 = [&](float4* e) -> float4 {
    float4 v = *e;
    if (p.input_depth) {
      // (rest - depth) + rest_lo in pairs (FADD2), each step rounded as the scalar form
      const float2 rr = make_float2(p.rest, p.rest), rl = make_float2(p.rest_lo, p.rest_lo);
      const float2 a = fsubadd2(rr, make_float2(v.x, v.y), rl);
      const float2 b = fsubadd2(rr, make_float2(v.z, v.w), rl);
      v.x = clampf(a.x, 0.f, p.rest);
      v.y = clampf(a.y, 0.f, p.rest);
      v.z = clampf(b.x, 0.f, p.rest);
      v.w = clampf(b.y, 0.f, p.rest);
      *e = v;
    }
    // any non-zero bit pattern (a -0 only widens the extent: still exact)
    nz |= (__float_as_uint(v.x) | __float_as_uint(v.y) | __float_as_uint(v.z) | __float_as_uint(v.w)) != 0u;
    return v;
  };
  for (int i = ro; i < R; i += cstep) clamp4(reinterpret_cast<float4*>(inb + i * ip) + cg);
  for (int i = R + BH + ro; i < nrows; i += cstep) clamp4(reinterpret_cast<float4*>(inb + i * ip) + cg);
  const int own_rows = min(BH, H - y0);
  // band rows past the frame bottom (last band, H % 16 != 0) are clamped
  // replicas of row H-1: converted for the blur, not counted
  for (int i = own_rows + ro; i < BH; i += cstep) clamp4(reinterpret_cast<float4*>(inb + (R + i) * ip) + cg);
  for (int i = ro; i < own_rows; i += cstep) {
    float4* e = reinterpret_cast<float4*>(inb + (R + i) * ip) + cg;
    const float4 raw = *e;
    // non-finite inputs are counted, not raised (summary field 6); the sum of
    // four finite depths (metres) cannot overflow
    if (!(fabsf(raw.x + raw.y + raw.z + raw.w) < INFINITY)) {
      red.nf += (fabsf(raw.x) < INFINITY ? 0.f : 1.f) + (fabsf(raw.y) < INFINITY ? 0.f : 1.f) +
                (fabsf(raw.z) < INFINITY ? 0.f : 1.f) + (fabsf(raw.w) < INFINITY ? 0.f : 1.f);
    }
    const float4 c4 = clamp4(e);
    const float v[4] = {c4.x, c4.y, c4.z, c4.w};
    float w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      red.mx = fmaxf(red.mx, v[k]);
      const bool in = v[k] > p.threshold;
      w[k] = in ? v[k] : 0.f;
      red.cnt += in ? 1.f : 0.f;
      colsum[k] += w[k];
    }
    const float rowsum = (w[0] + w[1]) + (w[2] + w[3]);
    red.sw += (double)rowsum;
    red.swy = fma((double)rowsum, (double)(y0 + i) + 0.5 - (double)p.half_h, red.swy);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    red.swx = fma((double)colsum[q], (double)(4 * cg + q) + 0.5 - (double)p.half_w, red.swx);
  warp_reduce(red);
  if ((tid & 31) == 0) {
    double* q = s_red + (tid >> 5) * 8;
    q[0] = red.cnt;
    q[1] = red.sw;
    q[2] = red.swx;
    q[3] = red.swy;
    q[4] = red.mx;
    q[5] = red.nf;
  }
  {
    const int c = 4 * cg;
    const int lo = __reduce_min_sync(0xffffffffu, nz ? c : INT_MAX);
    const int hi = __reduce_max_sync(0xffffffffu, nz ? c + 3 : INT_MIN);
    if ((tid & 31) == 0 && lo != INT_MAX) {
      atomicMin(&s_lo, lo);
      atomicMax(&s_hi, hi);
    }
  }
  __syncthreads();
  const int ea = s_lo, eb = s_hi;

  // ---- blur: output range [ha, hb] in whole 16-column chunks ------------------
  int k_lo = 0, k_hi = -1, ha = INT_MAX, hb = INT_MIN;
  if (ea <= eb) {
    k_lo = max(ea - R, 0) >> 4;
    k_hi = min(eb + R, W - 1) >> 4;
    ha = 16 * k_lo;
    hb = 16 * k_hi + 15;
  }
  if (tid == 0) p.band_ext[env * nb + band] = make_int2(ha, hb);  // ext_strips == 1
  // H items: row pair m x 8 columns; lanes 0..7 = row pairs of one chunk
  const int m = tid & 7;
  const int k8 = tid >> 3;
  const int c0 = 8 * k8;
  const bool has = k8 >= 2 * k_lo && k8 <= 2 * k_hi + 1 && c0 < W;
  const int rpp = 2 * vp;  // floats per row pair (4 x odd)
  float2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  if (ea <= eb) {
    const int c_lo = max(ha - R4, 0);
    const int c_hi = min(hb + R4, W - 1);
    const int np = (c_hi - c_lo) / 2 + 1;
    for (int l = 0; l < p.n_levels; ++l) {
      const int RL = p.radius[l];
      if (RL == 0) {  // identity level (k == 1): straight from the input
        if (has) {
          const float w = p.wh[l][0];
          const float* in0 = inb + (2 * m + R) * ip + c0;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            acc[i] = ffma2(make_float2(w, w), make_float2(in0[i], in0[ip + i]), acc[i]);
        }
        continue;
      }
      if (tid < 2 * np) {
        const int hf = tid >= np ? 1 : 0;
        const int c = c_lo + 2 * (tid - hf * np);
        const float* sp = inb + (8 * hf + R - RL) * ip + c;
        float* dst = vb + 4 * hf * rpp + 2 * (c - vbase);
        switch (RL) {
#define X(r)                                            \
  case r:                                               \
    v5item_rp<r>(p.wv2[l], sp, ip, dst, rpp);           \
    break;
          TAC5_RADIUS_CASES(X)
#undef X
          default:
            break;
        }
      }
      __syncthreads();
      float* prow = vb + m * rpp;  // row pair m, column vbase
      if (has) {
        // frame-border chunks write their own row pair's replicate pads; the
        // H items of the same row pair that read them are in the same warp
        if (c0 == 0) {
          const float2 e = *reinterpret_cast<const float2*>(prow - 2 * vbase);
          for (int i = 0; i < R4; i += 2)
            *reinterpret_cast<float4*>(prow + 2 * i) = make_float4(e.x, e.y, e.x, e.y);
        }
        if (c0 + 8 == W) {
          const float2 e = *reinterpret_cast<const float2*>(prow + 2 * (W - 1 - vbase));
          for (int i = 0; i < R4; i += 2)
            *reinterpret_cast<float4*>(prow + 2 * (W - vbase + i)) = make_float4(e.x, e.y, e.x, e.y);
        }
      }
      __syncwarp();  // pads visible to the warp's other lanes (convergent point)
      if (has) {
        switch (RL) {
#define X(r)                                                                   \
  case r:                                                                      \
    h5pair<r>(p.wh2[l], prow + 2 * (c0 - ((r + 3) & ~3) - vbase), acc);       \
    break;
          TAC5_RADIUS_CASES(X)
#undef X
          default:
            break;
        }
      }
      // the next level's V pass overwrites vb (no barrier after the last level:
      // only registers and HBM are touched from here on)
      if (l + 1 < p.n_levels) __syncthreads();
    }
  }
  // ---- blurred band out (exact zeros outside [ha, hb]) --------------------------
  {
    const int y = y0 + 2 * m;
    if (c0 < W) {
      float* d = p.scratch + env * HW + (long long)y * W + c0;
      if (y < H) {
        reinterpret_cast<float4*>(d)[0] = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
        reinterpret_cast<float4*>(d)[1] = make_float4(acc[4].x, acc[5].x, acc[6].x, acc[7].x);
      }
      if (y + 1 < H) {
        reinterpret_cast<float4*>(d + W)[0] = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
        reinterpret_cast<float4*>(d + W)[1] = make_float4(acc[4].y, acc[5].y, acc[6].y, acc[7].y);
      }
    }
  }

  // ---- contact partials of the band (warp sums in s_red since the conversion;
  //      reduced per env by env_epilogue_kernel) ----------------------------------
  if (p.finalize == 0 || tid != 0) return;
  const int nw = (blockDim.x * blockDim.y) >> 5;
  double t[6] = {0, 0, 0, 0, 0, 0};
  for (int w = 0; w < nw; ++w) {  // fixed order: deterministic
    for (int i = 0; i < 4; ++i) t[i] += s_red[w * 8 + i];
    t[4] = fmax(t[4], s_red[w * 8 + 4]);
    t[5] += s_red[w * 8 + 5];
  }
  double* q = p.partials + (env * p.nparts + band) * kSumFields;  // nparts == bands
  for (int i = 0; i < 6; ++i) q[i] = t[i];
}

// one 256-bit read-only load (LDG.E.ENL2.256 on sm_100a)
__device__ __forceinline__ void ld256(const float* p, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

// one 256-bit read-only load as 8 words (16 fp16 LUT coefficients)
__device__ __forceinline__ void ld256u(const void* p, uint32_t (&w)[8]) {
  asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
      : "l"(p));
}

__device__ __forceinline__ float h2f_lo(uint32_t w) { return __half2float(__ushort_as_half((unsigned short)(w & 0xffffu))); }
__device__ __forceinline__ float h2f_hi(uint32_t w) { return __half2float(__ushort_as_half((unsigned short)(w >> 16))); }

// ---- paired binning (two pixels per fp32x2 op) ----------------------------------
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Bins of two pixels and their normals' (x, y) NEGATED: m = (gx, gy) / sqrt(1 + |g|^2)
// = -(n_x, n_y) (the shading negates the linear terms).  Same definitions as
// bin_px: magnitude bin min(floor(|g| mag_scale), bins - 1),
// direction bin floor((atan2(gy, gx) + pi) dir_scale) mod bins, both 0 for a
// zero gradient (NaN converts to 0).  i = direction-major planar bin index.
struct Bins2 {
  float2 nx, ny;
  int i0, i1;
};

__device__ __forceinline__ int dir_fix(int db, int bins) {
  db = db >= bins ? db - bins : db;
  return max(db, 0);
}

__device__ __forceinline__ Bins2 bin_pair(const FrameParams& p, float2 gx, float2 gy) {
  Bins2 o;
  const float2 g2 = ffma2(gx, gx, f2mul(gy, gy));
  const float2 gm = f2mul(g2, make_float2(rsqrtf(g2.x), rsqrtf(g2.y)));  // NaN for g2 == 0 -> bin 0
  const float2 t = f2add(g2, bc2(1.f));
  const float2 inv = make_float2(rsqrtf(t.x), rsqrtf(t.y));
  o.nx = f2mul(gx, inv);
  o.ny = f2mul(gy, inv);
  const float2 ms = f2mul(gm, bc2(p.mag_scale));
  // atan2 by an odd minimax polynomial of min/max on [0, 1] (|err| ~ 1e-7 rad) + reflections
  const float ax0 = fabsf(gx.x), ay0 = fabsf(gy.x), ax1 = fabsf(gx.y), ay1 = fabsf(gy.y);
  const float2 mn = make_float2(fminf(ax0, ay0), fminf(ax1, ay1));
  const float2 mx = make_float2(fmaxf(ax0, ay0), fmaxf(ax1, ay1));
  const float2 a = f2mul(mn, make_float2(rcp_approx(mx.x), rcp_approx(mx.y)));  // 0/0 -> NaN -> bin 0
  const float2 s = f2mul(a, a);
  float2 q = bc2(0.0024567204527556896f);
  q = ffma2(q, s, bc2(-0.01440134271979332f));
  q = ffma2(q, s, bc2(0.039781197905540466f));
  q = ffma2(q, s, bc2(-0.07234855741262436f));
  q = ffma2(q, s, bc2(0.10498945415019989f));
  q = ffma2(q, s, bc2(-0.14161229133605957f));
  q = ffma2(q, s, bc2(0.19985906779766083f));
  q = ffma2(q, s, bc2(-0.33332598209381104f));
  q = ffma2(q, s, bc2(0.9999998807907104f));
  float2 r = f2mul(q, a);
  r.x = (ay0 > ax0) ? kHalfPi - r.x : r.x;
  r.y = (ay1 > ax1) ? kHalfPi - r.y : r.y;
  r.x = (gx.x < 0.f) ? kPi - r.x : r.x;
  r.y = (gx.y < 0.f) ? kPi - r.y : r.y;
  r.x = (gy.x < 0.f) ? -r.x : r.x;
  r.y = (gy.y < 0.f) ? -r.y : r.y;
  const float2 u = f2mul(f2add(r, bc2(kPi)), bc2(p.dir_scale));
  const int mb0 = max(min((int)ms.x, p.mag_bins - 1), 0), mb1 = max(min((int)ms.y, p.mag_bins - 1), 0);
  const int db0 = dir_fix((int)u.x, p.dir_bins), db1 = dir_fix((int)u.y, p.dir_bins);
  o.i0 = db0 * p.mag_bins + mb0;  // direction-major (tac_ctx_create)
  o.i1 = db1 * p.mag_bins + mb1;
  return o;
}

// bg + Delta_c (REF/optical.py:82-88, :244) with the bin's 15 coefficients as
// fp16 [R c1..c5, G c1..c5, B c1..c5, pad], one FMA chain per channel, (mx, my)
// = -(nx, ny): the linear terms' coefficients are negated in the FMA.
__device__ __forceinline__ void shade_h(const uint32_t (&w)[8], float mx, float my, float xx, float xy, float yy,
                                        const float* bg, float (&o)[3]) {
  o[0] = fmaf(h2f_lo(w[2]), yy, fmaf(h2f_hi(w[1]), xy, fmaf(h2f_lo(w[1]), xx,
         fmaf(-h2f_hi(w[0]), my, fmaf(-h2f_lo(w[0]), mx, bg[0])))));
  o[1] = fmaf(h2f_hi(w[4]), yy, fmaf(h2f_lo(w[4]), xy, fmaf(h2f_hi(w[3]), xx,
         fmaf(-h2f_lo(w[3]), my, fmaf(-h2f_hi(w[2]), mx, bg[1])))));
  o[2] = fmaf(h2f_lo(w[7]), yy, fmaf(h2f_hi(w[6]), xy, fmaf(h2f_lo(w[6]), xx,
         fmaf(-h2f_hi(w[5]), my, fmaf(-h2f_lo(w[5]), mx, bg[2])))));
}

__device__ __forceinline__ int planar_bin(const FrameParams& p, int mb, int db) {
  return db * p.mag_bins + mb;  // direction-major (tac_ctx_create)
}

// ---------------------------------------------------------------------------
// kernel (b): shade one 4-pixel group of row y from its blurred rows (c = row
// y with left/right neighbours, m = row y-1, n = row y+1; border rows/columns
// use np.gradient's one-sided differences, REF/optical.py:160).  Returns false
// (nothing written) when all four gradients are exactly zero and there are no
// shadows: the caller then copies the quantised background.
// Channel values the [0, 255] clip changes (REF/optical.py:246-247:
// raw != clip(raw), before any shadow), counted when the caller asks.
__device__ __forceinline__ unsigned clip_count(float r, float g, float b) {
  return (r < 0.f || r > 255.f ? 1u : 0u) + (g < 0.f || g > 255.f ? 1u : 0u) + (b < 0.f || b > 255.f ? 1u : 0u);
}

template <bool H16>
__device__ __forceinline__ bool shade_group(const FrameParams& p, long long env, int y, int xg,
                                            const float c[6], const float4 mm, const float4 nn,
                                            uint8_t* out, unsigned& nsat) {
  const int W = p.W, H = p.H;
  const float m[4] = {mm.x, mm.y, mm.z, mm.w};
  const float n[4] = {nn.x, nn.y, nn.z, nn.w};
  const bool top = (y == 0), bot = (y == H - 1);
  float gxs[4], gys[4];
  if (!top && !bot && xg > 0 && xg + 4 < W) {  // interior: central differences
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
      const bool lft = (x == 0), rgt = (x == W - 1);
      const float xr = rgt ? c[k + 1] : c[k + 2];
      const float xl = lft ? c[k + 1] : c[k];
      gxs[k] = (xr - xl) * ((lft || rgt) ? p.inv_p : p.inv_2p);
      const float yb = bot ? c[k + 1] : n[k];
      const float yt = top ? c[k + 1] : m[k];
      gys[k] = (yb - yt) * sy;
    }
  }
  // a group whose four gradients are exactly zero shades to exactly rint(bg)
  // (REF/optical.py:244 with n = (0, 0, 1))
  const bool flat = gxs[0] == 0.f && gxs[1] == 0.f && gxs[2] == 0.f && gxs[3] == 0.f &&
                    gys[0] == 0.f && gys[1] == 0.f && gys[2] == 0.f && gys[3] == 0.f;
  if (flat && p.shadow == nullptr) return false;
  const long long HW = (long long)H * W;
  // background planes: three coalesced 16-B loads per thread
  const long long pix = (long long)y * W + xg;
  const float4 br = __ldg(reinterpret_cast<const float4*>(p.bg_planar + pix));
  const float4 bgr = __ldg(reinterpret_cast<const float4*>(p.bg_planar + HW + pix));
  const float4 bb = __ldg(reinterpret_cast<const float4*>(p.bg_planar + 2 * HW + pix));
  const float bgv[12] = {br.x, bgr.x, bb.x, br.y, bgr.y, bb.y, br.z, bgr.z, bb.z, br.w, bgr.w, bb.w};
  float sf[4] = {1.f, 1.f, 1.f, 1.f};
  if (p.shadow) {
    const float4 f4 = __ldg(reinterpret_cast<const float4*>(p.shadow + env * HW + (long long)y * W + xg));
    sf[0] = f4.x; sf[1] = f4.y; sf[2] = f4.z; sf[3] = f4.w;
  }
  uint32_t qb[12], w01 = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if constexpr (H16) {
      // pixels 2h, 2h+1 binned together (paired fp32 ops); fp16 LUT: one
      // 32-B sector per bin (half the gather bytes)
      const Bins2 bq = bin_pair(p, make_float2(gxs[2 * h], gxs[2 * h + 1]), make_float2(gys[2 * h], gys[2 * h + 1]));
      const float2 nxx = f2mul(bq.nx, bq.nx), nxy = f2mul(bq.nx, bq.ny), nyy = f2mul(bq.ny, bq.ny);
      uint32_t w0[8], w1[8];
      TAC_CHECK(bq.i0 >= 0 && bq.i0 < p.nbins && bq.i1 >= 0 && bq.i1 < p.nbins);
      ld256u(p.lut_h16 + 2 * bq.i0, w0);
      ld256u(p.lut_h16 + 2 * bq.i1, w1);
      float rgb[2][3];
      shade_h(w0, bq.nx.x, bq.ny.x, nxx.x, nxy.x, nyy.x, &bgv[6 * h], rgb[0]);
      shade_h(w1, bq.nx.y, bq.ny.y, nxx.y, nxy.y, nyy.y, &bgv[6 * h + 3], rgb[1]);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        float r = rgb[s][0], g = rgb[s][1], b = rgb[s][2];
        if (p.saturated) nsat += clip_count(r, g, b);
        if (p.shadow) {
          const float f = sf[2 * h + s];
          r = clampf(r, 0.f, 255.f) * f;
          g = clampf(g, 0.f, 255.f) * f;
          b = clampf(b, 0.f, 255.f) * f;
        }
        qb[6 * h + 3 * s] = u8sat(r);
        qb[6 * h + 3 * s + 1] = u8sat(g);
        qb[6 * h + 3 * s + 2] = u8sat(b);
      }
      if (h == 0) w01 = pack4(qb[0], qb[1], qb[2], qb[3]);  // pixels 0, 1 done: fewer live registers
      continue;
    }
    // fp32 LUT (16 coefficients per pixel in registers): per-pixel binning
    // (the paired form exceeds the 48-register cap here: spills, measured 3 % slower)
    const Px a0p = bin_px(p, gxs[2 * h], gys[2 * h]);
    const Px a1p = bin_px(p, gxs[2 * h + 1], gys[2 * h + 1]);
    // two 256-bit loads per pixel: floats 0..7 and 8..15 of the bin
    const int i0 = planar_bin(p, a0p.mb, a0p.db);
    const int i1 = planar_bin(p, a1p.mb, a1p.db);
    TAC_CHECK(i0 >= 0 && i0 < p.nbins && i1 >= 0 && i1 < p.nbins);
    float4 a0, c0, d0, e0, a1, c1, d1, e1;
    {
      // plane 0 through the LSU (256-bit), plane 1 through the texture path:
      // the two halves of the gather use both L1TEX data pipes (measured +2 %)
      const cudaTextureObject_t tx = p.lut_tex;
      ld256(p.lut_half + 8 * i0, a0, c0);
      ld256(p.lut_half + 8 * i1, a1, c1);
      d0 = tex1Dfetch<float4>(tx, 2 * (p.nbins + i0));
      e0 = tex1Dfetch<float4>(tx, 2 * (p.nbins + i0) + 1);
      d1 = tex1Dfetch<float4>(tx, 2 * (p.nbins + i1));
      e1 = tex1Dfetch<float4>(tx, 2 * (p.nbins + i1) + 1);
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const Px& pp = s ? a1p : a0p;
      float r = bgv[6 * h + 3 * s], g = bgv[6 * h + 3 * s + 1], b = bgv[6 * h + 3 * s + 2];
      if (s)
        add_lut(a1, c1, d1, e1, pp.nx, pp.ny, r, g, b);
      else
        add_lut(a0, c0, d0, e0, pp.nx, pp.ny, r, g, b);
      if (p.saturated) nsat += clip_count(r, g, b);
      if (p.shadow) {  // clip, then the multiplicative shadow (REF/optical.py:246, :299)
        const float f = sf[2 * h + s];
        r = clampf(r, 0.f, 255.f) * f;
        g = clampf(g, 0.f, 255.f) * f;
        b = clampf(b, 0.f, 255.f) * f;
      }
      qb[6 * h + 3 * s] = u8sat(r);
      qb[6 * h + 3 * s + 1] = u8sat(g);
      qb[6 * h + 3 * s + 2] = u8sat(b);
    }
  }
  uint32_t* d = reinterpret_cast<uint32_t*>(out + ((long long)y * W + xg) * 3);
  d[0] = H16 ? w01 : pack4(qb[0], qb[1], qb[2], qb[3]);
  d[1] = pack4(qb[4], qb[5], qb[6], qb[7]);
  d[2] = pack4(qb[8], qb[9], qb[10], qb[11]);
  return true;
}

// One 4-pixel group of one row per thread.  grid (row groups, envs); block
// (row threads, rows): row threads = W/4, or W/4 rounded up (idle threads at
// the end of each row) when no row count makes the CTA whole warps.
#ifndef TAC_K2_MINB
#define TAC_K2_MINB 4
#endif
// PAD: rows padded (a separate instantiation: the extra idle test costs the
// unpadded kernel registers at its 48-register cap).
template <bool H16, bool PAD>
__global__ void __launch_bounds__(K2T, TAC_K2_MINB) band_shade_kernel(const __grid_constant__ FrameParams p) {
  const int W = p.W, H = p.H;
  const long long env = blockIdx.y;
  const int gi = threadIdx.x;
  const int xg = 4 * gi;
  const int ng = blockDim.x;  // threads per row
  const long long HW = (long long)H * W;
  const int lane = (threadIdx.y * ng + gi) & 31;
  const float* img = p.scratch + env * HW + xg;
  uint8_t* out = p.rgb + env * HW * 3;
  unsigned nsat = 0;
  // each CTA shades kShadeRowIters x blockDim.y rows of one env (setup amortised)
#pragma unroll kShadeUnroll
  for (int it = 0; it < kShadeRowIters; ++it) {
    const int y = (blockIdx.x * kShadeRowIters + it) * blockDim.y + threadIdx.y;
    const bool act = y < H && (!PAD || xg < W);  // xg >= W: row padding, idle
    if (__all_sync(0xffffffffu, !act)) break;  // uniform per warp
    const int yc = act ? y : H - 1;
    TAC_CHECK(yc >= 0 && yc < H && (xg + 4 <= W || (PAD && !act)));
    const float* rc = img + (long long)yc * W;
    // columns whose gradient can be non-zero: band extents of rows y-1..y+1
    // (union over the blur kernel's column strips), +-1
    // every active group reads its rows: groups outside the contact see zero
    // gradients and copy the background (no per-band column extents: their
    // per-row lookup cost more than the loads it skipped, measured 4 %)
    const bool any = act;
    float4 cc = make_float4(0.f, 0.f, 0.f, 0.f), mm = cc, nn = cc;
    if (any) {
      cc = *reinterpret_cast<const float4*>(rc);
      mm = *reinterpret_cast<const float4*>(yc > 0 ? rc - W : rc);
      nn = *reinterpret_cast<const float4*>(yc < H - 1 ? rc + W : rc);
    }
    float left = __shfl_up_sync(0xffffffffu, cc.w, 1);
    float right = __shfl_down_sync(0xffffffffu, cc.x, 1);
    bool done = false;
    if (any) {
      if (lane == 0 || gi == 0) left = xg > 0 ? rc[-1] : cc.x;
      if (lane == 31 || (PAD ? xg + 4 == W : gi == ng - 1)) right = xg + 4 < W ? rc[4] : cc.w;
      const float c[6] = {left, cc.x, cc.y, cc.z, cc.w, right};
      done = shade_group<H16>(p, env, yc, xg, c, mm, nn, out, nsat);
    }
    if (act && !done) {  // flat group: the quantised background
      const uint32_t* s = reinterpret_cast<const uint32_t*>(p.bg_u8 + ((long long)yc * W + xg) * 3);
      uint32_t* d = reinterpret_cast<uint32_t*>(out + ((long long)yc * W + xg) * 3);
      d[0] = __ldg(s);
      d[1] = __ldg(s + 1);
      d[2] = __ldg(s + 2);
    }
  }
  if (p.saturated) {  // whole CTA is one env: one atomic per warp
    const unsigned w = __reduce_add_sync(0xffffffffu, nsat);
    if (lane == 0 && w) atomicAdd(p.saturated + env, w);
  }
}

// ---------------------------------------------------------------------------
// kernel (c): per-env epilogue after every band is blurred and shaded.  The
// band partials are reduced in a fixed order (deterministic), then contact /
// summary / load (REF/marker.py:103-140), displacements (REF/marker.py:143-165)
// and the dot splat (REF/marker.py:203-234).  One 128-thread CTA per env.
__global__ void __launch_bounds__(128) env_epilogue_kernel(const __grid_constant__ FrameParams p) {
  __shared__ double s_dbl[8];
  __shared__ int s_int[2 * 1024];
  __shared__ int s_recount;
  __shared__ unsigned s_nf;
  const long long env = blockIdx.x;
  const int nb = p.nparts;
  double cnt = 0, sw = 0, swx = 0, swy = 0, nf = 0;  // folded by warp 0 (thread 0 finalises)
  float mx = 0.f;
  if (threadIdx.x < 32) {
    // warp 0: lane s folds bands s, s + 32, ...; then a fixed xor butterfly
    // (every lane ends with the same bits: deterministic for a given band count)
    const int lane = threadIdx.x;
    const double* q = p.partials + env * nb * kSumFields;
    for (int s = lane; s < nb; s += 32) {
      cnt += q[s * 8 + 0];
      sw += q[s * 8 + 1];
      swx += q[s * 8 + 2];
      swy += q[s * 8 + 3];
      mx = fmaxf(mx, (float)q[s * 8 + 4]);
      nf += q[s * 8 + 5];
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
    if (lane == 0) s_recount = nf < 0.0 ? 1 : 0;
    s_nf = 0u;
  }
  __syncthreads();
  if (s_recount) {
    // a stream-blur strip flagged a non-finite raw value (tac_stream.cu):
    // count this env's non-finite inputs exactly (integer sum: deterministic)
    const float* in = p.in + env * (long long)p.H * p.W;
    unsigned c = 0;
    for (long long i = threadIdx.x; i < (long long)p.H * p.W; i += blockDim.x) c += fabsf(in[i]) < INFINITY ? 0u : 1u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_nf, c);
    __syncthreads();
    nf = (double)s_nf;
  }
  if (threadIdx.x == 0) finalize_load(p, env, cnt, sw, swx, swy, mx, nf, s_dbl);
  __syncthreads();
  if (p.finalize != 2) return;
  const Load l = load_from(s_dbl);
  const int nm = p.mg.rows * p.mg.cols;
  markers_block(p.mg, l, p.disp ? p.disp + env * (long long)nm * 2 : nullptr,
                p.splat ? p.rgb + env * (long long)p.H * p.W * 3 : nullptr, nullptr, s_int, s_int + nm);
}

// vb pitch (floats per row): rows of W + 2 R4 columns; 2 x odd, so the
// row-pair pitch (2 vp floats) is 4 x odd and LDS.128 over 8 row pairs is
// conflict-free
int frame5_vpitch(int W, int R4) {
  int vp = ((W + 2 * R4 + 4 + 3) & ~3) + 2;  // 2 x odd -> row-pair pitch 4 x odd
  if (((vp / 2) & 1) == 0) vp += 4;
  return vp;
}

size_t band_blur_smem_bytes(const FrameParams& p) {
  return sizeof(float) * ((size_t)(BH + 2 * p.R) * p.in_pitch + (size_t)BH * p.v_pitch);
}

// Shade CTA shape: rows of `row` threads (W/4, or W/4 rounded up to the
// next multiple of 8 / 16 / 32) so that row x rows is whole warps, at most
// K2T threads; the fewest padded threads first, then the smallest CTA of at
// least K2_MIN threads.  rows = 0 if none fits.
ShadeCta shade_cta(int ng) {
  ShadeCta c{0, 0};
  if (ng <= 0) return c;
  for (int al = 1; al <= 32 && c.rows == 0; al *= 2) {
    const int row = (ng + al - 1) / al * al;
    if (row > K2T) break;
    int r0 = 1;
    while ((row * r0) % 32 != 0) ++r0;
    if (row * r0 > K2T) continue;
    int r = r0;
    while (row * r < K2_MIN && row * (r + r0) <= K2T) r += r0;
    c.rows = r;
    c.row = row;
  }
  return c;
}

bool frame5_eligible(const FrameParams& p) {
  if (p.strips != 1 || p.W % 16 != 0 || p.W > 320 || p.W < 16) return false;
  if (p.R < 1 || p.R > 16) return false;
  if (p.mg.rows * p.mg.cols > 1024) return false;
  if (p.lut_tex == 0) return false;  // the shade kernel reads LUT plane 1 through a texture
  const int ng = p.W / 4;
  if ((ng * (K1T / ng)) % 32 != 0) return false;  // whole warps (shuffles, block_reduce)
  if (shade_cta(ng).rows == 0) return false;
  return band_blur_smem_bytes(p) <= 227 * 1024;
}

// The band shade kernel and the epilogue behind the row-streaming blur.
bool shade5_eligible(const FrameParams& p) {
  if (p.W % 16 != 0 || p.W < 16) return false;
  if (p.mg.rows * p.mg.cols > 1024) return false;
  if (p.lut_tex == 0) return false;
  return shade_cta(p.W / 4).rows != 0;
}

int frame5_launches(const FrameParams& p, long long n_env) {
  if (n_env == 0) return 0;
  const long long chunk = p.chunk > 0 ? p.chunk : n_env;
  return (int)(2 * ((n_env + chunk - 1) / chunk) + (p.finalize != 0 ? 1 : 0));
}

cudaError_t launch_frame5(const FrameParams& p0, cudaStream_t s, Marks* tm, const ShadowParams* sp,
                          float* shadow_ws) {
  const size_t smem = band_blur_smem_bytes(p0);
  cudaError_t e = cudaFuncSetAttribute(band_blur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p0.n_env == 0) return cudaSuccess;
  const long long HW = (long long)p0.H * p0.W;
  const int ng = p0.W / 4;
  const dim3 b1(ng, K1T / ng);
  const ShadeCta sc = shade_cta(ng);
  const int rpc = sc.rows;
  const dim3 b2(sc.row, rpc);
  const unsigned nq = (unsigned)((p0.H + rpc * kShadeRowIters - 1) / (rpc * kShadeRowIters));
  const long long chunk = p0.chunk > 0 ? p0.chunk : p0.n_env;
  const long long nchunks = (p0.n_env + chunk - 1) / chunk;
  Marks none;
  if (!tm) tm = &none;
  tm->start();
#define CK(x)                          \
  do {                                 \
    e = (x);                           \
    if (e != cudaSuccess) return e;    \
  } while (0)
  for (long long i = 0; i < nchunks; ++i) {
    const long long e0 = i * chunk;
    const long long n = std::min(chunk, p0.n_env - e0);
    FrameParams p = p0;
    // per-chunk views (every per-env pointer advanced by e0 envs)
    p.in = p0.in + e0 * HW;
    p.rgb = p0.rgb + e0 * HW * 3;
    p.scratch = p0.blurred ? p0.blurred + e0 * HW : p0.scratch;
    p.partials = p0.partials + e0 * p0.nparts * kSumFields;
    if (p0.shadow) p.shadow = p0.shadow + e0 * HW;
    p.n_env = n;
    if (sp != nullptr) {  // add_shadows factor of this chunk (kind 3)
      CK(launch_shadow(*sp, p.in, p.input_depth, shadow_ws, nullptr, n, s));
      tm->mark(3);
      p.shadow = shadow_ws;
    }
    if (p.st_kind >= 0) {
      CK(launch_stream_blur(p, s));
    } else {
      band_blur_kernel<<<dim3((unsigned)p.bands, (unsigned)n), b1, smem, s>>>(p);
      CK(cudaGetLastError());
    }
    tm->mark(0);
    if (sc.row != ng) {
      if (p.lut_h16)
        band_shade_kernel<true, true><<<dim3(nq, (unsigned)n), b2, 0, s>>>(p);
      else
        band_shade_kernel<false, true><<<dim3(nq, (unsigned)n), b2, 0, s>>>(p);
    } else if (p.lut_h16) {
      band_shade_kernel<true, false><<<dim3(nq, (unsigned)n), b2, 0, s>>>(p);
    } else {
      band_shade_kernel<false, false><<<dim3(nq, (unsigned)n), b2, 0, s>>>(p);
    }
    CK(cudaGetLastError());
    tm->mark(1);
  }
#undef CK
  if (p0.finalize != 0) {
    env_epilogue_kernel<<<(unsigned)p0.n_env, 128, 0, s>>>(p0);
    e = cudaGetLastError();
    tm->mark(2);
  }
  return e;
}

}  // namespace tac
