// Slot-ring frame kernel (v4): kernel (a) clamp + multi-scale Gaussian pyramid,
// fused with kernel (b) gradient -> binned LUT -> background -> uint8 and the
// contact reductions / marker epilogue of kernel (c).  One launch per step.
//
// Differences from the strip-streaming v3 kernel (tac_frame.cu):
//  * the converted input lives in a ring of 3 slots of RB rows; TMA
//    (cp.async.bulk, one copy per row, clamped row index = replicate border of
//    REF/tactile.py:219-221) refills the slot of block b-1 with block b+2
//    while block b's horizontal pass runs, so no halo rows are ever shifted;
//  * every slot carries the column extent of its non-zero indentation.  The
//    blur of block b only touches columns within R of the union extent of
//    slots b-1..b+1, and the shading only shades columns whose 3x3 blurred
//    neighbourhood can be non-zero; everywhere else the blurred value is
//    exactly 0 and the RGB is exactly rint(background) (REF/optical.py:244-246
//    with a zero gradient) -- an exact skip, not an approximation;
//  * the vertical passes of all levels run in one phase and the horizontal
//    pass sums all levels per output (one store, no read-modify-write), so the
//    blur group passes 2 CTA-group barriers per 16-row block instead of ~11;
//  * the shade group shades 16 pixels per thread and writes RGB straight to
//    HBM with 16-byte stores (no staging buffer).
//
// Blur group = threads [0, 320), shade group = [320, 640), handing 16-row
// blocks over through a 2-slot blurred ring with FULL/EMPTY named barriers.
#include <climits>
#include <cstdio>

#include "tac_frame_common.cuh"

namespace tac {

namespace {

constexpr int kIn4 = 3;                 // input slots (R <= RB: window = slots of blocks b-1..b+1)
#ifndef TAC_V4_SLOTS
#define TAC_V4_SLOTS 2
#endif
constexpr int kSl4 = TAC_V4_SLOTS;      // blurred ring slots
constexpr int kRing4 = kSl4 * RB;
constexpr int kShade4 = 320;            // shade-group threads
enum : int { kB4Blur = 1, kB4Full = 3, kB4Empty = 3 + kSl4 };

__device__ __forceinline__ int ring4(int r) { return (r + kRing4) % kRing4; }
__device__ __forceinline__ void bsync4() { bar_sync(kB4Blur, kThreads); }
__device__ __forceinline__ int slot_of(int q) { return (q + kIn4) % kIn4; }  // q >= -1

// Shared state of one CTA besides the big buffers.
struct S4 {
  int ext_lo[kIn4], ext_hi[kIn4];  // non-zero column extent of each input slot (global cols)
  int sh_lo[kSl4], sh_hi[kSl4];    // shading column range of each blurred ring slot
};

// ---- vertical pass item: column pair x 8 rows of one level -------------------
// Output rows r0 + 8*hf + k (k < 8) need input rows r0 + 8*hf + k + t, |t| <= RL,
// i.e. offsets rel = 8*hf - RL + j from r0, j < 8 + 2*RL; rel < 0 lives in the
// slot of block b-1, rel >= RB in the slot of block b+1 (R <= RB).  The row
// pointer of load j is one of three per-item bases chosen by two compares
// (j < s1, j < s2), so the unrolled body is shared by both halves.
template <int RL>
__device__ __forceinline__ void vitem(const float* __restrict__ w1, const float* sp, const float* sc,
                                      const float* sn, int ip, int hf, int col, float* __restrict__ dst,
                                      int vp, bool st_y) {
  float2 w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = make_float2(w1[i], w1[i]);
  // row rel = 8*hf - RL + j: slot b-1 for j < s1, b for j < s2, else b+1
  const int s1 = RL - 8 * hf, s2 = RB + RL - 8 * hf;
  const float* b0 = sp + (8 * hf - RL + RB) * ip + col;
  const float* b1 = sc + (8 * hf - RL) * ip + col;
  const float* b2 = sn + (8 * hf - RL - RB) * ip + col;
  float2 acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 8 + 2 * RL; ++j) {
    const float* base = j < s1 ? b0 : (j < s2 ? b1 : b2);
    const float2 v = *reinterpret_cast<const float2*>(base + j * ip);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int t = j - k - RL;
      if (t >= -RL && t <= RL) acc[k] = ffma2(w[t < 0 ? -t : t], v, acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (st_y)
      *reinterpret_cast<float2*>(dst + k * vp) = acc[k];  // (c - vbase) and vp are even
    else
      dst[k * vp] = acc[k].x;
  }
}

// ---- horizontal pass: one row x 16 columns, all levels summed ----------------
// acc[i] = (out[c0 + 2i], out[c0 + 2i + 1]) += sum_t w[|t|] * v[c0 + 2i + t].
// `src` points at column c0 - RL4 of the level's vb row (16-B aligned).
// SLOW: the window leaves the computed vb columns [c_lo, chi] or the frame:
// column indices are clamped to the frame (replicate border, scipy
// mode="nearest") and uncomputed columns read as the exact zero they are.
template <int RL>
__device__ __forceinline__ void hlevel(const float* __restrict__ w1, const float* __restrict__ src,
                                       float2 acc[8]) {
  constexpr int RL4 = (RL + 3) & ~3;
  constexpr int NV = 16 + 2 * RL4;
  float v[NV];
#pragma unroll
  for (int q = 0; q < NV / 4; ++q) {
    const float4 f = *reinterpret_cast<const float4*>(src + 4 * q);
    v[4 * q] = f.x;
    v[4 * q + 1] = f.y;
    v[4 * q + 2] = f.z;
    v[4 * q + 3] = f.w;
  }
  float2 w[RL + 1];
#pragma unroll
  for (int i = 0; i <= RL; ++i) w[i] = make_float2(w1[i], w1[i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int t = -RL; t <= RL; ++t) {
      const int a = RL4 + 2 * i + t;  // index of out[c0 + 2i] + t in v
      acc[i] = ffma2(w[t < 0 ? -t : t], make_float2(v[a], v[a + 1]), acc[i]);
    }
  }
}

// Border/edge chunks: the window leaves the computed vb columns [c_lo, chi] or
// the frame.  Column indices are clamped to the frame (replicate border, scipy
// mode="nearest") and uncomputed columns read as the exact zero they are.
// Scalar FMAs, each loaded value consumed at once (no window in registers).
template <int RL>
__device__ __forceinline__ void hlevel_edge(const float* __restrict__ w1, const float* __restrict__ row0,
                                            int c0, int W, int c_lo, int chi, float2 acc[8]) {
  float s[16];
#pragma unroll
  for (int o = 0; o < 16; ++o) s[o] = 0.f;
#pragma unroll
  for (int j = 0; j < 16 + 2 * RL; ++j) {
    const int c = min(max(c0 - RL + j, 0), W - 1);
    const float v = (c >= c_lo && c <= chi) ? row0[c] : 0.f;
#pragma unroll
    for (int o = 0; o < 16; ++o) {
      const int t = j - RL - o;
      if (t >= -RL && t <= RL) s[o] = fmaf(w1[t < 0 ? -t : t], v, s[o]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i].x += s[2 * i];
    acc[i].y += s[2 * i + 1];
  }
}

#define TAC4_RADIUS_CASES(X) \
  X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

// ---- conversion of one input slot ----------------------------------------------
// Depth -> indentation in place (REF/tactile.py:193-197) for the RB rows of
// block q, folding the contact partials of REF/marker.py:109-121 (own rows and
// columns only) and the slot's non-zero column extent.
struct ConvMap {
  int cg, ro, cstep;  // float4 column group, first row, row step
  bool active;
  bool all_own;       // all four columns of the group are output columns of this strip
  bool cown[4];
};

__device__ __forceinline__ void conv_slot(const FrameParams& p, const Geo& g, const ConvMap& m,
                                          float* slot, int q, Red& red, float colsum[4],
                                          int* ext_lo, int* ext_hi) {
  bool nz = false;
  if (m.active) {
    for (int rr = m.ro; rr < RB; rr += m.cstep) {
      const int gr = q * RB + rr;
      float4* e = reinterpret_cast<float4*>(slot + rr * p.in_pitch) + m.cg;
      const float4 raw = *e;
      float v[4] = {raw.x, raw.y, raw.z, raw.w};
      const bool rown = gr >= 0 && gr < p.H;
      if (rown) {
        // non-finite inputs are counted, not raised (summary field 6)
        const bool bad = !(fabsf(v[0]) < INFINITY) || !(fabsf(v[1]) < INFINITY) ||
                         !(fabsf(v[2]) < INFINITY) || !(fabsf(v[3]) < INFINITY);
        if (bad) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (m.cown[k] && !(fabsf(v[k]) < INFINITY)) red.nf += 1.f;
        }
      }
      if (p.input_depth) {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = clampf((p.rest - v[k]) + p.rest_lo, 0.f, p.rest);
        *e = make_float4(v[0], v[1], v[2], v[3]);
      }
      nz |= (v[0] != 0.f) | (v[1] != 0.f) | (v[2] != 0.f) | (v[3] != 0.f);
      if (rown) {
        float rowsum = 0.f;
        if (m.all_own) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            red.mx = fmaxf(red.mx, v[k]);
            const bool in = v[k] > p.threshold;
            const float w = in ? v[k] : 0.f;
            red.cnt += in ? 1.f : 0.f;
            colsum[k] += w;
            rowsum += w;
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (!m.cown[k]) continue;
            red.mx = fmaxf(red.mx, v[k]);
            const bool in = v[k] > p.threshold;
            const float w = in ? v[k] : 0.f;
            red.cnt += in ? 1.f : 0.f;
            colsum[k] += w;
            rowsum += w;
          }
        }
        red.sw += (double)rowsum;
        red.swy = fma((double)rowsum, (double)gr + 0.5 - (double)p.half_h, red.swy);
      }
    }
  }
  // slot extent: one redux per warp, one shared atomic per warp
  const int c = g.lx0 + 4 * m.cg;
  const int lo = __reduce_min_sync(0xffffffffu, nz ? c : INT_MAX);
  const int hi = __reduce_max_sync(0xffffffffu, nz ? c + 3 : INT_MIN);
  if ((threadIdx.x & 31) == 0 && lo != INT_MAX) {
    atomicMin(ext_lo, lo);
    atomicMax(ext_hi, hi);
  }
}

// ---- shading ------------------------------------------------------------------
// One pixel, any position (border rules of np.gradient, REF/optical.py:160).
__device__ __forceinline__ void shade_px_slow(const FrameParams& p, const Geo& g, const float* bb,
                                              int y, int x, uint8_t* out, long long env) {
  const float* rc = bb + ring4(y) * p.b_pitch - g.bbase;
  const float* rm = bb + ring4(y - 1) * p.b_pitch - g.bbase;
  const float* rp = bb + ring4(y + 1) * p.b_pitch - g.bbase;
  const int xl = x > 0 ? x - 1 : x, xr = x < p.W - 1 ? x + 1 : x;
  const float gx = (rc[xr] - rc[xl]) * ((xr - xl == 2) ? p.inv_2p : p.inv_p);
  const float yb = (y < p.H - 1) ? rp[x] : rc[x];
  const float yt = (y > 0) ? rm[x] : rc[x];
  const float gy = (yb - yt) * ((y > 0 && y < p.H - 1) ? p.inv_2p : p.inv_p);
  const float* bgp = p.bg + ((long long)y * p.W + x) * 3;
  float r = __ldg(bgp), gg = __ldg(bgp + 1), b = __ldg(bgp + 2);
  shade_one(p, gx, gy, r, gg, b);
  if (p.shadow) {
    const float sf = __ldg(p.shadow + env * (long long)p.H * p.W + (long long)y * p.W + x);
    r = clampf(r, 0.f, 255.f) * sf;
    gg = clampf(gg, 0.f, 255.f) * sf;
    b = clampf(b, 0.f, 255.f) * sf;
  }
  uint8_t* d = out + ((long long)y * p.W + x) * 3;
  d[0] = (uint8_t)u8sat(r);
  d[1] = (uint8_t)u8sat(gg);
  d[2] = (uint8_t)u8sat(b);
}

// 16 pixels [xs, xs + 16) of row y, all interior to the 16-B aligned fast path:
// float4 ring reads, 4 x LDG.128 LUT gathers per pixel issued two pixels at a
// time, 12 x LDG.128 background, 3 x STG.128 RGB.
__device__ __forceinline__ void shade16(const FrameParams& p, const Geo& g, const float* bb, int y,
                                        int xs, uint8_t* out, long long env) {
  const float* rc = bb + ring4(y) * p.b_pitch + (xs - g.bbase);
  const float* rm = bb + ring4(y - 1) * p.b_pitch + (xs - g.bbase);
  const float* rp = bb + ring4(y + 1) * p.b_pitch + (xs - g.bbase);
  const bool top = (y == 0), bot = (y == p.H - 1);
  const bool lft = (xs == 0), rgt = (xs + 16 == p.W);
  const float sy = (top || bot) ? p.inv_p : p.inv_2p;
  const float* bgp = p.bg + ((long long)y * p.W + xs) * 3;
  const float* shp = p.shadow ? p.shadow + env * (long long)p.H * p.W + (long long)y * p.W + xs : nullptr;
  uint32_t word[12];
  float cprev = rc[-1];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 cc = *reinterpret_cast<const float4*>(rc + 4 * q);
    const float4 mm = *reinterpret_cast<const float4*>(rm + 4 * q);
    const float4 nn = *reinterpret_cast<const float4*>(rp + 4 * q);
    const float cnext = rc[4 * q + 4];
    const float c[6] = {cprev, cc.x, cc.y, cc.z, cc.w, cnext};
    const float m[4] = {mm.x, mm.y, mm.z, mm.w};
    const float n[4] = {nn.x, nn.y, nn.z, nn.w};
    cprev = cc.w;
    float gxs[4], gys[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool l0 = lft && q == 0 && k == 0;
      const bool r0 = rgt && q == 3 && k == 3;
      const float xr = r0 ? c[k + 1] : c[k + 2];
      const float xl = l0 ? c[k + 1] : c[k];
      gxs[k] = (xr - xl) * ((l0 || r0) ? p.inv_p : p.inv_2p);
      const float yb = bot ? c[k + 1] : n[k];
      const float yt = top ? c[k + 1] : m[k];
      gys[k] = (yb - yt) * sy;
    }
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(bgp) + 3 * q);
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(bgp) + 3 * q + 1);
    const float4 b2 = __ldg(reinterpret_cast<const float4*>(bgp) + 3 * q + 2);
    const float bgv[12] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w, b2.x, b2.y, b2.z, b2.w};
    float sf[4] = {1.f, 1.f, 1.f, 1.f};
    if (shp) {
      const float4 f4 = __ldg(reinterpret_cast<const float4*>(shp) + q);
      sf[0] = f4.x; sf[1] = f4.y; sf[2] = f4.z; sf[3] = f4.w;
    }
    uint32_t qb[12];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const Px p0 = bin_px(p, gxs[2 * h], gys[2 * h]);
      const Px p1 = bin_px(p, gxs[2 * h + 1], gys[2 * h + 1]);
      const float4 a0 = __ldg(p0.lut), c0 = __ldg(p0.lut + 1), d0 = __ldg(p0.lut + 2), e0 = __ldg(p0.lut + 3);
      const float4 a1 = __ldg(p1.lut), c1 = __ldg(p1.lut + 1), d1 = __ldg(p1.lut + 2), e1 = __ldg(p1.lut + 3);
      float r = bgv[6 * h], gg = bgv[6 * h + 1], b = bgv[6 * h + 2];
      add_lut(a0, c0, d0, e0, p0.nx, p0.ny, r, gg, b);
      if (shp) {  // clip, then the multiplicative shadow (REF/optical.py:246, :299)
        r = clampf(r, 0.f, 255.f) * sf[2 * h];
        gg = clampf(gg, 0.f, 255.f) * sf[2 * h];
        b = clampf(b, 0.f, 255.f) * sf[2 * h];
      }
      qb[6 * h] = u8sat(r);
      qb[6 * h + 1] = u8sat(gg);
      qb[6 * h + 2] = u8sat(b);
      r = bgv[6 * h + 3];
      gg = bgv[6 * h + 4];
      b = bgv[6 * h + 5];
      add_lut(a1, c1, d1, e1, p1.nx, p1.ny, r, gg, b);
      if (shp) {
        r = clampf(r, 0.f, 255.f) * sf[2 * h + 1];
        gg = clampf(gg, 0.f, 255.f) * sf[2 * h + 1];
        b = clampf(b, 0.f, 255.f) * sf[2 * h + 1];
      }
      qb[6 * h + 3] = u8sat(r);
      qb[6 * h + 4] = u8sat(gg);
      qb[6 * h + 5] = u8sat(b);
    }
    word[3 * q] = qb[0] | (qb[1] << 8) | (qb[2] << 16) | (qb[3] << 24);
    word[3 * q + 1] = qb[4] | (qb[5] << 8) | (qb[6] << 16) | (qb[7] << 24);
    word[3 * q + 2] = qb[8] | (qb[9] << 8) | (qb[10] << 16) | (qb[11] << 24);
  }
  uint4* d = reinterpret_cast<uint4*>(out + ((long long)y * p.W + xs) * 3);
  d[0] = make_uint4(word[0], word[1], word[2], word[3]);
  d[1] = make_uint4(word[4], word[5], word[6], word[7]);
  d[2] = make_uint4(word[8], word[9], word[10], word[11]);
}

}  // namespace

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads + kShade4, 1)
    frame4_kernel(const __grid_constant__ FrameParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Geo g = make_geo(p, kModeFused);
  const int R = p.R;
  const long long HW = (long long)p.H * p.W;
  const int tid = threadIdx.x;
  const int nb = (p.H + RB - 1) / RB;

  float* inb = reinterpret_cast<float*>(smem_raw);                    // kIn4 slots x RB rows
  float* vb = inb + kIn4 * RB * p.in_pitch;                           // n_levels x RB rows
  float* bb = vb + p.n_levels * RB * p.v_pitch;                       // kRing4 rows
  double* s_red = reinterpret_cast<double*>(bb + kRing4 * p.b_pitch);  // 20 warps x 8
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_red + 2 * (kThreads / 32) * 8);  // 1 mbarrier
  int* s_int = reinterpret_cast<int*>(bar + 2);
  __shared__ S4 st;
  __shared__ double s_dbl[8];
  __shared__ int s_flag;

  // diagnostics: per-block clock64 stamps (tac_set_profile_buffer)
  long long* prof = (p.prof != nullptr && g.env < p.prof_envs && g.strip == 0)
                        ? p.prof + g.env * (long long)nb * 8 : nullptr;
#define STAMP(b, k) \
  if (prof) prof[(b) * 8 + (k)] = clock64();
  const float* src = p.in + g.env * HW;
  const int LW = g.lx1 - g.lx0;
  const unsigned row_bytes = (unsigned)LW * 4u;
  const int R4 = (R + 3) & ~3;
  const int vbase = g.bx0 - R4;  // global column of vb column 0 (16-B aligned rows)

  // block q's RB rows (clamped) -> its slot, completing on mbarrier `mb` (thread 0)
  auto issue_block = [&](int q, uint64_t* mb) {
    float* slot = inb + slot_of(q) * RB * p.in_pitch;
    for (int i = 0; i < RB; ++i) {
      const int cr = min(max(q * RB + i, 0), p.H - 1);
      bulk_g2s(slot + i * p.in_pitch, src + (long long)cr * p.W + g.lx0, row_bytes, mb);
    }
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kIn4) {
    st.ext_lo[tid] = INT_MAX;
    st.ext_hi[tid] = INT_MIN;
  }
  __syncthreads();

  Red red = red_zero();
  float colsum[4] = {0.f, 0.f, 0.f, 0.f};
  ConvMap cm;
  {
    const int ng4 = LW >> 2;
    cm.cg = tid % ng4;
    cm.ro = tid / ng4;
    cm.cstep = kThreads / ng4;
    cm.active = tid < kThreads && cm.ro < cm.cstep;
    cm.all_own = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int gx = g.lx0 + 4 * cm.cg + k;
      cm.cown[k] = gx >= g.x0 && gx < g.x1;
      cm.all_own &= cm.cown[k];
    }
  }

  if (tid < kThreads) {
    // ======================= blur group ========================================
    if (tid == 0) {
      const int nq = min(nb, 1) + 2;  // blocks -1, 0, 1 (block nb is all clamped rows)
      mbar_expect_tx(bar, row_bytes * RB * (unsigned)nq);
      for (int q = -1; q < nq - 1; ++q) issue_block(q, bar);
    }
    mbar_wait(bar, 0);
    for (int q = -1; q <= min(1, nb); ++q)
      conv_slot(p, g, cm, inb + slot_of(q) * RB * p.in_pitch, q, red, colsum, &st.ext_lo[slot_of(q)],
                &st.ext_hi[slot_of(q)]);
    fence_proxy_async();
    bsync4();

    int prev_ha = INT_MAX, prev_hb = INT_MIN;  // H range of block b-1
    for (int b = 0; b < nb; ++b) {
      const int r0 = b * RB;
      const bool last = (b == nb - 1);
      if (tid == 0) STAMP(b, 0);
      const int sP = slot_of(b - 1), sC = slot_of(b), sN = slot_of(b + 1);
      const int ea = min(min(st.ext_lo[sP], st.ext_lo[sC]), st.ext_lo[sN]);
      const int eb = max(max(st.ext_hi[sP], st.ext_hi[sC]), st.ext_hi[sN]);
      const bool any = ea <= eb;
      // H output range, widened to whole 16-column chunks: every column the H pass
      // stores is computed from valid (computed or exactly-zero) vb columns
      int ha = INT_MAX, hb = INT_MIN, k_lo = 0, k_hi = -1;
      if (any) {
        const int a = max(ea - R, g.bx0), z = min(eb + R, g.bx1 - 1);
        if (a <= z) {
          k_lo = (a - g.bx0) >> 4;
          k_hi = (z - g.bx0) >> 4;
          ha = g.bx0 + 16 * k_lo;
          hb = min(g.bx0 + 16 * k_hi + 15, g.bx1 - 1);
        }
      }
      // ---- V: all levels, computed columns [c_lo, chi] -----------------------------
      int c_lo = 0, chi = -1;
      if (ha <= hb) {
        const float* sp = inb + sP * RB * p.in_pitch - g.lx0;
        const float* sc = inb + sC * RB * p.in_pitch - g.lx0;
        const float* sn = inb + sN * RB * p.in_pitch - g.lx0;
        const int ca0 = max(ea, max(ha - R, 0));
        const int cb0 = min(eb, min(hb + R, p.W - 1));
        c_lo = ca0 & ~1;
        const int np = (cb0 - c_lo) / 2 + 1;  // column pairs
        chi = min(c_lo + 2 * np - 1, p.W - 1);
        // levels with RL > 0, one 2*np-item stripe each
        int nlev = 0;
        for (int l = 0; l < p.n_levels; ++l) nlev += p.radius[l] > 0;
        const int per = 2 * np;
        for (int it = tid; it < nlev * per; it += kThreads) {
          int li = it / per;
          const int rem = it - li * per;
          int l = 0;
          for (; l < p.n_levels; ++l)
            if (p.radius[l] > 0 && li-- == 0) break;
          const int hf = rem >= np ? 1 : 0;
          const int c = c_lo + 2 * (rem - hf * np);
          float* dst = vb + l * RB * p.v_pitch + 8 * hf * p.v_pitch + (c - vbase);
          const bool st_y = c + 1 <= p.W - 1;
          switch (p.radius[l]) {
#define X(r)                                                                          \
  case r:                                                                             \
    vitem<r>(p.wv[l], sp, sc, sn, p.in_pitch, hf, c, dst, p.v_pitch, st_y);           \
    break;
            TAC4_RADIUS_CASES(X)
#undef X
            default:
              break;
          }
        }
      }
      fence_proxy_async();
      bsync4();
      if (tid == 0) STAMP(b, 1);
      // ---- refill: block b+2 into the slot of block b-1 (lands during H) -----------
      if (tid == 0 && b + 2 <= nb) {
        const int s2 = slot_of(b + 2);
        st.ext_lo[s2] = INT_MAX;
        st.ext_hi[s2] = INT_MIN;
        mbar_expect_tx(bar, row_bytes * RB);
        issue_block(b + 2, bar);
      }
      if (b >= kSl4) bar_sync(kB4Empty + b % kSl4, kThreads + kShade4);
      if (tid == 0) STAMP(b, 2);
      // ---- H: all levels summed, one row x 16 columns per item --------------------
      {
        float* ring = bb + ring4(r0) * p.b_pitch;  // slot rows r0 .. r0 + RB - 1
        const int EW = g.bx1 - g.bx0;
        const int nch = (EW + 15) >> 4;
        const int nk = k_hi - k_lo + 1;
        for (int it = tid; it < RB * nk; it += kThreads) {
          const int row = it & (RB - 1);
          const int k = k_lo + (it >> 4);
          const int c0 = g.bx0 + 16 * k;
          const bool fast = c0 - R4 >= c_lo && c0 + 15 + R4 <= chi;
          float2 acc[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
          for (int l = 0; l < p.n_levels; ++l) {
            const int RL = p.radius[l];
            if (RL == 0) {
              const float w = p.wh[l][0];
              const float* in = inb + sC * RB * p.in_pitch + row * p.in_pitch + (c0 - g.lx0);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int cc = c0 + 2 * i;
                const float a = cc < g.bx1 ? in[2 * i] : 0.f;
                const float bq = cc + 1 < g.bx1 ? in[2 * i + 1] : 0.f;
                acc[i] = ffma2(make_float2(w, w), make_float2(a, bq), acc[i]);
              }
              continue;
            }
            const float* vrow = vb + l * RB * p.v_pitch + row * p.v_pitch;
            switch (RL) {
#define X(r)                                                                              \
  case r:                                                                                 \
    if (fast)                                                                             \
      hlevel<r>(p.wh[l], vrow + (c0 - ((r + 3) & ~3) - vbase), acc);                      \
    else                                                                                  \
      hlevel_edge<r>(p.wh[l], vrow - vbase, c0, p.W, c_lo, chi, acc);                     \
    break;
              TAC4_RADIUS_CASES(X)
#undef X
              default:
                break;
            }
          }
          float* d = ring + row * p.b_pitch + (c0 - g.bbase);
          if (c0 + 16 <= g.bx1) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<float4*>(d)[i] =
                  make_float4(acc[2 * i].x, acc[2 * i].y, acc[2 * i + 1].x, acc[2 * i + 1].y);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (c0 + 2 * i < g.bx1) d[2 * i] = acc[i].x;
              if (c0 + 2 * i + 1 < g.bx1) d[2 * i + 1] = acc[i].y;
            }
          }
        }
        // exact zeros elsewhere in the slot (16-column chunks outside [k_lo, k_hi])
        const int nz = nch - nk;
        for (int it = tid; it < RB * nz * 4; it += kThreads) {
          const int row = it / (nz * 4);
          const int o = it - row * nz * 4;
          const int kk = o >> 2;
          const int k = kk < k_lo ? kk : kk + nk;
          const int c = g.bx0 + 16 * k + 4 * (o & 3);
          if (c < g.bx1) {
            float* d = ring + row * p.b_pitch + (c - g.bbase);
            if (c + 4 <= g.bx1)
              *reinterpret_cast<float4*>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
            else
              for (int i = 0; i < g.bx1 - c; ++i) d[i] = 0.f;
          }
        }
      }
      // ---- convert block b+2 (copied while H ran) ----------------------------------
      if (tid == 0) STAMP(b, 3);
      if (b + 2 <= nb) {
        const int q = b + 2;
        mbar_wait(bar, (unsigned)((b + 1) & 1));  // use b+1 of the mbarrier (prologue = 0)
        conv_slot(p, g, cm, inb + slot_of(q) * RB * p.in_pitch, q, red, colsum, &st.ext_lo[slot_of(q)],
                  &st.ext_hi[slot_of(q)]);
        fence_proxy_async();
      }
      bsync4();
      if (tid == 0) STAMP(b, 4);
      // ---- outputs ----------------------------------------------------------------
      if (p.blurred != nullptr) {
        float* dst = p.blurred + g.env * HW;
        const int OW = g.x1 - g.x0;
        const int nr = min(RB, p.H - r0);
        for (int it = tid; it < nr * OW; it += kThreads) {
          const int rr = it / OW;
          const int x = g.x0 + (it - rr * OW);
          dst[(long long)(r0 + rr) * p.W + x] = bb[ring4(r0 + rr) * p.b_pitch + (x - g.bbase)];
        }
      }
      if (tid == 0) {
        int sa = min(prev_ha, ha), sb = max(prev_hb, hb);
        if (sa <= sb) {
          sa = max(sa - 1, g.x0);
          sb = min(sb + 1, g.x1 - 1);
        }
        if (p.shadow != nullptr) {  // shadows reach flat regions
          sa = g.x0;
          sb = g.x1 - 1;
        }
        st.sh_lo[b % kSl4] = sa;
        st.sh_hi[b % kSl4] = sb;
      }
      prev_ha = ha;
      prev_hb = hb;
      (void)last;
      bar_arrive(kB4Full + b % kSl4, kThreads + kShade4);
    }
  } else {
    // ======================= shade group =======================================
    const int gtid = tid - kThreads;
    uint8_t* out = p.rgb + g.env * HW * 3;
    const int OW = g.x1 - g.x0;
    const int nch = (OW + 15) >> 4;
    const bool fast_ok = (p.W % 16) == 0;  // 16-B aligned RGB rows and background rows
    for (int b = 0; b < nb; ++b) {
      const int r0 = b * RB;
      const bool last = (b == nb - 1);
      bar_sync(kB4Full + b % kSl4, kThreads + kShade4);
      if (gtid == 0) STAMP(b, 5);
      const int y_lo = max(r0 - 1, 0);
      const int y_hi = last ? p.H : r0 + RB - 1;
      const int sa = st.sh_lo[b % kSl4], sb = st.sh_hi[b % kSl4];
      for (int it = gtid; it < (y_hi - y_lo) * nch; it += kShade4) {
        const int yy = it / nch;
        const int y = y_lo + yy;
        const int k = it - yy * nch;
        const int xs = g.x0 + 16 * k;
        const int xe = min(xs + 16, g.x1);
        const bool shade = sa <= sb && xs <= sb && xe - 1 >= sa;
        if (!shade) {
          const long long o = ((long long)y * p.W + xs) * 3;
          if (fast_ok && xe - xs == 16) {
            const uint4* s4 = reinterpret_cast<const uint4*>(p.bg_u8 + o);
            uint4* d4 = reinterpret_cast<uint4*>(out + o);
            d4[0] = __ldg(s4);
            d4[1] = __ldg(s4 + 1);
            d4[2] = __ldg(s4 + 2);
          } else {
            for (int i = 0; i < 3 * (xe - xs); ++i) out[o + i] = p.bg_u8[o + i];
          }
        } else if (fast_ok && xe - xs == 16) {
          shade16(p, g, bb, y, xs, out, g.env);
        } else {
          for (int x = xs; x < xe; ++x) shade_px_slow(p, g, bb, y, x, out, g.env);
        }
      }
      if (gtid == 0) STAMP(b, 6);
      // block b-1's slot (= block b+kSl4-1's) is no longer read
      if (b >= 1 && b + kSl4 - 1 < nb) bar_arrive(kB4Empty + (b + kSl4 - 1) % kSl4, kThreads + kShade4);
    }
  }

  // ---- reduction + env epilogue -------------------------------------------------
  if (p.finalize == 0) return;
  if (tid < kThreads) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      red.swx = fma((double)colsum[k], (double)(g.lx0 + 4 * cm.cg + k) + 0.5 - (double)p.half_w, red.swx);
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

size_t frame4_smem_bytes(const FrameParams& p) {
  size_t bytes = sizeof(float) * ((size_t)kIn4 * RB * p.in_pitch + (size_t)p.n_levels * RB * p.v_pitch +
                                  (size_t)kRing4 * p.b_pitch);
  bytes += sizeof(double) * 2 * (kThreads / 32) * 8;
  bytes += 2 * sizeof(uint64_t);
  bytes += 2 * sizeof(int) * (size_t)p.mg.rows * p.mg.cols;
  return (bytes + 127) & ~size_t(127);
}

bool frame4_eligible(const FrameParams& p) {
  if (p.R < 1 || p.R > RB) return false;      // window = slots b-1..b+1
  if (p.in_pitch % 4 != 0) return false;
  for (int l = 0; l < p.n_levels; ++l)
    if (p.radius[l] > 16) return false;
  return frame4_smem_bytes(p) <= 227 * 1024;
}

cudaError_t launch_frame4(const FrameParams& p, cudaStream_t s) {
  const size_t smem = frame4_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(frame4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = p.n_env * (long long)p.strips;
  if (blocks == 0) return cudaSuccess;
  frame4_kernel<<<(unsigned)blocks, kThreads + kShade4, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace tac
