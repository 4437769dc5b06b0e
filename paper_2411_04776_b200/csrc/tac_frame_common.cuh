// Device helpers shared by the frame kernels (tac_frame.cu: strip-streaming v3,
// tac_frame5.cu: band-tiled two-kernel path): TMA/mbarrier and named-barrier wrappers, strip
// geometry, paired FMA, the shading arithmetic (bins, LUT basis, uint8 rule),
// and the deterministic contact reductions + per-env finalisation.
#pragma once

#include "tac_internal.cuh"
#include "tac_marker.cuh"

namespace tac {

namespace {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kHalfPi = 1.57079632679489661923f;

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
  return fminf(fmaxf(v, lo), hi);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- TMA (bulk async copy) + mbarrier helpers ------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool bar_or(int id, int n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n .reg .pred pi, po;\n setp.ne.u32 pi, %1, 0;\n bar.red.or.pred po, %2, %3, pi;\n"
      " selp.u32 %0, 1, 0, po;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// ---- per-CTA geometry -------------------------------------------------------
struct Geo {
  long long env;
  int strip;
  int x0, x1;    // output columns
  int bx0, bx1;  // blurred columns (output + gradient ring)
  int vx0, vx1;  // in-frame vertical-pass columns
  int lx0, lx1;  // loaded columns (16-B aligned for TMA)
  int bbase;     // global column of blurred-buffer column 0 (4-aligned)
  int nblocks;
};

__device__ __forceinline__ Geo make_geo(const FrameParams& p, int mode) {
  Geo g;
  g.env = blockIdx.x / p.strips;
  g.strip = (int)(blockIdx.x - g.env * p.strips);
  g.x0 = g.strip * p.strip_w;
  g.x1 = min(g.x0 + p.strip_w, p.W);
  const int ring = mode == kModeFused ? 1 : 0;
  g.bx0 = max(g.x0 - ring, 0) & ~3;  // 4-aligned: float4 access to the blurred ring
  g.bx1 = min(g.x1 + ring, p.W);
  const int R = mode == kModeContact ? 0 : p.R;
  g.vx0 = max(g.bx0 - R, 0);
  g.vx1 = min(g.bx1 + R, p.W);
  if (p.use_tma) {
    g.lx0 = g.vx0 & ~3;
    g.lx1 = min((g.vx1 + 3) & ~3, p.W);
  } else {
    g.lx0 = g.vx0;
    g.lx1 = g.vx1;
  }
  g.bbase = g.bx0 & ~3;
  g.nblocks = (p.H + RB - 1) / RB;
  return g;
}

// ---- separable passes ---------------------------------------------------------
// Paired fp32 FMA (FFMA2 on sm_100a): two independent lanes of work per issue.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// Paired fp32 (a - b) + c, each step rounded (FADD2 x2 on sm_100a).
__device__ __forceinline__ float2 fsubadd2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n sub.rn.f32x2 rd, ra, rb;\n add.rn.f32x2 rd, rd, rc;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// ---- shading ------------------------------------------------------------------
// atan(a) for a in [0, 1]: odd minimax polynomial, |err| ~ 1e-7 rad in fp32.
__device__ __forceinline__ float atan01(float a) {
  const float s = a * a;
  float q = 0.0024567204527556896f;
  q = fmaf(q, s, -0.01440134271979332f);
  q = fmaf(q, s, 0.039781197905540466f);
  q = fmaf(q, s, -0.07234855741262436f);
  q = fmaf(q, s, 0.10498945415019989f);
  q = fmaf(q, s, -0.14161229133605957f);
  q = fmaf(q, s, 0.19985906779766083f);
  q = fmaf(q, s, -0.33332598209381104f);
  q = fmaf(q, s, 0.9999998807907104f);
  return q * a;
}

// atan2(y, x) for (x, y) != 0.
__device__ __forceinline__ float atan2_nz(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  float r = atan01(__fdividef(mn, mx));
  r = (ay > ax) ? kHalfPi - r : r;
  r = (x < 0.f) ? kPi - r : r;
  return (y < 0.f) ? -r : r;
}

__device__ __forceinline__ uint32_t u8sat(float v) {
  uint32_t r;
  asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

// Bins + normal of one pixel.  Branch-free: a zero gradient gives bin 0 and
// a zero basis, so its shading term is exactly 0 (the LUT is finite).
struct Px {
  const float4* lut;
  float nx, ny;
  int mb, db;  // magnitude / direction bin
};

__device__ __forceinline__ Px bin_px(const FrameParams& p, float gx, float gy) {
  const float g2 = fmaf(gx, gx, gy * gy);
  Px o;
  const float gm = g2 * rsqrtf(g2);        // NaN for g2 == 0 -> bin 0
  const float inv = rsqrtf(1.f + g2);
  o.nx = -gx * inv;
  o.ny = -gy * inv;
  const int mb = min((int)(gm * p.mag_scale), p.mag_bins - 1);
  int db = (int)((atan2_nz(gy, gx) + kPi) * p.dir_scale);  // NaN for (0,0) -> 0
  db = db >= p.dir_bins ? db - p.dir_bins : db;
  db = max(db, 0);
  o.mb = max(mb, 0);
  o.db = db;
  o.lut = p.lut + (o.mb * p.dir_bins + db) * 4;  // < 2^31 / 4 bins (host-checked)
  return o;
}

// Delta_c = c1 nx + c2 ny + c3 nx^2 + c4 nx ny + c5 ny^2 (REF/optical.py:82-88, :244)
// layout: a = R c1..c4 | c = R c5, G c1..c3 | d = G c4, c5, B c1, c2 | e = B c3..c5, pad
__device__ __forceinline__ void add_lut(const float4 a, const float4 c, const float4 d, const float4 e,
                                        float nx, float ny, float& r, float& g, float& b) {
  const float nxx = nx * nx, nxy = nx * ny, nyy = ny * ny;
  r += a.x * nx + a.y * ny + a.z * nxx + a.w * nxy + c.x * nyy;
  g += c.y * nx + c.z * ny + c.w * nxx + d.x * nxy + d.y * nyy;
  b += d.z * nx + d.w * ny + e.x * nxx + e.y * nxy + e.z * nyy;
}

// Read-only 16-B loads with L1 allocation hints: LUT gathers are kept in L1
// (evict_last), streamed operands (background, blurred rows) do not displace
// them (no_allocate).
__device__ __forceinline__ float4 ldg_keep(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}

// Four quantised channel bytes -> one little-endian word (3 PRMT).
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x3340), __byte_perm(c, d, 0x3340), 0x5410);
}

// Add the binned-LUT shading of gradient (gx, gy) to background (r, g, b).
__device__ __forceinline__ void shade_one(const FrameParams& p, float gx, float gy, float& r,
                                          float& g, float& b) {
  const Px q = bin_px(p, gx, gy);
  add_lut(__ldg(q.lut), __ldg(q.lut + 1), __ldg(q.lut + 2), __ldg(q.lut + 3), q.nx, q.ny, r, g, b);
}

// ---- reductions / epilogue ------------------------------------------------------
// Contact partials.  The first moments are accumulated in fp64: every
// product w*xc of an fp32 weight and a half-integer pixel coordinate is exact
// in fp64, so symmetric contacts cancel exactly (a centred flat press gives a
// centroid of exactly 0, as the fp64 reference does) and the dot centres do
// not flip on the .5 ties of REF/marker.py:221-225.
struct Red {
  float cnt, mx, nf;
  double sw, swx, swy;
};

__device__ __forceinline__ Red red_zero() {
  Red r;
  r.cnt = r.mx = r.nf = 0.f;
  r.sw = r.swx = r.swy = 0.0;
  return r;
}

// Warp-level part of block_reduce (fixed shuffle tree); result in every lane.
__device__ __forceinline__ void warp_reduce(Red& v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.cnt += __shfl_xor_sync(0xffffffffu, v.cnt, o);
    v.mx = fmaxf(v.mx, __shfl_xor_sync(0xffffffffu, v.mx, o));
    v.nf += __shfl_xor_sync(0xffffffffu, v.nf, o);
    v.sw += __shfl_xor_sync(0xffffffffu, v.sw, o);
    v.swx += __shfl_xor_sync(0xffffffffu, v.swx, o);
    v.swy += __shfl_xor_sync(0xffffffffu, v.swy, o);
  }
}

// Fixed shuffle tree + fixed warp order: deterministic.  Result in the thread
// with linear id 0.  `tid` / `nthreads`: linear thread id and block size (for
// 2-D blocks); nthreads is a multiple of 32.
__device__ __forceinline__ void block_reduce(Red& v, double* s_red, int tid, int nthreads) {
  const int lane = tid & 31, wid = tid >> 5, nw = nthreads / 32;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.cnt += __shfl_xor_sync(0xffffffffu, v.cnt, o);
    v.mx = fmaxf(v.mx, __shfl_xor_sync(0xffffffffu, v.mx, o));
    v.nf += __shfl_xor_sync(0xffffffffu, v.nf, o);
    v.sw += __shfl_xor_sync(0xffffffffu, v.sw, o);
    v.swx += __shfl_xor_sync(0xffffffffu, v.swx, o);
    v.swy += __shfl_xor_sync(0xffffffffu, v.swy, o);
  }
  if (lane == 0) {
    double* q = s_red + wid * 8;
    q[0] = v.cnt;
    q[1] = v.sw;
    q[2] = v.swx;
    q[3] = v.swy;
    q[4] = v.mx;
    q[5] = v.nf;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < nw; ++w) {
      const double* q = s_red + w * 8;
      v.cnt += (float)q[0];
      v.sw += q[1];
      v.swx += q[2];
      v.swy += q[3];
      v.mx = fmaxf(v.mx, (float)q[4]);
      v.nf += (float)q[5];
    }
  }
}

__device__ __forceinline__ void block_reduce(Red& v, double* s_red) {
  block_reduce(v, s_red, threadIdx.x, blockDim.x);
}

// Thread 0: totals (fp64) -> contact outputs + load; the load lands in s_dbl.
__device__ void finalize_load(const FrameParams& p, long long env, double cnt, double sw, double swx,
                              double swy, float mx, double nf, double* s_dbl) {
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
    s[7] = p.saturated != nullptr ? (float)p.saturated[env] : 0.f;
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
  load_store(s_dbl, l);
}

}  // namespace

}  // namespace tac
