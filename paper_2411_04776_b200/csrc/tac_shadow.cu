// add_shadows (REF/optical.py:261-300) on the GPU: per pixel and light, march
// `steps` pixels toward the light over the elevation map and darken the pixel
// multiplicatively when some sample rises above the light ray (soft edge).
//
// The per-step offsets (di, dj) and ray costs s * pitch * lz / lateral are the
// reference's (Python half-to-even rounding of s*dy, s*dx), built once on the
// host.
//
// shadow_tiled_kernel (default): one CTA per 24 x 160 output tile of one env.
// Per light the tile's region shifted by every offset of that light (the
// tile plus a one-sided halo along the light direction) is staged in shared
// memory once, with the row/column index clamped = replicate border
// (REF/optical.py:253-258); then every thread marches 15 pixels (3 rows x 5
// columns 32 apart: conflict-free LDS) with the step's byte offset and cost
// as uniform operands: one LDS + FADD + half an FMNMX3 per tap and pixel.
// The 240 taps of a pixel are served by shared memory instead of L1.
//
// shadow_kernel (fallback when a region exceeds shared memory, e.g. very
// long marches): every thread marches its own pixel through L1.
#include <algorithm>

#include "tac_internal.cuh"

namespace tac {

namespace {

constexpr int kShadowTX = 32, kShadowTY = 8;

__global__ void __launch_bounds__(kShadowTX * kShadowTY) shadow_kernel(
    const __grid_constant__ ShadowParams s, const float* __restrict__ in, int input_depth, float* __restrict__ factor,
    float* __restrict__ rgb, long long n_env) {
  extern __shared__ __align__(16) unsigned char smem[];
  int2* s_off = reinterpret_cast<int2*>(smem);
  float* s_cost = reinterpret_cast<float*>(s_off + s.n_lights * s.steps);
  const int n = s.n_lights * s.steps;
  const int tid = threadIdx.y * kShadowTX + threadIdx.x;
  for (int k = tid; k < n; k += kShadowTX * kShadowTY) {
    s_off[k] = s.off[k];
    s_cost[k] = s.cost[k];
  }
  __syncthreads();

  const int tiles_x = (s.W + kShadowTX - 1) / kShadowTX;
  const int tiles_y = (s.H + kShadowTY - 1) / kShadowTY;
  const long long T = (long long)tiles_x * tiles_y;
  const long long env = blockIdx.x / T;
  const int t = (int)(blockIdx.x - env * T);
  const int ty = t / tiles_x, tx = t - ty * tiles_x;
  const int i = ty * kShadowTY + threadIdx.y;
  const int j = tx * kShadowTX + threadIdx.x;
  const bool valid = i < s.H && j < s.W;
  const int ic = min(i, s.H - 1), jc = min(j, s.W - 1);
  const long long HW = (long long)s.H * s.W;
  const float* e = in + env * HW;
  // elevation: -depth for a HeightMap; the indentation differs from it by a
  // constant where the depth is within [0, rest], which cancels in occ
  const float sg = input_depth ? -1.f : 1.f;
  const float e0 = sg * __ldg(e + (long long)ic * s.W + jc);
  const bool interior = __all_sync(0xffffffffu, ic + s.di_min >= 0 && ic + s.di_max < s.H &&
                                                    jc + s.dj_min >= 0 && jc + s.dj_max < s.W);
  float F = 1.f;
  for (int l = 0; l < s.n_lights; ++l) {
    const int2* off = s_off + l * s.steps;
    const float* cost = s_cost + l * s.steps;
    float occ = -INFINITY;
    if (interior) {
      const float* base = e + (long long)ic * s.W + jc;
#pragma unroll 8
      for (int st = 0; st < s.steps; ++st) {
        const int2 o = off[st];
        occ = fmaxf(occ, fmaf(sg, __ldg(base + o.x * s.W + o.y), -cost[st]));
      }
    } else {
#pragma unroll 4
      for (int st = 0; st < s.steps; ++st) {
        const int2 o = off[st];
        const int ii = min(max(ic + o.x, 0), s.H - 1);
        const int jj = min(max(jc + o.y, 0), s.W - 1);
        occ = fmaxf(occ, fmaf(sg, __ldg(e + (long long)ii * s.W + jj), -cost[st]));
      }
    }
    // occ = max_s (elev(p + o_s) - s * rise) - elev(p)
    const float w = fminf(fmaxf((occ - e0) * s.inv_softness, 0.f), 1.f);
    F *= 1.f - s.one_minus_factor * w;
  }
  if (!valid) return;
  const long long pix = env * HW + (long long)i * s.W + j;
  if (factor != nullptr) factor[pix] = F;
  if (rgb != nullptr) {
    float* px = rgb + pix * 3;
    px[0] *= F;
    px[1] *= F;
    px[2] *= F;
  }
}

constexpr int kTileThreads = 256;  // 8 warps x 3 rows; lanes x 5 columns

// Paired fp32 addition (FADD2 on sm_100a).
__device__ __forceinline__ float2 fadd2s(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

__global__ void __launch_bounds__(kTileThreads, 3) shadow_tiled_kernel(
    const __grid_constant__ ShadowParams s, const float* __restrict__ in, int input_depth,
    float* __restrict__ factor, float* __restrict__ rgb, long long n_env) {
  extern __shared__ __align__(16) float reg[];
  constexpr int RPW = kShadowTH / 8;   // rows per warp
  constexpr int CPL = kShadowTW / 32;  // columns per lane
  const int tiles_x = (s.W + kShadowTW - 1) / kShadowTW;
  const int tiles_y = (s.H + kShadowTH - 1) / kShadowTH;
  const long long T = (long long)tiles_x * tiles_y;
  const long long env = blockIdx.x / T;
  const int t = (int)(blockIdx.x - env * T);
  const int ty = t / tiles_x, tx = t - ty * tiles_x;
  const int ti0 = ty * kShadowTH, tj0 = tx * kShadowTW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long HW = (long long)s.H * s.W;
  const float* e = in + env * HW;
  // elevation: -depth for a HeightMap; the indentation differs from it by a
  // constant where the depth is within [0, rest], which cancels in occ.  The
  // region holds the raw input; the sign is applied to the max below.
  const float sg = input_depth ? -1.f : 1.f;
  float F[RPW][CPL];
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int q = 0; q < CPL; ++q) F[r][q] = 1.f;
  for (int l = 0; l < s.n_lights; ++l) {
    const int rh = s.l_rh[l], rw = s.l_rw[l];
    const int r0 = ti0 + s.l_di_min[l], c0 = tj0 + s.l_dj_min[l];  // c0, rw: multiples of 4
    if (l) __syncthreads();  // the previous light's region is no longer read
    // stage the region: rows by warp, 16-B groups by lane; row index clamped
    // and groups outside [0, W) filled with the edge value (replicate border)
    for (int rr = warp; rr < rh; rr += 8) {
      const float* src = e + (long long)min(max(r0 + rr, 0), s.H - 1) * s.W;
      float4* dst = reinterpret_cast<float4*>(reg + rr * rw);
      for (int g = lane; g < (rw >> 2); g += 32) {
        const int cc = c0 + 4 * g;
        float4 v;
        if (cc < 0) {
          const float x = __ldg(src);
          v = make_float4(x, x, x, x);
        } else if (cc >= s.W) {
          const float x = __ldg(src + s.W - 1);
          v = make_float4(x, x, x, x);
        } else {
          v = __ldg(reinterpret_cast<const float4*>(src + cc));
        }
        dst[g] = v;
      }
    }
    __syncthreads();
    // elev - c = sg (x - sg c): occ' = max_s (x - sg c) for sg = 1, min_s for
    // sg = -1, and sg occ' = max_s (elev(p + o_s) - s rise), bit for bit
    float occ[RPW][CPL];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int q = 0; q < CPL; ++q) occ[r][q] = INFINITY;
    const char* base = reinterpret_cast<const char*>(reg + (warp * RPW) * rw + lane);
    const int* offb = s.offb[l];
    const float* cost = s.costs[l];
    int st = 0;
    for (; st + 1 < s.steps; st += 2) {
      const char* b0 = base + offb[st];
      const char* b1 = base + offb[st + 1];
      TAC_CHECK(b0 >= reinterpret_cast<const char*>(reg) && b1 >= reinterpret_cast<const char*>(reg) &&
                b0 + ((RPW - 1) * rw + 32 * (CPL - 1) + 1) * (int)sizeof(float) <=
                    reinterpret_cast<const char*>(reg + rh * rw) &&
                b1 + ((RPW - 1) * rw + 32 * (CPL - 1) + 1) * (int)sizeof(float) <=
                    reinterpret_cast<const char*>(reg + rh * rw));
      const float2 cs = make_float2(-sg * cost[st], -sg * cost[st + 1]);  // a = x - sg c
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int o = (r * rw + 32 * q) * (int)sizeof(float);
          // two steps of one pixel: one FADD2, one FMNMX3
          const float2 a = fadd2s(make_float2(*reinterpret_cast<const float*>(b0 + o),
                                              *reinterpret_cast<const float*>(b1 + o)), cs);
          occ[r][q] = sg < 0.f ? fminf(occ[r][q], fminf(a.x, a.y)) : fmaxf(occ[r][q], fmaxf(a.x, a.y));
        }
    }
    if (st < s.steps) {
      const char* b0 = base + offb[st];
      const float c0s = -sg * cost[st];
#pragma unroll
      for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const float a = *reinterpret_cast<const float*>(b0 + (r * rw + 32 * q) * (int)sizeof(float)) + c0s;
          occ[r][q] = sg < 0.f ? fminf(occ[r][q], a) : fmaxf(occ[r][q], a);
        }
    }
    // weight = clip((max_s(elev(p + o_s) - s rise) - elev(p)) / softness, 0, 1)
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int i = min(ti0 + warp * RPW + r, s.H - 1), j = min(tj0 + lane + 32 * q, s.W - 1);
        const float e0 = __ldg(e + (long long)i * s.W + j);
        const float w = fminf(fmaxf(sg * (occ[r][q] - e0) * s.inv_softness, 0.f), 1.f);
        F[r][q] *= 1.f - s.one_minus_factor * w;
      }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int i = ti0 + warp * RPW + r, j = tj0 + lane + 32 * q;
      if (i >= s.H || j >= s.W) continue;
      const long long pix = env * HW + (long long)i * s.W + j;
      if (factor != nullptr) factor[pix] = F[r][q];
      if (rgb != nullptr) {
        float* px = rgb + pix * 3;
        px[0] *= F[r][q];
        px[1] *= F[r][q];
        px[2] *= F[r][q];
      }
    }
}

size_t shadow_region_bytes(const ShadowParams& s) {
  size_t b = 0;
  for (int l = 0; l < s.n_lights; ++l) b = std::max(b, (size_t)s.l_rh[l] * s.l_rw[l] * sizeof(float));
  return b;
}

}  // namespace

cudaError_t launch_shadow(const ShadowParams& s, const float* in, int input_depth, float* factor,
                          float* rgb, long long n_env, cudaStream_t st) {
  if (s.tiled) {
    const long long tt = (long long)((s.W + kShadowTW - 1) / kShadowTW) * ((s.H + kShadowTH - 1) / kShadowTH);
    const long long nb = tt * n_env;
    const size_t smem = shadow_region_bytes(s);
    cudaError_t e = cudaFuncSetAttribute(shadow_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess || nb == 0) return e;
    shadow_tiled_kernel<<<(unsigned)nb, kTileThreads, smem, st>>>(s, in, input_depth, factor, rgb, n_env);
    return cudaGetLastError();
  }
  const long long tiles = (long long)((s.W + kShadowTX - 1) / kShadowTX) * ((s.H + kShadowTY - 1) / kShadowTY);
  const long long blocks = tiles * n_env;
  if (blocks == 0) return cudaSuccess;
  const size_t smem = (size_t)s.n_lights * s.steps * (sizeof(int2) + sizeof(float));
  shadow_kernel<<<(unsigned)blocks, dim3(kShadowTX, kShadowTY), smem, st>>>(s, in, input_depth, factor, rgb,
                                                                           n_env);
  return cudaGetLastError();
}

}  // namespace tac
