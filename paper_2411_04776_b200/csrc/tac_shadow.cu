// add_shadows (REF/optical.py:261-300) on the GPU: per pixel and light, march
// `steps` pixels toward the light over the elevation map and darken the pixel
// multiplicatively when some sample rises above the light ray (soft edge).
//
// The per-step offsets (di, dj) and ray costs s * pitch * lz / lateral are the
// reference's (Python half-to-even rounding of s*dy, s*dx), built once on the
// host; a CTA stages them in shared memory and every thread marches its own
// pixel, reading the elevation through L1 (the march of neighbouring pixels
// touches the same lines).  Borders replicate (REF/optical.py:253-258); warps
// whose whole march stays inside the frame skip the clamps.
#include "tac_internal.cuh"

namespace tac {

namespace {

constexpr int kShadowTX = 32, kShadowTY = 8;

__global__ void __launch_bounds__(kShadowTX * kShadowTY) shadow_kernel(
    const ShadowParams s, const float* __restrict__ in, int input_depth, float* __restrict__ factor,
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

}  // namespace

cudaError_t launch_shadow(const ShadowParams& s, const float* in, int input_depth, float* factor,
                          float* rgb, long long n_env, cudaStream_t st) {
  const long long tiles = (long long)((s.W + kShadowTX - 1) / kShadowTX) * ((s.H + kShadowTY - 1) / kShadowTY);
  const long long blocks = tiles * n_env;
  if (blocks == 0) return cudaSuccess;
  const size_t smem = (size_t)s.n_lights * s.steps * (sizeof(int2) + sizeof(float));
  shadow_kernel<<<(unsigned)blocks, dim3(kShadowTX, kShadowTY), smem, st>>>(s, in, input_depth, factor, rgb,
                                                                           n_env);
  return cudaGetLastError();
}

}  // namespace tac
