// Stand-alone element-wise and per-env kernels behind the un-fused entry
// points (the mirrors of the individual reference functions).
#include "tac_internal.cuh"
#include "tac_marker.cuh"

namespace tac {

namespace {

// indentation_from, REF/tactile.py:193-197, 128-bit vectorised.
__global__ void __launch_bounds__(256) indentation_kernel(const float4* __restrict__ d,
                                                          float4* __restrict__ o, float rest, float rest_lo,
                                                          long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldg(d + i);
    v.x = fminf(fmaxf((rest - v.x) + rest_lo, 0.f), rest);
    v.y = fminf(fmaxf((rest - v.y) + rest_lo, 0.f), rest);
    v.z = fminf(fmaxf((rest - v.z) + rest_lo, 0.f), rest);
    v.w = fminf(fmaxf((rest - v.w) + rest_lo, 0.f), rest);
    o[i] = v;
  }
}

__global__ void indentation_tail(const float* __restrict__ d, float* __restrict__ o, float rest,
                                 float rest_lo, long long start, long long n) {
  const long long i = start + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) o[i] = fminf(fmaxf((rest - d[i]) + rest_lo, 0.f), rest);
}

// normals_from, REF/optical.py:159-163 (np.gradient semantics).
__global__ void __launch_bounds__(256) normals_kernel(const float* __restrict__ e,
                                                      float* __restrict__ nrm, int H, int W,
                                                      float inv_p, float inv_2p, long long total) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long HW = (long long)H * W;
  const long long env = i / HW;
  const int pix = (int)(i - env * HW);
  const int y = pix / W, x = pix - y * W;
  const float* b = e + env * HW;
  float gx, gy;
  if (x == 0)
    gx = (b[pix + 1] - b[pix]) * inv_p;
  else if (x == W - 1)
    gx = (b[pix] - b[pix - 1]) * inv_p;
  else
    gx = (b[pix + 1] - b[pix - 1]) * inv_2p;
  if (y == 0)
    gy = (b[pix + W] - b[pix]) * inv_p;
  else if (y == H - 1)
    gy = (b[pix] - b[pix - W]) * inv_p;
  else
    gy = (b[pix + W] - b[pix - W]) * inv_2p;
  const float inv = rsqrtf(fmaf(gx, gx, fmaf(gy, gy, 1.f)));
  float* n = nrm + i * 3;
  n[0] = -gx * inv;
  n[1] = -gy * inv;
  n[2] = inv;
}

__global__ void quantize_bg_kernel(const float* __restrict__ bg, uint8_t* __restrict__ q,
                                   long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) q[i] = (uint8_t)min(max(__float2int_rn(bg[i]), 0), 255);
}

// track_load, REF/marker.py:124-140, one thread per env.
__global__ void track_load_kernel(double* __restrict__ state, const double* __restrict__ delta,
                                  const double* __restrict__ contact, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Load prev = load_from(state + i * 8);
  const Load c = load_from(contact + i * 8);
  const double* d = delta + i * 3;
  load_store(state + i * 8, track_load(prev, d[0], d[1], d[2], c));
}

// marker_displacements (+ optional splat), one CTA per env.
__global__ void __launch_bounds__(128) markers_kernel(const MarkerGeom g,
                                                      const double* __restrict__ loads,
                                                      float* __restrict__ disp,
                                                      const float* __restrict__ disp_in,
                                                      uint8_t* __restrict__ rgb) {
  extern __shared__ int s_cr[];
  const long long env = blockIdx.x;
  const int nm = g.rows * g.cols;
  const Load l = loads ? load_from(loads + env * 8) : load_zero();
  markers_block(g, l, disp ? disp + env * nm * 2 : nullptr, rgb ? rgb + env * (long long)g.H * g.W * 3 : nullptr,
                disp_in ? disp_in + env * nm * 2 : nullptr, s_cr, s_cr + nm);
}

}  // namespace

cudaError_t launch_indentation(const float* depth, float* ind, float rest, float rest_lo, long long n,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  long long n4 = 0;
  if (((reinterpret_cast<uintptr_t>(depth) | reinterpret_cast<uintptr_t>(ind)) & 15) == 0) {
    n4 = n / 4;
    if (n4 > 0) {
      const long long blocks = (n4 + 255) / 256;
      indentation_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
          reinterpret_cast<const float4*>(depth), reinterpret_cast<float4*>(ind), rest, rest_lo, n4);
    }
  }
  const long long start = n4 * 4;
  if (start < n)
    indentation_tail<<<(unsigned)((n - start + 255) / 256), 256, 0, s>>>(depth, ind, rest, rest_lo, start, n);
  return cudaGetLastError();
}

cudaError_t launch_normals(const float* elev, float* normals, int H, int W, float inv_p,
                           float inv_2p, long long n_env, cudaStream_t s) {
  const long long total = n_env * H * W;
  if (total == 0) return cudaSuccess;
  normals_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(elev, normals, H, W, inv_p, inv_2p,
                                                                 total);
  return cudaGetLastError();
}

cudaError_t launch_quantize_bg(const float* bg, uint8_t* bg_u8, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  quantize_bg_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(bg, bg_u8, n);
  return cudaGetLastError();
}

cudaError_t launch_track_load(double* state, const double* pose_delta, const double* contact,
                              long long n_env, cudaStream_t s) {
  if (n_env == 0) return cudaSuccess;
  track_load_kernel<<<(unsigned)((n_env + 127) / 128), 128, 0, s>>>(state, pose_delta, contact,
                                                                    n_env);
  return cudaGetLastError();
}

cudaError_t launch_marker_displacements(const MarkerGeom& m, const double* loads, float* disp,
                                        long long n_env, cudaStream_t s) {
  if (n_env == 0) return cudaSuccess;
  const size_t smem = 2 * sizeof(int) * (size_t)m.rows * m.cols;
  markers_kernel<<<(unsigned)n_env, 128, smem, s>>>(m, loads, disp, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_render_markers(const MarkerGeom& m, const float* disp, uint8_t* rgb,
                                  long long n_env, cudaStream_t s) {
  if (n_env == 0) return cudaSuccess;
  const size_t smem = 2 * sizeof(int) * (size_t)m.rows * m.cols;
  markers_kernel<<<(unsigned)n_env, 128, smem, s>>>(m, nullptr, nullptr, disp, rgb);
  return cudaGetLastError();
}

}  // namespace tac
