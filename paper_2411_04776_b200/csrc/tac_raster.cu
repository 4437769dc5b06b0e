// Row f2: render_heightmap (REF/tactile.py:129-190) -- orthographic z-buffer of
// camera-frame triangles, batched over envs that share one triangle list.
//
// The arithmetic is the reference's, in fp64, in the same operation order
// with every product / sum / quotient explicitly rounded (__dmul_rn & co., so
// the compiler cannot contract them into FMAs): the culling tests, the
// edge-on skip (|det| < 1e-18), the pixel-centre bounding box
// ceil/floor(min/max(x) / p + w/2 - 1/2), the barycentrics with the -1e-12
// inside tolerance, and z = l0 z0 + l1 z1 + l2 z2 <= rest.  The depth buffer
// holds order-preserving uint32 keys of the fp32 depth and is lowered with
// atomicMin (rounding to fp32 is monotonic, so min-then-round == round-then-
// min and the result equals fp32(reference fp64 depth) exactly, independent
// of triangle order).
//
// Work split: one thread per (env, triangle) does the setup; triangles whose
// bounding box has at most kSmall pixels are rasterised by that thread, the
// others are queued in shared memory and swept by the whole CTA.
#include <cstdint>
#include <cstring>
#include <algorithm>

#include "tac_internal.cuh"

namespace tac {

namespace {

constexpr int kRasterThreads = 256;
constexpr int kSmall = 32;

__host__ __device__ __forceinline__ uint32_t key_of(float f) {
#ifdef __CUDA_ARCH__
  const uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_of(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

struct Tri {
  double x0, y0, z0, x1, y1, z1, x2, y2, z2, det;
  int i0, i1, j0, j1;
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// Setup of one triangle; false if culled (REF/tactile.py:154-173).
__device__ bool tri_setup(const double* v, const int* t, int W, int H, double pitch, double rest,
                          Tri& o) {
  const double* a = v + 3 * t[0];
  const double* b = v + 3 * t[1];
  const double* c = v + 3 * t[2];
  o.x0 = a[0]; o.y0 = a[1]; o.z0 = a[2];
  o.x1 = b[0]; o.y1 = b[1]; o.z1 = b[2];
  o.x2 = c[0]; o.y2 = c[1]; o.z2 = c[2];
  const double zmin = fmin(fmin(o.z0, o.z1), o.z2);
  const double xmin = fmin(fmin(o.x0, o.x1), o.x2), xmax = fmax(fmax(o.x0, o.x1), o.x2);
  const double ymin = fmin(fmin(o.y0, o.y1), o.y2), ymax = fmax(fmax(o.y0, o.y1), o.y2);
  const double half_w = mul(mul(0.5, (double)W), pitch);
  const double half_h = mul(mul(0.5, (double)H), pitch);
  if (!(zmin <= rest) || !(xmax >= -half_w) || !(xmin <= half_w) || !(ymax >= -half_h) ||
      !(ymin <= half_h))
    return false;
  o.det = add(mul(sub(o.y1, o.y2), sub(o.x0, o.x2)), mul(sub(o.x2, o.x1), sub(o.y0, o.y2)));
  if (fabs(o.det) < 1e-18) return false;  // edge-on to the ray direction
  const double hw = mul(0.5, (double)W), hh = mul(0.5, (double)H);
  // clamp in fp64 before converting (huge triangles must not overflow int)
  o.j0 = (int)fmax(ceil(sub(add(__ddiv_rn(xmin, pitch), hw), 0.5)), 0.0);
  o.j1 = (int)fmin(floor(sub(add(__ddiv_rn(xmax, pitch), hw), 0.5)), (double)(W - 1));
  o.i0 = (int)fmax(ceil(sub(add(__ddiv_rn(ymin, pitch), hh), 0.5)), 0.0);
  o.i1 = (int)fmin(floor(sub(add(__ddiv_rn(ymax, pitch), hh), 0.5)), (double)(H - 1));
  return o.j1 >= o.j0 && o.i1 >= o.i0;
}

// One pixel (REF/tactile.py:179-190).
__device__ __forceinline__ void tri_pixel(const Tri& t, int i, int j, int W, int H, double pitch,
                                          double rest, uint32_t* keys) {
  const double px = mul(sub(add((double)j, 0.5), mul(0.5, (double)W)), pitch);
  const double py = mul(sub(add((double)i, 0.5), mul(0.5, (double)H)), pitch);
  const double dx = sub(px, t.x2), dy = sub(py, t.y2);
  const double l0 = __ddiv_rn(add(mul(sub(t.y1, t.y2), dx), mul(sub(t.x2, t.x1), dy)), t.det);
  const double l1 = __ddiv_rn(add(mul(sub(t.y2, t.y0), dx), mul(sub(t.x0, t.x2), dy)), t.det);
  const double l2 = sub(sub(1.0, l0), l1);
  const double eps = -1e-12;
  if (!(l0 >= eps && l1 >= eps && l2 >= eps)) return;
  const double z = add(add(mul(l0, t.z0), mul(l1, t.z1)), mul(l2, t.z2));
  if (!(z <= rest)) return;
  atomicMin(keys + (long long)i * W + j, key_of((float)z));
}

__global__ void __launch_bounds__(kRasterThreads) raster_init_kernel(uint32_t* keys, long long n, uint32_t k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    keys[i] = k;
}

// grid (ceil(T / 256), envs)
__global__ void __launch_bounds__(kRasterThreads) raster_kernel(const double* __restrict__ verts,
                                                                long long n_verts,
                                                                const int* __restrict__ tris, int n_tris,
                                                                uint32_t* __restrict__ keys, int W, int H,
                                                                double pitch, double rest) {
  __shared__ Tri big[kRasterThreads];
  __shared__ int n_big;
  const long long env = blockIdx.y;
  const double* v = verts + env * n_verts * 3;
  uint32_t* k = keys + env * (long long)H * W;
  if (threadIdx.x == 0) n_big = 0;
  __syncthreads();
  const int ti = blockIdx.x * kRasterThreads + threadIdx.x;
  Tri t;
  if (ti < n_tris && tri_setup(v, tris + 3 * ti, W, H, pitch, rest, t)) {
    const int nj = t.j1 - t.j0 + 1;
    const int npx = (t.i1 - t.i0 + 1) * nj;
    if (npx <= kSmall) {
      for (int q = 0; q < npx; ++q) tri_pixel(t, t.i0 + q / nj, t.j0 + q % nj, W, H, pitch, rest, k);
    } else {
      big[atomicAdd(&n_big, 1)] = t;
    }
  }
  __syncthreads();
  for (int b = 0; b < n_big; ++b) {  // large triangles: the whole CTA sweeps the box
    const Tri& tb = big[b];
    const int nj = tb.j1 - tb.j0 + 1;
    const int npx = (tb.i1 - tb.i0 + 1) * nj;
    for (int q = threadIdx.x; q < npx; q += kRasterThreads)
      tri_pixel(tb, tb.i0 + q / nj, tb.j0 + q % nj, W, H, pitch, rest, k);
  }
}

__global__ void __launch_bounds__(kRasterThreads) raster_finish_kernel(uint32_t* keys, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    reinterpret_cast<float*>(keys)[i] = float_of(keys[i]);
}

}  // namespace

// depth: [N][H][W] fp32, used in place as the key buffer.
cudaError_t launch_raster(const double* verts, long long n_verts, const int* tris, int n_tris, float* depth,
                          int H, int W, double pitch, double rest, long long n_env, cudaStream_t s) {
  const long long n = n_env * (long long)H * W;
  if (n == 0) return cudaSuccess;
  uint32_t* keys = reinterpret_cast<uint32_t*>(depth);
  const unsigned g = (unsigned)std::min<long long>((n + kRasterThreads - 1) / kRasterThreads, 148 * 16);
  raster_init_kernel<<<g, kRasterThreads, 0, s>>>(keys, n, key_of((float)rest));
  for (long long e0 = 0; n_tris > 0 && e0 < n_env; e0 += 65535) {  // grid.y <= 65535
    const long long ne = std::min<long long>(65535, n_env - e0);
    dim3 grid((unsigned)((n_tris + kRasterThreads - 1) / kRasterThreads), (unsigned)ne);
    raster_kernel<<<grid, kRasterThreads, 0, s>>>(verts + e0 * n_verts * 3, n_verts, tris, n_tris,
                                                  keys + e0 * (long long)H * W, W, H, pitch, rest);
  }
  raster_finish_kernel<<<g, kRasterThreads, 0, s>>>(keys, n);
  return cudaGetLastError();
}

}  // namespace tac
