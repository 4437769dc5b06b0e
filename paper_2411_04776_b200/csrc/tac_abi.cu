// C ABI: context lifetime, argument validation (error classes of
// REF/errors.py), and kernel launches.  No CPU fallback: every compute entry
// point enqueues CUDA work on the caller's stream or returns an error.
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_fp16.h>

#include "tac_internal.cuh"

using namespace tac;

struct tac_ctx {
  tac_config cfg;  // host pointers cleared after upload
  int device;
  float4* d_lut = nullptr;
  float* d_bg = nullptr;
  float4* d_lut_half = nullptr;    // [2][bins][8] float: plane h = floats 8h..8h+7 of every bin (256-bit loads)
  uint4* d_lut_h16 = nullptr;      // lut_dtype f16: [bins][16] fp16, direction-major (one 32-B sector per bin)
  cudaTextureObject_t lut_tex = 0;  // float4 texels over d_lut_half (texture path for the gathers)
  float* d_bg_planar = nullptr;    // [3][H*W]: R, G, B background planes (v5 shading)
  uint8_t* d_bg_u8 = nullptr;
  double* d_grid = nullptr;
  int2* d_shadow_off = nullptr;
  float* d_shadow_cost = nullptr;
  ShadowParams shadow;
  FrameParams fused, blur, contact;  // per-mode launch templates
  FrameParams fused5;                // two-kernel geometry (row-streaming or band-tiled blur)
  bool use5;                         // two-kernel path (TAC_PATH_STREAM or TAC_PATH_BAND)
  int path;                          // TAC_PATH_* taken for aligned input
  long long chunk5;                  // envs per blur/shade launch pair
  MarkerGeom mg;
  int max_tiles;  // max column strips per frame over the modes
  // diagnostics: kernel-boundary events of the pipeline calls between
  // tac_timing_begin and tac_timing_end (one session per context)
  mutable struct {
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
    std::vector<std::pair<int, int>> calls;  // [first event, count) of each recorded call
    int next = 0, max_calls = 0;
    bool on = false;
  } timing;
};

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(TAC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

static int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Geometry of the strip-streaming kernel for one mode (see tac_frame.cu).
void plan_strips(FrameParams& p, int mode, int max_strip) {
  if (mode == kModeContact) p.R = 0;
  const int R = p.R;
  if (p.W <= max_strip + max_strip / 10) {
    p.strips = 1;
    p.strip_w = p.W;
  } else {
    p.strips = (p.W + max_strip - 1) / max_strip;
    p.strip_w = round_up((p.W + p.strips - 1) / p.strips, 16);
    p.strips = (p.W + p.strip_w - 1) / p.strip_w;
  }
  const int ring = (mode == kModeFused && p.strips > 1) ? 1 : 0;
  const int ew = p.strip_w + 2 * ring + 3;        // blurred columns (origin 4-aligned)
  const int lw = (p.strips == 1) ? round_up(p.W, 4) : round_up(ew + 2 * R + 6, 4);
  p.in_pitch = round_up(lw, 4);
  p.in_rows = RB + 2 * R;
  int vp = round_up(ew, KH) + 2 * R + 1;
  if ((vp & 1) == 0) ++vp;  // odd: the H pass reads 16 rows x 2 chunks conflict-free
  p.v_pitch = vp;
  int bp = round_up(ew + 3 + 8, 4);
  if (((bp / 4) & 1) == 0) bp += 4;  // 4 x odd: float4 rows on distinct bank groups
  p.b_pitch = bp;
  (void)0;
  p.stage_bytes = (RB + 1) * p.strip_w * 3;
}

// Geometry of the band-tiled path (see tac_frame5.cu): input rows of W floats,
// vb rows from column -round_up(R, 4) to W + round_up(R, 4).
void plan_v5(FrameParams& p) {
  const int R4 = round_up(p.R, 4);
  p.bands = (p.H + 15) / 16;
  p.in_pitch = p.W;
  p.in_rows = 16 + 2 * p.R;
  p.v_pitch = frame5_vpitch(p.W, R4);  // layout-dependent (tac_frame5.cu)
  p.b_pitch = 0;
  p.stage_bytes = 0;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// v5 workspace (after the v3 region): band partials for every env, then the
// per-chunk band extents and blurred scratch.
size_t v5_workspace_bytes(const tac_ctx* c, int64_t n_env) {
  if (!c->use5) return 0;
  const long long C = std::min<long long>(n_env, c->chunk5);
  const FrameParams& p = c->fused5;
  return align256((size_t)n_env * p.nparts * kSumFields * sizeof(double)) +
         align256((size_t)C * p.bands * p.ext_strips * sizeof(int2)) + align256((size_t)C * p.H * p.W * sizeof(float));
}

// add_shadows factor computed by tac_pipeline itself (shadows on, no caller
// factor): one chunk on the two-kernel path, every env on the fused path.
size_t shadow_workspace_bytes(const tac_ctx* c, int64_t n_env) {
  if (c->shadow.n_lights == 0) return 0;
  const long long C = c->use5 ? std::min<long long>(n_env, c->chunk5) : n_env;
  return align256((size_t)C * c->cfg.height * c->cfg.width * sizeof(float));
}

size_t v3_workspace_bytes(const tac_ctx* c, int64_t n_env) {
  const size_t part = align256((size_t)n_env * c->max_tiles * kSumFields * sizeof(double));
  return part + align256((size_t)n_env * sizeof(unsigned int));
}

void bind_workspace5(const tac_ctx* c, FrameParams& p, void* ws, int64_t n_env) {
  const long long C = std::min<long long>(n_env, c->chunk5);
  char* b = reinterpret_cast<char*>(ws) + v3_workspace_bytes(c, n_env);
  p.partials = reinterpret_cast<double*>(b);
  b += align256((size_t)n_env * p.nparts * kSumFields * sizeof(double));
  p.band_ext = reinterpret_cast<int2*>(b);
  b += align256((size_t)C * p.bands * p.ext_strips * sizeof(int2));
  p.scratch = reinterpret_cast<float*>(b);
  p.chunk = C;
}

int free_ctx(tac_ctx* c) {
  if (!c) return TAC_OK;
  cudaFree(c->d_lut);
  cudaFree(c->d_bg);
  if (c->lut_tex) cudaDestroyTextureObject(c->lut_tex);
  cudaFree(c->d_lut_half);
  cudaFree(c->d_lut_h16);
  cudaFree(c->d_bg_planar);
  cudaFree(c->d_bg_u8);
  cudaFree(c->d_grid);
  cudaFree(c->d_shadow_off);
  cudaFree(c->d_shadow_cost);
  for (cudaEvent_t e : c->timing.ev) cudaEventDestroy(e);
  delete c;
  return TAC_OK;
}

int check_device(const tac_ctx* c) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev != c->device)
    return fail(TAC_ERR_INVALID, "context was created on device %d but the current device is %d",
                c->device, dev);
  return TAC_OK;
}

int common_checks(const tac_ctx* c, int64_t n_env) {
  if (!c) return fail(TAC_ERR_INVALID, "null context");
  if (n_env < 0) return fail(TAC_ERR_INVALID, "n_env must be >= 0");
  if (n_env > (int64_t)0x7fffffff / std::max(1, c->max_tiles))
    return fail(TAC_ERR_UNSUPPORTED, "n_env too large for one launch");
  return check_device(c);
}

int tma_ok(const FrameParams& p, const void* in) {
  return (p.W % 4 == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
}

// Strip-streaming kernel workspace: per-strip partials (always overwritten),
// then the per-env arrival counters of multi-strip frames, zeroed here on the
// call's stream (graph-capturable), so the workspace contents never matter.
cudaError_t bind_workspace(const tac_ctx* c, FrameParams& p, void* ws, int64_t n_env, cudaStream_t s) {
  p.partials = reinterpret_cast<double*>(ws);
  const size_t part_bytes = (((size_t)n_env * c->max_tiles * kSumFields * sizeof(double)) + 255) & ~size_t(255);
  p.counters = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(ws) + part_bytes);
  if (p.strips > 1 && n_env > 0) return cudaMemsetAsync(p.counters, 0, sizeof(unsigned int) * n_env, s);
  return cudaSuccess;
}

}  // namespace

extern "C" {

const char* tac_last_error(void) { return g_err.c_str(); }

int tac_ctx_create(const tac_config* cfg, tac_ctx** out) {
  if (!cfg || !out) return fail(TAC_ERR_INVALID, "null argument");
  *out = nullptr;
  if (cfg->struct_size != sizeof(tac_config))
    return fail(TAC_ERR_INVALID, "tac_config.struct_size is %u, this library expects %zu (header version %d)",
                cfg->struct_size, sizeof(tac_config), TAC_ABI_VERSION);
  const tac_config& k = *cfg;
  if (k.height < 2 || k.width < 2) return fail(TAC_ERR_INVALID, "image_size must be >= 2 x 2");
  if (!finite_pos(k.pixel_pitch)) return fail(TAC_ERR_INVALID, "pixel_pitch must be positive");
  if (!finite_pos(k.gel_thickness)) return fail(TAC_ERR_INVALID, "gelpad_thickness must be positive");
  if (k.n_levels < 1 || k.n_levels > TAC_MAX_LEVELS)
    return fail(TAC_ERR_INVALID, "pyramid needs 1..%d levels", TAC_MAX_LEVELS);
  int R = 0;
  for (int l = 0; l < k.n_levels; ++l) {
    if (k.radius[l] < 0) return fail(TAC_ERR_INVALID, "radius must be >= 0");
    if (k.radius[l] > TAC_MAX_RADIUS)
      return fail(TAC_ERR_UNSUPPORTED, "radius %d exceeds TAC_MAX_RADIUS=%d", k.radius[l], TAC_MAX_RADIUS);
    if (k.radius[l] > 0 && !finite_pos(k.sigma[l])) return fail(TAC_ERR_INVALID, "sigma must be positive");
    R = std::max(R, k.radius[l]);
  }
  if (k.mag_bins < 1 || k.dir_bins < 1) return fail(TAC_ERR_INVALID, "LUT bins must be >= 1");
  if (!finite_pos(k.g_max)) return fail(TAC_ERR_INVALID, "g_max must be positive");
  if (!k.lut || !k.background) return fail(TAC_ERR_INVALID, "lut and background are required");
  if (k.marker_rows < 1 || k.marker_cols < 1) return fail(TAC_ERR_INVALID, "marker_grid must be positive");
  const double lam[3] = {k.lambda_n, k.lambda_s, k.lambda_t};
  for (double v : lam)
    if (!finite_pos(v)) return fail(TAC_ERR_INVALID, "marker length scales must be positive");
  if (!std::isfinite(k.k_n) || !std::isfinite(k.k_t)) return fail(TAC_ERR_INVALID, "marker params must be finite");
  if (!finite_pos(k.contact_threshold)) return fail(TAC_ERR_INVALID, "threshold must be positive");
  if (k.dot_radius < 0 || k.dot_radius > 32) return fail(TAC_ERR_UNSUPPORTED, "dot_radius must be in 0..32");
  if (k.lut_dtype != TAC_LUT_F32 && k.lut_dtype != TAC_LUT_F16)
    return fail(TAC_ERR_INVALID, "unknown lut_dtype %d", k.lut_dtype);
  if (k.kernel_path < TAC_PATH_AUTO || k.kernel_path > TAC_PATH_STREAM)
    return fail(TAC_ERR_INVALID, "unknown kernel_path %d", k.kernel_path);
  if (k.chunk_envs < 0) return fail(TAC_ERR_INVALID, "chunk_envs must be >= 0");
  if (k.n_lights < 0 || k.n_lights > TAC_MAX_LIGHTS)
    return fail(TAC_ERR_INVALID, "n_lights must be in 0..%d", TAC_MAX_LIGHTS);
  if (!(k.shadow_factor >= 0.0 && k.shadow_factor <= 1.0))
    return fail(TAC_ERR_INVALID, "shadow factor must be in [0, 1]");
  const bool shadows_on = k.shadow_factor != 1.0 && k.n_lights > 0;
  if (shadows_on) {
    if (k.shadow_steps < 1 || k.shadow_steps > TAC_MAX_SHADOW_STEPS)
      return fail(TAC_ERR_UNSUPPORTED, "shadow steps must be in 1..%d", TAC_MAX_SHADOW_STEPS);
    if (!finite_pos(k.shadow_softness)) return fail(TAC_ERR_INVALID, "shadow softness must be positive");
    for (int l = 0; l < k.n_lights; ++l)
      for (int q = 0; q < 3; ++q)
        if (!std::isfinite(k.light_dir[l][q])) return fail(TAC_ERR_INVALID, "lighting values must be finite");
  }
  const size_t HW = (size_t)k.height * k.width;
  for (size_t i = 0; i < HW * 3; ++i)
    if (!std::isfinite(k.background[i])) return fail(TAC_ERR_INVALID, "table values must be finite");
  const size_t nbins = (size_t)k.mag_bins * k.dir_bins;
  for (size_t i = 0; i < nbins * 18; ++i)
    if (!std::isfinite(k.lut[i])) return fail(TAC_ERR_INVALID, "table values must be finite");

  tac_ctx* c = new tac_ctx();
  c->cfg = k;
  c->cfg.lut = nullptr;
  c->cfg.background = nullptr;
  c->cfg.rest_grid = nullptr;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) {
    free_ctx(c);
    return cuda_fail(e, "cudaGetDevice");
  }

  // LUT: [mag][dir][3][6] -> [mag*dir][16] = c1..c5 per channel + pad.
  // lut_dtype f16 rounds every coefficient to fp16 (nearest even) for ALL
  // shading paths, so they compute with the same table
  std::vector<float> lut(nbins * 16, 0.f);
  std::vector<__half> lut16(nbins * 16, __float2half_rn(0.f));
  for (size_t b = 0; b < nbins; ++b)
    for (int ch = 0; ch < 3; ++ch)
      for (int t = 1; t < 6; ++t) {
        float v = k.lut[(b * 3 + ch) * 6 + t];
        if (k.lut_dtype == TAC_LUT_F16) {
          const __half h = __float2half_rn(v);
          v = __half2float(h);
          const size_t mb = b / k.dir_bins, db = b % k.dir_bins;
          lut16[(db * k.mag_bins + mb) * 16 + ch * 5 + (t - 1)] = h;
        }
        lut[b * 16 + ch * 5 + (t - 1)] = v;
      }
  // half-planar LUT for the band shading kernel (plane h = floats 8h..8h+7 of
  // every bin, one 256-bit load each: a 128-B line holds 4 bins of a plane) and
  // R/G/B background planes (coalesced loads).  Bins in direction-major
  // order [dir][mag]: neighbouring pixels' bins share lines most often
  // (measured against [mag][dir] and 4x2 tiles in round 1)
  const size_t nbins_p = nbins;
  std::vector<float> luth(nbins_p * 16, 0.f);
  for (size_t b = 0; b < nbins; ++b) {
    const size_t mb = b / k.dir_bins, db = b % k.dir_bins;
    const size_t o = db * k.mag_bins + mb;
    for (int hh = 0; hh < 2; ++hh)
      for (int q = 0; q < 8; ++q) luth[(hh * nbins_p + o) * 8 + q] = lut[b * 16 + hh * 8 + q];
  }
  std::vector<float> bgp(HW * 3);
  for (size_t i = 0; i < HW; ++i)
    for (int ch = 0; ch < 3; ++ch) bgp[ch * HW + i] = k.background[i * 3 + ch];
  std::vector<uint8_t> bgq(HW * 3);
  for (size_t i = 0; i < HW * 3; ++i) {
    long v = std::lrint((double)k.background[i]);  // half-to-even (default rounding mode)
    bgq[i] = (uint8_t)std::min(255L, std::max(0L, v));
  }
  const int nm = k.marker_rows * k.marker_cols;
  std::vector<double> grid(nm * 2);
  if (cfg->rest_grid) {
    std::memcpy(grid.data(), cfg->rest_grid, sizeof(double) * nm * 2);
  } else {
    // grid_rest_positions, REF/marker.py:93-100; sensing area = (W p, H p)
    const double aw = k.width * k.pixel_pitch, ah = k.height * k.pixel_pitch;
    for (int i = 0; i < k.marker_rows; ++i)
      for (int j = 0; j < k.marker_cols; ++j) {
        grid[(i * k.marker_cols + j) * 2 + 0] = ((j + 0.5) / k.marker_cols - 0.5) * aw;
        grid[(i * k.marker_cols + j) * 2 + 1] = ((i + 0.5) / k.marker_rows - 0.5) * ah;
      }
  }
  struct Up {
    void** dst;
    const void* src;
    size_t bytes;
  } ups[] = {
      {(void**)&c->d_lut, lut.data(), lut.size() * sizeof(float)},
      {(void**)&c->d_bg, k.background, HW * 3 * sizeof(float)},
      {(void**)&c->d_bg_u8, bgq.data(), bgq.size()},
      {(void**)&c->d_lut_half, luth.data(), luth.size() * sizeof(float)},
      {(void**)&c->d_bg_planar, bgp.data(), bgp.size() * sizeof(float)},
      {(void**)&c->d_grid, grid.data(), grid.size() * sizeof(double)},
      {(void**)&c->d_lut_h16, lut16.data(), k.lut_dtype == TAC_LUT_F16 ? lut16.size() * sizeof(__half) : 0},
  };
  for (auto& u : ups) {
    if (u.bytes == 0) continue;
    e = cudaMalloc(u.dst, u.bytes);
    if (e == cudaSuccess) e = cudaMemcpy(*u.dst, u.src, u.bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_ctx(c);
      return cuda_fail(e, "context upload");
    }
  }

  // add_shadows march tables, exactly as REF/optical.py:283-291 in fp64
  {
    ShadowParams& sp = c->shadow;
    std::memset(&sp, 0, sizeof(sp));
    sp.H = k.height;
    sp.W = k.width;
    std::vector<int2> off;
    std::vector<float> cost;
    int lights = 0;
    if (shadows_on) {
      for (int l = 0; l < k.n_lights; ++l) {
        const double lx = k.light_dir[l][0], ly = k.light_dir[l][1], lz = k.light_dir[l][2];
        const double lateral = std::hypot(lx, ly);
        if (lateral < 1e-9) continue;  // overhead light casts no lateral shadow
        const double dx = lx / lateral, dy = ly / lateral;
        const double rise = k.pixel_pitch * lz / lateral;
        for (int st = 1; st <= k.shadow_steps; ++st) {
          int2 o;
          o.x = (int)std::nearbyint(st * dy);  // Python round: half to even
          o.y = (int)std::nearbyint(st * dx);
          off.push_back(o);
          cost.push_back((float)(st * rise));
          sp.di_min = std::min(sp.di_min, o.x);
          sp.di_max = std::max(sp.di_max, o.x);
          sp.dj_min = std::min(sp.dj_min, o.y);
          sp.dj_max = std::max(sp.dj_max, o.y);
        }
        ++lights;
      }
    }
    sp.n_lights = lights;
    sp.steps = lights ? k.shadow_steps : 0;
    sp.one_minus_factor = (float)(1.0 - k.shadow_factor);
    sp.inv_softness = shadows_on ? (float)(1.0 / k.shadow_softness) : 0.f;
    if (lights) {
      e = cudaMalloc(&c->d_shadow_off, off.size() * sizeof(int2));
      if (e == cudaSuccess) e = cudaMemcpy(c->d_shadow_off, off.data(), off.size() * sizeof(int2), cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMalloc(&c->d_shadow_cost, cost.size() * sizeof(float));
      if (e == cudaSuccess)
        e = cudaMemcpy(c->d_shadow_cost, cost.data(), cost.size() * sizeof(float), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        free_ctx(c);
        return cuda_fail(e, "shadow tables");
      }
    }
    sp.off = c->d_shadow_off;
    sp.cost = c->d_shadow_cost;
    // tiled-march geometry: per light, the region of a kShadowTH x kShadowTW
    // output tile shifted by every offset of that light
    size_t region = 0;
    for (int l = 0; l < lights; ++l) {
      int dimn = INT_MAX, dimx = INT_MIN, djmn = INT_MAX, djmx = INT_MIN;
      for (int st = 0; st < sp.steps; ++st) {
        const int2 o = off[l * sp.steps + st];
        dimn = std::min(dimn, o.x);
        dimx = std::max(dimx, o.x);
        djmn = std::min(djmn, o.y);
        djmx = std::max(djmx, o.y);
      }
      // region columns start at a multiple of 4 (tile origins are) so rows
      // stage with 16-B loads; width a multiple of 4
      const int dja = (int)std::floor(djmn / 4.0) * 4;
      sp.l_di_min[l] = dimn;
      sp.l_dj_min[l] = dja;
      sp.l_rh[l] = kShadowTH + dimx - dimn;
      sp.l_rw[l] = (kShadowTW + djmx - dja + 3) & ~3;
      region = std::max(region, (size_t)sp.l_rh[l] * sp.l_rw[l] * sizeof(float));
      for (int st = 0; st < sp.steps; ++st) {
        const int2 o = off[l * sp.steps + st];
        sp.offb[l][st] = ((o.x - dimn) * sp.l_rw[l] + (o.y - dja)) * (int)sizeof(float);
        sp.costs[l][st] = cost[l * sp.steps + st];
      }
    }
    sp.tiled = lights > 0 && region <= 72 * 1024 && k.width % 4 == 0;
  }

  MarkerGeom& mg = c->mg;
  mg.H = k.height;
  mg.W = k.width;
  mg.pitch = k.pixel_pitch;
  mg.rows = k.marker_rows;
  mg.cols = k.marker_cols;
  mg.rest_grid = c->d_grid;
  mg.k_n = k.k_n;
  mg.lambda_n = k.lambda_n;
  mg.lambda_s = k.lambda_s;
  mg.k_t = k.k_t;
  mg.lambda_t = k.lambda_t;
  mg.dot_radius = k.dot_radius;
  mg.dot_r = k.dot_color[0];
  mg.dot_g = k.dot_color[1];
  mg.dot_b = k.dot_color[2];

  FrameParams b;
  std::memset(&b, 0, sizeof(b));
  b.H = k.height;
  b.W = k.width;
  b.R = R;
  b.n_levels = k.n_levels;
  for (int l = 0; l < k.n_levels; ++l) {
    const int r = k.radius[l];
    b.radius[l] = r;
    // gaussian taps exactly as scipy's _gaussian_kernel1d, in fp64
    std::vector<double> w(r + 1);
    if (r == 0) {
      w[0] = 1.0;
    } else {
      double sum = 0.0;
      const double s2 = k.sigma[l] * k.sigma[l];
      std::vector<double> phi(2 * r + 1);
      for (int x = -r; x <= r; ++x) {
        phi[x + r] = std::exp(-0.5 / s2 * (double)x * (double)x);
        sum += phi[x + r];
      }
      for (int i = 0; i <= r; ++i) w[i] = phi[r + i] / sum;
    }
    for (int i = 0; i <= r; ++i) {
      b.wv[l][i] = (float)w[i];
      b.wh[l][i] = (float)(w[i] / k.n_levels);
      b.wv2[l][i] = make_float2(b.wv[l][i], b.wv[l][i]);
      b.wh2[l][i] = make_float2(b.wh[l][i], b.wh[l][i]);
    }
  }
  b.rest = (float)k.gel_thickness;
  b.rest_lo = (float)(k.gel_thickness - (double)b.rest);
  b.threshold = (float)k.contact_threshold;
  b.half_w = 0.5f * k.width;
  b.half_h = 0.5f * k.height;
  b.xoff = 0.5 - 0.5 * k.width;
  b.yoff = 0.5 - 0.5 * k.height;
  b.inv_p = (float)(1.0 / k.pixel_pitch);
  b.inv_2p = (float)(1.0 / (2.0 * k.pixel_pitch));
  b.mag_scale = (float)(k.mag_bins / k.g_max);
  b.dir_scale = (float)(k.dir_bins / (2.0 * M_PI));
  b.mag_bins = k.mag_bins;
  b.dir_bins = k.dir_bins;
  b.lut = c->d_lut;
  b.bg = c->d_bg;
  b.lut_half = reinterpret_cast<const float*>(c->d_lut_half);
  {
    cudaResourceDesc rd;
    std::memset(&rd, 0, sizeof(rd));
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = c->d_lut_half;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = luth.size() * sizeof(float);
    cudaTextureDesc td;
    std::memset(&td, 0, sizeof(td));
    td.readMode = cudaReadModeElementType;
    td.filterMode = cudaFilterModePoint;
    if (cudaCreateTextureObject(&c->lut_tex, &rd, &td, nullptr) != cudaSuccess) c->lut_tex = 0;
    cudaGetLastError();
  }
  b.lut_tex = c->lut_tex;
  b.bg_planar = c->d_bg_planar;
  b.lut_h16 = c->d_lut_h16;
  b.nbins = (int)nbins_p;
  b.bg_u8 = c->d_bg_u8;
  b.mg = mg;

  const int max_strip = 320;  // strip-streaming kernel: columns per CTA
  c->fused = b;
  plan_strips(c->fused, kModeFused, max_strip);
  c->blur = b;
  plan_strips(c->blur, kModeBlur, max_strip);
  c->contact = b;
  plan_strips(c->contact, kModeContact, max_strip);
  c->max_tiles = std::max({c->fused.strips, c->blur.strips, c->contact.strips});
  // tac_pipeline path: row-streaming blur (instantiated pyramids) > band blur
  // (W <= 320, R <= 16) > strip-streaming fused kernel (anything else)
  c->fused5 = c->fused;
  plan_v5(c->fused5);
  c->fused5.nparts = c->fused5.bands;
  c->fused5.ext_strips = 1;
  c->fused5.st_kind = -1;
  c->path = TAC_PATH_FUSED;
  {
    FrameParams st = c->fused5;
    plan_stream(st);
    const bool want = k.kernel_path == TAC_PATH_AUTO || k.kernel_path == TAC_PATH_STREAM;
    if (want && st.st_kind >= 0 && shade5_eligible(st)) {
      st.nparts = st.st_strips;
      st.ext_strips = st.st_strips;
      c->fused5 = st;
      c->path = TAC_PATH_STREAM;
    } else if ((k.kernel_path == TAC_PATH_AUTO || k.kernel_path == TAC_PATH_BAND) && frame5_eligible(c->fused5)) {
      c->path = TAC_PATH_BAND;
    }
  }
  if (k.kernel_path != TAC_PATH_AUTO && c->path != k.kernel_path) {
    free_ctx(c);
    return fail(TAC_ERR_UNSUPPORTED, "kernel_path %d is not available for this configuration", k.kernel_path);
  }
  c->use5 = c->path == TAC_PATH_STREAM || c->path == TAC_PATH_BAND;
  // default chunk: as many envs as fit a 10 GiB blurred scratch (one launch
  // pair for configs[4]'s 32768 envs of 240x320: fewer kernel tails; measured
  // 4096 -> 32768 envs per pair +2.8 %)
  c->chunk5 = k.chunk_envs > 0 ? k.chunk_envs
                               : std::max<long long>(1, (10ll << 30) / ((long long)k.height * k.width * 4));
  for (int mode = 0; mode < 3; ++mode) {
    FrameParams& p = mode == kModeFused ? c->fused : (mode == kModeBlur ? c->blur : c->contact);
    if (p.stage_bytes > (int)(RB * p.v_pitch * sizeof(float))) {
      free_ctx(c);
      return fail(TAC_ERR_UNSUPPORTED, "staging buffer does not fit (strip %d)", p.strip_w);
    }
    if (frame_smem_bytes(p) > 227 * 1024) {
      free_ctx(c);
      return fail(TAC_ERR_UNSUPPORTED,
                  "strip of %d columns with radius %d needs %zu B of shared memory (max 227 KB)",
                  p.strip_w, p.R, frame_smem_bytes(p));
    }
  }
  *out = c;
  return TAC_OK;
}

int tac_ctx_destroy(tac_ctx* ctx) { return free_ctx(ctx); }

size_t tac_workspace_bytes(const tac_ctx* c, int64_t n_env) {
  if (!c || n_env < 0) return 0;
  return v3_workspace_bytes(c, n_env) + v5_workspace_bytes(c, n_env) + shadow_workspace_bytes(c, n_env);
}

int32_t tac_tiles_per_frame(const tac_ctx* c) { return c ? c->fused.strips : 0; }


int tac_render_heightmap(const tac_ctx* c, const double* verts, int64_t n_verts, const int32_t* tris,
                         int64_t n_tris, float* depth, int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_verts < 0 || n_tris < 0) return fail(TAC_ERR_INVALID, "n_verts and n_tris must be >= 0");
  if (n_tris > 0x7fffffff / 3) return fail(TAC_ERR_UNSUPPORTED, "too many triangles");
  if (n_env && !depth) return fail(TAC_ERR_INVALID, "null depth buffer");
  if (n_env && n_tris && (!verts || !tris)) return fail(TAC_ERR_INVALID, "null vertex or triangle buffer");
  if (n_tris && n_verts == 0) return fail(TAC_ERR_INVALID, "triangles need vertices");
  cudaError_t e = launch_raster(verts, n_verts, tris, (int)n_tris, depth, c->cfg.height, c->cfg.width,
                                c->cfg.pixel_pitch, c->cfg.gel_thickness, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_render_heightmap");
}

int tac_indentation(const tac_ctx* c, const float* depth, float* ind, int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!depth || !ind)) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_indentation(depth, ind, c->fused.rest, c->fused.rest_lo,
                                     n_env * (long long)c->cfg.height * c->cfg.width,
                                     (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_indentation");
}

int tac_contact_blur(const tac_ctx* c, const float* in, int32_t input_kind, float* blurred,
                     float* summary, void* workspace, int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (input_kind != TAC_INPUT_DEPTH && input_kind != TAC_INPUT_INDENTATION)
    return fail(TAC_ERR_INVALID, "unknown input_kind %d", input_kind);
  if (n_env && (!in || !blurred)) return fail(TAC_ERR_INVALID, "null buffer");
  if (summary && !workspace) return fail(TAC_ERR_INVALID, "summary needs a workspace");
  FrameParams p = c->blur;
  p.in = in;
  p.use_tma = tma_ok(p, in);
  p.input_depth = input_kind == TAC_INPUT_DEPTH;
  p.blurred = blurred;
  p.n_env = n_env;
  p.finalize = summary ? 1 : 0;
  p.summary = summary;
  cudaError_t e = summary ? bind_workspace(c, p, workspace, n_env, (cudaStream_t)stream) : cudaSuccess;
  if (e == cudaSuccess) e = launch_frame(p, kModeBlur, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_contact_blur");
}

int tac_normals(const tac_ctx* c, const float* elev, float* normals, int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!elev || !normals)) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_normals(elev, normals, c->cfg.height, c->cfg.width, c->fused.inv_p,
                                 c->fused.inv_2p, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_normals");
}

int tac_shade_ex(const tac_ctx* c, const float* blurred, uint8_t* rgb, uint32_t* saturated, int64_t n_env,
                 void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!blurred || !rgb)) return fail(TAC_ERR_INVALID, "null buffer");
  FrameParams p = c->fused;
  p.n_env = n_env;
  cudaError_t e = launch_shade(p, blurred, rgb, saturated, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_shade");
}

int tac_shade(const tac_ctx* c, const float* blurred, uint8_t* rgb, int64_t n_env, void* stream) {
  return tac_shade_ex(c, blurred, rgb, nullptr, n_env, stream);
}

int tac_contact(const tac_ctx* c, const float* in, int32_t input_kind, double* contact,
                float* summary, void* workspace, int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (input_kind != TAC_INPUT_DEPTH && input_kind != TAC_INPUT_INDENTATION)
    return fail(TAC_ERR_INVALID, "unknown input_kind %d", input_kind);
  if (n_env && !in) return fail(TAC_ERR_INVALID, "null buffer");
  if (!workspace) return fail(TAC_ERR_INVALID, "tac_contact needs a workspace");
  FrameParams p = c->contact;
  p.in = in;
  p.use_tma = tma_ok(p, in);
  p.input_depth = input_kind == TAC_INPUT_DEPTH;
  p.n_env = n_env;
  p.finalize = 1;
  p.summary = summary;
  p.contact = contact;
  cudaError_t e = bind_workspace(c, p, workspace, n_env, (cudaStream_t)stream);
  if (e == cudaSuccess) e = launch_frame(p, kModeContact, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_contact");
}

int tac_track_load(const tac_ctx* c, double* state, const double* pose_delta, const double* contact,
                   int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!state || !pose_delta || !contact)) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_track_load(state, pose_delta, contact, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_track_load");
}

int tac_marker_displacements(const tac_ctx* c, const double* loads, float* disp, int64_t n_env,
                             void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!loads || !disp)) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_marker_displacements(c->mg, loads, disp, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_marker_displacements");
}

int tac_render_markers(const tac_ctx* c, const float* disp, uint8_t* rgb, int64_t n_env,
                       void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (n_env && (!disp || !rgb)) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_render_markers(c->mg, disp, rgb, n_env, (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_render_markers");
}

int tac_shadow(const tac_ctx* c, const float* in, int32_t input_kind, float* factor, float* rgb,
               int64_t n_env, void* stream) {
  int st = common_checks(c, n_env);
  if (st) return st;
  if (input_kind != TAC_INPUT_DEPTH && input_kind != TAC_INPUT_INDENTATION)
    return fail(TAC_ERR_INVALID, "unknown input_kind %d", input_kind);
  if (n_env && !in) return fail(TAC_ERR_INVALID, "null buffer");
  cudaError_t e = launch_shadow(c->shadow, in, input_kind == TAC_INPUT_DEPTH, factor, rgb, n_env,
                                (cudaStream_t)stream);
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_shadow");
}

int tac_pipeline(const tac_ctx* c, const tac_pipeline_args* a, void* stream) {
  if (!a) return fail(TAC_ERR_INVALID, "null args");
  if (a->struct_size != sizeof(tac_pipeline_args))
    return fail(TAC_ERR_INVALID, "tac_pipeline_args.struct_size is %u, this library expects %zu",
                a->struct_size, sizeof(tac_pipeline_args));
  int st = common_checks(c, a->n_env);
  if (st) return st;
  if (a->input_kind != TAC_INPUT_DEPTH && a->input_kind != TAC_INPUT_INDENTATION)
    return fail(TAC_ERR_INVALID, "unknown input_kind %d", a->input_kind);
  if (a->n_env && (!a->in || !a->rgb)) return fail(TAC_ERR_INVALID, "in and rgb are required");
  if (!a->workspace) return fail(TAC_ERR_INVALID, "tac_pipeline needs a workspace");
  if (a->load_mode == TAC_LOAD_GIVEN) {
    if (a->n_env && (!a->shear || !a->twist)) return fail(TAC_ERR_INVALID, "shear and twist are required");
  } else if (a->load_mode == TAC_LOAD_TRACK) {
    if (a->n_env && (!a->state || !a->pose_delta))
      return fail(TAC_ERR_INVALID, "state and pose_delta are required");
  } else {
    return fail(TAC_ERR_INVALID, "unknown load_mode %d", a->load_mode);
  }
  FrameParams p = c->fused;
  const bool tma = tma_ok(p, a->in);
  const bool v5 = c->use5 && tma;
  if (v5) p = c->fused5;
  p.in = a->in;
  p.use_tma = tma;
  p.input_depth = a->input_kind == TAC_INPUT_DEPTH;
  p.rgb = a->rgb;
  p.blurred = a->blurred;
  p.n_env = a->n_env;
  p.finalize = 2;
  p.summary = a->summary;
  p.contact = a->contact;
  p.load_mode = a->load_mode;
  p.shear = a->shear;
  p.twist = a->twist;
  p.state = a->state;
  p.pose_delta = a->pose_delta;
  p.disp = a->disp;
  p.splat = a->splat;
  p.saturated = a->saturated;
  if (a->saturated && a->n_env > 0) {
    if (!v5)
      return fail(TAC_ERR_UNSUPPORTED, "the saturation count needs the two-kernel path (this frame uses the fused kernel)");
    cudaError_t z = cudaMemsetAsync(a->saturated, 0, sizeof(uint32_t) * a->n_env, (cudaStream_t)stream);
    if (z != cudaSuccess) return cuda_fail(z, "tac_pipeline");
  }
  p.shadow = a->shadow;
  // diagnostics timeline (tac_timing_begin .. tac_timing_end)
  Marks tm;
  auto& tg = c->timing;
  if (tg.on && (int)tg.calls.size() < tg.max_calls && tg.next < (int)tg.ev.size()) {
    tm.ev = tg.ev.data() + tg.next;
    tm.kind = tg.kind.data() + tg.next;
    tm.cap = (int)tg.ev.size() - tg.next;
    tm.s = (cudaStream_t)stream;
  }
  cudaError_t e;
  // the add_shadows march runs here when the context has shadows on and the
  // caller gave no factor (REF/envs.py:1173 runs it on every observation)
  float* shadow_ws = nullptr;
  if (c->shadow.n_lights > 0 && a->shadow == nullptr)
    shadow_ws = reinterpret_cast<float*>(reinterpret_cast<char*>(a->workspace) + v3_workspace_bytes(c, a->n_env) +
                                         v5_workspace_bytes(c, a->n_env));
  if (v5) {
    bind_workspace5(c, p, a->workspace, a->n_env);
    e = launch_frame5(p, (cudaStream_t)stream, &tm, shadow_ws ? &c->shadow : nullptr, shadow_ws);
  } else {
    e = bind_workspace(c, p, a->workspace, a->n_env, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "tac_pipeline");
    tm.start();
    if (shadow_ws) {
      e = launch_shadow(c->shadow, a->in, p.input_depth, shadow_ws, nullptr, a->n_env, (cudaStream_t)stream);
      if (e != cudaSuccess) return cuda_fail(e, "tac_pipeline (shadows)");
      tm.mark(3);
      p.shadow = shadow_ws;
    }
    e = launch_frame(p, kModeFused, (cudaStream_t)stream);
    tm.mark(0);
  }
  if (tm.on() && tm.n > 1) {
    tg.calls.emplace_back(tg.next, tm.n);
    tg.next += tm.n;
  }
  return e == cudaSuccess ? TAC_OK : cuda_fail(e, "tac_pipeline");
}

int32_t tac_pipeline_path(const tac_ctx* c) {
  if (!c) return -1;
  return c->path;
}

int32_t tac_pipeline_launches(const tac_ctx* c, int64_t n_env) {
  if (!c || n_env < 0) return 0;
  if (c->use5) {
    FrameParams p = c->fused5;
    p.chunk = std::min<long long>(n_env, c->chunk5);
    p.finalize = 2;
    return frame5_launches(p, n_env);
  }
  return n_env > 0 ? 1 : 0;
}

int tac_timing_begin(const tac_ctx* c, int32_t max_calls) {
  if (!c) return fail(TAC_ERR_INVALID, "null context");
  if (max_calls < 1) return fail(TAC_ERR_INVALID, "max_calls must be >= 1");
  int st = check_device(c);
  if (st) return st;
  auto& tg = c->timing;
  // room for 2 launches per env chunk + 4 per call (shadow, epilogue, start)
  const size_t want = (size_t)max_calls * 24;
  while (tg.ev.size() < want) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) return cuda_fail(r, "cudaEventCreate");
    tg.ev.push_back(e);
  }
  tg.kind.assign(tg.ev.size(), -1);
  tg.calls.clear();
  tg.next = 0;
  tg.max_calls = max_calls;
  tg.on = true;
  return TAC_OK;
}

int tac_timing_end(const tac_ctx* c, float* kernel_ms, int32_t* calls) {
  if (!c || !kernel_ms || !calls) return fail(TAC_ERR_INVALID, "null argument");
  auto& tg = c->timing;
  tg.on = false;
  for (int k = 0; k < kTimingKinds; ++k) kernel_ms[k] = 0.f;
  *calls = (int32_t)tg.calls.size();
  if (tg.calls.empty()) return TAC_OK;
  cudaError_t r = cudaEventSynchronize(tg.ev[tg.next - 1]);
  if (r != cudaSuccess) return cuda_fail(r, "cudaEventSynchronize");
  double sum[kTimingKinds] = {0, 0, 0, 0};
  for (const auto& cl : tg.calls)
    for (int i = cl.first + 1; i < cl.first + cl.second; ++i) {
      float ms = 0.f;
      r = cudaEventElapsedTime(&ms, tg.ev[i - 1], tg.ev[i]);
      if (r != cudaSuccess) return cuda_fail(r, "cudaEventElapsedTime");
      if (tg.kind[i] >= 0 && tg.kind[i] < kTimingKinds) sum[tg.kind[i]] += ms;
    }
  for (int k = 0; k < kTimingKinds; ++k) kernel_ms[k] = (float)(sum[k] / tg.calls.size());
  tg.calls.clear();  // reported once
  tg.next = 0;
  return TAC_OK;
}

int tac_pipeline_profile(const tac_ctx* c, const tac_pipeline_args* a, void* stream, int32_t iters,
                         float* kernel_ms) {
  if (!kernel_ms || iters < 1) return fail(TAC_ERR_INVALID, "kernel_ms and iters >= 1 are required");
  int st = tac_timing_begin(c, iters);
  if (st) return st;
  for (int i = 0; i < iters; ++i) {
    st = tac_pipeline(c, a, stream);
    if (st) {
      c->timing.on = false;
      return st;
    }
  }
  int32_t n = 0;
  return tac_timing_end(c, kernel_ms, &n);
}

}  // extern "C"
