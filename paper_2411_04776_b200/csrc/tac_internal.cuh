// Internal device-side structures shared by the kernels and the C ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tac_b200.h"

// Debug bounds checks (build with -DTAC_DEBUG_CHECKS: `make CHECKS=1` ->
// libtac_b200_checks.so): a failed index check traps the kernel, so the call
// returns a CUDA error and the test fails.  compute-sanitizer is closed on the
// GPU pool; this build runs the GPU suite with every shared-memory and global
// index of the hot kernels checked.  Compiled out otherwise.
#ifdef TAC_DEBUG_CHECKS
#define TAC_CHECK(cond)      \
  do {                       \
    if (!(cond)) __trap();   \
  } while (0)
#else
#define TAC_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace tac {

// Strip-streaming frame kernel geometry (see tac_frame.cu).
constexpr int RB = 16;        // rows per row block (vertical-pass register block)
constexpr int KH = 16;        // horizontal-pass outputs per thread
constexpr int kThreads = 320; // threads per group (= 320 columns of a 320-wide strip)
#ifndef TAC_SHADE_WARPS
#define TAC_SHADE_WARPS 10
#endif
constexpr int kShadeThreads = 32 * TAC_SHADE_WARPS;  // shade group of the fused kernel
constexpr int kSlots = 3;      // blurred ring slots: blur runs up to two row blocks ahead of shading
constexpr int kRing = kSlots * RB;
constexpr int kSumFields = 8; // per-strip partial / per-env summary width

// Frame-kernel modes.
enum FrameMode : int {
  kModeBlur = 0,     // kernel (a) alone: writes blurred
  kModeFused = 1,    // kernel (a)+(b): blurred stays in smem, writes uint8 RGB
  kModeContact = 2,  // reduction only (contact_center)
};

// Marker geometry + model constants (REF/marker.py:25-40, :93-100, :203-234).
struct MarkerGeom {
  int H, W;
  double pitch;
  int rows, cols;
  const double* rest_grid;  // device [rows*cols][2] m
  double k_n, lambda_n, lambda_s, k_t, lambda_t;
  int dot_radius;
  unsigned char dot_r, dot_g, dot_b;
};

// Everything a frame kernel needs, passed by value (constant bank).
struct FrameParams {
  // geometry
  int H, W;
  int strips;            // column strips per frame (CTAs per env)
  int strip_w;           // output columns per strip (multiple of 16 unless W is smaller)
  int R;                 // max radius over levels (vertical halo rows)
  int in_rows, in_pitch; // input buffer: in_rows x in_pitch floats
  int v_pitch;           // vertical-pass buffer: RB x v_pitch floats (odd pitch)
  int b_pitch;           // blurred ring: kRing x b_pitch floats (multiple of 4, 4 x odd)
  int stage_bytes;       // uint8 RGB staging of the shade group
  int use_tma;           // rows 16-B aligned -> cp.async.bulk row loads
  // pyramid
  int n_levels;
  int radius[TAC_MAX_LEVELS];
  float wv[TAC_MAX_LEVELS][TAC_MAX_RADIUS + 1];  // vertical taps, centre first
  float wh[TAC_MAX_LEVELS][TAC_MAX_RADIUS + 1];  // horizontal taps, folded with 1/L
  float2 wv2[TAC_MAX_LEVELS][TAC_MAX_RADIUS + 1];  // (w, w) pairs of wv / wh for FFMA2
  float2 wh2[TAC_MAX_LEVELS][TAC_MAX_RADIUS + 1];
  // clamp / contact
  float rest;            // gel thickness rounded to fp32
  float rest_lo;         // rest - (double)rest: the clamp runs in ~fp64 accuracy
  float threshold;
  float half_w, half_h;  // W/2, H/2 (pixel-centre coordinates)
  double xoff, yoff;     // 0.5 - W/2, 0.5 - H/2: pixel-centre coordinate of column / row 0
  // shading
  float inv_p, inv_2p;
  float mag_scale;       // mag_bins / g_max
  float dir_scale;       // dir_bins / (2 pi)
  int mag_bins, dir_bins;
  const float4* lut;     // [mag*dir][4] float4 = c1..c5 per channel (15 used)
  const float* bg;       // [H][W][3] 8-bit units
  const uint8_t* bg_u8;  // [H][W][3] = clamp(rint(bg))
  const float* lut_half;     // [2][nbins][8]: plane h holds floats 8h..8h+7 of every bin
  unsigned long long lut_tex;  // cudaTextureObject_t over lut_half as float4 texels (0 = none)
  const float* bg_planar;    // [3][H][W]
  const uint4* lut_h16;      // lut_dtype f16: [nbins][2] uint4 = 16 fp16 (15 used), direction-major; else null
  int nbins;
  // io
  const float* in;
  int input_depth;
  float* blurred;        // nullable
  uint8_t* rgb;          // fused mode
  double* partials;      // workspace [N][strips][8]
  unsigned int* counters;// workspace [N]
  long long n_env;
  // finalize
  int finalize;          // 0 none, 1 contact/summary, 2 + markers
  float* summary;        // nullable [N][8]
  double* contact;       // nullable [N][8] fp64 LoadState
  // markers
  MarkerGeom mg;
  int load_mode;
  const double* shear;
  const double* twist;
  double* state;
  const double* pose_delta;
  float* disp;           // nullable
  int splat;
  const float* shadow;   // nullable [N][H][W] multiplicative shadow factor
  unsigned int* saturated;  // nullable [N]: clipped channel values per env (zeroed per call)
  // band-tiled two-kernel path (tac_frame5.cu)
  int bands;             // ceil(H / 16)
  long long chunk;       // envs per (blur, shade) launch pair
  int2* band_ext;        // workspace [chunk][bands][ext_strips] blurred non-zero column range
  float* scratch;        // workspace [chunk][H][W] blurred (or the caller's blurred output)
  int ext_strips;        // band_ext entries per band (column strips of the blur kernel)
  int nparts;            // contact partials per env (reduced by env_epilogue_kernel)
  // row-streaming blur (tac_stream.cu)
  int st_kind;           // pyramid instantiation (stream_kind); -1 = not eligible
  int st_strips;         // column strips per frame (CTAs per env)
  int st_ip;             // input slot row pitch (floats)
  int st_rpp;            // V buffer row-pair pitch (floats)
  int st_nvw, st_nhw;    // V / H warps per CTA
};

// In-stream kernel-boundary events of one tac_pipeline call (diagnostics):
// start() before the first launch, mark(kind) after each launch; the time
// between consecutive events is charged to the kind of the later one.  Kinds:
// 0 = blur (or a fused frame kernel), 1 = shade, 2 = per-env epilogue,
// 3 = shadow march.  No synchronisation: a timed loop runs unchanged.
constexpr int kTimingKinds = 4;
struct Marks {
  cudaEvent_t* ev = nullptr;  // pool slots [0, cap)
  int* kind = nullptr;
  int cap = 0, n = 0;
  cudaStream_t s = nullptr;
  bool on() const { return ev != nullptr; }
  void start() { put(-1); }
  void mark(int k) { put(k); }
  void put(int k) {
    if (!ev) return;
    if (n >= cap) {  // out of slots: this call is dropped (tac_timing_end counts complete calls)
      ev = nullptr;
      n = -1;
      return;
    }
    cudaEventRecord(ev[n], s);
    kind[n++] = k;
  }
};

// add_shadows march tables (REF/optical.py:283-299), built on the host.
constexpr int kShadowTH = 24, kShadowTW = 160;  // tiled march: output tile of one CTA
struct ShadowParams {
  int H, W;
  int n_lights, steps;
  const int2* off;       // [n_lights * steps] (di, dj)      (L1 fallback kernel)
  const float* cost;     // [n_lights * steps] s * pitch * lz / lateral
  float one_minus_factor;
  float inv_softness;
  int di_min, di_max, dj_min, dj_max;  // offset bounds over all lights (interior fast path)
  // tiled march: per light the tile's offset-range region [rh x rw] in smem
  int tiled;                            // 1: smem-tiled kernel (region fits)
  int l_di_min[TAC_MAX_LIGHTS], l_dj_min[TAC_MAX_LIGHTS];
  int l_rh[TAC_MAX_LIGHTS], l_rw[TAC_MAX_LIGHTS];
  int offb[TAC_MAX_LIGHTS][TAC_MAX_SHADOW_STEPS];    // byte offset of step s inside the light's region
  float costs[TAC_MAX_LIGHTS][TAC_MAX_SHADOW_STEPS]; // s * rise (fp32)
};

cudaError_t launch_shadow(const ShadowParams& s, const float* in, int input_depth, float* factor,
                          float* rgb, long long n_env, cudaStream_t st);

// Row f2: render_heightmap z-buffer (tac_raster.cu)
cudaError_t launch_raster(const double* verts, long long n_verts, const int* tris, int n_tris, float* depth,
                          int H, int W, double pitch, double rest, long long n_env, cudaStream_t s);

size_t frame_smem_bytes(const FrameParams& p);
cudaError_t launch_frame(const FrameParams& p, int mode, cudaStream_t s);
// band-tiled two-kernel path (tac_frame5.cu): one strip, W % 16 == 0, R <= 16
bool frame5_eligible(const FrameParams& p);
bool shade5_eligible(const FrameParams& p);
// sp / shadow_ws (nullable): run the add_shadows march per env chunk into
// shadow_ws (chunk x H x W) before the chunk's blur and shade with it.
cudaError_t launch_frame5(const FrameParams& p, cudaStream_t s, Marks* tm = nullptr, const ShadowParams* sp = nullptr,
                          float* shadow_ws = nullptr);
// row-streaming path (tac_stream.cu): plan (sets st_* / -1 when not
// eligible), smem bytes, and the blur launch of one env chunk.
void plan_stream(FrameParams& p);
size_t stream_smem_bytes(const FrameParams& p);
cudaError_t launch_stream_blur(const FrameParams& p, cudaStream_t s);

int frame5_launches(const FrameParams& p, long long n_env);
int frame5_vpitch(int W, int R4);
cudaError_t launch_indentation(const float* depth, float* ind, float rest, float rest_lo, long long n,
                               cudaStream_t s);
cudaError_t launch_normals(const float* elev, float* normals, int H, int W, float inv_p,
                           float inv_2p, long long n_env, cudaStream_t s);
cudaError_t launch_shade(const FrameParams& p, const float* blurred, uint8_t* rgb, unsigned int* saturated,
                         long long n_env, cudaStream_t s);
cudaError_t launch_track_load(double* state, const double* pose_delta, const double* contact,
                              long long n_env, cudaStream_t s);
cudaError_t launch_marker_displacements(const MarkerGeom& m, const double* loads,
                                        float* disp, long long n_env, cudaStream_t s);
cudaError_t launch_render_markers(const MarkerGeom& m, const float* disp, uint8_t* rgb,
                                  long long n_env, cudaStream_t s);

}  // namespace tac
