/*
 * tac_b200 — C ABI of the B200-native tactile-image path.
 *
 * Drop-in boundary for the per-sensor sensing layer of the reference
 * `tacsim` package (REF = /root/reference/pkg/src/tacsim).  The reference has
 * no FFI: its operator API is plain module functions on NumPy arrays,
 * re-exported at REF/__init__.py:59-81 and called per sensor by
 * Environment._observe (REF/envs.py:1156-1209) and cmd_render
 * (REF/cli.py:274-301).  Each entry point below replaces one of those
 * functions, batched over a leading env dimension; INTEGRATION.md shows the
 * ctypes binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (CUDA global memory), dense,
 *     row-major, with the leading dimension N = n_env.  fp32 unless noted.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *     only enqueues work; nothing synchronises the host.
 *   - The caller owns every buffer.  The library never allocates per call.
 *     Calls that reduce over a frame take a `workspace` of
 *     tac_workspace_bytes(ctx, n_env) bytes (device memory, contents
 *     irrelevant: every call initialises what it uses on its own stream, so
 *     a workspace can be reused by later calls of any size).  Calls running
 *     concurrently need distinct workspaces.
 *   - A context is immutable after creation: calls are reentrant across
 *     host threads and streams.  The only exception is the diagnostics pair
 *     tac_timing_begin / tac_timing_end (one timing session per context).
 *   - Structs passed by pointer start with `struct_size` = sizeof(struct);
 *     a mismatch returns TAC_ERR_INVALID instead of reading past the
 *     caller's struct.
 *   - Return value: TAC_OK or an error status; tac_last_error() returns a
 *     thread-local message for the last failing call on this thread.  The
 *     error classes mirror REF/errors.py:6-11 (InvalidArgumentError).
 *   - There is no CPU fallback inside the library.
 */
#ifndef TAC_B200_H
#define TAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAC_ABI_VERSION 2
#define TAC_MAX_LEVELS 8
#define TAC_MAX_RADIUS 24
#define TAC_MAX_LIGHTS 4
#define TAC_MAX_SHADOW_STEPS 256

enum {
  TAC_OK = 0,
  TAC_ERR_INVALID = 1,     /* precondition violated  -> InvalidArgumentError */
  TAC_ERR_CUDA = 2,        /* CUDA runtime error     -> RuntimeError */
  TAC_ERR_UNSUPPORTED = 3  /* valid but unsupported configuration */
};

/* Input kinds for entry points that accept either map. */
enum {
  TAC_INPUT_DEPTH = 0,       /* HeightMap values: depth from the camera plane (REF/tactile.py:72-87) */
  TAC_INPUT_INDENTATION = 1  /* IndentationMap values: penetration >= 0 (REF/tactile.py:90-107) */
};

/* LUT storage precision (tac_config.lut_dtype).  F32 is exact; F16 halves
 * the shade kernel's gather bytes (15 coefficients in one 32-B sector per
 * bin) at <= 2^-11 relative error per coefficient. */
enum {
  TAC_LUT_F32 = 0,
  TAC_LUT_F16 = 1
};

/* Kernel selection for tac_pipeline (tac_config.kernel_path). */
enum {
  TAC_PATH_AUTO = 0,   /* fastest eligible path (see tac_pipeline_path) */
  TAC_PATH_BAND = 1,   /* band-tiled blur + band shade (W <= 320, R <= 16) */
  TAC_PATH_FUSED = 2,  /* strip-streaming fused frame kernel (any shape) */
  TAC_PATH_STREAM = 3  /* row-streaming blur + band shade (W % 16 == 0, the pyramids
                          tac_stream.cu is instantiated for) */
};

/* Load sources for the marker stage of tac_pipeline. */
enum {
  TAC_LOAD_GIVEN = 0, /* shear[N,2] (m) and twist[N] (rad) supplied per env */
  TAC_LOAD_TRACK = 1  /* track_load: state[N,8] advanced by pose_delta[N,3] */
};

/*
 * Sensor + optical + marker configuration, uploaded once by tac_ctx_create.
 * Field sources: SensorConfig REF/tactile.py:31-69; smooth_pyramid levels
 * REF/tactile.py:200-222; PolyTable / binned LUT REF/optical.py:97-135;
 * MarkerParams REF/marker.py:25-40; DEFAULT_CONTACT_THRESHOLD REF/marker.py:22;
 * render_markers REF/marker.py:203-234.
 */
typedef struct tac_config {
  uint32_t struct_size;     /* = sizeof(tac_config); tac_ctx_create rejects any other
                               value (a caller built against a different header) */
  int32_t height, width;    /* image_size (H, W); both >= 2 */
  double pixel_pitch;       /* m per pixel (square pixels) */
  double gel_thickness;     /* rest surface depth, m */

  int32_t n_levels;                  /* 1..TAC_MAX_LEVELS */
  double sigma[TAC_MAX_LEVELS];      /* px; ignored when radius == 0 */
  int32_t radius[TAC_MAX_LEVELS];    /* 0..TAC_MAX_RADIUS; 0 = identity level (k == 1) */

  int32_t mag_bins, dir_bins;        /* LUT bins (125 x 180 in BASELINE configs) */
  double g_max;                      /* gradient magnitude mapped to the last magnitude bin */
  const float* lut;        /* HOST [mag_bins][dir_bins][3][6] fp32, 8-bit units; c0 unused */
  const float* background; /* HOST [H][W][3] fp32, 8-bit units */

  int32_t marker_rows, marker_cols;  /* marker_grid */
  const double* rest_grid; /* HOST [rows][cols][2] m, or NULL = grid_rest_positions (REF/marker.py:93-100) */
  double k_n, lambda_n, lambda_s, k_t, lambda_t; /* MarkerParams */
  double contact_threshold;          /* > 0 */
  int32_t dot_radius;                /* 0..12 */
  uint8_t dot_color[3];

  /* add_shadows (REF/optical.py:261-300).  shadow_factor == 1.0 disables the
   * stage (the reference's exact identity, REF/optical.py:281-282). */
  int32_t n_lights;                          /* 0..TAC_MAX_LIGHTS */
  double light_dir[TAC_MAX_LIGHTS][3];       /* surface -> light, any length */
  double shadow_factor;                      /* in [0, 1] */
  int32_t shadow_steps;                      /* max_steps, 1..TAC_MAX_SHADOW_STEPS */
  double shadow_softness;                    /* soft-edge width, m, > 0 */

  /* Execution choices (0 = library default).  They change speed, never the
   * arithmetic, except lut_dtype (see TAC_LUT_*). */
  int32_t lut_dtype;                         /* TAC_LUT_* */
  int32_t kernel_path;                       /* TAC_PATH_* */
  int32_t chunk_envs;                        /* envs per blur/shade launch pair; 0 = as many as
                                                fit a 10 GiB blurred scratch */
} tac_config;

typedef struct tac_ctx tac_ctx;
typedef struct tac_pipeline_args tac_pipeline_args; /* defined with tac_pipeline below */

/* Build a context: validates `cfg`, uploads the LUT (repacked), background,
 * quantised background, Gaussian taps and marker grid to the current device. */
int tac_ctx_create(const tac_config* cfg, tac_ctx** out);
int tac_ctx_destroy(tac_ctx* ctx);
const char* tac_last_error(void);
/* Bytes of workspace needed by reducing calls for n_env envs. */
size_t tac_workspace_bytes(const tac_ctx* ctx, int64_t n_env);
/* Tiles per frame used by the frame kernels (for diagnostics). */
int32_t tac_tiles_per_frame(const tac_ctx* ctx);
/* Diagnostics: TAC_PATH_* that tac_pipeline takes for 16-B aligned input. */
int32_t tac_pipeline_path(const tac_ctx* ctx);
/* Diagnostics: number of kernel launches one tac_pipeline call makes for n_env. */
int32_t tac_pipeline_launches(const tac_ctx* ctx, int64_t n_env);
/* Diagnostics: per-kernel timing.  kernel_ms has TAC_TIMING_KINDS slots:
 * [0] = blur (or the fused frame kernel), [1] = shade, [2] = per-env
 * epilogue, [3] = shadow march (0 when a kind does not run). */
#define TAC_TIMING_KINDS 4
/* Runs tac_pipeline `iters` times inside a timing session (below) and writes
 * the mean per-call milliseconds of each kernel kind. */
int tac_pipeline_profile(const tac_ctx* ctx, const tac_pipeline_args* args, void* stream,
                         int32_t iters, float* kernel_ms);
/* Between tac_timing_begin and tac_timing_end, the first max_calls
 * tac_pipeline calls on this context record CUDA events at their kernel
 * boundaries on the call's stream (no synchronisation, so a timed loop runs
 * unchanged).  tac_timing_end waits for the last event and writes the mean
 * per-call milliseconds of each kind (summed over a call's env chunks) and
 * the number of calls recorded.  One session per context at a time. */
int tac_timing_begin(const tac_ctx* ctx, int32_t max_calls);
int tac_timing_end(const tac_ctx* ctx, float* kernel_ms, int32_t* calls);

/* render_heightmap (REF/tactile.py:129-190): orthographic z-buffer of
 * camera-frame triangles.  verts: fp64 [N][n_verts][3] (camera frame, one
 * vertex set per env), tris: int32 [n_tris][3] shared by every env (indices
 * < n_verts, not checked on the device), depth out: fp32 [N][H][W] =
 * fp32(reference float64 depth) -- rest where no triangle is hit. */
int tac_render_heightmap(const tac_ctx* ctx, const double* verts, int64_t n_verts,
                         const int32_t* tris, int64_t n_tris, float* depth,
                         int64_t n_env, void* stream);

/* indentation_from (REF/tactile.py:193-197): ind = clip(rest - depth, 0, rest).
 * depth, ind: [N,H,W]. */
int tac_indentation(const tac_ctx* ctx, const float* depth, float* ind,
                    int64_t n_env, void* stream);

/* Kernel (a): indentation_from + smooth_pyramid (REF/tactile.py:193-222) with
 * the context's levels.  in: [N,H,W] of `input_kind`; blurred: [N,H,W].
 * summary (nullable): [N,8] contact summary as tac_contact. */
int tac_contact_blur(const tac_ctx* ctx, const float* in, int32_t input_kind,
                     float* blurred, float* summary, void* workspace,
                     int64_t n_env, void* stream);

/* normals_from (REF/optical.py:138-163) of an elevation map (IndentationMap
 * values): elev [N,H,W] -> normals [N,H,W,3]. */
int tac_normals(const tac_ctx* ctx, const float* elev, float* normals,
                int64_t n_env, void* stream);

/* Kernel (b): gradient -> bins -> LUT -> + background -> uint8 (shade,
 * REF/optical.py:233-250, with the binned LUT of DESIGN.md §3 and the uint8
 * rule of REF/cli.py:134-139).  blurred [N,H,W] -> rgb [N,H,W,3] uint8. */
int tac_shade(const tac_ctx* ctx, const float* blurred, uint8_t* rgb,
              int64_t n_env, void* stream);
/* tac_shade plus, per env, the number of channel values the [0, 255] clip
 * changed (the reference's `raw != clip(raw)` count behind its >1 %
 * saturation warning, REF/optical.py:246-249).  saturated: uint32 [N] (zeroed
 * here), nullable. */
int tac_shade_ex(const tac_ctx* ctx, const float* blurred, uint8_t* rgb, uint32_t* saturated,
                 int64_t n_env, void* stream);

/* contact_center (REF/marker.py:103-121) on the raw (unsmoothed) map.
 * contact (nullable): fp64 [N,8] LoadState layout (below) with shear/twist 0,
 *   exactly what the reference returns;
 * summary (nullable): fp32 [N,8] = {in_contact, area m^2, c_x m, c_y m,
 *   d_c m, force proxy m^3 (sum of indentation * p^2 over the contact mask),
 *   number of non-finite inputs, clipped channel values (tac_pipeline with
 *   a `saturated` output, else 0)}. */
int tac_contact(const tac_ctx* ctx, const float* in, int32_t input_kind,
                double* contact, float* summary, void* workspace, int64_t n_env,
                void* stream);

/* LoadState layout (REF/marker.py:43-70), fp64 [N,8]:
 *   {c_x, c_y, d_c, s_x, s_y, twist, in_contact (0/1), 0}. */

/* track_load (REF/marker.py:124-140).  state fp64 [N,8] in/out (LoadState);
 * pose_delta fp64 [N,3] = {dt_x, dt_y, rotvec_z} of the case pose delta;
 * contact fp64 [N,8] from tac_contact. */
int tac_track_load(const tac_ctx* ctx, double* state, const double* pose_delta,
                   const double* contact, int64_t n_env, void* stream);

/* marker_displacements (REF/marker.py:143-165).  loads fp64 [N,8]
 * (LoadState) -> disp fp32 [N,rows,cols,2] (m). */
int tac_marker_displacements(const tac_ctx* ctx, const double* loads, float* disp,
                             int64_t n_env, void* stream);

/* render_markers dot splat (REF/marker.py:203-234, arrows excluded): draws
 * filled dots of the context radius / colour at rest + disp into rgb. */
int tac_render_markers(const tac_ctx* ctx, const float* disp, uint8_t* rgb,
                       int64_t n_env, void* stream);

/* add_shadows (REF/optical.py:261-300): per light, march max_steps pixels
 * toward the light over the elevation (-depth, or the indentation for
 * TAC_INPUT_INDENTATION), occ = max_s(elev(p + o_s) - elev(p) - s * rise),
 * weight = clip(occ / softness, 0, 1), factor *= 1 - (1 - shadow_factor) * weight.
 * in: [N,H,W]; factor (nullable): [N,H,W] fp32 product over lights;
 * rgb (nullable): [N,H,W,3] fp32 multiplied in place. */
int tac_shadow(const tac_ctx* ctx, const float* in, int32_t input_kind, float* factor,
               float* rgb, int64_t n_env, void* stream);

/* The whole path in one call (on aligned frames of <= 320 columns: a band
 * blur kernel, a band shade kernel and a per-env epilogue, see
 * tac_pipeline_launches; otherwise one fused kernel).  depth -> rgb (with
 * dots), disp, summary (+ optional blurred) for every env.  No host
 * synchronisation, no allocation: CUDA-graph capturable.  Equivalent to, per env:
 * indentation_from -> smooth_pyramid -> shade -> uint8 ; contact_center ->
 * (given load | track_load) -> marker_displacements -> render_markers. */
struct tac_pipeline_args {
  uint32_t struct_size;     /* = sizeof(tac_pipeline_args) */
  const float* in;          /* [N,H,W] */
  int32_t input_kind;       /* TAC_INPUT_* */
  int32_t load_mode;        /* TAC_LOAD_* */
  const double* shear;      /* fp64 [N,2] m   (TAC_LOAD_GIVEN) */
  const double* twist;      /* fp64 [N]   rad (TAC_LOAD_GIVEN) */
  double* state;            /* fp64 [N,8] LoadState (TAC_LOAD_TRACK, in/out) */
  const double* pose_delta; /* fp64 [N,3] (TAC_LOAD_TRACK) */
  uint8_t* rgb;             /* [N,H,W,3] out */
  float* disp;              /* [N,rows,cols,2] out, nullable */
  float* summary;           /* [N,8] out, nullable (tac_contact layout) */
  double* contact;          /* fp64 [N,8] out, nullable (tac_contact layout) */
  float* blurred;           /* [N,H,W] out, nullable (parity/debug) */
  const float* shadow;      /* [N,H,W] shadow factor (e.g. from tac_shadow), nullable: with
                               shadows on in the context the call runs the march itself */
  int32_t splat;            /* nonzero: draw marker dots into rgb */
  uint32_t* saturated;      /* [N] out, nullable: channel values the [0, 255] clip changed (the
                               count behind REF/optical.py:246-249's >1 % warning); also
                               written to summary field 7 */
  void* workspace;
  int64_t n_env;
};

int tac_pipeline(const tac_ctx* ctx, const tac_pipeline_args* args, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TAC_B200_H */
