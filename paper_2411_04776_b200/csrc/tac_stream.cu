// Row-streaming, warp-specialised blur (kernel (a) of the default tac_pipeline path).
//
// indentation_from + smooth_pyramid (REF/tactile.py:193-222) + the contact
// partials of contact_center (REF/marker.py:103-121) for one env column strip
// (<= 320 output columns) per CTA, walking down the frame in blocks of SB = 8
// rows:
//
//   TMA      thread 0 streams 8-row input blocks into NS smem slots with
//            cp.async.bulk (mbarrier complete_tx), NS - 1 blocks ahead.
//   V warps  one lane per column pair.  Every input row is read from smem
//            ONCE, clamped (REF/tactile.py:195-196), folded into the contact
//            partials and pushed into a register ring of the last P rows.
//            Per output row pair the vertical pass of EVERY level is
//            evaluated from the ring with pair sums shared by the levels,
//            w0 x[y] + sum_t w_t (x[y+t] + x[y-t]): R_max FADD2 +
//            sum_l (R_l + 1) FFMA2 per output row of a column pair (36
//            instead of 45 for sigma 1,2,4), both rows of a pair sharing each
//            uniform-register tap load.  Outputs go to a double-buffered smem
//            block [level][row pair][column] with rows interleaved in pairs,
//            plus a per-row-pair bitmask of the non-zero column pairs.
//            Replicate borders: rows outside the frame are copies of the
//            edge row (ring fill); columns outside it are pads that the last
//            H warp writes (below): the V warps are the critical path.
//   H warps  the last H warp first writes the block's replicate column pads
//            (then an H-only named barrier); one (row pair, 8 columns) item
//            per lane and block, <= 2 items
//            per lane: the item's window of each level is loaded into
//            registers (LDS.128, every FFMA2 operand one aligned float2 of
//            the interleaved block) and convolved tap-outer, summed over the
//            levels, stored to HBM with 16-B stores.  Items whose window is
//            all zero (bitmask) store exact zeros.
//
// V and H warps hand blocks over with named barriers (FULL[s] / EMPTY[s],
// s = block parity); nothing else synchronises the CTA inside the loop.  The
// pyramid radii and the smem pitches are template parameters, so every ring
// index, smem offset and tap is static.
#include <climits>

#include "tac_frame_common.cuh"

namespace tac {

namespace {

constexpr int SB = 8;           // rows per stream block
constexpr int kMaxVW = 8;       // V warps per CTA
constexpr int kMaxStrip = 320;  // output columns per CTA

// barrier ids (0 = __syncthreads)
constexpr int kBarFull = 1;   // + block parity
constexpr int kBarEmpty = 3;  // + block parity
constexpr int kBarPad = 6;    // H warps: replicate pads written
constexpr int kBarV = 5;

template <int L_, int R0, int R1 = 0, int R2 = 0, int R3 = 0>
struct Pyr {
  static constexpr int L = L_;
  static constexpr int r(int l) { return l == 0 ? R0 : l == 1 ? R1 : l == 2 ? R2 : R3; }
  static constexpr int r4(int l) { return (r(l) + 3) & ~3; }
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int R = cmax(cmax(R0, L_ > 1 ? R1 : 0), cmax(L_ > 2 ? R2 : 0, L_ > 3 ? R3 : 0));
  static constexpr int R4 = (R + 3) & ~3;
  static constexpr int P = 2 * R + SB;                      // ring rows: an iteration's 8 outputs need 2R + 8
  static constexpr int NS = 4;                              // input slots: an iteration reads 2 blocks, + 2 ahead
  // 8 warps (4 per SMSP at 2 CTAs/SM: <= 128 registers) when the ring is short;
  // measured: 10 warps with a 96-register cap is 18 % slower
  static constexpr int MINB = (P <= 32 && L <= 3) ? 2 : 1;
  static constexpr int MAXT = MINB == 2 ? 256 : 384;
};

using Pyr0 = Pyr<3, 3, 6, 12>;      // sigma 1, 2, 4 (BASELINE configs[0-2, 4])
using Pyr1 = Pyr<4, 3, 6, 12, 24>;  // sigma 1, 2, 4, 8 (configs[3])
using Pyr2 = Pyr<4, 2, 5, 10, 15>;  // kernel sizes 5, 11, 21, 31 (REF DEFAULT_PYRAMID)
using Pyr3 = Pyr<3, 0, 2, 5>;       // kernel sizes 1, 5, 11

// Compile-time smem geometry of one instantiation: WIDE = frames split into
// column strips (V range = strip + R4 halo columns each side).
template <class PY, bool WIDE>
struct Geo5 {
  static constexpr int IP = (WIDE ? kMaxStrip + 2 * PY::R4 : kMaxStrip);  // input slot row (floats)
  static constexpr int VP0 = IP + 2 * PY::R4;                             // V row: pads + range
  static constexpr int VP = ((VP0 / 2) & 1) ? VP0 : VP0 + 2;              // row-pair pitch 2 VP = 4 x odd
  static constexpr int RPP = 2 * VP;                                      // floats per row pair
  static constexpr int VSLOT = PY::L * (SB / 2) * RPP;                    // floats per V block slot
  static constexpr size_t IN_OFF = 0;
  static constexpr size_t VB_OFF = ((size_t)PY::NS * SB * IP * 4 + 127) & ~size_t(127);
  static constexpr size_t NZ_OFF = VB_OFF + (size_t)2 * VSLOT * 4;
  static constexpr size_t RED_OFF = NZ_OFF + (size_t)2 * (SB / 2) * kMaxVW * 4;
  static constexpr size_t BAR_OFF = RED_OFF + (size_t)kMaxVW * 8 * 8;
  static constexpr size_t END = BAR_OFF + (size_t)PY::NS * 8;
  static size_t bytes(int, int) { return (END + 127) & ~size_t(127); }
};

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// The H item's window of non-zero flags: column pairs [qa, qb] of the V
// range (the widest level's taps around the item's 8 columns) lie in the
// bitmask words w and w + 1 (a window spans <= 2 R4 + 8 <= 56 columns, 28
// pairs); the item is non-zero if (nzs[w] & lo) | (nzs[w + 1] & hi).
struct HWin {
  int w;
  uint32_t lo, hi;
};
template <class PY>
__device__ __forceinline__ HWin h_window(int c0, int vx0, int npairs) {
  constexpr int R4 = PY::R4;
  static_assert(2 * R4 + 8 <= 64, "an H window spans at most two bitmask words");
  const int qa = max((c0 - R4 - vx0) >> 1, 0);
  const int qb = min((c0 + 8 + R4 - vx0) >> 1, npairs) - 1;
  HWin h;
  h.w = qa >> 5;
  const int a = qa & 31, b = max(qb - 32 * h.w, a);  // b in [a, 63]
  h.lo = (~0u << a) & (b >= 31 ? ~0u : ~0u >> (31 - b));
  h.hi = b >= 32 ? ~0u >> (63 - b) : 0u;
  return h;
}

// One H item: row pair m x 8 columns (acc[i] = (row 2m, row 2m+1) at column
// c0 + i) from the V block slot `vs` (column index 0 = global column vx0 - R4).
// Returns false (acc = 0) when the V window of the widest level is all zero.
template <class PY, class G>
__device__ __forceinline__ bool h_item(const FrameParams& p, const float* vs, const uint32_t* nzs, int m, int c0,
                                       int vx0, const HWin& hw, float2 (&acc)[8]) {
  constexpr int L = PY::L, R4 = PY::R4;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  // (hi == 0 when the window ends in word w: word w + 1 is then not read)
  const uint32_t bits = (nzs[hw.w] & hw.lo) | (hw.hi ? nzs[hw.w + 1] & hw.hi : 0u);
  if (bits == 0u) return false;
  // row pair m at column c0 - R4 (16-B aligned: every offset is a multiple of 4 columns)
  const float* base = vs + m * G::RPP + 2 * (c0 - vx0);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int rl_ = PY::r(l), r4l = PY::r4(l);
    float2 v[8 + 2 * PY::R4];
#pragma unroll
    for (int q = 0; q < (8 + 2 * r4l) / 2; ++q) {
      TAC_CHECK(2 * (c0 - vx0) + 2 * (R4 - r4l) + 4 * q >= 0 &&
                2 * (c0 - vx0) + 2 * (R4 - r4l) + 4 * q + 4 <= G::RPP);
      const float4 f = *reinterpret_cast<const float4*>(base + l * (SB / 2) * G::RPP + 2 * (R4 - r4l) + 4 * q);
      v[2 * q] = make_float2(f.x, f.y);
      v[2 * q + 1] = make_float2(f.z, f.w);
    }
    // tap-outer: each uniform-register tap serves the 8 outputs
#pragma unroll
    for (int t = -rl_; t <= rl_; ++t) {
      const float ws = p.wh[l][t < 0 ? -t : t];
      const float2 w = make_float2(ws, ws);  // scalar uniform operand (FFMA2 .F32 broadcast)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = ffma2(w, v[r4l + i + t], acc[i]);
    }
  }
  return true;
}

// Input block b (rows 8b..8b+7, columns [vx0, vx0 + ncols)) -> smem slot
// `dst` with bulk copies completing on `bar`.  Rows past the frame bottom are
// copies of row H-1 (replicate border, REF/tactile.py:220 mode="nearest").
// One thread; out of line: it runs once per block.
__device__ __forceinline__ void stream_issue(const float* src, float* dst, uint64_t* bar, int b, int ip, int H, int W,
                                          int vx0, int ncols) {
  const unsigned rbytes = (unsigned)ncols * 4u;
  mbar_expect_tx(bar, rbytes * (unsigned)SB);
  const float* g = src + vx0;
  if (ncols == W && W == ip && SB * b + SB <= H) {
    bulk_g2s(dst, g + (long long)SB * b * W, rbytes * (unsigned)SB, bar);  // contiguous rows
  } else {
    for (int i = 0; i < SB; ++i) bulk_g2s(dst + i * ip, g + (long long)min(SB * b + i, H - 1) * W, rbytes, bar);
  }
}

// Blocks [next, lim) into their slots (block b -> slot b % ns); returns lim.
__device__ __forceinline__ int stream_refill(const float* src, float* in_s, uint64_t* s_full, int next, int lim, int ns,
                                          int ip, int H, int W, int vx0, int ncols) {
#pragma unroll 1
  for (; next < lim; ++next) {
    const int slot = next % ns;
    stream_issue(src, in_s + slot * SB * ip, &s_full[slot], next, ip, H, W, vx0, ncols);
  }
  return next;
}

// ---------------------------------------------------------------------------
template <class PY, bool WIDE>
__global__ void __launch_bounds__(PY::MAXT, PY::MINB) stream_blur_kernel(const __grid_constant__ FrameParams p) {
  using G = Geo5<PY, WIDE>;
  constexpr int L = PY::L, R = PY::R, R4 = PY::R4, P = PY::P, NS = PY::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const long long env = blockIdx.x;
  const int strip = blockIdx.y;
  const int W = p.W, H = p.H;
  const long long HW = (long long)H * W;
  const int x0 = strip * p.strip_w;
  const int x1 = min(x0 + p.strip_w, W);
  const int vx0 = max(x0 - R4, 0);
  const int vx1 = min(x1 + R4, W);
  const int nvw = p.st_nvw, nhw = p.st_nhw;
  const int nthreads = 32 * (nvw + nhw);
  const int nbands = (H + 15) >> 4;
  const int nblk = (H + SB - 1) / SB;       // output blocks
  // input blocks: the last iteration reads rows up to 8 nblk - 1 + R (copies of row H-1 past the frame)
  const int nblk_in = nblk + (R + SB - 1) / SB;
  float* in_s = reinterpret_cast<float*>(smem_raw + G::IN_OFF);
  float* vb = reinterpret_cast<float*>(smem_raw + G::VB_OFF);
  uint32_t* s_nz = reinterpret_cast<uint32_t*>(smem_raw + G::NZ_OFF);
  double* s_red = reinterpret_cast<double*>(smem_raw + G::RED_OFF);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem_raw + G::BAR_OFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* src = p.in + env * HW;

  // thread 0 streams input block b (rows 8b..8b+7) into slot b % NS
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&s_full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    stream_refill(src, in_s, s_full, 0, min(NS, nblk_in), NS, G::IP, H, W, vx0, vx1 - vx0);
  }
  __syncthreads();

  if (warp < nvw) {
    // ======================= V warps: convert + vertical pass ===================
    const int q = warp * 32 + lane;  // column pair of the V range
    const int c = vx0 + 2 * q;
    const bool act = c < vx1;
    const int cr = act ? c : vx1 - 2;           // inactive lanes read a valid column
    const bool own = act && c >= x0 && c < x1;  // counted in this strip's contact partials
    const float* col = in_s + (cr - vx0);
    float* vcol = vb + 2 * (c - vx0 + R4);  // the pair's float4 in row pair 0, level 0, slot 0
    const float2 rr = make_float2(p.rest, p.rest), rl = make_float2(p.rest_lo, p.rest_lo);
    const float thr = p.threshold;
    const bool depth_in = p.input_depth != 0;
    const bool partials = p.finalize != 0 && own;
    const double yoff = 0.5 - (double)p.half_h;
    float mx = 0.f;
    float2 cnt2 = make_float2(0.f, 0.f);  // contact pixels of the pair's two columns
    float2 probe = make_float2(0.f, 0.f);  // sum of the raw values read (non-finite flag)
    float2 cs = make_float2(0.f, 0.f);  // fp32 column sums of the current input block
    double sw = 0.0, swx = 0.0, swy = 0.0;
    float2 win[P];
    int last_nz = INT_MIN / 2;  // last input row with a non-zero value in the warp's columns (warp-uniform)

    // read + convert one row y from smem slot / row; rows < H are folded into
    // the contact partials (rows >= H are replicas of row H-1)
    auto take = [&](int y, const float* src_row) -> float2 {
      TAC_CHECK(src_row >= in_s && src_row + 2 <= in_s + NS * SB * G::IP && (cr - vx0) + 2 <= G::IP);
      const float2 raw = *reinterpret_cast<const float2*>(src_row);
      float2 v = raw;
      if (depth_in) {
        v = fsubadd2(rr, raw, rl);
        v.x = clampf(v.x, 0.f, p.rest);
        v.y = clampf(v.y, 0.f, p.rest);
      }
      const bool nzw = __any_sync(0xffffffffu, (__float_as_uint(v.x) | __float_as_uint(v.y)) != 0u);
      // raw non-finite values clamp to 0 or rest; a running sum of the raw
      // values becomes non-finite if any is (or on a finite overflow): the
      // strip then flags its env and the epilogue counts them exactly
      // (summary field 6) -- one FADD2 per row instead of a per-row count
      probe = fadd2(probe, raw);
      if (nzw) {
        last_nz = y;
        if (partials && y < H) {
          mx = fmaxf(mx, fmaxf(v.x, v.y));
          // contact mask as 1/0 (v is finite and >= 0: v * 0 = +0, v * 1 = v)
          const float2 f = make_float2(v.x > thr ? 1.f : 0.f, v.y > thr ? 1.f : 0.f);
          const float2 w = fmul2(v, f);
          cnt2 = fadd2(cnt2, f);
          cs = fadd2(cs, w);
          const float rs = w.x + w.y;
          sw += (double)rs;
          swy = fma((double)rs, (double)y + yoff, swy);
        }
      }
      return v;
    };
    auto flush_cols = [&]() {
      if (partials && (cs.x != 0.f || cs.y != 0.f)) {
        const double xc0 = (double)c + p.xoff;
        swx = fma((double)cs.x, xc0, swx);
        swx = fma((double)cs.y, xc0 + 1.0, swx);
      }
      cs = make_float2(0.f, 0.f);
    };

    // ---- prologue: ring rows -R .. R-1 (rows < 0 replicate row 0) ----------
    // ring layout at the start of iteration j: win[t] = row 8j - R + t, t < 2R
#pragma unroll
    for (int y = 0; y < R; ++y) {
      if (y % SB == 0) mbar_wait(&s_full[(y / SB) % NS], ((y / SB) / NS) & 1);
      win[R + y] = take(y, col + ((y / SB) % NS * SB + y % SB) * G::IP);
      if (y == 0) {
#pragma unroll
        for (int t = 0; t < R; ++t) win[t] = win[R];
      }
    }
    flush_cols();

    // ---- main loop: iteration j = output rows 8j..8j+7 = input rows 8j+R.. ---
    // one iteration is unrolled; the ring shifts by 8 rows at its end
#pragma unroll 1
    for (int j = 0; j < nblk; ++j) {
      const int sv = j & 1;
      bar_sync_n(kBarEmpty + sv, nthreads);  // H finished block j-2; all V warps finished j-1
      float* vs = vcol + sv * G::VSLOT;
      uint32_t* nzs = s_nz + sv * (SB / 2) * kMaxVW + warp;
      // input rows 8j+R+i live in blocks b0 = j + R/8 and b0 + 1
      const int b0 = j + R / SB;
      const float* blk0 = col + (b0 % NS) * SB * G::IP;
      const float* blk1 = col + ((b0 + 1) % NS) * SB * G::IP;
#pragma unroll
      for (int k = 0; k < SB / 2; ++k) {
        // push input rows yi = 8j + R + 2k, +1
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * k + h;
          const int rb = (R + i) / SB - R / SB;  // 0: block b0, 1: block b0 + 1
          const int yi = SB * j + R + i;
          if (i == 0 || (R + i) % SB == 0) mbar_wait(&s_full[(b0 + rb) % NS], ((b0 + rb) / NS) & 1);
          win[2 * R + i] = take(yi, (rb ? blk1 : blk0) + ((R + i) % SB) * G::IP);
          if ((R + i) % SB == SB - 1) flush_cols();
        }
        // output rows yo = 8j + 2k (a) and yo + 1 (b): ring index R + 2k
        const int ro = R + 2 * k;
        float2 oa[L], ob[L];
        if (last_nz >= SB * j + 2 * k - R) {  // warp-uniform: a non-zero row in the window
#pragma unroll
          for (int l = 0; l < L; ++l) {
            oa[l] = ffma2(make_float2(p.wv[l][0], p.wv[l][0]), win[ro], make_float2(0.f, 0.f));
            ob[l] = ffma2(make_float2(p.wv[l][0], p.wv[l][0]), win[ro + 1], make_float2(0.f, 0.f));
          }
#pragma unroll
          for (int t = 1; t <= R; ++t) {
            const float2 pa = fadd2(win[ro + t], win[ro - t]);
            const float2 pb = fadd2(win[ro + 1 + t], win[ro + 1 - t]);
#pragma unroll
            for (int l = 0; l < L; ++l)
              if (t <= PY::r(l)) {
                oa[l] = ffma2(make_float2(p.wv[l][t], p.wv[l][t]), pa, oa[l]);
                ob[l] = ffma2(make_float2(p.wv[l][t], p.wv[l][t]), pb, ob[l]);
              }
          }
        } else {
#pragma unroll
          for (int l = 0; l < L; ++l) oa[l] = ob[l] = make_float2(0.f, 0.f);
        }
        // the widest level's window contains every level's: non-negative
        // inputs and positive taps make it zero only if all are
        const bool nz = (__float_as_uint(oa[L - 1].x) | __float_as_uint(oa[L - 1].y) |
                         __float_as_uint(ob[L - 1].x) | __float_as_uint(ob[L - 1].y)) != 0u;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          // rows (2k, 2k+1) x columns (c, c+1)
          TAC_CHECK(!act || (2 * (c - vx0 + R4) >= 0 && 2 * (c - vx0 + R4) + 4 <= G::RPP));
          if (act)
            *reinterpret_cast<float4*>(vs + (l * (SB / 2) + k) * G::RPP) =
                make_float4(oa[l].x, ob[l].x, oa[l].y, ob[l].y);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, act && nz);
        if (lane == 0) nzs[k * kMaxVW] = bal;
      }
      bar_arrive_n(kBarFull + sv, nthreads);
      // shift the ring by the 8 rows consumed
#pragma unroll
      for (int t = 0; t < 2 * R; ++t) win[t] = win[t + SB];
    }
    flush_cols();  // a partial last block
    // ---- contact partials of the strip: V warps only ----------------------------
    if (p.finalize == 0) return;
    Red red;
    red.cnt = cnt2.x + cnt2.y;
    red.mx = mx;
    red.nf = (partials && !(fabsf(probe.x + probe.y) < INFINITY)) ? -1.f : 0.f;  // < 0: recount
    red.sw = sw;
    red.swx = swx;
    red.swy = swy;
    warp_reduce(red);
    if (lane == 0) {
      double* qd = s_red + warp * 8;
      qd[0] = red.cnt;
      qd[1] = red.sw;
      qd[2] = red.swx;
      qd[3] = red.swy;
      qd[4] = red.mx;
      qd[5] = red.nf;
    }
    bar_sync_n(kBarV, 32 * nvw);
    if (threadIdx.x == 0) {
      double t[6] = {0, 0, 0, 0, 0, 0};
      for (int w = 0; w < nvw; ++w) {  // fixed order: deterministic
        for (int i = 0; i < 4; ++i) t[i] += s_red[w * 8 + i];
        t[4] = fmax(t[4], s_red[w * 8 + 4]);
        t[5] += s_red[w * 8 + 5];
      }
      double* qd = p.partials + (env * p.nparts + strip) * kSumFields;
      for (int i = 0; i < 6; ++i) qd[i] = t[i];
    }
  } else {
    // ======================= H warps: horizontal pass + store ===================
    // items = (row pair m, 8-column chunk) of a block; lane ht takes items ht
    // and ht + 32 nhw (the same chunks in every block)
    const int ht = threadIdx.x - 32 * nvw;
    const int nht = 32 * nhw;
    const int nitems = 4 * ((x1 - x0) >> 3);
    const int npairs = (vx1 - vx0) >> 1;
    // the (<= 2) items of this lane and their window masks (the same every block)
    const HWin hw0 = h_window<PY>(x0 + 8 * (ht >> 2), vx0, npairs);
    const HWin hw1 = h_window<PY>(x0 + 8 * ((ht + nht) >> 2), vx0, npairs);
    int next_issue = min(NS, nblk_in);  // (H thread 0) next input block to stream
    bar_arrive_n(kBarEmpty + 0, nthreads);
    if (nblk > 1) bar_arrive_n(kBarEmpty + 1, nthreads);
    for (int j = 0; j < nblk; ++j) {
      const int sv = j & 1;
      bar_sync_n(kBarFull + sv, nthreads);
      if (ht == 0) {
        // every V warp finished iteration j: the input blocks before the first
        // one iteration j+1 reads are free; refill their slots NS blocks ahead
        const int lim = min((SB * (j + 1) + R) / SB + NS, nblk_in);
        if (next_issue < lim)
          next_issue = stream_refill(src, in_s, s_full, next_issue, lim, NS, G::IP, H, W, vx0, vx1 - vx0);
      }
      {
        // the last H warp writes the block's replicate pads (columns left of
        // column 0 / right of column W-1, every level and row pair) from the
        // edge columns the V warps stored; the H warps then sync among
        // themselves (the V warps, the critical path, do no pad work)
        if (warp == nvw + nhw - 1 && (vx0 == 0 || vx1 == W)) {
          float* vblk = vb + sv * G::VSLOT;
#pragma unroll
          for (int l = 0; l < L; ++l) {
            const int np = PY::r4(l) / 2;  // float4 pads per side and row pair
            for (int i = lane; i < 4 * 2 * np; i += 32) {
              const int k = i / (2 * np), rem = i - k * 2 * np, side = rem >= np ? 1 : 0, t = rem - side * np;
              float* lrow = vblk + (l * (SB / 2) + k) * G::RPP;
              if (side == 0 && vx0 == 0) {
                TAC_CHECK(2 * (R4 - 2 * np + 2 * t) >= 0);
                const float2 e = *reinterpret_cast<const float2*>(lrow + 2 * R4);
                *reinterpret_cast<float4*>(lrow + 2 * (R4 - 2 * np + 2 * t)) = make_float4(e.x, e.y, e.x, e.y);
              } else if (side == 1 && vx1 == W) {
                TAC_CHECK(2 * (W - vx0 + R4 + 2 * t) + 4 <= G::RPP);
                const float2 e = *reinterpret_cast<const float2*>(lrow + 2 * (W - 1 - vx0 + R4));
                *reinterpret_cast<float4*>(lrow + 2 * (W - vx0 + R4 + 2 * t)) = make_float4(e.x, e.y, e.x, e.y);
              }
            }
          }
        }
        bar_sync_n(kBarPad, nht);
      }
      const float* vs = vb + sv * G::VSLOT;
#pragma unroll 1
      for (int item = ht; item < nitems; item += nht) {
        const int m = item & 3;
        const int c0 = x0 + 8 * (item >> 2);
        float2 acc[8];
        h_item<PY, G>(p, vs, s_nz + (sv * (SB / 2) + m) * kMaxVW, m, c0, vx0, item == ht ? hw0 : hw1, acc);
        const int y = SB * j + 2 * m;
        TAC_CHECK(c0 >= 0 && c0 + 8 <= W && m >= 0 && m < SB / 2);
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
      if (j + 2 < nblk) bar_arrive_n(kBarEmpty + sv, nthreads);
    }
  }
}

template <class PY, bool WIDE>
cudaError_t launch_kind(const FrameParams& p, cudaStream_t s) {
  using G = Geo5<PY, WIDE>;
  const size_t smem = G::bytes((p.H + 15) >> 4, p.st_nhw);
  cudaError_t e = cudaFuncSetAttribute(stream_blur_kernel<PY, WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (p.n_env == 0) return cudaSuccess;
  stream_blur_kernel<PY, WIDE>
      <<<dim3((unsigned)p.n_env, (unsigned)p.st_strips), 32 * (p.st_nvw + p.st_nhw), smem, s>>>(p);
  return cudaGetLastError();
}

template <class PY>
bool kind_matches(const FrameParams& p) {
  if (p.n_levels != PY::L) return false;
  for (int l = 0; l < PY::L; ++l)
    if (p.radius[l] != PY::r(l)) return false;
  return true;
}

// kind = 2 * pyramid + WIDE
int stream_kind_of(const FrameParams& p) {
  const int wide = p.W > kMaxStrip ? 1 : 0;
  if (kind_matches<Pyr0>(p)) return 0 + wide;
  if (kind_matches<Pyr1>(p)) return 2 + wide;
  if (kind_matches<Pyr2>(p)) return 4 + wide;
  if (kind_matches<Pyr3>(p)) return 6 + wide;
  return -1;
}

template <class PY>
void kind_info(bool wide, int nbands, int nhw, int& r4, int& maxt, size_t& smem) {
  r4 = PY::R4;
  maxt = PY::MAXT;
  smem = wide ? Geo5<PY, true>::bytes(nbands, nhw) : Geo5<PY, false>::bytes(nbands, nhw);
}

void kind_info(int k, int nbands, int nhw, int& r4, int& maxt, size_t& smem) {
  const bool wide = k & 1;
  switch (k >> 1) {
    case 0: kind_info<Pyr0>(wide, nbands, nhw, r4, maxt, smem); break;
    case 1: kind_info<Pyr1>(wide, nbands, nhw, r4, maxt, smem); break;
    case 2: kind_info<Pyr2>(wide, nbands, nhw, r4, maxt, smem); break;
    default: kind_info<Pyr3>(wide, nbands, nhw, r4, maxt, smem); break;
  }
}

}  // namespace

size_t stream_smem_bytes(const FrameParams& p) {
  int r4, maxt;
  size_t smem;
  kind_info(p.st_kind, (p.H + 15) >> 4, p.st_nhw, r4, maxt, smem);
  return smem;
}

// Strips of <= 320 output columns (multiples of 16); V range = strip +- R4
// columns clamped to the frame; one V lane per column pair, H lanes take
// <= 2 (row pair, 8 columns) items per block.
void plan_stream(FrameParams& p) {
  p.st_kind = -1;
  const int k = stream_kind_of(p);
  if (k < 0 || p.W % 16 != 0 || p.W < 16 || p.H < 1) return;
  if (p.mg.rows * p.mg.cols > 1024) return;  // epilogue scratch
  int r4, maxt;
  size_t smem;
  kind_info(k, 1, 1, r4, maxt, smem);
  int strips = (p.W + kMaxStrip - 1) / kMaxStrip;
  int sw = ((p.W + strips - 1) / strips + 15) & ~15;
  strips = (p.W + sw - 1) / sw;
  const int vw = std::min(sw + 2 * r4, p.W);  // widest V range (columns)
  const int nvw = (vw / 2 + 31) / 32;
  const int items = 4 * (sw / 8);
  int nhw = (items + 31) / 32;
  while (nhw > 1 && 32 * (nvw + nhw) > maxt) --nhw;
  if (nvw > kMaxVW || 32 * (nvw + nhw) > maxt || 2 * 32 * nhw < items) return;
  p.strip_w = sw;
  p.st_strips = strips;
  p.st_nvw = nvw;
  p.st_nhw = nhw;
  p.st_ip = 0;
  p.st_rpp = 0;
  p.st_kind = k;
  if (stream_smem_bytes(p) > 227 * 1024) p.st_kind = -1;
}

cudaError_t launch_stream_blur(const FrameParams& p, cudaStream_t s) {
  switch (p.st_kind) {
    case 0: return launch_kind<Pyr0, false>(p, s);
    case 1: return launch_kind<Pyr0, true>(p, s);
    case 2: return launch_kind<Pyr1, false>(p, s);
    case 3: return launch_kind<Pyr1, true>(p, s);
    case 4: return launch_kind<Pyr2, false>(p, s);
    case 5: return launch_kind<Pyr2, true>(p, s);
    case 6: return launch_kind<Pyr3, false>(p, s);
    case 7: return launch_kind<Pyr3, true>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tac
