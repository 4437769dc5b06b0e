// Row-streaming, warp-specialised blur (kernel (a), default tac_pipeline path).
//
// indentation_from + smooth_pyramid (REF/tactile.py:193-222) + the contact
// partials of contact_center (REF/marker.py:103-121) for one env column strip
// per CTA, walking down the frame in blocks of SB = 8 rows:
//
//   TMA      one elected thread streams 8-row input blocks into NS_IN smem
//            slots with cp.async.bulk (mbarrier complete_tx), NS_IN - 1
//            blocks ahead of the vertical pass.
//   V warps  one lane per column pair.  Every input row is read from smem
//            ONCE, clamped (REF/tactile.py:195-196), folded into the contact
//            partials, and pushed into a register ring of the last P rows;
//            the vertical pass of EVERY level is then evaluated from the ring
//            with pair sums shared by the levels, w0 x[y] + sum_t w_t (x[y+t]
//            + x[y-t]): R_max FADD2 + sum_l (R_l + 1) FFMA2 per output row
//            pair of columns (36 instead of 45 for sigma 1,2,4).  Outputs go
//            to a double-buffered smem block [level][row pair][column] with
//            rows interleaved in pairs, plus a per-row-pair bitmask of the
//            column pairs that are non-zero.  Replicate borders: rows
//            outside the frame are copies of the edge row (ring fill), the
//            edge column lanes write the column pads.
//   H warps  one (row pair, 8 columns) item per lane: every FFMA2 operand is
//            one aligned float2 of the interleaved block (LDS.128), summed
//            over the levels in registers, written to HBM with 16-B stores.
//            Items whose window is all zero (bitmask) store exact zeros.
//
// V and H warps hand blocks over with named barriers (FULL[s] / EMPTY[s],
// s = block parity); nothing else synchronises the CTA inside the loop.  The
// pyramid radii are template parameters (stream_kind), so every ring index,
// smem slot and tap is static: the inner loops are straight-line FFMA2.
#include <climits>

#include "tac_frame_common.cuh"

namespace tac {

namespace {

constexpr int SB = 8;          // rows per stream block
constexpr int kMaxVW = 8;      // V warps per CTA (<= 512 columns per strip)
constexpr int kStreamMaxT = 384;

// barrier ids (0 = __syncthreads)
constexpr int kBarFull = 1;    // + slot
constexpr int kBarEmpty = 3;   // + slot
constexpr int kBarV = 5;
constexpr int kBarH = 6;

template <int L_, int R0, int R1 = 0, int R2 = 0, int R3 = 0>
struct Pyr {
  static constexpr int L = L_;
  static constexpr int r(int l) { return l == 0 ? R0 : l == 1 ? R1 : l == 2 ? R2 : R3; }
  static constexpr int r4(int l) { return (r(l) + 3) & ~3; }
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int R = cmax(cmax(R0, L_ > 1 ? R1 : 0), cmax(L_ > 2 ? R2 : 0, L_ > 3 ? R3 : 0));
  static constexpr int R4 = (R + 3) & ~3;
  static constexpr int P = (2 * R + 1 + SB - 1) / SB * SB;  // ring rows (multiple of SB)
  static constexpr int NS = P / SB;                          // input slots: slot pattern repeats every P rows
  // two CTAs per SM (<= 102 registers) when the ring is short enough
  // (8 warps = 4 per SMSP: <= 128 registers per thread for the V ring)
  static constexpr int MINB = P <= 32 && L <= 3 ? 2 : 1;
  static constexpr int MAXT = MINB == 2 ? 256 : kStreamMaxT;
};

// stream_kind -> radii (host and device agree through this table)
using Pyr0 = Pyr<3, 3, 6, 12>;        // sigma 1, 2, 4 (BASELINE configs[0-2, 4])
using Pyr1 = Pyr<4, 3, 6, 12, 24>;    // sigma 1, 2, 4, 8 (configs[3])
using Pyr2 = Pyr<4, 2, 5, 10, 15>;    // kernel sizes 5, 11, 21, 31 (REF DEFAULT_PYRAMID)
using Pyr3 = Pyr<3, 0, 2, 5>;         // kernel sizes 1, 5, 11
constexpr int kStreamKinds = 4;

template <class PY>
struct KindOf;

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
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

// Shared-memory carve-up (dynamic smem), identical on host and device.
struct StreamSmem {
  size_t in_off, vb_off, nz_off, ext_off, red_off, bar_off, total;
};

__host__ __device__ inline StreamSmem stream_smem(int L, int NS, int ip, int rpp, int nbands, int nhw) {
  StreamSmem s;
  size_t o = 0;
  s.in_off = o;
  o += (size_t)NS * SB * ip * sizeof(float);
  o = (o + 127) & ~size_t(127);
  s.vb_off = o;
  o += (size_t)2 * L * (SB / 2) * rpp * sizeof(float);
  s.nz_off = o;
  o += (size_t)2 * (SB / 2) * kMaxVW * sizeof(uint32_t);
  s.ext_off = o;
  o += (size_t)nbands * nhw * sizeof(int2);
  o = (o + 7) & ~size_t(7);
  s.red_off = o;
  o += (size_t)kMaxVW * 8 * sizeof(double);
  s.bar_off = o;
  o += (size_t)NS * sizeof(uint64_t);
  s.total = (o + 127) & ~size_t(127);
  return s;
}

// One H item: row pair m x 8 columns of a block (acc[i] = (row 2m, row 2m+1)
// at column c0 + i).  Returns false (acc = 0) when the V window of the widest
// level is all zero, or for a lane without an item.
template <class PY>
__device__ __forceinline__ bool h_item(const FrameParams& p, const float* vslot, const uint32_t* nzb, int item,
                                       int nitems, int x0, int vx0, int npairs, float2 (&acc)[8]) {
  constexpr int L = PY::L, R4 = PY::R4;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  if (item >= nitems) return false;
  const int m = item & 3;
  const int c0 = x0 + 8 * (item >> 2);
  const uint32_t* nzs = nzb + m * kMaxVW;
  const int qa = max((c0 - R4 - vx0) >> 1, 0);
  const int qb = min((c0 + 8 + R4 - vx0) >> 1, npairs) - 1;
  bool any = false;
  for (int w = qa >> 5; w <= (qb >> 5); ++w) {
    uint32_t bits = nzs[w];
    const int b0 = w * 32;
    if (qa > b0) bits &= ~0u << (qa - b0);
    if (qb < b0 + 31) bits &= ~0u >> (b0 + 31 - qb);
    any |= bits != 0u;
  }
  if (!any) return false;
  const int rpp = p.st_rpp;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int rl_ = PY::r(l), r4l = PY::r4(l);
    // row pair m of level l from column c0 - r4l (16-B aligned: every offset is a multiple of 4 columns)
    const float* src_l = vslot + (size_t)(l * (SB / 2) + m) * rpp + 2 * (c0 - r4l - vx0 + R4);
    // the window 2 columns at a time: window column cc feeds output i with tap cc - r4l - i
#pragma unroll
    for (int qq = 0; qq < (8 + 2 * r4l) / 2; ++qq) {
      const float4 f = *reinterpret_cast<const float4*>(src_l + 4 * qq);
      const float2 va = make_float2(f.x, f.y), vbb = make_float2(f.z, f.w);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = 2 * qq + h;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int t = cc - r4l - i;
          if (t >= -rl_ && t <= rl_) acc[i] = ffma2(p.wh2[l][t < 0 ? -t : t], h ? vbb : va, acc[i]);
        }
      }
    }
  }
  return true;
}

__device__ __forceinline__ void h_store(const FrameParams& p, long long env, long long HW, int W, int H, int y0,
                                        int x0, int item, int nitems, const float2 (&acc)[8], bool any, int& lo,
                                        int& hi) {
  if (item >= nitems) return;
  const int m = item & 3;
  const int c0 = x0 + 8 * (item >> 2);
  const int y = y0 + 2 * m;
  float* d = p.scratch + env * HW + (long long)y * W + c0;
  if (y < H) {
    reinterpret_cast<float4*>(d)[0] = make_float4(acc[0].x, acc[1].x, acc[2].x, acc[3].x);
    reinterpret_cast<float4*>(d)[1] = make_float4(acc[4].x, acc[5].x, acc[6].x, acc[7].x);
  }
  if (y + 1 < H) {
    reinterpret_cast<float4*>(d + W)[0] = make_float4(acc[0].y, acc[1].y, acc[2].y, acc[3].y);
    reinterpret_cast<float4*>(d + W)[1] = make_float4(acc[4].y, acc[5].y, acc[6].y, acc[7].y);
  }
  if (any) {
    lo = min(lo, c0);
    hi = max(hi, c0 + 7);
  }
}

// ---------------------------------------------------------------------------
template <class PY>
__global__ void __launch_bounds__(PY::MAXT, PY::MINB) stream_blur_kernel(const __grid_constant__ FrameParams p) {
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
  const int ip = p.st_ip, rpp = p.st_rpp;
  const int nvw = p.st_nvw, nhw = p.st_nhw;
  const int nthreads = 32 * (nvw + nhw);
  const int nbands = (H + 15) >> 4;
  const int nblk = (H + SB - 1) / SB;  // output (and input) blocks
  const StreamSmem sm = stream_smem(L, NS, ip, rpp, nbands, nhw);
  float* in_s = reinterpret_cast<float*>(smem_raw + sm.in_off);
  float* vb = reinterpret_cast<float*>(smem_raw + sm.vb_off);
  uint32_t* s_nz = reinterpret_cast<uint32_t*>(smem_raw + sm.nz_off);
  int2* s_ext = reinterpret_cast<int2*>(smem_raw + sm.ext_off);
  double* s_red = reinterpret_cast<double*>(smem_raw + sm.red_off);
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem_raw + sm.bar_off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* src = p.in + env * HW;
  const unsigned rbytes = (unsigned)(vx1 - vx0) * 4u;

  // one thread streams input block b (rows 8b..) into slot b % NS
  auto issue = [&](int b) {
    const int slot = b % NS;
    const int rows = min(SB, H - b * SB);
    mbar_expect_tx(&s_full[slot], rbytes * (unsigned)rows);
    float* dst = in_s + slot * SB * ip;
    const float* g = src + (long long)b * SB * W + vx0;
    if (vx0 == 0 && vx1 == W && ip == W) {
      bulk_g2s(dst, g, rbytes * (unsigned)rows, &s_full[slot]);  // contiguous rows
    } else {
      for (int i = 0; i < rows; ++i) bulk_g2s(dst + i * ip, g + (long long)i * W, rbytes, &s_full[slot]);
    }
  };
  if (threadIdx.x == 0) {
    *reinterpret_cast<unsigned*>(s_red + kMaxVW * 8 - 1) = 0u;  // non-finite count
    for (int s = 0; s < NS; ++s) mbar_init(&s_full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int b = 0; b < NS && b < nblk; ++b) issue(b);
  }
  __syncthreads();

  if (warp < nvw) {
    // ======================= V warps: convert + vertical pass ===================
    const int q = warp * 32 + lane;  // column pair of the V range
    const int c = vx0 + 2 * q;
    const bool act = c < vx1;
    const int cr = act ? c : vx1 - 2;              // inactive lanes read a valid column
    const bool own = act && c >= x0 && c < x1;     // counted in this strip's contact partials
    const float* col = in_s + (cr - vx0);
    const bool padl = act && c == 0, padr = act && c + 2 == W;
    // warp-uniform: only the warps holding a frame-edge column write pads
    const bool pad_warp = __any_sync(0xffffffffu, padl || padr);
    unsigned* s_nf = reinterpret_cast<unsigned*>(s_red + kMaxVW * 8 - 1);  // non-finite count (rare path)
    const float2 rr = make_float2(p.rest, p.rest), rl = make_float2(p.rest_lo, p.rest_lo);
    const float thr = p.threshold;
    const bool depth_in = p.input_depth != 0;
    const bool partials = p.finalize != 0;
    const double yoff = 0.5 - (double)p.half_h;
    float cnt = 0.f, mx = 0.f;
    float cs0 = 0.f, cs1 = 0.f;  // fp32 column sums of the current block (flushed to fp64 per block)
    double sw = 0.0, swx = 0.0, swy = 0.0;
    float2 win[P];
    float2 last = make_float2(0.f, 0.f);
    int last_nz = INT_MIN / 2;  // last input row with a non-zero value in this pair

    // read + convert + fold one real row y (block already waited for)
    auto take = [&](int y, int slot, int row) -> float2 {
      const float2 raw = *reinterpret_cast<const float2*>(col + (slot * SB + row) * ip);
      float2 v = raw;
      if (depth_in) {
        v = fsubadd2(rr, raw, rl);
        v.x = clampf(v.x, 0.f, p.rest);
        v.y = clampf(v.y, 0.f, p.rest);
      }
      if (own && partials) {
        if (!(fabsf(raw.x + raw.y) < INFINITY))
          atomicAdd(s_nf, (fabsf(raw.x) < INFINITY ? 0u : 1u) + (fabsf(raw.y) < INFINITY ? 0u : 1u));
        mx = fmaxf(mx, fmaxf(v.x, v.y));
        const float w0 = v.x > thr ? v.x : 0.f, w1 = v.y > thr ? v.y : 0.f;
        cnt += (v.x > thr ? 1.f : 0.f) + (v.y > thr ? 1.f : 0.f);
        cs0 += w0;
        cs1 += w1;
        const float rs = w0 + w1;
        if (rs != 0.f) {
          sw += (double)rs;
          swy = fma((double)rs, (double)y + yoff, swy);
        }
      }
      if ((__float_as_uint(v.x) | __float_as_uint(v.y)) != 0u) last_nz = y;
      return v;
    };
    auto flush_cols = [&]() {
      if (own && partials && (cs0 != 0.f || cs1 != 0.f)) {
        const double xc0 = (double)c + 0.5 - (double)p.half_w;
        swx = fma((double)cs0, xc0, swx);
        swx = fma((double)cs1, xc0 + 1.0, swx);
      }
      cs0 = cs1 = 0.f;
    };

    // ---- prologue: ring rows -R .. R-1 (rows < 0 replicate row 0) ----------
    {
      int waited = -1;
#pragma unroll
      for (int y = 0; y < R; ++y) {
        if (y < H) {
          const int b = y / SB;
          if (b != waited) {
            mbar_wait(&s_full[b % NS], (b / NS) & 1);
            waited = b;
          }
          last = take(y, b % NS, y % SB);
        }
        win[(y % P + P) % P] = last;
        if (y == 0) {
#pragma unroll
          for (int t = 1; t <= R; ++t) win[((-t) % P + P) % P] = last;
        }
      }
      flush_cols();
    }

    // ---- main loop: iteration j = output rows 8j..8j+7 = input rows 8j+R.. ---
    int j = 0;
    int next_issue = min(NS, nblk);  // (thread 0) next input block to stream
    for (int jj = 0; jj < nblk; jj += NS) {
#pragma unroll
      for (int u = 0; u < NS; ++u) {
        j = jj + u;
        if (j >= nblk) break;
        const int sv = j & 1;
        bar_sync_n(kBarEmpty + sv, nthreads);  // H finished block j-2; all V warps finished j-1
        if (threadIdx.x == 0) {
          // input blocks before the first one iteration j reads are free:
          // refill their slots NS blocks ahead
          const int lim = min((SB * j + R) / SB + NS, nblk);
          while (next_issue < lim) issue(next_issue++);
        }
        float* vslot = vb + (size_t)sv * L * (SB / 2) * rpp;
        uint32_t* nzs = s_nz + sv * (SB / 2) * kMaxVW;
        float2 prev[L];
#pragma unroll
        for (int l = 0; l < L; ++l) prev[l] = make_float2(0.f, 0.f);
        bool prev_nz = false;
#pragma unroll
        for (int i = 0; i < SB; ++i) {
          // input row yi = 8j + R + i  (static slot / ring index within the unrolled P rows)
          const int yi = SB * j + R + i;
          const int ring_in = (SB * u + R + i) % P;
          const int slot_in = ring_in / SB;  // == (yi / SB) % NS since NS * SB == P
          if (yi < H) {
            if (i == 0 || ((R + i) % SB) == 0) mbar_wait(&s_full[slot_in], ((yi / SB) / NS) & 1);
            last = take(yi, slot_in, (R + i) % SB);
            if (((R + i) % SB) == SB - 1) flush_cols();
          }
          win[ring_in] = last;
          // output row yo = 8j + i from ring rows yo-R .. yo+R
          const int ro = (SB * u + i) % P;
          float2 o[L];
          const bool live = __any_sync(0xffffffffu, last_nz >= SB * j + i - R);
          if (live) {
            // w0 x[yo] + sum_t w_t (x[yo+t] + x[yo-t]): the pair sum of tap t is
            // shared by every level with radius >= t
#pragma unroll
            for (int l = 0; l < L; ++l) o[l] = ffma2(p.wv2[l][0], win[ro], make_float2(0.f, 0.f));
#pragma unroll
            for (int t = 1; t <= R; ++t) {
              const float2 ps = fadd2(win[(ro + t) % P], win[(ro - t + P) % P]);
#pragma unroll
              for (int l = 0; l < L; ++l)
                if (t <= PY::r(l)) o[l] = ffma2(p.wv2[l][t], ps, o[l]);
            }
          } else {
#pragma unroll
            for (int l = 0; l < L; ++l) o[l] = make_float2(0.f, 0.f);
          }
          bool nz = false;
#pragma unroll
          for (int l = 0; l < L; ++l) nz |= (__float_as_uint(o[l].x) | __float_as_uint(o[l].y)) != 0u;
          if (i & 1) {
            // row pair m = i/2: (rows 2m, 2m+1) x (columns c, c+1), one float4 per level
            const int m = i >> 1;
            if (act) {
#pragma unroll
              for (int l = 0; l < L; ++l) {
                float* d = vslot + (size_t)(l * (SB / 2) + m) * rpp;
                *reinterpret_cast<float4*>(d + 2 * (c - vx0 + R4)) =
                    make_float4(prev[l].x, o[l].x, prev[l].y, o[l].y);
                if (pad_warp && padl) {  // replicate columns -R4_l .. -1 (column 0)
                  const float4 e4 = make_float4(prev[l].x, o[l].x, prev[l].x, o[l].x);
#pragma unroll
                  for (int k = 0; k < PY::r4(l); k += 2)
                    *reinterpret_cast<float4*>(d + 2 * (R4 - PY::r4(l) + k)) = e4;
                }
                if (pad_warp && padr) {  // replicate columns W .. W+R4_l-1 (column W-1)
                  const float4 e4 = make_float4(prev[l].y, o[l].y, prev[l].y, o[l].y);
#pragma unroll
                  for (int k = 0; k < PY::r4(l); k += 2)
                    *reinterpret_cast<float4*>(d + 2 * (W - vx0 + R4 + k)) = e4;
                }
              }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, act && (nz || prev_nz));
            if (lane == 0) nzs[m * kMaxVW + warp] = bal;
          } else {
#pragma unroll
            for (int l = 0; l < L; ++l) prev[l] = o[l];
            prev_nz = nz;
          }
        }
        bar_arrive_n(kBarFull + sv, nthreads);
      }
    }
    flush_cols();  // a partial last block
    // ---- contact partials of the strip: V warps only ----------------------------
    if (p.finalize == 0) return;
    Red red;
    red.cnt = cnt;
    red.mx = mx;
    red.nf = 0.f;
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
      double t[6] = {0, 0, 0, 0, 0, (double)*s_nf};
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
    // items = (row pair m, 8-column chunk) of a block; a lane takes items
    // ht, ht + 32 nhw, ... (the same chunks in every block)
    const int ht = threadIdx.x - 32 * nvw;
    const int hw = warp - nvw;
    const int nht = 32 * nhw;
    const int nitems = 4 * ((x1 - x0) >> 3);
    const int npairs = (vx1 - vx0) >> 1;
    int lo = INT_MAX, hi = INT_MIN;  // non-zero output columns of the current band
    bar_arrive_n(kBarEmpty + 0, nthreads);
    if (nblk > 1) bar_arrive_n(kBarEmpty + 1, nthreads);
    for (int j = 0; j < nblk; ++j) {
      const int sv = j & 1;
      bar_sync_n(kBarFull + sv, nthreads);
      const float* vslot = vb + (size_t)sv * L * (SB / 2) * rpp;
      float2 acc0[8], acc1[8];
      const bool any0 = h_item<PY>(p, vslot, s_nz + sv * (SB / 2) * kMaxVW, ht, nitems, x0, vx0, npairs, acc0);
      const bool any1 = h_item<PY>(p, vslot, s_nz + sv * (SB / 2) * kMaxVW, ht + nht, nitems, x0, vx0, npairs, acc1);
      if (j + 2 < nblk) bar_arrive_n(kBarEmpty + sv, nthreads);
      h_store(p, env, HW, W, H, SB * j, x0, ht, nitems, acc0, any0, lo, hi);
      h_store(p, env, HW, W, H, SB * j, x0, ht + nht, nitems, acc1, any1, lo, hi);
      // band (16 rows = 2 blocks) complete: per-warp extent
      if ((j & 1) || j == nblk - 1) {
        const int blo = __reduce_min_sync(0xffffffffu, lo);
        const int bhi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) s_ext[(j >> 1) * nhw + hw] = make_int2(blo, bhi);
        lo = INT_MAX;
        hi = INT_MIN;
      }
    }
    bar_sync_n(kBarH, 32 * nhw);
    for (int b = ht; b < nbands; b += 32 * nhw) {
      int2 e = make_int2(INT_MAX, INT_MIN);
      for (int w = 0; w < nhw; ++w) {
        const int2 x = s_ext[b * nhw + w];
        e.x = min(e.x, x.x);
        e.y = max(e.y, x.y);
      }
      p.band_ext[(env * nbands + b) * p.ext_strips + strip] = e;
    }
  }
}

template <class PY>
cudaError_t launch_kind(const FrameParams& p, cudaStream_t s) {
  const size_t smem = stream_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(stream_blur_kernel<PY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (p.n_env == 0) return cudaSuccess;
  stream_blur_kernel<PY><<<dim3((unsigned)p.n_env, (unsigned)p.st_strips), 32 * (p.st_nvw + p.st_nhw), smem, s>>>(p);
  return cudaGetLastError();
}

template <class PY>
bool kind_matches(const FrameParams& p) {
  if (p.n_levels != PY::L) return false;
  for (int l = 0; l < PY::L; ++l)
    if (p.radius[l] != PY::r(l)) return false;
  return true;
}

int stream_kind_of(const FrameParams& p) {
  if (kind_matches<Pyr0>(p)) return 0;
  if (kind_matches<Pyr1>(p)) return 1;
  if (kind_matches<Pyr2>(p)) return 2;
  if (kind_matches<Pyr3>(p)) return 3;
  return -1;
}

int kind_L(int k) { return k == 0 ? Pyr0::L : k == 1 ? Pyr1::L : k == 2 ? Pyr2::L : Pyr3::L; }
int kind_R4(int k) { return k == 0 ? Pyr0::R4 : k == 1 ? Pyr1::R4 : k == 2 ? Pyr2::R4 : Pyr3::R4; }
int kind_NS(int k) { return k == 0 ? Pyr0::NS : k == 1 ? Pyr1::NS : k == 2 ? Pyr2::NS : Pyr3::NS; }

}  // namespace

size_t stream_smem_bytes(const FrameParams& p) {
  const int k = p.st_kind;
  return stream_smem(kind_L(k), kind_NS(k), p.st_ip, p.st_rpp, (p.H + 15) >> 4, p.st_nhw).total;
}

// Strips of <= 320 output columns (multiples of 16); V range = strip +- R4
// columns clamped to the frame; one V lane per column pair, one H lane per
// (row pair, 8 columns) of a 4-row-pair block.
void plan_stream(FrameParams& p) {
  p.st_kind = -1;
  const int k = stream_kind_of(p);
  if (k < 0 || p.W % 16 != 0 || p.W < 16 || p.H < 1) return;
  if (p.mg.rows * p.mg.cols > 1024) return;  // epilogue scratch
  const int R4 = kind_R4(k);
  int strips = (p.W + 319) / 320;
  int sw = ((p.W + strips - 1) / strips + 15) & ~15;
  strips = (p.W + sw - 1) / sw;
  const int vw = std::min(sw + 2 * R4, p.W);  // widest V range (columns)
  const int nvw = (vw / 2 + 31) / 32;
  const int maxt = k == 0 ? Pyr0::MAXT : k == 1 ? Pyr1::MAXT : k == 2 ? Pyr2::MAXT : Pyr3::MAXT;
  // H lanes take <= 2 (row pair, 8-column) items per block
  const int items = 4 * (sw / 8);
  int nhw = (items + 31) / 32;
  while (nhw > 1 && 32 * (nvw + nhw) > maxt) --nhw;
  if (nvw > kMaxVW || 32 * (nvw + nhw) > maxt || 2 * 32 * nhw < items) return;
  p.strip_w = sw;
  p.st_strips = strips;
  p.st_ip = (vw + 3) & ~3;
  int vp = p.st_ip + 2 * R4;  // floats per vb row: pads + V range
  if (((vp / 2) & 1) == 0) vp += 2;  // row-pair pitch 2 vp = 4 x odd: conflict-free LDS.128 over 4 row pairs
  p.st_rpp = 2 * vp;
  p.st_nvw = nvw;
  p.st_nhw = nhw;
  p.st_kind = k;
  if (stream_smem_bytes(p) > 227 * 1024) p.st_kind = -1;
}

cudaError_t launch_stream_blur(const FrameParams& p, cudaStream_t s) {
  switch (p.st_kind) {
    case 0:
      return launch_kind<Pyr0>(p, s);
    case 1:
      return launch_kind<Pyr1>(p, s);
    case 2:
      return launch_kind<Pyr2>(p, s);
    case 3:
      return launch_kind<Pyr3>(p, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tac
