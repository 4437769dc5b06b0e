// tcgen05 probe (diagnostics, not part of the library): one CTA computes
// D[M x N] = A[M x K] . B[N x K]^T with both operands K-major in shared memory
// (no swizzle, 8-row x 16-byte core matrices), the fp32 accumulator in TMEM,
// and reads it back with tcgen05.ld.  It pins down the descriptor conventions
// (which descriptor field strides along K, the M-field bit position) that a
// tensor-core pyramid pass would rely on.
//
//   probe <dtype: bf16|tf32> <M> <N> <K> <swap 0|1> <mbit 23|24> [bmaj 0|1] [gap 128|256]
// prints the max abs error against a CPU product of the same (rounded) inputs.
// bmaj 1 stores B MN-major (element (n, k) at (n / 8) * 128 + (k / 8) * sbo_b +
// (k % 8) * 16 + (n % 8) * 2, 16-bit types) with the transpose-B bit set.  All
// 128 TMEM lanes are dumped, and the host locates each row of D in them (the
// M = 64 accumulator layout).  gap: byte stride between the core matrices that
// are adjacent in shared memory (128 = packed; 256 separates the two strides).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, no swizzle
}

// es: element bytes (2 bf16, 4 tf32).  Element (r, k) of a K-major operand
// lives at (r / 8) * sbo + (k / cpe) * 128 + (r % 8) * 16 + (k % cpe) * es,
// cpe = 16 / es elements per core-matrix row; sbo = 128 * K / cpe.
__global__ void probe_kernel(const void* A, const void* B, float* D, int M, int N, int K, int es,
                             uint32_t idesc, int swap, int ncols, int bmaj, uint32_t gap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cpe = 16 / es;
  const uint32_t kstride = gap;
  const uint32_t sbo = gap * (uint32_t)(K / cpe);
  uint8_t* sa = smem;
  uint8_t* sb = smem + (size_t)M * K * es * (gap / 128);
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const size_t off = (size_t)(r / 8) * sbo + (k / cpe) * kstride + (r % 8) * 16 + (k % cpe) * es;
    memcpy(sa + off, (const uint8_t*)A + (size_t)i * es, es);
  }
  const uint32_t sbo_b = gap * (uint32_t)(N / 8);  // MN-major: stride between 8-k groups
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const size_t off = bmaj ? (size_t)(r / 8) * kstride + (size_t)(k / 8) * sbo_b + (k % 8) * 16 + (r % 8) * es
                            : (size_t)(r / 8) * sbo + (k / cpe) * kstride + (r % 8) * 16 + (k % cpe) * es;
    memcpy(sb + off, (const uint8_t*)B + (size_t)i * es, es);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  const uint32_t lbo_f = swap ? sbo : kstride, sbo_f = swap ? kstride : sbo;
  if (tid == 0) {
    const int kstep = 32 / es;  // K elements per MMA (32 bytes)
    for (int ks = 0; ks < K / kstep; ++ks) {
      const uint64_t da = sdesc(su32(sa) + ks * 2 * kstride, lbo_f, sbo_f);
      // MN-major B: a 16-k step is two 8-k groups
      const uint64_t db = bmaj ? sdesc(su32(sb) + ks * 2 * sbo_b, swap ? kstride : sbo_b, swap ? sbo_b : kstride)
                               : sdesc(su32(sb) + ks * 2 * kstride, lbo_f, sbo_f);
      const uint32_t acc = ks > 0;
      if (es == 2)
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      else
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&bar))
                 : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          " selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(tm + ((uint32_t)(32 * warp) << 16) + (uint32_t)c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 32 * warp + lane;  // TMEM lane
    for (int j = 0; j < 8; ++j) D[(size_t)row * N + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(ncols));
}

static float tf32_round(float x) {  // round to nearest even on the 13 dropped bits
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;
  memcpy(&x, &u, 4);
  return x;
}

int main(int argc, char** argv) {
  if (argc < 7) {
    fprintf(stderr, "usage: probe bf16|tf32 M N K swap mbit\n");
    return 2;
  }
  const bool bf = strcmp(argv[1], "bf16") == 0;
  const int M = atoi(argv[2]), N = atoi(argv[3]), K = atoi(argv[4]), swap = atoi(argv[5]),
            mbit = atoi(argv[6]), bmaj = argc > 7 ? atoi(argv[7]) : 0;
  const uint32_t gap = argc > 8 ? (uint32_t)atoi(argv[8]) : 128u;
  const int es = bf ? 2 : 4;
  uint32_t idesc = (1u << 4);                      // D format f32
  idesc |= (bf ? 1u : 2u) << 7;                    // A format: bf16 (kind::f16) / tf32
  idesc |= (bf ? 1u : 2u) << 10;                   // B format
  idesc |= (uint32_t)(N >> 3) << 17;               // N / 8
  if (bmaj) idesc |= 1u << 16;                     // B MN-major
  idesc |= (uint32_t)(M >> 4) << mbit;             // M / 16
  srand(1234);
  std::vector<float> a(M * K), b(N * K);
  std::vector<uint8_t> ab(M * K * es), bb(N * K * es);
  for (int i = 0; i < M * K; ++i) a[i] = (float)rand() / RAND_MAX - 0.5f;
  for (int i = 0; i < N * K; ++i) b[i] = (float)rand() / RAND_MAX - 0.5f;
  auto pack = [&](std::vector<float>& v, std::vector<uint8_t>& o) {
    for (size_t i = 0; i < v.size(); ++i) {
      if (bf) {
        __nv_bfloat16 h = __float2bfloat16(v[i]);
        v[i] = __bfloat162float(h);
        memcpy(&o[i * 2], &h, 2);
      } else {
        memcpy(&o[i * 4], &v[i], 4);  // hardware reads tf32 from fp32 bits
        v[i] = tf32_round(v[i]);
      }
    }
  };
  pack(a, ab);
  pack(b, bb);
  void *da, *db;
  float* dd;
  cudaMalloc(&da, ab.size());
  cudaMalloc(&db, bb.size());
  cudaMalloc(&dd, sizeof(float) * 128 * N);
  cudaMemcpy(da, ab.data(), ab.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, bb.data(), bb.size(), cudaMemcpyHostToDevice);
  cudaMemset(dd, 0, sizeof(float) * 128 * N);
  int ncols = 32;
  while (ncols < N) ncols *= 2;
  const size_t smem = (size_t)(M + N) * K * es * (gap / 128);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_kernel<<<1, 128, smem>>>(da, db, dd, M, N, K, es, idesc, swap, ncols, bmaj, gap);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s M=%d N=%d K=%d swap=%d mbit=%d: CUDA error %s\n", argv[1], M, N, K, swap, mbit,
           cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> d(128 * N);
  cudaMemcpy(d.data(), dd, sizeof(float) * 128 * N, cudaMemcpyDeviceToHost);
  // each row of the product -> the TMEM lane holding it (-1: none)
  double mx = 0, ref_mx = 0;
  const double tol = bf ? 1e-4 : 1e-2;
  char map[512] = {0};
  int pos = 0, found = 0;
  for (int i = 0; i < M; ++i) {
    std::vector<double> s(N, 0.0);
    for (int j = 0; j < N; ++j) {
      for (int k = 0; k < K; ++k) s[j] += (double)a[i * K + k] * b[j * K + k];
      ref_mx = fmax(ref_mx, fabs(s[j]));
    }
    int lane = -1;
    double best = 1e30;
    for (int l = 0; l < 128; ++l) {
      double e = 0;
      for (int j = 0; j < N; ++j) e = fmax(e, fabs(s[j] - d[l * N + j]));
      if (e < best) best = e, lane = l;
    }
    if (best < tol) ++found;
    mx = fmax(mx, best);
    if (i % 16 == 0 && pos < 480) pos += snprintf(map + pos, sizeof(map) - pos, " r%d->l%d", i, best < tol ? lane : -1);
  }
  printf("%s gap=%u M=%d N=%d K=%d swap=%d mbit=%d bmaj=%d: rows found %d/%d, max err %.3e (max |D| %.3f)%s %s\n",
         argv[1], gap, M, N, K, swap, mbit, bmaj, found, M, mx, ref_mx, map, found == M ? "OK" : "WRONG");
  return 0;
}
