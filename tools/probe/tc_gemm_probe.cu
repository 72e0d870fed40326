// Probe: one tcgen05.mma kind::tf32 GEMM D[128×N] = A[128×K]·B[N×K]ᵀ with
// K-major SWIZZLE_NONE operands, checked against a CPU fp64 reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_gemm_probe tc_gemm_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 64, K = 24;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// element (r, k) of an R×K K-major operand: core matrices of 8 rows × 16 B
__device__ __forceinline__ int kmaj(int r, int k, int R) {
  return (k >> 2) * (R * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int mode) {
  __shared__ __align__(1024) float sA[M * K], sAl[M * K];
  __shared__ __align__(1024) float sB[N * K], sBl[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int e = t; e < M * K; e += blockDim.x) {
    const float x = A[e], hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    sA[kmaj(e / K, e % K, M)] = hi; sAl[kmaj(e / K, e % K, M)] = x - hi;
  }
  for (int e = t; e < N * K; e += blockDim.x) {
    const float x = B[e], hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    sB[kmaj(e / K, e % K, N)] = hi; sBl[kmaj(e / K, e % K, N)] = x - hi;
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (t == 0) {
    const float* As[3] = {sA, sAl, sA};
    const float* Bs[3] = {sB, sB, sBl};
    const int npass = mode ? 3 : 1;
    for (int ps = 0; ps < npass; ++ps)
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t ad = sdesc(smem_u32(As[ps]) + kk * 2 * (M * 16), M * 16, 128);
      const uint64_t bd = sdesc(smem_u32(Bs[ps]) + kk * 2 * (N * 16), N * 16, 128);
      const uint32_t acc = (kk > 0 || ps > 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for phase 0
  asm volatile("{\n.reg .pred P1;\nWAIT:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@!P1 bra WAIT;\n}\n" ::"r"(smem_u32(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = t >> 5, lane = t & 31;
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      const int row = warp * 32 + lane;
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

int main(int argc, char** argv) {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX) - 0.5f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX) - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  probe<<<1, 256>>>(dA, dB, dD, mode);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("max |ref| %.4g  max err %.4g  rel %.3g  D[0]=%g D[last]=%g\n", maxref, maxerr, maxerr / maxref, D[0], D[M * N - 1]);
  return 0;
}
