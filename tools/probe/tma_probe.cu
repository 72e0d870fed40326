// TMA 3-D tile load probe: box (BX, BY, BZ) of a [Z][H][W] fp32 tensor at a
// (possibly negative) origin; compares the staged box with a host-built one.
// usage: tma_probe BX BY BZ x y z [desc_in_global]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, int x, int y,
                      int z, uint32_t bytes, int n, float* out) {
  extern __shared__ __align__(128) float s[];
  __shared__ __align__(8) uint64_t bar;
  const uint64_t desc = gtm ? (uint64_t)gtm : (uint64_t)&tm;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(s)), "l"(desc), "r"(x), "r"(y), "r"(z), "r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
               "@!P1 bra WAIT_%=;\n}\n" ::"r"(su32(&bar)) : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  const int BX = atoi(argv[1]), BY = atoi(argv[2]), BZ = atoi(argv[3]);
  const int x = atoi(argv[4]), y = atoi(argv[5]), z = atoi(argv[6]);
  const int glob = argc > 7 ? atoi(argv[7]) : 0;
  const int W = 64, H = 64, Z = 9;
  std::vector<float> h(W * H * Z);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i + 1);
  float *d, *o;
  const int n = BX * BY * BZ;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, n * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)Z};
  const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  const cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)BY, (cuuint32_t)BZ};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gm = nullptr;
  if (glob) {
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  }
  const size_t smem = (size_t)n * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<1, 256, smem>>>(m, gm, x, y, z, (uint32_t)(n * 4), n, o);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = 0;
  if (e == cudaSuccess) {
    std::vector<float> g(n);
    cudaMemcpy(g.data(), o, n * 4, cudaMemcpyDeviceToHost);
    for (int k = 0; k < BZ; ++k)
      for (int rr = 0; rr < BY; ++rr)
        for (int c = 0; c < BX; ++c) {
          const int gx = x + c, gy = y + rr, gz = z + k;
          const float want = (gx >= 0 && gx < W && gy >= 0 && gy < H && gz < Z) ? h[(gz * H + gy) * W + gx] : 0.f;
          if (g[(k * BY + rr) * BX + c] != want) ++bad;
        }
  }
  printf("box %d,%d,%d at %d,%d,%d glob=%d: encode %d, kernel %s, mismatches %d\n", BX, BY, BZ, x, y, z,
         glob, (int)r, cudaGetErrorString(e), bad);
  return 0;
}
