// inherit.cu — selective inheritance (Eq. 1) and its straight-through
// gradient plus the mask loss of Eq. 2.  Elementwise,
// HBM-bound (f3 of SURVEY §8(f)).
#include "common.cuh"

namespace dass {
namespace {

__global__ void __launch_bounds__(256) inherit_mask_kernel(int n, const float* __restrict__ m,
                                                          uint8_t* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // Quant(sigmoid(m)) with Quant(x) = 1[x >= 0.5]  <=>  m >= 0
  keep[i] = m[i] >= 0.f ? 1 : 0;
}

__global__ void __launch_bounds__(256) inherit_mask_bwd_kernel(
    int n, const float* __restrict__ m, const float4* __restrict__ pos_opa,
    const float4* __restrict__ scale, const float4* __restrict__ g_pos_opa,
    const float4* __restrict__ g_scale, float lambda_inher, float* g_m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float sig = 1.f / (1.f + __expf(-m[i]));
  const float dsig = sig * (1.f - sig);
  const float4 po = pos_opa[i], s = scale[i], gpo = g_pos_opa[i], gs = g_scale[i];
  const float dm_op = po.w * gpo.w + s.x * gs.x + s.y * gs.y + s.z * gs.z;
  g_m[i] += (dm_op + lambda_inher) * dsig;
}

}  // namespace

cudaError_t launch_inherit_mask(int n, const float* m, uint8_t* keep, cudaStream_t s) {
  inherit_mask_kernel<<<div_up(n, 256), 256, 0, s>>>(n, m, keep);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_inherit_mask_bwd(int n, const float* m, const float4* pos_opa,
                                    const float4* scale, const float4* g_pos_opa,
                                    const float4* g_scale, float lambda_inher, float* g_m,
                                    cudaStream_t s) {
  inherit_mask_bwd_kernel<<<div_up(n, 256), 256, 0, s>>>(n, m, pos_opa, scale, g_pos_opa, g_scale,
                                                         lambda_inher, g_m);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
