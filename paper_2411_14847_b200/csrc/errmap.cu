// errmap.cu — dass_error_map (§3.4; Alg. 1 P:403-415 with
// the garble fixed, A20-A22).  Two HBM-bound kernels: a pixel kernel (E and
// the D bitmask via warp ballot, 28 B/px) and a per-Gaussian Alg. 1 kernel
// that OR-accumulates s_err (17 B/G).  Both evaluate E with the same inline
// function, so D agrees between them bit-for-bit.
#include "common.cuh"

namespace dass {
namespace {

__device__ __forceinline__ float err_at(const float* __restrict__ a, const float* __restrict__ b,
                                        size_t pix, size_t np) {
  const float e0 = fabsf(a[pix] - b[pix]);
  const float e1 = fabsf(a[np + pix] - b[np + pix]);
  const float e2 = fabsf(a[2 * np + pix] - b[2 * np + pix]);
  return __fdiv_rn(__fadd_rn(__fadd_rn(e0, e1), e2), 3.0f);
}

__global__ void __launch_bounds__(256) error_pixels_kernel(int np, const float* __restrict__ a,
                                                          const float* __restrict__ b, float gamma,
                                                          float* err, uint32_t* dmask) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  float e = 0.f;
  if (p < np) {
    e = err_at(a, b, (size_t)p, (size_t)np);
    if (err) err[p] = e;
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, p < np && e > gamma);
  if (dmask && (threadIdx.x & 31) == 0 && p < np) dmask[p >> 5] = bits;
}

__global__ void __launch_bounds__(256) alg1_kernel(const __grid_constant__ CamParams cam,
                                                  int n_base, const float4* __restrict__ pos,
                                                  const float* __restrict__ a,
                                                  const float* __restrict__ b, float gamma,
                                                  uint8_t* s_err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_base) return;
  const float4 p = pos[i];
  const float* T = cam.T;
  // P_hom = [p, 1] · T  (row vector)
  float h[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) h[c] = p.x * T[c] + p.y * T[4 + c] + p.z * T[8 + c] + T[12 + c];
  if (!(h[3] > cam.near_plane)) return;
  const float xn = h[0] / h[3], yn = h[1] / h[3];
  // x_n = Round(0.5((x_norm + 1)·W − 1)), y_n from y_norm and H (A20), half away from zero
  const float fx = roundf(0.5f * ((xn + 1.f) * (float)cam.W - 1.f));
  const float fy = roundf(0.5f * ((yn + 1.f) * (float)cam.H - 1.f));
  if (!(fx >= 0.f && fx < (float)cam.W && fy >= 0.f && fy < (float)cam.H)) return;
  const size_t np = (size_t)cam.W * cam.H;
  const size_t pix = (size_t)fy * cam.W + (size_t)fx;
  if (err_at(a, b, pix, np) > gamma) s_err[i] = 1;
}

}  // namespace

cudaError_t launch_error_map(const CamParams& cam, const float* rendered, const float* gt,
                             float gamma, float* err, uint32_t* dmask, int n_base,
                             const float4* pos_opa, uint8_t* s_err, cudaStream_t s) {
  const int np = cam.W * cam.H;
  if (err || dmask) {
    error_pixels_kernel<<<div_up(np, 256), 256, 0, s>>>(np, rendered, gt, gamma, err, dmask);
    launch_counted();
  }
  if (s_err && n_base > 0) {
    alg1_kernel<<<div_up(n_base, 256), 256, 0, s>>>(cam, n_base, pos_opa, rendered, gt, gamma, s_err);
    launch_counted();
  }
  return cudaGetLastError();
}

}  // namespace dass
