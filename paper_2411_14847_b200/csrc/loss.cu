// loss.cu — dass_fidelity_loss: the fidelity loss of Eq. 3,
// L = (1−λ)·L1 + λ·(1 − SSIM) (A39), forward and ∂L/∂I.
//
// SSIM statistics are separable 11-tap Gaussian windows (σ = 1.5, zero
// padding).  Two stencil kernels on 32×32 output tiles with a 5-px halo
// staged in shared memory:
//   ssim_fwd:  5 windowed moments (μ_I, μ_G, E[I²], E[G²], E[IG]) → S(q) and the
//              three partials ∂S/∂μ_I, ∂S/∂E[I²], ∂S/∂E[IG] (to workspace), plus
//              block-reduced Σ S and Σ|I − G| (fp64 atomics);
//   ssim_bwd:  the partial maps windowed again (the transpose of the
//              zero-padded correlation is the same window) → ∂SSIM/∂I, fused
//              with the L1 term.  HBM/L2-bound (≈ 40 B/px/channel).
#include "common.cuh"

namespace dass {
namespace {

constexpr int LT = 32;          // output tile
constexpr int HALO = 5;
constexpr int LS = LT + 2 * HALO;  // 42 staged rows/cols
constexpr float SSIM_C1 = 0.01f * 0.01f;
constexpr float SSIM_C2 = 0.03f * 0.03f;

struct Win {
  float w[11];
};

Win make_window() {
  Win k;
  double g[11], s = 0;
  for (int i = 0; i < 11; ++i) { g[i] = exp(-((i - 5) * (i - 5)) / (2.0 * 1.5 * 1.5)); s += g[i]; }
  for (int i = 0; i < 11; ++i) k.w[i] = (float)(g[i] / s);
  return k;
}

__global__ void __launch_bounds__(256) ssim_fwd_kernel(int W, int H, const float* __restrict__ img,
                                                      const float* __restrict__ gt, Win win,
                                                      float* __restrict__ pmaps,
                                                      double* __restrict__ acc) {
  __shared__ float sI[LS][LS + 1], sG[LS][LS + 1];
  __shared__ float sH[5][LS][LT + 1];
  __shared__ double s_red[2][8];
  const int ch = blockIdx.z;
  const size_t np = (size_t)W * H;
  const float* I = img + ch * np;
  const float* G = gt + ch * np;
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const int t = threadIdx.x;
  for (int k = t; k < LS * LS; k += 256) {
    const int r = k / LS, c = k % LS;
    const int gy = y0 - HALO + r, gx = x0 - HALO + c;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    sI[r][c] = in ? I[(size_t)gy * W + gx] : 0.f;
    sG[r][c] = in ? G[(size_t)gy * W + gx] : 0.f;
  }
  __syncthreads();
  for (int k = t; k < LS * LT; k += 256) {
    const int r = k / LT, c = k % LT;
    float a = 0.f, b = 0.f, aa = 0.f, bb = 0.f, ab = 0.f;
#pragma unroll
    for (int d = 0; d < 11; ++d) {
      const float w = win.w[d], iv = sI[r][c + d], gv = sG[r][c + d];
      a += w * iv; b += w * gv; aa += w * iv * iv; bb += w * gv * gv; ab += w * iv * gv;
    }
    sH[0][r][c] = a; sH[1][r][c] = b; sH[2][r][c] = aa; sH[3][r][c] = bb; sH[4][r][c] = ab;
  }
  __syncthreads();
  const int tx = t & 31, ty = t >> 5;
  double sum_s = 0.0, sum_l1 = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int gy = y0 + r, gx = x0 + tx;
    if (gy >= H || gx >= W) continue;
    float m[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int d = 0; d < 11; ++d) {
      const float w = win.w[d];
#pragma unroll
      for (int q = 0; q < 5; ++q) m[q] += w * sH[q][r + d][tx];
    }
    const float m1 = m[0], m2 = m[1];
    const float v1 = m[2] - m1 * m1, v2 = m[3] - m2 * m2, v12 = m[4] - m1 * m2;
    const float A1 = 2.f * m1 * m2 + SSIM_C1, A2 = 2.f * v12 + SSIM_C2;
    const float B1 = m1 * m1 + m2 * m2 + SSIM_C1, B2 = v1 + v2 + SSIM_C2;
    const float iB = 1.f / (B1 * B2);
    const float S = A1 * A2 * iB;
    sum_s += S;
    sum_l1 += fabsf(sI[r + HALO][tx + HALO] - sG[r + HALO][tx + HALO]);
    const size_t q = (size_t)gy * W + gx;
    float* P = pmaps + (size_t)ch * 3 * np;
    P[q] = 2.f * m2 * (A2 - A1) * iB - 2.f * m1 * S * (B2 - B1) * iB;   // ∂S/∂μ_I
    P[np + q] = -S / B2;                                                 // ∂S/∂E[I²]
    P[2 * np + q] = 2.f * A1 * iB;                                       // ∂S/∂E[IG]
  }
  // block reduction of (Σ S, Σ|I − G|) → fp64 atomics
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum_s += __shfl_xor_sync(0xffffffffu, sum_s, o);
    sum_l1 += __shfl_xor_sync(0xffffffffu, sum_l1, o);
  }
  if (tx == 0) { s_red[0][ty] = sum_s; s_red[1][ty] = sum_l1; }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) { a += s_red[0][w]; b += s_red[1][w]; }
    atomicAdd(&acc[0], a);
    atomicAdd(&acc[1], b);
  }
}

__global__ void __launch_bounds__(256) ssim_bwd_kernel(int W, int H, const float* __restrict__ img,
                                                      const float* __restrict__ gt, Win win,
                                                      const float* __restrict__ pmaps, float lambda,
                                                      float* __restrict__ dL) {
  __shared__ float sP[3][LS][LS + 1];
  __shared__ float sH[3][LS][LT + 1];
  const int ch = blockIdx.z;
  const size_t np = (size_t)W * H;
  const float* P = pmaps + (size_t)ch * 3 * np;
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const int t = threadIdx.x;
  for (int k = t; k < LS * LS; k += 256) {
    const int r = k / LS, c = k % LS;
    const int gy = y0 - HALO + r, gx = x0 - HALO + c;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const size_t q = (size_t)gy * W + gx;
    sP[0][r][c] = in ? P[q] : 0.f;
    sP[1][r][c] = in ? P[np + q] : 0.f;
    sP[2][r][c] = in ? P[2 * np + q] : 0.f;
  }
  __syncthreads();
  for (int k = t; k < LS * LT; k += 256) {
    const int r = k / LT, c = k % LT;
    float a = 0.f, b = 0.f, e = 0.f;
#pragma unroll
    for (int d = 0; d < 11; ++d) {
      const float w = win.w[d];
      a += w * sP[0][r][c + d]; b += w * sP[1][r][c + d]; e += w * sP[2][r][c + d];
    }
    sH[0][r][c] = a; sH[1][r][c] = b; sH[2][r][c] = e;
  }
  __syncthreads();
  const int tx = t & 31, ty = t >> 5;
  const float invM = 1.f / (3.f * (float)np);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = ty + 8 * k;
    const int gy = y0 + r, gx = x0 + tx;
    if (gy >= H || gx >= W) continue;
    float c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
    for (int d = 0; d < 11; ++d) {
      const float w = win.w[d];
      c1 += w * sH[0][r + d][tx]; c2 += w * sH[1][r + d][tx]; c3 += w * sH[2][r + d][tx];
    }
    const size_t q = (size_t)gy * W + gx;
    const float iv = img[ch * np + q], gv = gt[ch * np + q];
    const float dssim = c1 + 2.f * iv * c2 + gv * c3;
    const float d = iv - gv;
    const float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
    dL[ch * np + q] = ((1.f - lambda) * sgn - lambda * dssim) * invM;
  }
}

__global__ void loss_finalize_kernel(const double* acc, double M, float lambda, float* loss) {
  const double ssim = acc[0] / M, l1 = acc[1] / M;
  loss[0] = (float)((1.0 - lambda) * l1 + lambda * (1.0 - ssim));
  loss[1] = (float)l1;
  loss[2] = (float)ssim;
}

}  // namespace

size_t fidelity_loss_workspace(int W, int H) {
  return 256 + sizeof(float) * 9 * (size_t)W * H;
}

cudaError_t launch_fidelity_loss(int W, int H, const float* img, const float* gt, float lambda,
                                 void* ws, float* loss, float* dL, cudaStream_t s) {
  double* acc = (double*)ws;
  float* pmaps = (float*)((char*)ws + 256);
  cudaError_t e = cudaMemsetAsync(acc, 0, 2 * sizeof(double), s);
  if (e != cudaSuccess) return e;
  static const Win win = make_window();
  const dim3 grid(div_up(W, LT), div_up(H, LT), 3);
  ssim_fwd_kernel<<<grid, 256, 0, s>>>(W, H, img, gt, win, pmaps, acc);
  launch_counted();
  loss_finalize_kernel<<<1, 1, 0, s>>>(acc, 3.0 * (double)W * H, lambda, loss);
  launch_counted();
  if (dL) {
    ssim_bwd_kernel<<<grid, 256, 0, s>>>(W, H, img, gt, win, pmaps, lambda, dL);
    launch_counted();
  }
  return cudaGetLastError();
}

}  // namespace dass
