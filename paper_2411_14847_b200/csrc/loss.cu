// loss.cu — dass_fidelity_loss: the fidelity loss of Eq. 3,
// L = (1−λ)·L1 + λ·(1 − SSIM) (A39), forward and ∂L/∂I.
//
// SSIM statistics are separable 11-tap Gaussian windows (σ = 1.5, zero
// padding).  Two stencil kernels on 32×32 output tiles with a 5-px halo
// staged in shared memory:
//   ssim_fwd:  4 windowed moments (μ_I, μ_G, E[I² + G²], E[IG]) → S(q) and the
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

// Both stencil kernels are register-blocked separable passes over a staged
// 42×42 tile: the horizontal pass gives each thread an 8-column strip of one
// row (18 inputs per 8 outputs instead of 11 per output), the vertical pass a
// 4-row strip of one column (14 inputs per 4 outputs), so shared-memory loads
// per output drop from ≈ 90 to ≈ 25 and the kernels become HBM-bound.
constexpr int HS = 8;                  // horizontal strip (columns per thread)
constexpr int VS = 4;                  // vertical strip (rows per thread)
constexpr int HTASKS = LS * (LT / HS); // 168 horizontal strips per tile

__global__ void __launch_bounds__(256) ssim_fwd_kernel(int W, int H, const float* __restrict__ img,
                                                      const float* __restrict__ gt, Win win,
                                                      float* __restrict__ pmaps,
                                                      double* __restrict__ acc) {
  __shared__ float sI[LS][LS + 1], sG[LS][LS + 1];
  __shared__ float sH[4][LS][LT + 1];   // μ_I, μ_G, E[I² + G²], E[IG] (B2 needs only σ_I² + σ_G²)
  __shared__ double s_red[2][8];
  const int ch = blockIdx.z;
  const size_t np = (size_t)W * H;
  const float* I = img + ch * np;
  const float* G = gt + ch * np;
  const int x0 = blockIdx.x * LT, y0 = blockIdx.y * LT;
  const int t = threadIdx.x;
  {
    // warp-per-row staging: coalesced row segments, no index division
    const int lane = t & 31;
    for (int r = t >> 5; r < LS; r += 8) {
      const int gy = y0 - HALO + r;
      const bool rin = gy >= 0 && gy < H;
      const size_t rowoff = (size_t)(rin ? gy : 0) * W;
#pragma unroll
      for (int c = lane; c < LS; c += 32) {
        const int gx = x0 - HALO + c;
        const bool in = rin && gx >= 0 && gx < W;
        sI[r][c] = in ? __ldg(I + rowoff + gx) : 0.f;
        sG[r][c] = in ? __ldg(G + rowoff + gx) : 0.f;
      }
    }
  }
  __syncthreads();
  if (t < HTASKS) {
    const int r = t >> 2, c0 = (t & 3) * HS;
    float xi[HS + 10], xg[HS + 10], xsq[HS + 10], xig[HS + 10];
#pragma unroll
    for (int k = 0; k < HS + 10; ++k) {
      xi[k] = sI[r][c0 + k]; xg[k] = sG[r][c0 + k];
      xsq[k] = fmaf(xi[k], xi[k], xg[k] * xg[k]); xig[k] = xi[k] * xg[k];
    }
#pragma unroll
    for (int o = 0; o < HS; ++o) {
      float a = 0.f, b = 0.f, sq = 0.f, ab = 0.f;
#pragma unroll
      for (int d = 0; d < 11; ++d) {
        const float w = win.w[d];
        a = fmaf(w, xi[o + d], a); b = fmaf(w, xg[o + d], b);
        sq = fmaf(w, xsq[o + d], sq); ab = fmaf(w, xig[o + d], ab);
      }
      sH[0][r][c0 + o] = a; sH[1][r][c0 + o] = b; sH[2][r][c0 + o] = sq; sH[3][r][c0 + o] = ab;
    }
  }
  __syncthreads();
  const int c = t & 31, r0 = (t >> 5) * VS;
  const int gx = x0 + c;
  float m[VS][4];
#pragma unroll
  for (int o = 0; o < VS; ++o)
#pragma unroll
    for (int q = 0; q < 4; ++q) m[o][q] = 0.f;
#pragma unroll
  for (int k = 0; k < VS + 10; ++k) {
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = sH[q][r0 + k][c];
#pragma unroll
    for (int o = 0; o < VS; ++o) {
      const int d = k - o;
      if (d >= 0 && d < 11) {
        const float w = win.w[d];
#pragma unroll
        for (int q = 0; q < 4; ++q) m[o][q] = fmaf(w, v[q], m[o][q]);
      }
    }
  }
  double sum_s = 0.0, sum_l1 = 0.0;
  float* P = pmaps + (size_t)ch * 3 * np;
#pragma unroll
  for (int o = 0; o < VS; ++o) {
    const int r = r0 + o, gy = y0 + r;
    if (gy >= H || gx >= W) continue;
    const float m1 = m[o][0], m2 = m[o][1];
    const float v12 = m[o][3] - m1 * m2;
    const float A1 = 2.f * m1 * m2 + SSIM_C1, A2 = 2.f * v12 + SSIM_C2;
    const float B1 = m1 * m1 + m2 * m2 + SSIM_C1, B2 = (m[o][2] - m1 * m1 - m2 * m2) + SSIM_C2;
    const float iB = 1.f / (B1 * B2);
    const float S = A1 * A2 * iB;
    sum_s += S;
    sum_l1 += fabsf(sI[r + HALO][c + HALO] - sG[r + HALO][c + HALO]);
    const size_t q = (size_t)gy * W + gx;
    P[q] = 2.f * m2 * (A2 - A1) * iB - 2.f * m1 * S * (B2 - B1) * iB;   // ∂S/∂μ_I
    P[np + q] = -S * B1 * iB;                                            // ∂S/∂E[I²] = −S/B2
    P[2 * np + q] = 2.f * A1 * iB;                                       // ∂S/∂E[IG]
  }
  // block reduction of (Σ S, Σ|I − G|) → fp64 atomics
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum_s += __shfl_xor_sync(0xffffffffu, sum_s, o);
    sum_l1 += __shfl_xor_sync(0xffffffffu, sum_l1, o);
  }
  const int w = t >> 5;
  if (c == 0) { s_red[0][w] = sum_s; s_red[1][w] = sum_l1; }
  __syncthreads();
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 8; ++k) { a += s_red[0][k]; b += s_red[1][k]; }
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
  {
    const int lane = t & 31;
    for (int r = t >> 5; r < LS; r += 8) {
      const int gy = y0 - HALO + r;
      const bool rin = gy >= 0 && gy < H;
      const size_t rowoff = (size_t)(rin ? gy : 0) * W;
#pragma unroll
      for (int c = lane; c < LS; c += 32) {
        const int gx = x0 - HALO + c;
        const bool in = rin && gx >= 0 && gx < W;
        const size_t q = rowoff + gx;
        sP[0][r][c] = in ? __ldg(P + q) : 0.f;
        sP[1][r][c] = in ? __ldg(P + np + q) : 0.f;
        sP[2][r][c] = in ? __ldg(P + 2 * np + q) : 0.f;
      }
    }
  }
  __syncthreads();
  if (t < HTASKS) {
    const int r = t >> 2, c0 = (t & 3) * HS;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float x[HS + 10];
#pragma unroll
      for (int k = 0; k < HS + 10; ++k) x[k] = sP[q][r][c0 + k];
#pragma unroll
      for (int o = 0; o < HS; ++o) {
        float a = 0.f;
#pragma unroll
        for (int d = 0; d < 11; ++d) a = fmaf(win.w[d], x[o + d], a);
        sH[q][r][c0 + o] = a;
      }
    }
  }
  __syncthreads();
  const int c = t & 31, r0 = (t >> 5) * VS;
  const int gx = x0 + c;
  float m[VS][3];
#pragma unroll
  for (int o = 0; o < VS; ++o) m[o][0] = m[o][1] = m[o][2] = 0.f;
#pragma unroll
  for (int k = 0; k < VS + 10; ++k) {
    const float v0 = sH[0][r0 + k][c], v1 = sH[1][r0 + k][c], v2 = sH[2][r0 + k][c];
#pragma unroll
    for (int o = 0; o < VS; ++o) {
      const int d = k - o;
      if (d >= 0 && d < 11) {
        const float w = win.w[d];
        m[o][0] = fmaf(w, v0, m[o][0]); m[o][1] = fmaf(w, v1, m[o][1]); m[o][2] = fmaf(w, v2, m[o][2]);
      }
    }
  }
  const float invM = 1.f / (3.f * (float)np);
#pragma unroll
  for (int o = 0; o < VS; ++o) {
    const int gy = y0 + r0 + o;
    if (gy >= H || gx >= W) continue;
    const size_t q = (size_t)gy * W + gx;
    const float iv = __ldg(img + ch * np + q), gv = __ldg(gt + ch * np + q);
    const float dssim = m[o][0] + 2.f * iv * m[o][1] + gv * m[o][2];
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
