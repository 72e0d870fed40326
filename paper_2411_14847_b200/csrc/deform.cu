// deform.cu — SURVEY §8(f) f2: the dual hash-grid deformation fields 𝓗_dyn /
// 𝓗_st of §3.3 (supplement §B), forward and backward, and
// the stable dynamic/static partition of the Gaussians that routes each one to
// its field.
//
// One field evaluation per Gaussian: I-NGP multiresolution hash encoding
// (trilinear over 8 lattice corners per level, A41) → MLP in → 64 → 64 → 7
// (ReLU) → μ = out[0:3], σ = e_w + out[3:7] (A42).
//
// Kernel shape (fwd and bwd alike): a persistent CTA of 256 threads owns tiles
// of 128 Gaussians, two threads per Gaussian (each half computes half of every
// layer's outputs and encodes / scatters half of the levels).  The MLP weights
// are staged once per CTA in shared memory and read as warp-uniform float4
// broadcasts; activations live in shared-memory rows of 68 floats (stride
// chosen so per-thread float4 row reads are bank-conflict free).  The weight
// gradients are block-level outer-product reductions over the tile (each thread
// owns a 4×4 block of dW, accumulated in registers across all tiles of the CTA
// and flushed once with atomics).  The table gradient is a scatter of
// red.global.add.v{4,2}.f32 into the L2-resident tables (8 MB / 1 MB).
//
// Everything is fp32 FFMA (SIMT): the MLP is ≈20 kFLOP per Gaussian; the
// tcgen05 version is listed as next work in DESIGN.md.
#include <cstdlib>

#include "common.cuh"

namespace dass {

namespace {

constexpr int HID = DASS_MLP_HIDDEN;  // 64
constexpr int NOUT = 7;
constexpr int GT = 128;               // Gaussians per tile
constexpr int NT = 256;               // 2 threads per Gaussian
constexpr int AS = HID + 4;           // activation row stride (floats)

__host__ __device__ inline int x_stride(int in) {
  // row stride s (floats) with s/4 odd → 8 consecutive rows hit 8 distinct
  // 4-bank groups for a float4 access (conflict-free quarter-warp phases)
  return ((in / 4) & 1) ? in + 4 : in + 8;
}

// levels handled per half-CTA thread: ⌈L/2⌉ rounded up so that Lh·F % 4 == 0
__host__ __device__ inline int half_levels(int L, int F) {
  int Lh = (L + 1) / 2;
  const int q = 4 / F;
  return (Lh + q - 1) / q * q;
}

__device__ __forceinline__ void red_add_v2(float* addr, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}

// The 8 (row, weight) pairs of level l (A41).
__device__ __forceinline__ void level_corners(const HashGridParams& g, int l, float3 p,
                                              uint32_t row[8], float wt[8]) {
  const int N = g.res[l];
  const float pc[3] = {p.x, p.y, p.z};
  uint32_t i0[3];
  float w[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float xh = (pc[k] - g.lo[k]) / g.span[k];
    xh = fminf(1.f, fmaxf(0.f, xh));
    const float s = xh * (float)N;
    const float f = fminf(floorf(s), (float)(N - 1));
    i0[k] = (uint32_t)f;
    w[k] = s - f;
  }
  const bool dense = (g.dense_mask >> l) & 1u;
  const uint32_t n1 = (uint32_t)N + 1u;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t x = i0[0] + (c & 1), y = i0[1] + ((c >> 1) & 1), z = i0[2] + ((c >> 2) & 1);
    row[c] = dense ? x + n1 * (y + n1 * z)
                   : ((x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u)) & g.Tmask;
    wt[c] = ((c & 1) ? w[0] : 1.f - w[0]) * (((c >> 1) & 1) ? w[1] : 1.f - w[1]) *
            (((c >> 2) & 1) ? w[2] : 1.f - w[2]);
  }
}

// enc for levels [l0, l1) of one Gaussian → x[(l − 0)·F + f] (x = the row base)
template <int F>
__device__ __forceinline__ void encode_levels(const HashGridParams& g, const float* __restrict__ table,
                                              float3 p, bool valid, int l0, int l1, float* x) {
  for (int l = l0; l < l1; ++l) {
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.f;
    if (valid) {
      uint32_t row[8];
      float wt[8];
      level_corners(g, l, p, row, wt);
      const float* tab = table + (size_t)l * g.T * F;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if constexpr (F == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(tab) + row[c]);
          acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y; acc[2] += wt[c] * v.z; acc[3] += wt[c] * v.w;
        } else if constexpr (F == 2) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(tab) + row[c]);
          acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y;
        } else {
          acc[0] += wt[c] * __ldg(tab + row[c]);
        }
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) x[l * F + f] = acc[f];
  }
}

// acc[o] = b[o] + Σ_j x[j]·Wt[j][o] for the 32 outputs this half owns.
// x: the Gaussian's own activation row (float4 reads); Wt: column block base
// of a [in][HID] matrix (warp-uniform float4 broadcasts).
__device__ __forceinline__ void dense32(const float* __restrict__ x, int in,
                                        const float* __restrict__ Wt,
                                        const float* __restrict__ b, float acc[32]) {
#pragma unroll
  for (int o4 = 0; o4 < 8; ++o4) {
    const float4 bb = reinterpret_cast<const float4*>(b)[o4];
    acc[4 * o4] = bb.x; acc[4 * o4 + 1] = bb.y; acc[4 * o4 + 2] = bb.z; acc[4 * o4 + 3] = bb.w;
  }
#pragma unroll 1
  for (int j = 0; j < in; j += 4) {
    const float4 xv = *reinterpret_cast<const float4*>(x + j);
    const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4* w = reinterpret_cast<const float4*>(Wt + (j + q) * HID);
#pragma unroll
      for (int o4 = 0; o4 < 8; ++o4) {
        const float4 ww = w[o4];
        acc[4 * o4] = fmaf(xs[q], ww.x, acc[4 * o4]);
        acc[4 * o4 + 1] = fmaf(xs[q], ww.y, acc[4 * o4 + 1]);
        acc[4 * o4 + 2] = fmaf(xs[q], ww.z, acc[4 * o4 + 2]);
        acc[4 * o4 + 3] = fmaf(xs[q], ww.w, acc[4 * o4 + 3]);
      }
    }
  }
}

__device__ __forceinline__ void store32(float* dst, const float v[32]) {
#pragma unroll
  for (int o4 = 0; o4 < 8; ++o4)
    reinterpret_cast<float4*>(dst)[o4] = make_float4(v[4 * o4], v[4 * o4 + 1], v[4 * o4 + 2], v[4 * o4 + 3]);
}

// stage the MLP (global layout W1[HID][in] b1 W2[HID][HID] b2 W3[7][HID] b3)
struct MlpOffsets {
  int W1, b1, W2, b2, W3, b3;
  __host__ __device__ explicit MlpOffsets(int in)
      : W1(0), b1(HID * in), W2(HID * in + HID), b2(HID * in + HID + HID * HID),
        W3(HID * in + 2 * HID + HID * HID), b3(HID * in + 2 * HID + HID * HID + NOUT * HID) {}
};

template <int F>
__global__ void __launch_bounds__(NT, 2)
deform_fwd_kernel(const __grid_constant__ HashGridParams g, const float* __restrict__ table,
                  const float* __restrict__ mlp, int n, const int* __restrict__ idx,
                  const int* __restrict__ count, const float4* __restrict__ pos_opa,
                  float4* __restrict__ mu, float4* __restrict__ sigma) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  const int in = g.in;
  float* sW1t = sm;                   // [in][HID]
  float* sb1 = sW1t + in * HID;       // [HID]
  float* sW2t = sb1 + HID;            // [HID][HID] (j-major)
  float* sb2 = sW2t + HID * HID;
  float* sW3 = sb2 + HID;             // [7][HID]
  float* sb3 = sW3 + NOUT * HID;      // [8]
  float* sA = sb3 + 8;                // [GT][AS]
  float* sB = sA + GT * AS;           // [GT][AS]
  const MlpOffsets off(in);
  const int t = threadIdx.x;
  for (int e = t; e < HID * in; e += NT) sW1t[(e % in) * HID + e / in] = mlp[off.W1 + e];
  for (int e = t; e < HID * HID; e += NT) sW2t[(e % HID) * HID + e / HID] = mlp[off.W2 + e];
  for (int e = t; e < NOUT * HID; e += NT) sW3[e] = mlp[off.W3 + e];
  if (t < HID) { sb1[t] = mlp[off.b1 + t]; sb2[t] = mlp[off.b2 + t]; }
  if (t < 8) sb3[t] = t < NOUT ? mlp[off.b3 + t] : 0.f;
  __syncthreads();

  const int m = count ? min(*count, n) : n;
  const int gi = t & (GT - 1), h = t >> 7;
  const int Lh = half_levels(g.L, F);
  const int l0 = min(g.L, h * Lh), l1 = min(g.L, (h + 1) * Lh);
  float* xa = sA + gi * AS;
  float* xb = sB + gi * AS;
  for (int tile = blockIdx.x; tile * GT < m; tile += gridDim.x) {
    const int k = tile * GT + gi;
    const bool valid = k < m;
    const int i = valid ? (idx ? idx[k] : k) : 0;
    float3 p = make_float3(0.f, 0.f, 0.f);
    if (valid) { const float4 po = pos_opa[i]; p = make_float3(po.x, po.y, po.z); }
    encode_levels<F>(g, table, p, valid, l0, l1, xa);
    __syncthreads();
    float acc[32];
    dense32(xa, in, sW1t + 32 * h, sb1 + 32 * h, acc);
#pragma unroll
    for (int o = 0; o < 32; ++o) acc[o] = fmaxf(acc[o], 0.f);
    store32(xb + 32 * h, acc);
    __syncthreads();
    dense32(xb, HID, sW2t + 32 * h, sb2 + 32 * h, acc);
#pragma unroll
    for (int o = 0; o < 32; ++o) acc[o] = fmaxf(acc[o], 0.f);
    store32(xa + 32 * h, acc);
    __syncthreads();
    // linear head: half 0 → out[0..3], half 1 → out[4..6]
    const int c0 = h ? 4 : 0;
    float o4[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) o4[c] = (c0 + c < NOUT) ? sb3[c0 + c] : 0.f;
#pragma unroll 4
    for (int j = 0; j < HID; j += 4) {
      const float4 hv = *reinterpret_cast<const float4*>(xa + j);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c0 + c < NOUT) {
          const float4 w = *reinterpret_cast<const float4*>(sW3 + (c0 + c) * HID + j);
          o4[c] = fmaf(hv.x, w.x, fmaf(hv.y, w.y, fmaf(hv.z, w.z, fmaf(hv.w, w.w, o4[c]))));
        }
      }
    }
    if (valid) {
      float* sg = reinterpret_cast<float*>(sigma + i);
      if (h == 0) {
        mu[i] = make_float4(o4[0], o4[1], o4[2], 0.f);
        sg[0] = 1.f + o4[3];
      } else {
        sg[1] = o4[0]; sg[2] = o4[1]; sg[3] = o4[2];
      }
    }
    __syncthreads();
  }
}

template <int F>
__global__ void __launch_bounds__(NT, 1)
deform_bwd_kernel(const __grid_constant__ HashGridParams g, const float* __restrict__ table,
                  const float* __restrict__ mlp, int n, const int* __restrict__ idx,
                  const int* __restrict__ count, const float4* __restrict__ pos_opa,
                  const float4* __restrict__ g_mu, const float4* __restrict__ g_sigma,
                  float* __restrict__ g_table, float* __restrict__ g_mlp) {
  extern __shared__ float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  const int in = g.in;
  const int XS = x_stride(in);
  float* sW1t = sm;                   // [in][HID]
  float* sW1 = sW1t + in * HID;       // [HID][in]
  float* sb1 = sW1 + HID * in;        // [HID]
  float* sW2t = sb1 + HID;            // [HID][HID] j-major
  float* sW2 = sW2t + HID * HID;      // [HID][HID] o-major
  float* sb2 = sW2 + HID * HID;
  float* sW3 = sb2 + HID;             // [7][HID]
  float* sX = sW3 + NOUT * HID;       // [GT][XS]
  float* sH1 = sX + GT * XS;          // [GT][AS]  h1, later ∂L/∂z1
  float* sH2 = sH1 + GT * AS;         // [GT][AS]  h2, later ∂L/∂z2
  float* sD3 = sH2 + GT * AS;         // [GT][8]   ∂L/∂out
  const MlpOffsets off(in);
  const int t = threadIdx.x;
  for (int e = t; e < HID * in; e += NT) {
    const float v = mlp[off.W1 + e];
    sW1[e] = v;
    sW1t[(e % in) * HID + e / in] = v;
  }
  for (int e = t; e < HID * HID; e += NT) {
    const float v = mlp[off.W2 + e];
    sW2[e] = v;
    sW2t[(e % HID) * HID + e / HID] = v;
  }
  for (int e = t; e < NOUT * HID; e += NT) sW3[e] = mlp[off.W3 + e];
  if (t < HID) { sb1[t] = mlp[off.b1 + t]; sb2[t] = mlp[off.b2 + t]; }
  __syncthreads();

  // persistent weight-gradient accumulators
  float a3[2] = {0.f, 0.f}, ab3 = 0.f;                 // dW3 elements t, t+256; db3[t]
  float a2[16], ab2[4];                                // dW2 4×4 block, db2 (j-block 0 only)
  float a1[16], ab1[4];                                // dW1 4×4 block, db1
#pragma unroll
  for (int q = 0; q < 16; ++q) { a2[q] = 0.f; a1[q] = 0.f; }
#pragma unroll
  for (int q = 0; q < 4; ++q) { ab2[q] = 0.f; ab1[q] = 0.f; }
  const int o2 = (t >> 4) * 4, j2 = (t & 15) * 4;      // dW2 block of this thread
  const int jb1 = in / 4;                              // j-blocks of dW1
  const bool has1 = t < 16 * jb1;
  const int o1 = has1 ? (t / jb1) * 4 : 0, j1 = has1 ? (t % jb1) * 4 : 0;

  const int m = count ? min(*count, n) : n;
  const int gi = t & (GT - 1), h = t >> 7;
  const int Lh = half_levels(g.L, F);
  const int l0 = min(g.L, h * Lh), l1 = min(g.L, (h + 1) * Lh);
  float* xr = sX + gi * XS;
  float* h1r = sH1 + gi * AS;
  float* h2r = sH2 + gi * AS;
  float* d3r = sD3 + gi * 8;
  for (int tile = blockIdx.x; tile * GT < m; tile += gridDim.x) {
    const int k = tile * GT + gi;
    const bool valid = k < m;
    const int i = valid ? (idx ? idx[k] : k) : 0;
    float3 p = make_float3(0.f, 0.f, 0.f);
    if (valid) { const float4 po = pos_opa[i]; p = make_float3(po.x, po.y, po.z); }
    encode_levels<F>(g, table, p, valid, l0, l1, xr);
    if (h == 0) {
      const float4 d = valid ? g_mu[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      d3r[0] = d.x; d3r[1] = d.y; d3r[2] = d.z; d3r[7] = 0.f;
    } else {
      const float4 d = valid ? g_sigma[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      d3r[3] = d.x; d3r[4] = d.y; d3r[5] = d.z; d3r[6] = d.w;
    }
    __syncthreads();
    float acc[32];
    dense32(xr, in, sW1t + 32 * h, sb1 + 32 * h, acc);
#pragma unroll
    for (int o = 0; o < 32; ++o) acc[o] = fmaxf(acc[o], 0.f);
    store32(h1r + 32 * h, acc);
    __syncthreads();
    dense32(h1r, HID, sW2t + 32 * h, sb2 + 32 * h, acc);
#pragma unroll
    for (int o = 0; o < 32; ++o) acc[o] = fmaxf(acc[o], 0.f);
    store32(h2r + 32 * h, acc);
    __syncthreads();

    // ---- head: dW3 += d3 ⊗ h2, db3 += d3; per Gaussian ∂L/∂z2 (registers)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = t + r * NT;
      if (e < NOUT * HID) {
        const int c = e >> 6, j = e & 63;
        float s = 0.f;
#pragma unroll 8
        for (int q = 0; q < GT; ++q) s = fmaf(sD3[q * 8 + c], sH2[q * AS + j], s);
        a3[r] += s;
      }
    }
    if (t < NOUT) {
      float s = 0.f;
      for (int q = 0; q < GT; ++q) s += sD3[q * 8 + t];
      ab3 += s;
    }
    {
      float d3[NOUT];
#pragma unroll
      for (int c = 0; c < NOUT; ++c) d3[c] = d3r[c];
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 hv = *reinterpret_cast<const float4*>(h2r + 32 * h + 4 * j4);
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int c = 0; c < NOUT; ++c) {
          const float4 w = *reinterpret_cast<const float4*>(sW3 + c * HID + 32 * h + 4 * j4);
          s.x = fmaf(w.x, d3[c], s.x); s.y = fmaf(w.y, d3[c], s.y);
          s.z = fmaf(w.z, d3[c], s.z); s.w = fmaf(w.w, d3[c], s.w);
        }
        acc[4 * j4] = hv.x > 0.f ? s.x : 0.f;
        acc[4 * j4 + 1] = hv.y > 0.f ? s.y : 0.f;
        acc[4 * j4 + 2] = hv.z > 0.f ? s.z : 0.f;
        acc[4 * j4 + 3] = hv.w > 0.f ? s.w : 0.f;
      }
    }
    __syncthreads();
    store32(h2r + 32 * h, acc);       // sH2 := ∂L/∂z2
    __syncthreads();

    // ---- layer 2: dW2 += d2 ⊗ h1, db2 += d2; per Gaussian ∂L/∂z1
#pragma unroll 4
    for (int q = 0; q < GT; ++q) {
      const float4 dv = *reinterpret_cast<const float4*>(sH2 + q * AS + o2);
      const float4 hv = *reinterpret_cast<const float4*>(sH1 + q * AS + j2);
      const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, hh[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 4; ++b) a2[4 * a + b] = fmaf(dd[a], hh[b], a2[4 * a + b]);
      }
      if (j2 == 0) { ab2[0] += dd[0]; ab2[1] += dd[1]; ab2[2] += dd[2]; ab2[3] += dd[3]; }
    }
    {
#pragma unroll
      for (int o = 0; o < 32; ++o) acc[o] = 0.f;
#pragma unroll 1
      for (int o = 0; o < HID; o += 4) {
        const float4 dv = *reinterpret_cast<const float4*>(h2r + o);
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4* w = reinterpret_cast<const float4*>(sW2 + (o + q) * HID + 32 * h);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 ww = w[j4];
            acc[4 * j4] = fmaf(dd[q], ww.x, acc[4 * j4]);
            acc[4 * j4 + 1] = fmaf(dd[q], ww.y, acc[4 * j4 + 1]);
            acc[4 * j4 + 2] = fmaf(dd[q], ww.z, acc[4 * j4 + 2]);
            acc[4 * j4 + 3] = fmaf(dd[q], ww.w, acc[4 * j4 + 3]);
          }
        }
      }
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 hv = *reinterpret_cast<const float4*>(h1r + 32 * h + 4 * j4);
        if (!(hv.x > 0.f)) acc[4 * j4] = 0.f;
        if (!(hv.y > 0.f)) acc[4 * j4 + 1] = 0.f;
        if (!(hv.z > 0.f)) acc[4 * j4 + 2] = 0.f;
        if (!(hv.w > 0.f)) acc[4 * j4 + 3] = 0.f;
      }
    }
    __syncthreads();
    store32(h1r + 32 * h, acc);       // sH1 := ∂L/∂z1
    __syncthreads();

    // ---- layer 1: dW1 += d1 ⊗ x, db1 += d1; per Gaussian ∂L/∂x → table
    if (has1) {
#pragma unroll 4
      for (int q = 0; q < GT; ++q) {
        const float4 dv = *reinterpret_cast<const float4*>(sH1 + q * AS + o1);
        const float4 xv = *reinterpret_cast<const float4*>(sX + q * XS + j1);
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int b = 0; b < 4; ++b) a1[4 * a + b] = fmaf(dd[a], xx[b], a1[4 * a + b]);
        }
        if (j1 == 0) { ab1[0] += dd[0]; ab1[1] += dd[1]; ab1[2] += dd[2]; ab1[3] += dd[3]; }
      }
    }
    if (valid && l1 > l0) {
      const int jlo = l0 * F;
      const int cnt = (l1 - l0) * F;   // ≤ 32 columns of ∂L/∂x owned by this half
#pragma unroll
      for (int o = 0; o < 32; ++o) acc[o] = 0.f;
#pragma unroll 1
      for (int o = 0; o < HID; o += 4) {
        const float4 dv = *reinterpret_cast<const float4*>(h1r + o);
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4* w = reinterpret_cast<const float4*>(sW1 + (o + q) * in + jlo);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            if (4 * j4 < cnt) {   // cnt is a multiple of 4 (half_levels, in % 4 == 0)
              const float4 ww = w[j4];
              acc[4 * j4] = fmaf(dd[q], ww.x, acc[4 * j4]);
              acc[4 * j4 + 1] = fmaf(dd[q], ww.y, acc[4 * j4 + 1]);
              acc[4 * j4 + 2] = fmaf(dd[q], ww.z, acc[4 * j4 + 2]);
              acc[4 * j4 + 3] = fmaf(dd[q], ww.w, acc[4 * j4 + 3]);
            }
          }
        }
      }
      float* gt = g_table;
#pragma unroll
      for (int ll = 0; ll < 32 / F; ++ll) {
        const int l = l0 + ll;
        if (l < l1) {
          uint32_t row[8];
          float wt[8];
          level_corners(g, l, p, row, wt);
          float* tab = gt + (size_t)l * g.T * F;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if constexpr (F == 4) {
              red_add_v4(reinterpret_cast<float4*>(tab) + row[c],
                         make_float4(wt[c] * acc[4 * ll], wt[c] * acc[4 * ll + 1],
                                     wt[c] * acc[4 * ll + 2], wt[c] * acc[4 * ll + 3]));
            } else if constexpr (F == 2) {
              red_add_v2(tab + (size_t)row[c] * 2, wt[c] * acc[2 * ll], wt[c] * acc[2 * ll + 1]);
            } else {
              atomicAdd(tab + row[c], wt[c] * acc[ll]);
            }
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- flush the weight gradients (once per CTA)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = t + r * NT;
    if (e < NOUT * HID) atomicAdd(g_mlp + off.W3 + e, a3[r]);
  }
  if (t < NOUT) atomicAdd(g_mlp + off.b3 + t, ab3);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int b = 0; b < 4; ++b) atomicAdd(g_mlp + off.W2 + (o2 + a) * HID + j2 + b, a2[4 * a + b]);
    if (j2 == 0) atomicAdd(g_mlp + off.b2 + o2 + a, ab2[a]);
  }
  if (has1) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int b = 0; b < 4; ++b) atomicAdd(g_mlp + off.W1 + (o1 + a) * in + j1 + b, a1[4 * a + b]);
      if (j1 == 0) atomicAdd(g_mlp + off.b1 + o1 + a, ab1[a]);
    }
  }
}

// ---------------------------------------------------------------------------
// Tensor-core forward (tcgen05.mma kind::tf32, sm_100a).  Same tile/thread
// shape as deform_fwd_kernel; the three layers are GEMMs D[128×N] = A[128×K]·Bᵀ
// (A = the tile's activations, B = a weight matrix [N×K], both K-major in the
// canonical no-swizzle core-matrix layout: 8 rows × 16 B per 128-B core
// matrix, row groups 128 B apart, 4-float k-chunks R·16 B apart), issued by one
// thread, accumulated in TMEM and read back with tcgen05.ld for the bias/ReLU
// epilogue, which writes the next layer's A operand.  Precision: 3×TF32 — every
// operand x = hi + lo with hi = x with the low 13 mantissa bits cleared (exactly
// a TF32 value) and lo = x − hi, and D = A_hi·B_hi + A_lo·B_hi + A_hi·B_lo, which
// keeps the products at ≈ fp32 accuracy (the dropped lo·lo term is ≤ 2⁻²²·|ab|).
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// float offset of element (r, k) of an R-row K-major operand
__device__ __forceinline__ int kmaj(int r, int k, int R) {
  return (k >> 2) * (R * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  return d;                 // base offset 0, no swizzle
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M×N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               ::"r"(smem_u32(mbar)));
}
__device__ __forceinline__ void wait(uint64_t* mbar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\n"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
               "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(mbar)), "r"(parity));
}
__device__ __forceinline__ void ld16(uint32_t taddr, float v[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
                 "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[128×N] (=|+=) A·Bᵀ over K with the 3×TF32 split: A hi/lo [128×K], B hi/lo [N×K]
__device__ __forceinline__ void gemm3(uint32_t tmem, const float* Ah, const float* Al,
                                      const float* Bh, const float* Bl, int N, int K) {
  const uint32_t id = idesc_tf32(128, N);
  const float* As[3] = {Ah, Al, Ah};
  const float* Bs[3] = {Bh, Bh, Bl};
#pragma unroll
  for (int ps = 0; ps < 3; ++ps)
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t a = sdesc(smem_u32(As[ps]) + kk * 2 * (128 * 16), 128 * 16, 128);
      const uint64_t b = sdesc(smem_u32(Bs[ps]) + kk * 2 * (N * 16), N * 16, 128);
      mma(tmem, a, b, id, (ps > 0 || kk > 0) ? 1u : 0u);
    }
}

}  // namespace tc

// stage a weight matrix W[N][K] (global, row-major) as hi/lo K-major operands
// (rows ≥ Nreal are zero)
__device__ __forceinline__ void stage_weight(const float* __restrict__ W, int Nreal, int N, int K,
                                             float* hi, float* lo) {
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e - r * K;
    const float x = r < Nreal ? W[r * K + k] : 0.f;
    const float h = tc::tf32_hi(x);
    hi[tc::kmaj(r, k, N)] = h;
    lo[tc::kmaj(r, k, N)] = x - h;
  }
}

// enc for levels [l0, l1) of one Gaussian, written as hi/lo into the K-major A
// operand (row g of 128)
template <int F>
__device__ __forceinline__ void encode_levels_tc(const HashGridParams& g, const float* __restrict__ table,
                                                 float3 p, bool valid, int l0, int l1, int row,
                                                 float* xh, float* xl) {
  for (int l = l0; l < l1; ++l) {
    float acc[F];
#pragma unroll
    for (int f = 0; f < F; ++f) acc[f] = 0.f;
    if (valid) {
      uint32_t rw[8];
      float wt[8];
      level_corners(g, l, p, rw, wt);
      const float* tab = table + (size_t)l * g.T * F;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if constexpr (F == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(tab) + rw[c]);
          acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y; acc[2] += wt[c] * v.z; acc[3] += wt[c] * v.w;
        } else if constexpr (F == 2) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(tab) + rw[c]);
          acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y;
        } else {
          acc[0] += wt[c] * __ldg(tab + rw[c]);
        }
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const int o = tc::kmaj(row, l * F + f, GT);
      const float h = tc::tf32_hi(acc[f]);
      xh[o] = h;
      xl[o] = acc[f] - h;
    }
  }
}

// bias + ReLU of 16·NCH accumulator columns [c0, c0 + 16·NCH) of this thread's
// row, written as the next layer's hi/lo A operand (float4 per 4 columns)
template <int NCH>
__device__ __forceinline__ void relu_epilogue(uint32_t taddr, const float* __restrict__ bias, int c0,
                                              int row, float* hh, float* hl) {
#pragma unroll
  for (int half = 0; half < NCH; ++half) {
    float v[16];
    tc::ld16(taddr + half * 16, v);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + half * 16 + 4 * q;
      float4 h4, l4;
      float* hp = &h4.x;
      float* lp = &l4.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x = fmaxf(v[4 * q + j] + bias[c + j], 0.f);
        hp[j] = tc::tf32_hi(x);
        lp[j] = x - hp[j];
      }
      const int o = tc::kmaj(row, c, GT);   // 4 consecutive columns: one 16-B chunk
      *reinterpret_cast<float4*>(hh + o) = h4;
      *reinterpret_cast<float4*>(hl + o) = l4;
    }
  }
}

constexpr int NT_TC = 512;   // 4 threads per Gaussian row; 16 warps = 4 TMEM lane quadrants × 4 column groups

template <int F>
__global__ void __launch_bounds__(NT_TC, 1)
deform_fwd_tc_kernel(const __grid_constant__ HashGridParams g, const float* __restrict__ table,
                     const float* __restrict__ mlp, int n, const int* __restrict__ idx,
                     const int* __restrict__ count, const float4* __restrict__ pos_opa,
                     float4* __restrict__ mu, float4* __restrict__ sigma) {
  extern __shared__ __align__(1024) float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int in = g.in;
  float* W1h = sm;                      // [64][in]
  float* W1l = W1h + HID * in;
  float* W2h = W1l + HID * in;          // [64][64]
  float* W2l = W2h + HID * HID;
  float* W3h = W2l + HID * HID;         // [16][64] (rows ≥ 7 zero)
  float* W3l = W3h + 16 * HID;
  float* b1 = W3l + 16 * HID;
  float* b2 = b1 + HID;
  float* b3 = b2 + HID;                 // [16]
  float* Xh = b3 + 16;                  // [128][in]
  float* Xl = Xh + GT * in;
  float* Hh = Xl + GT * in;             // [128][64]
  float* Hl = Hh + GT * HID;
  const MlpOffsets off(in);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  stage_weight(mlp + off.W1, HID, HID, in, W1h, W1l);
  stage_weight(mlp + off.W2, HID, HID, HID, W2h, W2l);
  stage_weight(mlp + off.W3, NOUT, 16, HID, W3h, W3l);
  if (t < HID) { b1[t] = mlp[off.b1 + t]; b2[t] = mlp[off.b2 + t]; }
  if (t < 16) b3[t] = t < NOUT ? mlp[off.b3 + t] : 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;"
                 ::"r"(tc::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_async_smem();
  tc::before_sync();
  __syncthreads();
  tc::after_sync();
  const uint32_t tmem = tbase;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;   // this warp's TMEM lanes
  const int row = (warp & 3) * 32 + lane;                          // tile row = TMEM lane
  const int h = warp >> 2;                                         // column group (16 columns)
  uint32_t phase = 0;

  const int m = count ? min(*count, n) : n;
  const int gi = t & (GT - 1), qq = t >> 7;                         // encode quarter
  int Lq = (g.L + 3) / 4;
  Lq = (Lq + (4 / F) - 1) / (4 / F) * (4 / F);                     // Lq·F % 4 == 0
  const int l0 = min(g.L, qq * Lq), l1 = min(g.L, (qq + 1) * Lq);
  for (int tile = blockIdx.x; tile * GT < m; tile += gridDim.x) {
    {
      const int k = tile * GT + gi;
      const bool valid = k < m;
      const int i = valid ? (idx ? idx[k] : k) : 0;
      float3 p = make_float3(0.f, 0.f, 0.f);
      if (valid) { const float4 po = pos_opa[i]; p = make_float3(po.x, po.y, po.z); }
      encode_levels_tc<F>(g, table, p, valid, l0, l1, gi, Xh, Xl);
    }
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // layer 1: Z1 = X·W1ᵀ → TMEM columns [0, 64)
      tc::gemm3(tmem, Xh, Xl, W1h, W1l, HID, in);
      tc::commit(&mbar);
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    relu_epilogue<1>(tmem + lane_base + 16 * h, b1, 16 * h, row, Hh, Hl);
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // layer 2: Z2 = H1·W2ᵀ → TMEM columns [64, 128)
      tc::gemm3(tmem + 64, Hh, Hl, W2h, W2l, HID, HID);
      tc::commit(&mbar);
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    relu_epilogue<1>(tmem + lane_base + 64 + 16 * h, b2, 16 * h, row, Hh, Hl);
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // head: OUT = H2·W3ᵀ (N = 16, rows ≥ 7 zero) → TMEM columns [0, 16)
      tc::gemm3(tmem, Hh, Hl, W3h, W3l, 16, HID);
      tc::commit(&mbar);
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    if (h == 0) {
      float v[16];
      tc::ld16(tmem + lane_base, v);
      const int k = tile * GT + row;
      if (k < m) {
        const int i = idx ? idx[k] : k;
        mu[i] = make_float4(v[0] + b3[0], v[1] + b3[1], v[2] + b3[2], 0.f);
        sigma[i] = make_float4(1.f + (v[3] + b3[3]), v[4] + b3[4], v[5] + b3[5], v[6] + b3[6]);
      }
    }
    tc::before_sync();
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// Tensor-core backward (tcgen05, 3×TF32).  Tiles of GB = 64 Gaussians (M = 64
// keeps every operand in shared memory: 198 KB at in = 32): the recompute
// Z1 = X·W1ᵀ, Z2 = H1·W2ᵀ and the δ chain ∂L/∂H1 = D2·W2, ∂L/∂X = D1·W1 are
// tcgen05 GEMMs; the weight gradients (reductions over the tile's rows) are
// FP32 outer products from the same shared-memory operands (hi + lo = the exact
// fp32 value), accumulated in registers across the CTA's tiles.  Activation
// operands use a padded k-chunk stride ((R + 1)·16 B, LBO) so the row-fixed
// float4 reads of those outer products are bank-conflict free.  M = 64 TMEM
// mapping (probed): row r ↔ lane 32⌊r/16⌋ + r mod 16.
constexpr int GB = 64;

namespace tc {
// padded K-major offset (k-chunk stride (R + 1)·4 floats)
__device__ __forceinline__ int kmajp(int r, int k, int R) {
  return (k >> 2) * ((R + 1) * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3);
}
// D[M×N] (=) A·Bᵀ over K, 3×TF32; A padded (R = M), B unpadded (R = N)
template <int M>
__device__ __forceinline__ void gemm3p(uint32_t tmem, const float* Ah, const float* Al,
                                       const float* Bh, const float* Bl, int N, int K) {
  const uint32_t id = idesc_tf32(M, N);
  const float* As[3] = {Ah, Al, Ah};
  const float* Bs[3] = {Bh, Bh, Bl};
  constexpr uint32_t lboA = (M + 1) * 16;
#pragma unroll
  for (int ps = 0; ps < 3; ++ps)
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t a = sdesc(smem_u32(As[ps]) + kk * 2 * lboA, lboA, 128);
      const uint64_t b = sdesc(smem_u32(Bs[ps]) + kk * 2 * (N * 16), N * 16, 128);
      mma(tmem, a, b, id, (ps > 0 || kk > 0) ? 1u : 0u);
    }
}
}  // namespace tc

// stage Wᵀ of W[N][K] (row-major global) as an unpadded K-major operand of
// Kt = N ... i.e. operand rows = K (the new N), operand k = N
__device__ __forceinline__ void stage_weight_t(const float* __restrict__ W, int N, int K, float* hi,
                                               float* lo) {
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e - r * K;   // W[r][k] → operand element (k, r), K rows
    const float x = W[e];
    const float h = tc::tf32_hi(x);
    hi[tc::kmaj(k, r, K)] = h;
    lo[tc::kmaj(k, r, K)] = x - h;
  }
}

__device__ __forceinline__ float4 ld_hl(const float* hi, const float* lo, int off) {
  const float4 a = *reinterpret_cast<const float4*>(hi + off);
  const float4 b = *reinterpret_cast<const float4*>(lo + off);
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ void st_hl(float* hi, float* lo, int off, const float v[4]) {
  float4 h, l;
  float* hp = &h.x;
  float* lp = &l.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) { hp[j] = tc::tf32_hi(v[j]); lp[j] = v[j] - hp[j]; }
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}

template <int F>
__global__ void __launch_bounds__(NT, 1)
deform_bwd_tc_kernel(const __grid_constant__ HashGridParams g, const float* __restrict__ table,
                     const float* __restrict__ mlp, int n, const int* __restrict__ idx,
                     const int* __restrict__ count, const float4* __restrict__ pos_opa,
                     const float4* __restrict__ g_mu, const float4* __restrict__ g_sigma,
                     float* __restrict__ g_table, float* __restrict__ g_mlp) {
  extern __shared__ __align__(1024) float4 smem4[];
  float* sm = reinterpret_cast<float*>(smem4);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int in = g.in;
  constexpr int PS = (GB + 1) * 4;           // padded k-chunk stride (floats)
  float* W1h = sm;                           // [64][in]  (n = o, k = j)
  float* W1l = W1h + HID * in;
  float* W2h = W1l + HID * in;               // [64][64]  (n = o, k = j)
  float* W2l = W2h + HID * HID;
  float* W2Th = W2l + HID * HID;             // [64][64]  (n = j, k = o)
  float* W2Tl = W2Th + HID * HID;
  float* W1Th = W2Tl + HID * HID;            // [in][64]  (n = j, k = o)
  float* W1Tl = W1Th + in * HID;
  float* sW3 = W1Tl + in * HID;              // fp32 [7][64] (+ pad)
  float* b1 = sW3 + 8 * HID;
  float* b2 = b1 + HID;
  float* Xh = b2 + HID;                      // [64][in] padded
  float* Xl = Xh + (in / 4) * PS;
  float* Ah = Xl + (in / 4) * PS;            // [64][64] padded: H1, then ∂L/∂Z1
  float* Al = Ah + (HID / 4) * PS;
  float* Dh = Al + (HID / 4) * PS;           // [64][64] padded: ∂L/∂Z2
  float* Dl = Dh + (HID / 4) * PS;
  float* H2 = Dl + (HID / 4) * PS;           // fp32 [64][68]
  float* D3 = H2 + GB * AS;                  // [64][8] ∂L/∂out
  const MlpOffsets off(in);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  stage_weight(mlp + off.W1, HID, HID, in, W1h, W1l);
  stage_weight(mlp + off.W2, HID, HID, HID, W2h, W2l);
  stage_weight_t(mlp + off.W2, HID, HID, W2Th, W2Tl);
  stage_weight_t(mlp + off.W1, HID, in, W1Th, W1Tl);
  for (int e = t; e < NOUT * HID; e += NT) sW3[e] = mlp[off.W3 + e];
  if (t < HID) { b1[t] = mlp[off.b1 + t]; b2[t] = mlp[off.b2 + t]; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;"
                 ::"r"(tc::smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_async_smem();
  tc::before_sync();
  __syncthreads();
  tc::after_sync();
  const uint32_t tmem = tbase;
  uint32_t phase = 0;

  // epilogue role: warp quadrant q (TMEM lanes 32q..), rows 16q + lane (lane < 16),
  // column half ch of a 64-column accumulator
  const int q = warp & 3, ch = warp >> 2;
  const bool erow = lane < 16;
  const int row = 16 * q + (lane & 15);
  const uint32_t lane_base = (uint32_t)(32 * q) << 16;

  // weight-gradient accumulators (registers, whole CTA lifetime)
  float a3[2] = {0.f, 0.f}, ab3 = 0.f;
  float a2[16], ab2[4], a1[16], ab1[4];
#pragma unroll
  for (int k = 0; k < 16; ++k) { a2[k] = 0.f; a1[k] = 0.f; }
#pragma unroll
  for (int k = 0; k < 4; ++k) { ab2[k] = 0.f; ab1[k] = 0.f; }
  const int o2 = (t >> 4) * 4, j2 = (t & 15) * 4;
  const int jb1 = in / 4;
  const bool has1 = t < 16 * jb1;
  const int o1 = has1 ? (t / jb1) * 4 : 0, j1 = has1 ? (t % jb1) * 4 : 0;

  const int m = count ? min(*count, n) : n;
  const int gi = t & (GB - 1), qq = t >> 6;
  int Lq = (g.L + 3) / 4;
  Lq = (Lq + (4 / F) - 1) / (4 / F) * (4 / F);
  const int l0 = min(g.L, qq * Lq), l1 = min(g.L, (qq + 1) * Lq);
  for (int tile = blockIdx.x; tile * GB < m; tile += gridDim.x) {
    // ---- encode X (hi/lo) and ∂L/∂out
    {
      const int k = tile * GB + gi;
      const bool valid = k < m;
      const int i = valid ? (idx ? idx[k] : k) : 0;
      float3 p = make_float3(0.f, 0.f, 0.f);
      if (valid) { const float4 po = pos_opa[i]; p = make_float3(po.x, po.y, po.z); }
      for (int l = l0; l < l1; ++l) {
        float acc[F];
#pragma unroll
        for (int f = 0; f < F; ++f) acc[f] = 0.f;
        if (valid) {
          uint32_t rw[8];
          float wt[8];
          level_corners(g, l, p, rw, wt);
          const float* tab = table + (size_t)l * g.T * F;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if constexpr (F == 4) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(tab) + rw[c]);
              acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y; acc[2] += wt[c] * v.z; acc[3] += wt[c] * v.w;
            } else if constexpr (F == 2) {
              const float2 v = __ldg(reinterpret_cast<const float2*>(tab) + rw[c]);
              acc[0] += wt[c] * v.x; acc[1] += wt[c] * v.y;
            } else {
              acc[0] += wt[c] * __ldg(tab + rw[c]);
            }
          }
        }
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const int o = tc::kmajp(gi, l * F + f, GB);
          const float h = tc::tf32_hi(acc[f]);
          Xh[o] = h;
          Xl[o] = acc[f] - h;
        }
      }
      if (qq == 0) {
        const float4 d = valid ? g_mu[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        D3[gi * 8 + 0] = d.x; D3[gi * 8 + 1] = d.y; D3[gi * 8 + 2] = d.z; D3[gi * 8 + 7] = 0.f;
      } else if (qq == 1) {
        const float4 d = valid ? g_sigma[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        D3[gi * 8 + 3] = d.x; D3[gi * 8 + 4] = d.y; D3[gi * 8 + 5] = d.z; D3[gi * 8 + 6] = d.w;
      }
    }
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // Z1 = X·W1ᵀ → TMEM [0, 64)
      tc::gemm3p<GB>(tmem, Xh, Xl, W1h, W1l, HID, in);
      tc::commit(&mbar);
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    uint32_t m1 = 0;   // ReLU mask of this thread's 32 columns of row `row`
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      float v[16];
      tc::ld16(tmem + lane_base + 32 * ch + 16 * hlf, v);
      if (erow) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int c = 32 * ch + 16 * hlf + 4 * q4;
          float h[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float z = v[4 * q4 + j] + b1[c + j];
            h[j] = fmaxf(z, 0.f);
            if (z > 0.f) m1 |= 1u << (16 * hlf + 4 * q4 + j);
          }
          st_hl(Ah, Al, tc::kmajp(row, c, GB), h);
        }
      }
    }
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // Z2 = H1·W2ᵀ → TMEM [64, 128)
      tc::gemm3p<GB>(tmem + 64, Ah, Al, W2h, W2l, HID, HID);
      tc::commit(&mbar);
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    {
      float d3[NOUT];
#pragma unroll
      for (int c = 0; c < NOUT; ++c) d3[c] = D3[row * 8 + c];
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        float v[16];
        tc::ld16(tmem + lane_base + 64 + 32 * ch + 16 * hlf, v);
        if (erow) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int c = 32 * ch + 16 * hlf + 4 * q4;
            float d[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float z = v[4 * q4 + j] + b2[c + j];
              H2[row * AS + c + j] = fmaxf(z, 0.f);
              float sacc = 0.f;
#pragma unroll
              for (int cc = 0; cc < NOUT; ++cc) sacc = fmaf(sW3[cc * HID + c + j], d3[cc], sacc);
              d[j] = z > 0.f ? sacc : 0.f;
            }
            st_hl(Dh, Dl, tc::kmajp(row, c, GB), d);
          }
        }
      }
    }
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // ∂L/∂H1 = D2·W2 → TMEM [64, 128)
      tc::gemm3p<GB>(tmem + 64, Dh, Dl, W2Th, W2Tl, HID, HID);
      tc::commit(&mbar);
    }
    // FP32 weight gradients from shared memory while the MMA runs
#pragma unroll 4
    for (int r = 0; r < GB; ++r) {
      const float4 dv = ld_hl(Dh, Dl, tc::kmajp(r, o2, GB));
      const float4 hv = ld_hl(Ah, Al, tc::kmajp(r, j2, GB));
      const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, hh[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int b = 0; b < 4; ++b) a2[4 * a + b] = fmaf(dd[a], hh[b], a2[4 * a + b]);
      }
      if (j2 == 0) { ab2[0] += dd[0]; ab2[1] += dd[1]; ab2[2] += dd[2]; ab2[3] += dd[3]; }
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int e = t + rr * NT;
      if (e < NOUT * HID) {
        const int c = e >> 6, j = e & 63;
        float sacc = 0.f;
#pragma unroll 8
        for (int r = 0; r < GB; ++r) sacc = fmaf(D3[r * 8 + c], H2[r * AS + j], sacc);
        a3[rr] += sacc;
      }
    }
    if (t < NOUT) {
      float sacc = 0.f;
      for (int r = 0; r < GB; ++r) sacc += D3[r * 8 + t];
      ab3 += sacc;
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    __syncthreads();   // every read of H1 (A buffer) is done before ∂L/∂Z1 overwrites it
#pragma unroll
    for (int hlf = 0; hlf < 2; ++hlf) {
      float v[16];
      tc::ld16(tmem + lane_base + 64 + 32 * ch + 16 * hlf, v);
      if (erow) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int c = 32 * ch + 16 * hlf + 4 * q4;
          float d[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) d[j] = ((m1 >> (16 * hlf + 4 * q4 + j)) & 1u) ? v[4 * q4 + j] : 0.f;
          st_hl(Ah, Al, tc::kmajp(row, c, GB), d);
        }
      }
    }
    tc::fence_async_smem();
    tc::before_sync();
    __syncthreads();
    tc::after_sync();
    if (t == 0) {   // ∂L/∂X = D1·W1 → TMEM [0, in)
      tc::gemm3p<GB>(tmem, Ah, Al, W1Th, W1Tl, in, HID);
      tc::commit(&mbar);
    }
    if (has1) {
#pragma unroll 4
      for (int r = 0; r < GB; ++r) {
        const float4 dv = ld_hl(Ah, Al, tc::kmajp(r, o1, GB));
        const float4 xv = ld_hl(Xh, Xl, tc::kmajp(r, j1, GB));
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, xx[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int b = 0; b < 4; ++b) a1[4 * a + b] = fmaf(dd[a], xx[b], a1[4 * a + b]);
        }
        if (j1 == 0) { ab1[0] += dd[0]; ab1[1] += dd[1]; ab1[2] += dd[2]; ab1[3] += dd[3]; }
      }
    }
    tc::wait(&mbar, phase); phase ^= 1u;
    tc::after_sync();
    // ∂L/∂X columns [16·ch, 16·ch + 16) of row `row` → table scatter
    if (16 * ch < in) {
      float v[16];
      tc::ld16(tmem + lane_base + 16 * ch, v);
      const int k = tile * GB + row;
      if (erow && k < m) {
        const int i = idx ? idx[k] : k;
        const float4 po = pos_opa[i];
        const float3 p = make_float3(po.x, po.y, po.z);
        constexpr int LPC = 16 / F;   // levels per 16 columns
#pragma unroll
        for (int ll = 0; ll < LPC; ++ll) {
          const int l = 16 * ch / F + ll;
          if (l < g.L) {
            uint32_t rw[8];
            float wt[8];
            level_corners(g, l, p, rw, wt);
            float* tab = g_table + (size_t)l * g.T * F;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              if constexpr (F == 4) {
                red_add_v4(reinterpret_cast<float4*>(tab) + rw[c],
                           make_float4(wt[c] * v[4 * ll], wt[c] * v[4 * ll + 1],
                                       wt[c] * v[4 * ll + 2], wt[c] * v[4 * ll + 3]));
              } else if constexpr (F == 2) {
                red_add_v2(tab + (size_t)rw[c] * 2, wt[c] * v[2 * ll], wt[c] * v[2 * ll + 1]);
              } else {
                atomicAdd(tab + rw[c], wt[c] * v[ll]);
              }
            }
          }
        }
      }
    }
    tc::before_sync();
    __syncthreads();
  }

  // ---- flush the weight gradients (once per CTA)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int e = t + r * NT;
    if (e < NOUT * HID) atomicAdd(g_mlp + off.W3 + e, a3[r]);
  }
  if (t < NOUT) atomicAdd(g_mlp + off.b3 + t, ab3);
#pragma unroll
  for (int a = 0; a < 4; ++a) {
#pragma unroll
    for (int b = 0; b < 4; ++b) atomicAdd(g_mlp + off.W2 + (o2 + a) * HID + j2 + b, a2[4 * a + b]);
    if (j2 == 0) atomicAdd(g_mlp + off.b2 + o2 + a, ab2[a]);
  }
  if (has1) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int b = 0; b < 4; ++b) atomicAdd(g_mlp + off.W1 + (o1 + a) * in + j1 + b, a1[4 * a + b]);
      if (j1 == 0) atomicAdd(g_mlp + off.b1 + o1 + a, ab1[a]);
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---- stable partition: idx_dyn = ascending {i : mask[i] ≠ 0}, idx_st = the rest
constexpr int PB = 1024;

__global__ void __launch_bounds__(PB) part_count_kernel(int n, const uint8_t* __restrict__ mask,
                                                       int* __restrict__ bcount) {
  __shared__ int wsum[PB / 32];
  const int i = blockIdx.x * PB + threadIdx.x;
  const bool d = i < n && mask[i] != 0;
  const unsigned b = __ballot_sync(0xffffffffu, d);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = wsum[threadIdx.x];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
    if (threadIdx.x == 0) bcount[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(PB) part_scan_kernel(int nb, int n, const int* __restrict__ bcount,
                                                      int* __restrict__ boff, int* __restrict__ counts) {
  __shared__ int wsum[PB / 32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += PB) {
    const int b = base + threadIdx.x;
    const int v = b < nb ? bcount[b] : 0;
    int incl = v;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, s);
      if (lane >= s) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int x = wsum[lane];
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, x, s);
        if (lane >= s) x += u;
      }
      wsum[lane] = x;   // inclusive warp totals
    }
    __syncthreads();
    const int c = carry;
    if (b < nb) boff[b] = c + (w ? wsum[w - 1] : 0) + incl - v;
    __syncthreads();
    if (threadIdx.x == PB - 1) carry = c + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) { counts[0] = carry; counts[1] = n - carry; }
}

__global__ void __launch_bounds__(PB) part_scatter_kernel(int n, const uint8_t* __restrict__ mask,
                                                         const int* __restrict__ boff,
                                                         int* __restrict__ idx_dyn,
                                                         int* __restrict__ idx_st) {
  __shared__ int wsum[PB / 32];
  const int i = blockIdx.x * PB + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool in_range = i < n;
  const bool d = in_range && mask[i] != 0;
  const unsigned b = __ballot_sync(0xffffffffu, d);
  if (lane == 0) wsum[w] = __popc(b);
  __syncthreads();
  int before = 0;   // dynamic Gaussians in earlier warps of this block
  for (int q = 0; q < w; ++q) before += wsum[q];
  const int rank = before + __popc(b & ((1u << lane) - 1u));
  if (!in_range) return;
  const int dyn_base = boff[blockIdx.x];
  if (d) {
    idx_dyn[dyn_base + rank] = i;
  } else if (idx_st != nullptr) {
    const int st_base = blockIdx.x * PB - dyn_base;
    idx_st[st_base + (threadIdx.x - rank)] = i;
  }
}

template <int F>
size_t fwd_smem(int in) {
  return sizeof(float) * (size_t)(in * HID + HID + HID * HID + HID + NOUT * HID + 8 + 2 * GT * AS);
}
template <int F>
size_t bwd_smem(int in) {
  return sizeof(float) * (size_t)(2 * in * HID + HID + 2 * HID * HID + HID + NOUT * HID +
                                  GT * x_stride(in) + 2 * GT * AS + GT * 8);
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

size_t fwd_tc_smem(int in) {
  return sizeof(float) * (size_t)(2 * HID * in + 2 * HID * HID + 2 * 16 * HID + 2 * HID + 16 +
                                  2 * GT * in + 2 * GT * HID);
}

// The tcgen05 kernels serve every field shape they are defined for (K a
// multiple of 8: kind::tf32 consumes K in steps of 8); other shapes, and the
// F = 2 backward (measured slower on tcgen05), run the FP32 SIMT
// kernels.
constexpr bool use_tc() { return true; }

template <int F>
cudaError_t fwd_launch(const HashGridParams& g, const float* table, const float* mlp, int n,
                       const int* idx, const int* count, const float4* pos_opa, float4* mu,
                       float4* sigma, cudaStream_t s) {
  if (use_tc() && g.in % 8 == 0) {   // kind::tf32 consumes K in steps of 8
    const size_t sm = fwd_tc_smem(g.in);
    cudaError_t e = cudaFuncSetAttribute(deform_fwd_tc_kernel<F>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = max(1, min(div_up(n, GT), sm_count()));
    deform_fwd_tc_kernel<F><<<grid, NT_TC, sm, s>>>(g, table, mlp, n, idx, count, pos_opa, mu, sigma);
    launch_counted();
    return cudaGetLastError();
  }
  const size_t sm = fwd_smem<F>(g.in);
  cudaError_t e = cudaFuncSetAttribute(deform_fwd_kernel<F>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int grid = max(1, min(div_up(n, GT), 2 * sm_count()));
  deform_fwd_kernel<F><<<grid, NT, sm, s>>>(g, table, mlp, n, idx, count, pos_opa, mu, sigma);
  launch_counted();
  return cudaGetLastError();
}

size_t bwd_tc_smem(int in) {
  const int PS = (GB + 1) * 4;
  return sizeof(float) * (size_t)(2 * HID * in + 2 * HID * HID + 2 * HID * HID + 2 * in * HID +
                                  8 * HID + 2 * HID + 2 * (in / 4) * PS + 4 * (HID / 4) * PS +
                                  GB * AS + GB * 8);
}

template <int F>
cudaError_t bwd_launch(const HashGridParams& g, const float* table, const float* mlp, int n,
                       const int* idx, const int* count, const float4* pos_opa,
                       const float4* g_mu, const float4* g_sigma, float* g_table, float* g_mlp,
                       cudaStream_t s) {
  // The tcgen05 backward is used where it measured faster: the F = 4 field (𝓗_dyn, in = 32:
  // 287 → 243 µs for 90k Gaussians).  For 𝓗_st (F = 2, in = 16) its serialised per-tile
  // MMA/epilogue phases cost more than they save (415 → 444 µs), so the SIMT kernel runs;
  // in > 32 would not fit the M = 64 operands in shared memory.
  if (use_tc() && F == 4 && g.in <= 32 && g.in % 8 == 0) {
    const size_t sm = bwd_tc_smem(g.in);
    cudaError_t e = cudaFuncSetAttribute(deform_bwd_tc_kernel<F>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const int grid = max(1, min(div_up(n, GB), sm_count()));
    deform_bwd_tc_kernel<F><<<grid, NT, sm, s>>>(g, table, mlp, n, idx, count, pos_opa, g_mu,
                                                 g_sigma, g_table, g_mlp);
    launch_counted();
    return cudaGetLastError();
  }
  const size_t sm = bwd_smem<F>(g.in);
  cudaError_t e = cudaFuncSetAttribute(deform_bwd_kernel<F>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  const int grid = max(1, min(div_up(n, GT), sm_count()));
  deform_bwd_kernel<F><<<grid, NT, sm, s>>>(g, table, mlp, n, idx, count, pos_opa, g_mu, g_sigma,
                                            g_table, g_mlp);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace

size_t partition_workspace(int n) { return sizeof(int) * 2 * (size_t)max(1, div_up(n, PB)); }

cudaError_t launch_partition(int n, const uint8_t* mask, int* idx_dyn, int* idx_st, int* counts,
                             void* ws, cudaStream_t s) {
  const int nb = max(1, div_up(n, PB));
  int* bcount = static_cast<int*>(ws);
  int* boff = bcount + nb;
  part_count_kernel<<<nb, PB, 0, s>>>(n, mask, bcount);
  part_scan_kernel<<<1, PB, 0, s>>>(nb, n, bcount, boff, counts);
  part_scatter_kernel<<<nb, PB, 0, s>>>(n, mask, boff, idx_dyn, idx_st);
  launch_counted(3);
  return cudaGetLastError();
}

cudaError_t launch_deform_fwd(const HashGridParams& g, const float* table, const float* mlp, int n,
                              const int* idx, const int* count, const float4* pos_opa, float4* mu,
                              float4* sigma, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (g.F) {
    case 4: return fwd_launch<4>(g, table, mlp, n, idx, count, pos_opa, mu, sigma, s);
    case 2: return fwd_launch<2>(g, table, mlp, n, idx, count, pos_opa, mu, sigma, s);
    default: return fwd_launch<1>(g, table, mlp, n, idx, count, pos_opa, mu, sigma, s);
  }
}

cudaError_t launch_deform_bwd(const HashGridParams& g, const float* table, const float* mlp, int n,
                              const int* idx, const int* count, const float4* pos_opa,
                              const float4* g_mu, const float4* g_sigma, float* g_table,
                              float* g_mlp, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (g.F) {
    case 4: return bwd_launch<4>(g, table, mlp, n, idx, count, pos_opa, g_mu, g_sigma, g_table, g_mlp, s);
    case 2: return bwd_launch<2>(g, table, mlp, n, idx, count, pos_opa, g_mu, g_sigma, g_table, g_mlp, s);
    default: return bwd_launch<1>(g, table, mlp, n, idx, count, pos_opa, g_mu, g_sigma, g_table, g_mlp, s);
  }
}

}  // namespace dass
