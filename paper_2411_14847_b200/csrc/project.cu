// project.cu — dass_project / dass_project_views: EWA projection + SH colour
// (Eqs. 5-7, colour P:351).  One thread per Gaussian, looping over
// the views of the launch so the 240 B/G of parameters are read once for all
// views (multi-view batching).  HBM-bound.
//
// Three precisions, by purpose:
//  * the KEY CHAIN (depth bits, pixel box, visibility) in IEEE fp32 with
//    explicit-rounding intrinsics, in exactly the op order documented in
//    include/dass.h, so the (tile|depth) keys are reproducible bit-for-bit;
//  * the per-pixel records (u, v, conic) in fp64 then rounded once to fp32:
//    the mean is stored as fp32 hi + fp16 lo so the renderer can form the
//    tile-local offset u − X to ~1e-7 px instead of ulp(1000) = 6e-5 px;
//  * the SH colour in fp32.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "sh.cuh"

namespace dass {
namespace {

constexpr int MAXV = 32;  // views per launch (kernel-parameter budget)

struct ProjectArgs {
  CamParams cam[MAXV];
  int vpt;                 // views per thread (blockIdx.y groups)
  int num_views;
  int n;
  int view_offset;  // records of view v go to [(view_offset + v)·n, …)
  const float4* pos_opa;
  const float4* scale;
  const float4* rot;
  const float4* sh;
  const uint8_t* keep;
  float4* xy_depth;
  float4* conic_opa;
  float4* rgb;
  uint2* box;
  uint4* rows;      // A50 tile-row spans
  uint32_t* tiles;
};

#define FM __fmul_rn
#define FA __fadd_rn
#define FS __fsub_rn
#define FD __fdiv_rn

struct KeyResult {
  bool visible;
  float z;
  int x0, x1, y0, y1;
  uint32_t tiles;
  uint4 rows;
};

// KEY CHAIN steps 12-13 of include/dass.h (A50): per tile row of the box, the
// tile columns the ellipse {d : dᵀ Σ'⁻¹ d ≤ R2} reaches in the row's band of pixel
// rows, padded by one pixel; R2 = an upper bound of 2·ln(255·o) (ln m ≤ m − 1 on
// the mantissa) × 1.01 + 0.05.  Boxes of more than 8 tile rows or 255 tile
// columns keep every box tile (rows = all ones).  Every op individually rounded
// (the oracle's replica must get the same bits).  Returns the tile count.
// Step 12: the threshold R2 from o (view-independent).
__device__ __forceinline__ float footprint_r2(float o) {
  const float xo = FM(255.0f, o);
  const uint32_t bits = __float_as_uint(xo);
  const int e = (int)(bits >> 23) - 127;
  const float mf = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);
  const float L = FA(FM((float)e, 0.693147182f), FS(mf, 1.0f));
  return FA(FM(FM(2.0f, L), 1.01f), 0.05f);
}

// Step 13 for one view.
__device__ __forceinline__ uint32_t footprint_rows(float ca, float cb, float cc, float det, float u,
                                                   float v, float R2, int x0, int x1, int y0, int y1,
                                                   uint4& rows) {
  const int tx0 = x0 / 16, tx1 = x1 / 16, ty0 = y0 / 16, ty1 = y1 / 16;
  if (ty1 - ty0 + 1 > 8 || tx1 - tx0 + 1 > 255) {
    rows = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    return (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
  }
  const float sxa = __fsqrt_rn(FM(R2, ca));
  const float tq = __fsqrt_rn(FD(R2, ca));
  const float dyL = -FM(cb, tq), dyR = FM(cb, tq);
  const float crr = FM(cc, R2);
  const float ey = __fsqrt_rn(crr);
  const float icc = FD(1.0f, cc);
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  uint32_t total = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int ty = ty0 + k;
    uint32_t span = 0x00FFu;   // empty: lo = 255 > hi = 0
    if (ty <= ty1) {
      const int Y0 = max(y0, 16 * ty), Y1 = min(y1, 16 * ty + 15);
      const float d0 = fmaxf(FS((float)Y0, v), -ey);
      const float d1 = fminf(FS((float)Y1, v), ey);
      if (d0 <= d1) {
        const float h0 = __fsqrt_rn(fmaxf(0.0f, FM(det, FS(crr, FM(d0, d0)))));
        const float h1 = __fsqrt_rn(fmaxf(0.0f, FM(det, FS(crr, FM(d1, d1)))));
        const float l0 = FM(FS(FM(cb, d0), h0), icc), l1 = FM(FS(FM(cb, d1), h1), icc);
        const float r0 = FM(FA(FM(cb, d0), h0), icc), r1 = FM(FA(FM(cb, d1), h1), icc);
        const float lo = (d0 <= dyL && dyL <= d1) ? -sxa : fminf(l0, l1);
        const float hi = (d0 <= dyR && dyR <= d1) ? sxa : fmaxf(r0, r1);
        const float X0f = fmaxf((float)x0, FS(FA(u, lo), 1.0f));
        const float X1f = fminf((float)x1, FA(FA(u, hi), 1.0f));
        const float c0 = ceilf(X0f), c1 = floorf(X1f);
        if (c0 <= c1) {
          const int lo_t = (int)c0 / 16 - tx0, hi_t = (int)c1 / 16 - tx0;
          span = (uint32_t)lo_t | ((uint32_t)hi_t << 8);
          total += (uint32_t)(hi_t - lo_t + 1);
        }
      }
    }
    w[k >> 1] |= span << (16 * (k & 1));
  }
  rows = make_uint4(w[0], w[1], w[2], w[3]);
  return total;
}

// The view-independent part of the KEY CHAIN (steps 3-5 and 12): q̂, R(q̂) and
// Σ = m mᵀ with m = R·diag(s), and R2.  Computed once per Gaussian by the keys
// kernel; the per-view part below uses the same values in the same op order, so
// the result is the chain of include/dass.h bit for bit.
struct KeyPrep {
  bool qok;        // nq > 0 and finite
  float S[6];      // Σ00, Σ01, Σ02, Σ11, Σ12, Σ22
  float R2;
};

__device__ __forceinline__ KeyPrep key_prep(float o, float s0, float s1, float s2, float4 q) {
  KeyPrep kp;
  kp.R2 = footprint_r2(o);
  const float nn = FA(FA(FA(FM(q.x, q.x), FM(q.y, q.y)), FM(q.z, q.z)), FM(q.w, q.w));
  const float nq = __fsqrt_rn(nn);
  kp.qok = (nq > 0.f) && isfinite(nq);
  if (!kp.qok) {
#pragma unroll
    for (int k = 0; k < 6; ++k) kp.S[k] = 0.f;
    return kp;
  }
  const float w = FD(q.x, nq), x = FD(q.y, nq), y = FD(q.z, nq), z = FD(q.w, nq);
  const float xx = FM(x, x), yy = FM(y, y), zz = FM(z, z), xy = FM(x, y), xz = FM(x, z),
              yz = FM(y, z), wx = FM(w, x), wy = FM(w, y), wz = FM(w, z);
  float R[3][3];
  R[0][0] = FS(1.f, FM(2.f, FA(yy, zz)));
  R[0][1] = FM(2.f, FS(xy, wz));
  R[0][2] = FM(2.f, FA(xz, wy));
  R[1][0] = FM(2.f, FA(xy, wz));
  R[1][1] = FS(1.f, FM(2.f, FA(xx, zz)));
  R[1][2] = FM(2.f, FS(yz, wx));
  R[2][0] = FM(2.f, FS(xz, wy));
  R[2][1] = FM(2.f, FA(yz, wx));
  R[2][2] = FS(1.f, FM(2.f, FA(xx, yy)));
  const float s[3] = {s0, s1, s2};
  float m[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) m[a][b] = FM(R[a][b], s[b]);
  int k = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = a; b < 3; ++b)
      kp.S[k++] = FA(FA(FM(m[a][0], m[b][0]), FM(m[a][1], m[b][1])), FM(m[a][2], m[b][2]));
  return kp;
}

// The per-view part of the KEY CHAIN (steps 1-2, 6-11, 13).  lx, ly: step 6's
// clamp limits of this camera (computed once per block, same ops).
__device__ __forceinline__ KeyResult key_view(const CamParams& c, float lx, float ly, float px,
                                              float py, float pz, float o, const KeyPrep& kp) {
  KeyResult k;
  k.visible = false; k.z = 0.f; k.x0 = 1; k.x1 = 0; k.y0 = 1; k.y1 = 0;
  k.tiles = 0; k.rows = make_uint4(0u, 0u, 0u, 0u);
  const float* V = c.V;
  float t[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    t[a] = FA(FA(FA(FM(V[4 * a + 0], px), FM(V[4 * a + 1], py)), FM(V[4 * a + 2], pz)), V[4 * a + 3]);
  if (!(t[2] > c.near_plane)) return k;
  if (!kp.qok) return k;
  const float S[3][3] = {{kp.S[0], kp.S[1], kp.S[2]}, {kp.S[1], kp.S[3], kp.S[4]}, {kp.S[2], kp.S[4], kp.S[5]}};
  const float Wf = (float)c.W, Hf = (float)c.H;
  const float xt = FM(fminf(lx, fmaxf(-lx, FD(t[0], t[2]))), t[2]);
  const float yt = FM(fminf(ly, fmaxf(-ly, FD(t[1], t[2]))), t[2]);
  const float tz2 = FM(t[2], t[2]);
  const float J00 = FD(c.fx, t[2]);
  const float J02 = -FD(FM(c.fx, xt), tz2);
  const float J11 = FD(c.fy, t[2]);
  const float J12 = -FD(FM(c.fy, yt), tz2);
  float M[2][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    M[0][b] = FA(FM(J00, V[0 * 4 + b]), FM(J02, V[2 * 4 + b]));
    M[1][b] = FA(FM(J11, V[1 * 4 + b]), FM(J12, V[2 * 4 + b]));
  }
  float P[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      P[a][b] = FA(FA(FM(M[a][0], S[0][b]), FM(M[a][1], S[1][b])), FM(M[a][2], S[2][b]));
  const float ca = FA(FA(FA(FM(P[0][0], M[0][0]), FM(P[0][1], M[0][1])), FM(P[0][2], M[0][2])), 0.3f);
  const float cb = FA(FA(FM(P[0][0], M[1][0]), FM(P[0][1], M[1][1])), FM(P[0][2], M[1][2]));
  const float cc = FA(FA(FA(FM(P[1][0], M[1][0]), FM(P[1][1], M[1][1])), FM(P[1][2], M[1][2])), 0.3f);
  const float det = FS(FM(ca, cc), FM(cb, cb));
  if (!(det > 0.f)) return k;
  const float mid = FM(0.5f, FA(ca, cc));
  const float lam = FA(mid, __fsqrt_rn(fmaxf(0.1f, FS(FM(mid, mid), det))));
  const float r = ceilf(FM(3.0f, __fsqrt_rn(lam)));
  const float u = FA(FD(FM(c.fx, t[0]), t[2]), c.cx);
  const float v = FA(FD(FM(c.fy, t[1]), t[2]), c.cy);
  if (!isfinite(u) || !isfinite(v) || !isfinite(lam)) return k;
  const float fx0 = fmaxf(0.f, ceilf(FS(u, r)));
  const float fx1 = fminf(FS(Wf, 1.f), floorf(FA(u, r)));
  const float fy0 = fmaxf(0.f, ceilf(FS(v, r)));
  const float fy1 = fminf(FS(Hf, 1.f), floorf(FA(v, r)));
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) return k;
  if (!(o >= ALPHA_MIN)) return k;
  k.visible = true;
  k.z = t[2];
  k.x0 = (int)fx0; k.x1 = (int)fx1; k.y0 = (int)fy0; k.y1 = (int)fy1;
  k.tiles = footprint_rows(ca, cb, cc, det, u, v, kp.R2, k.x0, k.x1, k.y0, k.y1, k.rows);   // 12-13
  return k;
}

#undef FM
#undef FA
#undef FS
#undef FD

// fp64 records: tile-independent mean (hi/lo) and the conic of Eq. 7 in its
// Cholesky form (A, β, γ): K = [[A, B], [B, C]] with B = A·β, C = γ + A·β²,
// so A dx² + 2B dx dy + C dy² = A(dx + β dy)² + γ dy² (common.cuh, A35).
struct Records {
  float u_hi, v_hi;
  __half u_lo, v_lo;
  float A, beta, gamma;
};

__device__ __forceinline__ Records accurate_records(const CamParams& c, float4 po, float4 sc,
                                                    float4 q, float keepf) {
  Records r;
  const double px = po.x, py = po.y, pz = po.z;
  double t[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    t[a] = (double)c.V[4 * a] * px + (double)c.V[4 * a + 1] * py + (double)c.V[4 * a + 2] * pz +
           (double)c.V[4 * a + 3];
  const double nq = sqrt((double)q.x * q.x + (double)q.y * q.y + (double)q.z * q.z + (double)q.w * q.w);
  const double inq = 1.0 / nq;   // reciprocals instead of repeated fp64 divisions
  const double w = q.x * inq, x = q.y * inq, y = q.z * inq, z = q.w * inq;
  double R[3][3];
  R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
  R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
  R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
  const double s[3] = {(double)sc.x * keepf, (double)sc.y * keepf, (double)sc.z * keepf};
  // N = J W R S (2×3); Σ' = N Nᵀ + 0.3 I
  const double lx = 1.3 * c.W / (2.0 * c.fx), ly = 1.3 * c.H / (2.0 * c.fy);
  const double itz = 1.0 / t[2], itz2 = itz * itz;
  const double xt = t[2] * fmin(lx, fmax(-lx, t[0] * itz));
  const double yt = t[2] * fmin(ly, fmax(-ly, t[1] * itz));
  const double J00 = c.fx * itz, J02 = -c.fx * xt * itz2;
  const double J11 = c.fy * itz, J12 = -c.fy * yt * itz2;
  double M[2][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    M[0][b] = J00 * c.V[b] + J02 * c.V[8 + b];
    M[1][b] = J11 * c.V[4 + b] + J12 * c.V[8 + b];
  }
  double N[2][3];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      N[a][b] = (M[a][0] * R[0][b] + M[a][1] * R[1][b] + M[a][2] * R[2][b]) * s[b];
  const double a2 = N[0][0] * N[0][0] + N[0][1] * N[0][1] + N[0][2] * N[0][2] + 0.3;
  const double b2 = N[0][0] * N[1][0] + N[0][1] * N[1][1] + N[0][2] * N[1][2];
  const double c2 = N[1][0] * N[1][0] + N[1][1] * N[1][1] + N[1][2] * N[1][2] + 0.3;
  const double det = a2 * c2 - b2 * b2;
  const double ic = 1.0 / c2;
  r.A = (float)(c2 / det);
  r.beta = (float)(-b2 * ic);    // B/A = (−b/det)/(c/det)
  r.gamma = (float)ic;           // C − B²/A = (ac − b²)/(det·c) = 1/c
  const double u = c.fx * t[0] * itz + c.cx;
  const double v = c.fy * t[1] * itz + c.cy;
  r.u_hi = (float)u;
  r.v_hi = (float)v;
  r.u_lo = __double2half(u - (double)r.u_hi);
  r.v_lo = __double2half(v - (double)r.v_hi);
  return r;
}

// The projection runs as two launches ("a1 in two parts"):
//  * project_keys_kernel — the KEY CHAIN and its footprint: depth, box, tile rows,
//    tile count, i.e. everything dass_bin_sort reads; xy_depth gets (0, 0, z, 0);
//  * project_records_kernel — the fp64 records and the SH colour, which only the
//    raster kernels read: xy_depth's (u_hi, v_hi) and lo word, conic_opa, rgb.
// The two write disjoint bytes, so the records may run on a side stream while the
// views' sorts (which read xy_depth.z only) run — off the step's critical path.
__global__ void __launch_bounds__(256) project_keys_kernel(const __grid_constant__ ProjectArgs a) {
  // step 6's per-camera clamp limits, once per block (the same ops as the chain)
  __shared__ float s_l[MAXV][2];
  const int va = blockIdx.y * a.vpt, vb = min(a.num_views, va + a.vpt);
  if ((int)threadIdx.x < vb - va) {
    const CamParams& c = a.cam[va + threadIdx.x];
    s_l[threadIdx.x][0] = __fdiv_rn(__fmul_rn(1.3f, (float)c.W), __fmul_rn(2.0f, c.fx));
    s_l[threadIdx.x][1] = __fdiv_rn(__fmul_rn(1.3f, (float)c.H), __fmul_rn(2.0f, c.fy));
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const float4 po = a.pos_opa[i];
  const float4 sc = a.scale[i];
  const float4 q = a.rot[i];
  const bool kept = a.keep == nullptr || a.keep[i] != 0;
  const float o_eff = kept ? po.w : 0.f;
  const float keepf = kept ? 1.f : 0.f;
  const KeyPrep kp = key_prep(o_eff, sc.x * keepf, sc.y * keepf, sc.z * keepf, q);
  for (int v = va; v < vb; ++v) {
    const CamParams& c = a.cam[v];
    const size_t o = (size_t)(a.view_offset + v) * a.n + i;
    const KeyResult k = key_view(c, s_l[v - va][0], s_l[v - va][1], po.x, po.y, po.z, o_eff, kp);
    if (!k.visible) {
      a.xy_depth[o] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.box[o] = make_uint2(1u, 1u);     // x0 = 1 > x1 = 0: the invisible sentinel
      a.rows[o] = make_uint4(0u, 0u, 0u, 0u);
      a.tiles[o] = 0u;
      continue;
    }
    a.xy_depth[o] = make_float4(0.f, 0.f, k.z, 0.f);
    a.box[o] = make_uint2((uint32_t)k.x0 | ((uint32_t)k.x1 << 16), (uint32_t)k.y0 | ((uint32_t)k.y1 << 16));
    a.rows[o] = k.rows;
    a.tiles[o] = k.tiles;
  }
}

template <int DEG>
__global__ void __launch_bounds__(256) project_records_kernel(const __grid_constant__ ProjectArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const float4 po = a.pos_opa[i];
  const float4 sc = a.scale[i];
  const float4 q = a.rot[i];
  const bool kept = a.keep == nullptr || a.keep[i] != 0;
  const float o_eff = kept ? po.w : 0.f;
  const float keepf = kept ? 1.f : 0.f;
  using L = SHLayout<DEG>;
  const int va = blockIdx.y * a.vpt, vb = min(a.num_views, va + a.vpt);
  for (int v = va; v < vb; ++v) {
    const CamParams& c = a.cam[v];
    const size_t o = (size_t)(a.view_offset + v) * a.n + i;
    const uint2 bx = a.box[o];           // the key chain's visibility decision
    if ((bx.x & 0xFFFFu) > (bx.x >> 16)) {
      a.conic_opa[o] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.rgb[o] = make_float4(0.f, 0.f, 0.f, 0.f);
      continue;
    }
    const Records r = accurate_records(c, po, sc, q, keepf);
    // colour: d = (p − c_cam)/‖p − c_cam‖, col = Σ Y_k(d) sh_k + 0.5, clamp ≥ 0
    float dx = po.x - c.campos[0], dy = po.y - c.campos[1], dz = po.z - c.campos[2];
    const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
    dx *= inv; dy *= inv; dz *= inv;
    float Y[L::NC];
    sh_eval<DEG>(dx, dy, dz, Y);
    // SH planes re-read per view (L1/L2-resident after the first view) instead
    // of pinning 4·K4 registers across the view loop
    float col[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int j = 0; j < L::K4; ++j) {
      const float4 c4 = __ldg(a.sh + (size_t)j * a.n + i);
      const float cf[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int f = 4 * j + e;   // coefficient-major, channel-minor: f = 3·kk + ch
        if (f < L::NF) col[f % 3] += Y[f / 3] * cf[e];
      }
    }
    int bits = 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      if (col[ch] < 0.f) { bits |= 1 << ch; col[ch] = 0.f; }
    const __half2 lo = __halves2half2(r.u_lo, r.v_lo);
    float* xyd = reinterpret_cast<float*>(a.xy_depth + o);   // z (word 2) is the key chain's
    *reinterpret_cast<float2*>(xyd) = make_float2(r.u_hi, r.v_hi);
    xyd[3] = __uint_as_float(*(const uint32_t*)&lo);
    a.conic_opa[o] = make_float4(r.A, r.beta, r.gamma, o_eff);
    a.rgb[o] = make_float4(col[0], col[1], col[2], (float)bits);
  }
}

}  // namespace

static ProjectArgs project_args(const CamParams* cams, int v0, int num_views, int n,
                                const float4* pos_opa, const float4* scale, const float4* rot,
                                const float4* sh, const uint8_t* keep, float4* xy_depth,
                                float4* conic_opa, float4* rgb, uint2* box, uint4* rows,
                                uint32_t* tiles) {
  ProjectArgs a;
  a.num_views = num_views - v0 < MAXV ? num_views - v0 : MAXV;
  for (int v = 0; v < a.num_views; ++v) a.cam[v] = cams[v0 + v];
  a.n = n; a.view_offset = v0;
  a.pos_opa = pos_opa; a.scale = scale; a.rot = rot; a.sh = sh; a.keep = keep;
  a.xy_depth = xy_depth; a.conic_opa = conic_opa; a.rgb = rgb; a.box = box; a.rows = rows;
  a.tiles = tiles;
  a.vpt = MAXV;   // every view of the launch per thread (measured fastest)
  return a;
}

cudaError_t launch_project_part(int part, const CamParams* cams, int num_views, int n,
                                int sh_degree, const float4* pos_opa, const float4* scale,
                                const float4* rot, const float4* sh, const uint8_t* keep,
                                float4* xy_depth, float4* conic_opa, float4* rgb, uint2* box,
                                uint4* rows, uint32_t* tiles, cudaStream_t s) {
  for (int v0 = 0; v0 < num_views; v0 += MAXV) {
    const ProjectArgs a = project_args(cams, v0, num_views, n, pos_opa, scale, rot, sh, keep,
                                       xy_depth, conic_opa, rgb, box, rows, tiles);
    const dim3 grid(div_up(n, 256), div_up(a.num_views, a.vpt));
    if (part & PROJECT_KEYS) {
      project_keys_kernel<<<grid, 256, 0, s>>>(a);
      launch_counted();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    if (part & PROJECT_RECORDS) {
      switch (sh_degree) {
        case 0: project_records_kernel<0><<<grid, 256, 0, s>>>(a); break;
        case 1: project_records_kernel<1><<<grid, 256, 0, s>>>(a); break;
        case 2: project_records_kernel<2><<<grid, 256, 0, s>>>(a); break;
        default: project_records_kernel<3><<<grid, 256, 0, s>>>(a); break;
      }
      launch_counted();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace dass
