// render.cu — dass_render_fwd / dass_render_bwd (Eq. 8 P:349-351 and its
// reverse-mode derivative).
//
// Tile kernels: one CTA per 16×16 tile, NT = 256/PPT threads, each thread
// owning PPT pixels of one column.  The tile's sorted list is streamed in
// batches of NT entries staged into shared memory (gathered by sorted id), in
// a tile-local frame: u_rel = (u_hi − tileX0) + u_lo keeps the mean offset
// accurate to ~1e-7 px, and the integer pixel box becomes a 16+16-bit
// column/row mask so the per-pixel box test (A05) is one LOP3 + compare.
//
// Backward reduction (hard part 2): per (warp, entry) the 9 per-pixel
// gradient terms are summed with a reduce-scatter butterfly (12 SHFL for 9
// values instead of 45), skipped when no lane of the warp contributes; the
// warp result is added into a shared-memory accumulator of the batch entry,
// and the batch is flushed with two 128-bit vector reductions
// (red.global.add.v4.f32) + one scalar per Gaussian and tile.
//
// The per-pixel terms are accumulated in a "moment" form that folds the
// per-Gaussian constants out of the pixel loop: with e = G·∂L/∂α (0 when α is
// clamped), the pixel contributes (e·dx, e·dy, e·dx², e·dx·dy, e·dy², e,
// αT·g_r, αT·g_g, αT·g_b), and the preprocess kernel forms
// ∂L/∂u = −o(A Σe·dx + B Σe·dy), ∂L/∂A = −½ o Σe·dx², … (exact algebra).
#include <cstdlib>

#include "common.cuh"
#include "sh.cuh"

namespace dass {
namespace {

// Staged entry (48 B in three 16-B shared arrays so a warp can test the
// box mask with one LDS.128 before touching the rest):
//   s_a  = (u_rel, v_rel, p_thr, box mask bits)   p_thr: conservative power
//          threshold ln(α_min/o) − 1e-3 below which α < 1/255 for sure, so the
//          exp is skipped without changing any decision
//   s_co = (A, B, C, o)    s_c = (r, g, b, −)
// Tile-local row/column mask of the pixels an entry can possibly be accepted
// at: the integer pixel box (A05) intersected with the bounding box of the
// α ≥ 1/255 support ellipse {½ dᵀK d ≤ −p_thr}, whose half-extents are
// √(2(−p_thr)·Σ'_xx) and √(2(−p_thr)·Σ'_yy) with Σ' = K⁻¹.  Conservative
// (p_thr carries a 1e-3 margin and the extents a relative + absolute pad), so
// every pixel it excludes would have been rejected by the exact per-pixel test:
// decisions, and hence results, are unchanged (A05's box stays the rule).
// Minimum over the rectangle [a0,a1]×[b0,b1] (offsets from the mean) of the
// convex quadratic q(d) = A dx² + 2B dx dy + C dy²: 0 if the mean is inside,
// else the minimum over the four edges (1-D minimisation, clamped).
__device__ __forceinline__ float rect_qmin(float A, float B, float C, float a0, float a1, float b0,
                                           float b1) {
  if (a0 <= 0.f && a1 >= 0.f && b0 <= 0.f && b1 >= 0.f) return 0.f;
  const float iA = 1.f / A, iC = 1.f / C;
  float best = INFINITY;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float dx = e ? a1 : a0;
    const float dy = fminf(fmaxf(-B * dx * iC, b0), b1);
    best = fminf(best, A * dx * dx + 2.f * B * dx * dy + C * dy * dy);
    const float ey = e ? b1 : b0;
    const float ex = fminf(fmaxf(-B * ey * iA, a0), a1);
    best = fminf(best, A * ex * ex + 2.f * B * ex * ey + C * ey * ey);
  }
  return best;
}

// Tile-local row/column mask of the pixels an entry can possibly be accepted
// at: the integer pixel box (A05) intersected with the bounding box of the
// α ≥ 1/255 support ellipse {dᵀK d ≤ R² = −2·p_thr}, whose half-extents are
// √(R²·Σ'_xx) and √(R²·Σ'_yy) with Σ' = K⁻¹; then, for every warp region of
// RPW rows, the region's row bits are cleared when the ellipse misses the
// region entirely (exact ellipse-rectangle test, A36).  Conservative (p_thr
// carries a 1e-3 margin, the extents and the ellipse test carry relative and
// absolute pads), so every pixel it excludes would have been rejected by the
// exact per-pixel test: decisions, and hence results, are unchanged.
template <int RPW>
__device__ __forceinline__ uint32_t support_mask(uint2 b, int tx0, int ty0, float ux, float uy,
                                                 float4 co, float pthr) {
  int x0 = max((int)(b.x & 0xFFFFu) - tx0, 0), x1 = min((int)(b.x >> 16) - tx0, TILE - 1);
  int y0 = max((int)(b.y & 0xFFFFu) - ty0, 0), y1 = min((int)(b.y >> 16) - ty0, TILE - 1);
  const float det = co.x * co.z - co.y * co.y;
  const float r2 = -2.f * pthr;
  bool tight = false;
  if (det > 0.f && r2 > 0.f) {
    const float hx = sqrtf(r2 * co.z / det) * 1.0001f + 1e-3f;
    const float hy = sqrtf(r2 * co.x / det) * 1.0001f + 1e-3f;
    if (isfinite(hx) && isfinite(hy)) {
      tight = true;
      x0 = max(x0, (int)ceilf(fmaxf(ux - hx, -1.f)));
      x1 = min(x1, (int)floorf(fminf(ux + hx, 16.f)));
      y0 = max(y0, (int)ceilf(fmaxf(uy - hy, -1.f)));
      y1 = min(y1, (int)floorf(fminf(uy + hy, 16.f)));
    }
  }
  if (x0 > x1 || y0 > y1) return 0u;
  const uint32_t mx = ((2u << x1) - 1u) & ~((1u << x0) - 1u);
  uint32_t my = ((2u << y1) - 1u) & ~((1u << y0) - 1u);
  if (tight && RPW < 16) {
    const float lim = r2 * 1.0001f + 1e-3f;
#pragma unroll
    for (int w = 0; w < 16 / RPW; ++w) {
      const int ry0 = max(y0, w * RPW), ry1 = min(y1, w * RPW + RPW - 1);
      if (ry0 > ry1) continue;
      const float q = rect_qmin(co.x, co.y, co.z, (float)x0 - ux, (float)x1 - ux, (float)ry0 - uy,
                                (float)ry1 - uy);
      if (q > lim) my &= ~(((1u << RPW) - 1u) << (w * RPW));
    }
  }
  return my ? (mx | (my << 16)) : 0u;
}

struct Staged {  // one entry: three 16-B fields at fixed offsets from one base address
  float4 a, co, c;
};

template <int RPW>
__device__ __forceinline__ void stage(uint32_t id, const float4* __restrict__ xy_depth,
                                      const float4* __restrict__ conic_opa,
                                      const float4* __restrict__ rgb, const uint2* __restrict__ box,
                                      int tx0, int ty0, float4& a, float4& co, float4& c) {
  const float4 xy = xy_depth[id];
  const uint32_t lo_bits = __float_as_uint(xy.w);
  const __half2 lo = *reinterpret_cast<const __half2*>(&lo_bits);
  co = conic_opa[id];
  const float4 cc = rgb[id];
  a.x = __fadd_rn(xy.x - (float)tx0, __low2float(lo));
  a.y = __fadd_rn(xy.y - (float)ty0, __high2float(lo));
  a.z = __logf(ALPHA_MIN / co.w) - 1e-3f;
  a.w = __uint_as_float(support_mask<RPW>(box[id], tx0, ty0, a.x, a.y, co, a.z));
  c = make_float4(cc.x, cc.y, cc.z, 0.f);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Warp-row mask: warp w owns thread rows 2w, 2w+1 → pixel rows [2w·PPT, 2w·PPT + 2·PPT).
template <int PPT>
__device__ __forceinline__ uint32_t warp_row_mask(int warp) {
  return (((1u << (2 * PPT)) - 1u) << (16 + warp * 2 * PPT));
}

// ------------------------------------------------------------- forward ----
template <int PPT>
__global__ void __launch_bounds__(256 / PPT, 768 / (256 / PPT)) render_fwd_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const float4* __restrict__ rgb,
    const uint2* __restrict__ box, float3 bg, float* __restrict__ out_img,
    float* __restrict__ out_T, uint32_t* __restrict__ out_last) {
  constexpr int NT = 256 / PPT;
  constexpr int BATCH = 2 * NT;
  __shared__ Staged s_st[BATCH];
  const int tile = blockIdx.x;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const int t = threadIdx.x;
  const int lx = t & 15, ly0 = (t >> 4) * PPT;
  const int X = tx0 + lx;
  const uint32_t wmask = warp_row_mask<PPT>(t >> 5);
  const uint32_t colbit = 1u << lx;
  const uint2 range = ranges[tile];
  float T[PPT], C[PPT][3];
  uint32_t last[PPT];
  bool done[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int Y = ty0 + ly0 + p;
    T[p] = 1.f; C[p][0] = C[p][1] = C[p][2] = 0.f;
    last[p] = range.x;
    done[p] = !(X < cam.W && Y < cam.H);
  }
  const float fx = (float)lx;
  float fy[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) fy[p] = (float)(ly0 + p);
  for (uint32_t b0 = range.x; b0 < range.y; b0 += BATCH) {
    bool alive = false;
#pragma unroll
    for (int p = 0; p < PPT; ++p) alive |= !done[p];
    if (__syncthreads_count(alive) == 0) break;
    for (int k = t; k < BATCH; k += NT)
      if (b0 + k < range.y) stage<16>(ids[b0 + k], xy_depth, conic_opa, rgb, box, tx0, ty0, s_st[k].a, s_st[k].co, s_st[k].c);
    __syncthreads();
    const int cnt = __any_sync(0xffffffffu, alive) ? (int)min((uint32_t)BATCH, range.y - b0) : 0;
    for (int j = 0; j < cnt; ++j) {
      const Staged& st = s_st[j];
      const float4 a = st.a;
      const uint32_t m = __float_as_uint(a.w);
      if ((m & wmask) == 0u) continue;   // warp-uniform: box misses this warp's rows
      if ((m & colbit) == 0u) continue;
      const float4 co = st.co;
      const ColTerms ct = col_terms(co.x, co.y, co.z, a.x - fx);
      const uint32_t mr = m >> (16 + ly0);   // this thread's PPT row bits
      float pw[PPT];
      bool ok[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) {   // independent per pixel: no branches, full ILP
        pw[p] = splat_power(ct, a.y - fy[p]);
        ok[p] = !done[p] && ((mr >> p) & 1u) && !(pw[p] > 0.f) && !(pw[p] < a.z);
      }
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (!ok[p]) continue;
        const float alpha = splat_alpha(co.w, splat_exp(pw[p]));
        if (alpha < ALPHA_MIN) continue;
        const float tn = __fmul_rn(T[p], __fsub_rn(1.f, alpha));
        if (tn < T_MIN) { done[p] = true; continue; }
        const float4 c = st.c;
        const float w = alpha * T[p];
        C[p][0] += c.x * w; C[p][1] += c.y * w; C[p][2] += c.z * w;
        T[p] = tn;
        last[p] = b0 + j + 1;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int Y = ty0 + ly0 + p;
    if (X < cam.W && Y < cam.H) {
      const size_t pix = (size_t)Y * cam.W + X, np = (size_t)cam.W * cam.H;
      out_img[pix] = C[p][0] + T[p] * bg.x;
      out_img[np + pix] = C[p][1] + T[p] * bg.y;
      out_img[2 * np + pix] = C[p][2] + T[p] * bg.z;
      out_T[pix] = T[p];
      out_last[pix] = last[p];
    }
  }
}

// ------------------------------------------------ backward: raster part ----
// Reduce-scatter butterfly for 9 values (pad 10): after 5 rounds (12 SHFL)
// every even lane holds the warp sum of one value index.  Lane predicates
// and the owned index are loop-invariant and computed once per thread.
struct LaneRS {
  bool b16, b8, b4, b2;
  int slot;  // value index this lane owns after the butterfly, −1 if none
  __device__ __forceinline__ void init() {
    const uint32_t lane = threadIdx.x & 31u;
    b16 = lane & 16; b8 = lane & 8; b4 = lane & 4; b2 = lane & 2;
    const int pos = (b8 ? 3 : 0) + (b4 ? 2 : 0) + (b2 ? 1 : 0);
    const bool valid = (lane & 1) == 0 && (b8 ? pos <= 4 : pos <= 2);
    const int idx = (b16 ? 5 : 0) + pos;
    slot = (valid && idx < 9) ? idx : -1;
  }
  __device__ __forceinline__ float reduce(const float (&v)[9]) const {
    float r[6];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const float lo_v = v[i];
      const float hi_v = i + 5 < 9 ? v[i + 5] : 0.f;
      r[i] = (b16 ? hi_v : lo_v) + __shfl_xor_sync(0xffffffffu, b16 ? lo_v : hi_v, 16);
    }
    r[5] = 0.f;
    float s[4];
#pragma unroll
    for (int i = 0; i < 3; ++i)
      s[i] = (b8 ? r[i + 3] : r[i]) + __shfl_xor_sync(0xffffffffu, b8 ? r[i] : r[i + 3], 8);
    s[3] = 0.f;
    float q[2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
      q[i] = (b4 ? s[i + 2] : s[i]) + __shfl_xor_sync(0xffffffffu, b4 ? s[i] : s[i + 2], 4);
    float out = (b2 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, b2 ? q[0] : q[1], 2);
    out += __shfl_xor_sync(0xffffffffu, out, 1);
    return out;
  }
};

template <int PPT, int MINB>
__global__ void __launch_bounds__(256 / PPT, MINB) render_bwd_raster_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const float4* __restrict__ rgb,
    const uint2* __restrict__ box, float3 bg, const float* __restrict__ out_T,
    const uint32_t* __restrict__ out_last, const float* __restrict__ dL_dimg,
    float4* __restrict__ g2d) {
  constexpr int NT = 256 / PPT;
  constexpr int NW = NT / 32;
  constexpr int BATCH = 64;  // s_acc = NW·BATCH·36 B; small enough not to limit occupancy
  __shared__ Staged s_st[BATCH];
  __shared__ uint32_t s_id[BATCH];
  __shared__ float s_acc[NW][BATCH][9];
  __shared__ uint32_t s_wlast[NW];
  const int tile = blockIdx.x;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const int t = threadIdx.x;
  const int warp = t >> 5;
  const int lx = t & 15, ly0 = (t >> 4) * PPT;
  const int X = tx0 + lx;
  const uint32_t wmask = warp_row_mask<PPT>(warp);
  const uint32_t colbit = 1u << lx;
  const uint2 range = ranges[tile];
  LaneRS rs;
  rs.init();
  float T[PPT], gR[PPT], g[PPT][3];
  uint32_t last[PPT];
  uint32_t mylast = range.x;
  const size_t np = (size_t)cam.W * cam.H;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int Y = ty0 + ly0 + p;
    if (X < cam.W && Y < cam.H) {
      const size_t pix = (size_t)Y * cam.W + X;
      T[p] = out_T[pix];
      last[p] = out_last[pix];
      g[p][0] = dL_dimg[pix]; g[p][1] = dL_dimg[np + pix]; g[p][2] = dL_dimg[2 * np + pix];
    } else {
      T[p] = 1.f; last[p] = range.x;
      g[p][0] = g[p][1] = g[p][2] = 0.f;
    }
    gR[p] = T[p] * (g[p][0] * bg.x + g[p][1] * bg.y + g[p][2] * bg.z);
    mylast = max(mylast, last[p]);
  }
  const uint32_t wlast = __reduce_max_sync(0xffffffffu, mylast);
  if ((t & 31) == 0) s_wlast[warp] = wlast;
  __syncthreads();
  uint32_t end = range.x;
#pragma unroll
  for (int w = 0; w < NW; ++w) end = max(end, s_wlast[w]);
  const float fx = (float)lx;
  float fy[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) fy[p] = (float)(ly0 + p);
  for (uint32_t b1 = end; b1 > range.x;) {
    const uint32_t b0 = b1 - range.x > (uint32_t)BATCH ? b1 - BATCH : range.x;
    const int cnt = (int)(b1 - b0);
    __syncthreads();  // previous batch flushed
    for (int k = t; k < cnt; k += NT) {
      const uint32_t id = ids[b0 + k];
      s_id[k] = id;
      stage<2 * PPT>(id, xy_depth, conic_opa, rgb, box, tx0, ty0, s_st[k].a, s_st[k].co, s_st[k].c);
#pragma unroll
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int q = 0; q < 9; ++q) s_acc[w][k][q] = 0.f;
    }
    __syncthreads();
    for (int j = cnt - 1; j >= 0; --j) {
      const uint32_t gidx = b0 + j;
      if (gidx >= wlast) continue;          // warp-uniform: past every pixel's last
      const Staged& st = s_st[j];
      const float4 a = st.a;
      const uint32_t m = __float_as_uint(a.w);
      if ((m & wmask) == 0u) continue;      // warp-uniform: box misses this warp's rows
      float v[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) v[q] = 0.f;
      bool any = false;
      if (m & colbit) {
        const float4 co = st.co;
        const float dx = a.x - fx;
        const ColTerms ct = col_terms(co.x, co.y, co.z, dx);
        const uint32_t mr = m >> (16 + ly0);   // this thread's PPT row bits
        float pw[PPT];
        bool ok[PPT];
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          pw[p] = splat_power(ct, a.y - fy[p]);
          ok[p] = gidx < last[p] && ((mr >> p) & 1u) && !(pw[p] > 0.f) && !(pw[p] < a.z);
        }
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          if (!ok[p]) continue;
          const float G = splat_exp(pw[p]);
          const float oG = __fmul_rn(co.w, G);
          const float alpha = fminf(ALPHA_MAX, oG);
          if (alpha < ALPHA_MIN) continue;
          any = true;
          const float dy = a.y - fy[p];
          const float4 c = st.c;
          const float inv = rcp_approx(1.f - alpha);
          T[p] *= inv;                        // transmittance before this entry
          const float w = alpha * T[p];
          const float gc = g[p][0] * c.x + g[p][1] * c.y + g[p][2] * c.z;
          const float dLda = T[p] * gc - inv * gR[p];
          gR[p] += gc * w;                    // g·(S + T_final·bg), S = suffix colour
          v[6] += w * g[p][0]; v[7] += w * g[p][1]; v[8] += w * g[p][2];
          const float e = oG < ALPHA_MAX ? G * dLda : 0.f;
          const float ex = e * dx, ey = e * dy;
          v[0] += ex; v[1] += ey; v[2] += ex * dx; v[3] += ex * dy; v[4] += ey * dy; v[5] += e;
        }
      }
      if (__any_sync(0xffffffffu, any)) {
        const float sum = rs.reduce(v);
        if (rs.slot >= 0) s_acc[warp][j][rs.slot] = sum;
      }
    }
    __syncthreads();
    for (int k = t; k < cnt; k += NT) {
      float a9[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) s += s_acc[w][k][q];
        a9[q] = s;
      }
      bool nz = false;
#pragma unroll
      for (int q = 0; q < 9; ++q) nz |= a9[q] != 0.f;
      if (nz) {
        float4* dst = g2d + 3 * (size_t)s_id[k];
        red_add_v4(dst, make_float4(a9[0], a9[1], a9[2], a9[3]));
        red_add_v4(dst + 1, make_float4(a9[4], a9[5], a9[6], a9[7]));
        atomicAdd(&dst[2].x, a9[8]);
      }
    }
    b1 = b0;
  }
}

// --------------------------------------------- backward: preprocess part ----
// Per Gaussian, over V views: each view's 2D moments → ∂L/∂(u, v, A, B, C, o,
// rgb) → chained through Eqs. 5-7 and the SH colour.  The parameters are read
// once, R and Σ are built once, and the view-independent ∂L/∂Σ is summed over
// the views before the scale/rotation chain, so every output is updated once
// (+=) per launch (multi-view batching).
constexpr int PRE_MAXV = 32;  // views per launch (kernel-parameter budget)

struct PreArgs {
  CamParams cam[PRE_MAXV];
  int num_views, n;
  const float4* pos_opa;
  const float4* scale;
  const float4* rot;
  const float4* sh;
  const uint8_t* keep;
  const float4* conic_opa;  // [V][N]
  const float4* rgb;        // [V][N]
  const uint2* box;         // [V][N]
  const float4* g2d;        // [V][N][3]
  float4* g_pos_opa;
  float4* g_scale;
  float4* g_rot;
  float4* g_sh;
  float* gradstat_sum;
  uint32_t* gradstat_cnt;
};

template <int DEG>
__global__ void __launch_bounds__(256, 2) preprocess_views_kernel(const __grid_constant__ PreArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int n = a.n;
  using L = SHLayout<DEG>;
  const bool kp = a.keep == nullptr || a.keep[i] != 0;
  const float4 po = a.pos_opa[i];
  const float4 q = a.rot[i];
  const float4 sc = a.scale[i];
  // view-independent geometry: q̂, R, s, Σ
  const float qn = sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
  const float qi = 1.f / qn;
  const float w = q.x * qi, x = q.y * qi, y = q.z * qi, z = q.w * qi;
  float R[3][3];
  R[0][0] = 1.f - 2.f * (y * y + z * z); R[0][1] = 2.f * (x * y - w * z); R[0][2] = 2.f * (x * z + w * y);
  R[1][0] = 2.f * (x * y + w * z); R[1][1] = 1.f - 2.f * (x * x + z * z); R[1][2] = 2.f * (y * z - w * x);
  R[2][0] = 2.f * (x * z - w * y); R[2][1] = 2.f * (y * z + w * x); R[2][2] = 1.f - 2.f * (x * x + y * y);
  const float s[3] = {kp ? sc.x : 0.f, kp ? sc.y : 0.f, kp ? sc.z : 0.f};
  float Sig[3][3];
#pragma unroll
  for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
    for (int c0 = 0; c0 < 3; ++c0)
      Sig[r0][c0] = R[r0][0] * s[0] * s[0] * R[c0][0] + R[r0][1] * s[1] * s[1] * R[c0][1] +
                    R[r0][2] * s[2] * s[2] * R[c0][2];
  // accumulators over views
  float gp[3] = {0.f, 0.f, 0.f};
  float go = 0.f;
  float GS[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
  float gsh[4 * L::K4];
#pragma unroll
  for (int f = 0; f < 4 * L::K4; ++f) gsh[f] = 0.f;
  float gstat = 0.f;
  uint32_t nvis = 0;
  for (int v = 0; v < a.num_views; ++v) {
    const size_t o = (size_t)v * n + i;
    const uint2 bx = a.box[o];
    if ((bx.x & 0xFFFFu) > (bx.x >> 16)) continue;  // culled in this view
    const CamParams& cam = a.cam[v];
    ++nvis;
    const float4 m0 = a.g2d[3 * o], m1 = a.g2d[3 * o + 1], m2 = a.g2d[3 * o + 2];
    const float4 co = a.conic_opa[o];
    const float A = co.x, B = co.y, Cc = co.z, op = co.w;
    // 2D gradients from the moments
    const float gu = -op * (A * m0.x + B * m0.y);
    const float gv = -op * (B * m0.x + Cc * m0.y);
    const float gA = -0.5f * op * m0.z;
    const float gB = -op * m0.w;
    const float gC = -0.5f * op * m1.x;
    go += m1.y;
    const int bits = (int)a.rgb[o].w;
    const float gcol[3] = {(bits & 1) ? 0.f : m1.z, (bits & 2) ? 0.f : m1.w, (bits & 4) ? 0.f : m2.x};
    {
      const float ga = gu * 0.5f * cam.W, gb = gv * 0.5f * cam.H;
      gstat += sqrtf(ga * ga + gb * gb);
    }
    // ---- colour / SH (direction from this view's camera centre)
    {
      float dx = po.x - cam.campos[0], dy = po.y - cam.campos[1], dz = po.z - cam.campos[2];
      const float dist = sqrtf(dx * dx + dy * dy + dz * dz);
      const float inv = 1.f / dist;
      dx *= inv; dy *= inv; dz *= inv;
      float Y[L::NC];
      sh_eval<DEG>(dx, dy, dz, Y);
      float wk[L::NC];
#pragma unroll
      for (int k = 0; k < L::NC; ++k) wk[k] = 0.f;
#pragma unroll
      for (int j = 0; j < L::K4; ++j) {
        // re-read per view (L1-resident) instead of pinning 48 registers
        const float4 c4 = a.sh[(size_t)j * n + i];
        const float cf[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int f = 4 * j + e;
          if (f < L::NF) {
            const int k = f / 3, ch = f % 3;
            wk[k] += gcol[ch] * cf[e];
            gsh[f] += Y[k] * gcol[ch];
          }
        }
      }
      if (DEG > 0) {
        const float3 gd = sh_dir_grad<DEG>(dx, dy, dz, wk);
        const float dd = dx * gd.x + dy * gd.y + dz * gd.z;
        gp[0] += (gd.x - dx * dd) * inv;
        gp[1] += (gd.y - dy * dd) * inv;
        gp[2] += (gd.z - dz * dd) * inv;
      }
    }
    // ---- projection chain for this view
    const float* V = cam.V;
    float t[3];
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0)
      t[r0] = V[4 * r0] * po.x + V[4 * r0 + 1] * po.y + V[4 * r0 + 2] * po.z + V[4 * r0 + 3];
    const float lx = 1.3f * cam.W / (2.f * cam.fx), ly = 1.3f * cam.H / (2.f * cam.fy);
    const float txtz = t[0] / t[2], tytz = t[1] / t[2];
    const bool clx = txtz < -lx || txtz > lx, cly = tytz < -ly || tytz > ly;
    const float xt = t[2] * fminf(lx, fmaxf(-lx, txtz));
    const float yt = t[2] * fminf(ly, fmaxf(-ly, tytz));
    const float tz = t[2], tz2 = tz * tz, tz3 = tz2 * tz;
    const float J00 = cam.fx / tz, J02 = -cam.fx * xt / tz2;
    const float J11 = cam.fy / tz, J12 = -cam.fy * yt / tz2;
    float M[2][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      M[0][b] = J00 * V[b] + J02 * V[8 + b];
      M[1][b] = J11 * V[4 + b] + J12 * V[8 + b];
    }
    // conic → Σ': Gs = −K Ĝ K, Ĝ = [[gA, gB/2],[gB/2, gC]]
    const float G01h = 0.5f * gB;
    const float KG00 = A * gA + B * G01h, KG01 = A * G01h + B * gC;
    const float KG10 = B * gA + Cc * G01h, KG11 = B * G01h + Cc * gC;
    const float Gs00 = -(KG00 * A + KG01 * B);
    const float Gs01 = -(KG00 * B + KG01 * Cc);
    const float Gs11 = -(KG10 * B + KG11 * Cc);
    float GM1[2][3];  // Gs M
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      GM1[0][b] = Gs00 * M[0][b] + Gs01 * M[1][b];
      GM1[1][b] = Gs01 * M[0][b] + Gs11 * M[1][b];
    }
    // ∂L/∂Σ += Mᵀ Gs M  (summed over views, chained once below)
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
      for (int c0 = 0; c0 < 3; ++c0) GS[r0][c0] += M[0][r0] * GM1[0][c0] + M[1][r0] * GM1[1][c0];
    // ∂L/∂M = 2 Gs M Σ → ∂L/∂J = ∂L/∂M Wᵀ
    float GM[2][3];
#pragma unroll
    for (int r0 = 0; r0 < 2; ++r0)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        GM[r0][b] = 2.f * (GM1[r0][0] * Sig[0][b] + GM1[r0][1] * Sig[1][b] + GM1[r0][2] * Sig[2][b]);
    const float GJ00 = GM[0][0] * V[0] + GM[0][1] * V[1] + GM[0][2] * V[2];
    const float GJ02 = GM[0][0] * V[8] + GM[0][1] * V[9] + GM[0][2] * V[10];
    const float GJ11 = GM[1][0] * V[4] + GM[1][1] * V[5] + GM[1][2] * V[6];
    const float GJ12 = GM[1][0] * V[8] + GM[1][1] * V[9] + GM[1][2] * V[10];
    float gt[3] = {0.f, 0.f, 0.f};
    gt[2] += GJ00 * (-cam.fx / tz2) + GJ11 * (-cam.fy / tz2);
    if (!clx) {
      gt[0] += GJ02 * (-cam.fx / tz2);
      gt[2] += GJ02 * (2.f * cam.fx * t[0] / tz3);
    } else {
      gt[2] += GJ02 * (cam.fx * xt / tz3);
    }
    if (!cly) {
      gt[1] += GJ12 * (-cam.fy / tz2);
      gt[2] += GJ12 * (2.f * cam.fy * t[1] / tz3);
    } else {
      gt[2] += GJ12 * (cam.fy * yt / tz3);
    }
    gt[0] += gu * cam.fx / tz;
    gt[2] += gu * (-cam.fx * t[0] / tz2);
    gt[1] += gv * cam.fy / tz;
    gt[2] += gv * (-cam.fy * t[1] / tz2);
#pragma unroll
    for (int c0 = 0; c0 < 3; ++c0) gp[c0] += V[c0] * gt[0] + V[4 + c0] * gt[1] + V[8 + c0] * gt[2];
  }
  if (nvis == 0) return;
  if (a.gradstat_sum) a.gradstat_sum[i] += gstat;
  if (a.gradstat_cnt) a.gradstat_cnt[i] += nvis;
  if (a.g_sh) {
#pragma unroll
    for (int j = 0; j < L::K4; ++j) {
      const size_t off = (size_t)j * n + i;
      float4 gg = a.g_sh[off];
      gg.x += gsh[4 * j]; gg.y += gsh[4 * j + 1];
      if (4 * j + 2 < L::NF) gg.z += gsh[4 * j + 2];
      if (4 * j + 3 < L::NF) gg.w += gsh[4 * j + 3];
      a.g_sh[off] = gg;
    }
  }
  if (a.g_pos_opa) {
    float4 gpo = a.g_pos_opa[i];
    gpo.x += gp[0]; gpo.y += gp[1]; gpo.z += gp[2];
    gpo.w += kp ? go : 0.f;
    a.g_pos_opa[i] = gpo;
  }
  if (!a.g_scale && !a.g_rot) return;
  // Σ = R diag(s²) Rᵀ : dL/ds_k = 2 s_k (Rᵀ GΣ R)_kk ; dL/dR = 2 GΣ R diag(s²)
  float GR[3][3];
  float gs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float GSr[3];
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0) GSr[r0] = GS[r0][0] * R[0][k] + GS[r0][1] * R[1][k] + GS[r0][2] * R[2][k];
    gs[k] = 2.f * s[k] * (R[0][k] * GSr[0] + R[1][k] * GSr[1] + R[2][k] * GSr[2]);
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0) GR[r0][k] = 2.f * GSr[r0] * s[k] * s[k];
  }
  if (a.g_scale) {
    float4 g4 = a.g_scale[i];
    if (kp) { g4.x += gs[0]; g4.y += gs[1]; g4.z += gs[2]; }
    a.g_scale[i] = g4;
  }
  if (a.g_rot) {
    float gq[4];
    gq[0] = GR[0][1] * (-2.f * z) + GR[0][2] * (2.f * y) + GR[1][0] * (2.f * z) + GR[1][2] * (-2.f * x) +
            GR[2][0] * (-2.f * y) + GR[2][1] * (2.f * x);
    gq[1] = GR[0][1] * (2.f * y) + GR[0][2] * (2.f * z) + GR[1][0] * (2.f * y) + GR[1][1] * (-4.f * x) +
            GR[1][2] * (-2.f * w) + GR[2][0] * (2.f * z) + GR[2][1] * (2.f * w) + GR[2][2] * (-4.f * x);
    gq[2] = GR[0][0] * (-4.f * y) + GR[0][1] * (2.f * x) + GR[0][2] * (2.f * w) + GR[1][0] * (2.f * x) +
            GR[1][2] * (2.f * z) + GR[2][0] * (-2.f * w) + GR[2][1] * (2.f * z) + GR[2][2] * (-4.f * y);
    gq[3] = GR[0][0] * (-4.f * z) + GR[0][1] * (-2.f * w) + GR[0][2] * (2.f * x) + GR[1][0] * (2.f * w) +
            GR[1][1] * (-4.f * z) + GR[1][2] * (2.f * y) + GR[2][0] * (2.f * x) + GR[2][1] * (2.f * y);
    const float dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
    float4 g4 = a.g_rot[i];
    g4.x += (gq[0] - w * dot) * qi;
    g4.y += (gq[1] - x * dot) * qi;
    g4.z += (gq[2] - y * dot) * qi;
    g4.w += (gq[3] - z * dot) * qi;
    a.g_rot[i] = g4;
  }
}

// Pixels per thread of the raster kernels (tuning knob; DASS_FWD_PPT /
// DASS_BWD_PPT override the default for experiments, read once per process).
static int ppt_from_env(const char* name, int dflt) {
  const char* v = getenv(name);
  if (!v) return dflt;
  const int p = atoi(v);
  return (p == 1 || p == 2 || p == 4 || p == 8) ? p : dflt;
}
static int fwd_ppt() { static const int p = ppt_from_env("DASS_FWD_PPT", 4); return p; }
static int bwd_ppt() { static const int p = ppt_from_env("DASS_BWD_PPT", 4); return p; }
static int bwd_minb() {
  static const int m = [] {
    const char* v = getenv("DASS_BWD_MINB");
    const int p = v ? atoi(v) : 16;
    return (p == 8 || p == 12 || p == 16) ? p : 16;
  }();
  return bwd_ppt() == 4 ? m : (bwd_ppt() == 1 ? 16 : (bwd_ppt() == 2 ? 8 : 16));
}

}  // namespace

cudaError_t launch_render_fwd(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, float* out_img, float* out_T,
                              uint32_t* out_last, cudaStream_t s) {
  const int ntiles = cam.tiles_x * cam.tiles_y;
#define FWD(P)                                                                                   \
  render_fwd_kernel<P><<<ntiles, 256 / P, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, rgb, box, \
                                                  bg, out_img, out_T, out_last)
  switch (fwd_ppt()) {
    case 1: FWD(1); break;
    case 2: FWD(2); break;
    case 8: FWD(8); break;
    default: FWD(4); break;
  }
#undef FWD
  launch_counted();
  return cudaGetLastError();
}

size_t render_bwd_workspace(int n) { return sizeof(float4) * 3 * (size_t)(n > 0 ? n : 1); }

cudaError_t launch_render_bwd_raster(const CamParams& cam, int n, const uint2* ranges,
                                     const uint32_t* ids, const float4* xy_depth,
                                     const float4* conic_opa, const float4* rgb, const uint2* box,
                                     float3 bg, const float* out_T, const uint32_t* out_last,
                                     const float* dL_dimg, float4* g2d, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(g2d, 0, render_bwd_workspace(n), s);
  if (e != cudaSuccess) return e;
  const int ntiles = cam.tiles_x * cam.tiles_y;
#define BWD(P, MB)                                                                          \
  render_bwd_raster_kernel<P, MB><<<ntiles, 256 / P, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, \
                                                             rgb, box, bg, out_T, out_last, dL_dimg, g2d)
  switch (bwd_ppt() * 100 + bwd_minb()) {
    case 116: BWD(1, 4); break;
    case 208: BWD(2, 8); break;
    case 816: BWD(8, 16); break;
    case 412: BWD(4, 12); break;
    case 408: BWD(4, 8); break;
    default: BWD(4, 16); break;
  }
#undef BWD
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_preprocess_views(const CamParams* cams, int num_views, int n, int sh_degree,
                                    const float4* pos_opa, const float4* scale, const float4* rot,
                                    const float4* sh, const uint8_t* keep,
                                    const float4* conic_opa, const float4* rgb, const uint2* box,
                                    const float4* g2d, float4* g_pos_opa, float4* g_scale,
                                    float4* g_rot, float4* g_sh, float* gradstat_sum,
                                    uint32_t* gradstat_cnt, cudaStream_t s) {
  for (int v0 = 0; v0 < num_views; v0 += PRE_MAXV) {
    PreArgs a;
    a.num_views = num_views - v0 < PRE_MAXV ? num_views - v0 : PRE_MAXV;
    for (int v = 0; v < a.num_views; ++v) a.cam[v] = cams[v0 + v];
    const size_t off = (size_t)v0 * n;
    a.n = n;
    a.pos_opa = pos_opa; a.scale = scale; a.rot = rot; a.sh = sh; a.keep = keep;
    a.conic_opa = conic_opa + off; a.rgb = rgb + off; a.box = box + off; a.g2d = g2d + 3 * off;
    a.g_pos_opa = g_pos_opa; a.g_scale = g_scale; a.g_rot = g_rot; a.g_sh = g_sh;
    a.gradstat_sum = gradstat_sum; a.gradstat_cnt = gradstat_cnt;
    const int grid = div_up(n, 256);
    switch (sh_degree) {
      case 0: preprocess_views_kernel<0><<<grid, 256, 0, s>>>(a); break;
      case 1: preprocess_views_kernel<1><<<grid, 256, 0, s>>>(a); break;
      case 2: preprocess_views_kernel<2><<<grid, 256, 0, s>>>(a); break;
      default: preprocess_views_kernel<3><<<grid, 256, 0, s>>>(a); break;
    }
    launch_counted();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_render_bwd(const CamParams& cam, int n, int sh_degree, const float4* pos_opa,
                              const float4* scale, const float4* rot, const float4* sh,
                              const uint8_t* keep, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, const float* out_T,
                              const uint32_t* out_last, const float* dL_dimg, void* ws,
                              float4* g_pos_opa, float4* g_scale, float4* g_rot, float4* g_sh,
                              float* gradstat_sum, uint32_t* gradstat_cnt, cudaStream_t s) {
  float4* g2d = (float4*)ws;
  cudaError_t e = launch_render_bwd_raster(cam, n, ranges, ids, xy_depth, conic_opa, rgb, box, bg,
                                           out_T, out_last, dL_dimg, g2d, s);
  if (e != cudaSuccess) return e;
  return launch_preprocess_views(&cam, 1, n, sh_degree, pos_opa, scale, rot, sh, keep, conic_opa,
                                 rgb, box, g2d, g_pos_opa, g_scale, g_rot, g_sh, gradstat_sum,
                                 gradstat_cnt, s);
}

}  // namespace dass
