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
#include "common.cuh"
#include "sh.cuh"

#ifndef PRE1_MINB
#define PRE1_MINB 3   // preprocess PART 1: 3 blocks/SM (166 registers, no spill) with the cp.async view pipeline: 0.352 ms per 20 views against 0.397 at 4 blocks (128 registers, spills)
#endif

namespace dass {
namespace {

// Staged entry (48 B in three 16-B shared arrays so a warp can test the
// box mask with one LDS.128 before touching the rest):
//   s_a  = (u_rel, v_rel, p_thr, box mask bits)   p_thr: conservative power
//          threshold ln(α_min/o) − 1e-3 below which α < 1/255 for sure, so the
//          exp is skipped without changing any decision
//   s_co = (s, sβ, g, o) (conic_staged)    s_c = (r, g, b, −)
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
  // co = (A, β, γ, o): K = [[A, Aβ], [Aβ, γ + Aβ²]], det K = Aγ, Σ' = K⁻¹ with
  // Σ'_xx = 1/A + β²/γ and Σ'_yy = 1/γ
  int x0 = max((int)(b.x & 0xFFFFu) - tx0, 0), x1 = min((int)(b.x >> 16) - tx0, TILE - 1);
  int y0 = max((int)(b.y & 0xFFFFu) - ty0, 0), y1 = min((int)(b.y >> 16) - ty0, TILE - 1);
  const float r2 = -2.f * pthr;
  bool tight = false;
  if (co.x > 0.f && co.z > 0.f && r2 > 0.f) {
    const float sxx = 1.f / co.x + co.y * co.y / co.z, syy = 1.f / co.z;
    const float hx = sqrtf(r2 * sxx) * 1.0001f + 1e-3f;
    const float hy = sqrtf(r2 * syy) * 1.0001f + 1e-3f;
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
    const float B = co.x * co.y, C = co.z + co.x * co.y * co.y;
#pragma unroll
    for (int w = 0; w < 16 / RPW; ++w) {
      const int ry0 = max(y0, w * RPW), ry1 = min(y1, w * RPW + RPW - 1);
      if (ry0 > ry1) continue;
      const float q = rect_qmin(co.x, B, C, (float)x0 - ux, (float)x1 - ux, (float)ry0 - uy,
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
  const float4 con = conic_opa[id];
  co = conic_staged(con);   // (s, sβ, g, o)
  const float4 cc = rgb[id];
  a.x = __fadd_rn(xy.x - (float)tx0, __low2float(lo));
  a.y = __fadd_rn(xy.y - (float)ty0, __high2float(lo));
  a.z = __logf(ALPHA_MIN / co.w) - 1e-3f;
  a.w = __uint_as_float(support_mask<RPW>(box[id], tx0, ty0, a.x, a.y, con, a.z));
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

// Per-tile acceptance lists written by the forward (A38; one warp per tile,
// TW pixel map): for every tile-list entry accepted by at least one pixel of
// the tile, its absolute list index idx[range.x + k] and 32 bytes
// bytes[(range.x + k)·32 + lane] — the 8-bit set of lane's pixels that
// accepted it; cnt[tile] = the number of such entries.  The backward walks
// exactly these (pixel, entry) pairs.
struct AcceptLists {
  uint32_t* cnt;
  uint32_t* idx;
  uint8_t* bytes;
  uint32_t* order;   // launch order of the tiles (longest list first)
  uint32_t cap;      // pair capacity the lists were sized for
};

// Pixel ownership of a tile CTA (NT = 256/PPT threads, 16×16 pixels).
//   PPT = 4 ("quadrant map", the list path): warp w owns the 16×8 half-tile of
//     rows [8w, 8w+8); lane l owns one pixel in each of its four 8×4
//     quadrants, (cx + 8·(p&1), cy + 4·(p>>1)) with cx = l&7, cy = 8w + (l>>3).
//     A compact footprint covers few quadrants, so the per-p pixel blocks a
//     warp executes for one entry (any lane with bit p) drop from 3.5 to 2.5
//     per accepted warp-entry on the C3 scene; two
//     columns and two rows per lane keep dx/dy at two values each.
//   other PPT ("row map"): thread t owns column t&15, rows (t>>4)·PPT + p.
template <int PPT>
struct PixMap {
  static constexpr bool QUAD = PPT == 4;
  int cx, cy;
  __device__ __forceinline__ explicit PixMap(int t) {
    if (QUAD) { cx = t & 7; cy = ((t >> 5) << 3) + ((t >> 3) & 3); }
    else { cx = t & 15; cy = (t >> 4) * PPT; }
  }
  __device__ __forceinline__ int x(int p) const { return QUAD ? cx + 8 * (p & 1) : cx; }
  __device__ __forceinline__ int y(int p) const { return QUAD ? cy + 4 * (p >> 1) : cy + p; }
  // bit p set iff pixel p's column and row bits are both set in the entry's
  // tile-local support mask m (columns in bits 0-15, rows in bits 16-31)
  __device__ __forceinline__ uint32_t cand(uint32_t m) const {
    if (QUAD) {
      const uint32_t c2 = ((m >> cx) & 1u) | ((m >> (cx + 7)) & 2u);
      const uint32_t r = m >> (16 + cy);
      return ((r & 1u) ? c2 : 0u) | ((r & 16u) ? (c2 << 2) : 0u);
    }
    return ((m >> cx) & 1u) ? ((m >> (16 + cy)) & ((1u << PPT) - 1u)) : 0u;
  }
};

// ------------------------------------------------------------- forward ----
// Without acceptance lists (dass_render_fwd with accept = nullptr): one CTA of
// 64 threads per tile, PPT = 4 quadrant map, batches of 128 staged entries.
template <int PPT, int MINB = 768 / (256 / PPT)>
__global__ void __launch_bounds__(256 / PPT, MINB) render_fwd_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const float4* __restrict__ rgb,
    const uint2* __restrict__ box, float3 bg, float* __restrict__ out_img,
    float* __restrict__ out_T, uint32_t* __restrict__ out_last) {
  static_assert(PPT == 4, "the quadrant map");
  constexpr int NT = 256 / PPT;
  constexpr int BATCH = 2 * NT;
  __shared__ Staged s_st[BATCH];
  const int tile = cam.tile0 + blockIdx.x * cam.tstride;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const int t = threadIdx.x;
  const PixMap<PPT> pm(t);
  const uint32_t wmask = warp_row_mask<PPT>(t >> 5);
  const uint2 range = ranges[tile];
  float T[PPT], C[PPT][3];
  uint32_t last[PPT];
  uint32_t live = 0;   // bit p: pixel p is inside the image and not terminated
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    T[p] = 1.f; C[p][0] = C[p][1] = C[p][2] = 0.f;
    last[p] = range.x;
    if (tx0 + pm.x(p) < cam.W && ty0 + pm.y(p) < cam.H) live |= 1u << p;
  }
  // tile-relative pixel coordinates: columns fxc[p & 1], rows fy[p]
  const float fxc[2] = {(float)pm.x(0), (float)pm.x(1)};
  const float fy0 = (float)pm.y(0), fy1 = (float)pm.y(2);
  for (uint32_t b0 = range.x; b0 < range.y; b0 += BATCH) {
    const bool alive = live != 0u;
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
      // candidate pixels: column and row in the support mask, still live
      const uint32_t cand = pm.cand(m) & live;
      if (!cand) continue;
      const float4 co = st.co;
      const float dx0 = a.x - fxc[0], dx1 = a.x - fxc[1];
      const float dy0 = a.y - fy0, dy1 = a.y - fy1;
      const float X0 = col_term(co, dx0), X1 = col_term(co, dx1);
      const RowTerms R0 = row_terms(co, dy0), R1 = row_terms(co, dy1);
      float pw[PPT];
      pw[0] = splat_power(X0, R0); pw[1] = splat_power(X1, R0);
      pw[2] = splat_power(X0, R1); pw[3] = splat_power(X1, R1);
      uint32_t ok = 0;
#pragma unroll
      for (int p = 0; p < PPT; ++p)   // independent per pixel: no branches, full ILP
        ok |= (!(pw[p] > 0.f) && !(pw[p] < a.z)) ? (1u << p) : 0u;
      ok &= cand;
      if (!ok) continue;
      const float4 c = st.c;
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (!((ok >> p) & 1u)) continue;
        const float alpha = splat_alpha(co.w, splat_exp(pw[p]));
        if (alpha < ALPHA_MIN) continue;
        const float tn = __fmul_rn(T[p], __fsub_rn(1.f, alpha));
        if (tn < T_MIN) { live &= ~(1u << p); continue; }
        const float w = alpha * T[p];
        C[p][0] += c.x * w; C[p][1] += c.y * w; C[p][2] += c.z * w;
        T[p] = tn;
        last[p] = b0 + j + 1;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int X = tx0 + pm.x(p), Y = ty0 + pm.y(p);
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

// ------------------------------------- identity-feature render (Eq. 9) ----
// M = Σ_i e_i α_i Π_{j<i}(1 − α_j) (f4, A47): the forward's tile walk,
// PPT = 4 mapping, support masks and canonical α decisions, with NV float4
// feature planes per entry in place of the colour and no background.
template <int NV>
__global__ void __launch_bounds__(64) render_features_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const uint2* __restrict__ box,
    const float4* __restrict__ feat, float* __restrict__ out) {
  constexpr int PPT = 4;
  constexpr int NT = 64;
  constexpr int BATCH = 2 * NT;
  __shared__ Staged s_st[BATCH];
  __shared__ float4 s_f[BATCH][NV];
  const int tile = cam.tile0 + blockIdx.x * cam.tstride;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const int t = threadIdx.x;
  const int lx = t & 15, ly0 = (t >> 4) * PPT;
  const int X = tx0 + lx;
  const uint32_t wmask = warp_row_mask<PPT>(t >> 5);
  const uint32_t colbit = 1u << lx;
  const uint2 range = ranges[tile];
  float T[PPT];
  float4 M[PPT][NV];
  bool done[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int Y = ty0 + ly0 + p;
    T[p] = 1.f;
#pragma unroll
    for (int v = 0; v < NV; ++v) M[p][v] = make_float4(0.f, 0.f, 0.f, 0.f);
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
    for (int k = t; k < BATCH; k += NT) {
      if (b0 + k < range.y) {
        const uint32_t id = ids[b0 + k];
        stage<16>(id, xy_depth, conic_opa, conic_opa, box, tx0, ty0, s_st[k].a, s_st[k].co, s_st[k].c);
#pragma unroll
        for (int v = 0; v < NV; ++v) s_f[k][v] = feat[(size_t)id * NV + v];
      }
    }
    __syncthreads();
    const int cnt = (int)min((uint32_t)BATCH, range.y - b0);
    for (int j = 0; j < cnt; ++j) {
      const float4 a = s_st[j].a;
      const uint32_t m = __float_as_uint(a.w);
      if ((m & wmask) == 0u || !(m & colbit)) continue;
      const float4 co = s_st[j].co;
      const float dx = a.x - fx;
      const uint32_t mr = m >> (16 + ly0);
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (done[p] || !((mr >> p) & 1u)) continue;
        const float dy = a.y - fy[p];
        const float pw = splat_power(co, dx, dy);
        if (pw > 0.f || pw < a.z) continue;
        const float alpha = splat_alpha(co.w, splat_exp(pw));
        if (alpha < ALPHA_MIN) continue;
        const float tn = __fmul_rn(T[p], __fsub_rn(1.f, alpha));
        if (tn < T_MIN) { done[p] = true; continue; }
        const float w = alpha * T[p];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const float4 e = s_f[j][v];
          M[p][v].x += e.x * w; M[p][v].y += e.y * w; M[p][v].z += e.z * w; M[p][v].w += e.w * w;
        }
        T[p] = tn;
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int Y = ty0 + ly0 + p;
    if (X < cam.W && Y < cam.H) {
      const size_t pix = (size_t)Y * cam.W + X, np = (size_t)cam.W * cam.H;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        out[(4 * v + 0) * np + pix] = M[p][v].x;
        out[(4 * v + 1) * np + pix] = M[p][v].y;
        out[(4 * v + 2) * np + pix] = M[p][v].z;
        out[(4 * v + 3) * np + pix] = M[p][v].w;
      }
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
  const int tile = cam.tile0 + blockIdx.x * cam.tstride;
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
        const uint32_t mr = m >> (16 + ly0);   // this thread's PPT row bits
        float pw[PPT];
        bool ok[PPT];
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          const float dyp = a.y - fy[p];
          pw[p] = splat_power(co, dx, dyp);
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
          const float ey = e * dy;
          v[1] += ey; v[4] += ey * dy; v[5] += e;
        }
        // the lane's PPT pixels share one column, so dx factors out of the
        // dx-moments: Σe·dx = dx·Σe, Σe·dx² = dx·(dx·Σe), Σe·dx·dy = dx·Σe·dy
        v[0] = v[5] * dx; v[2] = v[0] * dx; v[3] = v[1] * dx;
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

// ------------------------------------- tile-warp list path (TW, PPT = 8) ----
#ifndef TW_BWD_CHUNK
#define TW_BWD_CHUNK 16
#endif
#ifndef TW_FWD_BATCH
#define TW_FWD_BATCH 32
#endif
// One warp per 16×16 tile (32-thread CTAs).  Lane l owns the eight pixels
// (cx + 8·(p>>2), cy + 4·(p&3)), cx = l&7, cy = l>>3: one per 8×4 block of
// the tile, so a compact footprint covers few blocks p.  Against the two
// half-tile warps of the PPT = 4 path, an entry whose accepted pixels span
// both halves is walked, staged and reduced once instead of twice (a CPU
// replay of a C3 view: 0.67× the warp-entries, identical pixel blocks).  The
// list is one per tile: entry k of tile t at [range.x + k], byte `lane` = the
// lane's 8-bit accepted set, cnt[t].
struct TileMap {
  int cx, cy;
  __device__ __forceinline__ explicit TileMap(int lane) : cx(lane & 7), cy(lane >> 3) {}
  __device__ __forceinline__ int x(int p) const { return cx + 8 * (p >> 2); }
  __device__ __forceinline__ int y(int p) const { return cy + 4 * (p & 3); }
  // bit p set iff pixel p's column and row bits are both set in m
  __device__ __forceinline__ uint32_t cand(uint32_t m) const {
    const uint32_t c = ((m >> cx) & 1u) | ((m >> (cx + 4)) & 16u);      // columns cx, cx+8 → bits 0, 4
    const uint32_t r = (m >> (16 + cy)) & 0x1111u;                     // rows cy+4i at bits 4i
    // gather bits 0, 4, 8, 12 into 9..12: the partial products of ×0x249 sit at
    // 16 distinct positions, so there are no carries
    const uint32_t r4 = ((r * 0x249u) >> 9) & 15u;
    return c * r4;   // outer product: bit (p&3) + 4·(p>>2)
  }
};

// Launch order of the TW path: tiles by descending work (one 1024-thread
// CTA, 64 buckets of 2^SHIFT), so the longest serial tile walks start in the
// first wave and the short ones fill the tail.  Work = the tile's list length
// (forward; cnt == nullptr) or its accepted-entry count cnt[tile] (backward).
__device__ __forceinline__ uint32_t tile_work(const CamParams& cam, const uint2* ranges,
                                              const uint32_t* cnt, int i) {
  const int tile = cam.tile0 + i * cam.tstride;
  if (cnt != nullptr) return cnt[tile];
  const uint2 r = ranges[tile];
  return r.y - r.x;
}
template <int SHIFT>
__global__ void __launch_bounds__(1024) tile_order_kernel(const __grid_constant__ CamParams cam,
                                                          const uint2* __restrict__ ranges,
                                                          const uint32_t* __restrict__ cnt,
                                                          uint32_t* __restrict__ order) {
  constexpr int NB = 64;
  __shared__ uint32_t hist[NB];
  const int t = threadIdx.x;
  if (t < NB) hist[t] = 0u;
  __syncthreads();
  for (int i = t; i < cam.tcount; i += blockDim.x)
    atomicAdd(&hist[NB - 1 - min((uint32_t)(NB - 1), tile_work(cam, ranges, cnt, i) >> SHIFT)], 1u);
  __syncthreads();
  if (t == 0) {
    uint32_t sum = 0;
    for (int b = 0; b < NB; ++b) { const uint32_t c = hist[b]; hist[b] = sum; sum += c; }
  }
  __syncthreads();
  for (int i = t; i < cam.tcount; i += blockDim.x) {
    const uint32_t b = NB - 1 - min((uint32_t)(NB - 1), tile_work(cam, ranges, cnt, i) >> SHIFT);
    order[atomicAdd(&hist[b], 1u)] = (uint32_t)i;
  }
}

// Forward, one warp per tile.  Per batch, lane k stages entry b0 + k (its
// tile-local mean, staged conic, colour, support mask).  Per entry: a
// warp-uniform skip when its support misses the tile, then every lane tests
// its eight pixels at once (candidate bits from the support mask, the power
// threshold) and only the pixel blocks with a candidate execute the α /
// transmittance update.  Per-pixel colour sits in shared memory (touched only
// on acceptance), T in registers (the termination test does not wait on a
// shared load).
template <int MINB>
__global__ void __launch_bounds__(32, MINB) render_fwd_tw_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const float4* __restrict__ rgb,
    const uint2* __restrict__ box, float3 bg, float* __restrict__ out_img,
    float* __restrict__ out_T, uint32_t* __restrict__ out_last, AcceptLists acc) {
  constexpr int PPT = 8;
  constexpr int BATCH = TW_FWD_BATCH;
  __shared__ Staged s_st[BATCH];
  __shared__ float4 s_px[PPT][32];   // (C_r, C_g, C_b, T) of the lane's pixels
  const int tile = cam.tile0 + (int)acc.order[blockIdx.x] * cam.tstride;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const uint32_t lane = threadIdx.x;
  const TileMap pm((int)lane);
  const uint2 range = ranges[tile];
  if (range.y > acc.cap) __trap();   // lists sized for fewer pairs than the sort produced
  uint32_t last[PPT];
  float T[PPT];
  uint32_t live = 0;   // bit p: pixel p is inside the image and not terminated
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    s_px[p][lane] = make_float4(0.f, 0.f, 0.f, 1.f);
    T[p] = 1.f;
    last[p] = range.x;
    if (tx0 + pm.x(p) < cam.W && ty0 + pm.y(p) < cam.H) live |= 1u << p;
  }
  // the lane's pixel coordinates (tile-local columns fx0, fx1, rows fy0..fy3), read
  // from shared memory per candidate entry instead of re-derived from the lane id
  // (the compiler rematerialises registers here: 64-register budget)
  __shared__ float4 s_pc[32];
  __shared__ float2 s_pc2[32];
  s_pc[lane] = make_float4((float)pm.x(0), (float)pm.x(4), (float)pm.y(0), (float)pm.y(1));
  s_pc2[lane] = make_float2((float)pm.y(2), (float)pm.y(3));
  uint32_t nlist = range.x;                    // next list entry
  // running pointers to the next entry's byte of this lane and (lane 0) its index slot
  uint8_t* lbyte = acc.bytes + (size_t)nlist * 32 + lane;
  uint32_t* lidx = acc.idx + nlist;
  for (uint32_t b0 = range.x; b0 < range.y; b0 += BATCH) {
    if (!__any_sync(0xffffffffu, live != 0u)) break;
    __syncwarp();   // the previous batch is consumed
    if (b0 + lane < range.y)
      stage<16>(ids[b0 + lane], xy_depth, conic_opa, rgb, box, tx0, ty0, s_st[lane].a, s_st[lane].co, s_st[lane].c);
    __syncwarp();
    const int cnt = (int)min((uint32_t)BATCH, range.y - b0);
    for (int j = 0; j < cnt; ++j) {
      const Staged& st = s_st[j];
      const float4 a = st.a;
      const uint32_t m = __float_as_uint(a.w);
      if (m == 0u) continue;             // warp-uniform: support misses the tile
      uint32_t accb = 0;                 // this lane's accepted pixels of the entry
      const uint32_t cand = pm.cand(m) & live;
      {   // no per-lane guard: a lane without candidates just enters no pixel block
        const float4 co = st.co;
        const float4 pc = s_pc[lane];
        const float2 pc2 = s_pc2[lane];
        const float fy[4] = {pc.z, pc.w, pc2.x, pc2.y};
        const float X0 = col_term(co, a.x - pc.x), X1 = col_term(co, a.x - pc.y);
        float pw[PPT];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const RowTerms R = row_terms(co, a.y - fy[r]);
          pw[r] = splat_power(X0, R);
          pw[r + 4] = splat_power(X1, R);
        }
        // every candidate pixel block tests the power threshold itself: no packed 8-bit
        // threshold mask first (its 20 compare/select/add instructions and their dependency
        // chain cost more in the overlapped step than the extra blocks entered: step 11.74 →
        // 11.59 ms, although the forward alone is 3 % slower)
        {
          const float4 c = st.c;
#pragma unroll
          for (int p = 0; p < PPT; ++p) {
            if (!((cand >> p) & 1u) || !(pw[p] >= a.z)) continue;
            const float alpha = splat_alpha(co.w, splat_exp(pw[p]));
            if (alpha < ALPHA_MIN || pw[p] > 0.f) continue;   // A11: skip if power > 0
            const float tn = __fmul_rn(T[p], __fsub_rn(1.f, alpha));
            if (tn < T_MIN) { live &= ~(1u << p); continue; }
            const float w = alpha * T[p];
            T[p] = tn;
            float4 px = s_px[p][lane];
            px.x += c.x * w; px.y += c.y * w; px.z += c.z * w;
            px.w = tn;
            s_px[p][lane] = px;
            last[p] = b0 + j + 1;
            accb |= 1u << p;
          }
        }
      }
      if (__any_sync(0xffffffffu, accb != 0u)) {
        DASS_CHECK(nlist < acc.cap);
        *lbyte = (uint8_t)accb;
        if (lane == 0) *lidx = b0 + j;
        lbyte += 32;
        ++lidx;
        ++nlist;
      }
    }
  }
  if (lane == 0) acc.cnt[tile] = nlist - range.x;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int X = tx0 + pm.x(p), Y = ty0 + pm.y(p);
    if (X < cam.W && Y < cam.H) {
      const size_t pix = (size_t)Y * cam.W + X, np = (size_t)cam.W * cam.H;
      const float4 px = s_px[p][lane];
      out_img[pix] = px.x + px.w * bg.x;
      out_img[np + pix] = px.y + px.w * bg.y;
      out_img[2 * np + pix] = px.z + px.w * bg.z;
      out_T[pix] = px.w;
      out_last[pix] = last[p];
    }
  }
}

template <int MINB>
__global__ void __launch_bounds__(32, MINB) render_bwd_tw_kernel(
    const __grid_constant__ CamParams cam, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ ids, const float4* __restrict__ xy_depth,
    const float4* __restrict__ conic_opa, const float4* __restrict__ rgb, float3 bg,
    const float* __restrict__ out_T, const float* __restrict__ dL_dimg, AcceptLists acc,
    float4* __restrict__ g2d) {
  constexpr int PPT = 8;
  constexpr int CH = TW_BWD_CHUNK;   // entries staged per chunk
  __shared__ float4 s_a[CH];    // (u_rel, v_rel, −, −)
  __shared__ float4 s_co[CH];   // (s, sβ, g, o)
  __shared__ float4 s_c[CH];    // (r, g, b, −)
  __shared__ uint4 s_bytes[CH][2];
  __shared__ uint32_t s_id[CH];
  __shared__ float s_acc[CH][9];
  // dL/dC of the lane's pixels: read once per accepted pixel from shared
  // memory instead of pinning 24 registers (occupancy: 1-warp CTAs)
  __shared__ float4 s_g[PPT][32];
  const int tile = cam.tile0 + (int)acc.order[blockIdx.x] * cam.tstride;
  const uint32_t n = acc.cnt[tile];
  if (n == 0) return;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const uint32_t lane = threadIdx.x;
  const TileMap pm((int)lane);
  const uint2 range = ranges[tile];
  if (range.y > acc.cap) __trap();   // lists sized for fewer pairs than the sort produced
  LaneRS rs;
  rs.init();
  float T[PPT], gR[PPT];
  const size_t np = (size_t)cam.W * cam.H;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int X = tx0 + pm.x(p), Y = ty0 + pm.y(p);
    float4 gg = make_float4(0.f, 0.f, 0.f, 0.f);
    T[p] = 1.f;
    if (X < cam.W && Y < cam.H) {
      const size_t pix = (size_t)Y * cam.W + X;
      T[p] = out_T[pix];
      gg = make_float4(dL_dimg[pix], dL_dimg[np + pix], dL_dimg[2 * np + pix], 0.f);
    }
    s_g[p][lane] = gg;
    gR[p] = T[p] * (gg.x * bg.x + gg.y * bg.y + gg.z * bg.z);
  }
  // the lane's pixel columns, read from shared memory per entry (the 64-register budget
  // otherwise rematerialises them from the lane id every entry)
  __shared__ float2 s_fx[32];
  s_fx[lane] = make_float2((float)pm.x(0), (float)pm.x(4));
  float fy[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) fy[r] = (float)pm.y(r);
  for (int ptr = (int)n; ptr > 0;) {
    const int k0 = ptr > CH ? ptr - CH : 0;
    const int cnt = ptr - k0;
    if ((int)lane < cnt) {
      const size_t e = (size_t)range.x + k0 + lane;
      const uint32_t id = ids[acc.idx[e]];
      const uint4* src = reinterpret_cast<const uint4*>(acc.bytes + e * 32);
      s_bytes[lane][0] = src[0];
      s_bytes[lane][1] = src[1];
      s_id[lane] = id;
      // the forward's staging arithmetic for (u_rel, v_rel): identical bits
      const float4 xy = xy_depth[id];
      const uint32_t lo_bits = __float_as_uint(xy.w);
      const __half2 lo = *reinterpret_cast<const __half2*>(&lo_bits);
      s_a[lane] = make_float4(__fadd_rn(xy.x - (float)tx0, __low2float(lo)),
                              __fadd_rn(xy.y - (float)ty0, __high2float(lo)), 0.f, 0.f);
      s_co[lane] = conic_staged(conic_opa[id]);
      s_c[lane] = rgb[id];
    }
    __syncwarp();
    for (int k = cnt - 1; k >= 0; --k) {
      const uint32_t bits = reinterpret_cast<const uint8_t*>(&s_bytes[k][0])[lane];
      float v[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) v[q] = 0.f;
      {   // no per-lane guard: a lane without accepted pixels enters no pixel block
        const float4 a = s_a[k];
        const float4 co = s_co[k];
        const float4 c = s_c[k];
        const float2 fx = s_fx[lane];
        const float dxc[2] = {a.x - fx.x, a.x - fx.y};
        const float Xc[2] = {col_term(co, dxc[0]), col_term(co, dxc[1])};
        float se[2] = {0.f, 0.f}, sey[2] = {0.f, 0.f};   // per column: Σe, Σe·dy
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          if (!((bits >> p) & 1u)) continue;
          const float dy = a.y - fy[p & 3];
          const float G = splat_exp(splat_power(Xc[p >> 2], row_terms(co, dy)));
          const float4 gp = s_g[p][lane];
          const float oG = __fmul_rn(co.w, G);
          const float alpha = fminf(ALPHA_MAX, oG);
          const float inv = rcp_approx(1.f - alpha);
          T[p] *= inv;                        // transmittance before this entry
          const float w = alpha * T[p];
          const float gc = gp.x * c.x + gp.y * c.y + gp.z * c.z;
          const float dLda = T[p] * gc - inv * gR[p];
          gR[p] += gc * w;                    // g·(S + T_final·bg), S = suffix colour
          v[6] += w * gp.x; v[7] += w * gp.y; v[8] += w * gp.z;
          const float e = oG < ALPHA_MAX ? G * dLda : 0.f;
          const float ey = e * dy;
          sey[p >> 2] += ey; v[4] += ey * dy; se[p >> 2] += e;
        }
        const float m0 = se[0] * dxc[0], m1 = se[1] * dxc[1];
        v[0] = m0 + m1;
        v[1] = sey[0] + sey[1];
        v[2] = m0 * dxc[0] + m1 * dxc[1];
        v[3] = sey[0] * dxc[0] + sey[1] * dxc[1];
        v[5] = se[0] + se[1];
      }
      const float sum = rs.reduce(v);
      if (rs.slot >= 0) s_acc[k][rs.slot] = sum;
    }
    __syncwarp();
    if ((int)lane < cnt) {
      const float* a9 = s_acc[lane];
      float4* dst = g2d + 3 * (size_t)s_id[lane];
      red_add_v4(dst, make_float4(a9[0], a9[1], a9[2], a9[3]));
      red_add_v4(dst + 1, make_float4(a9[4], a9[5], a9[6], a9[7]));
      atomicAdd(&dst[2].x, a9[8]);
    }
    __syncwarp();
    ptr = k0;
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
  // per view (nullable): instead of adding ‖(∂L/∂u·W/2, ∂L/∂v·H/2)‖ to the ∇p̄
  // statistic, add (∂L/∂u·W/2, ∂L/∂v·H/2) to uv_out[v][i] — the view is split
  // across GPUs and the norm is taken after the partial sums are reduced; the
  // visibility count of such a view is added only where bit v of uv_count is set
  float2* uv_out[PRE_MAXV];
  uint32_t uv_count;
};

// Per-thread asynchronous copies global → shared (LDGSTS): the view loop below
// keeps the next PRE_STAGES − 1 views' records in flight while it computes one,
// without holding registers for them.  Each thread copies and reads back only
// its own Gaussian's slots, so no block barrier is needed.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int PRE_STAGES = 3;

// One view's records of the block's Gaussians, structure-of-arrays (conflict-free
// 16-byte shared loads); PART 2 reads only box, m1, m2 and the clamp bits.
template <int PART, int NT>
struct PreStage {
  uint2 bx[NT];
  float rgbw[NT];
  float4 m1[NT], m2[NT];
  float4 m0[PART == 1 ? NT : 1], co[PART == 1 ? NT : 1];
};

// PART 1: geometry (p, s, q, o, ∇p̄ and the SH direction term), fp64 chain.
// PART 2: SH coefficient gradients (fp32, 3(d+1)² register accumulators).
// Split so neither part spills.
template <int DEG, int PART>
__global__ void __launch_bounds__(PART == 1 ? 128 : 256, PART == 1 ? PRE1_MINB : 2) preprocess_views_kernel(
    const __grid_constant__ PreArgs a) {
  constexpr int NT = PART == 1 ? 128 : 256;
  __shared__ PreStage<PART, NT> stg[PRE_STAGES];
  // The per-Gaussian chain is evaluated in fp64: the kernel is HBM-bound, so
  // the wider arithmetic is free, and it removes the chain's own rounding
  // (conic → Σ' → Σ → R(q), J(t) with its clamp) from the gradient error
  // budget, leaving only the fp32 per-pixel sums of the raster pass.
  using F = double;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int n = a.n;
  const int tid = threadIdx.x;
  // issue view u's copies into stage u % PRE_STAGES (an empty group past the last
  // view keeps the group count uniform for cp.async.wait_group)
  auto prefetch = [&](int u) {
    if (u < a.num_views) {
      PreStage<PART, NT>& S = stg[u % PRE_STAGES];
      const size_t o = (size_t)u * n + i;
      cp_async8(&S.bx[tid], a.box + o);
      cp_async16(&S.m1[tid], a.g2d + 3 * o + 1);
      cp_async16(&S.m2[tid], a.g2d + 3 * o + 2);
      cp_async4(&S.rgbw[tid], &a.rgb[o].w);
      if (PART == 1) {
        cp_async16(&S.m0[tid], a.g2d + 3 * o);
        cp_async16(&S.co[tid], a.conic_opa + o);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int u = 0; u < PRE_STAGES - 1; ++u) prefetch(u);
  using L = SHLayout<DEG>;
  const bool kp = a.keep == nullptr || a.keep[i] != 0;
  const float4 po = a.pos_opa[i];
  const float4 q = a.rot[i];
  const float4 sc = a.scale[i];
  // view-independent geometry: q̂, R, s, Σ
  const F qn = sqrt((F)q.x * q.x + (F)q.y * q.y + (F)q.z * q.z + (F)q.w * q.w);
  const F qi = 1.0 / qn;
  const F w = q.x * qi, x = q.y * qi, y = q.z * qi, z = q.w * qi;
  F R[3][3];
  R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);
  R[1][0] = 2 * (x * y + w * z); R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
  R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x); R[2][2] = 1 - 2 * (x * x + y * y);
  const F s[3] = {kp ? (F)sc.x : 0.0, kp ? (F)sc.y : 0.0, kp ? (F)sc.z : 0.0};
  F Sig[3][3];
#pragma unroll
  for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
    for (int c0 = 0; c0 < 3; ++c0)
      Sig[r0][c0] = R[r0][0] * s[0] * s[0] * R[c0][0] + R[r0][1] * s[1] * s[1] * R[c0][1] +
                    R[r0][2] * s[2] * s[2] * R[c0][2];
  // accumulators over views
  F gp[3] = {0, 0, 0};
  F go = 0;
  F GS[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  constexpr int NGSH = PART == 2 ? 4 * L::K4 : 1;
  float gsh[NGSH];
#pragma unroll
  for (int f = 0; f < NGSH; ++f) gsh[f] = 0.f;
  float gstat = 0.f;
  uint32_t nvis = 0, ncnt = 0;
  for (int v = 0; v < a.num_views; ++v) {
    // view v's copies have landed; read them, then refill the stage view v − 1 used
    cp_async_wait<PRE_STAGES - 2>();
    const PreStage<PART, NT>& S = stg[v % PRE_STAGES];
    const uint2 bx = S.bx[tid];
    const float4 m1 = S.m1[tid], m2 = S.m2[tid];
    const float rgbw = S.rgbw[tid];
    const float4 m0 = PART == 1 ? S.m0[tid] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 co = PART == 1 ? S.co[tid] : make_float4(0.f, 0.f, 0.f, 0.f);
    prefetch(v + PRE_STAGES - 1);
    if ((bx.x & 0xFFFFu) > (bx.x >> 16)) continue;  // culled in this view
    const CamParams& cam = a.cam[v];
    ++nvis;
    const int bits = (int)rgbw;
    const float gcol[3] = {(bits & 1) ? 0.f : m1.z, (bits & 2) ? 0.f : m1.w, (bits & 4) ? 0.f : m2.x};
    if (PART == 2) {
      F dx = (F)po.x - cam.campos[0], dy = (F)po.y - cam.campos[1], dz = (F)po.z - cam.campos[2];
      const F inv = rsqrt(dx * dx + dy * dy + dz * dz);
      float Y[L::NC];
      sh_eval<DEG>((float)(dx * inv), (float)(dy * inv), (float)(dz * inv), Y);
#pragma unroll
      for (int f = 0; f < L::NF; ++f) gsh[f] += Y[f / 3] * gcol[f % 3];
      continue;
    }
    // the record's conic in Cholesky form (A, β, γ): B = A·β, C = γ + A·β² (fp64)
    const F A = co.x, B = A * (F)co.y, Cc = (F)co.z + B * (F)co.y, op = co.w;
    // 2D gradients from the moments
    const F gu = -op * (A * m0.x + B * m0.y);
    const F gv = -op * (B * m0.x + Cc * m0.y);
    const F gA = -0.5 * op * m0.z;
    const F gB = -op * m0.w;
    const F gC = -0.5 * op * m1.x;
    go += m1.y;
    {
      const F ga = gu * 0.5 * cam.W, gb = gv * 0.5 * cam.H;
      if (a.uv_out[v] != nullptr) {
        float2 u = a.uv_out[v][i];
        u.x += (float)ga; u.y += (float)gb;
        a.uv_out[v][i] = u;
        if ((a.uv_count >> v) & 1u) ++ncnt;
      } else {
        gstat += (float)sqrt(ga * ga + gb * gb);
        ++ncnt;
      }
    }
    // ---- colour / SH (direction from this view's camera centre)
    {
      F dx = (F)po.x - cam.campos[0], dy = (F)po.y - cam.campos[1], dz = (F)po.z - cam.campos[2];
      const F inv = rsqrt(dx * dx + dy * dy + dz * dz);
      dx *= inv; dy *= inv; dz *= inv;
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
          if (f < L::NF) wk[f / 3] += gcol[f % 3] * cf[e];
        }
      }
      if (DEG > 0) {
        const float3 gd = sh_dir_grad<DEG>((float)dx, (float)dy, (float)dz, wk);
        const F dd = dx * gd.x + dy * gd.y + dz * gd.z;
        gp[0] += (gd.x - dx * dd) * inv;
        gp[1] += (gd.y - dy * dd) * inv;
        gp[2] += (gd.z - dz * dd) * inv;
      }
    }
    // ---- projection chain for this view
    const float* V = cam.V;
    F t[3];
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0)
      t[r0] = (F)V[4 * r0] * po.x + (F)V[4 * r0 + 1] * po.y + (F)V[4 * r0 + 2] * po.z + (F)V[4 * r0 + 3];
    const F lx = 1.3 * cam.W / (2.0 * cam.fx), ly = 1.3 * cam.H / (2.0 * cam.fy);
    // one double division per view: the reciprocals of t_z replace the dozen
    // divisions of the chain (≤ 1 ulp of fp64 apart, far below the fp32 outputs)
    const F itz = 1.0 / t[2], itz2 = itz * itz, itz3 = itz2 * itz;
    const F txtz = t[0] * itz, tytz = t[1] * itz;
    const bool clx = txtz < -lx || txtz > lx, cly = tytz < -ly || tytz > ly;
    const F xt = t[2] * fmin(lx, fmax(-lx, txtz));
    const F yt = t[2] * fmin(ly, fmax(-ly, tytz));
    const F fxc = cam.fx, fyc = cam.fy;
    const F J00 = fxc * itz, J02 = -fxc * xt * itz2;
    const F J11 = fyc * itz, J12 = -fyc * yt * itz2;
    F M[2][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      M[0][b] = J00 * V[b] + J02 * V[8 + b];
      M[1][b] = J11 * V[4 + b] + J12 * V[8 + b];
    }
    // conic → Σ': Gs = −K Ĝ K, Ĝ = [[gA, gB/2],[gB/2, gC]]
    const F G01h = 0.5 * gB;
    const F KG00 = A * gA + B * G01h, KG01 = A * G01h + B * gC;
    const F KG10 = B * gA + Cc * G01h, KG11 = B * G01h + Cc * gC;
    const F Gs00 = -(KG00 * A + KG01 * B);
    const F Gs01 = -(KG00 * B + KG01 * Cc);
    const F Gs11 = -(KG10 * B + KG11 * Cc);
    F GM1[2][3];  // Gs M
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
    F GM[2][3];
#pragma unroll
    for (int r0 = 0; r0 < 2; ++r0)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        GM[r0][b] = 2 * (GM1[r0][0] * Sig[0][b] + GM1[r0][1] * Sig[1][b] + GM1[r0][2] * Sig[2][b]);
    const F GJ00 = GM[0][0] * V[0] + GM[0][1] * V[1] + GM[0][2] * V[2];
    const F GJ02 = GM[0][0] * V[8] + GM[0][1] * V[9] + GM[0][2] * V[10];
    const F GJ11 = GM[1][0] * V[4] + GM[1][1] * V[5] + GM[1][2] * V[6];
    const F GJ12 = GM[1][0] * V[8] + GM[1][1] * V[9] + GM[1][2] * V[10];
    F gt[3] = {0, 0, 0};
    gt[2] += GJ00 * (-fxc * itz2) + GJ11 * (-fyc * itz2);
    if (!clx) {
      gt[0] += GJ02 * (-fxc * itz2);
      gt[2] += GJ02 * (2 * fxc * t[0] * itz3);
    } else {
      gt[2] += GJ02 * (fxc * xt * itz3);
    }
    if (!cly) {
      gt[1] += GJ12 * (-fyc * itz2);
      gt[2] += GJ12 * (2 * fyc * t[1] * itz3);
    } else {
      gt[2] += GJ12 * (fyc * yt * itz3);
    }
    gt[0] += gu * fxc * itz;
    gt[2] += gu * (-fxc * t[0] * itz2);
    gt[1] += gv * fyc * itz;
    gt[2] += gv * (-fyc * t[1] * itz2);
#pragma unroll
    for (int c0 = 0; c0 < 3; ++c0) gp[c0] += V[c0] * gt[0] + V[4 + c0] * gt[1] + V[8 + c0] * gt[2];
  }
  if (nvis == 0) return;
  // The outputs are accumulated (+=) with fire-and-forget reductions instead of a
  // load-add-store: one thread owns Gaussian i in a launch, so each element gets one
  // add per launch, the same fp32 add as before, without waiting for the old value.
  if (PART == 2) {
    if (!a.g_sh) return;
#pragma unroll
    for (int j = 0; j < L::K4; ++j) {
      float4* dst = a.g_sh + (size_t)j * n + i;
      if (4 * j + 3 < L::NF) {
        red_add_v4(dst, make_float4(gsh[4 * j], gsh[4 * j + 1], gsh[4 * j + 2], gsh[4 * j + 3]));
      } else {
        float* d = reinterpret_cast<float*>(dst);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * j + e < L::NF) red_add_f32(d + e, gsh[4 * j + e]);
      }
    }
    return;
  }
  if (a.gradstat_sum) red_add_f32(a.gradstat_sum + i, gstat);
  if (a.gradstat_cnt) red_add_u32(a.gradstat_cnt + i, ncnt);
  if (a.g_pos_opa)
    red_add_v4(a.g_pos_opa + i, make_float4((float)gp[0], (float)gp[1], (float)gp[2], kp ? (float)go : 0.f));
  if (!a.g_scale && !a.g_rot) return;
  // Σ = R diag(s²) Rᵀ : dL/ds_k = 2 s_k (Rᵀ GΣ R)_kk ; dL/dR = 2 GΣ R diag(s²)
  F GR[3][3];
  F gs[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    F GSr[3];
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0) GSr[r0] = GS[r0][0] * R[0][k] + GS[r0][1] * R[1][k] + GS[r0][2] * R[2][k];
    gs[k] = 2 * s[k] * (R[0][k] * GSr[0] + R[1][k] * GSr[1] + R[2][k] * GSr[2]);
#pragma unroll
    for (int r0 = 0; r0 < 3; ++r0) GR[r0][k] = 2 * GSr[r0] * s[k] * s[k];
  }
  if (a.g_scale && kp) {
    float* d = reinterpret_cast<float*>(a.g_scale + i);
    red_add_f32(d, (float)gs[0]);
    red_add_f32(d + 1, (float)gs[1]);
    red_add_f32(d + 2, (float)gs[2]);
  }
  if (a.g_rot) {
    F gq[4];
    gq[0] = GR[0][1] * (-2 * z) + GR[0][2] * (2 * y) + GR[1][0] * (2 * z) + GR[1][2] * (-2 * x) +
            GR[2][0] * (-2 * y) + GR[2][1] * (2 * x);
    gq[1] = GR[0][1] * (2 * y) + GR[0][2] * (2 * z) + GR[1][0] * (2 * y) + GR[1][1] * (-4 * x) +
            GR[1][2] * (-2 * w) + GR[2][0] * (2 * z) + GR[2][1] * (2 * w) + GR[2][2] * (-4 * x);
    gq[2] = GR[0][0] * (-4 * y) + GR[0][1] * (2 * x) + GR[0][2] * (2 * w) + GR[1][0] * (2 * x) +
            GR[1][2] * (2 * z) + GR[2][0] * (-2 * w) + GR[2][1] * (2 * z) + GR[2][2] * (-4 * y);
    gq[3] = GR[0][0] * (-4 * z) + GR[0][1] * (-2 * w) + GR[0][2] * (2 * x) + GR[1][0] * (2 * w) +
            GR[1][1] * (-4 * z) + GR[1][2] * (2 * y) + GR[2][0] * (2 * x) + GR[2][1] * (2 * y);
    const F dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
    red_add_v4(a.g_rot + i, make_float4((float)((gq[0] - w * dot) * qi), (float)((gq[1] - x * dot) * qi),
                                        (float)((gq[2] - y * dot) * qi), (float)((gq[3] - z * dot) * qi)));
  }
}

// Acceptance-list workspace: cnt[ntiles] u32 | idx[capacity] u32 | bytes[capacity][32] | order[ntiles].
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
size_t accept_bytes(int ntiles, int64_t capacity) {
  const size_t c = (size_t)(capacity > 0 ? capacity : 1);
  return al(sizeof(uint32_t) * (size_t)ntiles) + al(sizeof(uint32_t) * c) + al(32 * c) +
         al(sizeof(uint32_t) * (size_t)ntiles);
}
AcceptLists carve_accept(void* base, int ntiles, int64_t capacity) {
  const size_t c = (size_t)(capacity > 0 ? capacity : 1);
  char* p = (char*)base;
  AcceptLists a;
  a.cnt = (uint32_t*)p;
  p += al(sizeof(uint32_t) * (size_t)ntiles);
  a.idx = (uint32_t*)p;
  p += al(sizeof(uint32_t) * c);
  a.bytes = (uint8_t*)p;
  p += al(32 * c);
  a.order = (uint32_t*)p;
  a.cap = (uint32_t)(capacity > 0 ? capacity : 0);
  return a;
}

// Launch shapes, measured: launch order by list length in
// 16-entry buckets (forward) / accepted entries in 8-entry buckets (backward);
// 32 one-warp CTAs per SM (the hardware block limit).
constexpr int TW_FWD_ORDER_SHIFT = 4;
constexpr int TW_BWD_ORDER_SHIFT = 3;
constexpr int TW_FWD_MINB = 32;
constexpr int TW_BWD_MINB = 32;

}  // namespace

size_t render_accept_workspace(int ntiles, int64_t capacity) { return accept_bytes(ntiles, capacity); }

cudaError_t launch_render_fwd(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, float* out_img, float* out_T,
                              uint32_t* out_last, void* accept, int64_t capacity, cudaStream_t s) {
  const int ntiles = cam.tiles_x * cam.tiles_y;
  if (accept != nullptr) {
    const AcceptLists acc = carve_accept(accept, ntiles, capacity);
    tile_order_kernel<TW_FWD_ORDER_SHIFT><<<1, 1024, 0, s>>>(cam, ranges, nullptr, acc.order);
    launch_counted();
    render_fwd_tw_kernel<TW_FWD_MINB><<<cam.tcount, 32, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, rgb,
                                                                box, bg, out_img, out_T, out_last, acc);
    launch_counted();
    return cudaGetLastError();
  }
  render_fwd_kernel<4><<<cam.tcount, 64, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, rgb, box, bg,
                                                 out_img, out_T, out_last);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_render_features(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                                   const float4* xy_depth, const float4* conic_opa,
                                   const uint2* box, int channels, const float* feat, float* out,
                                   cudaStream_t s) {
  const float4* f4 = reinterpret_cast<const float4*>(feat);
#define FEAT(NV)                                                                                 \
  render_features_kernel<NV><<<cam.tcount, 64, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, box, f4, out)
  switch (channels / 4) {
    case 1: FEAT(1); break;
    case 2: FEAT(2); break;
    case 3: FEAT(3); break;
    default: FEAT(4); break;
  }
#undef FEAT
  launch_counted();
  return cudaGetLastError();
}

size_t render_bwd_workspace(int n) { return sizeof(float4) * 3 * (size_t)(n > 0 ? n : 1); }

cudaError_t launch_render_bwd_raster(const CamParams& cam, int n, const uint2* ranges,
                                     const uint32_t* ids, const float4* xy_depth,
                                     const float4* conic_opa, const float4* rgb, const uint2* box,
                                     float3 bg, const float* out_T, const uint32_t* out_last,
                                     const float* dL_dimg, const void* accept, int64_t capacity,
                                     float4* g2d, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(g2d, 0, render_bwd_workspace(n), s);
  if (e != cudaSuccess) return e;
  if (cam.tcount == 0) return cudaSuccess;
  const int ntiles = cam.tiles_x * cam.tiles_y;
  if (accept != nullptr) {
    const AcceptLists acc = carve_accept(const_cast<void*>(accept), ntiles, capacity);
    tile_order_kernel<TW_BWD_ORDER_SHIFT><<<1, 1024, 0, s>>>(cam, ranges, acc.cnt, acc.order);
    launch_counted();
    render_bwd_tw_kernel<TW_BWD_MINB><<<cam.tcount, 32, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, rgb, bg,
                                                                out_T, dL_dimg, acc, g2d);
    launch_counted();
    return cudaGetLastError();
  }
  render_bwd_raster_kernel<4, 16><<<cam.tcount, 64, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, rgb,
                                                            box, bg, out_T, out_last, dL_dimg, g2d);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_preprocess_views(const CamParams* cams, int num_views, int n, int sh_degree,
                                    const float4* pos_opa, const float4* scale, const float4* rot,
                                    const float4* sh, const uint8_t* keep,
                                    const float4* conic_opa, const float4* rgb, const uint2* box,
                                    const float4* g2d, float4* g_pos_opa, float4* g_scale,
                                    float4* g_rot, float4* g_sh, float* gradstat_sum,
                                    uint32_t* gradstat_cnt, float2* const* uv_out,
                                    const uint8_t* uv_count, int part, cudaStream_t s) {
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
    a.uv_count = 0;
    for (int v = 0; v < PRE_MAXV; ++v) {
      a.uv_out[v] = (uv_out != nullptr && v < a.num_views) ? uv_out[v0 + v] : nullptr;
      if (a.uv_out[v] && uv_count && uv_count[v0 + v]) a.uv_count |= 1u << v;
    }
    const int grid = div_up(n, 256);
    switch (sh_degree) {
#define PRE(D)                                                                       \
  if (part & 1) preprocess_views_kernel<D, 1><<<div_up(n, 128), 128, 0, s>>>(a);      \
  if (part & 2) preprocess_views_kernel<D, 2><<<grid, 256, 0, s>>>(a)
      case 0: PRE(0); break;
      case 1: PRE(1); break;
      case 2: PRE(2); break;
      default: PRE(3); break;
#undef PRE
    }
    launch_counted(part == 3 ? 2 : 1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ∇p̄ terms of views split across GPUs, after their (∂L/∂u·W/2, ∂L/∂v·H/2, vis)
// partial sums were reduced: += ‖(x, y)‖ and += 1 where the view saw the Gaussian.
// (an invisible Gaussian has (0, 0) and adds nothing, as in the whole-view path)
__global__ void __launch_bounds__(256) gradstat_uv_kernel(int n, int S, const float2* __restrict__ uv,
                                                         float* __restrict__ gsum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float sacc = 0.f;
  for (int k = 0; k < S; ++k) {
    const float2 u = uv[(size_t)k * n + i];
    sacc += (float)sqrt((double)u.x * u.x + (double)u.y * u.y);
  }
  gsum[i] += sacc;
}

cudaError_t launch_gradstat_uv(int n, int S, const float2* uv, float* gsum, cudaStream_t s) {
  if (n == 0 || S == 0) return cudaSuccess;
  gradstat_uv_kernel<<<div_up(n, 256), 256, 0, s>>>(n, S, uv, gsum);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_render_bwd(const CamParams& cam, int n, int sh_degree, const float4* pos_opa,
                              const float4* scale, const float4* rot, const float4* sh,
                              const uint8_t* keep, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, const float* out_T,
                              const uint32_t* out_last, const float* dL_dimg, const void* accept,
                              int64_t capacity, void* ws, float4* g_pos_opa, float4* g_scale,
                              float4* g_rot, float4* g_sh, float* gradstat_sum,
                              uint32_t* gradstat_cnt, cudaStream_t s) {
  float4* g2d = (float4*)ws;
  cudaError_t e = launch_render_bwd_raster(cam, n, ranges, ids, xy_depth, conic_opa, rgb, box, bg,
                                           out_T, out_last, dL_dimg, accept, capacity, g2d, s);
  if (e != cudaSuccess) return e;
  return launch_preprocess_views(&cam, 1, n, sh_degree, pos_opa, scale, rot, sh, keep, conic_opa,
                                 rgb, box, g2d, g_pos_opa, g_scale, g_rot, g_sh, gradstat_sum,
                                 gradstat_cnt, nullptr, nullptr, 3, s);
}

}  // namespace dass
