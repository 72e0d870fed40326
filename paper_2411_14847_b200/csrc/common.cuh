// common.cuh — shared device helpers of libdass.so (sm_100a).
// The CUDA path shares nothing with oracle/ (see DESIGN.md §Boundary).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "dass.h"

// Device-side checks of the checked build (`python -m paper_2411_14847_b200.build --checked`
// → libdass_checked.so, -DDASS_CHECKED): index bounds and count invariants on the
// scatter / emission / list paths, a printf and a trap on violation.  This pool has
// compute-sanitizer closed, so tools/gpu_checked.sh runs the GPU tests on this build
// instead.  In the product build the checks compile to nothing.
#ifdef DASS_CHECKED
#include <cstdio>
#define DASS_CHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("DASS_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,      \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                 \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define DASS_CHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace dass {

constexpr int TILE = DASS_TILE;  // 16×16 pixel tiles (A04)
constexpr float ALPHA_MIN = 1.0f / 255.0f;  // A11
constexpr float ALPHA_MAX = 0.99f;          // A11
constexpr float T_MIN = 1e-4f;              // A12
constexpr float LOG2E = 1.4426950408889634f;

// Camera passed by value as a kernel parameter (__grid_constant__).
struct CamParams {
  int W, H, tiles_x, tiles_y;
  float fx, fy, cx, cy;
  float V[12];       // world→camera [R|t] row-major
  float near_plane;
  float campos[3];   // −Rᵀ t (SH direction origin)
  float T[16];       // Alg. 1 full projection (row-vector convention)
  // tile subset rendered by the tile kernels: tile = tile0 + blockIdx.x·tstride,
  // blockIdx.x < tcount (whole image: 0, 1, tiles_x·tiles_y)
  int tile0, tstride, tcount;
};

void launch_counted(int n = 1);  // bumps the dass_kernel_launches() counter

// Per-pixel power of Eq. 8, shared by every kernel that takes a per-pixel
// decision (render_fwd, render_bwd, render_stats, render_features) so all of
// them get identical fp32 bits (A35).
//
// The projected conic record (dass_project) is the Cholesky form of the 2×2
// inverse covariance K = [[A, B], [B, C]]:
//   conic_opa = (A, β, γ, o),  β = B/A = −Σ′_xy/Σ′_yy,  γ = C − B²/A = 1/Σ′_yy
// (β and γ from the fp64 Σ′, then rounded once), because
//   power = −½(A dx² + 2B dx dy + C dy²) = −[(s·dx + sβ·dy)² + (g·dy)²],
//   s = √(A/2), g = √(γ/2),
// is then minus a sum of two squares: an elongated splat's cross term no longer
// cancels against the diagonal terms (the form −½(A dx² + C dy²) − B dx dy
// lost up to ~1e-4 of the power in fp32 for needle-like splats, enough to move
// T by 4e-3 relative after a few dozen entries).  Staged as (s, sβ, g, o), a
// pixel (dx, dy) costs
//   column term X = s·dx,  row terms Y = sβ·dy, N = −(g·dy)·(g·dy)
//   t = X + Y;  power = fma(−t, t, N)          (all explicitly rounded)
// i.e. one FADD and one FFMA per pixel when X / (Y, N) are shared by the
// pixels of a column / row.
__device__ __forceinline__ float4 conic_staged(float4 co) {
  const float s = __fsqrt_rn(__fmul_rn(0.5f, co.x));
  return make_float4(s, __fmul_rn(s, co.y), __fsqrt_rn(__fmul_rn(0.5f, co.z)), co.w);
}
struct RowTerms {
  float y, n;   // sβ·dy, −(g·dy)²
};
__device__ __forceinline__ float col_term(const float4& sc, float dx) { return __fmul_rn(sc.x, dx); }
__device__ __forceinline__ RowTerms row_terms(const float4& sc, float dy) {
  const float z = __fmul_rn(sc.z, dy);
  return RowTerms{__fmul_rn(sc.y, dy), -__fmul_rn(z, z)};
}
__device__ __forceinline__ float splat_power(float X, const RowTerms& r) {
  const float t = __fadd_rn(X, r.y);
  return __fmaf_rn(-t, t, r.n);
}
__device__ __forceinline__ float splat_power(const float4& sc, float dx, float dy) {
  return splat_power(col_term(sc, dx), row_terms(sc, dy));
}

// exp(power) on the MUFU pipe: ex2.approx(power · log2 e).
__device__ __forceinline__ float splat_exp(float power) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(power, LOG2E)));
  return y;
}

// α = min(0.99, o·G) — Eq. 8's α_i with the 0.99 cap (A11).
__device__ __forceinline__ float splat_alpha(float o, float G) {
  return fminf(ALPHA_MAX, __fmul_rn(o, G));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// Vector reduction to global memory (sm_90+): one instruction adds 4 floats.
__device__ __forceinline__ void red_add_v4(float4* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ void red_add_f32(float* addr, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" :: "l"(addr), "f"(v) : "memory");
}
// Programmatic dependent launch (a kernel launched with the programmatic stream
// serialisation attribute may start before its predecessor on the stream ends):
// pdl_wait() blocks until the predecessor grid has completed and its writes are
// visible — every such kernel calls it before reading what the predecessor wrote;
// pdl_trigger() lets the dependent grid's blocks be scheduled once every block of
// this grid has issued it.  Both are no-ops for a kernel launched without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void red_add_u32(uint32_t* addr, uint32_t v) {
  asm volatile("red.global.add.u32 [%0], %1;" :: "l"(addr), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int div_up(int a, int b) { return (a + b - 1) / b; }

// Kernel-side copy of dass_hashgrid (f2), passed by value (__grid_constant__).
struct HashGridParams {
  int L, F, in;          // levels, features per entry, MLP inputs = L·F
  uint32_t T, Tmask;     // table rows per level (2^log2_table), T − 1
  uint32_t dense_mask;   // bit l: (res_l + 1)³ ≤ T → direct indexing
  int res[16];
  float lo[3], span[3];  // AABB min and (max − min)
};

}  // namespace dass

// Internal launchers (defined in the .cu files, called by api.cu).
namespace dass {
cudaError_t launch_shift(int n, const float4* pos, const float4* rot, const float4* mu,
                         const float4* sigma, const uint8_t* mask, float4* pos_out,
                         float4* rot_out, cudaStream_t s);
cudaError_t launch_shift_bwd(int n, const float4* rot, const float4* sigma, const uint8_t* mask,
                             const float4* g_pos_out, const float4* g_rot_out, float4* g_mu,
                             float4* g_sigma, cudaStream_t s);
// part: PROJECT_KEYS (key chain + footprint), PROJECT_RECORDS (fp64 records +
// colour; needs the keys' box), or both in that order
constexpr int PROJECT_KEYS = 1, PROJECT_RECORDS = 2;
cudaError_t launch_project_part(int part, const CamParams* cams, int num_views, int n,
                                int sh_degree, const float4* pos_opa, const float4* scale,
                                const float4* rot, const float4* sh, const uint8_t* keep,
                                float4* xy_depth, float4* conic_opa, float4* rgb, uint2* box,
                                uint4* rows, uint32_t* tiles, cudaStream_t s);
size_t binsort_workspace(int n, int num_tiles, int64_t capacity);
cudaError_t launch_binsort(const CamParams& cam, int n, const float4* xy_depth, const uint2* box,
                           const uint4* rows, const uint32_t* tiles, void* ws, int64_t capacity,
                           uint64_t* sorted_keys, uint32_t* sorted_ids, uint2* ranges,
                           uint32_t* num_pairs_dev, int pair_grid, cudaStream_t s);
// dass_bin_sort_shared's pair-pass grid (blocks that loop over the key tiles)
constexpr int BINSORT_SHARED_GRID = 74;
size_t render_accept_workspace(int ntiles, int64_t capacity);
cudaError_t launch_render_fwd(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, float* out_img, float* out_T,
                              uint32_t* out_last, void* accept, int64_t capacity, cudaStream_t s);
size_t render_bwd_workspace(int n);
cudaError_t launch_render_bwd(const CamParams& cam, int n, int sh_degree, const float4* pos_opa,
                              const float4* scale, const float4* rot, const float4* sh,
                              const uint8_t* keep, const uint2* ranges, const uint32_t* ids,
                              const float4* xy_depth, const float4* conic_opa, const float4* rgb,
                              const uint2* box, float3 bg, const float* out_T,
                              const uint32_t* out_last, const float* dL_dimg, const void* accept,
                              int64_t capacity, void* ws, float4* g_pos_opa, float4* g_scale,
                              float4* g_rot, float4* g_sh, float* gradstat_sum,
                              uint32_t* gradstat_cnt, cudaStream_t s);
cudaError_t launch_render_bwd_raster(const CamParams& cam, int n, const uint2* ranges,
                                     const uint32_t* ids, const float4* xy_depth,
                                     const float4* conic_opa, const float4* rgb, const uint2* box,
                                     float3 bg, const float* out_T, const uint32_t* out_last,
                                     const float* dL_dimg, const void* accept, int64_t capacity,
                                     float4* g2d, cudaStream_t s);
cudaError_t launch_preprocess_views(const CamParams* cams, int num_views, int n, int sh_degree,
                                    const float4* pos_opa, const float4* scale, const float4* rot,
                                    const float4* sh, const uint8_t* keep,
                                    const float4* conic_opa, const float4* rgb, const uint2* box,
                                    const float4* g2d, float4* g_pos_opa, float4* g_scale,
                                    float4* g_rot, float4* g_sh, float* gradstat_sum,
                                    uint32_t* gradstat_cnt, float2* const* uv_out,
                                    const uint8_t* uv_count, int part, cudaStream_t s);
cudaError_t launch_gradstat_uv(int n, int S, const float2* uv, float* gsum, cudaStream_t s);
size_t fidelity_loss_workspace(int W, int H);
cudaError_t launch_fidelity_loss(int W, int H, const float* img, const float* gt, float lambda,
                                 float dssim_scale, void* ws, float* loss, float* dL,
                                 cudaStream_t s);
cudaError_t launch_inherit_mask(int n, const float* m, uint8_t* keep, cudaStream_t s);
cudaError_t launch_inherit_mask_bwd(int n, const float* m, const float4* pos_opa,
                                    const float4* scale, const float4* g_pos_opa,
                                    const float4* g_scale, float lambda_inher, float* g_m,
                                    cudaStream_t s);
cudaError_t launch_render_features(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                                   const float4* xy_depth, const float4* conic_opa,
                                   const uint2* box, int channels, const float* feat, float* out,
                                   cudaStream_t s);
cudaError_t launch_densify_select(int n, const float* gsum, const uint32_t* gcnt,
                                  const uint8_t* s_err, float tau_pos, float tau_err,
                                  uint8_t* in_S, int* idx, int* counts, void* ws, cudaStream_t s);
cudaError_t launch_prune_select(int n, int first, const float4* pos_opa, float min_opacity,
                                uint8_t* keep, int* idx, int* counts, void* ws, cudaStream_t s);
cudaError_t launch_gather(int n_src, int k4, const float4* pos_opa, const float4* scale,
                          const float4* rot, const float4* sh, const uint8_t* dyn, int m,
                          const int* idx, int n_dst, int dst_offset, float4* o_pos_opa,
                          float4* o_scale, float4* o_rot, float4* o_sh, uint8_t* o_dyn,
                          cudaStream_t s);
cudaError_t launch_spawn_children(int n_src, int k4, const float4* pos_opa, const float4* scale,
                                  const float4* rot, const float4* sh, const uint8_t* dyn, int m,
                                  const int* idx, int K, float shrink, float child_opacity,
                                  uint64_t seed, int n_dst, int dst_offset, float4* o_pos_opa,
                                  float4* o_scale, float4* o_rot, float4* o_sh, uint8_t* o_dyn,
                                  cudaStream_t s);
size_t partition_workspace(int n);
cudaError_t launch_partition(int n, const uint8_t* mask, int* idx_dyn, int* idx_st, int* counts,
                             void* ws, cudaStream_t s);
cudaError_t launch_deform_fwd(const HashGridParams& g, const float* table, const float* mlp, int n,
                              const int* idx, const int* count, const float4* pos_opa, float4* mu,
                              float4* sigma, cudaStream_t s);
cudaError_t launch_deform_bwd(const HashGridParams& g, const float* table, const float* mlp, int n,
                              const int* idx, const int* count, const float4* pos_opa,
                              const float4* g_mu, const float4* g_sigma, float* g_table,
                              float* g_mlp, cudaStream_t s);
cudaError_t launch_error_map(const CamParams& cam, const float* rendered, const float* gt,
                             float gamma, float* err, uint32_t* dmask, int n_base,
                             const float4* pos_opa, uint8_t* s_err, cudaStream_t s);
size_t binsort_views_workspace(int V, int n, int64_t view_capacity);
cudaError_t launch_binsort_views(const CamParams& cam, int V, int n, const float4* xy_depth,
                                 const uint2* box, const uint4* rows, const uint32_t* tiles,
                                 void* ws_ptr,
                                 int64_t view_capacity, uint32_t* sorted_ids, uint2* ranges,
                                 uint32_t* view_pairs, cudaStream_t s);
cudaError_t launch_timestamp(uint64_t* out, cudaStream_t s);
cudaError_t launch_nonfinite(const float* x, long long n, uint32_t* count, cudaStream_t s);
cudaError_t launch_render_stats(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                                const float4* xy_depth, const float4* conic_opa, const uint2* box,
                                const float* out_T, const uint32_t* out_last,
                                unsigned long long* counters, cudaStream_t s);
}  // namespace dass
