// api.cu — the extern "C" boundary of libdass.so (include/dass.h).
// Argument validation happens here, before anything is enqueued; the kernels
// live in the other translation units.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace dass {

static std::atomic<uint64_t> g_launches{0};
void launch_counted(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

static thread_local std::string t_last_error;

static int fail(int status, const char* fmt, const char* what = "") {
  char buf[512];
  snprintf(buf, sizeof(buf), fmt, what);
  t_last_error = buf;
  return status;
}

static int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return DASS_OK;
  t_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return DASS_ERR_CUDA;
}

static int check_camera(const dass_camera* c) {
  if (c == nullptr) return fail(DASS_ERR_INVALID_ARG, "camera is null%s");
  if (c->width < 1 || c->width > 65535 || c->height < 1 || c->height > 65535)
    return fail(DASS_ERR_INVALID_ARG, "camera width/height must be in [1, 65535]%s");
  if (!(c->fx > 0.0f) || !(c->fy > 0.0f) || !std::isfinite(c->fx) || !std::isfinite(c->fy))
    return fail(DASS_ERR_INVALID_ARG, "camera fx, fy must be finite and > 0%s");
  return DASS_OK;
}

static CamParams to_params(const dass_camera* c) {
  CamParams p;
  p.W = c->width;
  p.H = c->height;
  p.tiles_x = div_up(c->width, TILE);
  p.tiles_y = div_up(c->height, TILE);
  p.fx = c->fx; p.fy = c->fy; p.cx = c->cx; p.cy = c->cy;
  for (int i = 0; i < 12; ++i) p.V[i] = c->viewmat[i];
  p.near_plane = c->near_plane;
  // camera centre −Rᵀ t (SH direction origin)
  for (int a = 0; a < 3; ++a)
    p.campos[a] = -(c->viewmat[0 * 4 + a] * c->viewmat[3] + c->viewmat[1 * 4 + a] * c->viewmat[7] +
                    c->viewmat[2 * 4 + a] * c->viewmat[11]);
  for (int i = 0; i < 16; ++i) p.T[i] = c->full_proj[i];
  p.tile0 = 0;
  p.tstride = 1;
  p.tcount = p.tiles_x * p.tiles_y;
  return p;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static int to_hashgrid(const dass_hashgrid* c, HashGridParams* g) {
  if (!c) return fail(DASS_ERR_INVALID_ARG, "hash-grid config is null%s");
  if (c->levels < 1 || c->levels > 16) return fail(DASS_ERR_INVALID_ARG, "levels must be in [1, 16]%s");
  if (c->features != 1 && c->features != 2 && c->features != 4)
    return fail(DASS_ERR_INVALID_ARG, "features must be 1, 2 or 4%s");
  const int in = c->levels * c->features;
  if (in % 4 != 0 || in > 64)
    return fail(DASS_ERR_INVALID_ARG, "levels*features must be a multiple of 4 and <= 64%s");
  if (c->log2_table < 1 || c->log2_table > 24)
    return fail(DASS_ERR_INVALID_ARG, "log2_table must be in [1, 24]%s");
  g->L = c->levels; g->F = c->features; g->in = in;
  g->T = 1u << c->log2_table; g->Tmask = g->T - 1u;
  g->dense_mask = 0;
  for (int l = 0; l < 16; ++l) g->res[l] = 1;
  for (int l = 0; l < c->levels; ++l) {
    const int N = c->resolution[l];
    if (N < 1 || N > (1 << 20)) return fail(DASS_ERR_INVALID_ARG, "resolution[l] must be in [1, 2^20]%s");
    g->res[l] = N;
    const uint64_t n1 = (uint64_t)N + 1;
    if (n1 * n1 * n1 <= (uint64_t)g->T) g->dense_mask |= 1u << l;
  }
  for (int k = 0; k < 3; ++k) {
    if (!std::isfinite(c->aabb_min[k]) || !std::isfinite(c->aabb_max[k]) ||
        !(c->aabb_max[k] > c->aabb_min[k]))
      return fail(DASS_ERR_INVALID_ARG, "aabb must be finite with max > min%s");
    g->lo[k] = c->aabb_min[k];
    g->span[k] = c->aabb_max[k] - c->aabb_min[k];
  }
  return DASS_OK;
}

}  // namespace dass

using namespace dass;

extern "C" {

const char* dass_status_string(int status) {
  switch (status) {
    case DASS_OK: return "ok";
    case DASS_ERR_INVALID_ARG: return "invalid argument";
    case DASS_ERR_DATA: return "data error";
    case DASS_ERR_NUMERICAL: return "numerical error";
    case DASS_ERR_CAPACITY: return "pair capacity exceeded";
    case DASS_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char* dass_last_error(void) { return t_last_error.c_str(); }

int dass_abi_version(void) { return DASS_ABI_VERSION; }

uint64_t dass_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int dass_apply_shift(int32_t n, const float* pos_opa, const float* rot, const float* mu,
                     const float* sigma, const uint8_t* dyn_mask, float* pos_opa_out,
                     float* rot_out, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!pos_opa || !rot || !mu || !sigma || !pos_opa_out || !rot_out)
    return fail(DASS_ERR_INVALID_ARG, "dass_apply_shift: null required pointer%s");
  if (!aligned16(pos_opa) || !aligned16(rot) || !aligned16(mu) || !aligned16(sigma) ||
      !aligned16(pos_opa_out) || !aligned16(rot_out))
    return fail(DASS_ERR_INVALID_ARG, "dass_apply_shift: float4 arrays must be 16-byte aligned%s");
  return cuda_status(launch_shift(n, (const float4*)pos_opa, (const float4*)rot, (const float4*)mu,
                                  (const float4*)sigma, dyn_mask, (float4*)pos_opa_out,
                                  (float4*)rot_out, (cudaStream_t)stream),
                     "dass_apply_shift");
}

int dass_apply_shift_bwd(int32_t n, const float* rot, const float* sigma, const uint8_t* dyn_mask,
                         const float* g_pos_out, const float* g_rot_out, float* g_mu,
                         float* g_sigma, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0 || (!g_mu && !g_sigma)) return DASS_OK;
  if (!rot || !sigma || !g_pos_out || !g_rot_out)
    return fail(DASS_ERR_INVALID_ARG, "dass_apply_shift_bwd: null required pointer%s");
  return cuda_status(launch_shift_bwd(n, (const float4*)rot, (const float4*)sigma, dyn_mask,
                                      (const float4*)g_pos_out, (const float4*)g_rot_out,
                                      (float4*)g_mu, (float4*)g_sigma, (cudaStream_t)stream),
                     "dass_apply_shift_bwd");
}

static int project_common(int part, const dass_camera* cams, int32_t num_views, int32_t n,
                          int32_t sh_degree, const float* pos_opa, const float* scale, const float* rot,
                          const float* sh, const uint8_t* keep, float* xy_depth, float* conic_opa,
                          float* rgb, uint32_t* box, uint32_t* tile_rows, uint32_t* tiles,
                          void* stream) {
  if (num_views < 1 || num_views > 64)
    return fail(DASS_ERR_INVALID_ARG, "num_views must be in [1, 64]%s");
  for (int v = 0; v < num_views; ++v) {
    int st = check_camera(cams + v);
    if (st) return st;
  }
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (sh_degree < 0 || sh_degree > 3) return fail(DASS_ERR_INVALID_ARG, "sh_degree must be in [0, 3]%s");
  if (part < DASS_PROJECT_KEYS || part > DASS_PROJECT_ALL)
    return fail(DASS_ERR_INVALID_ARG, "dass_project_views_part: part must be 1, 2 or 3%s");
  if (n == 0) return DASS_OK;
  if (!pos_opa || !scale || !rot || !sh || !xy_depth || !conic_opa || !rgb || !box || !tile_rows ||
      !tiles)
    return fail(DASS_ERR_INVALID_ARG, "dass_project: null required pointer%s");
  if (!aligned16(tile_rows)) return fail(DASS_ERR_INVALID_ARG, "dass_project: tile_rows must be 16-byte aligned%s");
  CamParams cp[64];
  for (int v = 0; v < num_views; ++v) cp[v] = to_params(cams + v);
  return cuda_status(launch_project_part(part, cp, num_views, n, sh_degree, (const float4*)pos_opa,
                                         (const float4*)scale, (const float4*)rot,
                                         (const float4*)sh, keep, (float4*)xy_depth,
                                         (float4*)conic_opa, (float4*)rgb, (uint2*)box,
                                         (uint4*)tile_rows, tiles, (cudaStream_t)stream),
                     "dass_project");
}

int dass_project(const dass_camera* cam, int32_t n, int32_t sh_degree, const float* pos_opa,
                 const float* scale, const float* rot, const float* sh, const uint8_t* keep_mask,
                 float* xy_depth, float* conic_opa, float* rgb, uint32_t* box,
                 uint32_t* tile_rows, uint32_t* tiles_touched, void* stream) {
  return project_common(DASS_PROJECT_ALL, cam, 1, n, sh_degree, pos_opa, scale, rot, sh,
                        keep_mask, xy_depth, conic_opa, rgb, box, tile_rows, tiles_touched, stream);
}

int dass_project_views(const dass_camera* cams, int32_t num_views, int32_t n, int32_t sh_degree,
                       const float* pos_opa, const float* scale, const float* rot, const float* sh,
                       const uint8_t* keep_mask, float* xy_depth, float* conic_opa, float* rgb,
                       uint32_t* box, uint32_t* tile_rows, uint32_t* tiles_touched, void* stream) {
  if (cams == nullptr) return fail(DASS_ERR_INVALID_ARG, "cams is null%s");
  return project_common(DASS_PROJECT_ALL, cams, num_views, n, sh_degree, pos_opa, scale, rot, sh,
                        keep_mask, xy_depth, conic_opa, rgb, box, tile_rows, tiles_touched, stream);
}

int dass_project_views_part(int32_t part, const dass_camera* cams, int32_t num_views, int32_t n,
                            int32_t sh_degree, const float* pos_opa, const float* scale,
                            const float* rot, const float* sh, const uint8_t* keep_mask,
                            float* xy_depth, float* conic_opa, float* rgb, uint32_t* box,
                            uint32_t* tile_rows, uint32_t* tiles_touched, void* stream) {
  if (cams == nullptr) return fail(DASS_ERR_INVALID_ARG, "cams is null%s");
  return project_common(part, cams, num_views, n, sh_degree, pos_opa, scale, rot, sh, keep_mask,
                        xy_depth, conic_opa, rgb, box, tile_rows, tiles_touched, stream);
}

int dass_bin_sort_workspace(int32_t n, int32_t num_tiles, int64_t pair_capacity, size_t* bytes) {
  if (!bytes) return fail(DASS_ERR_INVALID_ARG, "bytes is null%s");
  if (n < 0 || n >= (1 << 30) || num_tiles < 1 || pair_capacity < 0 ||
      pair_capacity >= (int64_t(1) << 30))
    return fail(DASS_ERR_INVALID_ARG, "need 0 <= n < 2^30, num_tiles >= 1, 0 <= pair_capacity < 2^30%s");
  *bytes = binsort_workspace(n, num_tiles, pair_capacity);
  return DASS_OK;
}

static int bin_sort_common(int pair_grid, const dass_camera* cam, int32_t n, const float* xy_depth,
                           const uint32_t* box, const uint32_t* tile_rows,
                           const uint32_t* tiles_touched, void* ws, size_t ws_bytes,
                           int64_t pair_capacity, uint64_t* sorted_keys, uint32_t* sorted_ids,
                           uint32_t* tile_ranges, uint32_t* num_pairs_dev,
                           int64_t* num_pairs_host, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  // the onesweep look-back packs counts into 30 bits (binsort.cu)
  if (n < 0 || n >= (1 << 30)) return fail(DASS_ERR_INVALID_ARG, "n must be in [0, 2^30)%s");
  if (pair_capacity < 0 || pair_capacity >= (int64_t(1) << 30))
    return fail(DASS_ERR_INVALID_ARG, "pair_capacity must be in [0, 2^30)%s");
  CamParams cp = to_params(cam);
  const int ntiles = cp.tiles_x * cp.tiles_y;
  if (!tile_ranges || !num_pairs_dev || !sorted_ids)
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort: null required pointer%s");
  if (n > 0 && (!xy_depth || !box || !tile_rows || !tiles_touched))
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort: null record pointer%s");
  const size_t need = binsort_workspace(n, ntiles, pair_capacity);
  if (ws_bytes < need || (need > 0 && ws == nullptr))
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort: workspace too small%s");
  cudaStream_t s = (cudaStream_t)stream;
  st = cuda_status(launch_binsort(cp, n, (const float4*)xy_depth, (const uint2*)box,
                                  (const uint4*)tile_rows, tiles_touched,
                                  ws, pair_capacity, sorted_keys, sorted_ids, (uint2*)tile_ranges,
                                  num_pairs_dev, pair_grid, s),
                   "dass_bin_sort");
  if (st || num_pairs_host == nullptr) return st;
  uint32_t h[2];
  st = cuda_status(cudaMemcpyAsync(h, num_pairs_dev, sizeof(h), cudaMemcpyDeviceToHost, s),
                   "dass_bin_sort: read K");
  if (st) return st;
  st = cuda_status(cudaStreamSynchronize(s), "dass_bin_sort: sync");
  if (st) return st;
  *num_pairs_host = (int64_t)h[0];
  if (h[1]) {
    char buf[128];
    snprintf(buf, sizeof(buf), "K = %u pairs exceed capacity %lld", h[0], (long long)pair_capacity);
    t_last_error = buf;
    return DASS_ERR_CAPACITY;
  }
  return DASS_OK;
}

int dass_bin_sort(const dass_camera* cam, int32_t n, const float* xy_depth, const uint32_t* box,
                  const uint32_t* tile_rows, const uint32_t* tiles_touched, void* ws,
                  size_t ws_bytes, int64_t pair_capacity,
                  uint64_t* sorted_keys, uint32_t* sorted_ids, uint32_t* tile_ranges,
                  uint32_t* num_pairs_dev, int64_t* num_pairs_host, void* stream) {
  return bin_sort_common(0, cam, n, xy_depth, box, tile_rows, tiles_touched, ws, ws_bytes,
                         pair_capacity, sorted_keys, sorted_ids, tile_ranges, num_pairs_dev,
                         num_pairs_host, stream);
}

int dass_bin_sort_shared(const dass_camera* cam, int32_t n, const float* xy_depth,
                         const uint32_t* box, const uint32_t* tile_rows,
                         const uint32_t* tiles_touched, void* ws, size_t ws_bytes,
                         int64_t pair_capacity, uint64_t* sorted_keys, uint32_t* sorted_ids,
                         uint32_t* tile_ranges, uint32_t* num_pairs_dev,
                         int64_t* num_pairs_host, void* stream) {
  return bin_sort_common(BINSORT_SHARED_GRID, cam, n, xy_depth, box, tile_rows, tiles_touched, ws,
                         ws_bytes, pair_capacity, sorted_keys, sorted_ids, tile_ranges,
                         num_pairs_dev, num_pairs_host, stream);
}

int dass_bin_sort_views_workspace(int32_t num_views, int32_t n, int64_t view_capacity,
                                  size_t* bytes) {
  if (!bytes) return fail(DASS_ERR_INVALID_ARG, "bytes is null%s");
  if (num_views < 1 || num_views > 64 || n < 0 || (int64_t)num_views * n >= (int64_t(1) << 30) ||
      view_capacity < 0 || view_capacity >= (int64_t(1) << 30) / num_views)
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views_workspace: bad sizes (V·n and V·capacity must be < 2^30)%s");
  *bytes = binsort_views_workspace(num_views, n, view_capacity);
  return DASS_OK;
}

int dass_bin_sort_views(const dass_camera* cams, int32_t num_views, int32_t n,
                        const float* xy_depth, const uint32_t* box, const uint32_t* tile_rows,
                        const uint32_t* tiles_touched,
                        void* ws, size_t ws_bytes, int64_t view_capacity, uint32_t* sorted_ids,
                        uint32_t* tile_ranges, uint32_t* num_pairs_dev, void* stream) {
  if (!cams) return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: cams is null%s");
  if (num_views < 1 || num_views > 64)
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: num_views must be in [1, 64]%s");
  for (int v = 0; v < num_views; ++v) {
    int st = check_camera(&cams[v]);
    if (st) return st;
    if (cams[v].width != cams[0].width || cams[v].height != cams[0].height)
      return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: cameras differ in size%s");
  }
  if (n < 0 || (int64_t)num_views * n >= (int64_t(1) << 30))
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: need 0 <= V·n < 2^30%s");
  if (view_capacity < 0 || view_capacity >= (int64_t(1) << 30) / num_views)
    return fail(DASS_ERR_INVALID_ARG, "view_capacity must be in [0, 2^30 / V)%s");
  if (!sorted_ids || !tile_ranges || !num_pairs_dev)
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: null required pointer%s");
  if (n > 0 && (!xy_depth || !box || !tile_rows || !tiles_touched))
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: null record pointer%s");
  const size_t need = binsort_views_workspace(num_views, n, view_capacity);
  if (ws_bytes < need || (need > 0 && ws == nullptr))
    return fail(DASS_ERR_INVALID_ARG, "dass_bin_sort_views: workspace too small%s");
  CamParams cp = to_params(&cams[0]);
  return cuda_status(launch_binsort_views(cp, num_views, n, (const float4*)xy_depth,
                                          (const uint2*)box, (const uint4*)tile_rows, tiles_touched, ws, view_capacity,
                                          sorted_ids, (uint2*)tile_ranges, num_pairs_dev,
                                          (cudaStream_t)stream),
                     "dass_bin_sort_views");
}

int dass_render_accept_workspace(int32_t num_tiles, int64_t pair_capacity, size_t* bytes) {
  if (!bytes || num_tiles < 1 || pair_capacity < 0 || pair_capacity >= (int64_t(1) << 30))
    return fail(DASS_ERR_INVALID_ARG, "need num_tiles >= 1 and 0 <= pair_capacity < 2^30%s");
  *bytes = render_accept_workspace(num_tiles, pair_capacity);
  return DASS_OK;
}

// Acceptance-list buffer (A38): 16-byte aligned, at least the workspace the
// image's tile count and pair_capacity need, pair_capacity ∈ [0, 2^30).
static int check_accept(const CamParams& cp, const void* accept, size_t accept_bytes,
                        int64_t pair_capacity, const char* where) {
  if (accept == nullptr) return DASS_OK;
  char buf[192];
  if (pair_capacity < 0 || pair_capacity >= (int64_t(1) << 30) || !aligned16(accept)) {
    snprintf(buf, sizeof(buf), "%s: accept needs a 16-byte aligned buffer and 0 <= pair_capacity < 2^30", where);
    t_last_error = buf;
    return DASS_ERR_INVALID_ARG;
  }
  const size_t need = render_accept_workspace(cp.tiles_x * cp.tiles_y, pair_capacity);
  if (accept_bytes < need) {
    snprintf(buf, sizeof(buf), "%s: accept buffer of %zu bytes < %zu needed", where, accept_bytes, need);
    t_last_error = buf;
    return DASS_ERR_INVALID_ARG;
  }
  return DASS_OK;
}

static int tile_subset(const dass_camera* cam, int32_t tile_begin, int32_t tile_stride,
                       int32_t tile_count, CamParams* cp) {
  const int nt = cp->tiles_x * cp->tiles_y;
  if (tile_count < 0) { cp->tile0 = 0; cp->tstride = 1; cp->tcount = nt; return DASS_OK; }
  if (tile_stride < 1 || tile_begin < 0 ||
      (tile_count > 0 && (int64_t)tile_begin + (int64_t)(tile_count - 1) * tile_stride >= nt))
    return fail(DASS_ERR_INVALID_ARG, "tile subset outside the image's tiles%s");
  cp->tile0 = tile_begin; cp->tstride = tile_stride; cp->tcount = tile_count;
  (void)cam;
  return DASS_OK;
}

int dass_render_fwd_tiles(const dass_camera* cam, int32_t tile_begin, int32_t tile_stride,
                          int32_t tile_count, const uint32_t* tile_ranges,
                          const uint32_t* sorted_ids, const float* xy_depth,
                          const float* conic_opa, const float* rgb, const uint32_t* box,
                          const float* bg, float* out_img, float* out_T, uint32_t* out_last,
                          void* accept, size_t accept_bytes, int64_t pair_capacity, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (!tile_ranges || !out_img || !out_T || !out_last)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_fwd: null required pointer%s");
  if (!sorted_ids || !xy_depth || !conic_opa || !rgb || !box)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_fwd: null record pointer%s");
  CamParams cp = to_params(cam);
  if ((st = check_accept(cp, accept, accept_bytes, pair_capacity, "dass_render_fwd"))) return st;
  if ((st = tile_subset(cam, tile_begin, tile_stride, tile_count, &cp))) return st;
  if (cp.tcount == 0) return DASS_OK;
  float3 b = bg ? make_float3(bg[0], bg[1], bg[2]) : make_float3(0.f, 0.f, 0.f);
  return cuda_status(launch_render_fwd(cp, (const uint2*)tile_ranges, sorted_ids,
                                       (const float4*)xy_depth, (const float4*)conic_opa,
                                       (const float4*)rgb, (const uint2*)box, b, out_img, out_T,
                                       out_last, accept, pair_capacity, (cudaStream_t)stream),
                     "dass_render_fwd");
}

int dass_render_fwd(const dass_camera* cam, const uint32_t* tile_ranges, const uint32_t* sorted_ids,
                    const float* xy_depth, const float* conic_opa, const float* rgb,
                    const uint32_t* box, const float* bg, float* out_img, float* out_T,
                    uint32_t* out_last, void* accept, size_t accept_bytes, int64_t pair_capacity,
                    void* stream) {
  return dass_render_fwd_tiles(cam, 0, 1, -1, tile_ranges, sorted_ids, xy_depth, conic_opa, rgb,
                               box, bg, out_img, out_T, out_last, accept, accept_bytes,
                               pair_capacity, stream);
}

int dass_render_bwd_workspace(int32_t n, size_t* bytes) {
  if (!bytes || n < 0) return fail(DASS_ERR_INVALID_ARG, "bad arguments%s");
  *bytes = render_bwd_workspace(n);
  return DASS_OK;
}

int dass_render_bwd(const dass_camera* cam, int32_t n, int32_t sh_degree, const float* pos_opa,
                    const float* scale, const float* rot, const float* sh,
                    const uint8_t* keep_mask, const uint32_t* tile_ranges,
                    const uint32_t* sorted_ids, const float* xy_depth, const float* conic_opa,
                    const float* rgb, const uint32_t* box, const float* bg, const float* out_T,
                    const uint32_t* out_last, const float* dL_dimg, const void* accept,
                    size_t accept_bytes, int64_t pair_capacity, void* ws, size_t ws_bytes,
                    float* g_pos_opa, float* g_scale, float* g_rot, float* g_sh,
                    float* gradstat_sum, uint32_t* gradstat_cnt, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (sh_degree < 0 || sh_degree > 3) return fail(DASS_ERR_INVALID_ARG, "sh_degree must be in [0, 3]%s");
  if (n == 0) return DASS_OK;
  if (!pos_opa || !scale || !rot || !sh || !tile_ranges || !sorted_ids || !xy_depth || !conic_opa ||
      !rgb || !box || !out_T || !out_last || !dL_dimg)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd: null required pointer%s");
  if (ws_bytes < render_bwd_workspace(n) || !ws)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd: workspace too small%s");
  if (!aligned16(ws)) return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd: workspace must be 16-byte aligned%s");
  CamParams cp = to_params(cam);
  if ((st = check_accept(cp, accept, accept_bytes, pair_capacity, "dass_render_bwd"))) return st;
  float3 b = bg ? make_float3(bg[0], bg[1], bg[2]) : make_float3(0.f, 0.f, 0.f);
  return cuda_status(
      launch_render_bwd(cp, n, sh_degree, (const float4*)pos_opa, (const float4*)scale,
                        (const float4*)rot, (const float4*)sh, keep_mask,
                        (const uint2*)tile_ranges, sorted_ids, (const float4*)xy_depth,
                        (const float4*)conic_opa, (const float4*)rgb, (const uint2*)box, b, out_T,
                        out_last, dL_dimg, accept, pair_capacity, ws, (float4*)g_pos_opa, (float4*)g_scale,
                        (float4*)g_rot, (float4*)g_sh, gradstat_sum, gradstat_cnt,
                        (cudaStream_t)stream),
      "dass_render_bwd");
}

int dass_render_bwd_raster_tiles(const dass_camera* cam, int32_t tile_begin, int32_t tile_stride,
                                 int32_t tile_count, int32_t n, const uint32_t* tile_ranges,
                                 const uint32_t* sorted_ids, const float* xy_depth,
                                 const float* conic_opa, const float* rgb, const uint32_t* box,
                                 const float* bg, const float* out_T, const uint32_t* out_last,
                                 const float* dL_dimg, const void* accept, size_t accept_bytes,
                                 int64_t pair_capacity, float* g2d, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!tile_ranges || !sorted_ids || !xy_depth || !conic_opa || !rgb || !box || !out_T ||
      !out_last || !dL_dimg || !g2d)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd_raster: null required pointer%s");
  if (!aligned16(g2d)) return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd_raster: g2d must be 16-byte aligned%s");
  CamParams cp = to_params(cam);
  if ((st = check_accept(cp, accept, accept_bytes, pair_capacity, "dass_render_bwd_raster"))) return st;
  if ((st = tile_subset(cam, tile_begin, tile_stride, tile_count, &cp))) return st;
  float3 b = bg ? make_float3(bg[0], bg[1], bg[2]) : make_float3(0.f, 0.f, 0.f);
  return cuda_status(launch_render_bwd_raster(cp, n, (const uint2*)tile_ranges, sorted_ids,
                                              (const float4*)xy_depth, (const float4*)conic_opa,
                                              (const float4*)rgb, (const uint2*)box, b, out_T,
                                              out_last, dL_dimg, accept, pair_capacity,
                                              (float4*)g2d, (cudaStream_t)stream),
                     "dass_render_bwd_raster");
}

int dass_render_bwd_raster(const dass_camera* cam, int32_t n, const uint32_t* tile_ranges,
                           const uint32_t* sorted_ids, const float* xy_depth,
                           const float* conic_opa, const float* rgb, const uint32_t* box,
                           const float* bg, const float* out_T, const uint32_t* out_last,
                           const float* dL_dimg, const void* accept, size_t accept_bytes,
                           int64_t pair_capacity, float* g2d, void* stream) {
  return dass_render_bwd_raster_tiles(cam, 0, 1, -1, n, tile_ranges, sorted_ids, xy_depth,
                                      conic_opa, rgb, box, bg, out_T, out_last, dL_dimg, accept,
                                      accept_bytes, pair_capacity, g2d, stream);
}

int dass_render_bwd_preprocess_views_part(int32_t part, const dass_camera* cams, int32_t num_views,
                                          int32_t n, int32_t sh_degree, const float* pos_opa,
                                          const float* scale, const float* rot, const float* sh,
                                          const uint8_t* keep_mask, const float* conic_opa,
                                          const float* rgb, const uint32_t* box, const float* g2d,
                                          float* g_pos_opa, float* g_scale, float* g_rot,
                                          float* g_sh, float* gradstat_sum,
                                          uint32_t* gradstat_cnt, float* const* uv_out,
                                          const uint8_t* uv_count, void* stream) {
  if (part < DASS_PREPROCESS_GEOMETRY || part > DASS_PREPROCESS_ALL)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd_preprocess_views_part: part must be 1, 2 or 3%s");
  if (cams == nullptr) return fail(DASS_ERR_INVALID_ARG, "cams is null%s");
  if (num_views < 1 || num_views > 64) return fail(DASS_ERR_INVALID_ARG, "num_views must be in [1, 64]%s");
  for (int v = 0; v < num_views; ++v) {
    int st = check_camera(cams + v);
    if (st) return st;
  }
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (sh_degree < 0 || sh_degree > 3) return fail(DASS_ERR_INVALID_ARG, "sh_degree must be in [0, 3]%s");
  if (n == 0) return DASS_OK;
  if (!pos_opa || !scale || !rot || !sh || !conic_opa || !rgb || !box || !g2d)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd_preprocess_views: null required pointer%s");
  if (uv_out)
    for (int v = 0; v < num_views; ++v)
      if (uv_out[v] && ((uintptr_t)uv_out[v] & 7u))
        return fail(DASS_ERR_INVALID_ARG, "dass_render_bwd_preprocess_views: uv_out must be 8-byte aligned%s");
  CamParams cp[64];
  for (int v = 0; v < num_views; ++v) cp[v] = to_params(cams + v);
  return cuda_status(launch_preprocess_views(cp, num_views, n, sh_degree, (const float4*)pos_opa,
                                             (const float4*)scale, (const float4*)rot,
                                             (const float4*)sh, keep_mask,
                                             (const float4*)conic_opa, (const float4*)rgb,
                                             (const uint2*)box, (const float4*)g2d,
                                             (float4*)g_pos_opa, (float4*)g_scale,
                                             (float4*)g_rot, (float4*)g_sh, gradstat_sum,
                                             gradstat_cnt,
                                             reinterpret_cast<float2* const*>(uv_out), uv_count,
                                             part, (cudaStream_t)stream),
                     "dass_render_bwd_preprocess_views");
}

int dass_render_bwd_preprocess_views_uv(const dass_camera* cams, int32_t num_views, int32_t n,
                                        int32_t sh_degree, const float* pos_opa,
                                        const float* scale, const float* rot, const float* sh,
                                        const uint8_t* keep_mask, const float* conic_opa,
                                        const float* rgb, const uint32_t* box, const float* g2d,
                                        float* g_pos_opa, float* g_scale, float* g_rot,
                                        float* g_sh, float* gradstat_sum,
                                        uint32_t* gradstat_cnt, float* const* uv_out,
                                        const uint8_t* uv_count, void* stream) {
  return dass_render_bwd_preprocess_views_part(DASS_PREPROCESS_ALL, cams, num_views, n, sh_degree,
                                               pos_opa, scale, rot, sh, keep_mask, conic_opa, rgb,
                                               box, g2d, g_pos_opa, g_scale, g_rot, g_sh,
                                               gradstat_sum, gradstat_cnt, uv_out, uv_count, stream);
}

int dass_render_bwd_preprocess_views(const dass_camera* cams, int32_t num_views, int32_t n,
                                     int32_t sh_degree, const float* pos_opa,
                                     const float* scale, const float* rot, const float* sh,
                                     const uint8_t* keep_mask, const float* conic_opa,
                                     const float* rgb, const uint32_t* box, const float* g2d,
                                     float* g_pos_opa, float* g_scale, float* g_rot,
                                     float* g_sh, float* gradstat_sum,
                                     uint32_t* gradstat_cnt, void* stream) {
  return dass_render_bwd_preprocess_views_uv(cams, num_views, n, sh_degree, pos_opa, scale, rot,
                                             sh, keep_mask, conic_opa, rgb, box, g2d, g_pos_opa,
                                             g_scale, g_rot, g_sh, gradstat_sum, gradstat_cnt,
                                             nullptr, nullptr, stream);
}

int dass_gradstat_from_uv(int32_t n, int32_t num_split, const float* uv, float* gradstat_sum,
                          void* stream) {
  if (n < 0 || num_split < 0) return fail(DASS_ERR_INVALID_ARG, "n and num_split must be >= 0%s");
  if (n == 0 || num_split == 0) return DASS_OK;
  if (!uv || ((uintptr_t)uv & 7u) || !gradstat_sum)
    return fail(DASS_ERR_INVALID_ARG, "dass_gradstat_from_uv: null or misaligned pointer%s");
  return cuda_status(launch_gradstat_uv(n, num_split, (const float2*)uv, gradstat_sum,
                                        (cudaStream_t)stream),
                     "dass_gradstat_from_uv");
}

int dass_fidelity_loss_workspace(int32_t width, int32_t height, size_t* bytes) {
  if (!bytes || width < 1 || height < 1 || width > 65535 || height > 65535)
    return fail(DASS_ERR_INVALID_ARG, "width/height must be in [1, 65535]%s");
  *bytes = fidelity_loss_workspace(width, height);
  return DASS_OK;
}

int dass_fidelity_loss(int32_t width, int32_t height, const float* img, const float* gt,
                       float lambda, float dssim_scale, void* ws, size_t ws_bytes, float* loss,
                       float* dL_dimg, void* stream) {
  if (width < 1 || height < 1 || width > 65535 || height > 65535)
    return fail(DASS_ERR_INVALID_ARG, "width/height must be in [1, 65535]%s");
  if (!(lambda >= 0.f && lambda <= 1.f)) return fail(DASS_ERR_INVALID_ARG, "lambda must be in [0, 1]%s");
  if (!(dssim_scale > 0.f && dssim_scale <= 1.f))
    return fail(DASS_ERR_INVALID_ARG, "dssim_scale must be in (0, 1]%s");
  if (!img || !gt || !loss) return fail(DASS_ERR_INVALID_ARG, "dass_fidelity_loss: null required pointer%s");
  if (!ws || ws_bytes < fidelity_loss_workspace(width, height) || ((uintptr_t)ws & 15u))
    return fail(DASS_ERR_INVALID_ARG, "dass_fidelity_loss: workspace too small or unaligned%s");
  return cuda_status(launch_fidelity_loss(width, height, img, gt, lambda, dssim_scale, ws, loss,
                                          dL_dimg, (cudaStream_t)stream),
                     "dass_fidelity_loss");
}

int dass_inherit_mask(int32_t n, const float* m, uint8_t* keep, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!m || !keep) return fail(DASS_ERR_INVALID_ARG, "dass_inherit_mask: null required pointer%s");
  return cuda_status(launch_inherit_mask(n, m, keep, (cudaStream_t)stream), "dass_inherit_mask");
}

int dass_inherit_mask_bwd(int32_t n, const float* m, const float* pos_opa, const float* scale,
                          const float* g_pos_opa, const float* g_scale, float lambda_inher,
                          float* g_m, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!m || !pos_opa || !scale || !g_pos_opa || !g_scale || !g_m)
    return fail(DASS_ERR_INVALID_ARG, "dass_inherit_mask_bwd: null required pointer%s");
  if (!std::isfinite(lambda_inher)) return fail(DASS_ERR_INVALID_ARG, "lambda_inher must be finite%s");
  return cuda_status(launch_inherit_mask_bwd(n, m, (const float4*)pos_opa, (const float4*)scale,
                                             (const float4*)g_pos_opa, (const float4*)g_scale,
                                             lambda_inher, g_m, (cudaStream_t)stream),
                     "dass_inherit_mask_bwd");
}

int dass_deform_param_count(const dass_hashgrid* cfg, int64_t* table_floats, int64_t* mlp_floats) {
  HashGridParams g;
  const int st = to_hashgrid(cfg, &g);
  if (st) return st;
  const int64_t H = DASS_MLP_HIDDEN;
  if (table_floats) *table_floats = (int64_t)g.L * g.T * g.F;
  if (mlp_floats) *mlp_floats = H * g.in + H + H * H + H + 7 * H + 7;
  return DASS_OK;
}

static int check_table_align(const HashGridParams& g, const void* p) {
  const uintptr_t a = (uintptr_t)p;
  if ((g.F == 4 && (a & 15u)) || (g.F == 2 && (a & 7u)) || (a & 3u))
    return fail(DASS_ERR_INVALID_ARG, "table pointer misaligned for its feature width%s");
  return DASS_OK;
}

int dass_deform_fwd(const dass_hashgrid* cfg, const float* table, const float* mlp, int32_t n,
                    const int32_t* idx, const int32_t* count, const float* pos_opa, float* mu,
                    float* sigma, void* stream) {
  HashGridParams g;
  int st = to_hashgrid(cfg, &g);
  if (st) return st;
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!table || !mlp || !pos_opa || !mu || !sigma)
    return fail(DASS_ERR_INVALID_ARG, "dass_deform_fwd: null required pointer%s");
  if ((st = check_table_align(g, table))) return st;
  if (!aligned16(pos_opa) || !aligned16(mu) || !aligned16(sigma))
    return fail(DASS_ERR_INVALID_ARG, "dass_deform_fwd: float4 arrays must be 16-byte aligned%s");
  return cuda_status(launch_deform_fwd(g, table, mlp, n, idx, count, (const float4*)pos_opa,
                                       (float4*)mu, (float4*)sigma, (cudaStream_t)stream),
                     "dass_deform_fwd");
}

int dass_deform_bwd(const dass_hashgrid* cfg, const float* table, const float* mlp, int32_t n,
                    const int32_t* idx, const int32_t* count, const float* pos_opa,
                    const float* g_mu, const float* g_sigma, float* g_table, float* g_mlp,
                    void* stream) {
  HashGridParams g;
  int st = to_hashgrid(cfg, &g);
  if (st) return st;
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (n == 0) return DASS_OK;
  if (!table || !mlp || !pos_opa || !g_mu || !g_sigma || !g_table || !g_mlp)
    return fail(DASS_ERR_INVALID_ARG, "dass_deform_bwd: null required pointer%s");
  if ((st = check_table_align(g, table)) || (st = check_table_align(g, g_table))) return st;
  if (!aligned16(pos_opa) || !aligned16(g_mu) || !aligned16(g_sigma))
    return fail(DASS_ERR_INVALID_ARG, "dass_deform_bwd: float4 arrays must be 16-byte aligned%s");
  return cuda_status(launch_deform_bwd(g, table, mlp, n, idx, count, (const float4*)pos_opa,
                                       (const float4*)g_mu, (const float4*)g_sigma, g_table,
                                       g_mlp, (cudaStream_t)stream),
                     "dass_deform_bwd");
}

int dass_partition_workspace(int32_t n, size_t* bytes) {
  if (n < 0 || !bytes) return fail(DASS_ERR_INVALID_ARG, "n < 0 or bytes is null%s");
  *bytes = partition_workspace(n);
  return DASS_OK;
}

int dass_partition(int32_t n, const uint8_t* mask, int32_t* idx_dyn, int32_t* idx_st,
                   int32_t* counts, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if (!mask && n > 0) return fail(DASS_ERR_INVALID_ARG, "dass_partition: mask is null%s");
  if (!idx_dyn || !idx_st || !counts)
    return fail(DASS_ERR_INVALID_ARG, "dass_partition: null required pointer%s");
  if (!ws || ws_bytes < partition_workspace(n) || ((uintptr_t)ws & 3u))
    return fail(DASS_ERR_INVALID_ARG, "dass_partition: workspace too small or misaligned%s");
  return cuda_status(launch_partition(n, mask, idx_dyn, idx_st, counts, ws, (cudaStream_t)stream),
                     "dass_partition");
}

static int sh_k4(int deg) { return (3 * (deg + 1) * (deg + 1) + 3) / 4; }

int dass_densify_select(int32_t n, const float* gradstat_sum, const uint32_t* gradstat_cnt,
                        const uint8_t* s_err, float tau_pos, float tau_err, uint8_t* in_S,
                        int32_t* idx, int32_t* counts, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if ((n > 0 && (!gradstat_sum || !gradstat_cnt || !in_S || !idx)) || !counts)
    return fail(DASS_ERR_INVALID_ARG, "dass_densify_select: null required pointer%s");
  if (!std::isfinite(tau_pos) || !std::isfinite(tau_err))
    return fail(DASS_ERR_INVALID_ARG, "dass_densify_select: thresholds must be finite%s");
  if (!ws || ws_bytes < partition_workspace(n) || ((uintptr_t)ws & 3u))
    return fail(DASS_ERR_INVALID_ARG, "dass_densify_select: workspace too small or misaligned%s");
  return cuda_status(launch_densify_select(n, gradstat_sum, gradstat_cnt, s_err, tau_pos, tau_err,
                                           in_S, idx, counts, ws, (cudaStream_t)stream),
                     "dass_densify_select");
}

int dass_prune_select(int32_t n, int32_t first, const float* pos_opa, float min_opacity,
                      uint8_t* keep, int32_t* idx, int32_t* counts, void* ws, size_t ws_bytes,
                      void* stream) {
  if (n < 0) return fail(DASS_ERR_INVALID_ARG, "n < 0%s");
  if ((n > 0 && (!pos_opa || !keep || !idx)) || !counts)
    return fail(DASS_ERR_INVALID_ARG, "dass_prune_select: null required pointer%s");
  if (pos_opa && !aligned16(pos_opa))
    return fail(DASS_ERR_INVALID_ARG, "dass_prune_select: pos_opa must be 16-byte aligned%s");
  if (!std::isfinite(min_opacity)) return fail(DASS_ERR_INVALID_ARG, "min_opacity must be finite%s");
  if (!ws || ws_bytes < partition_workspace(n) || ((uintptr_t)ws & 3u))
    return fail(DASS_ERR_INVALID_ARG, "dass_prune_select: workspace too small or misaligned%s");
  return cuda_status(launch_prune_select(n, first, (const float4*)pos_opa, min_opacity, keep, idx,
                                         counts, ws, (cudaStream_t)stream),
                     "dass_prune_select");
}

static int check_rows(const char* where, const float* a, const float* b, const float* c,
                      const float* d) {
  if (!a || !b || !c || !d) return fail(DASS_ERR_INVALID_ARG, "%s: null required pointer", where);
  if (!aligned16(a) || !aligned16(b) || !aligned16(c) || !aligned16(d))
    return fail(DASS_ERR_INVALID_ARG, "%s: float4 arrays must be 16-byte aligned", where);
  return DASS_OK;
}

int dass_gather(int32_t n, int32_t sh_degree, const float* pos_opa, const float* scale,
                const float* rot, const float* sh, const uint8_t* dyn, int32_t m,
                const int32_t* idx, float* out_pos_opa, float* out_scale, float* out_rot,
                float* out_sh, uint8_t* out_dyn, void* stream) {
  if (n < 0 || m < 0 || m > n) return fail(DASS_ERR_INVALID_ARG, "dass_gather: need 0 <= m <= n%s");
  if (sh_degree < 0 || sh_degree > 3) return fail(DASS_ERR_INVALID_ARG, "sh_degree must be in [0, 3]%s");
  if (m == 0) return DASS_OK;
  int st;
  if ((st = check_rows("dass_gather", pos_opa, scale, rot, sh)) ||
      (st = check_rows("dass_gather", out_pos_opa, out_scale, out_rot, out_sh)))
    return st;
  if (!idx) return fail(DASS_ERR_INVALID_ARG, "dass_gather: idx is null%s");
  return cuda_status(launch_gather(n, sh_k4(sh_degree), (const float4*)pos_opa, (const float4*)scale,
                                   (const float4*)rot, (const float4*)sh, dyn, m, idx, m, 0,
                                   (float4*)out_pos_opa, (float4*)out_scale, (float4*)out_rot,
                                   (float4*)out_sh, out_dyn, (cudaStream_t)stream),
                     "dass_gather");
}

int dass_spawn(int32_t n, int32_t sh_degree, const float* pos_opa, const float* scale,
               const float* rot, const float* sh, const uint8_t* dyn, int32_t m,
               const int32_t* idx, int32_t spawn_count, float scale_shrink, float child_opacity,
               uint64_t seed, float* out_pos_opa, float* out_scale, float* out_rot, float* out_sh,
               uint8_t* out_dyn, void* stream) {
  if (n < 0 || m < 0) return fail(DASS_ERR_INVALID_ARG, "dass_spawn: n, m must be >= 0%s");
  if (sh_degree < 0 || sh_degree > 3) return fail(DASS_ERR_INVALID_ARG, "sh_degree must be in [0, 3]%s");
  if (spawn_count < 1 || !(scale_shrink > 0.f) || !std::isfinite(child_opacity))
    return fail(DASS_ERR_INVALID_ARG, "dass_spawn: need spawn_count >= 1, scale_shrink > 0, finite opacity%s");
  const int64_t n_out = (int64_t)n + (int64_t)m * spawn_count;
  if (n_out > INT32_MAX) return fail(DASS_ERR_INVALID_ARG, "dass_spawn: n + m*K overflows int32%s");
  if (n_out == 0) return DASS_OK;
  int st;
  if ((st = check_rows("dass_spawn", out_pos_opa, out_scale, out_rot, out_sh))) return st;
  if (n > 0 && (st = check_rows("dass_spawn", pos_opa, scale, rot, sh))) return st;
  if (m > 0 && !idx) return fail(DASS_ERR_INVALID_ARG, "dass_spawn: idx is null%s");
  if ((dyn == nullptr) != (out_dyn == nullptr))
    return fail(DASS_ERR_INVALID_ARG, "dass_spawn: dyn and out_dyn must both be given or both null%s");
  const int k4 = sh_k4(sh_degree);
  cudaError_t e = launch_gather(n, k4, (const float4*)pos_opa, (const float4*)scale,
                                (const float4*)rot, (const float4*)sh, dyn, n, nullptr, (int)n_out,
                                0, (float4*)out_pos_opa, (float4*)out_scale, (float4*)out_rot,
                                (float4*)out_sh, out_dyn, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_status(e, "dass_spawn");
  return cuda_status(launch_spawn_children(n, k4, (const float4*)pos_opa, (const float4*)scale,
                                           (const float4*)rot, (const float4*)sh, dyn, m, idx,
                                           spawn_count, scale_shrink, child_opacity, seed,
                                           (int)n_out, n, (float4*)out_pos_opa,
                                           (float4*)out_scale, (float4*)out_rot, (float4*)out_sh,
                                           out_dyn, (cudaStream_t)stream),
                     "dass_spawn");
}

int dass_render_features(const dass_camera* cam, const uint32_t* tile_ranges,
                         const uint32_t* sorted_ids, const float* xy_depth, const float* conic_opa,
                         const uint32_t* box, int32_t channels, const float* feat, float* out,
                         void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (channels != 4 && channels != 8 && channels != 12 && channels != 16)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_features: channels must be 4, 8, 12 or 16%s");
  if (!tile_ranges || !sorted_ids || !xy_depth || !conic_opa || !box || !feat || !out)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_features: null required pointer%s");
  if (!aligned16(feat)) return fail(DASS_ERR_INVALID_ARG, "dass_render_features: feat must be 16-byte aligned%s");
  CamParams cp = to_params(cam);
  return cuda_status(launch_render_features(cp, (const uint2*)tile_ranges, sorted_ids,
                                            (const float4*)xy_depth, (const float4*)conic_opa,
                                            (const uint2*)box, channels, feat, out,
                                            (cudaStream_t)stream),
                     "dass_render_features");
}

int dass_error_map(const dass_camera* cam, const float* rendered, const float* gt, float gamma_err,
                   float* err, uint32_t* dmask, int32_t n_base, const float* pos_opa,
                   uint8_t* s_err, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (!(gamma_err > 0.0f)) return fail(DASS_ERR_INVALID_ARG, "gamma_err must be > 0 (S:619)%s");
  if (n_base < 0) return fail(DASS_ERR_INVALID_ARG, "n_base < 0%s");
  if (!rendered || !gt) return fail(DASS_ERR_DATA, "dass_error_map: rendered and gt are required%s");
  if (s_err && n_base > 0 && !pos_opa)
    return fail(DASS_ERR_INVALID_ARG, "dass_error_map: s_err needs pos_opa%s");
  CamParams cp = to_params(cam);
  return cuda_status(launch_error_map(cp, rendered, gt, gamma_err, err, dmask, s_err ? n_base : 0,
                                      (const float4*)pos_opa, s_err, (cudaStream_t)stream),
                     "dass_error_map");
}

int dass_render_stats(const dass_camera* cam, const uint32_t* tile_ranges,
                      const uint32_t* sorted_ids, const float* xy_depth, const float* conic_opa,
                      const uint32_t* box, const float* out_T, const uint32_t* out_last,
                      uint64_t* counters, void* stream) {
  int st = check_camera(cam);
  if (st) return st;
  if (!tile_ranges || !sorted_ids || !xy_depth || !conic_opa || !box || !out_T || !out_last ||
      !counters)
    return fail(DASS_ERR_INVALID_ARG, "dass_render_stats: null required pointer%s");
  CamParams cp = to_params(cam);
  return cuda_status(launch_render_stats(cp, (const uint2*)tile_ranges, sorted_ids,
                                         (const float4*)xy_depth, (const float4*)conic_opa,
                                         (const uint2*)box, out_T, out_last,
                                         (unsigned long long*)counters, (cudaStream_t)stream),
                     "dass_render_stats");
}

int dass_timestamp(uint64_t* stamps, int32_t slot, void* stream) {
  if (!stamps || slot < 0) return fail(DASS_ERR_INVALID_ARG, "dass_timestamp: null stamps or slot < 0%s");
  return cuda_status(launch_timestamp(stamps + slot, (cudaStream_t)stream), "dass_timestamp");
}

int dass_scan_nonfinite(const float* data, int64_t count, uint32_t* bad_dev, int64_t* bad_host,
                        void* stream) {
  if (count < 0) return fail(DASS_ERR_INVALID_ARG, "dass_scan_nonfinite: count < 0%s");
  if (!bad_dev || (count > 0 && !data))
    return fail(DASS_ERR_INVALID_ARG, "dass_scan_nonfinite: null pointer%s");
  cudaStream_t s = (cudaStream_t)stream;
  int st = cuda_status(launch_nonfinite(data, (long long)count, bad_dev, s), "dass_scan_nonfinite");
  if (st || bad_host == nullptr) return st;
  uint32_t h = 0;
  st = cuda_status(cudaMemcpyAsync(&h, bad_dev, sizeof(h), cudaMemcpyDeviceToHost, s),
                   "dass_scan_nonfinite: read count");
  if (st) return st;
  st = cuda_status(cudaStreamSynchronize(s), "dass_scan_nonfinite: sync");
  if (st) return st;
  *bad_host = (int64_t)h;
  if (h) {
    char buf[96];
    snprintf(buf, sizeof(buf), "%u non-finite values", h);
    t_last_error = buf;
    return DASS_ERR_NUMERICAL;
  }
  return DASS_OK;
}

}  // extern "C"
