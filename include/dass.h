/*
 * dass.h — C-ABI of libdass.so, the B200 (sm_100a) hot path of DASS
 * (arXiv 2411.14847): the per-timestep tile-based differentiable 3D Gaussian
 * Splatting rasterizer every DASS stage optimises through, the masked
 * per-Gaussian shift, and the error map of error-guided densification.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (with its section/eq.);
 * "S:n" = SPEC.md line n; "A.." = a reading listed in DESIGN.md §Readings
 * (SURVEY.md §8(c) table).  Paper passages defining the operations:
 *   Eq. 5-8  (supplement §A.1): Gaussian, Σ = R S Sᵀ Rᵀ, EWA
 *            Σ_2D = J W Σ Wᵀ Jᵀ, front-to-back blending C = Σ c_i α_i Π(1-α_j).
 *   §3.3: shift p' = p + μ, q' = norm(q) × norm(σ).
 *   §3.4 + Alg. 1: error maps E^c, D_err^c,
 *            S_err; historical view-space positional gradient ∇p̄.
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every export
 * ---------------------------------------------------------------------------
 *  - Every pointer argument named *_dev / every array argument is a DEVICE
 *    pointer owned by the caller (normally a torch tensor's data_ptr()),
 *    16-byte aligned where the element is float4.  `const dass_camera*` and
 *    `const float bg[3]` are HOST pointers read during the call.
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it
 *    asynchronously.  Only dass_bin_sort in "host mode" synchronises.
 *  - The library never allocates device memory, keeps no mutable global
 *    state except a relaxed atomic launch counter (dass_kernel_launches) and
 *    a thread-local last-error string; calls on distinct streams are
 *    thread-safe.  Scratch memory is a caller-provided workspace whose size
 *    the matching *_workspace query returns.
 *  - Per-pixel outputs are OVERWRITTEN.  Per-Gaussian gradients and
 *    statistics are ACCUMULATED (+=): the caller zeroes them once per step so
 *    multi-view sums on one GPU cost nothing (A28).
 *  - Return value: a dass_status.  On error nothing has been enqueued (argument
 *    validation happens before any launch) unless the status is DASS_ERR_CUDA.
 *
 * Data layout in HBM (field-SoA of 16-byte records; one coalesced 128-bit load
 * per field per thread):
 *  Gaussian parameters, N = n:
 *    pos_opa  float4[N]   x, y, z (world), opacity o ∈ (0,1) (activated, A16)
 *    scale    float4[N]   sx, sy, sz > 0 (activated), w ignored
 *    rot      float4[N]   quaternion w, x, y, z (real first, raw, A15)
 *    sh       float4[K4][N]  coefficient PLANES: the 3·(d+1)² SH coefficients
 *             of Gaussian i, ordered coefficient-major/channel-minor
 *             (c[k*3+ch]), are split into K4 = ceil(3(d+1)²/4) float4 chunks;
 *             chunk j of every Gaussian forms plane j (sh[j*N + i]).  Padding
 *             floats are ignored on input and written 0 in gradients.
 *    Gradients use the identical layout (g_pos_opa.w = dL/do).
 *  Per-view projected records (outputs of dass_project):
 *    xy_depth  float4[N]  u, v (pixels), z (camera-frame depth), 0
 *    conic_opa float4[N]  A, β, γ, o_eff: the inverse 2D covariance
 *                         K = [[A, B], [B, C]] in Cholesky form, B = A·β,
 *                         C = γ + A·β² (β = −Σ'_xy/Σ'_yy, γ = 1/Σ'_yy, from
 *                         the fp64 Σ', rounded once), so the per-pixel power
 *                         −½(A dx² + 2B dx dy + C dy²) = −[(s dx + sβ dy)² +
 *                         (g dy)²], s = √(A/2), g = √(γ/2), is minus a sum of
 *                         squares (no cancellation for elongated splats)
 *    rgb       float4[N]  r, g, b (clamped ≥ 0), clamp bits (float 0..7,
 *                         bit ch set when channel ch was clamped)
 *    box       uint32[2N] per Gaussian {x0 | x1<<16, y0 | y1<<16}; a culled
 *                         Gaussian has x0 = 1 > x1 = 0 (and y likewise)
 *    tiles_touched uint32[N]
 *  Images: float32 planar [3][H][W] (PyTorch CHW).  Pixel (X, Y) has its
 *  centre at (X, Y) (A19); row-major pixel index Y·W + X.
 *  Tiles: 16×16 pixels, tile id = ty·tiles_x + tx, tiles_x = ceil(W/16),
 *  tiles_y = ceil(H/16) (A04).
 */
#ifndef DASS_H_
#define DASS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DASS_TILE 16
#define DASS_ABI_VERSION 3

typedef enum dass_status {
  DASS_OK = 0,
  DASS_ERR_INVALID_ARG = 1, /* usage error: bad size, null required pointer */
  DASS_ERR_DATA = 2,        /* data error: inputs inconsistent */
  DASS_ERR_NUMERICAL = 3,   /* non-finite values found (dass_scan_nonfinite) */
  DASS_ERR_CAPACITY = 4,    /* pair capacity too small (bin_sort host mode) */
  DASS_ERR_CUDA = 5         /* a CUDA runtime call failed */
} dass_status;

/*
 * Camera (D03; Alg. 1 input).
 *  - width, height ∈ [1, 65535]; fx, fy > 0.
 *  - viewmat: world→camera [R|t], row-major 3×4: t_cam = R·p + t.  R must be
 *    orthonormal (not checked).  Camera centre (SH direction origin) is −Rᵀt.
 *  - Pinhole: u = fx·t_x/t_z + cx, v = fy·t_y/t_z + cy, pixel centres at
 *    integers (A19): (W−1)/2 is the image centre.
 *  - near_plane: Gaussians with !(t_z > near_plane) are culled (A09).
 *  - full_proj: Alg. 1's "full projection matrix T", row-major 4×4 in
 *    the row-vector convention P_hom = [p, 1]·T; column 3 is the
 *    homogeneous coordinate.  Used only by dass_error_map.
 */
typedef struct dass_camera {
  int32_t width;
  int32_t height;
  float fx, fy, cx, cy;
  float viewmat[12];
  float near_plane;
  float full_proj[16];
} dass_camera;

/* Human-readable text for a status; never NULL. */
const char* dass_status_string(int status);
/* Thread-local message describing the last non-OK status of this thread. */
const char* dass_last_error(void);
/* DASS_ABI_VERSION of the loaded library. */
int dass_abi_version(void);
/* Total number of kernels this process has launched through libdass
 * (relaxed atomic; diagnostic for bench.py's gpu_launches). */
uint64_t dass_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * dass_apply_shift — masked per-Gaussian shift (§3.3; A24, A25)
 *   where dyn_mask[i] != 0:  p' = p + μ_i (xyz), o' = o,
 *                            q' = n(q) ⊗ n(σ_i) (Hamilton product, q on the
 *                            left; n(x) = x/‖x‖; ‖σ‖ < 1e-8 → σ := identity)
 *   where dyn_mask[i] == 0:  p', q' = exact copy.
 * mu, sigma: float4[n] (mu.w ignored; sigma = w,x,y,z).  dyn_mask: uint8[n],
 * nullable = all ones.  In-place (pos_opa_out == pos_opa, rot_out == rot) OK.
 * INVALID_ARG: n < 0, or n > 0 with a null required pointer.  n = 0 → OK.
 * ------------------------------------------------------------------------- */
int dass_apply_shift(int32_t n, const float* pos_opa, const float* rot,
                     const float* mu, const float* sigma,
                     const uint8_t* dyn_mask, float* pos_opa_out,
                     float* rot_out, void* stream);

/* dass_apply_shift_bwd — reverse of dass_apply_shift for the trained offsets
 * (the shift stage trains only the deformation outputs):
 *   g_mu    += mask · dL/dp'                         (xyz; w untouched)
 *   g_sigma += mask · (dL/dn(σ) − n(σ)(n(σ)·dL/dn(σ)))/‖σ‖ with
 *              dL/dn(σ) = L(n(q))ᵀ dL/dq' (L(a) = left-multiplication matrix);
 *              zero when ‖σ‖ < 1e-8.
 * rot is the PRE-shift quaternion.  g_pos_out/g_rot_out: gradients w.r.t. the
 * shifted pos_opa'/rot' (float4[n]).  g_mu, g_sigma nullable. */
int dass_apply_shift_bwd(int32_t n, const float* rot, const float* sigma,
                         const uint8_t* dyn_mask, const float* g_pos_out,
                         const float* g_rot_out, float* g_mu, float* g_sigma,
                         void* stream);

/* ---------------------------------------------------------------------------
 * dass_project — EWA projection + SH colour, one view (Eqs. 5-7, P:336-347;
 * colour P:351, A14).  Per Gaussian i:
 *  o_eff = keep_mask ? (keep_mask[i] ? o : 0) : o;  s_eff likewise (Eq. 1,
 *  P:94-95; a Quant = 0 Gaussian is culled by the opacity cull, A10).
 *
 *  KEY CHAIN — computed in IEEE fp32, every operation individually rounded
 *  (no FMA contraction), IEEE division and square root, in EXACTLY this order
 *  (a+b+c means ((a+b)+c); this is the bit-exact contract, hard part 1):
 *   1. t_a = ((V[a][0]·x + V[a][1]·y) + V[a][2]·z) + V[a][3], a = 0..2.
 *   2. cull unless t_z > near_plane.
 *   3. nq = sqrt(((w·w + x·x) + y·y) + z·z) of rot; cull unless nq > 0 and
 *      nq finite; q̂ = (w/nq, x/nq, y/nq, z/nq).
 *   4. R(q̂): with products xx=x·x, yy, zz, xy, xz, yz, wx, wy, wz:
 *      R00 = 1 − 2·(yy+zz), R01 = 2·(xy−wz), R02 = 2·(xz+wy),
 *      R10 = 2·(xy+wz), R11 = 1 − 2·(xx+zz), R12 = 2·(yz−wx),
 *      R20 = 2·(xz−wy), R21 = 2·(yz+wx), R22 = 1 − 2·(xx+yy).
 *   5. m_ak = R_ak·s_k;  Σ_ab = (m_a0·m_b0 + m_a1·m_b1) + m_a2·m_b2 (a ≤ b).
 *   6. lx = (1.3·W)/(2·fx), ly = (1.3·H)/(2·fy);
 *      x̃ = min(lx, max(−lx, t_x/t_z))·t_z, ỹ likewise;
 *      J00 = fx/t_z, J02 = −((fx·x̃)/(t_z·t_z)), J11 = fy/t_z,
 *      J12 = −((fy·ỹ)/(t_z·t_z)).
 *   7. M0k = J00·V[0][k] + J02·V[2][k];  M1k = J11·V[1][k] + J12·V[2][k].
 *      P_ak = (M_a0·Σ_0k + M_a1·Σ_1k) + M_a2·Σ_2k.
 *      a = ((P_00·M_00 + P_01·M_01) + P_02·M_02) + 0.3,
 *      b =  (P_00·M_10 + P_01·M_11) + P_02·M_12,
 *      c = ((P_10·M_10 + P_11·M_11) + P_12·M_12) + 0.3      (A07)
 *   8. det = a·c − b·b; cull unless det > 0.
 *   9. mid = 0.5·(a + c); λ = mid + sqrt(max(0.1, mid·mid − det));
 *      r = ceil(3·sqrt(λ))                                    (A06)
 *  10. u = (fx·t_x)/t_z + cx,  v = (fy·t_y)/t_z + cy  (unclamped);
 *      cull unless u, v, λ finite.
 *  11. x0 = max(0, ceil(u − r)), x1 = min(W − 1, floor(u + r)), y likewise
 *      (clamped in float before conversion to int); visible iff x0 ≤ x1,
 *      y0 ≤ y1 and o_eff ≥ 1/255 (A05, A10).
 *  12. Footprint threshold (A50): xo = 255·o_eff; with its IEEE bits, e =
 *      (bits >> 23) − 127 and m = the float with bits (bits & 0x7FFFFF) |
 *      0x3F800000 (m ∈ [1, 2)); L = ((float)e·0.693147182) + (m − 1)  (≥ ln xo);
 *      R2 = ((2·L)·1.01) + 0.05.
 *  13. Tile footprint: tx0 = x0/16, tx1 = x1/16, ty0 = y0/16, ty1 = y1/16.  If
 *      ty1 − ty0 + 1 > 8 or tx1 − tx0 + 1 > 255: every tile of the box, rows =
 *      all ones, tiles_touched = (tx1 − tx0 + 1)·(ty1 − ty0 + 1).  Otherwise,
 *      with sxa = sqrt(R2·a), tq = sqrt(R2/a), dyL = −(b·tq), dyR = b·tq,
 *      crr = c·R2, ey = sqrt(crr), icc = 1/c, for each tile row ty ∈ [ty0, ty1]
 *      (k = ty − ty0):
 *        Y0 = max(y0, 16·ty), Y1 = min(y1, 16·ty + 15);
 *        d0 = max((float)Y0 − v, −ey), d1 = min((float)Y1 − v, ey);
 *        if d0 ≤ d1: h_i = sqrt(max(0, det·(crr − d_i·d_i))),
 *          l_i = (b·d_i − h_i)·icc, r_i = (b·d_i + h_i)·icc (i = 0, 1);
 *          lo = −sxa if d0 ≤ dyL ≤ d1 else min(l0, l1);
 *          hi = sxa if d0 ≤ dyR ≤ d1 else max(r0, r1);
 *          X0 = max((float)x0, (u + lo) − 1), X1 = min((float)x1, (u + hi) + 1);
 *          if ceil(X0) ≤ floor(X1): row k spans the tiles ceil(X0)/16 …
 *          floor(X1)/16;
 *      (the tile columns the ellipse {d : dᵀ Σ'⁻¹ d ≤ R2} reaches in the row's
 *      band of pixel rows, padded by one pixel; every pixel with α ≥ 1/255
 *      lies inside it, so the tiled sequences equal the tile-free ones).
 *      tile_rows[4i..4i+3] (uint32 ×4, 16-byte aligned): row k in bits
 *      16·(k&1) … of word k>>1 as lo | hi << 8 (tile offsets from tx0; an
 *      empty row and rows past ty1 are lo = 255, hi = 0);
 *      tiles_touched = the number of tiles of the rows.
 *  The conic record is (A, β, γ) = (c/det, −b/c, 1/c), i.e. the conic
 *  (c, −b, a)/det of Eq. 7 in Cholesky form (see the layout above).  Colour (fast math
 *  allowed): d = (p − c_cam)/‖p − c_cam‖, col = Σ_k Y_k(d)·sh_k + 0.5 with the
 *  real SH basis of degree ≤ 3 listed in DESIGN.md (A14); a channel < 0 sets
 *  its clamp bit and is clamped to 0.
 * Culled Gaussians: tiles_touched = 0, box = {1, 1} (x0 > x1), tile_rows and
 * other records zero.  A visible Gaussian (box non-empty, o_eff ≥ 1/255) may
 * still have tiles_touched = 0 (its support reaches no pixel of the image).
 * Degenerate q is culled, not an error (A15).
 * INVALID_ARG: bad camera, n < 0, sh_degree ∉ [0,3], null required pointer.
 * ------------------------------------------------------------------------- */
int dass_project(const dass_camera* cam, int32_t n, int32_t sh_degree,
                 const float* pos_opa, const float* scale, const float* rot,
                 const float* sh, const uint8_t* keep_mask, float* xy_depth,
                 float* conic_opa, float* rgb, uint32_t* box,
                 uint32_t* tile_rows, uint32_t* tiles_touched, void* stream);

/* dass_project_views — the same as V calls of dass_project (one per camera),
 * in one launch that reads the parameters once for all V views (a2, "multi-
 * view batched").  Record arrays are [V][N] concatenations of the per-view
 * layout above (view v's xy_depth at xy_depth + 4·v·N, etc.). */
int dass_project_views(const dass_camera* cams, int32_t num_views, int32_t n,
                       int32_t sh_degree, const float* pos_opa,
                       const float* scale, const float* rot, const float* sh,
                       const uint8_t* keep_mask, float* xy_depth,
                       float* conic_opa, float* rgb, uint32_t* box,
                       uint32_t* tile_rows, uint32_t* tiles_touched, void* stream);

/* dass_project_views_part — dass_project_views in two parts that may run on two
 * streams (same arguments, plus `part`):
 *  DASS_PROJECT_KEYS (1): the KEY CHAIN with its footprint — writes xy_depth
 *    as (0, 0, z, 0), box, tile_rows, tiles_touched: everything dass_bin_sort
 *    reads.  sh and conic_opa / rgb are not touched.
 *  DASS_PROJECT_RECORDS (2): reads box (the keys' visibility decision) and
 *    writes words 0, 1 and 3 of xy_depth (u_hi, v_hi, the fp16 lo pair),
 *    conic_opa and rgb.  Must be ordered after the KEYS part of the same
 *    arrays; writes no byte the KEYS part or dass_bin_sort reads, so it may run
 *    concurrently with dass_bin_sort of the same views.  The raster calls
 *    must be ordered after it.
 *  DASS_PROJECT_ALL (3): both in order on `stream` (= dass_project_views).
 * After both parts every output equals dass_project_views' bit for bit.
 * INVALID_ARG as dass_project_views, or part ∉ {1, 2, 3}. */
#define DASS_PROJECT_KEYS 1
#define DASS_PROJECT_RECORDS 2
#define DASS_PROJECT_ALL 3
int dass_project_views_part(int32_t part, const dass_camera* cams, int32_t num_views,
                            int32_t n, int32_t sh_degree, const float* pos_opa,
                            const float* scale, const float* rot, const float* sh,
                            const uint8_t* keep_mask, float* xy_depth,
                            float* conic_opa, float* rgb, uint32_t* box,
                            uint32_t* tile_rows, uint32_t* tiles_touched, void* stream);

/* ---------------------------------------------------------------------------
 * dass_bin_sort — tile binning + sort + per-tile ranges (a3-a5; P:29
 * "tile-based"; A03, A04, A50).  For every visible Gaussian i and every tile
 * (tx, ty) of its footprint (tile_rows of dass_project, KEY CHAIN step 13: a
 * subset of its pixel box's tiles) emit the pair key = (tile_id << 32) |
 * bits_u32(z_i), value = i.  Output: the
 * pairs in ascending (key, i) order — i.e. lexicographic (tile, depth bits,
 * Gaussian index) — and ranges[t] = [first, one-past-last) of tile t in that
 * order, [0, 0) for an empty tile.  Integer work: bit-exact by contract.
 *
 *  ws, ws_bytes: workspace of at least dass_bin_sort_workspace(n, num_tiles,
 *    pair_capacity) bytes.
 *  sorted_keys: uint64[pair_capacity], nullable (skips writing the keys).
 *  sorted_ids: uint32[pair_capacity].  tile_ranges: uint32[2·num_tiles].
 *  num_pairs_dev: uint32[2] device: [0] = K (total pairs, even on overflow),
 *    [1] = 1 if K > pair_capacity (then every range is [0,0)), else 0.
 *  num_pairs_host: nullable.  Non-null = HOST MODE: the call synchronises the
 *    stream once, stores K, and returns DASS_ERR_CAPACITY if K > capacity.
 *    Null = GRAPH MODE: no synchronisation (capturable in a CUDA graph); the
 *    caller reads num_pairs_dev later.
 * Requires 0 ≤ pair_capacity < 2^30 and 0 ≤ n < 2^30 (the onesweep
 * look-back packs counts into 30 bits).
 * ------------------------------------------------------------------------- */
int dass_bin_sort_workspace(int32_t n, int32_t num_tiles,
                            int64_t pair_capacity, size_t* bytes);
int dass_bin_sort(const dass_camera* cam, int32_t n, const float* xy_depth,
                  const uint32_t* box, const uint32_t* tile_rows,
                  const uint32_t* tiles_touched, void* ws, size_t ws_bytes,
                  int64_t pair_capacity,
                  uint64_t* sorted_keys, uint32_t* sorted_ids,
                  uint32_t* tile_ranges, uint32_t* num_pairs_dev,
                  int64_t* num_pairs_host, void* stream);

/* dass_bin_sort_shared — dass_bin_sort (same arguments, workspace, outputs and
 * errors, bit for bit the same results) for a view sorted while other views'
 * kernels share the GPU, as in the multi-view step.  K is known on the
 * device only, so dass_bin_sort launches the pair passes for the capacity, one
 * block per 2048-key tile; here a fixed grid of 74 blocks loops over the key
 * tiles instead: slower alone, but fewer resident blocks next to the other
 * views' sorts and raster kernels (C3 step 11.32 → 11.29 ms against a
 * one-block-per-SM grid, 11.44 against the capacity grid). */
int dass_bin_sort_shared(const dass_camera* cam, int32_t n, const float* xy_depth,
                         const uint32_t* box, const uint32_t* tile_rows,
                         const uint32_t* tiles_touched, void* ws, size_t ws_bytes,
                         int64_t pair_capacity,
                         uint64_t* sorted_keys, uint32_t* sorted_ids,
                         uint32_t* tile_ranges, uint32_t* num_pairs_dev,
                         int64_t* num_pairs_host, void* stream);

/* ---------------------------------------------------------------------------
 * dass_bin_sort_views — dass_bin_sort for V views of one timestep at once
 * (a3-a5 batched over the views of P:74; A03, A04).  All cameras share W×H
 * (the tile grid T); the records are the [V][N] arrays of
 * dass_project_views.  Per view v the outputs equal, bit for bit, those of
 * dass_bin_sort on view v alone (graph mode): sorted_ids[v·view_capacity + k]
 * for k < K_v, tile_ranges[(v·T + t)·2 + {0,1}] view-relative [s, e) (empty
 * tiles [0, 0)), num_pairs_dev[2v] = K_v, num_pairs_dev[2v+1] = 1 if K_v >
 * view_capacity (that view's ranges then stay empty; if the batch total
 * exceeds V·view_capacity every view is flagged).  One depth presort of the
 * V·N (view, Gaussian) keys, one emission and one sort of all pairs on the
 * combined index v·T + tile: a few large kernels instead of V latency-bound
 * chains.  No host synchronisation.
 *  INVALID_ARG: V ∉ [1, 64], cameras of different sizes, n < 0, view_capacity
 *   ∉ [0, 2^30 / V), a null required pointer, workspace too small.
 * ------------------------------------------------------------------------- */
int dass_bin_sort_views_workspace(int32_t num_views, int32_t n,
                                  int64_t view_capacity, size_t* bytes);
int dass_bin_sort_views(const dass_camera* cams, int32_t num_views, int32_t n,
                        const float* xy_depth, const uint32_t* box,
                        const uint32_t* tile_rows, const uint32_t* tiles_touched,
                        void* ws, size_t ws_bytes,
                        int64_t view_capacity, uint32_t* sorted_ids,
                        uint32_t* tile_ranges, uint32_t* num_pairs_dev,
                        void* stream);

/* ---------------------------------------------------------------------------
 * dass_render_fwd — front-to-back compositing (Eq. 8; A01, A05,
 * A11-A13).  For pixel (X, Y), over the tile's sorted list, skipping entries
 * whose box does not contain the pixel:
 *   dx = u − X, dy = v − Y; power = −0.5·(A·dx² + C·dy²) − B·dx·dy
 *   (evaluated as −[(s dx + sβ dy)² + (g dy)²], the same fp32 bits in every
 *   kernel, A35);
 *   skip if power > 0; α = min(0.99, o·exp(power)); skip if α < 1/255;
 *   if T·(1 − α) < 1e-4 stop (the entry is NOT added);
 *   otherwise C += rgb·α·T, T ← T·(1 − α).      (T starts at 1)
 * out_img[ch] = C + T·bg[ch] (bg: host float[3], nullable = black);
 * out_T = final T; out_last = one past the sorted-list index of the last
 * accepted entry (the range start if none).  Both are needed by the backward.
 *
 * accept (nullable): acceptance-list workspace of dass_render_accept_workspace
 *   (num_tiles, pair_capacity) bytes.  When given, the forward also records,
 *   for every tile and every list entry accepted by at least one of its
 *   pixels, the entry index and which of the tile's pixels accepted it (one
 *   list per tile, plus the tiles' launch order); dass_render_bwd* then walk
 *   only those (A38).  pair_capacity must be at least the pair count of the
 *   sort that produced tile_ranges (the one given to dass_bin_sort): a tile
 *   range ending past it traps on the device.  Opaque layout; valid until the
 *   next dass_render_fwd on the same buffer.  accept_bytes = its size.
 *   INVALID_ARG: accept not 16-byte aligned, accept_bytes below the workspace
 *   size, pair_capacity ∉ [0, 2^30).  The same holds for the accept argument
 *   of every dass_render_bwd* call.
 * ------------------------------------------------------------------------- */
int dass_render_accept_workspace(int32_t num_tiles, int64_t pair_capacity,
                                 size_t* bytes);
int dass_render_fwd(const dass_camera* cam, const uint32_t* tile_ranges,
                    const uint32_t* sorted_ids, const float* xy_depth,
                    const float* conic_opa, const float* rgb,
                    const uint32_t* box, const float* bg, float* out_img,
                    float* out_T, uint32_t* out_last, void* accept,
                    size_t accept_bytes, int64_t pair_capacity, void* stream);

/* ---------------------------------------------------------------------------
 * dass_render_bwd — reverse-mode gradient of dass_project + dass_render_fwd
 * for one view (a7, a8; reverse of Eqs. 5-8; P:159 for ∇p̄).  The exact
 * derivative of the forward holding the accepted set and clamp states fixed
 * (A17, A18): α clamped at 0.99 → ∂α/∂(o, G) = 0; clamped colour channels get
 * no gradient; J's clamp differentiated exactly (A08).
 * Gradients are w.r.t. the ACTIVATED scale and opacity and the RAW
 * quaternion (A16), accumulated (+=) into g_* (nullable: a null output skips
 * its work), summed over pixels and views (A27).
 *   gradstat_sum[i] += ‖(dL/du·W/2, dL/dv·H/2)‖₂ and gradstat_cnt[i] += 1 for
 *   every Gaussian visible in this view (A23).  Both nullable.
 * The caller must pass the SAME records and fwd outputs; the ABI
 * cannot check this.  dL_dimg: float [3][H][W].  ws: dass_render_bwd_workspace.
 * accept/pair_capacity: the forward's acceptance lists (nullable: the pass
 * then re-derives the accepted set from out_last; same result).
 * ------------------------------------------------------------------------- */
int dass_render_bwd_workspace(int32_t n, size_t* bytes);
int dass_render_bwd(const dass_camera* cam, int32_t n, int32_t sh_degree,
                    const float* pos_opa, const float* scale, const float* rot,
                    const float* sh, const uint8_t* keep_mask,
                    const uint32_t* tile_ranges, const uint32_t* sorted_ids,
                    const float* xy_depth, const float* conic_opa,
                    const float* rgb, const uint32_t* box, const float* bg,
                    const float* out_T, const uint32_t* out_last,
                    const float* dL_dimg, const void* accept, size_t accept_bytes,
                    int64_t pair_capacity, void* ws, size_t ws_bytes,
                    float* g_pos_opa, float* g_scale, float* g_rot,
                    float* g_sh, float* gradstat_sum, uint32_t* gradstat_cnt,
                    void* stream);

/* ---------------------------------------------------------------------------
 * Two-phase backward for multi-view batches (same mathematics as
 * dass_render_bwd, which is exactly phase 1 + phase 2 for V = 1):
 *
 * dass_render_bwd_raster — phase 1, one view: the per-pixel reverse pass of
 *   Eq. 8.  Writes (overwrites) the view's per-Gaussian 2D moment workspace
 *   g2d: float[N][12] (3 float4 per Gaussian, dass_render_bwd_workspace
 *   bytes): (Σe·dx, Σe·dy, Σe·dx², Σe·dx·dy, Σe·dy², Σe, Σ αT·g_rgb) with
 *   e = G·∂L/∂α (0 where α is clamped).  Views on distinct streams may run
 *   concurrently (each writes only its own g2d).
 *
 * dass_render_bwd_preprocess_views — phase 2, V views at once: chains every
 *   view's moments through Eqs. 5-7 and the SH colour into ∂L/∂(p, s, q, o,
 *   sh) and ∇p̄, reading the parameters once and updating each output once
 *   (+=).  cams[V]; records as written by dass_project_views ([V][N]
 *   concatenations of conic_opa, rgb, box); g2d: V phase-1 workspaces
 *   concatenated ([V][N][12] floats).
 * ------------------------------------------------------------------------- */
int dass_render_bwd_raster(const dass_camera* cam, int32_t n, const uint32_t* tile_ranges,
                           const uint32_t* sorted_ids, const float* xy_depth,
                           const float* conic_opa, const float* rgb, const uint32_t* box,
                           const float* bg, const float* out_T, const uint32_t* out_last,
                           const float* dL_dimg, const void* accept, size_t accept_bytes,
                           int64_t pair_capacity, float* g2d, void* stream);
int dass_render_bwd_preprocess_views(const dass_camera* cams, int32_t num_views, int32_t n,
                                     int32_t sh_degree, const float* pos_opa,
                                     const float* scale, const float* rot, const float* sh,
                                     const uint8_t* keep_mask, const float* conic_opa,
                                     const float* rgb, const uint32_t* box, const float* g2d,
                                     float* g_pos_opa, float* g_scale, float* g_rot,
                                     float* g_sh, float* gradstat_sum,
                                     uint32_t* gradstat_cnt, void* stream);

/* ---------------------------------------------------------------------------
 * Tile subsets and split views (multi-GPU load balance).  A view
 * can be rendered in parts: each part is a tile subset, and the parts' results
 * add up to the whole view.
 *
 * dass_render_fwd_tiles / dass_render_bwd_raster_tiles: as dass_render_fwd /
 *   dass_render_bwd_raster, restricted to tiles tile_begin + k·tile_stride,
 *   k < tile_count (tile index = ty·tiles_x + tx; tile_count < 0 = every tile).
 *   Only those tiles' pixels are written.  g2d is overwritten with the subset's
 *   partial moments; moments are sums over pixels, so the subsets' g2d add up to
 *   the whole view's.  INVALID_ARG: tile_stride < 1, tile_begin < 0, or a
 *   subset reaching past the last tile.
 *
 * dass_render_bwd_preprocess_views_uv: dass_render_bwd_preprocess_views with
 *   uv_out, a host array of num_views device pointers (array nullable; entries
 *   nullable, else 8-byte aligned float2[n]), and uv_count, a host uint8 array
 *   (nullable).  Every gradient is linear in g2d, so partial-view moments give
 *   partial gradients, except the ∇p̄ norm.  For a view with uv_out[v] set, the
 *   kernel therefore adds to uv_out[v][i], instead of the norm,
 *     (∂L/∂u·W/2, ∂L/∂v·H/2)           for every Gaussian visible in the view,
 *   and adds the view's gradstat_cnt term only if uv_count[v] ≠ 0 (exactly one
 *   of the GPUs sharing a view sets it: visibility is the same on each).  The
 *   caller sums the partials (e.g. inside the gradient all_reduce).
 * dass_gradstat_from_uv: then, for the num_split reduced blocks
 *   uv[num_split][n] (float2), adds gradstat_sum[i] += Σ_k ‖uv[k][i]‖₂ — the
 *   terms the whole views would have contributed (A23; an invisible Gaussian
 *   has (0, 0) and adds nothing in either form).
 * ------------------------------------------------------------------------- */
int dass_render_fwd_tiles(const dass_camera* cam, int32_t tile_begin, int32_t tile_stride,
                          int32_t tile_count, const uint32_t* tile_ranges,
                          const uint32_t* sorted_ids, const float* xy_depth,
                          const float* conic_opa, const float* rgb, const uint32_t* box,
                          const float* bg, float* out_img, float* out_T, uint32_t* out_last,
                          void* accept, size_t accept_bytes, int64_t pair_capacity, void* stream);
int dass_render_bwd_raster_tiles(const dass_camera* cam, int32_t tile_begin, int32_t tile_stride,
                                 int32_t tile_count, int32_t n, const uint32_t* tile_ranges,
                                 const uint32_t* sorted_ids, const float* xy_depth,
                                 const float* conic_opa, const float* rgb, const uint32_t* box,
                                 const float* bg, const float* out_T, const uint32_t* out_last,
                                 const float* dL_dimg, const void* accept, size_t accept_bytes,
                                 int64_t pair_capacity, float* g2d, void* stream);
int dass_render_bwd_preprocess_views_uv(const dass_camera* cams, int32_t num_views, int32_t n,
                                        int32_t sh_degree, const float* pos_opa,
                                        const float* scale, const float* rot, const float* sh,
                                        const uint8_t* keep_mask, const float* conic_opa,
                                        const float* rgb, const uint32_t* box, const float* g2d,
                                        float* g_pos_opa, float* g_scale, float* g_rot,
                                        float* g_sh, float* gradstat_sum,
                                        uint32_t* gradstat_cnt, float* const* uv_out,
                                        const uint8_t* uv_count, void* stream);

/* dass_render_bwd_preprocess_views_part — dass_render_bwd_preprocess_views_uv in
 * two parts that write disjoint outputs and may run on two streams:
 *  DASS_PREPROCESS_GEOMETRY (1): ∂L/∂(p, o, s, q), the ∇p̄ statistic (or the
 *    split views' uv blocks) and the visibility counts;
 *  DASS_PREPROCESS_SH (2): ∂L/∂SH coefficients (g_sh);
 *  DASS_PREPROCESS_ALL (3): both in order on `stream` (= the _uv call).
 * Both parts only read the records and the 2-D moments.  INVALID_ARG as the
 * _uv call, or part ∉ {1, 2, 3}. */
#define DASS_PREPROCESS_GEOMETRY 1
#define DASS_PREPROCESS_SH 2
#define DASS_PREPROCESS_ALL 3
int dass_render_bwd_preprocess_views_part(int32_t part, const dass_camera* cams, int32_t num_views,
                                          int32_t n, int32_t sh_degree, const float* pos_opa,
                                          const float* scale, const float* rot, const float* sh,
                                          const uint8_t* keep_mask, const float* conic_opa,
                                          const float* rgb, const uint32_t* box, const float* g2d,
                                          float* g_pos_opa, float* g_scale, float* g_rot,
                                          float* g_sh, float* gradstat_sum,
                                          uint32_t* gradstat_cnt, float* const* uv_out,
                                          const uint8_t* uv_count, void* stream);
int dass_gradstat_from_uv(int32_t n, int32_t num_split, const float* uv, float* gradstat_sum,
                          void* stream);

/* ---------------------------------------------------------------------------
 * dass_fidelity_loss — the fidelity loss of Eq. 3, "the fidelity
 * loss in the vanilla 3DGS": L = (1−λ)·L1 + λ·D-SSIM with
 * D-SSIM = dssim_scale·(1 − SSIM): 1 is the 3DGS code's 1 − SSIM (A39, the
 * default of the Python binding), 0.5 SPEC's (1 − SSIM)/2; with
 *   L1 = mean over the 3·H·W values of |img − gt|;
 *   SSIM = mean over 3·H·W of S = ((2μ_Iμ_G + C1)(2σ_IG + C2)) /
 *          ((μ_I² + μ_G² + C1)(σ_I² + σ_G² + C2)), per channel, windowed
 *          statistics over an 11×11 Gaussian window (σ = 1.5, normalised),
 *          zero padding outside the image, C1 = 0.01², C2 = 0.03².
 * img, gt: float [3][H][W].  λ ∈ [0, 1] (0.2 in 3DGS); dssim_scale ∈ (0, 1].  loss: device float[3]
 * = (L, L1, SSIM), written.  dL_dimg: float [3][H][W] = ∂L/∂img, written
 * (nullable: forward only; sign(0) = 0 for the L1 term).  ws: workspace of
 * dass_fidelity_loss_workspace bytes, 16-byte aligned.  Any img/gt alignment
 * is accepted: when W % 4 == 0 and the planes are 16-byte aligned the halo
 * tiles are staged by TMA (cp.async.bulk.tensor), else by plain loads; both
 * stage the same values, so the results are bit-identical.
 * ------------------------------------------------------------------------- */
int dass_fidelity_loss_workspace(int32_t width, int32_t height, size_t* bytes);
int dass_fidelity_loss(int32_t width, int32_t height, const float* img,
                       const float* gt, float lambda, float dssim_scale, void* ws,
                       size_t ws_bytes, float* loss, float* dL_dimg, void* stream);

/* ---------------------------------------------------------------------------
 * Selective inheritance, Eq. 1 with the straight-through estimator
 * — SURVEY §8(f) f3.
 *
 * dass_inherit_mask: keep[i] = Quant(sigmoid(m_i)) with Quant(x) = 1[x ≥ 0.5]
 *   (A26), i.e. keep = 1[m ≥ 0] (sigmoid(0) = 0.5 keeps).  Feed `keep`
 *   as keep_mask to dass_project / dass_render_bwd*: o_r = keep·o and
 *   s_r = keep·s, and a Quant = 0 Gaussian is culled (A10).  m: float[n].
 *
 * dass_inherit_mask_bwd: the STE gradient of m_op = detach(Quant(σ(m)) − σ(m))
 *   + σ(m) plus the mask loss λ_inher·Σ σ(m) of Eq. 2:
 *     g_m[i] += (o_i·∂L/∂o_r,i + Σ_k s_i,k·∂L/∂s_r,i,k + λ_inher)·σ'(m_i),
 *   σ'(m) = σ(m)(1 − σ(m)).  ∂L/∂o_r and ∂L/∂s_r are g_pos_opa.w and g_scale
 *   from dass_render_bwd* (gradients w.r.t. the effective o, s; zero for
 *   culled Gaussians).  pos_opa/scale: the un-masked o, s.
 * ------------------------------------------------------------------------- */
int dass_inherit_mask(int32_t n, const float* m, uint8_t* keep, void* stream);
int dass_inherit_mask_bwd(int32_t n, const float* m, const float* pos_opa,
                          const float* scale, const float* g_pos_opa,
                          const float* g_scale, float lambda_inher, float* g_m,
                          void* stream);

/* ---------------------------------------------------------------------------
 * Dual hash-grid deformation (§3.3; supplement §B) —
 * SURVEY §8(f) f2.  Each field 𝓗 (𝓗_dyn for the dynamic group, 𝓗_st for the
 * static one) maps a Gaussian position p to (μ, σ):
 *   enc(p):  per level l < levels with resolution N_l = resolution[l]:
 *            x̂ = clamp((p − aabb_min)/(aabb_max − aabb_min), 0, 1),
 *            s = x̂·N_l, i0 = min(⌊s⌋, N_l − 1), w = s − i0 (per axis);
 *            the 8 corners i0 + c, c ∈ {0,1}³, read table row
 *              (N_l+1)³ ≤ T:  x + y(N_l+1) + z(N_l+1)²               (dense)
 *              otherwise:     (x ⊕ y·2654435761 ⊕ z·805459861) mod T (u32)
 *            weighted Π_k (c_k ? w_k : 1 − w_k); features of the levels
 *            concatenated (I-NGP; A41).
 *   MLP:     in = levels·features → 64 → 64 → 7, ReLU hidden, linear head.
 *   μ = out[0:3], σ = (1, 0, 0, 0) + out[3:7] (a zero head is the identity
 *   deformation; A42).  Feed μ, σ to dass_apply_shift (q' = n(q) ⊗ n(σ)).
 * T_Hash / F_Hash per group and dataset: N3DV 2^16/4 (dyn), 2^14/2 (st); Meet
 * Room 2^15/4, 2^13/2.
 *
 * Memory (all device, caller-owned, float32):
 *   table: [levels][T][features] (16-byte aligned for features = 4, 8 for 2);
 *   mlp:   flat W1[64][in] b1[64] W2[64][64] b2[64] W3[7][64] b3[7]
 *          (dass_deform_param_count gives both sizes);
 *   pos_opa, mu, sigma, g_mu, g_sigma: float4[n_gauss] (16-byte aligned);
 *     mu.w is written 0; sigma = (w, x, y, z).
 * Rows: row k < (count ? *count : n) processes Gaussian i = idx ? idx[k] : k
 * (count is a DEVICE int, so a partition can feed it without a host sync;
 * n bounds it and sizes the grid).  Rows ≥ the count are untouched.
 * dass_deform_fwd writes mu[i], sigma[i].  dass_deform_bwd recomputes the
 * forward and ACCUMULATES (+=) ∂L/∂table into g_table and ∂L/∂mlp into g_mlp
 * from ∂L/∂μ = g_mu[i].xyz and ∂L/∂σ = g_sigma[i] (float atomics: the
 * summation order is not deterministic).  ReLU'(0) = 0.
 * INVALID_ARG: levels ∉ [1, 16], features ∉ {1, 2, 4}, in = levels·features
 *   not a multiple of 4 or > 64, log2_table ∉ [1, 24], resolution[l] ∉
 *   [1, 2^20], aabb not finite or max ≤ min, n < 0, a null required pointer
 *   or a misaligned one.
 *
 * dass_partition: the stable split of the Gaussians by the dynamics mask
 *   (§3.3): idx_dyn = ascending {i : mask[i] ≠ 0}, idx_st = ascending
 *   {i : mask[i] = 0} (each int32[n]), counts (device int32[2]) = (#dyn, #st).
 *   ws: dass_partition_workspace bytes (4-byte aligned).  Deterministic.
 * ------------------------------------------------------------------------- */
#define DASS_MLP_HIDDEN 64
typedef struct dass_hashgrid {
  int32_t levels;          /* L */
  int32_t log2_table;      /* T = 2^log2_table rows per level (T_Hash) */
  int32_t features;        /* F_Hash */
  int32_t reserved;        /* 0 */
  int32_t resolution[16];  /* N_l, l < levels */
  float aabb_min[3];
  float aabb_max[3];
} dass_hashgrid;

int dass_deform_param_count(const dass_hashgrid* cfg, int64_t* table_floats,
                            int64_t* mlp_floats);
int dass_deform_fwd(const dass_hashgrid* cfg, const float* table, const float* mlp,
                    int32_t n, const int32_t* idx, const int32_t* count,
                    const float* pos_opa, float* mu, float* sigma, void* stream);
int dass_deform_bwd(const dass_hashgrid* cfg, const float* table, const float* mlp,
                    int32_t n, const int32_t* idx, const int32_t* count,
                    const float* pos_opa, const float* g_mu, const float* g_sigma,
                    float* g_table, float* g_mlp, void* stream);
int dass_partition_workspace(int32_t n, size_t* bytes);
int dass_partition(int32_t n, const uint8_t* mask, int32_t* idx_dyn, int32_t* idx_st,
                   int32_t* counts, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Error-guided densification (§3.4) — SURVEY §8(f) f4.
 *
 * dass_densify_select: Eq. 4
 *     S = {n : ∇p̄_n > τ_pos} ∪ (S_err ∩ {n : ∇p̄_n > τ_err}),
 *   ∇p̄_n = gradstat_sum[n] / gradstat_cnt[n] (one IEEE fp32 division; 0 when
 *   the count is 0; A44), S_err = {n : s_err[n] ≠ 0} from dass_error_map
 *   (nullable: ∅).  in_S: uint8[n] written (1 = selected); idx: int32[n],
 *   the first |S| entries = ascending members of S; counts: device int32[2]
 *   = (|S|, n − |S|).  ws: dass_partition_workspace(n) bytes.  Deterministic.
 *
 * dass_spawn: spawn densification (A45).  Writes n_out = n + m·K rows
 *   to the out arrays (sh planes with stride n_out): rows [0, n) copy the
 *   input, and child j < K of the k-th listed parent i = idx[k] (k < m, host
 *   int, e.g. counts[0] of dass_densify_select) goes to row n + k·K + j:
 *     z ~ N(0, I₃) from Philox4x64-10(counter = (k·K + j, 0, 0, 0),
 *                                     key = (seed, 0x44415353)),
 *       Box-Muller on u_a = ((x_a >> 40) + ½)·2⁻²⁴:
 *       z = (r₀cos 2πu₁, r₀sin 2πu₁, r₁cos 2πu₃), r_b = √(−2 ln u_{2b}),
 *     p_child = p + R(n(q))·(s ∘ z)   (a sample of N(p, Σ), Σ = R S Sᵀ Rᵀ),
 *     s_child = s / scale_shrink, o_child = child_opacity,
 *     q, SH and the dynamic flag copied.
 *   dyn/out_dyn nullable (both or neither).  K ≥ 1, scale_shrink > 0.
 *
 * dass_prune_select: opacity pruning of the candidates (A46): keep
 *   row i iff i < first (the frozen base rows) or o_i ≥ min_opacity.  keep:
 *   uint8[n] written; idx / counts as for dass_densify_select (the kept rows,
 *   ascending).  ws: dass_partition_workspace(n) bytes.
 *
 * dass_gather: out row k ← input row idx[k] for k < m (host int), all fields
 *   (pos_opa, scale, rot, the K4 SH planes with strides n and m, dyn).  With
 *   dass_prune_select's idx and m = counts[0] it is the pruned set.
 *
 * INVALID_ARG: n < 0, m < 0, sh_degree ∉ [0, 3], a null required pointer,
 *   misaligned float4 arrays, K < 1 or scale_shrink ≤ 0 (spawn), m > n (gather).
 * ------------------------------------------------------------------------- */
int dass_densify_select(int32_t n, const float* gradstat_sum, const uint32_t* gradstat_cnt,
                        const uint8_t* s_err, float tau_pos, float tau_err, uint8_t* in_S,
                        int32_t* idx, int32_t* counts, void* ws, size_t ws_bytes,
                        void* stream);
int dass_spawn(int32_t n, int32_t sh_degree, const float* pos_opa, const float* scale,
               const float* rot, const float* sh, const uint8_t* dyn, int32_t m,
               const int32_t* idx, int32_t spawn_count, float scale_shrink,
               float child_opacity, uint64_t seed, float* out_pos_opa, float* out_scale,
               float* out_rot, float* out_sh, uint8_t* out_dyn, void* stream);
int dass_prune_select(int32_t n, int32_t first, const float* pos_opa, float min_opacity,
                      uint8_t* keep, int32_t* idx, int32_t* counts, void* ws,
                      size_t ws_bytes, void* stream);
int dass_gather(int32_t n, int32_t sh_degree, const float* pos_opa, const float* scale,
                const float* rot, const float* sh, const uint8_t* dyn, int32_t m,
                const int32_t* idx, float* out_pos_opa, float* out_scale, float* out_rot,
                float* out_sh, uint8_t* out_dyn, void* stream);

/* ---------------------------------------------------------------------------
 * dass_render_features — identity-feature render, Eq. 9 (A47):
 *   M = Σ_i e_i α_i Π_{j<i}(1 − α_j)
 * over the same sorted tile lists, records, α decisions (Eq. 8, A09-A12,
 * A35-A36) and early stop as dass_render_fwd, with per-Gaussian features
 * e (float [n][channels], 16-byte aligned; channels ∈ {4, 8, 12, 16}; 16 in
 * Gaussian Grouping) in place of the colour and no background term.
 * out: float [channels][H][W], overwritten.  Inputs as for dass_render_fwd.
 * ------------------------------------------------------------------------- */
int dass_render_features(const dass_camera* cam, const uint32_t* tile_ranges,
                         const uint32_t* sorted_ids, const float* xy_depth,
                         const float* conic_opa, const uint32_t* box, int32_t channels,
                         const float* feat, float* out, void* stream);

/* ---------------------------------------------------------------------------
 * dass_error_map — error map, binarisation and Alg. 1 (§3.4 P:164-165, P:174;
 * Alg. 1 P:403-415 with the garble fixed, A20-A22).
 *   E(X,Y) = (1/3)·Σ_ch |rendered − gt|  → err (float [H][W], nullable)
 *   D = E > gamma_err (strict)           → dmask (uint32[ceil(HW/32)],
 *       bit (p & 31) of word p >> 5 for pixel p = Y·W + X; nullable)
 *   For n < n_base (𝒢^base only): P_hom = [p_n, 1]·T (T = full_proj);
 *   x_norm = P_hom.x/P_hom.w, y_norm = P_hom.y/P_hom.w;
 *   x_n = round(0.5·((x_norm + 1)·W − 1)), y_n = round(0.5·((y_norm + 1)·H − 1))
 *   (round half away from zero); skipped if P_hom.w ≤ near_plane or the pixel
 *   is outside the image; otherwise s_err[n] |= D[y_n][x_n]  (uint8, nullable).
 * INVALID_ARG: gamma_err ≤ 0, bad camera.  DATA: rendered or gt null.
 * ------------------------------------------------------------------------- */
int dass_error_map(const dass_camera* cam, const float* rendered,
                   const float* gt, float gamma_err, float* err,
                   uint32_t* dmask, int32_t n_base, const float* pos_opa,
                   uint8_t* s_err, void* stream);

/* ---------------------------------------------------------------------------
 * dass_render_stats — scene statistics of one rendered view,
 * diagnostic, not on the timed path.  counters: uint64[8] device, overwritten:
 *   [0] P_fwd   Σ_px entries whose box contains the pixel, visited by the
 *               forward up to and including its terminating entry
 *   [1] P_bwd   Σ_px entries with index < out_last whose box contains the pixel
 *   [2] accepted Σ_px accepted (composited) entries
 *   [3] pixels that terminated early (T·(1−α) < 1e-4 reached)
 *   [4] Σ_tiles list length, [5] max list length, [6] non-empty tiles,
 *   [7] Σ_px entries in the pixel's tile list up to out_last (box-unfiltered)
 * ------------------------------------------------------------------------- */
int dass_render_stats(const dass_camera* cam, const uint32_t* tile_ranges,
                      const uint32_t* sorted_ids, const float* xy_depth,
                      const float* conic_opa, const uint32_t* box,
                      const float* out_T, const uint32_t* out_last,
                      uint64_t* counters, void* stream);

/* ---------------------------------------------------------------------------
 * dass_scan_nonfinite — numerical validation, SPEC's "numerical" exit code
 * (S:795): bad_dev[0] += the number of NaN / ±Inf values in data[0, count)
 * (float, device; the caller zeroes bad_dev, so several arrays can share one
 * counter).  bad_host: nullable.  Non-null = HOST MODE: the call synchronises
 * the stream, stores the counter and returns DASS_ERR_NUMERICAL if it is
 * non-zero.  Null = GRAPH MODE (capturable): the caller reads bad_dev later
 * (paper_2411_14847_b200/step.py runs it on the step's gradients when asked).
 * INVALID_ARG: count < 0, null bad_dev, null data with count > 0.
 * ------------------------------------------------------------------------- */
int dass_scan_nonfinite(const float* data, int64_t count, uint32_t* bad_dev,
                        int64_t* bad_host, void* stream);

/* ---------------------------------------------------------------------------
 * dass_timestamp — diagnostic: one single-thread kernel on `stream` writes the
 * GPU global timer (ns) to stamps[slot] when it runs, so a captured CUDA graph
 * can be given a per-stream timeline (tools/timeline.py).  stamps: uint64
 * device array owned by the caller.  INVALID_ARG if stamps is null or slot < 0.
 * Not on the hot path.
 * ------------------------------------------------------------------------- */
int dass_timestamp(uint64_t* stamps, int32_t slot, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DASS_H_ */
