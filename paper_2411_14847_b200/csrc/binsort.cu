// binsort.cu — dass_bin_sort: tile binning, in-house onesweep LSD radix sort
// and per-tile ranges ("tile-based"; A03, A04).
//
// Contract: the pairs (key = tile<<32 | bits(z), value = Gaussian id) in
// ascending (tile, depth bits, id) order.  Equivalent, cheaper order of work
// (SURVEY §7.3 hard part 4): (1) a stable onesweep sort of the N Gaussians by
// their 32 depth bits (key = zbits<<32 | id, 4 passes over N, not over K);
// (2) an exclusive scan of tiles_touched in that depth order (decoupled
// look-back); (3) emission of the pairs in depth order, so the pair array is
// already ordered by (depth bits, id) within every tile; (4) a stable onesweep
// sort of the K pairs on the tile bits only (ceil(tile_bits/8) passes, 2 at
// 1352×1014); (5) ids + ranges.  All of it is integer work and bit-exact.
//
// Onesweep pass (Adinets & Merrill 2022 design, written for sm_100a): one
// global histogram per digit pass computed up front (fused into the producer
// kernels), then per pass one kernel whose blocks (a) claim a tile of 2048
// keys through an atomic counter (forward progress for the look-back),
// (b) rank digits within each warp with __match_any_sync (stable: item order
// is (warp, round, lane)), (c) publish per-digit block counts and resolve the
// exclusive prefix by decoupled look-back over predecessor blocks, (d) scatter.
// No host synchronisation anywhere: K stays on the device (graph mode).
#include "common.cuh"

namespace dass {
namespace {

constexpr int SORT_THREADS = 256;
constexpr int SORT_IPT = 8;
constexpr int SORT_ITEMS = SORT_THREADS * SORT_IPT;  // 2048 keys per block
constexpr int RADIX = 256;
constexpr int MAX_PASSES = 8;  // hist slots: 0..3 depth presort, 4..7 pair sort
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1u;
constexpr unsigned long long SFLAG_AGG = 1ull << 62;
constexpr unsigned long long SFLAG_INC = 2ull << 62;
constexpr unsigned long long SVAL_MASK = (1ull << 62) - 1ull;
constexpr int NUM_COUNTERS = 16;   // 0-3 presort, 4 scan, 5-8 pair passes, 12-13 batch K
constexpr int MAX_SORT_VIEWS = 64;
#ifndef SPIN_NS
#define SPIN_NS 64
#endif

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

struct WS {
  uint64_t* dkeysA;
  uint64_t* dkeysB;
  uint32_t* offsets;
  uint64_t* pkeysA;
  uint64_t* pkeysB;
  uint32_t* hist;                  // [MAX_PASSES][256]
  uint32_t* counters;              // [NUM_COUNTERS]
  unsigned long long* scan_status; // [scan blocks]
  uint32_t* dstatus;               // [4][nblk_n][256]
  uint32_t* pstatus;               // [MAX_PASSES-4][nblk_cap][256]
  size_t ctrl_bytes;               // hist + counters (memset every call)
  size_t total;
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

WS carve(void* base, int n, int64_t cap) {
  WS w;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += align_up(bytes); return r; };
  const size_t nblk_n = (size_t)div_up(n > 0 ? n : 1, SORT_ITEMS);
  const size_t nblk_cap = (size_t)((cap + SORT_ITEMS - 1) / SORT_ITEMS) + 1;
  w.hist = (uint32_t*)take(sizeof(uint32_t) * MAX_PASSES * RADIX);
  w.counters = (uint32_t*)take(sizeof(uint32_t) * NUM_COUNTERS);
  w.ctrl_bytes = off;
  w.scan_status = (unsigned long long*)take(sizeof(unsigned long long) * nblk_n);
  w.dstatus = (uint32_t*)take(sizeof(uint32_t) * 4 * nblk_n * RADIX);
  w.pstatus = (uint32_t*)take(sizeof(uint32_t) * (MAX_PASSES - 4) * nblk_cap * RADIX);
  w.dkeysA = (uint64_t*)take(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  w.dkeysB = (uint64_t*)take(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  w.offsets = (uint32_t*)take(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  w.pkeysA = (uint64_t*)take(sizeof(uint64_t) * (size_t)(cap > 0 ? cap : 1));
  w.pkeysB = (uint64_t*)take(sizeof(uint64_t) * (size_t)(cap > 0 ? cap : 1));
  w.total = off;
  return w;
}

// ---------------------------------------------------------------- kernels --

// Depth-presort keys zbits<<32 | i (culled: all-ones depth → sorted last),
// fused with the 4 digit histograms of bits 32..63 and the clearing of the
// presort look-back status words.
__global__ void __launch_bounds__(256) presort_init_kernel(int n, const float4* __restrict__ xy_depth,
                                                          const uint32_t* __restrict__ tiles,
                                                          uint64_t* keys, uint32_t* hist,
                                                          uint32_t* dstatus, size_t dstatus_words,
                                                          unsigned long long* scan_status,
                                                          int scan_blocks) {
  __shared__ uint32_t sh[4][RADIX];
  for (int k = threadIdx.x; k < 4 * RADIX; k += blockDim.x) (&sh[0][0])[k] = 0u;
  __syncthreads();
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (size_t i = gid; i < (size_t)n; i += gstride) {
    const uint32_t zb = tiles[i] ? __float_as_uint(xy_depth[i].z) : 0xFFFFFFFFu;
    keys[i] = ((uint64_t)zb << 32) | (uint64_t)i;
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&sh[p][(zb >> (8 * p)) & 255u], 1u);
  }
  for (size_t k = gid; k < dstatus_words; k += gstride) dstatus[k] = 0u;
  for (size_t k = gid; k < (size_t)scan_blocks; k += gstride) scan_status[k] = 0ull;
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * RADIX; k += blockDim.x) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(&hist[k], v);
  }
}

// One onesweep LSD pass over bits [shift, shift+8) of 64-bit keys.
template <typename KT = uint64_t>
__global__ void __launch_bounds__(SORT_THREADS) onesweep_kernel(
    const KT* __restrict__ in, KT* __restrict__ out, int n_static,
    const uint32_t* __restrict__ n_dev, const uint32_t* __restrict__ hist, uint32_t* status,
    uint32_t* counter, int shift) {
  // per-warp digit counts, then per-warp exclusive offsets: ≤ SORT_ITEMS, so 16 bits
  // (4 KB instead of 8: a smaller footprint next to the raster CTAs of other views)
  __shared__ uint16_t s_whist[SORT_THREADS / 32][RADIX];
  __shared__ uint32_t s_gbase[RADIX];
  __shared__ uint32_t s_wsum[SORT_THREADS / 32];
  __shared__ uint32_t s_blk;
  const int t = threadIdx.x;
  const int warp = t >> 5;
  const uint32_t lane = lane_id();
  const int n = n_static >= 0 ? n_static : (n_dev[1] ? 0 : (int)n_dev[0]);
  // blocks past the end (the pair passes launch for the capacity, K is on the
  // device) leave right after their claim, before touching shared memory
  if (t == 0) s_blk = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const long long base = (long long)blk * SORT_ITEMS;
  if (base >= n) return;
  for (int k = t; k < (SORT_THREADS / 32) * RADIX; k += SORT_THREADS) (&s_whist[0][0])[k] = 0u;
  __syncthreads();

  KT keys[SORT_IPT];
  uint32_t digit[SORT_IPT];
  uint32_t rank[SORT_IPT];
  const long long wbase = base + warp * (SORT_IPT * 32);
#pragma unroll
  for (int j = 0; j < SORT_IPT; ++j) {
    const long long idx = wbase + j * 32 + lane;
    if (idx < n) {
      keys[j] = in[idx];
      digit[j] = (uint32_t)(keys[j] >> shift) & 255u;
    } else {
      keys[j] = 0;
      digit[j] = 256u;  // invalid: ranks only among invalid lanes, never scattered
    }
  }
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < SORT_IPT; ++j) {
    const uint32_t d = digit[j];
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    uint32_t pre = 0u;
    if (d < 256u) pre = s_whist[warp][d];
    __syncwarp();
    if (d < 256u) {
      rank[j] = pre + __popc(peers & lt_mask);
      const uint32_t leader = 31u - __clz(peers);
      if (lane == leader) s_whist[warp][d] = (uint16_t)(pre + __popc(peers));
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive scan over warps, block count
  uint32_t count = 0u;
#pragma unroll
  for (int w = 0; w < SORT_THREADS / 32; ++w) {
    const uint32_t c = s_whist[w][t];
    s_whist[w][t] = (uint16_t)count;
    count += c;
  }
  // exclusive scan of the global histogram over digits (digit = t)
  const uint32_t hv = hist[t];
  uint32_t incl = hv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  // decoupled look-back for digit t
  uint32_t excl = 0u;
  uint32_t* my = status + (size_t)blk * RADIX + t;
  if (blk == 0) {
    st_relaxed(my, FLAG_INC | count);
  } else {
    st_relaxed(my, FLAG_AGG | count);
    long long j = (long long)blk - 1;
    while (true) {
      const uint32_t v = ld_relaxed(status + (size_t)j * RADIX + t);
      const uint32_t f = v & ~VAL_MASK;
      if (f == 0u) {  // predecessor not published yet: back off, do not burn issue slots
        __nanosleep(SPIN_NS);
        continue;
      }
      excl += v & VAL_MASK;
      if (f == FLAG_INC) break;
      --j;
    }
    st_relaxed(my, FLAG_INC | (excl + count));
  }
  __syncthreads();
  uint32_t gofs = incl - hv;
  for (int w = 0; w < warp; ++w) gofs += s_wsum[w];
  s_gbase[t] = gofs + excl;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < SORT_IPT; ++j) {
    const uint32_t d = digit[j];
    if (d < 256u) out[s_gbase[d] + s_whist[warp][d] + rank[j]] = keys[j];
  }
}

// Exclusive scan of tiles_touched in depth order → offsets; K and the
// overflow flag → num_pairs_dev.  Single pass, decoupled look-back.
__global__ void __launch_bounds__(256) tile_scan_kernel(int n, const uint64_t* __restrict__ dkeys,
                                                       const uint32_t* __restrict__ tiles,
                                                       uint32_t* offsets,
                                                       unsigned long long* status,
                                                       uint32_t* counter, long long cap,
                                                       uint32_t* num_pairs_dev) {
  constexpr int IPT = 8;
  __shared__ unsigned long long s_w[8];
  __shared__ unsigned long long s_excl;
  __shared__ uint32_t s_blk;
  const int t = threadIdx.x;
  const uint32_t lane = lane_id();
  const int warp = t >> 5;
  if (t == 0) s_blk = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t blk = s_blk;
  const long long base = (long long)blk * (256 * IPT) + (long long)t * IPT;
  uint32_t c[IPT];
  unsigned long long tsum = 0ull;
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const long long r = base + j;
    c[j] = r < n ? tiles[(uint32_t)dkeys[r]] : 0u;
    tsum += c[j];
  }
  unsigned long long incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  unsigned long long wexcl = 0ull, btotal = 0ull;
  for (int w = 0; w < 8; ++w) {
    if (w < warp) wexcl += s_w[w];
    btotal += s_w[w];
  }
  if (t == 0) {
    unsigned long long* my = status + blk;
    unsigned long long excl = 0ull;
    if (blk == 0) {
      st_relaxed64(my, SFLAG_INC | btotal);
    } else {
      st_relaxed64(my, SFLAG_AGG | btotal);
      long long j = (long long)blk - 1;
      while (true) {
        const unsigned long long v = ld_relaxed64(status + j);
        const unsigned long long f = v & ~SVAL_MASK;
        if (f == 0ull) {
          __nanosleep(SPIN_NS);
          continue;
        }
        excl += v & SVAL_MASK;
        if (f == SFLAG_INC) break;
        --j;
      }
      st_relaxed64(my, SFLAG_INC | (excl + btotal));
    }
    s_excl = excl;
    if (blk == gridDim.x - 1) {
      const unsigned long long K = excl + btotal;
      num_pairs_dev[0] = K > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)K;
      num_pairs_dev[1] = K > (unsigned long long)cap ? 1u : 0u;
    }
  }
  __syncthreads();
  unsigned long long run = s_excl + wexcl + (incl - tsum);
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const long long r = base + j;
    if (r < n) offsets[r] = (uint32_t)run;
    run += c[j];
  }
}

// Emit pairs (tile<<32 | id) in depth order; histogram their tile digits;
// clear the pair-sort look-back status words for the blocks that will run.
// The tile of a Gaussian's local pair index j (A50, include/dass.h KEY CHAIN
// step 13): rows = 8 row spans of 16 bits (lo | hi << 8, relative to the box's
// first tile column; lo > hi: no tile) or all ones = every tile of the box, in
// (row, column) order; w = the box's width in tiles.
__device__ __forceinline__ void footprint_tile(uint4 rows, uint32_t w, uint32_t j, uint32_t& dy,
                                               uint32_t& dx) {
  if ((rows.x & rows.y & rows.z & rows.w) == 0xFFFFFFFFu) {
    dy = j / w;
    dx = j - dy * w;
    return;
  }
  const uint32_t wd[4] = {rows.x, rows.y, rows.z, rows.w};
  dy = 0;
  dx = 0;
  uint32_t rem = j;
  bool found = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t span = (wd[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
    const uint32_t lo = span & 0xFFu, hi = span >> 8;
    const uint32_t width = lo <= hi ? hi - lo + 1u : 0u;
    if (!found && rem < width) {
      dy = (uint32_t)k;
      dx = lo + rem;
      found = true;
    }
    if (!found) rem -= width;
  }
}

__global__ void __launch_bounds__(256) emit_kernel(int n, const uint64_t* __restrict__ dkeys,
                                                  const uint32_t* __restrict__ tiles,
                                                  const uint2* __restrict__ box,
                                                  const uint4* __restrict__ rowspans,
                                                  const uint32_t* __restrict__ offsets,
                                                  const uint32_t* __restrict__ num_pairs_dev,
                                                  int tiles_x, int npass, uint64_t* pkeys,
                                                  uint32_t* hist, uint32_t* pstatus,
                                                  size_t pstatus_stride, int view_n = 0,
                                                  int view_tiles = 0) {
  __shared__ uint32_t sh[MAX_PASSES - 4][RADIX];
  if (num_pairs_dev[1]) return;  // overflow: every range stays [0,0)
  for (int k = threadIdx.x; k < (MAX_PASSES - 4) * RADIX; k += blockDim.x) (&sh[0][0])[k] = 0u;
  __syncthreads();
  const uint32_t K = num_pairs_dev[0];
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t words = (size_t)div_up((int)K, SORT_ITEMS) * RADIX;
  for (int p = 0; p < npass; ++p)
    for (size_t k = gid; k < words; k += gstride) pstatus[p * pstatus_stride + k] = 0u;
  // Warp-cooperative emission: a warp owns 32 consecutive depth-ordered
  // Gaussians, whose pairs are one contiguous run of pkeys (offsets is their
  // exclusive scan), and writes that run with consecutive lanes (coalesced);
  // lane j finds its Gaussian by a binary search over the warp's inclusive
  // counts.  Histogram increments are aggregated per distinct tile.
  const uint32_t lane = threadIdx.x & 31u;
  const size_t wid = gid >> 5, nwarps = gstride >> 5;
  for (size_t base = wid * 32; base < (size_t)n; base += nwarps * 32) {
    const size_t r = base + lane;
    uint32_t id = 0, cnt = 0, w = 1;
    int tx0 = 0, ty0 = 0;
    uint4 rw = make_uint4(0u, 0u, 0u, 0u);
    if (r < (size_t)n) {
      id = (uint32_t)dkeys[r];
      cnt = tiles[id];
      if (cnt) {
        const uint2 b = box[id];
        tx0 = (int)(b.x & 0xFFFFu) / TILE;
        ty0 = (int)(b.y & 0xFFFFu) / TILE;
        w = (uint32_t)((int)(b.x >> 16) / TILE - tx0 + 1);
        rw = rowspans[id];
      }
    }
    uint32_t incl = cnt;   // inclusive scan of the counts over the warp
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (uint32_t)d) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    const uint32_t o0 = __shfl_sync(0xffffffffu, r < (size_t)n ? offsets[r] : 0u, 0);
    for (uint32_t j0 = 0; j0 < total; j0 += 32) {
      const uint32_t j = j0 + lane;
      // owner: the first lane whose inclusive count exceeds j
      uint32_t lo = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + st - 1);
        if (v <= j) lo += st;
      }
      const uint32_t owner = lo < 32 ? lo : 31;
      const uint32_t excl = __shfl_sync(0xffffffffu, incl - cnt, owner);
      const uint32_t oid = __shfl_sync(0xffffffffu, id, owner);
      const uint32_t ow = __shfl_sync(0xffffffffu, w, owner);
      const int otx0 = __shfl_sync(0xffffffffu, tx0, owner);
      const int oty0 = __shfl_sync(0xffffffffu, ty0, owner);
      const uint4 orw = make_uint4(__shfl_sync(0xffffffffu, rw.x, owner), __shfl_sync(0xffffffffu, rw.y, owner),
                                   __shfl_sync(0xffffffffu, rw.z, owner), __shfl_sync(0xffffffffu, rw.w, owner));
      const bool act = j < total;
      uint32_t tile = 0xFFFFFFFFu;
      if (act) {
        const uint32_t local = j - excl;
        uint32_t dy, dx;
        footprint_tile(orw, ow, local, dy, dx);
        tile = (uint32_t)((oty0 + (int)dy) * tiles_x + otx0 + (int)dx);
        uint32_t gid = oid;
        if (view_n > 0) {   // multi-view batch: Gaussian index v·N + i → (v·T + tile, i)
          const uint32_t v = oid / (uint32_t)view_n;
          gid = oid - v * (uint32_t)view_n;
          tile += v * (uint32_t)view_tiles;
        }
        pkeys[o0 + j] = ((uint64_t)tile << 32) | gid;
      }
      const uint32_t peers = __match_any_sync(0xffffffffu, tile);
      if (act && lane == (uint32_t)(__ffs(peers) - 1)) {
        const uint32_t c = (uint32_t)__popc(peers);
        for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(tile >> (8 * p)) & 255u], c);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < npass * RADIX; k += blockDim.x) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(&hist[4 * RADIX + k], v);
  }
}

// Multi-view batch: the pairs sorted by (v·T + tile, depth bits, i) → per view v
// its ids at sorted_ids[v·view_cap + k − off_v], view-relative tile ranges and
// (K_v, overflow_v).  off_v = first sorted position of view v (binary search on the
// monotone combined tile index).  A view with K_v > view_cap keeps empty ranges.
__global__ void __launch_bounds__(256) finalize_views_kernel(const uint64_t* __restrict__ pk,
                                                            const uint32_t* __restrict__ num_pairs_g,
                                                            int V, int T, long long view_cap,
                                                            uint32_t* ids, uint2* ranges,
                                                            uint32_t* view_pairs) {
  __shared__ uint32_t s_off[MAX_SORT_VIEWS + 1];
  const int t = threadIdx.x;
  if (num_pairs_g[1]) {   // the batch overflowed its total capacity: every view is flagged
    if (blockIdx.x == 0)
      for (int v = t; v < V; v += blockDim.x) {
        view_pairs[2 * v] = num_pairs_g[0];
        view_pairs[2 * v + 1] = 1u;
      }
    return;
  }
  const uint32_t K = num_pairs_g[0];
  for (int v = t; v <= V; v += blockDim.x) {
    const uint64_t key = (uint64_t)((uint32_t)v * (uint32_t)T) << 32;
    uint32_t lo = 0, hi = K;   // first k with pk[k] >= key
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (pk[mid] < key) lo = mid + 1; else hi = mid;
    }
    s_off[v] = lo;
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int v = t; v < V; v += blockDim.x) {
      const uint32_t kv = s_off[v + 1] - s_off[v];
      view_pairs[2 * v] = kv;
      view_pairs[2 * v + 1] = (long long)kv > view_cap ? 1u : 0u;
    }
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + t; k < K; k += gstride) {
    const uint64_t key = pk[k];
    const uint32_t ct = (uint32_t)(key >> 32);
    const uint32_t v = ct / (uint32_t)T, tile = ct - v * (uint32_t)T;
    const uint32_t off = s_off[v], end = s_off[v + 1];
    if ((long long)(end - off) > view_cap) continue;
    const uint32_t kr = (uint32_t)k - off;
    ids[(size_t)v * (size_t)view_cap + kr] = (uint32_t)key;
    uint2* r = ranges + (size_t)v * T + tile;
    if (k == off || (uint32_t)(pk[k - 1] >> 32) != ct) r->x = kr;
    if (k + 1 == end || (uint32_t)(pk[k + 1] >> 32) != ct) r->y = kr + 1;
  }
}

// ------------------------------------------------ per-view bucket sort ----
// dass_bin_sort (one view): the pairs are bucketed by tile with atomics and each
// tile's bucket is then sorted on (depth bits, id) in shared memory — no depth
// presort over N, no look-back chains ("option A").  Order of
// work: (1) count the pairs of every tile, (2) scan the counts → ranges and
// scatter cursors, (3) scatter (zbits << 32 | id) into the buckets (arbitrary
// order within a bucket), (4) sort every bucket: one warp per bucket of
// ≤ SEG_SMALL pairs (register bitonic), one CTA per bucket of ≤ SEG_LARGE
// (shared-memory bitonic), and a CTA-wide stable LSD radix sort through global
// memory beyond that.  Small CTAs throughout: the sort's kernels must find room
// next to other views' raster CTAs in the overlapped step.  The result is the contract's total order
// (tile, depth bits, id), so it is bit-exact whatever order the atomics took.
constexpr int SEG_SMALL = 512;    // one warp per bucket, 16 keys per lane in registers
constexpr int SEG_MED = 1024;     // one warp per bucket, 32 keys per lane (listed buckets)
constexpr int SEG_LARGE = 4096;   // one 256-thread CTA, 32 KB of shared memory
constexpr int SEG_GRID = 148;   // CTAs of the long- and huge-bucket kernels

struct BWS {
  uint32_t* diff;      // [ty_n][tx_n + 1] per tile row: +1 at a run's first tile, −1 past its last (zeroed)
  uint32_t* ctrl;      // [4]: [0] long, [1] huge, [2] medium buckets (zeroed every call)
  uint32_t* count;     // [T] pairs per tile (the scan's row prefix of diff)
  uint32_t* cursor;    // [T] scatter cursors (absolute positions, written by the scan)
  uint32_t* med_ids;   // [T] tiles with SEG_SMALL < count ≤ SEG_MED
  uint32_t* long_ids;  // [T] tiles with SEG_MED < count ≤ SEG_LARGE
  uint32_t* huge_ids;  // [T] tiles with count > SEG_LARGE
  uint64_t* keys;      // [cap] (zbits << 32 | id), bucketed by tile
  uint64_t* tmp;       // [cap] ping-pong of the huge-bucket radix sort
  size_t zero_bytes;   // count + ctrl
  size_t total;
};

// diff_entries: tiles_y·(tiles_x + 1) at launch; the size query, which knows only
// T = tiles_x·tiles_y, takes the bound 2T (tiles_y ≤ T), so a launch's layout
// never outgrows the queried workspace.
BWS carve_bucket(void* base, size_t diff_entries, size_t num_tiles, int64_t cap) {
  BWS w;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += align_up(bytes); return r; };
  const size_t T = num_tiles > 0 ? num_tiles : 1;
  const size_t c = (size_t)(cap > 0 ? cap : 1);
  w.diff = (uint32_t*)(p ? p : nullptr);
  off += sizeof(uint32_t) * (diff_entries > 0 ? diff_entries : 1);
  w.ctrl = (uint32_t*)(p ? p + off : nullptr);           // diff and ctrl adjacent: one memset
  off += sizeof(uint32_t) * 4;
  w.zero_bytes = off;
  off = align_up(off);
  w.count = (uint32_t*)take(sizeof(uint32_t) * T);
  w.cursor = (uint32_t*)take(sizeof(uint32_t) * T);
  w.med_ids = (uint32_t*)take(sizeof(uint32_t) * T);
  w.long_ids = (uint32_t*)take(sizeof(uint32_t) * T);
  w.huge_ids = (uint32_t*)take(sizeof(uint32_t) * T);
  w.keys = (uint64_t*)take(sizeof(uint64_t) * c);
  w.tmp = (uint64_t*)take(sizeof(uint64_t) * c);
  w.total = off;
  return w;
}

// The pairs of Gaussians [0, n) in index order, expanded warp-cooperatively (a
// warp owns 32 consecutive Gaussians and hands out their pairs to consecutive
// lanes; lane j finds its Gaussian by a binary search over the warp's inclusive
// counts).  f(act, tile, id, zbits) is called by all 32 lanes (warp-synchronous);
// inactive lanes get tile = 0xFFFFFFFF.
template <class F>
__device__ __forceinline__ void expand_pairs(int n, const float4* __restrict__ xy_depth,
                                             const uint32_t* __restrict__ tiles,
                                             const uint2* __restrict__ box,
                                             const uint4* __restrict__ rowspans, int tiles_x, F&& f) {
  const uint32_t lane = threadIdx.x & 31u;
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t wid = gid >> 5, nwarps = gstride >> 5;
  for (size_t base = wid * 32; base < (size_t)n; base += nwarps * 32) {
    const size_t i = base + lane;
    uint32_t cnt = 0, w = 1, zb = 0;
    int tx0 = 0, ty0 = 0;
    uint4 rw = make_uint4(0u, 0u, 0u, 0u);
    if (i < (size_t)n) {
      cnt = tiles[i];
      if (cnt) {
        const uint2 b = box[i];
        tx0 = (int)(b.x & 0xFFFFu) / TILE;
        ty0 = (int)(b.y & 0xFFFFu) / TILE;
        w = (uint32_t)((int)(b.x >> 16) / TILE - tx0 + 1);
        rw = rowspans[i];
        zb = __float_as_uint(xy_depth[i].z);
      }
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= (uint32_t)d) incl += u;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    for (uint32_t j0 = 0; j0 < total; j0 += 32) {
      const uint32_t j = j0 + lane;
      uint32_t lo = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, lo + st - 1);
        if (v <= j) lo += st;
      }
      const uint32_t owner = lo < 32 ? lo : 31;
      const uint32_t excl = __shfl_sync(0xffffffffu, incl - cnt, owner);
      const uint32_t ow = __shfl_sync(0xffffffffu, w, owner);
      const int otx0 = __shfl_sync(0xffffffffu, tx0, owner);
      const int oty0 = __shfl_sync(0xffffffffu, ty0, owner);
      const uint32_t ozb = __shfl_sync(0xffffffffu, zb, owner);
      const uint4 orw = make_uint4(__shfl_sync(0xffffffffu, rw.x, owner), __shfl_sync(0xffffffffu, rw.y, owner),
                                   __shfl_sync(0xffffffffu, rw.z, owner), __shfl_sync(0xffffffffu, rw.w, owner));
      const bool act = j < total;
      uint32_t tile = 0xFFFFFFFFu;
      if (act) {
        uint32_t dy, dx;
        footprint_tile(orw, ow, j - excl, dy, dx);
        tile = (uint32_t)((oty0 + (int)dy) * tiles_x + otx0 + (int)dx);
      }
      f(act, tile, (uint32_t)(base + owner), ozb);
    }
  }
}

// Pair counts per tile as run-length differences: every footprint row is one run
// of consecutive tiles [lo, hi] (KEY CHAIN step 13; a full box: every row of the
// box), so one thread per Gaussian adds +1 at lo and −1 at hi + 1 of the row's
// difference array — two atomics per row instead of one per pair.
__global__ void __launch_bounds__(256) bucket_count_kernel(int n, const uint32_t* __restrict__ tiles,
                                                           const uint2* __restrict__ box,
                                                           const uint4* __restrict__ rowspans,
                                                           int tiles_x, uint32_t* diff) {
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  const int stride = tiles_x + 1;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (size_t)n; i += gstride) {
    if (!tiles[i]) continue;
    const uint2 b = box[i];
    const int tx0 = (int)(b.x & 0xFFFFu) / TILE, tx1 = (int)(b.x >> 16) / TILE;
    const int ty0 = (int)(b.y & 0xFFFFu) / TILE, ty1 = (int)(b.y >> 16) / TILE;
    const uint4 rw = rowspans[i];
    if ((rw.x & rw.y & rw.z & rw.w) == 0xFFFFFFFFu) {   // every tile of the box
      for (int ty = ty0; ty <= ty1; ++ty) {
        atomicAdd(&diff[ty * stride + tx0], 1u);
        atomicAdd(&diff[ty * stride + tx1 + 1], 0xFFFFFFFFu);
      }
      continue;
    }
    const uint32_t wd[4] = {rw.x, rw.y, rw.z, rw.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t span = (wd[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
      const uint32_t lo = span & 0xFFu, hi = span >> 8;
      if (lo <= hi) {
        atomicAdd(&diff[(ty0 + k) * stride + tx0 + (int)lo], 1u);
        atomicAdd(&diff[(ty0 + k) * stride + tx0 + (int)hi + 1], 0xFFFFFFFFu);
      }
    }
  }
}

// One CTA: K = Σ counts → num_pairs_dev (overflow: stop, every range stays [0,0));
// else the exclusive scan → ranges (empty tile [0,0)), cursors, and the lists of
// long and huge buckets.
__global__ void __launch_bounds__(1024) bucket_scan_kernel(int tiles_x, int tiles_y,
                                                           const uint32_t* __restrict__ diff,
                                                           uint32_t* count, long long cap, uint32_t* cursor,
                                                           uint2* ranges, uint32_t* num_pairs_dev,
                                                           uint32_t* ctrl, uint32_t* med_ids,
                                                           uint32_t* long_ids, uint32_t* huge_ids) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const int t = threadIdx.x;
  const uint32_t lane = lane_id();
  const int warp = t >> 5;
  const int T = tiles_x * tiles_y;
  // counts = the row prefix of the difference arrays (a warp per tile row)
  for (int row = warp; row < tiles_y; row += (int)(blockDim.x >> 5)) {
    uint32_t carry = 0;
    for (int c0 = 0; c0 < tiles_x; c0 += 32) {
      const int c = c0 + (int)lane;
      uint32_t v = c < tiles_x ? diff[row * (tiles_x + 1) + c] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (uint32_t)o) v += y;
      }
      v += carry;
      if (c < tiles_x) count[row * tiles_x + c] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  unsigned long long part = 0;
  for (int k = t; k < T; k += blockDim.x) part += count[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) s_w[warp] = part;
  __syncthreads();
  if (t == 0) {
    unsigned long long K = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) K += s_w[w];
    num_pairs_dev[0] = K > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)K;
    num_pairs_dev[1] = K > (unsigned long long)cap ? 1u : 0u;
    s_carry = K > (unsigned long long)cap ? ~0ull : 0ull;
  }
  __syncthreads();
  if (s_carry == ~0ull) return;   // overflow
  __syncthreads();
  for (int k0 = 0; k0 < T; k0 += blockDim.x) {
    const int k = k0 + t;
    const uint32_t c = k < T ? count[k] : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    unsigned long long wpre = s_carry;
    for (int w = 0; w < warp; ++w) wpre += s_w[w];
    const uint32_t start = (uint32_t)(wpre + incl - c);   // < cap < 2^30
    if (k < T) {
      cursor[k] = start;
      if (c) {
        ranges[k] = make_uint2(start, start + c);
        if (c > (uint32_t)SEG_LARGE) huge_ids[atomicAdd(&ctrl[1], 1u)] = (uint32_t)k;
        else if (c > (uint32_t)SEG_MED) long_ids[atomicAdd(&ctrl[0], 1u)] = (uint32_t)k;
        else if (c > (uint32_t)SEG_SMALL) med_ids[atomicAdd(&ctrl[2], 1u)] = (uint32_t)k;
      }
    }
    __syncthreads();
    if (t == (int)blockDim.x - 1) s_carry = wpre + incl;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) bucket_scatter_kernel(int n, const float4* __restrict__ xy_depth,
                                                             const uint32_t* __restrict__ tiles,
                                                             const uint2* __restrict__ box,
                                                             const uint4* __restrict__ rowspans,
                                                             int tiles_x, const uint32_t* __restrict__ num_pairs_dev,
                                                             uint32_t* cursor, uint64_t* keys) {
  if (num_pairs_dev[1]) return;
  const uint32_t lt_mask = (1u << lane_id()) - 1u;
  expand_pairs(n, xy_depth, tiles, box, rowspans, tiles_x,
               [&](bool act, uint32_t tile, uint32_t id, uint32_t zb) {
                 const uint32_t peers = __match_any_sync(0xffffffffu, tile);
                 const uint32_t leader = (uint32_t)(__ffs(peers) - 1);
                 uint32_t b = 0;
                 if (act && lane_id() == leader) b = atomicAdd(&cursor[tile], (uint32_t)__popc(peers));
                 b = __shfl_sync(0xffffffffu, b, leader);
                 if (act) keys[b + __popc(peers & lt_mask)] = ((uint64_t)zb << 32) | id;
               });
}

// Bitonic sort of s[0, P) (P a power of two ≥ 2) by the threads [0, nthr) of
// `sync`'s group: P/2 compare-exchanges per stage, spread over the threads.
template <class Sync>
__device__ __forceinline__ void bitonic_shared(uint64_t* s, uint32_t P, uint32_t tid, uint32_t nthr,
                                               Sync&& sync) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t q = tid; q < (P >> 1); q += nthr) {
        const uint32_t i = ((q & ~(j - 1u)) << 1) | (q & (j - 1u));   // lower index of (i, i + j)
        const uint64_t a = s[i], b = s[i + j];
        const bool up = (i & k) == 0;
        if ((a > b) == up) { s[i] = b; s[i + j] = a; }
      }
      sync();
    }
  }
}

__device__ __forceinline__ void write_bucket(const uint64_t* s, uint32_t cnt, uint32_t start, uint32_t tile,
                                             uint32_t tid, uint32_t nthr, uint32_t* ids,
                                             uint64_t* sorted_keys) {
  for (uint32_t k = tid; k < cnt; k += nthr) {
    const uint64_t key = s[k];
    ids[start + k] = (uint32_t)key;
    if (sorted_keys) sorted_keys[start + k] = ((uint64_t)tile << 32) | (key >> 32);
  }
}

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) { return x <= 2u ? 2u : 1u << (32 - __clz(x - 1u)); }

// Bitonic sort of 32·E keys held in registers, blocked layout: lane l holds the
// keys of positions l·E … l·E + E − 1.  Exchange distances j ≥ E pair lane l with
// lane l ^ (j/E) through shuffles (one runtime-parameterised stage); j < E stay
// in the lane's registers (one compile-time stage per j, so no register array is
// indexed dynamically).  The k and j loops are not unrolled: the fully unrolled
// network of the larger E overflowed the instruction cache.
template <int E>
__device__ __forceinline__ void cross_stage(uint64_t (&x)[E], uint32_t lane, uint32_t k, uint32_t lm) {
  const bool lower = (lane & lm) == 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool up = ((lane * E + e) & k) == 0;
    const uint64_t o = __shfl_xor_sync(0xffffffffu, x[e], lm);
    const uint64_t lo = x[e] < o ? x[e] : o, hi = x[e] < o ? o : x[e];
    x[e] = lower == up ? lo : hi;
  }
}
template <int E, int J>
__device__ __forceinline__ void reg_stage(uint64_t (&x)[E], uint32_t lane, uint32_t k) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & J) == 0) {
      const int f = e | J;
      const bool up = ((lane * E + e) & k) == 0;
      const uint64_t a = x[e], b = x[f];
      const bool sw = (a > b) == up;
      x[e] = sw ? b : a;
      x[f] = sw ? a : b;
    }
  }
}
template <int E>
__device__ __forceinline__ void warp_bitonic(uint64_t (&x)[E], uint32_t lane) {
  static_assert(E >= 1 && E <= 32 && (E & (E - 1)) == 0, "E: a power of two ≤ 32");
#pragma unroll 1
  for (uint32_t k = 2; k <= 32u * E; k <<= 1) {
    uint32_t j = k >> 1;
#pragma unroll 1
    for (; j >= (uint32_t)E; j >>= 1) cross_stage<E>(x, lane, k, j / E);
#pragma unroll 1
    for (; j > 0; j >>= 1) {
      if constexpr (E > 16) { if (j == 16) reg_stage<E, 16>(x, lane, k); }
      if constexpr (E > 8) { if (j == 8) reg_stage<E, 8>(x, lane, k); }
      if constexpr (E > 4) { if (j == 4) reg_stage<E, 4>(x, lane, k); }
      if constexpr (E > 2) { if (j == 2) reg_stage<E, 2>(x, lane, k); }
      if constexpr (E > 1) { if (j == 1) reg_stage<E, 1>(x, lane, k); }
    }
  }
}

template <int E>
__device__ __forceinline__ void sort_bucket_warp(const uint64_t* __restrict__ keys, uint32_t cnt,
                                                 uint32_t start, uint32_t tile, uint32_t lane,
                                                 uint32_t* ids, uint64_t* sorted_keys) {
  uint64_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t k = lane * E + e;
    x[e] = k < cnt ? keys[start + k] : ~0ull;
  }
  warp_bitonic<E>(x, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t k = lane * E + e;
    if (k < cnt) {
      ids[start + k] = (uint32_t)x[e];
      if (sorted_keys) sorted_keys[start + k] = ((uint64_t)tile << 32) | (x[e] >> 32);
    }
  }
}

// One warp per bucket of ≤ SEG_SMALL pairs (register bitonic of 32·E ≥ count keys).
__global__ void __launch_bounds__(32) seg_sort_small_kernel(const uint2* __restrict__ ranges,
                                                            const uint32_t* __restrict__ num_pairs_dev,
                                                            const uint64_t* __restrict__ keys, uint32_t* ids,
                                                            uint64_t* sorted_keys) {
  if (num_pairs_dev[1]) return;
  const uint32_t tile = blockIdx.x;
  const uint2 r = ranges[tile];
  const uint32_t cnt = r.y - r.x;
  if (cnt == 0 || cnt > (uint32_t)SEG_SMALL) return;
  const uint32_t lane = threadIdx.x;
  if (cnt <= 32) sort_bucket_warp<1>(keys, cnt, r.x, tile, lane, ids, sorted_keys);
  else if (cnt <= 64) sort_bucket_warp<2>(keys, cnt, r.x, tile, lane, ids, sorted_keys);
  else if (cnt <= 128) sort_bucket_warp<4>(keys, cnt, r.x, tile, lane, ids, sorted_keys);
  else if (cnt <= 256) sort_bucket_warp<8>(keys, cnt, r.x, tile, lane, ids, sorted_keys);
  else sort_bucket_warp<16>(keys, cnt, r.x, tile, lane, ids, sorted_keys);
}

// One warp per listed bucket of SEG_SMALL < count ≤ SEG_MED (32 keys per lane;
// a kernel of its own so the small-bucket kernel keeps its lower register count).
__global__ void __launch_bounds__(32) seg_sort_med_kernel(const uint2* __restrict__ ranges,
                                                          const uint32_t* __restrict__ num_pairs_dev,
                                                          const uint32_t* __restrict__ ctrl,
                                                          const uint32_t* __restrict__ med_ids,
                                                          const uint64_t* __restrict__ keys, uint32_t* ids,
                                                          uint64_t* sorted_keys) {
  if (num_pairs_dev[1]) return;
  const uint32_t nm = ctrl[2];
  for (uint32_t q = blockIdx.x; q < nm; q += gridDim.x) {
    const uint32_t tile = med_ids[q];
    const uint2 r = ranges[tile];
    sort_bucket_warp<32>(keys, r.y - r.x, r.x, tile, threadIdx.x, ids, sorted_keys);
  }
}

// One 256-thread CTA per bucket of SEG_MED < count ≤ SEG_LARGE (listed by the scan).
__global__ void __launch_bounds__(256) seg_sort_large_kernel(const uint2* __restrict__ ranges,
                                                             const uint32_t* __restrict__ num_pairs_dev,
                                                             const uint32_t* __restrict__ ctrl,
                                                             const uint32_t* __restrict__ long_ids,
                                                             const uint64_t* __restrict__ keys, uint32_t* ids,
                                                             uint64_t* sorted_keys) {
  __shared__ uint64_t s_dyn[SEG_LARGE];
  if (num_pairs_dev[1]) return;
  const uint32_t nl = ctrl[0];
  for (uint32_t q = blockIdx.x; q < nl; q += gridDim.x) {
    const uint32_t tile = long_ids[q];
    const uint2 r = ranges[tile];
    const uint32_t cnt = r.y - r.x;
    const uint32_t P = pow2_ceil(cnt);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < P; k += blockDim.x) s_dyn[k] = k < cnt ? keys[r.x + k] : ~0ull;
    __syncthreads();
    bitonic_shared(s_dyn, P, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    write_bucket(s_dyn, cnt, r.x, tile, threadIdx.x, blockDim.x, ids, sorted_keys);
  }
}

// One 256-thread CTA per bucket of more than SEG_LARGE pairs: a stable LSD radix
// sort of the bucket through global memory (keys ↔ tmp), 8 bits per pass over the
// id bits and the 32 depth bits, each pass in chunks of 256 keys ranked with
// __match_any_sync (item order = thread order, so every pass is stable).
__global__ void __launch_bounds__(256) seg_sort_huge_kernel(const uint2* __restrict__ ranges,
                                                             const uint32_t* __restrict__ num_pairs_dev,
                                                             const uint32_t* __restrict__ ctrl,
                                                             const uint32_t* __restrict__ huge_ids,
                                                             int id_bits, uint64_t* keys, uint64_t* tmp,
                                                             uint32_t* ids, uint64_t* sorted_keys) {
  __shared__ uint32_t s_hist[RADIX];
  __shared__ uint32_t s_base[RADIX];
  __shared__ uint32_t s_tot[RADIX];
  __shared__ uint16_t s_w[8][RADIX];
  if (num_pairs_dev[1]) return;
  const uint32_t nh = ctrl[1];
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  for (uint32_t q = blockIdx.x; q < nh; q += gridDim.x) {
    const uint32_t tile = huge_ids[q];
    const uint2 r = ranges[tile];
    const uint32_t cnt = r.y - r.x;
    uint64_t* src = keys + r.x;
    uint64_t* dst = tmp + r.x;
    for (int shift = 0; shift < 64; shift += 8) {
      if (shift < 32 && shift >= id_bits) continue;   // id bits above the largest id are all zero
      __syncthreads();
      if (t < RADIX) s_hist[t] = 0u;
      __syncthreads();
      for (uint32_t k = t; k < cnt; k += blockDim.x) atomicAdd(&s_hist[(uint32_t)(src[k] >> shift) & 255u], 1u);
      __syncthreads();
      if (t == 0) {
        uint32_t run = 0;
        for (int d = 0; d < RADIX; ++d) { s_base[d] = run; run += s_hist[d]; }
      }
      __syncthreads();
      for (uint32_t c0 = 0; c0 < cnt; c0 += blockDim.x) {
        const uint32_t k = c0 + t;
        const bool valid = k < cnt;
        const uint64_t key = valid ? src[k] : 0ull;
        const uint32_t d = valid ? ((uint32_t)(key >> shift) & 255u) : 256u;
        for (uint32_t z = t; z < 8 * RADIX; z += blockDim.x) (&s_w[0][0])[z] = 0u;
        __syncthreads();
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid && lane == (uint32_t)(__ffs(peers) - 1)) s_w[warp][d] = (uint16_t)__popc(peers);
        __syncthreads();
        if (t < RADIX) {   // exclusive over warps, per digit
          uint32_t run = 0;
          for (int w = 0; w < 8; ++w) { const uint32_t c = s_w[w][t]; s_w[w][t] = (uint16_t)run; run += c; }
          s_tot[t] = run;
        }
        __syncthreads();
        if (valid) dst[s_base[d] + s_w[warp][d] + __popc(peers & lt_mask)] = key;
        __syncthreads();
        if (t < RADIX) s_base[t] += s_tot[t];
      }
      uint64_t* x = src; src = dst; dst = x;
    }
    __syncthreads();
    for (uint32_t k = t; k < cnt; k += blockDim.x) {
      const uint64_t key = src[k];
      ids[r.x + k] = (uint32_t)key;
      if (sorted_keys) sorted_keys[r.x + k] = ((uint64_t)tile << 32) | (key >> 32);
    }
  }
}

}  // namespace

size_t binsort_workspace(int n, int num_tiles, int64_t capacity) {
  (void)n;
  const size_t T = (size_t)(num_tiles > 0 ? num_tiles : 1);
  return carve_bucket(nullptr, 2 * T, T, capacity).total;
}

cudaError_t launch_binsort(const CamParams& cam, int n, const float4* xy_depth, const uint2* box,
                           const uint4* rows, const uint32_t* tiles, void* ws_ptr, int64_t capacity,
                           uint64_t* sorted_keys, uint32_t* sorted_ids, uint2* ranges,
                           uint32_t* num_pairs_dev, cudaStream_t s) {
  const int num_tiles = cam.tiles_x * cam.tiles_y;
  BWS w = carve_bucket(ws_ptr, (size_t)cam.tiles_y * (size_t)(cam.tiles_x + 1), (size_t)num_tiles,
                       capacity);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)num_tiles, s))) return e;
  if ((e = cudaMemsetAsync(w.diff, 0, w.zero_bytes, s))) return e;
  if (n == 0) return cudaMemsetAsync(num_pairs_dev, 0, 2 * sizeof(uint32_t), s);
  const int grid_n = div_up(n, 256) < 148 * 8 ? div_up(n, 256) : 148 * 8;
  bucket_count_kernel<<<grid_n, 256, 0, s>>>(n, tiles, box, rows, cam.tiles_x, w.diff);
  launch_counted();
  bucket_scan_kernel<<<1, 1024, 0, s>>>(cam.tiles_x, cam.tiles_y, w.diff, w.count, (long long)capacity,
                                        w.cursor, ranges, num_pairs_dev, w.ctrl, w.med_ids, w.long_ids,
                                        w.huge_ids);
  launch_counted();
  bucket_scatter_kernel<<<grid_n, 256, 0, s>>>(n, xy_depth, tiles, box, rows, cam.tiles_x,
                                               num_pairs_dev, w.cursor, w.keys);
  launch_counted();
  seg_sort_small_kernel<<<num_tiles, 32, 0, s>>>(ranges, num_pairs_dev, w.keys, sorted_ids, sorted_keys);
  launch_counted();
  seg_sort_med_kernel<<<4 * SEG_GRID, 32, 0, s>>>(ranges, num_pairs_dev, w.ctrl, w.med_ids, w.keys,
                                                  sorted_ids, sorted_keys);
  launch_counted();
  seg_sort_large_kernel<<<SEG_GRID, 256, 0, s>>>(ranges, num_pairs_dev, w.ctrl, w.long_ids, w.keys,
                                                 sorted_ids, sorted_keys);
  launch_counted();
  const int id_bits = n > 1 ? 32 - __builtin_clz((unsigned)(n - 1)) : 1;
  seg_sort_huge_kernel<<<SEG_GRID, 256, 0, s>>>(ranges, num_pairs_dev, w.ctrl, w.huge_ids, id_bits,
                                                w.keys, w.tmp, sorted_ids, sorted_keys);
  launch_counted();
  return cudaGetLastError();
}

size_t binsort_views_workspace(int V, int n, int64_t view_capacity) {
  return carve(nullptr, V * n, (int64_t)V * view_capacity).total;
}

// V views at once (same image size): one depth presort over the V·N (view,
// Gaussian) keys, one emission, one sort of all pairs on the combined tile
// index v·T + tile, per-view outputs.  Equal to V dass_bin_sort calls
// (bit-exact) with a handful of large kernels instead of V chains of small,
// latency-bound ones.
cudaError_t launch_binsort_views(const CamParams& cam, int V, int n, const float4* xy_depth,
                                 const uint2* box, const uint4* rows, const uint32_t* tiles,
                                 void* ws_ptr,
                                 int64_t view_capacity, uint32_t* sorted_ids, uint2* ranges,
                                 uint32_t* view_pairs, cudaStream_t s) {
  const int T = cam.tiles_x * cam.tiles_y;
  const int nn = V * n;
  const int64_t cap = (int64_t)V * view_capacity;
  WS w = carve(ws_ptr, nn, cap);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)V * T, s))) return e;
  if ((e = cudaMemsetAsync(w.hist, 0, w.ctrl_bytes, s))) return e;
  if (nn == 0) return cudaMemsetAsync(view_pairs, 0, 2 * sizeof(uint32_t) * (size_t)V, s);
  uint32_t* kg = w.counters + 12;   // (K_total, overflow) of the batch
  const int vt = V * T;
  const int ct_bits = vt > 1 ? 32 - __builtin_clz((unsigned)(vt - 1)) : 0;
  const int npass = (ct_bits + 7) / 8;
  if (npass > MAX_PASSES - 4) return cudaErrorInvalidValue;
  const int nblk_n = div_up(nn, SORT_ITEMS);
  const size_t nblk_cap = (size_t)((cap + SORT_ITEMS - 1) / SORT_ITEMS) + 1;
  const int grid_n = div_up(nn, 256) < 148 * 8 ? div_up(nn, 256) : 148 * 8;
  presort_init_kernel<<<grid_n, 256, 0, s>>>(nn, xy_depth, tiles, w.dkeysA, w.hist, w.dstatus,
                                             (size_t)4 * nblk_n * RADIX, w.scan_status, nblk_n);
  launch_counted();
  uint64_t* a = w.dkeysA;
  uint64_t* b = w.dkeysB;
  for (int p = 0; p < 4; ++p) {
    onesweep_kernel<uint64_t><<<nblk_n, SORT_THREADS, 0, s>>>(a, b, nn, nullptr, w.hist + p * RADIX,
                                                    w.dstatus + (size_t)p * nblk_n * RADIX,
                                                    w.counters + p, 32 + 8 * p);
    launch_counted();
    uint64_t* tmp = a; a = b; b = tmp;
  }
  tile_scan_kernel<<<nblk_n, 256, 0, s>>>(nn, a, tiles, w.offsets, w.scan_status, w.counters + 4,
                                          (long long)cap, kg);
  launch_counted();
  emit_kernel<<<grid_n, 256, 0, s>>>(nn, a, tiles, box, rows, w.offsets, kg, cam.tiles_x, npass, w.pkeysA,
                                     w.hist, w.pstatus, nblk_cap * RADIX, n, T);
  launch_counted();
  uint64_t* pa = w.pkeysA;
  uint64_t* pb = w.pkeysB;
  for (int p = 0; p < npass; ++p) {
    onesweep_kernel<uint64_t><<<(int)nblk_cap, SORT_THREADS, 0, s>>>(pa, pb, -1, kg, w.hist + (4 + p) * RADIX,
                                                           w.pstatus + (size_t)p * nblk_cap * RADIX,
                                                           w.counters + 5 + p, 32 + 8 * p);
    launch_counted();
    uint64_t* tmp = pa; pa = pb; pb = tmp;
  }
  finalize_views_kernel<<<148 * 8, 256, 0, s>>>(pa, kg, V, T, (long long)view_capacity, sorted_ids,
                                                ranges, view_pairs);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
