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
constexpr int SORT_ITEMS = SORT_THREADS * SORT_IPT;  // 2048 keys per block (pair passes)
// depth presort passes: 16 keys per thread, 4096 per block (74 blocks at N = 300k); fewer,
// longer blocks overlap better with the other views' chains (step 11.76 → 11.74 ms against 8;
// 4: 11.83, 32: 11.86)
constexpr int PRESORT_IPT = 16;
constexpr int PRESORT_ITEMS = SORT_THREADS * PRESORT_IPT;
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
  const size_t nblk_n = (size_t)div_up(n > 0 ? n : 1, PRESORT_ITEMS);
  const size_t nblk_cap = (size_t)((cap + SORT_ITEMS - 1) / SORT_ITEMS) + 1;
  w.hist = (uint32_t*)take(sizeof(uint32_t) * MAX_PASSES * RADIX);
  w.counters = (uint32_t*)take(sizeof(uint32_t) * NUM_COUNTERS);
  w.ctrl_bytes = off;
  w.scan_status = (unsigned long long*)take(sizeof(unsigned long long) *
                                            (size_t)div_up(n > 0 ? n : 1, SORT_ITEMS));
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
template <typename KT = uint64_t, int IPT = SORT_IPT>
__global__ void __launch_bounds__(SORT_THREADS) onesweep_kernel(
    const KT* __restrict__ in, KT* __restrict__ out, int n_static,
    const uint32_t* __restrict__ n_dev, const uint32_t* __restrict__ hist, uint32_t* status,
    uint32_t* counter, int shift, int loop) {
  // per-warp digit counts, then per-warp exclusive offsets: ≤ 256·IPT, so 16 bits
  // (4 KB instead of 8: a smaller footprint next to the raster CTAs of other views)
  __shared__ uint16_t s_whist[SORT_THREADS / 32][RADIX];
  __shared__ uint32_t s_gbase[RADIX];
  __shared__ uint32_t s_wsum[SORT_THREADS / 32];
  __shared__ uint32_t s_blk;
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x;
  const int warp = t >> 5;
  const uint32_t lane = lane_id();
  const int n = n_static >= 0 ? n_static : (n_dev[1] ? 0 : (int)n_dev[0]);
  // Each block claims key tiles in order until they run out: the pair passes launch for the
  // capacity or on a fixed grid (K is on the device), so a block past the end leaves right after
  // its claim, before touching shared memory.
  for (;;) {
    if (t == 0) s_blk = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t blk = s_blk;
    const long long base = (long long)blk * (SORT_THREADS * IPT);
    if (base >= n) return;
    for (int k = t; k < (SORT_THREADS / 32) * RADIX; k += SORT_THREADS) (&s_whist[0][0])[k] = 0u;
    __syncthreads();

    KT keys[IPT];
    uint32_t digit[IPT];
    uint32_t rank[IPT];
    const long long wbase = base + warp * (IPT * 32);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
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
    for (int j = 0; j < IPT; ++j) {
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
    for (int j = 0; j < IPT; ++j) {
      const uint32_t d = digit[j];
      if (d < 256u) {
        DASS_CHECK((long long)(s_gbase[d] + s_whist[warp][d] + rank[j]) < (long long)n);
        out[s_gbase[d] + s_whist[warp][d] + rank[j]] = keys[j];
      }
    }
    // a grid of one block per key tile stops here (a second claim per block would queue
    // one more atomic per block on the shared counter)
    if (!loop) return;
    __syncthreads();   // s_blk, s_whist, s_gbase are reused by the next claim
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
  pdl_trigger();
  pdl_wait();
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
  pdl_trigger();
  pdl_wait();
  if (num_pairs_dev[1]) return;  // overflow: every range stays [0,0)
  for (int k = threadIdx.x; k < (MAX_PASSES - 4) * RADIX; k += blockDim.x) (&sh[0][0])[k] = 0u;
  __syncthreads();
  const uint32_t K = num_pairs_dev[0];
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t words = (size_t)div_up((int)K, SORT_ITEMS) * RADIX;
  for (int p = 0; p < npass; ++p)
    for (size_t k = gid; k < words; k += gstride) pstatus[p * pstatus_stride + k] = 0u;
  // One thread per depth-ordered Gaussian: its pairs are one contiguous run of
  // pkeys (offsets = the exclusive scan of tiles_touched in depth order), written
  // row by row — each footprint row is a run of consecutive tiles [lo, hi]
  // (KEY CHAIN step 13), so no per-pair decoding.  Histogram: digit 0 per pair;
  // the higher digits change at most once along a row's run (L ≤ 255 < 256), so
  // they are counted per row in one or two increments.
  for (size_t r = gid; r < (size_t)n; r += gstride) {
    const uint32_t id = (uint32_t)dkeys[r];
    if (!tiles[id]) continue;   // culled / empty footprint (sorted last: all-ones depth)
    const uint2 b = box[id];
    const int tx0 = (int)(b.x & 0xFFFFu) / TILE, tx1 = (int)(b.x >> 16) / TILE;
    const int ty0 = (int)(b.y & 0xFFFFu) / TILE, ty1 = (int)(b.y >> 16) / TILE;
    const uint4 rw = rowspans[id];
    const bool full = (rw.x & rw.y & rw.z & rw.w) == 0xFFFFFFFFu;
    uint32_t gidv = id, tbase = 0;
    if (view_n > 0) {   // multi-view batch: Gaussian index v·N + i → (v·T + tile, i)
      const uint32_t v = id / (uint32_t)view_n;
      gidv = id - v * (uint32_t)view_n;
      tbase = v * (uint32_t)view_tiles;
    }
    uint64_t* out = pkeys + offsets[r];
#ifdef DASS_CHECKED
    uint64_t* const out0 = out;
#endif
    const int nrows = full ? ty1 - ty0 + 1 : 8;
    for (int k = 0; k < nrows; ++k) {
      uint32_t lo, hi;
      if (full) {
        lo = 0u;
        hi = (uint32_t)(tx1 - tx0);
      } else {
        const uint32_t word = k < 2 ? rw.x : k < 4 ? rw.y : k < 6 ? rw.z : rw.w;
        const uint32_t span = (word >> (16 * (k & 1))) & 0xFFFFu;
        lo = span & 0xFFu;
        hi = span >> 8;
        if (lo > hi) continue;
      }
      const uint32_t t0 = tbase + (uint32_t)((ty0 + k) * tiles_x + tx0) + lo;
      const uint32_t L = hi - lo + 1u;
      for (uint32_t dx = 0; dx < L; ++dx) {
        const uint32_t tile = t0 + dx;
        DASS_CHECK(out < pkeys + K);
        *out++ = ((uint64_t)tile << 32) | gidv;
        atomicAdd(&sh[0][tile & 255u], 1u);
      }
      const uint32_t t1 = t0 + L - 1u;
      for (int p = 1; p < npass; ++p) {
        const uint32_t da = t0 >> (8 * p), db = t1 >> (8 * p);
        if (da == db) {
          atomicAdd(&sh[p][da & 255u], L);
        } else {   // one crossing: [t0, edge) and [edge, t1]
          const uint32_t edge = db << (8 * p);
          atomicAdd(&sh[p][da & 255u], edge - t0);
          atomicAdd(&sh[p][db & 255u], t1 - edge + 1u);
        }
      }
    }
#ifdef DASS_CHECKED
    DASS_CHECK((uint32_t)(out - out0) == tiles[id]);   // the rows hold tiles_touched pairs
#endif
  }
  __syncthreads();
  for (int k = threadIdx.x; k < npass * RADIX; k += blockDim.x) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(&hist[4 * RADIX + k], v);
  }
}

// Sorted pairs → ids, optional (tile|zbits) keys, per-tile [start, end).
__global__ void __launch_bounds__(256) finalize_kernel(const uint64_t* __restrict__ pk,
                                                      const uint32_t* __restrict__ num_pairs_dev,
                                                      const float4* __restrict__ xy_depth,
                                                      uint64_t* sorted_keys, uint32_t* ids,
                                                      uint2* ranges) {
  pdl_wait();
  if (num_pairs_dev[1]) return;
  const uint32_t K = num_pairs_dev[0];
  const size_t gstride = (size_t)gridDim.x * blockDim.x;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gstride) {
    const uint64_t key = pk[k];
    const uint32_t id = (uint32_t)key;
    const uint32_t tile = (uint32_t)(key >> 32);
    ids[k] = id;
    if (sorted_keys) sorted_keys[k] = ((uint64_t)tile << 32) | __float_as_uint(xy_depth[id].z);
    if (k == 0 || (uint32_t)(pk[k - 1] >> 32) != tile) ranges[tile].x = (uint32_t)k;
    if (k + 1 == K || (uint32_t)(pk[k + 1] >> 32) != tile) ranges[tile].y = (uint32_t)(k + 1);
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

}  // namespace

// A chain kernel launched with programmatic stream serialisation: its blocks may be
// scheduled while the previous kernel of the view's chain drains (they wait in
// pdl_wait() for its completion), which shortens the 10-kernel chain's gaps.
template <typename... P, typename... A>
cudaError_t launch_pdl(void (*k)(P...), int grid, int block, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<P>(args)...);
}

size_t binsort_workspace(int n, int num_tiles, int64_t capacity) {
  (void)num_tiles;
  return carve(nullptr, n, capacity).total;
}

cudaError_t launch_binsort(const CamParams& cam, int n, const float4* xy_depth, const uint2* box,
                           const uint4* rows, const uint32_t* tiles, void* ws_ptr, int64_t capacity,
                           uint64_t* sorted_keys, uint32_t* sorted_ids, uint2* ranges,
                           uint32_t* num_pairs_dev, int pair_grid, cudaStream_t s) {
  const int num_tiles = cam.tiles_x * cam.tiles_y;
  WS w = carve(ws_ptr, n, capacity);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)num_tiles, s))) return e;
  if ((e = cudaMemsetAsync(w.hist, 0, w.ctrl_bytes, s))) return e;
  if (n == 0) {
    return cudaMemsetAsync(num_pairs_dev, 0, 2 * sizeof(uint32_t), s);
  }
  const int tile_bits = num_tiles > 1 ? 32 - __builtin_clz((unsigned)(num_tiles - 1)) : 0;
  const int npass = (tile_bits + 7) / 8;
  const int nblk_n = div_up(n, PRESORT_ITEMS);
  const size_t nblk_cap = (size_t)((capacity + SORT_ITEMS - 1) / SORT_ITEMS) + 1;
  const int grid_n = div_up(n, 256) < 148 * 8 ? div_up(n, 256) : 148 * 8;
  // two blocks per SM: every block flushes its 4×256 shared histogram bins with global
  // atomics onto the same 1024 words, so fewer, longer blocks contend less
  const int grid_i = div_up(n, 256) < 148 * 2 ? div_up(n, 256) : 148 * 2;
  // emit on two blocks per SM too (same histogram flush; measured 11.94 -> 11.89 ms in the
  // step, four per SM 11.90)
  const int grid_e = div_up(n, 256) < 148 * 2 ? div_up(n, 256) : 148 * 2;
  const int nblk_s = div_up(n, SORT_ITEMS);   // tile_scan blocks (2048 Gaussians each)
  presort_init_kernel<<<grid_i, 256, 0, s>>>(n, xy_depth, tiles, w.dkeysA, w.hist, w.dstatus,
                                             (size_t)4 * nblk_n * RADIX, w.scan_status, nblk_s);
  launch_counted();
  uint64_t* a = w.dkeysA;
  uint64_t* b = w.dkeysB;
  for (int p = 0; p < 4; ++p) {
    if ((e = launch_pdl(onesweep_kernel<uint64_t, PRESORT_IPT>, nblk_n, SORT_THREADS, s, a, b, n,
                        (const uint32_t*)nullptr, w.hist + p * RADIX,
                        w.dstatus + (size_t)p * nblk_n * RADIX, w.counters + p, 32 + 8 * p, 0))) return e;
    launch_counted();
    uint64_t* tmp = a; a = b; b = tmp;
  }
  // a = depth-sorted (zbits, id)
  if ((e = launch_pdl(tile_scan_kernel, nblk_s, 256, s, n, a, tiles, w.offsets, w.scan_status,
                      w.counters + 4, (long long)capacity, num_pairs_dev))) return e;
  launch_counted();
  if ((e = launch_pdl(emit_kernel, grid_e, 256, s, n, a, tiles, box, rows, w.offsets, num_pairs_dev,
                      cam.tiles_x, npass, w.pkeysA, w.hist, w.pstatus, nblk_cap * RADIX, 0, 0))) return e;
  launch_counted();
  uint64_t* pa = w.pkeysA;
  uint64_t* pb = w.pkeysB;
  // K ≤ capacity is known on the device only, so the pair passes launch for the capacity:
  // pair_grid = 0, one block per capacity tile (most leave empty; the fastest alone);
  // pair_grid > 0, that many blocks, each looping over key tiles — fewer resident blocks
  // next to the other views' kernels (dass_bin_sort_shared)
  const int grid_cap = pair_grid <= 0 || (int)nblk_cap < pair_grid ? (int)nblk_cap : pair_grid;
  for (int p = 0; p < npass; ++p) {
    if ((e = launch_pdl(onesweep_kernel<uint64_t, SORT_IPT>, grid_cap, SORT_THREADS, s, pa, pb, -1,
                        num_pairs_dev, w.hist + (4 + p) * RADIX,
                        w.pstatus + (size_t)p * nblk_cap * RADIX, w.counters + 5 + p, 32 + 8 * p,
                        grid_cap < (int)nblk_cap ? 1 : 0))) return e;
    launch_counted();
    uint64_t* tmp = pa; pa = pb; pb = tmp;
  }
  const int grid_f = 148 * 8;
  if ((e = launch_pdl(finalize_kernel, grid_f, 256, s, pa, num_pairs_dev, xy_depth, sorted_keys,
                      sorted_ids, ranges))) return e;
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
  const int nblk_n = div_up(nn, PRESORT_ITEMS);
  const size_t nblk_cap = (size_t)((cap + SORT_ITEMS - 1) / SORT_ITEMS) + 1;
  const int grid_n = div_up(nn, 256) < 148 * 8 ? div_up(nn, 256) : 148 * 8;
  const int nblk_s = div_up(nn, SORT_ITEMS);
  presort_init_kernel<<<grid_n, 256, 0, s>>>(nn, xy_depth, tiles, w.dkeysA, w.hist, w.dstatus,
                                             (size_t)4 * nblk_n * RADIX, w.scan_status, nblk_s);
  launch_counted();
  uint64_t* a = w.dkeysA;
  uint64_t* b = w.dkeysB;
  for (int p = 0; p < 4; ++p) {
    onesweep_kernel<uint64_t, PRESORT_IPT><<<nblk_n, SORT_THREADS, 0, s>>>(a, b, nn, nullptr, w.hist + p * RADIX,
                                                    w.dstatus + (size_t)p * nblk_n * RADIX,
                                                    w.counters + p, 32 + 8 * p, 0);
    launch_counted();
    uint64_t* tmp = a; a = b; b = tmp;
  }
  tile_scan_kernel<<<nblk_s, 256, 0, s>>>(nn, a, tiles, w.offsets, w.scan_status, w.counters + 4,
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
                                                           w.counters + 5 + p, 32 + 8 * p, 0);
    launch_counted();
    uint64_t* tmp = pa; pa = pb; pb = tmp;
  }
  finalize_views_kernel<<<148 * 8, 256, 0, s>>>(pa, kg, V, T, (long long)view_capacity, sorted_ids,
                                                ranges, view_pairs);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
