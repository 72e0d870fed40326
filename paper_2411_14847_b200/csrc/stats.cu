// stats.cu — dass_render_stats: scene statistics of one rendered view
// (SURVEY §8(d)): P_fwd, P_bwd, accepted entries, early-terminated pixels and
// tile-list lengths.  Diagnostic (not on the timed path): it replays the
// forward's per-pixel decisions with the same inline functions as
// render_fwd, so its counts are those of the kernels being measured.
#include "common.cuh"

namespace dass {
namespace {

__global__ void __launch_bounds__(256) stats_kernel(const __grid_constant__ CamParams cam,
                                                   const uint2* __restrict__ ranges,
                                                   const uint32_t* __restrict__ ids,
                                                   const float4* __restrict__ xy_depth,
                                                   const float4* __restrict__ conic_opa,
                                                   const uint2* __restrict__ box,
                                                   const uint32_t* __restrict__ out_last,
                                                   unsigned long long* counters) {
  __shared__ unsigned long long s_c[8];
  const int tile = blockIdx.x;
  const int tyi = tile / cam.tiles_x, txi = tile - tyi * cam.tiles_x;
  const int tx0 = txi * TILE, ty0 = tyi * TILE;
  const int t = threadIdx.x;
  if (t < 8) s_c[t] = 0ull;
  __syncthreads();
  const int X = tx0 + (t & 15), Y = ty0 + (t >> 4);
  const uint2 range = ranges[tile];
  unsigned long long pf = 0, pb = 0, acc = 0, term = 0, upto = 0;
  if (X < cam.W && Y < cam.H) {
    const uint32_t last = out_last[(size_t)Y * cam.W + X];
    float T = 1.f;
    bool done = false;
    for (uint32_t k = range.x; k < range.y; ++k) {
      const uint32_t id = ids[k];
      const uint2 b = box[id];
      const bool inbox = X >= (int)(b.x & 0xFFFFu) && X <= (int)(b.x >> 16) &&
                         Y >= (int)(b.y & 0xFFFFu) && Y <= (int)(b.y >> 16);
      if (k < last) {
        ++upto;
        if (inbox) ++pb;
      }
      if (done || !inbox) continue;
      ++pf;
      const float4 xy = xy_depth[id];
      const uint32_t lo_bits = __float_as_uint(xy.w);
      const __half2 lo = *reinterpret_cast<const __half2*>(&lo_bits);
      const float u = __fadd_rn(xy.x - (float)tx0, __low2float(lo));
      const float v = __fadd_rn(xy.y - (float)ty0, __high2float(lo));
      const float4 co = conic_staged(conic_opa[id]);
      const float power = splat_power(co, u - (float)(t & 15), v - (float)(t >> 4));
      if (power > 0.f) continue;
      const float alpha = splat_alpha(co.w, splat_exp(power));
      if (alpha < ALPHA_MIN) continue;
      const float tn = __fmul_rn(T, __fsub_rn(1.f, alpha));
      if (tn < T_MIN) { done = true; ++term; continue; }
      T = tn;
      ++acc;
    }
  }
  atomicAdd(&s_c[0], pf);
  atomicAdd(&s_c[1], pb);
  atomicAdd(&s_c[2], acc);
  atomicAdd(&s_c[3], term);
  atomicAdd(&s_c[7], upto);
  __syncthreads();
  if (t == 0) {
    const unsigned long long len = range.y - range.x;
    atomicAdd(&counters[0], s_c[0]);
    atomicAdd(&counters[1], s_c[1]);
    atomicAdd(&counters[2], s_c[2]);
    atomicAdd(&counters[3], s_c[3]);
    atomicAdd(&counters[4], len);
    atomicMax(&counters[5], len);
    if (len) atomicAdd(&counters[6], 1ull);
    atomicAdd(&counters[7], s_c[7]);
  }
}

}  // namespace

cudaError_t launch_render_stats(const CamParams& cam, const uint2* ranges, const uint32_t* ids,
                                const float4* xy_depth, const float4* conic_opa, const uint2* box,
                                const float* out_T, const uint32_t* out_last,
                                unsigned long long* counters, cudaStream_t s) {
  (void)out_T;
  cudaError_t e = cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  stats_kernel<<<cam.tiles_x * cam.tiles_y, 256, 0, s>>>(cam, ranges, ids, xy_depth, conic_opa, box,
                                                         out_last, counters);
  launch_counted();
  return cudaGetLastError();
}

namespace {
__global__ void timestamp_kernel(uint64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace

// Numerical validation (DASS_ERR_NUMERICAL): count the non-finite values.
__global__ void __launch_bounds__(256) nonfinite_kernel(const float* __restrict__ x, long long n,
                                                       uint32_t* __restrict__ count) {
  uint32_t c = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    c += isfinite(x[i]) ? 0u : 1u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(count, c);
}

cudaError_t launch_nonfinite(const float* x, long long n, uint32_t* count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long blocks = (n + 255) / 256;
  nonfinite_kernel<<<(int)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, s>>>(x, n, count);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_timestamp(uint64_t* out, cudaStream_t s) {
  timestamp_kernel<<<1, 1, 0, s>>>(out);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
