// densify.cu — SURVEY §8(f) f4: error-guided densification (§3.4).
//   densify_select: Eq. 4 per Gaussian, then a stable compaction of S;
//   spawn:          children sampled from N(p, Σ) of each selected parent (A45),
//                   drawn from a counter-based Philox4x64-10 (no generator state);
//   prune_select:   the keep list of the opacity pruning (A46);
//   gather:         row compaction / concatenation of the Gaussian arrays.
// All HBM-bound row kernels; the compaction is the stable partition of deform.cu.
#include "common.cuh"

namespace dass {
namespace {

__global__ void __launch_bounds__(256) select_flags_kernel(int n, const float* __restrict__ gsum,
                                                          const uint32_t* __restrict__ gcnt,
                                                          const uint8_t* __restrict__ s_err,
                                                          float tau_pos, float tau_err,
                                                          uint8_t* __restrict__ in_S) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = gcnt[i];
  const float g = c ? __fdiv_rn(gsum[i], (float)c) : 0.f;   // ∇p̄ (one IEEE fp32 division, A44)
  const bool a = g > tau_pos;
  const bool b = s_err != nullptr && s_err[i] != 0 && g > tau_err;
  in_S[i] = (a || b) ? 1 : 0;
}

__global__ void __launch_bounds__(256) prune_flags_kernel(int n, int first,
                                                         const float4* __restrict__ pos_opa,
                                                         float min_opacity,
                                                         uint8_t* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keep[i] = (i < first || !(pos_opa[i].w < min_opacity)) ? 1 : 0;
}

// dst row dst_offset + k ← src row (idx ? idx[k] : k), for every field.
__global__ void __launch_bounds__(256) gather_kernel(int n_src, int k4, const float4* __restrict__ pos_opa,
                                                    const float4* __restrict__ scale,
                                                    const float4* __restrict__ rot,
                                                    const float4* __restrict__ sh,
                                                    const uint8_t* __restrict__ dyn, int m,
                                                    const int* __restrict__ idx, int n_dst,
                                                    int dst_offset, float4* __restrict__ o_pos_opa,
                                                    float4* __restrict__ o_scale,
                                                    float4* __restrict__ o_rot,
                                                    float4* __restrict__ o_sh,
                                                    uint8_t* __restrict__ o_dyn) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int i = idx ? idx[k] : k;
  const int d = dst_offset + k;
  o_pos_opa[d] = pos_opa[i];
  o_scale[d] = scale[i];
  o_rot[d] = rot[i];
  for (int q = 0; q < k4; ++q) o_sh[(size_t)q * n_dst + d] = sh[(size_t)q * n_src + i];
  if (o_dyn) o_dyn[d] = dyn ? dyn[i] : 0;
}

__device__ __forceinline__ void philox4x64(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = c[0] * 0xD2E7470EE14C6C93ull, hi0 = __umul64hi(c[0], 0xD2E7470EE14C6C93ull);
    const uint64_t lo1 = c[2] * 0xCA5A826395121157ull, hi1 = __umul64hi(c[2], 0xCA5A826395121157ull);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

// One thread per child c = k·K + j of the k-th selected parent (A45).
__global__ void __launch_bounds__(256) spawn_kernel(int n_src, int k4, const float4* __restrict__ pos_opa,
                                                   const float4* __restrict__ scale,
                                                   const float4* __restrict__ rot,
                                                   const float4* __restrict__ sh,
                                                   const uint8_t* __restrict__ dyn, int m,
                                                   const int* __restrict__ idx, int K, float shrink,
                                                   float child_opacity, uint64_t seed, int n_dst,
                                                   int dst_offset, float4* __restrict__ o_pos_opa,
                                                   float4* __restrict__ o_scale,
                                                   float4* __restrict__ o_rot,
                                                   float4* __restrict__ o_sh,
                                                   uint8_t* __restrict__ o_dyn) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (long long)m * K) return;
  const int k = (int)(c / K);
  const int i = idx[k];
  uint64_t r[4] = {(uint64_t)c, 0ull, 0ull, 0ull};
  philox4x64(r, seed, 0x44415353ull);
  float u[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) u[a] = ((float)(r[a] >> 40) + 0.5f) * (1.0f / 16777216.0f);
  const float r0 = sqrtf(-2.f * logf(u[0])), r1 = sqrtf(-2.f * logf(u[2]));
  float s1, c1, s3, c3;
  sincospif(2.f * u[1], &s1, &c1);
  sincospif(2.f * u[3], &s3, &c3);
  const float z[3] = {r0 * c1, r0 * s1, r1 * c3};
  const float4 p = pos_opa[i], s = scale[i], q = rot[i];
  const float inv = rsqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
  const float w = q.x * inv, x = q.y * inv, y = q.z * inv, zq = q.w * inv;
  const float R[3][3] = {{1.f - 2.f * (y * y + zq * zq), 2.f * (x * y - w * zq), 2.f * (x * zq + w * y)},
                         {2.f * (x * y + w * zq), 1.f - 2.f * (x * x + zq * zq), 2.f * (y * zq - w * x)},
                         {2.f * (x * zq - w * y), 2.f * (y * zq + w * x), 1.f - 2.f * (x * x + y * y)}};
  const float v[3] = {s.x * z[0], s.y * z[1], s.z * z[2]};
  const int d = dst_offset + (int)c;
  o_pos_opa[d] = make_float4(p.x + R[0][0] * v[0] + R[0][1] * v[1] + R[0][2] * v[2],
                             p.y + R[1][0] * v[0] + R[1][1] * v[1] + R[1][2] * v[2],
                             p.z + R[2][0] * v[0] + R[2][1] * v[1] + R[2][2] * v[2], child_opacity);
  o_scale[d] = make_float4(__fdiv_rn(s.x, shrink), __fdiv_rn(s.y, shrink), __fdiv_rn(s.z, shrink), 0.f);
  o_rot[d] = q;
  for (int qq = 0; qq < k4; ++qq) o_sh[(size_t)qq * n_dst + d] = sh[(size_t)qq * n_src + i];
  if (o_dyn) o_dyn[d] = dyn ? dyn[i] : 0;
}

}  // namespace

cudaError_t launch_densify_select(int n, const float* gsum, const uint32_t* gcnt,
                                  const uint8_t* s_err, float tau_pos, float tau_err,
                                  uint8_t* in_S, int* idx, int* counts, void* ws, cudaStream_t s) {
  if (n > 0) {
    select_flags_kernel<<<div_up(n, 256), 256, 0, s>>>(n, gsum, gcnt, s_err, tau_pos, tau_err, in_S);
    launch_counted();
  }
  return launch_partition(n, in_S, idx, nullptr, counts, ws, s);
}

cudaError_t launch_prune_select(int n, int first, const float4* pos_opa, float min_opacity,
                                uint8_t* keep, int* idx, int* counts, void* ws, cudaStream_t s) {
  if (n > 0) {
    prune_flags_kernel<<<div_up(n, 256), 256, 0, s>>>(n, first, pos_opa, min_opacity, keep);
    launch_counted();
  }
  return launch_partition(n, keep, idx, nullptr, counts, ws, s);
}

cudaError_t launch_gather(int n_src, int k4, const float4* pos_opa, const float4* scale,
                          const float4* rot, const float4* sh, const uint8_t* dyn, int m,
                          const int* idx, int n_dst, int dst_offset, float4* o_pos_opa,
                          float4* o_scale, float4* o_rot, float4* o_sh, uint8_t* o_dyn,
                          cudaStream_t s) {
  if (m <= 0) return cudaSuccess;
  gather_kernel<<<div_up(m, 256), 256, 0, s>>>(n_src, k4, pos_opa, scale, rot, sh, dyn, m, idx,
                                               n_dst, dst_offset, o_pos_opa, o_scale, o_rot, o_sh,
                                               o_dyn);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_spawn_children(int n_src, int k4, const float4* pos_opa, const float4* scale,
                                  const float4* rot, const float4* sh, const uint8_t* dyn, int m,
                                  const int* idx, int K, float shrink, float child_opacity,
                                  uint64_t seed, int n_dst, int dst_offset, float4* o_pos_opa,
                                  float4* o_scale, float4* o_rot, float4* o_sh, uint8_t* o_dyn,
                                  cudaStream_t s) {
  const long long total = (long long)m * K;
  if (total <= 0) return cudaSuccess;
  spawn_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      n_src, k4, pos_opa, scale, rot, sh, dyn, m, idx, K, shrink, child_opacity, seed, n_dst,
      dst_offset, o_pos_opa, o_scale, o_rot, o_sh, o_dyn);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
