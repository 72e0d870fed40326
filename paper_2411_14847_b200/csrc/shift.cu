// shift.cu — masked per-Gaussian shift (§3.3) and its backward.
// HBM-bound elementwise kernels: one thread per Gaussian, float4 loads.
#include "common.cuh"

namespace dass {
namespace {

__device__ __forceinline__ float4 qmul(float4 a, float4 b) {  // Hamilton, (w,x,y,z)
  return make_float4(a.x * b.x - a.y * b.y - a.z * b.z - a.w * b.w,
                     a.x * b.y + a.y * b.x + a.z * b.w - a.w * b.z,
                     a.x * b.z - a.y * b.w + a.z * b.x + a.w * b.y,
                     a.x * b.w + a.y * b.z - a.z * b.y + a.w * b.x);
}

__device__ __forceinline__ float norm4(float4 a) {
  return sqrtf(a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w);
}

__global__ void __launch_bounds__(256) shift_kernel(int n, const float4* __restrict__ pos,
                                                    const float4* __restrict__ rot,
                                                    const float4* __restrict__ mu,
                                                    const float4* __restrict__ sigma,
                                                    const uint8_t* __restrict__ mask,
                                                    float4* pos_out, float4* rot_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float4 p = pos[i];
  float4 q = rot[i];
  if (mask == nullptr || mask[i]) {
    const float4 m = mu[i];
    float4 s = sigma[i];
    p.x += m.x; p.y += m.y; p.z += m.z;
    const float nq = norm4(q);
    q = make_float4(q.x / nq, q.y / nq, q.z / nq, q.w / nq);
    const float ns = norm4(s);
    s = ns < 1e-8f ? make_float4(1.f, 0.f, 0.f, 0.f)
                   : make_float4(s.x / ns, s.y / ns, s.z / ns, s.w / ns);
    q = qmul(q, s);  // q' = n(q) ⊗ n(σ)
  }
  pos_out[i] = p;
  rot_out[i] = q;
}

__global__ void __launch_bounds__(256) shift_bwd_kernel(int n, const float4* __restrict__ rot,
                                                        const float4* __restrict__ sigma,
                                                        const uint8_t* __restrict__ mask,
                                                        const float4* __restrict__ gp,
                                                        const float4* __restrict__ gq,
                                                        float4* g_mu, float4* g_sigma) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mask != nullptr && !mask[i]) return;
  if (g_mu) {
    const float4 g = gp[i];
    float4 o = g_mu[i];
    o.x += g.x; o.y += g.y; o.z += g.z;
    g_mu[i] = o;
  }
  if (g_sigma) {
    float4 s = sigma[i];
    const float ns = norm4(s);
    if (ns < 1e-8f) return;
    float4 q = rot[i];
    const float nq = norm4(q);
    q = make_float4(q.x / nq, q.y / nq, q.z / nq, q.w / nq);
    s = make_float4(s.x / ns, s.y / ns, s.z / ns, s.w / ns);
    const float4 g = gq[i];
    // dL/dŝ = L(q̂)ᵀ dL/dq'  with L(a) the left-multiplication matrix
    const float4 gs = make_float4(q.x * g.x + q.y * g.y + q.z * g.z + q.w * g.w,
                                  -q.y * g.x + q.x * g.y + q.w * g.z - q.z * g.w,
                                  -q.z * g.x - q.w * g.y + q.x * g.z + q.y * g.w,
                                  -q.w * g.x + q.z * g.y - q.y * g.z + q.x * g.w);
    const float dot = s.x * gs.x + s.y * gs.y + s.z * gs.z + s.w * gs.w;
    const float inv = 1.0f / ns;
    float4 o = g_sigma[i];
    o.x += (gs.x - s.x * dot) * inv;
    o.y += (gs.y - s.y * dot) * inv;
    o.z += (gs.z - s.z * dot) * inv;
    o.w += (gs.w - s.w * dot) * inv;
    g_sigma[i] = o;
  }
}

}  // namespace

cudaError_t launch_shift(int n, const float4* pos, const float4* rot, const float4* mu,
                         const float4* sigma, const uint8_t* mask, float4* pos_out,
                         float4* rot_out, cudaStream_t s) {
  shift_kernel<<<div_up(n, 256), 256, 0, s>>>(n, pos, rot, mu, sigma, mask, pos_out, rot_out);
  launch_counted();
  return cudaGetLastError();
}

cudaError_t launch_shift_bwd(int n, const float4* rot, const float4* sigma, const uint8_t* mask,
                             const float4* g_pos_out, const float4* g_rot_out, float4* g_mu,
                             float4* g_sigma, cudaStream_t s) {
  shift_bwd_kernel<<<div_up(n, 256), 256, 0, s>>>(n, rot, sigma, mask, g_pos_out, g_rot_out,
                                                  g_mu, g_sigma);
  launch_counted();
  return cudaGetLastError();
}

}  // namespace dass
