// sh.cuh — real spherical harmonics of degree ≤ 3 (3DGS/Plenoxels constants
// and ordering, A14) for the view-dependent colour c_i.
#pragma once
#include "common.cuh"

namespace dass {

struct SHConst {
  static constexpr float C0 = 0.28209479177387814f;
  static constexpr float C1 = 0.4886025119029199f;
  static constexpr float C2_0 = 1.0925484305920792f;
  static constexpr float C2_1 = -1.0925484305920792f;
  static constexpr float C2_2 = 0.31539156525252005f;
  static constexpr float C2_3 = -1.0925484305920792f;
  static constexpr float C2_4 = 0.5462742152960396f;
  static constexpr float C3_0 = -0.5900435899266435f;
  static constexpr float C3_1 = 2.890611442640554f;
  static constexpr float C3_2 = -0.4570457994644658f;
  static constexpr float C3_3 = 0.3731763325901154f;
  static constexpr float C3_4 = -0.4570457994644658f;
  static constexpr float C3_5 = 1.445305721320277f;
  static constexpr float C3_6 = -0.5900435899266435f;
};

// Basis values Y[0..(DEG+1)²) at unit direction (x, y, z).
template <int DEG>
__device__ __forceinline__ void sh_eval(float x, float y, float z, float* Y) {
  Y[0] = SHConst::C0;
  if (DEG >= 1) {
    Y[1] = -SHConst::C1 * y;
    Y[2] = SHConst::C1 * z;
    Y[3] = -SHConst::C1 * x;
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    Y[4] = SHConst::C2_0 * x * y;
    Y[5] = SHConst::C2_1 * y * z;
    Y[6] = SHConst::C2_2 * (2.f * zz - xx - yy);
    Y[7] = SHConst::C2_3 * x * z;
    Y[8] = SHConst::C2_4 * (xx - yy);
    if (DEG >= 3) {
      Y[9] = SHConst::C3_0 * y * (3.f * xx - yy);
      Y[10] = SHConst::C3_1 * x * y * z;
      Y[11] = SHConst::C3_2 * y * (4.f * zz - xx - yy);
      Y[12] = SHConst::C3_3 * z * (2.f * zz - 3.f * xx - 3.f * yy);
      Y[13] = SHConst::C3_4 * x * (4.f * zz - xx - yy);
      Y[14] = SHConst::C3_5 * z * (xx - yy);
      Y[15] = SHConst::C3_6 * x * (xx - 3.f * yy);
    }
  }
}

// Gradient of Σ_k Y_k(d)·w_k w.r.t. the (unnormalised-independent) direction
// components, given per-basis weights w_k (= Σ_ch g_ch · sh_k,ch).
template <int DEG>
__device__ __forceinline__ float3 sh_dir_grad(float x, float y, float z, const float* w) {
  float gx = 0.f, gy = 0.f, gz = 0.f;
  if (DEG >= 1) {
    gy += -SHConst::C1 * w[1];
    gz += SHConst::C1 * w[2];
    gx += -SHConst::C1 * w[3];
  }
  if (DEG >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    gx += SHConst::C2_0 * y * w[4];
    gy += SHConst::C2_0 * x * w[4];
    gy += SHConst::C2_1 * z * w[5];
    gz += SHConst::C2_1 * y * w[5];
    gx += SHConst::C2_2 * (-2.f * x) * w[6];
    gy += SHConst::C2_2 * (-2.f * y) * w[6];
    gz += SHConst::C2_2 * (4.f * z) * w[6];
    gx += SHConst::C2_3 * z * w[7];
    gz += SHConst::C2_3 * x * w[7];
    gx += SHConst::C2_4 * (2.f * x) * w[8];
    gy += SHConst::C2_4 * (-2.f * y) * w[8];
    if (DEG >= 3) {
      gx += SHConst::C3_0 * 6.f * x * y * w[9];
      gy += SHConst::C3_0 * (3.f * xx - 3.f * yy) * w[9];
      gx += SHConst::C3_1 * y * z * w[10];
      gy += SHConst::C3_1 * x * z * w[10];
      gz += SHConst::C3_1 * x * y * w[10];
      gx += SHConst::C3_2 * (-2.f * x * y) * w[11];
      gy += SHConst::C3_2 * (4.f * zz - xx - 3.f * yy) * w[11];
      gz += SHConst::C3_2 * (8.f * y * z) * w[11];
      gx += SHConst::C3_3 * (-6.f * x * z) * w[12];
      gy += SHConst::C3_3 * (-6.f * y * z) * w[12];
      gz += SHConst::C3_3 * (6.f * zz - 3.f * xx - 3.f * yy) * w[12];
      gx += SHConst::C3_4 * (4.f * zz - 3.f * xx - yy) * w[13];
      gy += SHConst::C3_4 * (-2.f * x * y) * w[13];
      gz += SHConst::C3_4 * (8.f * x * z) * w[13];
      gx += SHConst::C3_5 * (2.f * x * z) * w[14];
      gy += SHConst::C3_5 * (-2.f * y * z) * w[14];
      gz += SHConst::C3_5 * (xx - yy) * w[14];
      gx += SHConst::C3_6 * (3.f * xx - 3.f * yy) * w[15];
      gy += SHConst::C3_6 * (-6.f * x * y) * w[15];
    }
  }
  return make_float3(gx, gy, gz);
}

// Coefficient f (= k*3 + ch) of Gaussian i in the plane layout sh[f/4][i].f%4.
template <int DEG>
struct SHLayout {
  static constexpr int NC = (DEG + 1) * (DEG + 1);  // coefficients per channel
  static constexpr int NF = 3 * NC;                  // floats per Gaussian
  static constexpr int K4 = (NF + 3) / 4;            // float4 planes
};

}  // namespace dass
