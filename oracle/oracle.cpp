// oracle/oracle.cpp — the CPU ORACLE for the DASS hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  The
// product path (libdass.so + its Python binding) never links, imports or calls
// it, and this file shares no code, header, constant table or helper with the
// CUDA path (paper_2411_14847_b200/csrc).
//
// What it computes, each function citing the passage it follows
// (P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n; A.. = the
// readings in DESIGN.md §Readings):
//   O1  oracle_shift / oracle_shift_bwd     §3.3 P:128 (A24, A25)
//   O2  oracle_project                       Eqs. 5-7, colour P:351
//       + the fp32 KEY REPLICA (depth bits, pixel box, visibility) following
//         the op order documented in include/dass.h (typed independently here)
//   O3  oracle_bin_sort                      brute-force enumeration + sort (A03-A04)
//   O4  oracle_render (literal & scatter)    Eq. 8 P:349-351 (A01, A05, A11-A13)
//   O5  oracle_render_bwd                    exact derivative of O2+O4 (A16-A18)
//   O6  gradstat                             §3.4 P:159 (A23)
//   O7  oracle_error_map                     §3.4, Alg. 1 P:403-415 (A20-A22)
// Everything image/gradient-valued is double.  The only float arithmetic is the
// key replica, compiled with -ffp-contract=off so each operation rounds once.
//
// Parity pins: see tests/test_oracle_*.py.  SH sign/ordering convention (A14)
// is "parity unpinned" against the paper (the paper never states it).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// Memory layout identical to the camera record the input generator builds
// (paper_2411_14847_b200/synth.py CAMERA_DTYPE); declared here on its own.
struct OCam {
  int32_t width, height;
  float fx, fy, cx, cy;
  float viewmat[12];
  float near_plane;
  float full_proj[16];
};

int oracle_version(void) { return 1; }

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// OpenMP threads of the following calls (bench.py times the oracle single-threaded
// and on every host core).
void oracle_set_threads(int k) {
#ifdef _OPENMP
  if (k > 0) omp_set_num_threads(k);
#else
  (void)k;
#endif
}

}  // extern "C"

namespace {

// ---------------------------------------------------------------- O1 shift --
// Hamilton product, real part first (A25).
void qmul(const double a[4], const double b[4], double o[4]) {
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

double norm4(const double a[4]) {
  return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2] + a[3] * a[3]);
}

// ------------------------------------------------------ SH basis (A14) -----
// Real SH, degree <= 3, 3DGS/Plenoxels constants and ordering.
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792,
                         0.31539156525252005, -1.0925484305920792,
                         0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554,
                         -0.4570457994644658, 0.3731763325901154,
                         -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};

// Y[k] and dY[k][0..2] = ∂Y_k/∂(x,y,z) at direction d (treated as free vars).
void sh_basis(int deg, const double d[3], double Y[16], double dY[16][3]) {
  const double x = d[0], y = d[1], z = d[2];
  for (int k = 0; k < 16; ++k) { Y[k] = 0; dY[k][0] = dY[k][1] = dY[k][2] = 0; }
  Y[0] = SH_C0;
  if (deg < 1) return;
  Y[1] = -SH_C1 * y;  dY[1][1] = -SH_C1;
  Y[2] = SH_C1 * z;   dY[2][2] = SH_C1;
  Y[3] = -SH_C1 * x;  dY[3][0] = -SH_C1;
  if (deg < 2) return;
  Y[4] = SH_C2[0] * x * y;               dY[4][0] = SH_C2[0] * y; dY[4][1] = SH_C2[0] * x;
  Y[5] = SH_C2[1] * y * z;               dY[5][1] = SH_C2[1] * z; dY[5][2] = SH_C2[1] * y;
  Y[6] = SH_C2[2] * (2 * z * z - x * x - y * y);
  dY[6][0] = SH_C2[2] * (-2 * x); dY[6][1] = SH_C2[2] * (-2 * y); dY[6][2] = SH_C2[2] * (4 * z);
  Y[7] = SH_C2[3] * x * z;               dY[7][0] = SH_C2[3] * z; dY[7][2] = SH_C2[3] * x;
  Y[8] = SH_C2[4] * (x * x - y * y);     dY[8][0] = SH_C2[4] * 2 * x; dY[8][1] = SH_C2[4] * (-2 * y);
  if (deg < 3) return;
  Y[9] = SH_C3[0] * y * (3 * x * x - y * y);
  dY[9][0] = SH_C3[0] * 6 * x * y; dY[9][1] = SH_C3[0] * (3 * x * x - 3 * y * y);
  Y[10] = SH_C3[1] * x * y * z;
  dY[10][0] = SH_C3[1] * y * z; dY[10][1] = SH_C3[1] * x * z; dY[10][2] = SH_C3[1] * x * y;
  Y[11] = SH_C3[2] * y * (4 * z * z - x * x - y * y);
  dY[11][0] = SH_C3[2] * (-2 * x * y);
  dY[11][1] = SH_C3[2] * (4 * z * z - x * x - 3 * y * y);
  dY[11][2] = SH_C3[2] * (8 * y * z);
  Y[12] = SH_C3[3] * z * (2 * z * z - 3 * x * x - 3 * y * y);
  dY[12][0] = SH_C3[3] * (-6 * x * z); dY[12][1] = SH_C3[3] * (-6 * y * z);
  dY[12][2] = SH_C3[3] * (6 * z * z - 3 * x * x - 3 * y * y);
  Y[13] = SH_C3[4] * x * (4 * z * z - x * x - y * y);
  dY[13][0] = SH_C3[4] * (4 * z * z - 3 * x * x - y * y);
  dY[13][1] = SH_C3[4] * (-2 * x * y); dY[13][2] = SH_C3[4] * (8 * x * z);
  Y[14] = SH_C3[5] * z * (x * x - y * y);
  dY[14][0] = SH_C3[5] * 2 * x * z; dY[14][1] = SH_C3[5] * (-2 * y * z);
  dY[14][2] = SH_C3[5] * (x * x - y * y);
  Y[15] = SH_C3[6] * x * (x * x - 3 * y * y);
  dY[15][0] = SH_C3[6] * (3 * x * x - 3 * y * y); dY[15][1] = SH_C3[6] * (-6 * x * y);
}

// ---------------------------------------------------- parameter access -----
struct Params {
  int n, deg;
  const float* pos_opa;  // [n][4]
  const float* scale;    // [n][4]
  const float* rot;      // [n][4]
  const float* sh;       // [K4][n][4] planes
  const uint8_t* keep;   // nullable
  int ncoef() const { return (deg + 1) * (deg + 1); }
  int k4() const { return (3 * ncoef() + 3) / 4; }
  // coefficient k, channel ch of Gaussian i (coefficient-major, channel-minor)
  double shc(int i, int k, int ch) const {
    int f = k * 3 + ch;
    return (double)sh[((size_t)(f / 4) * n + i) * 4 + (f % 4)];
  }
  bool kept(int i) const { return keep == nullptr || keep[i] != 0; }
};

// ------------------------------------------ O2-key: the fp32 replica -------
// Exactly the op order of include/dass.h "KEY CHAIN", one rounding per op.
struct KeyReplica {
  bool visible;
  float z;
  uint32_t zbits;
  int x0, x1, y0, y1;
  uint32_t tiles;
  uint32_t rows[4];   // A50 tile-row spans (8 × 16 bits) or the full-box sentinel
};

// A50, KEY CHAIN steps 12-13 of include/dass.h, typed from that text: the tile
// footprint is, per tile row of the box, the tile columns the ellipse
// {d : dᵀ Σ'⁻¹ d ≤ R2} reaches in the row's band of pixel rows, padded by one
// pixel, with R2 ≥ 1.01·2·ln(255·o) + 0.05 an upper bound of the α ≥ 1/255
// support (ln m ≤ m − 1 on the mantissa).  Boxes of more than 8 tile rows or
// 255 tile columns keep every box tile (sentinel rows = all ones).  Returns the
// tile count.
uint32_t footprint_rows(float ca, float cb, float cc, float det, float u, float v, float o,
                        int x0, int x1, int y0, int y1, uint32_t rows[4]) {
  const int tx0 = x0 / 16, tx1 = x1 / 16, ty0 = y0 / 16, ty1 = y1 / 16;
  if (ty1 - ty0 + 1 > 8 || tx1 - tx0 + 1 > 255) {
    for (int w = 0; w < 4; ++w) rows[w] = 0xFFFFFFFFu;
    return (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
  }
  // 12. the threshold
  const float xo = 255.0f * o;
  uint32_t bits;
  std::memcpy(&bits, &xo, 4);
  const int e = (int)(bits >> 23) - 127;
  const uint32_t mbits = (bits & 0x007FFFFFu) | 0x3F800000u;
  float mf;
  std::memcpy(&mf, &mbits, 4);
  float L = (float)e * 0.693147182f;
  L = L + (mf - 1.0f);
  float R2 = (2.0f * L) * 1.01f;
  R2 = R2 + 0.05f;
  // 13. per tile row
  const float sxa = std::sqrt(R2 * ca);
  const float tq = std::sqrt(R2 / ca);
  const float dyL = -(cb * tq), dyR = cb * tq;
  const float crr = cc * R2;
  const float ey = std::sqrt(crr);
  const float icc = 1.0f / cc;
  auto half = [&](float d) {   // √(det·(cc·R2 − d²)), clamped at 0
    float r = crr - d * d;
    r = det * r;
    return std::sqrt(std::fmax(0.0f, r));
  };
  uint32_t total = 0;
  for (int w = 0; w < 4; ++w) rows[w] = 0;
  for (int ty = ty0; ty <= ty1; ++ty) {
    const int k = ty - ty0;
    uint32_t span = 0x00FFu;   // empty: lo = 255 > hi = 0
    const int Y0 = std::max(y0, 16 * ty), Y1 = std::min(y1, 16 * ty + 15);
    float d0 = (float)Y0 - v, d1 = (float)Y1 - v;
    d0 = std::fmax(d0, -ey);
    d1 = std::fmin(d1, ey);
    if (d0 <= d1) {
      const float h0 = half(d0), h1 = half(d1);
      const float l0 = (cb * d0 - h0) * icc, l1 = (cb * d1 - h1) * icc;
      const float r0 = (cb * d0 + h0) * icc, r1 = (cb * d1 + h1) * icc;
      const float lo = (d0 <= dyL && dyL <= d1) ? -sxa : std::fmin(l0, l1);
      const float hi = (d0 <= dyR && dyR <= d1) ? sxa : std::fmax(r0, r1);
      float X0f = u + lo;
      X0f = X0f - 1.0f;
      X0f = std::fmax((float)x0, X0f);
      float X1f = u + hi;
      X1f = X1f + 1.0f;
      X1f = std::fmin((float)x1, X1f);
      const float c0 = std::ceil(X0f), c1 = std::floor(X1f);
      if (c0 <= c1) {
        const int lo_t = (int)c0 / 16 - tx0, hi_t = (int)c1 / 16 - tx0;
        span = (uint32_t)lo_t | ((uint32_t)hi_t << 8);
        total += (uint32_t)(hi_t - lo_t + 1);
      }
    }
    rows[k >> 1] |= span << (16 * (k & 1));
  }
  for (int k = ty1 - ty0 + 1; k < 8; ++k) rows[k >> 1] |= 0x00FFu << (16 * (k & 1));
  return total;
}

KeyReplica key_replica(const OCam& c, const Params& P, int i) {
  KeyReplica k;
  k.visible = false; k.z = 0; k.zbits = 0; k.x0 = 1; k.x1 = 0; k.y0 = 1; k.y1 = 0; k.tiles = 0;
  k.rows[0] = k.rows[1] = k.rows[2] = k.rows[3] = 0;
  const float* V = c.viewmat;
  const float px = P.pos_opa[4 * i + 0], py = P.pos_opa[4 * i + 1], pz = P.pos_opa[4 * i + 2];
  const float o = P.kept(i) ? P.pos_opa[4 * i + 3] : 0.0f;
  float s[3];
  for (int a = 0; a < 3; ++a) s[a] = P.kept(i) ? P.scale[4 * i + a] : 0.0f;
  // 1. camera transform
  float t[3];
  for (int a = 0; a < 3; ++a) {
    float acc = V[4 * a + 0] * px;
    acc = acc + V[4 * a + 1] * py;
    acc = acc + V[4 * a + 2] * pz;
    acc = acc + V[4 * a + 3];
    t[a] = acc;
  }
  // 2. near cull
  if (!(t[2] > c.near_plane)) return k;
  // 3. quaternion normalisation
  const float qw = P.rot[4 * i + 0], qx = P.rot[4 * i + 1], qy = P.rot[4 * i + 2], qz = P.rot[4 * i + 3];
  float nn = qw * qw;
  nn = nn + qx * qx;
  nn = nn + qy * qy;
  nn = nn + qz * qz;
  const float nq = std::sqrt(nn);
  if (!(nq > 0.0f) || !std::isfinite(nq)) return k;
  const float w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
  // 4. rotation matrix
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, xz = x * z, yz = y * z;
  const float wx = w * x, wy = w * y, wz = w * z;
  float R[3][3];
  R[0][0] = 1.0f - 2.0f * (yy + zz); R[0][1] = 2.0f * (xy - wz); R[0][2] = 2.0f * (xz + wy);
  R[1][0] = 2.0f * (xy + wz); R[1][1] = 1.0f - 2.0f * (xx + zz); R[1][2] = 2.0f * (yz - wx);
  R[2][0] = 2.0f * (xz - wy); R[2][1] = 2.0f * (yz + wx); R[2][2] = 1.0f - 2.0f * (xx + yy);
  // 5. Σ = (R diag(s)) (R diag(s))^T
  float m[3][3];
  for (int a = 0; a < 3; ++a)
    for (int kk = 0; kk < 3; ++kk) m[a][kk] = R[a][kk] * s[kk];
  float S[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b) {
      float acc = m[a][0] * m[b][0];
      acc = acc + m[a][1] * m[b][1];
      acc = acc + m[a][2] * m[b][2];
      S[a][b] = acc; S[b][a] = acc;
    }
  // 6. clamped Jacobian
  const float W = (float)c.width, H = (float)c.height;
  const float lx = (1.3f * W) / (2.0f * c.fx);
  const float ly = (1.3f * H) / (2.0f * c.fy);
  const float xt = std::fmin(lx, std::fmax(-lx, t[0] / t[2])) * t[2];
  const float yt = std::fmin(ly, std::fmax(-ly, t[1] / t[2])) * t[2];
  const float tz2 = t[2] * t[2];
  const float J00 = c.fx / t[2];
  const float J02 = -((c.fx * xt) / tz2);
  const float J11 = c.fy / t[2];
  const float J12 = -((c.fy * yt) / tz2);
  // 7. M = J W, Σ' = M Σ M^T + 0.3 I
  float M[2][3];
  for (int kk = 0; kk < 3; ++kk) {
    M[0][kk] = J00 * V[0 * 4 + kk] + J02 * V[2 * 4 + kk];
    M[1][kk] = J11 * V[1 * 4 + kk] + J12 * V[2 * 4 + kk];
  }
  float Pm[2][3];
  for (int a = 0; a < 2; ++a)
    for (int kk = 0; kk < 3; ++kk) {
      float acc = M[a][0] * S[0][kk];
      acc = acc + M[a][1] * S[1][kk];
      acc = acc + M[a][2] * S[2][kk];
      Pm[a][kk] = acc;
    }
  float ca = Pm[0][0] * M[0][0];
  ca = ca + Pm[0][1] * M[0][1];
  ca = ca + Pm[0][2] * M[0][2];
  ca = ca + 0.3f;
  float cb = Pm[0][0] * M[1][0];
  cb = cb + Pm[0][1] * M[1][1];
  cb = cb + Pm[0][2] * M[1][2];
  float cc = Pm[1][0] * M[1][0];
  cc = cc + Pm[1][1] * M[1][1];
  cc = cc + Pm[1][2] * M[1][2];
  cc = cc + 0.3f;
  // 8. determinant
  const float det = ca * cc - cb * cb;
  if (!(det > 0.0f)) return k;
  // 9. radius
  const float mid = 0.5f * (ca + cc);
  const float lam = mid + std::sqrt(std::fmax(0.1f, mid * mid - det));
  const float r = std::ceil(3.0f * std::sqrt(lam));
  // 10. mean
  const float u = (c.fx * t[0]) / t[2] + c.cx;
  const float v = (c.fy * t[1]) / t[2] + c.cy;
  if (!std::isfinite(u) || !std::isfinite(v) || !std::isfinite(lam)) return k;
  // 11. box
  const float fx0 = std::fmax(0.0f, std::ceil(u - r));
  const float fx1 = std::fmin(W - 1.0f, std::floor(u + r));
  const float fy0 = std::fmax(0.0f, std::ceil(v - r));
  const float fy1 = std::fmin(H - 1.0f, std::floor(v + r));
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) return k;
  if (!(o >= 1.0f / 255.0f)) return k;
  k.visible = true;
  k.z = t[2];
  std::memcpy(&k.zbits, &k.z, 4);
  k.x0 = (int)fx0; k.x1 = (int)fx1; k.y0 = (int)fy0; k.y1 = (int)fy1;
  // 12-13. the tile footprint (A50)
  k.tiles = footprint_rows(ca, cb, cc, det, u, v, o, k.x0, k.x1, k.y0, k.y1, k.rows);
  return k;
}

// Whether pixel (X, Y)'s tile is in the A50 footprint of k (the tile lists the
// GPU walks): the visited-entry statistics P_fwd / P_bwd count only those.
inline bool in_footprint(const KeyReplica& k, int X, int Y) {
  if (k.rows[0] == 0xFFFFFFFFu && k.rows[1] == 0xFFFFFFFFu && k.rows[2] == 0xFFFFFFFFu &&
      k.rows[3] == 0xFFFFFFFFu)
    return true;
  const int kk = Y / 16 - k.y0 / 16;
  if (kk < 0 || kk > 7) return false;
  const uint32_t span = (k.rows[kk >> 1] >> (16 * (kk & 1))) & 0xFFFFu;
  const int tx = X / 16 - k.x0 / 16;
  return (int)(span & 0xFFu) <= tx && tx <= (int)(span >> 8);
}

// ------------------------------------------------ O2: double projection ----
struct Proj {
  KeyReplica key;
  // double quantities (O2)
  double p[3], t[3];
  double qn, qh[4];
  double R[3][3];
  double s[3];
  double Sig[3][3];
  double lx, ly, txtz, tytz;
  bool clx, cly;  // Jacobian clamp active
  double J00, J02, J11, J12;
  double M[2][3];
  double a, b, c, det;
  double A, B, C;
  double u, v, o;
  double dir[3], dist;
  double col[3];
  int clampbits;
};

Proj project_one(const OCam& c, const Params& P, int i) {
  Proj g;
  std::memset(&g, 0, sizeof(g));
  g.key = key_replica(c, P, i);
  if (!g.key.visible) return g;
  const bool kp = P.kept(i);
  double V[3][4];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 4; ++b) V[a][b] = c.viewmat[4 * a + b];
  for (int a = 0; a < 3; ++a) g.p[a] = P.pos_opa[4 * i + a];
  g.o = kp ? (double)P.pos_opa[4 * i + 3] : 0.0;
  for (int a = 0; a < 3; ++a) g.s[a] = kp ? (double)P.scale[4 * i + a] : 0.0;
  // 1. t = W p + t_w  (Eq. 7's viewing transform W)
  for (int a = 0; a < 3; ++a) g.t[a] = V[a][0] * g.p[0] + V[a][1] * g.p[1] + V[a][2] * g.p[2] + V[a][3];
  // 3. q̂ (R from a quaternion)
  double q[4];
  for (int a = 0; a < 4; ++a) q[a] = P.rot[4 * i + a];
  g.qn = norm4(q);
  for (int a = 0; a < 4; ++a) g.qh[a] = q[a] / g.qn;
  const double w = g.qh[0], x = g.qh[1], y = g.qh[2], z = g.qh[3];
  // 4. R(q̂)
  g.R[0][0] = 1 - 2 * (y * y + z * z); g.R[0][1] = 2 * (x * y - w * z); g.R[0][2] = 2 * (x * z + w * y);
  g.R[1][0] = 2 * (x * y + w * z); g.R[1][1] = 1 - 2 * (x * x + z * z); g.R[1][2] = 2 * (y * z - w * x);
  g.R[2][0] = 2 * (x * z - w * y); g.R[2][1] = 2 * (y * z + w * x); g.R[2][2] = 1 - 2 * (x * x + y * y);
  // 5. Σ = R S S^T R^T (Eq. 6)
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += g.R[a][k] * g.s[k] * g.s[k] * g.R[b][k];
      g.Sig[a][b] = acc;
    }
  // 6. J, the affine Jacobian of the projection (Eq. 7), guard band (A08)
  g.lx = 1.3 * c.width / (2.0 * c.fx);
  g.ly = 1.3 * c.height / (2.0 * c.fy);
  g.txtz = g.t[0] / g.t[2];
  g.tytz = g.t[1] / g.t[2];
  g.clx = (g.txtz < -g.lx) || (g.txtz > g.lx);
  g.cly = (g.tytz < -g.ly) || (g.tytz > g.ly);
  const double xt = g.t[2] * std::min(g.lx, std::max(-g.lx, g.txtz));
  const double yt = g.t[2] * std::min(g.ly, std::max(-g.ly, g.tytz));
  g.J00 = c.fx / g.t[2];
  g.J02 = -c.fx * xt / (g.t[2] * g.t[2]);
  g.J11 = c.fy / g.t[2];
  g.J12 = -c.fy * yt / (g.t[2] * g.t[2]);
  // 7. Σ_2D = J W Σ W^T J^T + 0.3 I (Eq. 7; low-pass A07)
  for (int k = 0; k < 3; ++k) {
    g.M[0][k] = g.J00 * V[0][k] + g.J02 * V[2][k];
    g.M[1][k] = g.J11 * V[1][k] + g.J12 * V[2][k];
  }
  double S2[2][2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) acc += g.M[a][k] * g.Sig[k][l] * g.M[b][l];
      S2[a][b] = acc;
    }
  g.a = S2[0][0] + 0.3;
  g.b = S2[0][1];
  g.c = S2[1][1] + 0.3;
  // 8. conic = Σ_2D^{-1}
  g.det = g.a * g.c - g.b * g.b;
  g.A = g.c / g.det;
  g.B = -g.b / g.det;
  g.C = g.a / g.det;
  // 10. pixel mean (pinhole, A19)
  g.u = c.fx * g.t[0] / g.t[2] + c.cx;
  g.v = c.fy * g.t[1] / g.t[2] + c.cy;
  // 12. view-dependent colour c_i (A14)
  double cam[3];
  for (int a = 0; a < 3; ++a) cam[a] = -(V[0][a] * V[0][3] + V[1][a] * V[1][3] + V[2][a] * V[2][3]);
  double dv[3] = {g.p[0] - cam[0], g.p[1] - cam[1], g.p[2] - cam[2]};
  g.dist = std::sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
  for (int a = 0; a < 3; ++a) g.dir[a] = dv[a] / g.dist;
  double Y[16], dY[16][3];
  sh_basis(P.deg, g.dir, Y, dY);
  g.clampbits = 0;
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.5;
    for (int k = 0; k < P.ncoef(); ++k) acc += Y[k] * P.shc(i, k, ch);
    if (acc < 0) { g.clampbits |= (1 << ch); acc = 0; }
    g.col[ch] = acc;
  }
  return g;
}

std::vector<Proj> project_all(const OCam& c, const Params& P) {
  std::vector<Proj> out(P.n);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < P.n; ++i) out[i] = project_one(c, P, i);
  return out;
}

// Global front-to-back order: visible Gaussians by (fp32 depth bits, index)
// (A01-A03).
std::vector<int> depth_order(const std::vector<Proj>& G) {
  std::vector<int> ord;
  for (int i = 0; i < (int)G.size(); ++i)
    if (G[i].key.visible) ord.push_back(i);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) {
    if (G[a].key.zbits != G[b].key.zbits) return G[a].key.zbits < G[b].key.zbits;
    return a < b;
  });
  return ord;
}

// ------------------------------------------ per-pixel evaluation (O4) ------
struct Eval {
  bool inbox;
  double dx, dy, power, G, oG, alpha;
};

inline bool box_has(const Proj& g, int X, int Y) {
  return X >= g.key.x0 && X <= g.key.x1 && Y >= g.key.y0 && Y <= g.key.y1;
}

inline Eval eval_at(const Proj& g, int X, int Y) {
  Eval e;
  e.inbox = box_has(g, X, Y);
  e.dx = g.u - X;
  e.dy = g.v - Y;
  e.power = -0.5 * (g.A * e.dx * e.dx + g.C * e.dy * e.dy) - g.B * e.dx * e.dy;
  e.G = std::exp(e.power);
  e.oG = g.o * e.G;
  e.alpha = std::min(0.99, e.oG);
  return e;
}

const double ALPHA_MIN = 1.0 / 255.0;
const double T_MIN = 1e-4;

// Tie margins (A29): relative widths around each decision threshold.
struct TieEps {
  double alpha_rel;   // |α − 1/255| < alpha_rel·(1/255)
  double t_rel;       // |T(1−α) − 1e-4| < t_rel·1e-4
  double clamp_rel;   // |oG − 0.99| < clamp_rel·0.99  (gradient kink only)
  double power_rel;   // |power| < power_rel·(|A dx²| + |C dy²| + |2B dx dy|) + 1e-12
};

TieEps tie_from(const double* eps) {
  TieEps t;
  t.alpha_rel = eps ? eps[0] : 1e-5;
  t.t_rel = eps ? eps[1] : 3e-5;
  t.clamp_rel = eps ? eps[2] : 1e-5;
  t.power_rel = eps ? eps[3] : 1e-6;
  return t;
}

// Which decisions of one (pixel, entry) evaluation lie inside their tie margin:
// bit 0 the power > 0 guard, bit 1 the α < 1/255 skip, bit 2 the α = 0.99 clamp
// (a derivative kink only), bit 3 the T(1−α) < 1e-4 termination.
enum { TIE_POWER = 1, TIE_ALPHA = 2, TIE_CLAMP = 4, TIE_TERM = 8 };
inline int tie_bits(const Proj& g, const Eval& e, double T, const TieEps& te) {
  const double mag = std::fabs(g.A * e.dx * e.dx) + std::fabs(g.C * e.dy * e.dy) +
                     std::fabs(2 * g.B * e.dx * e.dy);
  int b = 0;
  if (std::fabs(e.power) < te.power_rel * mag + 1e-12 && e.power != 0.0) b |= TIE_POWER;
  if (std::fabs(e.alpha - ALPHA_MIN) < te.alpha_rel * ALPHA_MIN) b |= TIE_ALPHA;
  if (std::fabs(e.oG - 0.99) < te.clamp_rel * 0.99) b |= TIE_CLAMP;
  // the termination test is a decision only for an entry that passes (or ties
  // at) the power and α tests: a skipped entry's T(1 − α) decides nothing
  const bool reaches_term = (!(e.power > 0) || (b & TIE_POWER)) &&
                            (!(e.alpha < ALPHA_MIN) || (b & TIE_ALPHA));
  if (reaches_term && std::fabs(T * (1 - e.alpha) - T_MIN) < te.t_rel * T_MIN) b |= TIE_TERM;
  return b;
}
inline bool is_tie(const Proj& g, const Eval& e, double T, const TieEps& te) {
  return tie_bits(g, e, T, te) != 0;
}

// Output of a forward pass.
struct FwdOut {
  double* img;       // [3][H][W]
  double* Tfin;      // [H][W]
  int32_t* nacc;     // [H][W] accepted count
  int32_t* last_id;  // [H][W] Gaussian id of last accepted, -1 if none
  int32_t* last_pos; // [H][W] position in the global order of last accepted, -1
  uint8_t* tie;      // [H][W]
  uint8_t* term;     // [H][W] 1 if terminated early
  int64_t* pfwd;     // [H][W] entries visited (inbox, incl. terminating)
  int64_t* pbwd;     // [H][W] inbox entries up to last accepted
};

// One pixel, literal form: the definition of Eq. 8.
void pixel_forward(const std::vector<Proj>& G, const std::vector<int>& ord, int X, int Y,
                   const double bg[3], const TieEps& te, double C[3], double& T, int& nacc,
                   int& last_id, int& last_pos, bool& tie, bool& term, int64_t& pf, int64_t& pb) {
  C[0] = C[1] = C[2] = 0;
  T = 1;
  nacc = 0; last_id = -1; last_pos = -1; tie = false; term = false; pf = 0; pb = 0;
  int64_t inbox_count = 0;
  int64_t inbox_at_last = 0;
  for (int pos = 0; pos < (int)ord.size(); ++pos) {
    const Proj& g = G[ord[pos]];
    if (!box_has(g, X, Y)) continue;
    Eval e = eval_at(g, X, Y);
    if (in_footprint(g.key, X, Y)) ++inbox_count;
    if (is_tie(g, e, T, te)) tie = true;
    if (e.power > 0) continue;
    if (e.alpha < ALPHA_MIN) continue;
    const double tn = T * (1 - e.alpha);
    if (tn < T_MIN) { term = true; break; }
    for (int ch = 0; ch < 3; ++ch) C[ch] += g.col[ch] * e.alpha * T;
    T = tn;
    ++nacc;
    last_id = ord[pos];
    last_pos = pos;
    inbox_at_last = inbox_count;
  }
  pf = inbox_count;
  pb = inbox_at_last;
  for (int ch = 0; ch < 3; ++ch) C[ch] += T * bg[ch];
}

struct Grad2D {
  double u, v, A, B, C, o, col[3];
};

// Accumulate one pixel's terms into the sum and, for the conditioning
// measure κ (Σ_px |term|, used to recognise cancelling sums), their magnitudes.
inline void accumulate(Grad2D& sum, Grad2D& kap, const Grad2D& t) {
  sum.u += t.u; sum.v += t.v; sum.A += t.A; sum.B += t.B; sum.C += t.C; sum.o += t.o;
  kap.u += std::fabs(t.u); kap.v += std::fabs(t.v); kap.A += std::fabs(t.A);
  kap.B += std::fabs(t.B); kap.C += std::fabs(t.C); kap.o += std::fabs(t.o);
  for (int ch = 0; ch < 3; ++ch) { sum.col[ch] += t.col[ch]; kap.col[ch] += std::fabs(t.col[ch]); }
}

// The 9 per-pixel terms of one accepted entry (O5).
inline Grad2D pixel_terms(double A, double B, double C, double o, const double* col,
                          double alpha, double G, double oG, double dx, double dy, double Tk,
                          double dL_dalpha, const double g[3], int clamped = -1) {
  Grad2D t{0, 0, 0, 0, 0, 0, {0, 0, 0}};
  (void)col;
  for (int ch = 0; ch < 3; ++ch) t.col[ch] = alpha * Tk * g[ch];
  if (clamped < 0 ? oG < 0.99 : clamped == 0) {  // unclamped α: α = o·G (A17)
    t.o = G * dL_dalpha;
    const double dpow = o * G * dL_dalpha;
    t.u = dpow * (-(A * dx + B * dy));
    t.v = dpow * (-(B * dx + C * dy));
    t.A = dpow * (-0.5 * dx * dx);
    t.B = dpow * (-dx * dy);
    t.C = dpow * (-0.5 * dy * dy);
  }
  return t;
}

// Gradients of one pixel's composite w.r.t. its accepted entries (O5),
// literal form: explicit accepted list, suffix sums (derivative of Eq. 8).
void pixel_backward(const std::vector<Proj>& G, const std::vector<int>& ord, int X, int Y,
                    const double bg[3], const double g[3], std::vector<Grad2D>& g2d,
                    std::vector<Grad2D>& kap) {
  struct Acc { int id; Eval e; double T; };
  std::vector<Acc> acc;
  double T = 1;
  for (int pos = 0; pos < (int)ord.size(); ++pos) {
    const Proj& p = G[ord[pos]];
    if (!box_has(p, X, Y)) continue;
    Eval e = eval_at(p, X, Y);
    if (e.power > 0 || e.alpha < ALPHA_MIN) continue;
    const double tn = T * (1 - e.alpha);
    if (tn < T_MIN) break;
    acc.push_back({ord[pos], e, T});
    T = tn;
  }
  const double Tfin = T;
  double S[3] = {0, 0, 0};  // Σ_{j>k} col_j α_j T_j
  for (int k = (int)acc.size() - 1; k >= 0; --k) {
    const Proj& p = G[acc[k].id];
    const Eval& e = acc[k].e;
    const double Tk = acc[k].T;
    double dL_dalpha = 0;
    for (int ch = 0; ch < 3; ++ch)
      dL_dalpha += g[ch] * (p.col[ch] * Tk - (S[ch] + Tfin * bg[ch]) / (1 - e.alpha));
    accumulate(g2d[acc[k].id], kap[acc[k].id],
               pixel_terms(p.A, p.B, p.C, p.o, p.col, e.alpha, e.G, e.oG, e.dx, e.dy, Tk, dL_dalpha, g));
    for (int ch = 0; ch < 3; ++ch) S[ch] += p.col[ch] * e.alpha * Tk;
  }
}

// Tie slack (A29): the per-pixel 2D terms of every entry of one pixel's sequence
// when its flip_k-th tie decision point (0-based; −1: none, the oracle's own
// decisions) is taken the other way — every decision inside its margin at that
// entry is inverted, the rest of the sequence re-evaluated.  A tie pixel's
// contribution to a gradient may legitimately be either branch's, so the
// comparison allows Σ_tie px |terms_A − terms_B| there instead of excluding
// whole Gaussians.  Returns the number of tie decision points (branch A).
int pixel_branch_terms(const std::vector<Proj>& G, const std::vector<int>& ord, int X, int Y,
                       const double bg[3], const double g[3], const TieEps& te, int flip_k,
                       std::vector<std::pair<int, Grad2D>>& out) {
  struct Acc { int id; Eval e; double T; int clamped; };
  std::vector<Acc> acc;
  double T = 1;
  int nt = 0;
  for (int pos = 0; pos < (int)ord.size(); ++pos) {
    const Proj& p = G[ord[pos]];
    if (!box_has(p, X, Y)) continue;
    const Eval e = eval_at(p, X, Y);
    const int tb = tie_bits(p, e, T, te);
    int flip = 0;
    if (tb) { if (nt == flip_k) flip = tb; ++nt; }
    bool skip_pow = e.power > 0, skip_a = e.alpha < ALPHA_MIN;
    int clamped = e.oG >= 0.99 ? 1 : 0;
    if (flip & TIE_POWER) skip_pow = !skip_pow;
    if (flip & TIE_ALPHA) skip_a = !skip_a;
    if (flip & TIE_CLAMP) clamped = 1 - clamped;
    if (skip_pow || skip_a) continue;
    const double tn = T * (1 - e.alpha);
    bool stop = tn < T_MIN;
    if (flip & TIE_TERM) stop = !stop;
    if (stop) break;
    acc.push_back({ord[pos], e, T, clamped});
    T = tn;
  }
  const double Tfin = T;
  double S[3] = {0, 0, 0};
  out.clear();
  for (int k = (int)acc.size() - 1; k >= 0; --k) {
    const Proj& p = G[acc[k].id];
    const Eval& e = acc[k].e;
    const double Tk = acc[k].T;
    double dL_dalpha = 0;
    for (int ch = 0; ch < 3; ++ch)
      dL_dalpha += g[ch] * (p.col[ch] * Tk - (S[ch] + Tfin * bg[ch]) / (1 - e.alpha));
    out.push_back({acc[k].id, pixel_terms(p.A, p.B, p.C, p.o, p.col, e.alpha, e.G, e.oG, e.dx,
                                          e.dy, Tk, dL_dalpha, g, acc[k].clamped)});
    for (int ch = 0; ch < 3; ++ch) S[ch] += p.col[ch] * e.alpha * Tk;
  }
  return nt;
}

// ---------------------------------------- O5 preprocess backward (chain) ---
struct Grad3D {
  double p[3], o, s[3], q[4];
  double sh[16][3];
};

void preprocess_backward(const OCam& c, const Params& P, int i, const Proj& g,
                         const Grad2D& d, Grad3D& out) {
  std::memset(&out, 0, sizeof(out));
  if (!g.key.visible) return;
  const bool kp = P.kept(i);
  double V[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) V[a][b] = c.viewmat[4 * a + b];
  // colour: clamped channels carry no gradient
  double gcol[3];
  for (int ch = 0; ch < 3; ++ch) gcol[ch] = (g.clampbits >> ch) & 1 ? 0.0 : d.col[ch];
  double Y[16], dY[16][3];
  sh_basis(P.deg, g.dir, Y, dY);
  double gdir[3] = {0, 0, 0};
  for (int k = 0; k < P.ncoef(); ++k)
    for (int ch = 0; ch < 3; ++ch) {
      out.sh[k][ch] = Y[k] * gcol[ch];
      for (int a = 0; a < 3; ++a) gdir[a] += gcol[ch] * P.shc(i, k, ch) * dY[k][a];
    }
  // d = (p − cam)/‖p − cam‖ → dL/dp += (I − d dᵀ) dL/dd / dist
  const double dd = g.dir[0] * gdir[0] + g.dir[1] * gdir[1] + g.dir[2] * gdir[2];
  for (int a = 0; a < 3; ++a) out.p[a] += (gdir[a] - g.dir[a] * dd) / g.dist;
  // opacity (Eq. 1: o_r = keep·o)
  out.o = kp ? d.o : 0.0;
  // conic → Σ_2D:  dL/dΣ' = −K Ĝ K with Ĝ = [[gA, gB/2],[gB/2, gC]]
  const double K[2][2] = {{g.A, g.B}, {g.B, g.C}};
  const double Gh[2][2] = {{d.A, 0.5 * d.B}, {0.5 * d.B, d.C}};
  double KG[2][2], Gs[2][2];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) KG[a][b] = K[a][0] * Gh[0][b] + K[a][1] * Gh[1][b];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) Gs[a][b] = -(KG[a][0] * K[0][b] + KG[a][1] * K[1][b]);
  // Σ' = M Σ Mᵀ + 0.3 I:  dL/dΣ = Mᵀ Gs M ;  dL/dM = 2 Gs M Σ
  double GSig[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) acc += g.M[k][a] * Gs[k][l] * g.M[l][b];
      GSig[a][b] = acc;
    }
  double GM[2][3];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 3; ++l) acc += Gs[a][k] * g.M[k][l] * g.Sig[l][b];
      GM[a][b] = 2 * acc;
    }
  // M = J W → dL/dJ = dL/dM Wᵀ  (only J00, J02, J11, J12 are variables)
  double GJ[2][3];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 3; ++b) GJ[a][b] = GM[a][0] * V[b][0] + GM[a][1] * V[b][1] + GM[a][2] * V[b][2];
  // J(t) with the exact derivative of the guard-band clamp (A08)
  const double tx = g.t[0], ty = g.t[1], tz = g.t[2];
  const double tz2 = tz * tz, tz3 = tz2 * tz;
  const double xt = tz * std::min(g.lx, std::max(-g.lx, g.txtz));
  const double yt = tz * std::min(g.ly, std::max(-g.ly, g.tytz));
  double gt[3] = {0, 0, 0};
  // J00 = fx/tz, J11 = fy/tz
  gt[2] += GJ[0][0] * (-c.fx / tz2) + GJ[1][1] * (-c.fy / tz2);
  // J02 = −fx x̃/tz²
  if (!g.clx) {
    gt[0] += GJ[0][2] * (-c.fx / tz2);
    gt[2] += GJ[0][2] * (2 * c.fx * tx / tz3);
  } else {
    gt[2] += GJ[0][2] * (c.fx * xt / tz3);
  }
  if (!g.cly) {
    gt[1] += GJ[1][2] * (-c.fy / tz2);
    gt[2] += GJ[1][2] * (2 * c.fy * ty / tz3);
  } else {
    gt[2] += GJ[1][2] * (c.fy * yt / tz3);
  }
  // mean: u = fx tx/tz + cx, v = fy ty/tz + cy
  gt[0] += d.u * c.fx / tz;
  gt[2] += d.u * (-c.fx * tx / tz2);
  gt[1] += d.v * c.fy / tz;
  gt[2] += d.v * (-c.fy * ty / tz2);
  // t = W p + t_w → dL/dp = Wᵀ dL/dt
  for (int a = 0; a < 3; ++a) out.p[a] += V[0][a] * gt[0] + V[1][a] * gt[1] + V[2][a] * gt[2];
  // Σ = R diag(s²) Rᵀ
  double RtGR[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) acc += g.R[k][a] * GSig[k][l] * g.R[l][b];
      RtGR[a][b] = acc;
    }
  for (int k = 0; k < 3; ++k) out.s[k] = kp ? 2 * g.s[k] * RtGR[k][k] : 0.0;
  double GR[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += GSig[a][k] * g.R[k][b];
      GR[a][b] = 2 * acc * g.s[b] * g.s[b];
    }
  // R(q̂) partials
  const double w = g.qh[0], x = g.qh[1], y = g.qh[2], z = g.qh[3];
  double gq[4] = {0, 0, 0, 0};
  gq[0] = GR[0][1] * (-2 * z) + GR[0][2] * (2 * y) + GR[1][0] * (2 * z) + GR[1][2] * (-2 * x) +
          GR[2][0] * (-2 * y) + GR[2][1] * (2 * x);
  gq[1] = GR[0][1] * (2 * y) + GR[0][2] * (2 * z) + GR[1][0] * (2 * y) + GR[1][1] * (-4 * x) +
          GR[1][2] * (-2 * w) + GR[2][0] * (2 * z) + GR[2][1] * (2 * w) + GR[2][2] * (-4 * x);
  gq[2] = GR[0][0] * (-4 * y) + GR[0][1] * (2 * x) + GR[0][2] * (2 * w) + GR[1][0] * (2 * x) +
          GR[1][2] * (2 * z) + GR[2][0] * (-2 * w) + GR[2][1] * (2 * z) + GR[2][2] * (-4 * y);
  gq[3] = GR[0][0] * (-4 * z) + GR[0][1] * (-2 * w) + GR[0][2] * (2 * x) + GR[1][0] * (2 * w) +
          GR[1][1] * (-4 * z) + GR[1][2] * (2 * y) + GR[2][0] * (2 * x) + GR[2][1] * (2 * y);
  // q̂ = q/‖q‖
  const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
  for (int a = 0; a < 4; ++a) out.q[a] = (gq[a] - g.qh[a] * dot) / g.qn;
}

struct RenderCtx {
  OCam cam;
  Params P;
  std::vector<Proj> G;
  std::vector<int> ord;
};

void make_ctx(RenderCtx& R, const OCam* cam, int n, int deg, const float* pos_opa,
              const float* scale, const float* rot, const float* sh, const uint8_t* keep) {
  R.cam = *cam;
  R.P.n = n; R.P.deg = deg; R.P.pos_opa = pos_opa; R.P.scale = scale; R.P.rot = rot;
  R.P.sh = sh; R.P.keep = keep;
  R.G = project_all(R.cam, R.P);
  R.ord = depth_order(R.G);
}

// Scatter form of O4: walks the global order once, splatting each Gaussian
// into its box while carrying every pixel's (C, T, done) state.  Per pixel it
// performs exactly the op sequence of pixel_forward (bit-identical results),
// at O(Σ box area) cost.  Row bands are independent → OpenMP over bands.
void scatter_forward(const RenderCtx& R, const double bg[3], const TieEps& te, FwdOut& o) {
  const int W = R.cam.width, H = R.cam.height;
  const size_t np = (size_t)W * H;
  std::vector<uint8_t> done(np, 0);
  std::vector<int64_t> inbox(np, 0), inbox_last(np, 0);
  for (size_t p = 0; p < np; ++p) {
    o.img[p] = o.img[np + p] = o.img[2 * np + p] = 0;
    o.Tfin[p] = 1; o.nacc[p] = 0; o.last_id[p] = -1; o.last_pos[p] = -1; o.tie[p] = 0; o.term[p] = 0;
  }
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  const int band = std::max(1, (H + nth * 4 - 1) / (nth * 4));
  const int nb = (H + band - 1) / band;
#pragma omp parallel for schedule(dynamic, 1)
  for (int bi = 0; bi < nb; ++bi) {
    const int ylo = bi * band, yhi = std::min(H - 1, ylo + band - 1);
    for (int pos = 0; pos < (int)R.ord.size(); ++pos) {
      const Proj& g = R.G[R.ord[pos]];
      const int y0 = std::max(g.key.y0, ylo), y1 = std::min(g.key.y1, yhi);
      for (int Y = y0; Y <= y1; ++Y)
        for (int X = g.key.x0; X <= g.key.x1; ++X) {
          const size_t p = (size_t)Y * W + X;
          if (done[p]) continue;
          Eval e = eval_at(g, X, Y);
          if (in_footprint(g.key, X, Y)) ++inbox[p];
          double& T = o.Tfin[p];
          if (is_tie(g, e, T, te)) o.tie[p] = 1;
          if (e.power > 0 || e.alpha < ALPHA_MIN) continue;
          const double tn = T * (1 - e.alpha);
          if (tn < T_MIN) { done[p] = 1; o.term[p] = 1; continue; }
          for (int ch = 0; ch < 3; ++ch) o.img[ch * np + p] += g.col[ch] * e.alpha * T;
          T = tn;
          o.nacc[p] += 1;
          o.last_id[p] = R.ord[pos];
          o.last_pos[p] = pos;
          inbox_last[p] = inbox[p];
        }
    }
  }
  for (size_t p = 0; p < np; ++p) {
    for (int ch = 0; ch < 3; ++ch) o.img[ch * np + p] += o.Tfin[p] * bg[ch];
    if (o.pfwd) o.pfwd[p] = inbox[p];
    if (o.pbwd) o.pbwd[p] = inbox_last[p];
  }
}

// Scatter form of O5's raster part: reverse global order; per pixel the
// transmittance before entry k is recovered as T_k = T_{k+1}/(1−α_k) in double.
void scatter_backward(const RenderCtx& R, const double bg[3], const float* dL, const double* Tfin,
                      const int32_t* last_pos, std::vector<Grad2D>& g2d, std::vector<Grad2D>& kap) {
  const int W = R.cam.width, H = R.cam.height;
  const size_t np = (size_t)W * H;
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  const int band = std::max(1, (H + nth * 4 - 1) / (nth * 4));
  const int nb = (H + band - 1) / band;
  std::vector<double> Tcur(Tfin, Tfin + np);
  std::vector<double> S(3 * np, 0.0);
  std::vector<std::vector<Grad2D>> part(nb), kpart(nb);
#pragma omp parallel for schedule(dynamic, 1)
  for (int bi = 0; bi < nb; ++bi) {
    std::vector<Grad2D>& mine = part[bi];
    std::vector<Grad2D>& kmine = kpart[bi];
    mine.assign(R.G.size(), Grad2D{0, 0, 0, 0, 0, 0, {0, 0, 0}});
    kmine.assign(R.G.size(), Grad2D{0, 0, 0, 0, 0, 0, {0, 0, 0}});
    const int ylo = bi * band, yhi = std::min(H - 1, ylo + band - 1);
    for (int pos = (int)R.ord.size() - 1; pos >= 0; --pos) {
      const int id = R.ord[pos];
      const Proj& g = R.G[id];
      const int y0 = std::max(g.key.y0, ylo), y1 = std::min(g.key.y1, yhi);
      for (int Y = y0; Y <= y1; ++Y)
        for (int X = g.key.x0; X <= g.key.x1; ++X) {
          const size_t p = (size_t)Y * W + X;
          if (pos > last_pos[p]) continue;
          Eval e = eval_at(g, X, Y);
          if (e.power > 0 || e.alpha < ALPHA_MIN) continue;
          const double Tk = Tcur[p] / (1 - e.alpha);
          const double gg[3] = {dL[p], dL[np + p], dL[2 * np + p]};
          double dL_dalpha = 0;
          for (int ch = 0; ch < 3; ++ch)
            dL_dalpha += gg[ch] * (g.col[ch] * Tk - (S[ch * np + p] + Tfin[p] * bg[ch]) / (1 - e.alpha));
          accumulate(mine[id], kmine[id],
                     pixel_terms(g.A, g.B, g.C, g.o, g.col, e.alpha, e.G, e.oG, e.dx, e.dy, Tk, dL_dalpha, gg));
          for (int ch = 0; ch < 3; ++ch) S[ch * np + p] += g.col[ch] * e.alpha * Tk;
          Tcur[p] = Tk;
        }
    }
  }
  // deterministic reduction in band order
  for (int bi = 0; bi < nb; ++bi)
    for (size_t i = 0; i < R.G.size(); ++i) {
      Grad2D z{0, 0, 0, 0, 0, 0, {0, 0, 0}};
      accumulate(g2d[i], z, part[bi][i]);
      accumulate(kap[i], z, kpart[bi][i]);
    }
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------ O1 -----
// §3.3: p' = p + μ, q' = norm(q) × norm(σ) where mask = 1; copy else.
int oracle_shift(int n, const float* pos_opa, const float* rot, const float* mu,
                 const float* sigma, const uint8_t* mask, double* pos_out, double* rot_out) {
  for (int i = 0; i < n; ++i) {
    const bool m = mask == nullptr || mask[i] != 0;
    for (int a = 0; a < 4; ++a) {
      pos_out[4 * i + a] = pos_opa[4 * i + a];
      rot_out[4 * i + a] = rot[4 * i + a];
    }
    if (!m) continue;
    for (int a = 0; a < 3; ++a) pos_out[4 * i + a] = (double)pos_opa[4 * i + a] + (double)mu[4 * i + a];
    double q[4], s[4];
    for (int a = 0; a < 4; ++a) { q[a] = rot[4 * i + a]; s[a] = sigma[4 * i + a]; }
    const double nq = norm4(q), ns = norm4(s);
    for (int a = 0; a < 4; ++a) q[a] /= nq;
    if (ns < 1e-8) { s[0] = 1; s[1] = s[2] = s[3] = 0; }
    else for (int a = 0; a < 4; ++a) s[a] /= ns;
    double o[4];
    qmul(q, s, o);
    for (int a = 0; a < 4; ++a) rot_out[4 * i + a] = o[a];
  }
  return 0;
}

// Reverse of O1 w.r.t. (μ, σ) (SURVEY O5 "Shift").
int oracle_shift_bwd(int n, const float* rot, const float* sigma, const uint8_t* mask,
                     const double* g_pos_out, const double* g_rot_out, double* g_mu,
                     double* g_sigma) {
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 4; ++a) { g_mu[4 * i + a] = 0; g_sigma[4 * i + a] = 0; }
    const bool m = mask == nullptr || mask[i] != 0;
    if (!m) continue;
    for (int a = 0; a < 3; ++a) g_mu[4 * i + a] = g_pos_out[4 * i + a];
    double q[4], s[4];
    for (int a = 0; a < 4; ++a) { q[a] = rot[4 * i + a]; s[a] = sigma[4 * i + a]; }
    const double nq = norm4(q), ns = norm4(s);
    if (ns < 1e-8) continue;
    for (int a = 0; a < 4; ++a) { q[a] /= nq; s[a] /= ns; }
    // q' = L(q̂) ŝ  →  dL/dŝ = L(q̂)ᵀ dL/dq'
    const double L[4][4] = {{q[0], -q[1], -q[2], -q[3]},
                            {q[1], q[0], -q[3], q[2]},
                            {q[2], q[3], q[0], -q[1]},
                            {q[3], -q[2], q[1], q[0]}};
    double gs[4];
    for (int b = 0; b < 4; ++b) {
      gs[b] = 0;
      for (int a = 0; a < 4; ++a) gs[b] += L[a][b] * g_rot_out[4 * i + a];
    }
    const double dot = s[0] * gs[0] + s[1] * gs[1] + s[2] * gs[2] + s[3] * gs[3];
    for (int a = 0; a < 4; ++a) g_sigma[4 * i + a] = (gs[a] - s[a] * dot) / ns;
  }
  return 0;
}

// ------------------------------------------------------------------ O2 -----
// Outputs (all [n]-major): uvz double[3n]; conic double[3n] (A,B,C);
// opa double[n]; rgb double[3n]; clampbits int32[n];
// key replica: zf float[n], zbits uint32[n], box int32[4n] (x0,x1,y0,y1),
// tiles uint32[n], visible uint8[n].  Any output may be null.
int oracle_project(const OCam* cam, int n, int deg, const float* pos_opa, const float* scale,
                   const float* rot, const float* sh, const uint8_t* keep, double* uvz,
                   double* conic, double* opa, double* rgb, int32_t* clampbits, float* zf,
                   uint32_t* zbits, int32_t* box, uint32_t* tiles, uint8_t* visible,
                   uint32_t* rows) {
  Params P{n, deg, pos_opa, scale, rot, sh, keep};
  std::vector<Proj> G = project_all(*cam, P);
  for (int i = 0; i < n; ++i) {
    const Proj& g = G[i];
    if (uvz) { uvz[3 * i] = g.u; uvz[3 * i + 1] = g.v; uvz[3 * i + 2] = g.t[2]; }
    if (conic) { conic[3 * i] = g.A; conic[3 * i + 1] = g.B; conic[3 * i + 2] = g.C; }
    if (opa) opa[i] = g.o;
    if (rgb) for (int ch = 0; ch < 3; ++ch) rgb[3 * i + ch] = g.col[ch];
    if (clampbits) clampbits[i] = g.clampbits;
    if (zf) zf[i] = g.key.z;
    if (zbits) zbits[i] = g.key.zbits;
    if (box) { box[4 * i] = g.key.x0; box[4 * i + 1] = g.key.x1; box[4 * i + 2] = g.key.y0; box[4 * i + 3] = g.key.y1; }
    if (tiles) tiles[i] = g.key.tiles;
    if (visible) visible[i] = g.key.visible ? 1 : 0;
    if (rows) for (int w = 0; w < 4; ++w) rows[4 * i + w] = g.key.rows[w];
  }
  return 0;
}

// Σ' entries (a, b, c) and det in double, for the EWA pins.
int oracle_cov2d(const OCam* cam, int n, const float* pos_opa, const float* scale,
                 const float* rot, double* abcd) {
  std::vector<float> sh(4 * (size_t)n, 0.0f);
  Params P{n, 0, pos_opa, scale, rot, sh.data(), nullptr};
  for (int i = 0; i < n; ++i) {
    Proj g = project_one(*cam, P, i);
    abcd[4 * i] = g.a; abcd[4 * i + 1] = g.b; abcd[4 * i + 2] = g.c; abcd[4 * i + 3] = g.det;
  }
  return 0;
}

// Rotation matrix and covariance of a single Gaussian (pins S:42-62).
int oracle_rotmat_cov(const float* rot4, const float* scale3, double* R9, double* S9) {
  float pos[4] = {0, 0, 5, 1}, sc[4] = {scale3[0], scale3[1], scale3[2], 0};
  float sh[4] = {0, 0, 0, 0};
  OCam c;
  std::memset(&c, 0, sizeof(c));
  c.width = 64; c.height = 64; c.fx = 64; c.fy = 64; c.cx = 31.5f; c.cy = 31.5f;
  c.viewmat[0] = c.viewmat[5] = c.viewmat[10] = 1; c.near_plane = 0.2f;
  Params P{1, 0, pos, sc, rot4, sh, nullptr};
  Proj g = project_one(c, P, 0);
  if (!g.key.visible) return 1;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) { R9[3 * a + b] = g.R[a][b]; S9[3 * a + b] = g.Sig[a][b]; }
  return 0;
}

// SH basis values (for the orthonormality pin).
int oracle_sh_basis(int deg, int m, const double* dirs, double* Y) {
  for (int j = 0; j < m; ++j) {
    double y[16], dy[16][3];
    sh_basis(deg, dirs + 3 * j, y, dy);
    for (int k = 0; k < 16; ++k) Y[16 * j + k] = y[k];
  }
  return 0;
}

// ------------------------------------------------------------------ O3 -----
// Brute-force binning: enumerate every (visible Gaussian, tile of its box)
// pair with key = (tile << 32) | zbits, sort by (key, id).  Returns K; writes
// at most `cap` pairs; ranges [2*num_tiles] ([0,0) for empty tiles).
// O3 with the A50 footprint: the tiles of Gaussian i are, for each tile row k of
// its box, the columns tx0 + lo_k … tx0 + hi_k of rows[i] (row k = 16 bits:
// lo | hi << 8; lo > hi: none); all ones = every tile of the box.  rows null: the
// box rule of A05.
int64_t oracle_bin_sort(const OCam* cam, int n, const uint8_t* visible, const uint32_t* zbits,
                        const int32_t* box, int64_t cap, uint64_t* keys, uint32_t* ids,
                        uint32_t* ranges, const uint32_t* rows) {
  const int tx_n = (cam->width + 15) / 16, ty_n = (cam->height + 15) / 16;
  std::vector<std::pair<uint64_t, uint32_t>> pairs;
  for (int i = 0; i < n; ++i) {
    if (!visible[i]) continue;
    const int tx0 = box[4 * i] / 16, tx1 = box[4 * i + 1] / 16;
    const int ty0 = box[4 * i + 2] / 16, ty1 = box[4 * i + 3] / 16;
    const bool full = rows == nullptr || (rows[4 * i] == 0xFFFFFFFFu && rows[4 * i + 1] == 0xFFFFFFFFu &&
                                          rows[4 * i + 2] == 0xFFFFFFFFu && rows[4 * i + 3] == 0xFFFFFFFFu);
    for (int ty = ty0; ty <= ty1; ++ty) {
      int lo = tx0, hi = tx1;
      if (!full) {
        const int k = ty - ty0;
        const uint32_t span = (rows[4 * i + (k >> 1)] >> (16 * (k & 1))) & 0xFFFFu;
        lo = tx0 + (int)(span & 0xFFu);
        hi = tx0 + (int)(span >> 8);
      }
      for (int tx = lo; tx <= hi; ++tx) {
        const uint64_t tile = (uint64_t)(ty * tx_n + tx);
        pairs.push_back({(tile << 32) | zbits[i], (uint32_t)i});
      }
    }
  }
  std::sort(pairs.begin(), pairs.end());
  const int64_t K = (int64_t)pairs.size();
  if (ranges) for (int t = 0; t < 2 * tx_n * ty_n; ++t) ranges[t] = 0;
  for (int64_t k = 0; k < K && k < cap; ++k) {
    if (keys) keys[k] = pairs[k].first;
    if (ids) ids[k] = pairs[k].second;
  }
  if (ranges && K <= cap) {
    for (int64_t k = 0; k < K; ++k) {
      const uint32_t t = (uint32_t)(pairs[k].first >> 32);
      if (k == 0 || (uint32_t)(pairs[k - 1].first >> 32) != t) ranges[2 * t] = (uint32_t)k;
      if (k == K - 1 || (uint32_t)(pairs[k + 1].first >> 32) != t) ranges[2 * t + 1] = (uint32_t)(k + 1);
    }
  }
  return K;
}

// ------------------------------------------------------------------ O4 -----
// mode 0 = literal (every pixel over every depth-sorted Gaussian), 1 = scatter.
// Outputs: img double[3*H*W], Tfin double[H*W]; nacc/last_id/tie/term/pfwd/pbwd
// per pixel (nullable).  tie_eps: double[4] (nullable → defaults, A29).
int oracle_render(const OCam* cam, int n, int deg, const float* pos_opa, const float* scale,
                  const float* rot, const float* sh, const uint8_t* keep, const float* bg3,
                  int mode, const double* tie_eps, double* img, double* Tfin, int32_t* nacc,
                  int32_t* last_id, uint8_t* tie, uint8_t* term, int64_t* pfwd, int64_t* pbwd) {
  RenderCtx R;
  make_ctx(R, cam, n, deg, pos_opa, scale, rot, sh, keep);
  const double bg[3] = {bg3 ? bg3[0] : 0.0, bg3 ? bg3[1] : 0.0, bg3 ? bg3[2] : 0.0};
  const TieEps te = tie_from(tie_eps);
  const int W = cam->width, H = cam->height;
  const size_t np = (size_t)W * H;
  std::vector<int32_t> nacc_v(np), lid_v(np), lpos_v(np);
  std::vector<uint8_t> tie_v(np), term_v(np);
  std::vector<int64_t> pf_v(np), pb_v(np);
  std::vector<double> T_v(np);
  FwdOut o{img, T_v.data(), nacc_v.data(), lid_v.data(), lpos_v.data(), tie_v.data(),
           term_v.data(), pf_v.data(), pb_v.data()};
  if (mode == 0) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int Y = 0; Y < H; ++Y)
      for (int X = 0; X < W; ++X) {
        const size_t p = (size_t)Y * W + X;
        double C[3], T;
        int na, li, lp;
        bool ti, tm;
        int64_t pf, pb;
        pixel_forward(R.G, R.ord, X, Y, bg, te, C, T, na, li, lp, ti, tm, pf, pb);
        for (int ch = 0; ch < 3; ++ch) img[ch * np + p] = C[ch];
        T_v[p] = T; nacc_v[p] = na; lid_v[p] = li; lpos_v[p] = lp; tie_v[p] = ti; term_v[p] = tm;
        pf_v[p] = pf; pb_v[p] = pb;
      }
  } else {
    scatter_forward(R, bg, te, o);
  }
  for (size_t p = 0; p < np; ++p) {
    if (Tfin) Tfin[p] = T_v[p];
    if (nacc) nacc[p] = nacc_v[p];
    if (last_id) last_id[p] = lid_v[p];
    if (tie) tie[p] = tie_v[p];
    if (term) term[p] = term_v[p];
    if (pfwd) pfwd[p] = pf_v[p];
    if (pbwd) pbwd[p] = pb_v[p];
  }
  return 0;
}

// ------------------------------------------------------------------ O5 -----
// Full backward of one view.  dL_dimg float[3][H][W].  Outputs (=, not +=):
//   g_pos_opa double[4n] (x,y,z, o), g_scale double[4n], g_rot double[4n],
//   g_sh double[n*(d+1)²*3] coefficient-major, g2d double[9n] (u,v,A,B,C,o,r,g,b)
//   gradstat_sum double[n], gradstat_cnt int32[n].  Any output nullable.
// Also renders the forward (img/T nullable).  Tie pixels (A29): for a pixel
// with one tie decision point, t_* (nullable, same layouts as g_*; t_gradstat
// double[n]) receive the |difference| between its two decision branches'
// contributions pushed through |Jacobian| — the amount by which a correct
// fp32 implementation may differ there; Gaussians whose box holds a pixel
// with two or more tie points are flagged in gtie (uint8[n], nullable).
// κ outputs (nullable, same layouts as g_*): the conditioning of each
// gradient entry, Σ_px |L_i|·|per-pixel 2D terms| where L_i is the linear
// preprocess map of Gaussian i (columns by unit probes).  A gradient with
// κ ≫ |g| is a cancelling sum whose fp32 value is only accurate to ~eps·κ.
int oracle_render_bwd(const OCam* cam, int n, int deg, const float* pos_opa, const float* scale,
                      const float* rot, const float* sh, const uint8_t* keep, const float* bg3,
                      const float* dL_dimg, int mode, const double* tie_eps, double* g_pos_opa,
                      double* g_scale, double* g_rot, double* g_sh, double* g2d_out,
                      double* gradstat_sum, int32_t* gradstat_cnt, uint8_t* gtie, double* img_out,
                      double* T_out, double* k_pos_opa, double* k_scale, double* k_rot,
                      double* k_sh, double* t_pos_opa, double* t_scale, double* t_rot,
                      double* t_sh, double* t_gradstat) {
  RenderCtx R;
  make_ctx(R, cam, n, deg, pos_opa, scale, rot, sh, keep);
  const double bg[3] = {bg3 ? bg3[0] : 0.0, bg3 ? bg3[1] : 0.0, bg3 ? bg3[2] : 0.0};
  const TieEps te = tie_from(tie_eps);
  const int W = cam->width, H = cam->height;
  const size_t np = (size_t)W * H;
  std::vector<double> img(3 * np), Tfin(np);
  std::vector<int32_t> nacc(np), lid(np), lpos(np);
  std::vector<uint8_t> tie(np), term(np);
  FwdOut o{img.data(), Tfin.data(), nacc.data(), lid.data(), lpos.data(), tie.data(), term.data(),
           nullptr, nullptr};
  scatter_forward(R, bg, te, o);
  const Grad2D zero{0, 0, 0, 0, 0, 0, {0, 0, 0}};
  std::vector<Grad2D> g2d(n, zero), kap(n, zero);
  if (mode == 0) {
    // literal: every pixel independently, explicit accepted list
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    std::vector<std::vector<Grad2D>> part(nth), kpart(nth);
#pragma omp parallel
    {
      int tid = 0;
#ifdef _OPENMP
      tid = omp_get_thread_num();
#endif
      part[tid].assign(n, zero);
      kpart[tid].assign(n, zero);
#pragma omp for schedule(static)
      for (int Y = 0; Y < H; ++Y)
        for (int X = 0; X < W; ++X) {
          const size_t p = (size_t)Y * W + X;
          const double gg[3] = {dL_dimg[p], dL_dimg[np + p], dL_dimg[2 * np + p]};
          pixel_backward(R.G, R.ord, X, Y, bg, gg, part[tid], kpart[tid]);
        }
    }
    for (int t = 0; t < nth; ++t)
      for (int i = 0; i < n; ++i) {
        Grad2D z = zero;
        accumulate(g2d[i], z, part[t][i]);
        accumulate(kap[i], z, kpart[t][i]);
      }
  } else {
    scatter_backward(R, bg, dL_dimg, Tfin.data(), lpos.data(), g2d, kap);
  }
  // A29 tie slack: for every pixel with exactly one tie decision point, the
  // per-Gaussian |terms_A − terms_B| of its two branches (pixel_branch_terms);
  // a pixel with two or more tie points ("multi-tie") instead flags the
  // Gaussians whose box holds it (gtie), which the comparison excludes.
  std::vector<Grad2D> slack(n, zero);
  std::vector<uint8_t> multi(np, 0);
  const bool want_t = t_pos_opa || t_scale || t_rot || t_sh || t_gradstat || gtie;
  if (want_t) {
    std::vector<size_t> tps;
    for (size_t p = 0; p < np; ++p)
      if (tie[p]) tps.push_back(p);
#pragma omp parallel
    {
      std::vector<std::pair<int, Grad2D>> local, a, b;
#pragma omp for schedule(dynamic, 4)
      for (long k = 0; k < (long)tps.size(); ++k) {
        const size_t p = tps[k];
        const int X = (int)(p % W), Y = (int)(p / W);
        const double gg[3] = {dL_dimg[p], dL_dimg[np + p], dL_dimg[2 * np + p]};
        const int nt = pixel_branch_terms(R.G, R.ord, X, Y, bg, gg, te, -1, a);
        if (nt >= 2) { multi[p] = 1; continue; }
        if (nt == 0) continue;
        pixel_branch_terms(R.G, R.ord, X, Y, bg, gg, te, 0, b);
        std::vector<std::pair<int, Grad2D>> d;   // id → terms_B − terms_A
        auto add = [&](int id, const Grad2D& t, double sgn) {
          for (auto& q : d)
            if (q.first == id) {
              Grad2D& r = q.second;
              r.u += sgn * t.u; r.v += sgn * t.v; r.A += sgn * t.A; r.B += sgn * t.B;
              r.C += sgn * t.C; r.o += sgn * t.o;
              for (int ch = 0; ch < 3; ++ch) r.col[ch] += sgn * t.col[ch];
              return;
            }
          Grad2D r = zero;
          d.push_back({id, r});
          Grad2D& q = d.back().second;
          q.u = sgn * t.u; q.v = sgn * t.v; q.A = sgn * t.A; q.B = sgn * t.B; q.C = sgn * t.C;
          q.o = sgn * t.o;
          for (int ch = 0; ch < 3; ++ch) q.col[ch] = sgn * t.col[ch];
        };
        for (const auto& q : a) add(q.first, q.second, -1.0);
        for (const auto& q : b) add(q.first, q.second, 1.0);
        for (const auto& q : d) local.push_back(q);
      }
#pragma omp critical
      for (const auto& q : local) {
        Grad2D dummy = zero;
        Grad2D z = zero;
        accumulate(dummy, slack[q.first], q.second);   // slack += |Δterms|
        (void)z;
      }
    }
  }
  const int nc = (deg + 1) * (deg + 1);
  const bool want_k = k_pos_opa || k_scale || k_rot || k_sh;
  const bool want_ts = t_pos_opa || t_scale || t_rot || t_sh;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    Grad3D d;
    preprocess_backward(R.cam, R.P, i, R.G[i], g2d[i], d);
    if (g_pos_opa) { for (int a = 0; a < 3; ++a) g_pos_opa[4 * i + a] = d.p[a]; g_pos_opa[4 * i + 3] = d.o; }
    if (g_scale) { for (int a = 0; a < 3; ++a) g_scale[4 * i + a] = d.s[a]; g_scale[4 * i + 3] = 0; }
    if (g_rot) for (int a = 0; a < 4; ++a) g_rot[4 * i + a] = d.q[a];
    if (g_sh) for (int k = 0; k < nc; ++k) for (int ch = 0; ch < 3; ++ch) g_sh[((size_t)i * nc + k) * 3 + ch] = d.sh[k][ch];
    if (want_k) {
      Grad3D kk;
      std::memset(&kk, 0, sizeof(kk));
      const double k9[9] = {kap[i].u, kap[i].v, kap[i].A, kap[i].B, kap[i].C, kap[i].o,
                            kap[i].col[0], kap[i].col[1], kap[i].col[2]};
      for (int c = 0; c < 9; ++c) {
        if (k9[c] == 0) continue;
        Grad2D e = zero;
        double* f[9] = {&e.u, &e.v, &e.A, &e.B, &e.C, &e.o, &e.col[0], &e.col[1], &e.col[2]};
        *f[c] = 1.0;
        Grad3D col;
        preprocess_backward(R.cam, R.P, i, R.G[i], e, col);
        for (int a = 0; a < 3; ++a) { kk.p[a] += std::fabs(col.p[a]) * k9[c]; kk.s[a] += std::fabs(col.s[a]) * k9[c]; }
        kk.o += std::fabs(col.o) * k9[c];
        for (int a = 0; a < 4; ++a) kk.q[a] += std::fabs(col.q[a]) * k9[c];
        for (int k = 0; k < nc; ++k) for (int ch = 0; ch < 3; ++ch) kk.sh[k][ch] += std::fabs(col.sh[k][ch]) * k9[c];
      }
      if (k_pos_opa) { for (int a = 0; a < 3; ++a) k_pos_opa[4 * i + a] = kk.p[a]; k_pos_opa[4 * i + 3] = kk.o; }
      if (k_scale) { for (int a = 0; a < 3; ++a) k_scale[4 * i + a] = kk.s[a]; k_scale[4 * i + 3] = 0; }
      if (k_rot) for (int a = 0; a < 4; ++a) k_rot[4 * i + a] = kk.q[a];
      if (k_sh) for (int k = 0; k < nc; ++k) for (int ch = 0; ch < 3; ++ch) k_sh[((size_t)i * nc + k) * 3 + ch] = kk.sh[k][ch];
    }
    if (want_ts) {   // the tie slack through |preprocess Jacobian|, as κ
      Grad3D kk;
      std::memset(&kk, 0, sizeof(kk));
      const double k9[9] = {slack[i].u, slack[i].v, slack[i].A, slack[i].B, slack[i].C,
                            slack[i].o, slack[i].col[0], slack[i].col[1], slack[i].col[2]};
      for (int c = 0; c < 9; ++c) {
        if (k9[c] == 0) continue;
        Grad2D e = zero;
        double* f[9] = {&e.u, &e.v, &e.A, &e.B, &e.C, &e.o, &e.col[0], &e.col[1], &e.col[2]};
        *f[c] = 1.0;
        Grad3D col;
        preprocess_backward(R.cam, R.P, i, R.G[i], e, col);
        for (int a = 0; a < 3; ++a) { kk.p[a] += std::fabs(col.p[a]) * k9[c]; kk.s[a] += std::fabs(col.s[a]) * k9[c]; }
        kk.o += std::fabs(col.o) * k9[c];
        for (int a = 0; a < 4; ++a) kk.q[a] += std::fabs(col.q[a]) * k9[c];
        for (int k = 0; k < nc; ++k) for (int ch = 0; ch < 3; ++ch) kk.sh[k][ch] += std::fabs(col.sh[k][ch]) * k9[c];
      }
      if (t_pos_opa) { for (int a = 0; a < 3; ++a) t_pos_opa[4 * i + a] = kk.p[a]; t_pos_opa[4 * i + 3] = kk.o; }
      if (t_scale) { for (int a = 0; a < 3; ++a) t_scale[4 * i + a] = kk.s[a]; t_scale[4 * i + 3] = 0; }
      if (t_rot) for (int a = 0; a < 4; ++a) t_rot[4 * i + a] = kk.q[a];
      if (t_sh) for (int k = 0; k < nc; ++k) for (int ch = 0; ch < 3; ++ch) t_sh[((size_t)i * nc + k) * 3 + ch] = kk.sh[k][ch];
    }
    if (t_gradstat) t_gradstat[i] = slack[i].u * 0.5 * W + slack[i].v * 0.5 * H;
    if (g2d_out) {
      const Grad2D& s = g2d[i];
      const double v9[9] = {s.u, s.v, s.A, s.B, s.C, s.o, s.col[0], s.col[1], s.col[2]};
      for (int a = 0; a < 9; ++a) g2d_out[9 * i + a] = v9[a];
    }
    // O6: ∇p̄ statistic (A23): NDC-scaled 2D position gradient norm
    if (gradstat_sum) {
      if (R.G[i].key.visible) {
        const double gu = g2d[i].u * 0.5 * W, gv = g2d[i].v * 0.5 * H;
        gradstat_sum[i] = std::sqrt(gu * gu + gv * gv);
      } else {
        gradstat_sum[i] = 0;
      }
    }
    if (gradstat_cnt) gradstat_cnt[i] = R.G[i].key.visible ? 1 : 0;
    if (gtie) {
      uint8_t f = 0;
      const Proj& g = R.G[i];
      if (g.key.visible)
        for (int Y = g.key.y0; Y <= g.key.y1 && !f; ++Y)
          for (int X = g.key.x0; X <= g.key.x1; ++X)
            if (multi[(size_t)Y * W + X]) { f = 1; break; }
      gtie[i] = f;
    }
  }
  if (img_out) std::memcpy(img_out, img.data(), sizeof(double) * 3 * np);
  if (T_out) std::memcpy(T_out, Tfin.data(), sizeof(double) * np);
  return 0;
}

// ------------------------------------------------------------ f1 / Eq. 3 ---
// Fidelity loss: L = (1−λ)·L1 + λ·L_D-SSIM, "the fidelity loss in
// the vanilla 3DGS": L1 = mean |I − G| over 3HW values; D-SSIM = 1 − SSIM
// (A39); SSIM = mean over 3HW of S(q) = ((2μ_Iμ_G + C1)(2σ_IG + C2)) /
// ((μ_I² + μ_G² + C1)(σ_I² + σ_G² + C2)) with windowed statistics over an
// 11×11 Gaussian window (σ = 1.5, normalised to sum 1), per channel, zero
// padding outside the image, C1 = 0.01², C2 = 0.03² (S:306-307 design choice).
// Direct (non-separable) window sums: O(121·HW) per statistic, plain.
namespace {
void gauss_window(double w[11][11]) {
  double g[11], sum = 0;
  for (int k = 0; k < 11; ++k) { g[k] = std::exp(-((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5)); sum += g[k]; }
  for (int a = 0; a < 11; ++a)
    for (int b = 0; b < 11; ++b) w[a][b] = (g[a] / sum) * (g[b] / sum);
}
}  // namespace

// loss_out[0] = L, [1] = L1, [2] = SSIM.  dL (double[3HW], nullable) = ∂L/∂I.
// L = (1 − λ)·L1 + λ·D-SSIM with D-SSIM = dssim_scale·(1 − SSIM): 1 for the 3DGS
// code's 1 − SSIM (A39), 0.5 for SPEC's (1 − SSIM)/2.
int oracle_fidelity_loss(int W, int H, const float* img, const float* gt, double lambda,
                         double dssim_scale, double* loss_out, double* dL) {
  const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
  double w[11][11];
  gauss_window(w);
  const size_t np = (size_t)W * H;
  const double M = 3.0 * (double)np;
  std::vector<double> P1(3 * np), P2(3 * np), P3(3 * np);
  double sum_l1 = 0, sum_s = 0;
  for (int ch = 0; ch < 3; ++ch) {
    const float* I = img + ch * np;
    const float* G = gt + ch * np;
#pragma omp parallel for reduction(+ : sum_l1, sum_s) schedule(static)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        double m1 = 0, m2 = 0, s11 = 0, s22 = 0, s12 = 0;
        for (int a = -5; a <= 5; ++a)
          for (int b = -5; b <= 5; ++b) {
            const int yy = y + a, xx = x + b;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;  // zero padding
            const double wi = w[a + 5][b + 5];
            const double iv = I[(size_t)yy * W + xx], gv = G[(size_t)yy * W + xx];
            m1 += wi * iv; m2 += wi * gv; s11 += wi * iv * iv; s22 += wi * gv * gv; s12 += wi * iv * gv;
          }
        const double v1 = s11 - m1 * m1, v2 = s22 - m2 * m2, v12 = s12 - m1 * m2;
        const double A1 = 2 * m1 * m2 + C1, A2 = 2 * v12 + C2;
        const double B1 = m1 * m1 + m2 * m2 + C1, B2 = v1 + v2 + C2;
        const double S = A1 * A2 / (B1 * B2);
        sum_s += S;
        const size_t q = (size_t)y * W + x;
        sum_l1 += std::fabs((double)I[q] - (double)G[q]);
        // ∂S/∂μ_I, ∂S/∂E[I²], ∂S/∂E[IG] at q (μ_G, E[G²] do not depend on I)
        P1[ch * np + q] = 2 * m2 * (A2 - A1) / (B1 * B2) - 2 * m1 * A1 * A2 * (B2 - B1) / (B1 * B1 * B2 * B2);
        P2[ch * np + q] = -A1 * A2 / (B1 * B2 * B2);
        P3[ch * np + q] = 2 * A1 / (B1 * B2);
      }
  }
  const double L1 = sum_l1 / M, SSIM = sum_s / M;
  loss_out[0] = (1 - lambda) * L1 + lambda * dssim_scale * (1 - SSIM);
  loss_out[1] = L1;
  loss_out[2] = SSIM;
  if (!dL) return 0;
  for (int ch = 0; ch < 3; ++ch) {
    const float* I = img + ch * np;
    const float* G = gt + ch * np;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const size_t p = (size_t)y * W + x;
        // ∂SSIM/∂I(p) = (1/M) Σ_q w(p − q) [P1(q) + 2 I(p) P2(q) + G(p) P3(q)]
        double acc = 0;
        for (int a = -5; a <= 5; ++a)
          for (int b = -5; b <= 5; ++b) {
            const int yy = y + a, xx = x + b;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const size_t q = (size_t)yy * W + xx;
            const double wi = w[a + 5][b + 5];
            acc += wi * (P1[ch * np + q] + 2 * (double)I[p] * P2[ch * np + q] + (double)G[p] * P3[ch * np + q]);
          }
        const double d = (double)I[p] - (double)G[p];
        const double sgn = d > 0 ? 1.0 : (d < 0 ? -1.0 : 0.0);
        dL[ch * np + p] = (1 - lambda) * sgn / M - lambda * dssim_scale * acc / M;
      }
  }
  return 0;
}

// ------------------------------------------------------------ f3 / Eq. 1 ---
// Selective inheritance: o_r = Quant(sigmoid(m))∘o, s_r = Quant(sigmoid(m))∘s
// with Quant(x) = 1[x ≥ 0.5] (A26).
int oracle_inherit(int n, const float* m, uint8_t* keep) {
  for (int i = 0; i < n; ++i) {
    const double sig = 1.0 / (1.0 + std::exp(-(double)m[i]));
    keep[i] = sig >= 0.5 ? 1 : 0;
  }
  return 0;
}

// STE: m_op = detach(Quant(σ(m)) − σ(m)) + σ(m), so ∂m_op/∂m = σ'(m);
// with o_r = m_op·o and s_r = m_op·s, ∂L/∂m_op = o·∂L/∂o_r + Σ_k s_k·∂L/∂s_r,k.
// Mask loss λ_inher·Σσ(m) of Eq. 2 adds λ_inher·σ'(m).  g_m is written (=).
int oracle_inherit_bwd(int n, const float* m, const float* pos_opa, const float* scale,
                       const double* g_pos_opa, const double* g_scale, double lambda_inher,
                       double* g_m) {
  for (int i = 0; i < n; ++i) {
    const double sig = 1.0 / (1.0 + std::exp(-(double)m[i]));
    const double dsig = sig * (1.0 - sig);
    double dmop = (double)pos_opa[4 * i + 3] * g_pos_opa[4 * i + 3];
    for (int k = 0; k < 3; ++k) dmop += (double)scale[4 * i + k] * g_scale[4 * i + k];
    g_m[i] = (dmop + lambda_inher) * dsig;
  }
  return 0;
}

// ------------------------------------------------------------------ O7 -----
// §3.4: E = channel-mean |rendered − gt|, D = E > γ (strict,
// S:626).  Alg. 1 (garble fixed per A20): s_err |= D[y_n][x_n] for
// n < n_base.  Outputs: err double[H*W], D uint8[H*W], s_err uint8[n] (|=),
// xy int32[2n] (−1 if excluded), tie_g uint8[n] (pixel coordinate within
// 1e-4 of a rounding boundary), tie_px uint8[H*W] (|E − γ| < 1e-6).
int oracle_error_map(const OCam* cam, const float* rendered, const float* gt, double gamma,
                     int n_base, const float* pos_opa, double* err, uint8_t* D, uint8_t* s_err,
                     int32_t* xy, uint8_t* tie_g, uint8_t* tie_px) {
  const int W = cam->width, H = cam->height;
  const size_t np = (size_t)W * H;
  std::vector<double> E(np);
  std::vector<uint8_t> Dv(np);
  for (size_t p = 0; p < np; ++p) {
    double acc = 0;
    for (int ch = 0; ch < 3; ++ch) acc += std::fabs((double)rendered[ch * np + p] - (double)gt[ch * np + p]);
    E[p] = acc / 3.0;
    Dv[p] = E[p] > gamma ? 1 : 0;
    if (err) err[p] = E[p];
    if (D) D[p] = Dv[p];
    if (tie_px) tie_px[p] = std::fabs(E[p] - gamma) < 1e-6 ? 1 : 0;
  }
  double T[4][4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) T[a][b] = cam->full_proj[4 * a + b];
  for (int i = 0; i < n_base; ++i) {
    const double ph[4] = {pos_opa[4 * i], pos_opa[4 * i + 1], pos_opa[4 * i + 2], 1.0};
    double h[4];
    for (int b = 0; b < 4; ++b) h[b] = ph[0] * T[0][b] + ph[1] * T[1][b] + ph[2] * T[2][b] + ph[3] * T[3][b];
    if (xy) { xy[2 * i] = -1; xy[2 * i + 1] = -1; }
    if (tie_g) tie_g[i] = 0;
    if (!(h[3] > cam->near_plane)) continue;
    const double xn = h[0] / h[3], yn = h[1] / h[3];
    const double fxp = 0.5 * ((xn + 1.0) * W - 1.0);
    const double fyp = 0.5 * ((yn + 1.0) * H - 1.0);
    const double rx = std::round(fxp), ry = std::round(fyp);  // half away from zero
    if (tie_g) {
      const double ex = std::fabs(std::fabs(fxp - std::trunc(fxp)) - 0.5);
      const double ey = std::fabs(std::fabs(fyp - std::trunc(fyp)) - 0.5);
      if (ex < 1e-4 || ey < 1e-4) tie_g[i] = 1;
    }
    if (!(rx >= 0 && rx < W && ry >= 0 && ry < H)) continue;
    const int X = (int)rx, Y = (int)ry;
    if (xy) { xy[2 * i] = X; xy[2 * i + 1] = Y; }
    if (tie_px && tie_g && tie_px[(size_t)Y * W + X]) tie_g[i] = 1;
    if (s_err && Dv[(size_t)Y * W + X]) s_err[i] = 1;
  }
  return 0;
}

}  // extern "C"

// ------------------------------------------------------------ f2 -----------
// Dual hash-grid deformation (§3.3; supplement §B).  Each
// field 𝓗 maps a Gaussian position p_n to (μ_n, σ_n) = MLP(enc(p_n)) through
// an I-NGP multiresolution hash encoding and a small MLP (A41-A43):
//   enc: per level l (resolution N_l), x̂ = clamp((p − lo)/(hi − lo), 0, 1),
//        s = x̂·N_l, i0 = min(⌊s⌋, N_l − 1), w = s − i0; the 8 lattice corners
//        i0 + c (c ∈ {0,1}³) are read from level l's table row
//          (N_l+1)³ ≤ T:  x + y(N_l+1) + z(N_l+1)²               (dense)
//          otherwise:     (x·1 ⊕ y·2654435761 ⊕ z·805459861) mod T   (hash, u32)
//        and trilinearly weighted, Π_k (c_k ? w_k : 1 − w_k); levels concatenated.
//   MLP: in = L·F → 64 → 64 → 7, ReLU on the hidden layers, linear head;
//        params flat: W1[64][in], b1[64], W2[64][64], b2[64], W3[7][64], b3[7].
//   μ = out[0:3];  σ = (1, 0, 0, 0) + out[3:7]  (zero head = identity, A42).
// Everything in double from the fp32 inputs.
struct OHash {
  int32_t L, log2T, F, pad;
  int32_t res[16];
  float lo[3], hi[3];
};

namespace {
constexpr int OH = 64;  // hidden width (A41)

uint64_t hash_row(const OHash& c, int l, uint32_t x, uint32_t y, uint32_t z) {
  const uint64_t T = 1ull << c.log2T;
  const uint64_t n1 = (uint64_t)c.res[l] + 1;
  if (n1 * n1 * n1 <= T) return x + y * n1 + z * n1 * n1;
  const uint32_t h = (x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u);
  return h & (uint32_t)(T - 1);
}

// the 8 (row, weight) pairs of level l for position p
void corners(const OHash& c, int l, const float* p, uint64_t row[8], double wt[8]) {
  uint32_t i0[3];
  double w[3];
  for (int k = 0; k < 3; ++k) {
    double xh = ((double)p[k] - (double)c.lo[k]) / ((double)c.hi[k] - (double)c.lo[k]);
    xh = std::min(1.0, std::max(0.0, xh));
    const double s = xh * c.res[l];
    const double f = std::min(std::floor(s), (double)(c.res[l] - 1));
    i0[k] = (uint32_t)f;
    w[k] = s - f;
  }
  for (int cc = 0; cc < 8; ++cc) {
    const uint32_t bx = cc & 1, by = (cc >> 1) & 1, bz = (cc >> 2) & 1;
    row[cc] = hash_row(c, l, i0[0] + bx, i0[1] + by, i0[2] + bz);
    wt[cc] = (bx ? w[0] : 1.0 - w[0]) * (by ? w[1] : 1.0 - w[1]) * (bz ? w[2] : 1.0 - w[2]);
  }
}

struct MlpView {
  const float *W1, *b1, *W2, *b2, *W3, *b3;
  MlpView(const float* p, int in)
      : W1(p), b1(p + OH * in), W2(b1 + OH), b2(W2 + OH * OH), W3(b2 + OH), b3(W3 + 7 * OH) {}
};
}  // namespace

extern "C" {

int oracle_hash_params(int in) { return OH * in + OH + OH * OH + OH + 7 * OH + 7; }

// enc(p) for m positions: feat double[m][L·F]
int oracle_hash_encode(const OHash* c, const float* table, int m, const float* pos_opa,
                       double* feat) {
  const int L = c->L, F = c->F, in = L * F;
  const uint64_t T = 1ull << c->log2T;
  for (int i = 0; i < m; ++i) {
    for (int l = 0; l < L; ++l) {
      uint64_t row[8];
      double wt[8];
      corners(*c, l, pos_opa + 4 * i, row, wt);
      for (int f = 0; f < F; ++f) {
        double acc = 0;
        for (int cc = 0; cc < 8; ++cc) acc += wt[cc] * (double)table[((uint64_t)l * T + row[cc]) * F + f];
        feat[(size_t)i * in + l * F + f] = acc;
      }
    }
  }
  return 0;
}

// (μ, σ) for m positions.  mu, sigma: double[m][4] (mu.w = 0).  tie (nullable,
// uint8[m]): some hidden pre-activation within 1e-5·(1 + Σ|terms|) of 0, i.e. a
// ReLU decision that fp32 rounding may take differently (A43).
int oracle_deform_fwd(const OHash* c, const float* table, const float* mlp, int m,
                      const float* pos_opa, double* mu, double* sigma, uint8_t* tie) {
  const int in = c->L * c->F;
  const MlpView P(mlp, in);
  std::vector<double> x(in), h1(OH), h2(OH);
  for (int i = 0; i < m; ++i) {
    oracle_hash_encode(c, table, 1, pos_opa + 4 * i, x.data());
    bool t = false;
    for (int o = 0; o < OH; ++o) {
      double z = P.b1[o], k = std::fabs((double)P.b1[o]);
      for (int j = 0; j < in; ++j) { z += (double)P.W1[o * in + j] * x[j]; k += std::fabs((double)P.W1[o * in + j] * x[j]); }
      t |= std::fabs(z) < 1e-5 * (1.0 + k);
      h1[o] = z > 0 ? z : 0.0;
    }
    for (int o = 0; o < OH; ++o) {
      double z = P.b2[o], k = std::fabs((double)P.b2[o]);
      for (int j = 0; j < OH; ++j) { z += (double)P.W2[o * OH + j] * h1[j]; k += std::fabs((double)P.W2[o * OH + j] * h1[j]); }
      t |= std::fabs(z) < 1e-5 * (1.0 + k);
      h2[o] = z > 0 ? z : 0.0;
    }
    double out[7];
    for (int o = 0; o < 7; ++o) {
      double z = P.b3[o];
      for (int j = 0; j < OH; ++j) z += (double)P.W3[o * OH + j] * h2[j];
      out[o] = z;
    }
    mu[4 * i + 0] = out[0]; mu[4 * i + 1] = out[1]; mu[4 * i + 2] = out[2]; mu[4 * i + 3] = 0.0;
    sigma[4 * i + 0] = 1.0 + out[3];
    sigma[4 * i + 1] = out[4]; sigma[4 * i + 2] = out[5]; sigma[4 * i + 3] = out[6];
    if (tie) tie[i] = t ? 1 : 0;
  }
  return 0;
}

// Reverse of oracle_deform_fwd for ∂L/∂μ (g_mu[m][4], xyz) and ∂L/∂σ
// (g_sigma[m][4], wxyz): accumulates (+=) ∂L/∂table (double[L][T][F]) and
// ∂L/∂params (double, the flat MLP layout).  kt / km (nullable): Σ|term| of
// the same sums (conditioning, A43).
int oracle_deform_bwd(const OHash* c, const float* table, const float* mlp, int m,
                      const float* pos_opa, const double* g_mu, const double* g_sigma,
                      double* g_table, double* g_mlp, double* kt, double* km) {
  const int L = c->L, F = c->F, in = L * F;
  const uint64_t T = 1ull << c->log2T;
  const MlpView P(mlp, in);
  double* gW1 = g_mlp;
  double* gb1 = gW1 + OH * in;
  double* gW2 = gb1 + OH;
  double* gb2 = gW2 + OH * OH;
  double* gW3 = gb2 + OH;
  double* gb3 = gW3 + 7 * OH;
  const size_t koff[6] = {0, (size_t)OH * in, (size_t)OH * in + OH, (size_t)OH * in + OH + OH * OH,
                          (size_t)OH * in + 2 * OH + OH * OH, (size_t)OH * in + 2 * OH + OH * OH + 7 * OH};
  std::vector<double> x(in), z1(OH), h1(OH), z2(OH), h2(OH), d2(OH), d1(OH), dx(in);
  for (int i = 0; i < m; ++i) {
    oracle_hash_encode(c, table, 1, pos_opa + 4 * i, x.data());
    for (int o = 0; o < OH; ++o) {
      double z = P.b1[o];
      for (int j = 0; j < in; ++j) z += (double)P.W1[o * in + j] * x[j];
      z1[o] = z; h1[o] = z > 0 ? z : 0.0;
    }
    for (int o = 0; o < OH; ++o) {
      double z = P.b2[o];
      for (int j = 0; j < OH; ++j) z += (double)P.W2[o * OH + j] * h1[j];
      z2[o] = z; h2[o] = z > 0 ? z : 0.0;
    }
    // ∂L/∂out: μ = out[0:3], σ = e_w + out[3:7]
    const double d3[7] = {g_mu[4 * i], g_mu[4 * i + 1], g_mu[4 * i + 2], g_sigma[4 * i],
                          g_sigma[4 * i + 1], g_sigma[4 * i + 2], g_sigma[4 * i + 3]};
    for (int o = 0; o < 7; ++o) {
      gb3[o] += d3[o];
      if (km) km[koff[5] + o] += std::fabs(d3[o]);
      for (int j = 0; j < OH; ++j) {
        gW3[o * OH + j] += d3[o] * h2[j];
        if (km) km[koff[4] + o * OH + j] += std::fabs(d3[o] * h2[j]);
      }
    }
    for (int j = 0; j < OH; ++j) {
      double s = 0;
      for (int o = 0; o < 7; ++o) s += (double)P.W3[o * OH + j] * d3[o];
      d2[j] = z2[j] > 0 ? s : 0.0;
    }
    for (int o = 0; o < OH; ++o) {
      gb2[o] += d2[o];
      if (km) km[koff[3] + o] += std::fabs(d2[o]);
      for (int j = 0; j < OH; ++j) {
        gW2[o * OH + j] += d2[o] * h1[j];
        if (km) km[koff[2] + o * OH + j] += std::fabs(d2[o] * h1[j]);
      }
    }
    for (int j = 0; j < OH; ++j) {
      double s = 0;
      for (int o = 0; o < OH; ++o) s += (double)P.W2[o * OH + j] * d2[o];
      d1[j] = z1[j] > 0 ? s : 0.0;
    }
    for (int o = 0; o < OH; ++o) {
      gb1[o] += d1[o];
      if (km) km[koff[1] + o] += std::fabs(d1[o]);
      for (int j = 0; j < in; ++j) {
        gW1[o * in + j] += d1[o] * x[j];
        if (km) km[koff[0] + o * in + j] += std::fabs(d1[o] * x[j]);
      }
    }
    for (int j = 0; j < in; ++j) {
      double s = 0;
      for (int o = 0; o < OH; ++o) s += (double)P.W1[o * in + j] * d1[o];
      dx[j] = s;
    }
    // enc is linear in the table: ∂feat_{l,f}/∂table[l][row_c][f] = wt_c
    for (int l = 0; l < L; ++l) {
      uint64_t row[8];
      double wt[8];
      corners(*c, l, pos_opa + 4 * i, row, wt);
      for (int cc = 0; cc < 8; ++cc)
        for (int f = 0; f < F; ++f) {
          const size_t e = ((uint64_t)l * T + row[cc]) * F + f;
          g_table[e] += wt[cc] * dx[l * F + f];
          if (kt) kt[e] += std::fabs(wt[cc] * dx[l * F + f]);
        }
    }
  }
  return 0;
}

}  // extern "C"

// ------------------------------------------------------------ f4 -----------
// Error-guided densification (§3.4) and the identity-feature
// render of Gaussian Grouping (Eq. 9, §A.2).  A44-A47.
extern "C" {

// Eq. 4, literal set evaluation: S = {n : ∇p̄_n > τ_pos} ∪
// (S_err ∩ {n : ∇p̄_n > τ_err}), ∇p̄_n = gradstat_sum_n / gradstat_cnt_n (0 when
// never counted).  The threshold decisions are taken in fp32, the kernel's
// precision (A44): ∇p̄ is one IEEE fp32 division of the fp32 inputs.
// in_S uint8[n] (written).  Returns |S|.
int oracle_densify_select(int n, const float* gsum, const uint32_t* gcnt, const uint8_t* s_err,
                          float tau_pos, float tau_err, uint8_t* in_S) {
  int count = 0;
  for (int i = 0; i < n; ++i) {
    const float g = gcnt[i] ? gsum[i] / (float)gcnt[i] : 0.0f;
    const bool a = g > tau_pos;                          // {∇p̄ > τ_pos}
    const bool b = s_err && s_err[i] && g > tau_err;     // S_err ∩ {∇p̄ > τ_err}
    in_S[i] = (a || b) ? 1 : 0;
    count += in_S[i];
  }
  return count;
}

// Philox4x64-10 (Salmon et al., SC'11): the counter-based generator both
// sides implement for the spawn samples (A45).  out = Philox(ctr, key).
void oracle_philox4x64(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const unsigned __int128 p0 = (unsigned __int128)c0 * 0xD2E7470EE14C6C93ull;
    const unsigned __int128 p1 = (unsigned __int128)c2 * 0xCA5A826395121157ull;
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Spawn densification (A45): for the k-th selected parent i = idx[k]
// and child j < K, draw z ~ N(0, I₃) from Philox(ctr = (k·K + j, 0, 0, 0),
// key = (seed, 0x44415353)) via Box-Muller on u = ((x >> 40) + ½)·2⁻²⁴ and
// place the child at p + R(n(q))·(s ∘ z), i.e. a sample of N(p, Σ) with
// Σ = R S Sᵀ Rᵀ (Eq. 6); scale s/shrink, opacity child_opacity,
// rotation, SH and dynamic flag copied.  Outputs (double): child_pos_opa
// [m·K][4], child_scale [m·K][4]; z (nullable) [m·K][3].
int oracle_spawn(int m, const int32_t* idx, int K, double shrink, double child_opacity,
                 uint64_t seed, const float* pos_opa, const float* scale, const float* rot,
                 double* child_pos_opa, double* child_scale, double* zout) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int k = 0; k < m; ++k) {
    const int i = idx[k];
    double q[4];
    for (int a = 0; a < 4; ++a) q[a] = rot[4 * i + a];
    const double nq = norm4(q);
    for (int a = 0; a < 4; ++a) q[a] /= nq;
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                            {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                            {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
    for (int j = 0; j < K; ++j) {
      const uint64_t ctr[4] = {(uint64_t)k * (uint64_t)K + (uint64_t)j, 0, 0, 0};
      const uint64_t key[2] = {seed, 0x44415353ull};
      uint64_t r[4];
      oracle_philox4x64(ctr, key, r);
      double u[4];
      for (int a = 0; a < 4; ++a) u[a] = ((double)(r[a] >> 40) + 0.5) * (1.0 / 16777216.0);
      const double r0 = std::sqrt(-2.0 * std::log(u[0])), r1 = std::sqrt(-2.0 * std::log(u[2]));
      const double zz[3] = {r0 * std::cos(two_pi * u[1]), r0 * std::sin(two_pi * u[1]),
                            r1 * std::cos(two_pi * u[3])};
      const size_t c = (size_t)k * K + j;
      for (int a = 0; a < 3; ++a) {
        double off = 0;
        for (int b = 0; b < 3; ++b) off += R[a][b] * (double)scale[4 * i + b] * zz[b];
        child_pos_opa[4 * c + a] = (double)pos_opa[4 * i + a] + off;
        child_scale[4 * c + a] = (double)scale[4 * i + a] / shrink;
        if (zout) zout[3 * c + a] = zz[a];
      }
      child_pos_opa[4 * c + 3] = child_opacity;
      child_scale[4 * c + 3] = 0.0;
    }
  }
  return 0;
}

// Identity-feature render, Eq. 9: M = Σ_i e_i α_i Π_{j<i}(1 − α_j)
// with α, the order, the 1/255 skip and the early stop exactly as in Eq. 8's
// compositor (O4; A47), features e [n][C] in place of colours, no background.
// out double[C][H][W]; tie uint8[H][W] (nullable, A29).  Scatter form.
int oracle_render_features(const OCam* cam, int n, const float* pos_opa, const float* scale,
                           const float* rot, const uint8_t* keep, int C, const float* feat,
                           double* out, uint8_t* tie) {
  std::vector<float> sh0((size_t)n * 4, 0.0f);   // colours are not used (degree 0 placeholder)
  RenderCtx R;
  make_ctx(R, cam, n, 0, pos_opa, scale, rot, sh0.data(), keep);
  const TieEps te = tie_from(nullptr);
  const int W = cam->width, H = cam->height;
  const size_t np = (size_t)W * H;
  std::vector<double> T(np, 1.0);
  std::vector<uint8_t> done(np, 0), tv(np, 0);
  for (size_t e = 0; e < (size_t)C * np; ++e) out[e] = 0.0;
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  const int band = std::max(1, (H + nth * 4 - 1) / (nth * 4));
  const int nb = (H + band - 1) / band;
#pragma omp parallel for schedule(dynamic, 1)
  for (int bi = 0; bi < nb; ++bi) {
    const int ylo = bi * band, yhi = std::min(H - 1, ylo + band - 1);
    for (int pos = 0; pos < (int)R.ord.size(); ++pos) {
      const int gi = R.ord[pos];
      const Proj& g = R.G[gi];
      const int y0 = std::max(g.key.y0, ylo), y1 = std::min(g.key.y1, yhi);
      for (int Y = y0; Y <= y1; ++Y)
        for (int X = g.key.x0; X <= g.key.x1; ++X) {
          const size_t p = (size_t)Y * W + X;
          if (done[p]) continue;
          Eval e = eval_at(g, X, Y);
          if (is_tie(g, e, T[p], te)) tv[p] = 1;
          if (e.power > 0 || e.alpha < ALPHA_MIN) continue;
          const double tn = T[p] * (1 - e.alpha);
          if (tn < T_MIN) { done[p] = 1; continue; }
          for (int ch = 0; ch < C; ++ch) out[ch * np + p] += (double)feat[(size_t)gi * C + ch] * e.alpha * T[p];
          T[p] = tn;
        }
    }
  }
  if (tie)
    for (size_t p = 0; p < np; ++p) tie[p] = tv[p];
  return 0;
}

}  // extern "C"

extern "C" {
// Opacity pruning ("eliminate excessive Gaussian candidates with very
// low opacity"; A46): rows i < first (the frozen base) are kept; a candidate
// is kept iff o_i ≥ min_opacity.  keep uint8[n].  Returns the kept count.
int oracle_prune_keep(int n, int first, const float* pos_opa, float min_opacity, uint8_t* keep) {
  int c = 0;
  for (int i = 0; i < n; ++i) {
    keep[i] = (i < first || !(pos_opa[4 * i + 3] < min_opacity)) ? 1 : 0;
    c += keep[i];
  }
  return c;
}
}  // extern "C"
