// params.cuh — construction of the per-recolouring constant blocks (StrictP,
// FastP) from (source i0, OD table, basis, factors, target basis/i0), shared by
// the host C ABI (api.cu) and the device-side batch builder (batch.cu) so both
// produce bit-identical parameters.  Compiled with -ffp-contract=off on the
// host; device code uses explicit __dmul_rn/__dadd_rn where the reference's
// operation order matters.
#pragma once
#include <cmath>
#include <cstdint>

#include "spcn_device.cuh"

namespace spcn {

__host__ __device__ inline double p_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ inline double p_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}

// Gram entries in the reference's scalar order (src/stain_sep.py:197-199).
__host__ __device__ inline void gram3x2(const double* w, double& g00, double& g01, double& g11) {
  g00 = p_add(p_add(p_mul(w[0], w[0]), p_mul(w[2], w[2])), p_mul(w[4], w[4]));
  g11 = p_add(p_add(p_mul(w[1], w[1]), p_mul(w[3], w[3])), p_mul(w[5], w[5]));
  g01 = p_add(p_add(p_mul(w[0], w[1]), p_mul(w[2], w[3])), p_mul(w[4], w[5]));
}

// Everything except the 3x256 table (which the caller copies in).
__host__ __device__ inline void fill_strict_scalars(StrictP& sp, const double* ws, const double* wt,
                                                    const double* f, const double* i0t, double lam,
                                                    int max_sweeps) {
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < 2; ++j) {
      sp.ws[c][j] = ws ? ws[c * 2 + j] : 0.0;
      sp.wt[c][j] = wt ? wt[c * 2 + j] : 0.0;
    }
  sp.f[0] = f ? f[0] : 1.0;
  sp.f[1] = f ? f[1] : 1.0;
  for (int c = 0; c < 3; ++c) sp.i0t[c] = i0t ? i0t[c] : 255.0;
  if (ws) {
    gram3x2(ws, sp.g00, sp.g01, sp.g11);
    sp.det = p_add(p_mul(sp.g00, sp.g11), -p_mul(sp.g01, sp.g01));
  } else {
    sp.g00 = sp.g01 = sp.g11 = sp.det = 0.0;
  }
  sp.lam = lam;
  sp.tol = 0.0;
  sp.max_sweeps = max_sweeps;
  sp.pad_ = 0;
}

// fp32 coefficients + the analytic certification bound (DESIGN.md §Certified
// rounding).  Reads sp (scalars and table).  Returns false when the fast path
// must not be used: ill-conditioned basis, target i0 outside [0, 255], or (in
// EXACT mode) a bound too loose to be useful or a target i0 on a rounding tie.
// The fp32 table is written only when `lut` is non-null.
__host__ __device__ inline bool fill_fast_scalars(FastS& fp, const StrictP& sp, bool exact,
                                                  float (*lut)[256]) {
  const double g00 = sp.g00, g01 = sp.g01, g11 = sp.g11, det = sp.det;
  if (!(det > 1e-6 * g00 * g11) || !(g00 > 0) || !(g11 > 0)) return false;
  for (int c = 0; c < 3; ++c)
    if (!(sp.i0t[c] >= 0.0 && sp.i0t[c] <= 255.0)) return false;
  if (lut)
    for (int c = 0; c < 3; ++c)
      for (int i = 0; i < 256; ++i) lut[c][i] = static_cast<float>(sp.lut[c][i]);
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < 2; ++j) fp.w[c][j] = static_cast<float>(sp.ws[c][j]);
  fp.nlam = static_cast<float>(-sp.lam);
  const double A = g11 / det, C = g01 / det, E = 1.0 / g11, F = g01 / g11, G = 1.0 / g00,
               H = g01 / g00;
  fp.A = (float)A;
  fp.nC = -(float)C;
  fp.E = (float)E;
  fp.nF2 = -(float)F * 0.5f;
  fp.G = (float)G;
  fp.nH2 = -(float)H * 0.5f;
  for (int c = 0; c < 3; ++c) fp.I[c].x = fp.I[c].y = 0.0f;
  // Background skip: a byte x >= i0_c has OD exactly 0, so a
  // pixel with every channel there has h = 0 and renders floor(i0_t + 0.5)
  // (src/optics.py:89-94, src/normalize.py:146-150).  T = the smallest byte
  // value with OD 0 in every channel; the kernel tests "all bits of wmask set"
  // for every byte, i.e. x >= 256 - 2^k >= T (conservative).
  {
    int T = 0;
    for (int c = 0; c < 3; ++c) {
      int x = 255;
      while (x > 0 && sp.lut[c][x - 1] == 0.0) --x;
      if (!(sp.lut[c][255] == 0.0)) x = 256;   // no background byte in this channel
      T = x > T ? x : T;
    }
    fp.wmask = 0;
    if (T <= 255) {
      int k = 0;
      while ((2 << k) <= 256 - T) ++k;          // 2^k <= 256 - T < 2^(k+1)
      const uint32_t mb = (~((1u << k) - 1u)) & 0xffu;
      fp.wmask = mb * 0x01010101u;
    }
    uint32_t ob[3];
    for (int c = 0; c < 3; ++c) {
      double y = floor(p_add(static_cast<double>(sp.i0t[c]), 0.5));
      y = y < 0.0 ? 0.0 : (y > 255.0 ? 255.0 : y);
      ob[c] = static_cast<uint32_t>(y);
    }
    for (int wd = 0; wd < 3; ++wd) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) v |= ob[(4 * wd + b) % 3] << (8 * b);
      fp.wout[wd] = v;
    }
  }
  const double log2e = 1.4426950408889634;
  double Kabs[3][2];
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < 2; ++j) {
      const double k = -log2e * sp.wt[c][j] * sp.f[j];
      fp.K2[c][j] = static_cast<float>(k) * 0.5f;
      Kabs[c][j] = fabs(k);
    }
  for (int c = 0; c < 3; ++c) fp.i0t[c] = static_cast<float>(sp.i0t[c]);
  fp.lam4 = static_cast<float>(4.0 * sp.lam);
  // error chain, per unit u*T (u = 2^-24, T = t0 + t1 + 4 lam)
  const double P0 = A + C, D0 = 8.0 * (A + C);
  const double D1 = 7.0 * E + F * D0 + 3.0 * F * P0;
  const double P1 = E + F * P0;
  const double Dh0 = 7.0 * G + H * D1 + 3.0 * H * P1;
  const double H0 = G + H * P1;
  double L = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double l =
        Kabs[c][0] * Dh0 + Kabs[c][1] * D1 + 3.0 * (Kabs[c][0] * H0 + Kabs[c][1] * P1);
    L = l > L ? l : L;
  }
  const double u = 5.9604644775390625e-08, ln2 = 0.6931471805599453;  // u = 2^-24
  const double a1 = 1.25 * ln2 * u * L * 1.001;
  const double a0 = 1.25 * (2 * 4.76837158203125e-07);                // 2^-21 twice
  fp.a1 = static_cast<float>(a1 * (1.0 + 1e-6));
  fp.a0 = static_cast<float>(a0 * (1.0 + 1e-6));
  if (!exact) return true;
  double tmax = 4.0 * sp.lam;    // worst-case T over all u8 inputs (OD largest at i = 0)
  for (int c = 0; c < 3; ++c) tmax += (sp.ws[c][0] + sp.ws[c][1]) * sp.lut[c][0];
  if (a1 * tmax + a0 > 1e-3) return false;
  // zero-density pixels render exactly i0_t; an exact tie (i0_t = k + 0.5)
  // can never certify, so such targets take the strict path
  const double a_zero = a1 * 4.0 * sp.lam + a0;
  for (int c = 0; c < 3; ++c) {
    const double fr = sp.i0t[c] - floor(sp.i0t[c]);
    if (fabs(fr - 0.5) <= 2.0 * a_zero * sp.i0t[c] + 1e-9) return false;
  }
  return true;
}

// Per-pixel error bound of the fp32 densities (fast_density) against the
// reference's fp64 coder: |h_j - h_ref,j| <= coef[j] * T + 1e-30, T the
// pixel's t0 + t1 + 4 lam.  Same instruction-by-instruction chain and safety
// factor as the certification bound in fill_fast_scalars (h0 <- Dh0, h1 <- D1).
__host__ __device__ inline void density_error_coeffs(const StrictP& sp, double coef[2]) {
  const double g00 = sp.g00, g01 = sp.g01, g11 = sp.g11, det = sp.det;
  const double A = g11 / det, C = g01 / det, E = 1.0 / g11, F = g01 / g11, G = 1.0 / g00,
               H = g01 / g00;
  const double P0 = A + C, D0 = 8.0 * (A + C);
  const double D1 = 7.0 * E + F * D0 + 3.0 * F * P0;
  const double P1 = E + F * P0;
  const double Dh0 = 7.0 * G + H * D1 + 3.0 * H * P1;
  const double u = 5.9604644775390625e-08;   // 2^-24
  coef[0] = 1.25 * 1.001 * u * Dh0;
  coef[1] = 1.25 * 1.001 * u * D1;
}

}  // namespace spcn
