// op5.cuh -- the 5-point symmetric operator family evaluated from staged
// (shared-memory) values: face coefficients and one cell of y = A x plus the
// diagonal d (kernels_cg5.cu header).  Shared by the TMA-ring
// CG kernels.
#pragma once
#include "common.cuh"

namespace chb {

struct Op5T {
  const double* a;
  const double* w;
  double s, kscale, rho_n, rho_s;
  double ascal;   // AM == 2: constant diagonal coefficient (no array)
};

// diagonal coefficient at flat offset o: AM = 0 none, 1 array a[], 2 scalar
template <int AM>
__device__ __forceinline__ double a_at(const Op5T& op, size_t o) {
  return AM == 2 ? op.ascal : (AM ? op.a[o] : 0.0);
}

template <int KM>
__device__ __forceinline__ double kfaceT(const Op5T& op, double w1, double w2) {
  if (KM == 0) return 1.0;
  const double m = 0.5 * (w1 + w2);
  if (KM == 1) return op.kscale * m;
  const double f = fmin(fmax(m, 0.0), 1.0);   // volume fraction (R24)
  return 1.0 / (op.rho_s + f * (op.rho_n - op.rho_s));
}

template <int BC, int AM, int KM>
__device__ __forceinline__ void eval5T(const Op5T& op, const Geom& g, int gj, double ac, double wc,
                                       double ww, double we, double ws, double wn, double xc,
                                       double xw, double xe, double xs, double xn, double& y,
                                       double& d) {
  if (BC == BC_VFACE && gj == 0) {
    y = xc;
    d = 1.0;
    return;
  }
  const double kE = kfaceT<KM>(op, wc, we), kW = kfaceT<KM>(op, ww, wc);
  const double kN = kfaceT<KM>(op, wc, wn), kS = kfaceT<KM>(op, ws, wc);
  double fS = 1.0, fN = 1.0;
  if (BC == BC_MIRROR) {
    fS = (gj == 0) ? 0.0 : 1.0;
    fN = (gj == g.ny - 1) ? 0.0 : 1.0;
  } else if (BC == BC_ODD) {
    fS = (gj == 0) ? 2.0 : 1.0;
    fN = (gj == g.ny - 1) ? 2.0 : 1.0;
  }
  const double a = AM ? ac : 0.0;
  y = a * xc + op.s * ((kE * (xc - xe) + kW * (xc - xw)) * g.ihx2 +
                       (kN * (xc - xn) + kS * (xc - xs)) * g.ihy2);
  d = a + op.s * ((kE + kW) * g.ihx2 + (fN * kN + fS * kS) * g.ihy2);
}

// Split form for kernels that apply the same operator twice per cell (the
// single-reduction CG): face coefficients + diagonal once, then y = A x.
// Arithmetic identical to eval5T.
struct Cf5 {
  double kE, kW, kN, kS, a, d;
};

// WALLS = false: caller guarantees gj is neither a wall row nor (v) row 0.
template <int BC, int AM, int KM, bool WALLS = true>
__device__ __forceinline__ Cf5 coef5(const Op5T& op, const Geom& g, int gj, double ac, double wc,
                                     double ww, double we, double ws, double wn) {
  Cf5 c;
  if (WALLS && BC == BC_VFACE && gj == 0) {
    c.kE = c.kW = c.kN = c.kS = c.a = 0.0;
    c.d = 1.0;
    return c;
  }
  c.kE = kfaceT<KM>(op, wc, we);
  c.kW = kfaceT<KM>(op, ww, wc);
  c.kN = kfaceT<KM>(op, wc, wn);
  c.kS = kfaceT<KM>(op, ws, wc);
  double fS = 1.0, fN = 1.0;
  if (WALLS && BC == BC_MIRROR) {
    fS = (gj == 0) ? 0.0 : 1.0;
    fN = (gj == g.ny - 1) ? 0.0 : 1.0;
  } else if (WALLS && BC == BC_ODD) {
    fS = (gj == 0) ? 2.0 : 1.0;
    fN = (gj == g.ny - 1) ? 2.0 : 1.0;
  }
  c.a = AM ? ac : 0.0;
  c.d = c.a + op.s * ((c.kE + c.kW) * g.ihx2 + (fN * c.kN + fS * c.kS) * g.ihy2);
  return c;
}

template <int BC, bool WALLS = true>
__device__ __forceinline__ double apply5(const Cf5& c, const Op5T& op, const Geom& g, int gj,
                                         double xc, double xw, double xe, double xs, double xn) {
  if (WALLS && BC == BC_VFACE && gj == 0) return xc;
  return c.a * xc + op.s * ((c.kE * (xc - xe) + c.kW * (xc - xw)) * g.ihx2 +
                            (c.kN * (xc - xn) + c.kS * (xc - xs)) * g.ihy2);
}

}  // namespace chb
