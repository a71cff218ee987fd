// kernels_rhs.cu -- explicit parts of one time step (run once per step):
// CH right-hand side + phi* + Jacobi diagonal, nutrient RHS + coefficients,
// momentum RHS + coefficients, MAC divergence, projection.
// PAPER.md Eq. 16 (lines 108-114), Eq. 17-21 (lines 122-141); DESIGN.md §2.
// One thread per cell/face, neighbours through L1; these kernels are a small
// share of a step (the Krylov sweeps dominate), so clarity wins here.
#include "common.cuh"
#include "launch.h"

namespace chb {

#define CHB_CELL_PREAMBLE(g)                                  \
  const int i = blockIdx.x * blockDim.x + threadIdx.x;        \
  const int jl = blockIdx.y * blockDim.y + threadIdx.y;       \
  if (i >= (g).nx || jl >= (g).nyl) return;                   \
  const int j = (g).j0 + jl;                                  \
  const int iw = wrapc(i - 1, (g).nx), ie = wrapc(i + 1, (g).nx);

static dim3 grid2(const Geom& g) { return dim3((g.nx + 31) / 32, (g.nyl + 7) / 8); }
static const dim3 blk2(32, 8);

__device__ __forceinline__ double fprime(double p, double G2) {
  return 2.0 * G2 * p * (1.0 - p) * (1.0 - 2.0 * p);
}

// Material laws and rates take the physical volume fraction clip(phi, 0, 1) (R24).
__device__ __forceinline__ double vfrac(double p) { return fmin(fmax(p, 0.0), 1.0); }

// ------------------------------------------------------------------ CH RHS
// b = phi/dt + L_{M*}(F'(phi*) - (1-th) G1 Delta phi) - (1-ta) Adv(phi; v^n) + g_n(phi*, c)
// (th = theta_ch, ta = theta_adv of this step; R5, R12, R23)
__global__ void __launch_bounds__(256) k_ch_rhs(Geom g, Phys ph, StateP s, double* phis_out,
                                                double* dinv, double* b) {
  CHB_CELL_PREAMBLE(g)
  auto PHI = [&](int jj, int ii) { return ldf<BC_MIRROR>(s.phi, g, jj, ii); };
  auto PS = [&](int jj, int ii) {
    return 1.5 * ldf<BC_MIRROR>(s.phi, g, jj, ii) - 0.5 * ldf<BC_MIRROR>(s.phip, g, jj, ii);
  };
  auto LAP = [&](int jj, int ii) {
    const double c0 = PHI(jj, ii);
    return (PHI(jj, wrapc(ii + 1, g.nx)) - 2.0 * c0 + PHI(jj, wrapc(ii - 1, g.nx))) * g.ihx2 +
           (PHI(jj + 1, ii) - 2.0 * c0 + PHI(jj - 1, ii)) * g.ihy2;
  };
  const double g1e = (1.0 - ph.th_ch) * ph.Gamma1;
  auto MU = [&](int jj, int ii) { return fprime(PS(jj, ii), ph.Gamma2) - g1e * LAP(jj, ii); };
  const double pc = PS(j, i), pe = PS(j, ie), pw = PS(j, iw), pn = PS(j + 1, i), psv = PS(j - 1, i);
  const double L = ph.Lambda;
  const double mE = L * fmax(0.0, 0.5 * (pc + pe));
  const double mW = L * fmax(0.0, 0.5 * (pw + pc));
  const double mN = (j == g.ny - 1) ? 0.0 : L * fmax(0.0, 0.5 * (pc + pn));
  const double mS = (j == 0) ? 0.0 : L * fmax(0.0, 0.5 * (psv + pc));
  const double muc = MU(j, i);
  const double lm = (mE * (MU(j, ie) - muc) - mW * (muc - MU(j, iw))) * g.ihx2 +
                    (mN * (MU(j + 1, i) - muc) - mS * (muc - MU(j - 1, i))) * g.ihy2;
  const double uE = s.u[off(g, j, ie)], uW = s.u[off(g, j, i)];
  const double vN = ldf<BC_VFACE>(s.v, g, j + 1, i), vS = ldf<BC_VFACE>(s.v, g, j, i);
  const double fc = PHI(j, i);
  const double adv = (uE * 0.5 * (fc + PHI(j, ie)) - uW * 0.5 * (PHI(j, iw) + fc)) * g.ihx +
                     (vN * 0.5 * (fc + PHI(j + 1, i)) - vS * 0.5 * (PHI(j - 1, i) + fc)) * g.ihy;
  const size_t o = off(g, j, i);
  const double cval = s.c[o];
  const double grow = ph.eps * ph.mu * vfrac(pc) * cval / (ph.Kc + cval);
  b[o] = fc / ph.dt + lm - (1.0 - ph.th_adv) * adv + grow;
  phis_out[o] = pc;
  // Jacobi diagonal of I/dt + th G1 L_M Delta_h + ta Adv (mirror walls fold onto the cell)
  const double nwall = (j == 0 ? 1.0 : 0.0) + (j == g.ny - 1 ? 1.0 : 0.0);
  const double sx = (mE + mW) * g.ihx2, sy = (mN + mS) * g.ihy2;
  const double lapd = 2.0 * g.ihx2 + 2.0 * g.ihy2 - nwall * g.ihy2;
  const double adiag = 0.5 * ((uE - uW) * g.ihx + (vN - vS) * g.ihy);
  const double diag = 1.0 / ph.dt + ph.th_ch * ph.Gamma1 * ((sx + sy) * lapd + sx * g.ihx2 + sy * g.ihy2) +
                      ph.th_adv * adiag;
  dinv[o] = 1.0 / diag;
}

// ------------------------------------------------------------ nutrient RHS
// a = phi_s^{n+1}/dt + A/2 phi^{1/2};  w = phi_s^{1/2};  volume fractions clipped (R24)
// b = phi_s^n c/dt - Adv(phi_s^n c) + 1/2 L_K c - A/2 phi^{1/2} c,  K = Ds * face mean(w)
__global__ void __launch_bounds__(256) k_nut_rhs(Geom g, Phys ph, StateP s,
                                                 const double* __restrict__ phi1, double* a,
                                                 double* w, double* b) {
  CHB_CELL_PREAMBLE(g)
  auto SH = [&](int jj, int ii) {
    return 1.0 - vfrac(0.5 * (ldf<BC_MIRROR>(s.phi, g, jj, ii) + ldf<BC_MIRROR>(phi1, g, jj, ii)));
  };
  auto W = [&](int jj, int ii) {
    return (1.0 - vfrac(ldf<BC_MIRROR>(s.phi, g, jj, ii))) * ldf<BC_MIRROR>(s.c, g, jj, ii);
  };
  auto C = [&](int jj, int ii) { return ldf<BC_MIRROR>(s.c, g, jj, ii); };
  const size_t o = off(g, j, i);
  const double phin = s.phi[o], p1 = phi1[o];
  const double phalf = vfrac(0.5 * (phin + p1));
  const double sh = 1.0 - phalf;
  const double cc = s.c[o];
  a[o] = (1.0 - vfrac(p1)) / ph.dt + 0.5 * ph.A * phalf;
  w[o] = sh;
  const double wc = W(j, i), we = W(j, ie), ww = W(j, iw), wn = W(j + 1, i), ws = W(j - 1, i);
  const double uE = s.u[off(g, j, ie)], uW = s.u[off(g, j, i)];
  const double vN = ldf<BC_VFACE>(s.v, g, j + 1, i), vS = ldf<BC_VFACE>(s.v, g, j, i);
  const double adv = (uE * 0.5 * (wc + we) - uW * 0.5 * (ww + wc)) * g.ihx +
                     (vN * 0.5 * (wc + wn) - vS * 0.5 * (ws + wc)) * g.ihy;
  const double kE = ph.Ds * 0.5 * (sh + SH(j, ie)), kW = ph.Ds * 0.5 * (SH(j, iw) + sh);
  const double kN = ph.Ds * 0.5 * (sh + SH(j + 1, i)), kS = ph.Ds * 0.5 * (SH(j - 1, i) + sh);
  const double lk = (kE * (C(j, ie) - cc) - kW * (cc - C(j, iw))) * g.ihx2 +
                    (kN * (C(j + 1, i) - cc) - kS * (cc - C(j - 1, i))) * g.ihy2;
  b[o] = wc / ph.dt - adv + 0.5 * lk - 0.5 * ph.A * phalf * cc;
}

// -------------------------------------------------------- momentum pieces
// Mixture density and viscosity eta = 1/Re_a = f/Re_n + (1-f)/Re_s of the
// volume fraction f = clip(phi, 0, 1) (Eq. 15, R6, R24).
__device__ __forceinline__ double dens(const Phys& ph, double phi) {
  return ph.rho_s + vfrac(phi) * (ph.rho_n - ph.rho_s);
}
__device__ __forceinline__ double visc_eta(const Phys& ph, double phi) {
  const double f = vfrac(phi);
  return f / ph.Re_n + (1.0 - f) / ph.Re_s;
}

struct PhiStar {
  const double* p;
  Geom g;
  __device__ __forceinline__ double operator()(int jj, int ii) const {
    return ldf<BC_MIRROR>(p, g, jj, wrapc(ii, g.nx));
  }
  // corner (x = ii hx, y = jj hy) product phi_x phi_y
  __device__ __forceinline__ double txy(int jj, int ii) const {
    const double a = (*this)(jj, ii), b = (*this)(jj - 1, ii);
    const double c = (*this)(jj, ii - 1), d = (*this)(jj - 1, ii - 1);
    return ((a + b - c - d) * 0.5 * g.ihx) * ((a + c - b - d) * 0.5 * g.ihy);
  }
  __device__ __forceinline__ double txx(int jj, int ii) const {
    const double d = ((*this)(jj, ii + 1) - (*this)(jj, ii - 1)) * 0.5 * g.ihx;
    return d * d;
  }
  __device__ __forceinline__ double tyy(int jj, int ii) const {
    const double d = ((*this)(jj + 1, ii) - (*this)(jj - 1, ii)) * 0.5 * g.ihy;
    return d * d;
  }
  // phi at the u point (x-face) (jj, ii), at the v point (y-face) (jj, ii), at a corner
  __device__ __forceinline__ double fu(int jj, int ii) const {
    return 0.5 * ((*this)(jj, ii - 1) + (*this)(jj, ii));
  }
  __device__ __forceinline__ double fv(int jj, int ii) const {
    return 0.5 * ((*this)(jj - 1, ii) + (*this)(jj, ii));
  }
  __device__ __forceinline__ double fk(int jj, int ii) const {
    return 0.25 * ((*this)(jj, ii) + (*this)(jj, ii - 1) + (*this)(jj - 1, ii) +
                   (*this)(jj - 1, ii - 1));
  }
};

// u on x-faces (R6, R7; th = theta_visc, 1 = the viscous term at u^{n+1}, Eq. 19):
//   a = rho/dt, w = eta at the u point,
//   b = a u + (1-th) div(eta grad u) + th lid - rho (v.grad)u + R_x,
//   R = -G1 div(grad phi* grad phi*) + div(eta (grad v)^T)       (Eq. 17)
__global__ void __launch_bounds__(256) k_mom_rhs_u(Geom g, Phys ph, StateP s,
                                                   const double* __restrict__ phis, double* a,
                                                   double* w, double* b) {
  CHB_CELL_PREAMBLE(g)
  PhiStar P{phis, g};
  const double rho = dens(ph, P.fu(j, i));
  const double ec = visc_eta(ph, P.fu(j, i));
  const double Rx = -ph.Gamma1 * ((P.txx(j, i) - P.txx(j, i - 1)) * g.ihx +
                                  (P.txy(j + 1, i) - P.txy(j, i)) * g.ihy);
  auto U = [&](int jj, int ii) { return ld_u_lid(s.u, g, jj, ii, ph.lid_u); };
  auto V = [&](int jj, int ii) { return ldf<BC_VFACE>(s.v, g, jj, wrapc(ii, g.nx)); };
  const size_t o = off(g, j, i);
  const double uc = s.u[o];
  const double vbar = 0.25 * (V(j, iw) + V(j, i) + V(j + 1, iw) + V(j + 1, i));
  const double cu = uc * (U(j, ie) - U(j, iw)) * 0.5 * g.ihx +
                    vbar * (U(j + 1, i) - U(j - 1, i)) * 0.5 * g.ihy;
  // div(eta grad u): face coefficient = mean of eta at the two u points; the
  // coefficient's wall ghost is its mirror image (PhiStar's mirror rows)
  const double kE = 0.5 * (ec + visc_eta(ph, P.fu(j, ie))), kW = 0.5 * (ec + visc_eta(ph, P.fu(j, iw)));
  const double kN = 0.5 * (ec + visc_eta(ph, P.fu(j + 1, i)));
  const double kS = 0.5 * (ec + visc_eta(ph, P.fu(j - 1, i)));
  const double lap = (kE * (U(j, ie) - uc) - kW * (uc - U(j, iw))) * g.ihx2 +
                     (kN * (U(j + 1, i) - uc) - kS * (uc - U(j - 1, i))) * g.ihy2;
  // div(eta (grad v)^T): eta du/dx at the cells left/right, eta dv/dx at the corners below/above
  const double qR = visc_eta(ph, P(j, i)) * (U(j, ie) - uc) * g.ihx;
  const double qL = visc_eta(ph, P(j, i - 1)) * (uc - U(j, iw)) * g.ihx;
  const double rN = visc_eta(ph, P.fk(j + 1, i)) * (V(j + 1, i) - V(j + 1, i - 1)) * g.ihx;
  const double rS = visc_eta(ph, P.fk(j, i)) * (V(j, i) - V(j, i - 1)) * g.ihx;
  const double Tx = (qR - qL) * g.ihx + (rN - rS) * g.ihy;
  const double ac = rho / ph.dt;
  double rhs = ac * uc + (1.0 - ph.th_visc) * lap - rho * cu + Rx + Tx;
  if (j == g.ny - 1) rhs += ph.th_visc * kN * 2.0 * ph.lid_u * g.ihy2;
  a[o] = ac;
  w[o] = ec;
  b[o] = rhs;
}

// v on y-faces j >= 1 (row 0 = wall: identity row, b = 0; its w = eta(phi[0]) is
// the coefficient source of the face between rows 0 and 1)
__global__ void __launch_bounds__(256) k_mom_rhs_v(Geom g, Phys ph, StateP s,
                                                   const double* __restrict__ phis, double* a,
                                                   double* w, double* b) {
  CHB_CELL_PREAMBLE(g)
  PhiStar P{phis, g};
  const size_t o = off(g, j, i);
  if (j == 0) {
    a[o] = 1.0;
    w[o] = visc_eta(ph, P(0, i));
    b[o] = 0.0;
    return;
  }
  const double rho = dens(ph, P.fv(j, i));
  const double ec = visc_eta(ph, P.fv(j, i));
  const double Ry = -ph.Gamma1 * ((P.txy(j, i + 1) - P.txy(j, i)) * g.ihx +
                                  (P.tyy(j, i) - P.tyy(j - 1, i)) * g.ihy);
  auto V = [&](int jj, int ii) { return ldf<BC_VFACE>(s.v, g, jj, ii); };
  auto Uc = [&](int jj, int ii) { return s.u[off(g, jj, ii)]; };
  const double vc = s.v[o];
  const double ubar = 0.25 * (Uc(j - 1, i) + Uc(j - 1, ie) + Uc(j, i) + Uc(j, ie));
  const double cv = ubar * (V(j, ie) - V(j, iw)) * 0.5 * g.ihx +
                    vc * (V(j + 1, i) - V(j - 1, i)) * 0.5 * g.ihy;
  const double kE = 0.5 * (ec + visc_eta(ph, P.fv(j, ie))), kW = 0.5 * (ec + visc_eta(ph, P.fv(j, iw)));
  // eta at the v point below (row 0: eta(phi[0])), above (top ghost: the mirror, eta itself)
  const double eS = j == 1 ? visc_eta(ph, P(0, i)) : visc_eta(ph, P.fv(j - 1, i));
  const double eN = j == g.ny - 1 ? ec : visc_eta(ph, P.fv(j + 1, i));
  const double kN = 0.5 * (ec + eN), kS = 0.5 * (ec + eS);
  const double lap = (kE * (V(j, ie) - vc) - kW * (vc - V(j, iw))) * g.ihx2 +
                     (kN * (V(j + 1, i) - vc) - kS * (vc - V(j - 1, i))) * g.ihy2;
  // div(eta (grad v)^T): eta du/dy at the corners left/right, eta dv/dy at the cells below/above
  const double qR = visc_eta(ph, P.fk(j, i + 1)) * (Uc(j, ie) - Uc(j - 1, ie)) * g.ihy;
  const double qL = visc_eta(ph, P.fk(j, i)) * (Uc(j, i) - Uc(j - 1, i)) * g.ihy;
  const double rN = visc_eta(ph, P(j, i)) * (V(j + 1, i) - vc) * g.ihy;
  const double rS = visc_eta(ph, P(j - 1, i)) * (vc - V(j - 1, i)) * g.ihy;
  const double Ty = (qR - qL) * g.ihx + (rN - rS) * g.ihy;
  const double ac = rho / ph.dt;
  a[o] = ac;
  w[o] = ec;
  b[o] = ac * vc + (1.0 - ph.th_visc) * lap - rho * cv + Ry + Ty;
}

// ---------------------------------------------------------- projection
// b = D_h(u*, v*) (Eq. 20 RHS), reduced sum -> mean (null-space projection)
__global__ void __launch_bounds__(256) k_div(Geom g, const double* __restrict__ us,
                                             const double* __restrict__ vs, double* b,
                                             RedArgs ra) {
  // grid-strided over rows: the number of CTAs (= reduction partials) stays bounded
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (i < g.nx) {
    const int ie = wrapc(i + 1, g.nx);
    for (int jl = blockIdx.y * blockDim.y + threadIdx.y; jl < g.nyl;
         jl += gridDim.y * blockDim.y) {
      const int j = g.j0 + jl;
      const double d = (us[off(g, j, ie)] - us[off(g, j, i)]) * g.ihx +
                       (ldf<BC_VFACE>(vs, g, j + 1, i) - ldf<BC_VFACE>(vs, g, j, i)) * g.ihy;
      b[off(g, j, i)] = d;
      acc += d;
    }
  }
  double v[1] = {acc};
  block_reduce_finalize<1>(v, ra);
}

// v^{n+1} = u* + beta G_h p  (Eq. 21)
__global__ void __launch_bounds__(256) k_project(Geom g, Phys ph, const double* __restrict__ phi1,
                                                 const double* __restrict__ us,
                                                 const double* __restrict__ vs,
                                                 const double* __restrict__ p, double* u,
                                                 double* v) {
  CHB_CELL_PREAMBLE(g)
  (void)ie;
  const size_t o = off(g, j, i);
  const double fu = vfrac(0.5 * (phi1[off(g, j, iw)] + phi1[o]));
  const double bu = 1.0 / (ph.rho_s + fu * (ph.rho_n - ph.rho_s));
  u[o] = us[o] + bu * (p[o] - p[off(g, j, iw)]) * g.ihx;
  if (j == 0) {
    v[o] = 0.0;
  } else {
    const double fv = vfrac(0.5 * (phi1[off(g, j - 1, i)] + phi1[o]));
    const double bv = 1.0 / (ph.rho_s + fv * (ph.rho_n - ph.rho_s));
    v[o] = vs[o] + bv * (p[o] - p[off(g, j - 1, i)]) * g.ihy;
  }
}

void launch_ch_rhs(const Geom& g, const Phys& ph, StateP s, double* phis, double* dinv,
                   double* b, cudaStream_t st) {
  k_ch_rhs<<<grid2(g), blk2, 0, st>>>(g, ph, s, phis, dinv, b);
}
void launch_nut_rhs(const Geom& g, const Phys& ph, StateP s, const double* phi1, double* a,
                    double* w, double* b, cudaStream_t st) {
  k_nut_rhs<<<grid2(g), blk2, 0, st>>>(g, ph, s, phi1, a, w, b);
}
void launch_mom_rhs_u(const Geom& g, const Phys& ph, StateP s, const double* phis, double* a,
                      double* w, double* b, cudaStream_t st) {
  k_mom_rhs_u<<<grid2(g), blk2, 0, st>>>(g, ph, s, phis, a, w, b);
}
void launch_mom_rhs_v(const Geom& g, const Phys& ph, StateP s, const double* phis, double* a,
                      double* w, double* b, cudaStream_t st) {
  k_mom_rhs_v<<<grid2(g), blk2, 0, st>>>(g, ph, s, phis, a, w, b);
}
void launch_div(const Geom& g, const double* us, const double* vs, double* b, const RedArgs& ra,
                cudaStream_t st) {
  dim3 gr = grid2(g);
  if (gr.y > 256) gr.y = 256;   // <= 512 x 256 partials even at 16384^2
  k_div<<<gr, blk2, 0, st>>>(g, us, vs, b, ra);
}
void launch_project(const Geom& g, const Phys& ph, const double* phi1, const double* us,
                    const double* vs, const double* p, double* u, double* v, cudaStream_t st) {
  k_project<<<grid2(g), blk2, 0, st>>>(g, ph, phi1, us, vs, p, u, v);
}

}  // namespace chb
