// launch.h -- host-side launchers of the device kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace chb {

enum OpKind : int {
  OPK_POISSON_CONST = 0,
  OPK_POISSON_VAR = 1,
  OPK_NUTRIENT = 2,
  OPK_MOM_U = 3,
  OPK_MOM_V = 4,
  OPK_MOM_U_C = 5,   // momentum with constant density: a = rho/dt is a scalar (rho_n == rho_s)
  OPK_MOM_V_C = 6
};

// Operator descriptor for the 5-point family (op5.cuh, kernels_aux.cu, kernels_cgs.cu).
struct OpDesc {
  int kind;
  int strip;          // rows per marching strip (column-marching kernels)
  int strip2;         // rows per strip of the fused CG sweep (0 = one resident wave)
  int pdl;            // programmatic dependent launch for the fused CG sweeps
  const double* a;    // diagonal coefficient array (NUTRIENT, MOM_*)
  const double* w;    // cell coefficient (NUTRIENT: phi_s^{1/2}; POISSON_VAR: phi^{n+1})
  double s, kscale, rho_n, rho_s;
  double ascal;       // the diagonal coefficient of the *_C kinds
};

void launch_cg5_init(const OpDesc& d, const Geom& g, const double* x, const double* b,
                     int use_shift, double* z, const RedArgs& ra, cudaStream_t st);
void launch_op5_apply(const OpDesc& d, const Geom& g, const double* x, double* y,
                      cudaStream_t st);
void launch_cg5_finish(const Geom& g, double* x, const double* p, int nullspace, int odd_only,
                       const RedArgs& ra, cudaStream_t st);
// single-reduction CG (kernels_cgs.cu), even nx only
// tt = 1: three-term z recurrence (si = z_{i-1}, so unused); 0: s = A p recurrence
void launch_cgs_iter(const OpDesc& d, const Geom& g, const double* zi, double* zo,
                     const double* si, double* so, int first, int dir, int tt, const RedArgs& ra,
                     cudaStream_t st);
// one sweep launch over all local slabs (halo rows stored into the neighbours'
// ghost rows, cross-slab finalize by the last slab), common.cuh MsArgs
void launch_cgs_iter_ms(const OpDesc& d, const MsArgs& ms, int first, int dir, int tt,
                        const RedArgs& ra, cudaStream_t st);
struct ZList {
  const double* z[CGM];
};
void launch_cgs_px(const Geom& g, const ZList& zl, int n, int first_block, int write_p, int need,
                   const double* T, const KScal* sc, double* P, double* X, cudaStream_t st);

// peer-memory clique probe (xrank.cu): edge rows into the neighbours' ghost
// rows + one cross-rank combine, as one multi-slab CG iteration does them
void launch_peer_probe(const XPeers* xp, unsigned epoch, double* loc, int nloc, const Geom& g0,
                       double* lo, const Geom& g1, double* hi, double* out, cudaStream_t st);
void launch_cgs_delta0(const OpDesc& d, const Geom& g, const double* z, const RedArgs& ra,
                       cudaStream_t st);
double cgs_bytes(int kind, int first, int tt);
void launch_sum(const Geom& g, const double* x, const RedArgs& ra, cudaStream_t st);
void launch_sub_mean(const Geom& g, double* x, const KScal* sc, cudaStream_t st);
void launch_finalize_slabs(const double* tot, int nslabs, int K, const RedArgs& ra,
                           cudaStream_t st);

// ---- Cahn-Hilliard 13-point operator and BiCGStab / GMRES vector kernels
struct ChCoef {
  const double* phis;  // phi* (mobility source)
  const double* dinv;  // Jacobi inverse diagonal (nullptr: no scaling)
  const double* u;     // face velocities v^n of the implicit advection part
  const double* v;     //   (u == nullptr: no advection part)
  double dt, g1t, Lambda;  // g1t = theta_ch * Gamma1
  double tha;              // theta_adv
  int strip;               // forced rows per strip (0: one resident wave; env CHB_STRIP)
};
// y = A (dinv .* x)  [or A x when dinv == nullptr]; fused dots:
//   ndot = 0: none; 1: (y, d1); 2: (y, d1), (y, d2) where d2 == nullptr means (y, y)
void launch_ch_apply(const Geom& g, const ChCoef& cc, const double* x, double* y, int ndot,
                     const double* d1, const double* d2, int skip_if_done, int skip_if_half,
                     const RedArgs& ra, cudaStream_t st);

void launch_bi_init(const Geom& g, const double* y, const double* b, double* r, double* rhat,
                    const RedArgs& ra, cudaStream_t st);
void launch_bi_p(const Geom& g, const double* r, double* p, const double* v, int first,
                 const KScal* sc, cudaStream_t st);
void launch_bi_s(const Geom& g, const double* r, const double* v, double* s, const RedArgs& ra,
                 cudaStream_t st);
void launch_bi_xr(const Geom& g, double* x, const double* p, const double* s, const double* t,
                  double* r, const double* rhat, const double* dinv, const RedArgs& ra,
                  cudaStream_t st);

// GMRES (classical Gram-Schmidt with one re-orthogonalisation, CGS2); V has <= 66 vectors
void launch_gm_dots(const Geom& g, double* const* V, int k, const double* w, double* out,
                    double* part, unsigned int* ticket, cudaStream_t st);
void launch_gm_scale(const Geom& g, double* v, const double* coef, cudaStream_t st);
void launch_gm_axpy_multi(const Geom& g, double* const* V, int k, const double* coef, double* w,
                          cudaStream_t st);
void launch_gm_residual(const Geom& g, const double* y, const double* b, double* v0,
                        cudaStream_t st);
void launch_gm_update_x(const Geom& g, double* const* V, int k, const double* coef,
                        const double* dinv, double* x, cudaStream_t st);

// ---- explicit right-hand sides and projection (kernels_rhs.cu)
struct Phys {
  double dt, Gamma1, Gamma2, Lambda, mu, Kc, eps, A, Ds, Re_s, Re_n, rho_n, rho_s, lid_u;
  double th_ch, th_adv, th_visc;  // implicit weights of this step (R5, R12, R7, R23)
};
struct StateP {
  const double *phi, *phip, *c, *u, *v, *p;
};
void launch_ch_rhs(const Geom& g, const Phys& ph, StateP s, double* phis, double* dinv,
                   double* b, cudaStream_t st);
void launch_nut_rhs(const Geom& g, const Phys& ph, StateP s, const double* phi1, double* a,
                    double* w, double* b, cudaStream_t st);
void launch_mom_rhs_u(const Geom& g, const Phys& ph, StateP s, const double* phis, double* a,
                      double* w, double* b, cudaStream_t st);
void launch_mom_rhs_v(const Geom& g, const Phys& ph, StateP s, const double* phis, double* a,
                      double* w, double* b, cudaStream_t st);
void launch_div(const Geom& g, const double* us, const double* vs, double* b, const RedArgs& ra,
                cudaStream_t st);
void launch_project(const Geom& g, const Phys& ph, const double* phi1, const double* us,
                    const double* vs, const double* p, double* u, double* v, cudaStream_t st);

}  // namespace chb
