// common.cuh -- device-side building blocks shared by all kernels of the
// B200 hot path (slab geometry, wall ghost rules applied at read time,
// deterministic block reductions with a last-block finalizer, Krylov scalars).
//
// DESIGN.md §2 (discretisation) and §5 (layout).  Nothing here is shared with
// oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace chb {

constexpr int GH = 2;               // ghost rows stored below and above a slab
constexpr unsigned FULL = 0xffffffffu;

// Ghost rules of the unknown / field (R2-R4).
enum Bc : int {
  BC_MIRROR = 0,  // cell-centred scalar: s[-1-k] = s[k], s[ny+k] = s[ny-1-k]
  BC_ODD = 1,     // u on x-faces, homogeneous: u[-1-k] = -u[k] (lid handled by RHS)
  BC_VFACE = 2    // v on y-faces: v = 0 on the wall faces j = 0 and j = ny
};

// Geometry of one slab (rows [j0, j0+nyl) of the global nx x ny grid).
struct Geom {
  int nx, ny;       // global cells
  int j0, nyl;      // first global row, local row count
  int pitch;        // doubles per stored row (>= nx, multiple of 32)
  int pad;
  double hx, hy, ihx, ihy, ihx2, ihy2;
};

__device__ __forceinline__ size_t off(const Geom& g, int gj, int c) {
  return (size_t)(gj - g.j0 + GH) * (size_t)g.pitch + (size_t)c;
}

// Load value of a field with ghost rule BC at global row gj (|overhang| <= 2),
// column c in [0, nx).  Rows outside the slab but inside the domain come from
// the stored ghost rows (filled by the halo exchange).
template <int BC>
__device__ __forceinline__ double ldf(const double* __restrict__ a, const Geom& g, int gj, int c) {
  if (BC == BC_VFACE) {
    if (gj <= 0 || gj >= g.ny) return 0.0;
    return a[off(g, gj, c)];
  }
  if (gj < 0) {
    double v = a[off(g, -1 - gj, c)];
    return BC == BC_ODD ? -v : v;
  }
  if (gj >= g.ny) {
    double v = a[off(g, 2 * g.ny - 1 - gj, c)];
    return BC == BC_ODD ? -v : v;
  }
  return a[off(g, gj, c)];
}

// u (state) with the inhomogeneous wall values: no-slip below, lid above.
__device__ __forceinline__ double ld_u_lid(const double* __restrict__ u, const Geom& g, int gj,
                                           int c, double lid) {
  if (gj < 0) return -u[off(g, -1 - gj, c)];
  if (gj >= g.ny) return 2.0 * lid - u[off(g, 2 * g.ny - 1 - gj, c)];
  return u[off(g, gj, c)];
}

__device__ __forceinline__ int wrapc(int c, int nx) { return c < 0 ? c + nx : (c >= nx ? c - nx : c); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// ----------------------------------------------------------- Krylov scalars
struct KScal {
  double rho, rho_prev, alpha, beta, omega;
  double bb, tol2, rr, last;      // ||b||^2, rtol^2 ||b||^2, ||r||^2, scratch
  double mean;                    // mean used by null-space projections
  double aux[6];
  int iter, done, status, half;   // status: 0 ok, 1 breakdown, 2 maxit
  int zero, maxit, pad0, pad1;
};

enum Fin : int {
  FIN_NONE = 0,
  FIN_CG_INIT,     // [bb, rz, rr]
  FIN_CG_A,        // [pq]
  FIN_CG_B,        // [rz, rr]
  FIN_BI_INIT,     // [bb, rr]           (rhat = r  => rho = rr)
  FIN_BI_ALPHA,    // [rhat.v]
  FIN_BI_S,        // [s.s]
  FIN_BI_OMEGA,    // [t.s, t.t]
  FIN_BI_R,        // [r.r, rhat.r]
  FIN_MEAN,        // [sum]  -> mean = sum / ncells
  FIN_STORE,       // [v...] -> aux[k] = v[k]
  FIN_CGS_D0,      // [delta_0]                 single-reduction CG start
  FIN_CGS          // [gamma, r.r, delta]       single-reduction CG iteration
};

struct FinCtx {
  double rtol2;
  double ncells;
  double* tab;   // single-reduction CG with deferred p/x: coefficient tables of
                 // this system, [2][CGT] (block parity), see cgs_coef_update
  int m;         // iterations per deferred p/x block (0: p/x updated in-sweep)
  int pad;
};

// Deferred p/x of the single-reduction CG (kernels_cgs.cu).  Within a block of
// m iterations i0..i0+m-1 the directions and iterates are linear in the
// stored preconditioned residuals z_k:
//   p_i     = sum_k PZ[k] z_k + CPP p_{i0-1}
//   x_{i+1} = x_{i0} + sum_k CZ[k] z_k + CXP p_{i0-1}
// and the table follows the textbook updates p_i = z_i + beta_i p_{i-1},
// x_{i+1} = x_i + alpha_i p_i exactly (only the summation order of x differs).
constexpr int CGM = 64;   // max block length
constexpr int CGT = 136;  // table stride (>= 2 CGM + 3)
enum { CG_PZ = 0, CG_CZ = CGM, CG_CPP = 2 * CGM, CG_CXP = 2 * CGM + 1, CG_N = 2 * CGM + 2 };

__device__ inline void cgs_coef_update(double* tab, int m, int i, double alpha, double beta) {
  if (!tab || m <= 0) return;
  double* T = tab + ((i / m) & 1) * CGT;
  const int j = i % m;
  if (j == 0) {
    for (int k = 0; k < CGM; ++k) T[CG_PZ + k] = T[CG_CZ + k] = 0.0;
    T[CG_CPP] = 1.0;
    T[CG_CXP] = 0.0;
  }
  for (int k = 0; k < j; ++k) T[CG_PZ + k] *= beta;
  T[CG_CPP] *= beta;
  T[CG_PZ + j] = 1.0;
  for (int k = 0; k <= j; ++k) T[CG_CZ + k] += alpha * T[CG_PZ + k];
  T[CG_CXP] += alpha * T[CG_CPP];
  T[CG_N] = (double)(j + 1);
}

// The same update by the 32 lanes of one warp, lane l owning slots l, l + 32
// (CGM / 32 per lane): two dependent L2 round trips instead of ~2 j serial
// ones on the per-iteration critical path (the last CTA's finalize).
static_assert(CGM % 32 == 0 && CGM <= 64, "CGM / 32 deferred z slots per lane");
constexpr int CGS_SLOTS = CGM / 32;
__device__ inline void cgs_coef_update_warp(double* tab, int m, int i, double alpha, double beta,
                                            int lane) {
  if (!tab || m <= 0) return;
  double* T = tab + ((i / m) & 1) * CGT;
  const int j = i % m;
  double cpp = 1.0, cxp = 0.0;
  if (j != 0) {
    cpp = T[CG_CPP];
    cxp = T[CG_CXP];
  }
#pragma unroll
  for (int r = 0; r < CGS_SLOTS; ++r) {
    const int k = lane + 32 * r;
    double pz = 0.0, cz = 0.0;
    if (j != 0) {
      pz = T[CG_PZ + k];
      cz = T[CG_CZ + k];
    }
    if (k < j) pz *= beta;
    if (k == j) pz = 1.0;
    if (k <= j) cz += alpha * pz;
    T[CG_PZ + k] = pz;
    T[CG_CZ + k] = cz;
  }
  if (lane == 0) {
    cpp *= beta;
    cxp += alpha * cpp;
    T[CG_CPP] = cpp;
    T[CG_CXP] = cxp;
    T[CG_N] = (double)(j + 1);
  }
}

// A deferred coefficient-table update requested by finalize (see finalize_warp).
struct CoefReq {
  int valid, i;
  double alpha, beta;
};

__device__ __forceinline__ bool bad(double x) { return !(x == x) || x == 0.0; }
// CG on an SPD operator: (r, z), (A z, z) and the step denominator are > 0
// and finite; anything else means an indefinite operator or lost arithmetic.
__device__ __forceinline__ bool not_pos(double x) { return !(x > 0.0) || !(x < 1e308); }

// Breakdown codes in KScal.status (>= 3; 1 = generic, 2 = maxit), the value
// that tripped is left in KScal.last (reported by ch_last_error).
enum KStatus : int {
  KS_OK = 0, KS_BREAK = 1, KS_MAXIT = 2,
  KS_CG_GAMMA = 3,   // (r, z) <= 0 or not finite
  KS_CG_DELTA = 4,   // (A z, z) <= 0 or not finite
  KS_CG_DEN = 5,     // alpha's denominator delta - beta gamma / alpha <= 0
  KS_CG_OMEGA = 6,   // three-term recurrence omega not finite
  KS_BI_RHO = 7,     // BiCGStab (r^, r) = 0 or not finite
  KS_BI_RV = 8,      // BiCGStab (r^, v) = 0 or not finite
  KS_BI_TT = 9,      // BiCGStab (t, t) = 0 or not finite, or omega = 0
  KS_RES_NAN = 10,   // residual norm not finite
  KS_PEER_TIMEOUT = 11  // cross-rank combine: a rank's totals never arrived (~2 s)
};
__device__ __forceinline__ void kfail(KScal* s, int code, double val) {
  s->status = code;
  s->last = val;
  s->done = 1;
}

__device__ inline void finalize(int fin, const double* t, KScal* s, const FinCtx& fc,
                                CoefReq* req = nullptr) {
  switch (fin) {
    case FIN_CG_INIT: {
      s->bb = t[0];
      s->tol2 = fc.rtol2 * t[0];
      s->rho = t[1];
      s->rr = t[2];
      s->iter = 0;
      s->status = 0;
      s->half = 0;
      s->zero = (t[0] == 0.0);
      s->done = s->zero || (t[2] <= s->tol2);
      break;
    }
    case FIN_CG_A: {
      if (bad(t[0]) || !(s->rho == s->rho)) { s->status = 1; s->done = 1; break; }
      s->alpha = s->rho / t[0];
      break;
    }
    case FIN_CG_B: {
      s->iter += 1;
      s->rr = t[1];
      if (t[1] <= s->tol2) { s->done = 1; break; }
      if (s->iter >= s->maxit) { s->status = 2; s->done = 1; break; }
      s->beta = t[0] / s->rho;
      s->rho = t[0];
      break;
    }
    case FIN_BI_INIT: {
      s->bb = t[0];
      s->tol2 = fc.rtol2 * t[0];
      s->rr = t[1];
      s->rho = t[1];
      s->rho_prev = 1.0;
      s->alpha = 1.0;
      s->omega = 1.0;
      s->iter = 0;
      s->status = 0;
      s->half = 0;
      s->zero = (t[0] == 0.0);
      s->done = s->zero || (t[1] <= s->tol2);
      break;
    }
    case FIN_BI_ALPHA: {
      if (bad(t[0])) { kfail(s, KS_BI_RV, t[0]); break; }
      s->alpha = s->rho / t[0];
      break;
    }
    case FIN_BI_S: {
      s->half = (t[0] <= s->tol2);
      if (s->half) s->rr = t[0];
      break;
    }
    case FIN_BI_OMEGA: {
      if (s->half) break;
      if (bad(t[1])) { kfail(s, KS_BI_TT, t[1]); break; }
      s->omega = t[0] / t[1];
      break;
    }
    case FIN_BI_R: {
      s->iter += 1;
      if (s->half) { s->done = 1; break; }
      s->rr = t[0];
      if (t[0] <= s->tol2) { s->done = 1; break; }
      if (!(t[0] < 1e308)) { kfail(s, KS_RES_NAN, t[0]); break; }
      if (s->iter >= s->maxit) { s->status = 2; s->done = 1; break; }
      if (s->omega == 0.0) { kfail(s, KS_BI_TT, s->omega); break; }
      if (bad(t[1])) { kfail(s, KS_BI_RHO, t[1]); break; }
      s->rho_prev = s->rho;
      s->rho = t[1];
      break;
    }
    case FIN_MEAN: {
      s->mean = t[0] / fc.ncells;
      break;
    }
    case FIN_CGS_D0: {
      if (s->done) break;
      if (not_pos(t[0])) { kfail(s, KS_CG_DELTA, t[0]); break; }
      s->alpha = s->rho / t[0];
      s->beta = 0.0;
      s->aux[0] = 0.0;
      s->aux[4] = s->alpha;  // three-term z recurrence: gamma_0 = alpha_0, omega_1 = 1
      s->aux[5] = 1.0;
      if (req) *req = CoefReq{1, 0, s->alpha, 0.0};
      else cgs_coef_update(fc.tab, fc.m, 0, s->alpha, 0.0);
      break;
    }
    case FIN_CGS: {
      // Chronopoulos-Gear: beta = gamma'/gamma, alpha' = gamma'/(delta' - beta gamma'/alpha)
      s->iter += 1;
      s->rr = t[1];
      if (t[1] <= s->tol2) { s->done = 1; break; }
      if (!(t[1] < 1e308)) { kfail(s, KS_RES_NAN, t[1]); break; }
      if (s->iter >= s->maxit) { s->status = 2; s->done = 1; break; }
      if (not_pos(t[0])) { kfail(s, KS_CG_GAMMA, t[0]); break; }
      if (not_pos(t[2])) { kfail(s, KS_CG_DELTA, t[2]); break; }
      const double beta = t[0] / s->rho;
      const double den = t[2] - beta * t[0] / s->alpha;
      if (not_pos(den)) { kfail(s, KS_CG_DEN, den); break; }
      // three-term z recurrence (Concus-Golub-O'Leary form, kernels_cgs.cu):
      // gamma' = mu'/nu', omega' = 1 / (1 - (gamma'/gamma) (mu'/mu) / omega)
      const double gnew = t[0] / t[2];
      const double om = 1.0 / (1.0 - (gnew / s->aux[4]) * (t[0] / s->rho) / s->aux[5]);
      if (!(fabs(om) < 1e300)) { kfail(s, KS_CG_OMEGA, om); break; }
      s->aux[4] = gnew;
      s->aux[5] = om;
      s->aux[0] = s->alpha;  // alpha_{i} for the in-sweep x update over pairs
      s->beta = beta;
      s->alpha = t[0] / den;
      s->rho = t[0];
      if (req) *req = CoefReq{1, s->iter, s->alpha, beta};
      else cgs_coef_update(fc.tab, fc.m, s->iter, s->alpha, beta);
      break;
    }
    case FIN_STORE: {
      for (int k = 0; k < 6; ++k) s->aux[k] = t[k];
      break;
    }
    default:
      break;
  }
}

// finalize() run by all 32 lanes of a warp (t valid in lane 0): lane 0 updates
// the scalars, the lanes then share the coefficient-table update.
__device__ inline void finalize_warp(int fin, const double* t, KScal* s, const FinCtx& fc) {
  const int lane = threadIdx.x & 31;
  CoefReq req{0, 0, 0.0, 0.0};
  if (lane == 0) finalize(fin, t, s, fc, &req);
  req.valid = __shfl_sync(FULL, req.valid, 0);
  if (!req.valid) return;
  req.i = __shfl_sync(FULL, req.i, 0);
  req.alpha = __shfl_sync(FULL, req.alpha, 0);
  req.beta = __shfl_sync(FULL, req.beta, 0);
  cgs_coef_update_warp(fc.tab, fc.m, req.i, req.alpha, req.beta, lane);
}

// FIN_CGS with its scalar inputs prefetched (CgsPre, loaded by the sweep
// while its ring fills) and its coefficient-table slots loaded together with
// the partial sums: the last CTA's finalize then adds no global round trip
// to the critical path between sweeps.  Run by all 32 lanes of warp 0 (the
// scalar logic redundantly, lane 0 stores the scalars, lane k table slot k);
// same arithmetic and outcomes as finalize(FIN_CGS).
struct CgsPre {
  double rho, alpha, aux4, aux5, tol2;
  int iter, maxit;
};

__device__ inline void cgs_prefetch(CgsPre& p, const KScal* s, int lane) {
  if (lane == 0) {
    p.iter = __ldcg(&s->iter);
    p.maxit = __ldcg(&s->maxit);
    p.rho = __ldcg(&s->rho);
    p.alpha = __ldcg(&s->alpha);
    p.aux4 = __ldcg(&s->aux[4]);
    p.aux5 = __ldcg(&s->aux[5]);
    p.tol2 = __ldcg(&s->tol2);
  }
}

// table slot `lane` (+ CPP, CXP) of the iteration the finalize will record
struct CgsSlot {
  double pz[CGS_SLOTS], cz[CGS_SLOTS], cpp, cxp;
};
__device__ inline CgsSlot cgs_slot_load(const CgsPre& p, const FinCtx& fc, int lane) {
  CgsSlot o;
#pragma unroll
  for (int r = 0; r < CGS_SLOTS; ++r) o.pz[r] = o.cz[r] = 0.0;
  o.cpp = 1.0;
  o.cxp = 0.0;
  if (!fc.tab || fc.m <= 0) return o;
  const int i = p.iter + 1;
  const double* T = fc.tab + ((i / fc.m) & 1) * CGT;
#pragma unroll
  for (int r = 0; r < CGS_SLOTS; ++r) {
    o.pz[r] = __ldcg(T + CG_PZ + lane + 32 * r);
    o.cz[r] = __ldcg(T + CG_CZ + lane + 32 * r);
  }
  o.cpp = __ldcg(T + CG_CPP);
  o.cxp = __ldcg(T + CG_CXP);
  return o;
}

__device__ inline void finalize_cgs_pre(const double* t, const CgsPre& p, const CgsSlot& sl,
                                        KScal* s, const FinCtx& fc, int lane) {
  const int iter = p.iter + 1;
  int done = 0, status = 0;
  double beta = 0.0, alpha = 0.0, gnew = 0.0, om = 0.0, val = 0.0;
  if (t[1] <= p.tol2) {
    done = 1;
  } else if (!(t[1] < 1e308)) {
    status = KS_RES_NAN, val = t[1], done = 1;
  } else if (iter >= p.maxit) {
    status = KS_MAXIT;
    done = 1;
  } else if (not_pos(t[0])) {
    status = KS_CG_GAMMA, val = t[0], done = 1;
  } else if (not_pos(t[2])) {
    status = KS_CG_DELTA, val = t[2], done = 1;
  } else {
    beta = t[0] / p.rho;
    const double den = t[2] - beta * t[0] / p.alpha;
    gnew = t[0] / t[2];
    om = 1.0 / (1.0 - (gnew / p.aux4) * (t[0] / p.rho) / p.aux5);
    if (not_pos(den)) {
      status = KS_CG_DEN, val = den, done = 1;
    } else if (!(fabs(om) < 1e300)) {
      status = KS_CG_OMEGA, val = om, done = 1;
    } else {
      alpha = t[0] / den;
    }
  }
  if (lane == 0) {
    s->iter = iter;
    s->rr = t[1];
    if (done) {
      if (status) {
        s->status = status;
        s->last = val;
      }
      s->done = 1;
    } else {
      s->aux[4] = gnew;
      s->aux[5] = om;
      s->aux[0] = p.alpha;
      s->beta = beta;
      s->alpha = alpha;
      s->rho = t[0];
    }
  }
  if (done || !fc.tab || fc.m <= 0) return;
  double* T = fc.tab + ((iter / fc.m) & 1) * CGT;
  const int j = iter % fc.m;
  double cpp = 1.0, cxp = 0.0;
  if (j != 0) {
    cpp = sl.cpp;
    cxp = sl.cxp;
  }
#pragma unroll
  for (int r = 0; r < CGS_SLOTS; ++r) {
    const int k = lane + 32 * r;
    double pz = 0.0, cz = 0.0;
    if (j != 0) {
      pz = sl.pz[r];
      cz = sl.cz[r];
    }
    if (k < j) pz *= beta;
    if (k == j) pz = 1.0;
    if (k <= j) cz += alpha * pz;
    T[CG_PZ + k] = pz;
    T[CG_CZ + k] = cz;
  }
  if (lane == 0) {
    cpp *= beta;
    cxp += alpha * cpp;
    T[CG_CPP] = cpp;
    T[CG_CXP] = cxp;
    T[CG_N] = (double)(j + 1);
  }
}

#ifdef CHB_TRACE
// (kernels_cgs.cu) timing trace of the last k_cgs_iter launch (experiments only): per CTA
// globaltimer at entry, after griddepcontrol.wait, ring ready, loop end,
// after the reduction (+ finalize in the last CTA); clock64 of the same points
__device__ unsigned long long chb_trace[8192 * 16];
__device__ __forceinline__ void trace_now(unsigned long long& gt, unsigned long long& ck) {
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck));
}
__device__ __forceinline__ void trace_put(int i, unsigned long long gt, unsigned long long ck) {
  if (threadIdx.x != 0) return;
  chb_trace[blockIdx.x * 16 + i] = gt;
  chb_trace[blockIdx.x * 16 + 8 + i] = ck;
}
__device__ unsigned int chb_trace_smid[8192];
__device__ __forceinline__ void trace_smid() {
  if (threadIdx.x != 0) return;
  unsigned int sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  chb_trace_smid[blockIdx.x] = sm;
}
// dispatch order of the CTA on its SM: a per-SM counter taken at entry (the
// raw count; every launch adds its resident CTAs per SM, so count mod per-SM
// residency is the order within the launch)
__device__ unsigned int chb_trace_smctr[1024];
__device__ unsigned int chb_trace_order[8192];
__device__ __forceinline__ void trace_order() {
  if (threadIdx.x != 0) return;
  unsigned int sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  chb_trace_order[blockIdx.x] = atomicAdd(&chb_trace_smctr[sm & 1023], 1u);
}
__device__ __forceinline__ void trace_pt(int i) {
  unsigned long long gt, ck;
  trace_now(gt, ck);
  trace_put(i, gt, ck);
}
#define CHB_TP(i) trace_pt(i)
#else
#define CHB_TP(i) ((void)0)
#endif

// Reduction plumbing: every block writes K partial sums; the last block to
// finish (atomic ticket) sums the partials in fixed block order (deterministic)
// and either finalizes inline (single slab, single rank) or stores the slab
// total for a later cross-slab finalize.
// Cross-rank combine of the per-slab totals of one CG iteration over peer
// memory (NVLink P2P between the processes of a clique; within one process
// the same code with R = 1).  Every rank owns a totals area [2][XS_MAX][8]
// (double-buffered by iteration parity) and XR_MAX arrival flags; the last
// slab of a rank to finish pushes its slabs' totals into EVERY rank's area
// (peer stores), then stores the iteration's epoch into its flag on every
// rank (release, system scope), waits until all R flags on its own rank
// carry the epoch (acquire) and sums the totals in global slab order: every
// rank computes bit-identical scalars with no NCCL call and no extra launch.
constexpr int XR_MAX = 8, XS_MAX = 64;
struct XPeers {
  int R, rank;            // ranks in the clique, this rank
  int slab0, nslab_all;   // global index of this rank's first slab; slabs over all ranks
  double* tot[XR_MAX];    // rank q's totals area (peer-mapped; [rank] is local)
  unsigned* flag[XR_MAX]; // rank q's arrival flags [XR_MAX] (peer-mapped)
};

struct RedArgs {
  double* part;          // [nblocks * 8]
  unsigned int* ticket;  // zeroed; reset by the last block (multi-slab launch: one per slab)
  double* tot;           // [nslabs_total * 8] slab totals (when !inline_fin)
  KScal* sc;
  FinCtx fc;
  int fin;
  int inline_fin;
  int slab;              // index of this slab in tot
  int pad;
  // one launch over several slabs (nbs > 0): blocks [s*nbs, (s+1)*nbs) are slab
  // s, each slab's last block stores the slab total, the last slab to finish
  // (ticket2) combines the totals in slab order and finalizes
  int nbs;
  int nslab;
  unsigned int* ticket2;
  // multi-slab launch: cross-rank combine (xp: device XPeers; epoch: this
  // launch's number, > 0, the same on every rank)
  const XPeers* xp;
  unsigned epoch;
  int pad2;
};

// The combine of one rank's last slab (one warp, all lanes): push the nloc
// local slab totals (loc[s * 8 + k]) to every rank, arrive, wait for every
// rank, sum the totals of all slabs in slab order into t.  false: a rank did
// not arrive within ~2 s (the caller reports KS_PEER_TIMEOUT; never a hang).
template <int K>
__device__ __forceinline__ bool xrank_combine(const XPeers* xpp, unsigned epoch, const double* loc,
                                              int nloc, double (&t)[8]) {
  const int lane = threadIdx.x & 31;
  const int R = xpp->R, me = xpp->rank, slab0 = xpp->slab0, nall = xpp->nslab_all;
  const size_t par = (size_t)(epoch & 1u) * XS_MAX;
  const int n = R * nloc * K;
  for (int i = lane; i < n; i += 32) {
    const int q = i / (nloc * K), r = i % (nloc * K), sl = r / K, k = r % K;
    const double v = __ldcg(loc + sl * 8 + k);
    double* dst = xpp->tot[q] + (par + slab0 + sl) * 8 + k;
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(dst), "d"(v) : "memory");
  }
  // every lane's pushes are ordered before the flags (system scope)
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  __syncwarp();
  if (lane < R) {
    unsigned* f = xpp->flag[lane] + me;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
  // every lane acquires every rank's flag on this rank (so each lane's loads
  // below see every rank's pushes)
  const unsigned* myf = xpp->flag[me];
  int ok = 1;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < R && ok; ++q) {
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(myf + q) : "memory");
      if (v == epoch) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 2000000000ull) {   // 2 s
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
  }
  if (!__all_sync(0xffffffffu, ok)) return false;
  const double* mine = xpp->tot[me] + par * 8;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = 0.0;
    for (int sl = 0; sl < nall; ++sl) {
      double v;
      asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(mine + sl * 8 + k) : "memory");
      a += v;   // global slab order: identical on every rank
    }
    t[k] = a;
  }
  return true;
}

template <int K>
__device__ __forceinline__ void block_reduce_finalize(double (&v)[K], const RedArgs& ra,
                                                      const CgsPre* pre = nullptr) {
  __shared__ double sm[32][K > 0 ? K : 1];
  __shared__ int am_last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  const int gbid = blockIdx.x + blockIdx.y * gridDim.x;
  const int ms_slab = ra.nbs > 0 ? gbid / ra.nbs : ra.slab;
  const int bid = ra.nbs > 0 ? gbid % ra.nbs : gbid;
  const int nb = ra.nbs > 0 ? ra.nbs : gridDim.x * gridDim.y;
  double* const part = ra.nbs > 0 ? ra.part + (size_t)ms_slab * ra.nbs * 8 : ra.part;
  unsigned int* const ticket = ra.nbs > 0 ? ra.ticket + ms_slab : ra.ticket;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
  if (pre) CHB_TP(5);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sm[wid][k] = v[k];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = lane < nw ? sm[lane][k] : 0.0;
      t = warp_sum(t);
      if (lane == 0) part[(size_t)bid * 8 + k] = t;
    }
    if (lane == 0) {
      // acq_rel ticket: releases this CTA's partials; the last arrival
      // acquires everyone's (its threads' loads follow via the CTA barrier).
      // Replaces __threadfence() (MEMBAR.SC.GPU + L1 invalidate) on both sides.
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(ticket) : "memory");
      am_last = (prev == (unsigned)(nb - 1));
    }
  }
  __syncthreads();
  if (pre) CHB_TP(6);
  if (!am_last) return;
  CgsSlot slot;
  if (pre && wid == 0) slot = cgs_slot_load(*pre, ra.fc, lane);  // in flight with the partials
  // the last CTA sums the partials with all its warps (fixed partition and
  // order: deterministic), then one thread finalizes
  {
    // batches of 8 partials per thread, all loads in flight before the adds
    // (a load-add chain costs one L2 round trip per partial: ~4 us at 740
    // CTAs); fixed partition and order, so still deterministic
    constexpr int U = 8;
    const int nthr = nw * 32;
    double t[K > 0 ? K : 1];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = 0.0;
    for (int b0 = tid; b0 < nb; b0 += nthr * U) {
      double x[U][K > 0 ? K : 1];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int b = b0 + u * nthr;
#pragma unroll
        for (int k = 0; k < K; ++k) x[u][k] = b < nb ? __ldcg(part + (size_t)b * 8 + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] += x[u][k];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double w = warp_sum(t[k]);
      if (lane == 0) sm[wid][k] = w;
    }
  }
  __syncthreads();
  if (pre) CHB_TP(7);
  if (wid != 0) return;
  double res[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sm[w][k];
    res[k] = t;
  }
  if (lane == 0) *ticket = 0u;
  if (ra.inline_fin) {
    if (pre && ra.fin == FIN_CGS)
      finalize_cgs_pre(res, *pre, slot, ra.sc, ra.fc, lane);
    else
      finalize_warp(ra.fin, res, ra.sc, ra.fc);
  } else if (ra.nbs > 0) {
    // multi-slab launch: store this slab's total; the last slab combines
    unsigned prev = 0;
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) ra.tot[ms_slab * 8 + k] = res[k];
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(ra.ticket2) : "memory");
    }
    prev = __shfl_sync(FULL, prev, 0);
    if (prev != (unsigned)(ra.nslab - 1)) return;
    if (lane == 0) *ra.ticket2 = 0u;
    double t[8];
    if (ra.xp) {
      // across ranks (and the slabs of this one): peer-memory combine
      if (!xrank_combine<K>(ra.xp, ra.epoch, ra.tot, ra.nslab, t)) {
        if (lane == 0) kfail(ra.sc, KS_PEER_TIMEOUT, (double)ra.epoch);
        return;
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double a = 0.0;
        for (int s = 0; s < ra.nslab; ++s) a += __ldcg(ra.tot + s * 8 + k);   // slab order
        t[k] = a;
      }
    }
    finalize_warp(ra.fin, t, ra.sc, ra.fc);
  } else if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) ra.tot[ra.slab * 8 + k] = res[k];
  }
}

// Per-slab arguments of one CG sweep launch over all local slabs (virtual
// slabs of one process): the sweep of slab s stores its first / last two rows
// of z' (and s) also into the ghost rows of slab s-1 / s+1 -- the halo
// exchange happens inside the sweep, no copies, no extra launches.
constexpr int MS_MAX = 8;
struct MsArgs {
  int S;     // slabs in the launch (0 or 1: single-slab launch)
  int nbs;   // blocks per slab
  int sysfence;  // the edge rows go to another GPU (peer pointers): fence at system scope
  int pad;
  // neighbour arrays of slab s pre-offset so that [off(g[s], gq, c)] addresses
  // global row gq there (slab s-1 / s+1 of this process, or the neighbouring
  // rank's boundary slab through peer memory); nullptr at the domain walls
  double* zlo[MS_MAX];
  double* zhi[MS_MAX];
  double* slo[MS_MAX];
  double* shi[MS_MAX];
  Geom g[MS_MAX];
  const double* zi[MS_MAX];
  double* zo[MS_MAX];
  const double* si[MS_MAX];
  double* so[MS_MAX];
  const double* w[MS_MAX];
  const double* a[MS_MAX];
};

// Cross-slab finalize: sums slab totals in slab order, then finalizes.
__global__ void k_finalize_slabs(const double* tot, int nslabs, int K, RedArgs ra);

}  // namespace chb
