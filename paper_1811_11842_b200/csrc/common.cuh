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
constexpr int CGM = 32;  // max block length
constexpr int CGT = 80;  // table stride (>= 2 CGM + 3)
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

// The same update by the 32 lanes of one warp, lane k owning slot k (CGM ==
// 32): two dependent L2 round trips instead of ~2 j serial ones on the
// per-iteration critical path (the last CTA's finalize).
static_assert(CGM == 32, "one lane per deferred z slot");
__device__ inline void cgs_coef_update_warp(double* tab, int m, int i, double alpha, double beta,
                                            int lane) {
  if (!tab || m <= 0) return;
  double* T = tab + ((i / m) & 1) * CGT;
  const int j = i % m, k = lane;
  double pz = 0.0, cz = 0.0, cpp = 1.0, cxp = 0.0;
  if (j != 0) {
    pz = T[CG_PZ + k];
    cz = T[CG_CZ + k];
    cpp = T[CG_CPP];
    cxp = T[CG_CXP];
  }
  if (k < j) pz *= beta;
  if (k == j) pz = 1.0;
  if (k <= j) cz += alpha * pz;
  T[CG_PZ + k] = pz;
  T[CG_CZ + k] = cz;
  if (k == 0) {
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
      if (bad(t[0])) { s->status = 1; s->done = 1; break; }
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
      if (bad(t[1])) { s->status = 1; s->done = 1; break; }
      s->omega = t[0] / t[1];
      break;
    }
    case FIN_BI_R: {
      s->iter += 1;
      if (s->half) { s->done = 1; break; }
      s->rr = t[0];
      if (t[0] <= s->tol2) { s->done = 1; break; }
      if (s->iter >= s->maxit) { s->status = 2; s->done = 1; break; }
      if (t[1] == 0.0 || !(t[1] == t[1]) || s->omega == 0.0) { s->status = 1; s->done = 1; break; }
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
      if (bad(t[0])) { s->status = 1; s->done = 1; break; }
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
      if (s->iter >= s->maxit) { s->status = 2; s->done = 1; break; }
      if (bad(t[0]) || bad(s->rho) || bad(s->alpha)) { s->status = 1; s->done = 1; break; }
      const double beta = t[0] / s->rho;
      const double den = t[2] - beta * t[0] / s->alpha;
      if (bad(den)) { s->status = 1; s->done = 1; break; }
      // three-term z recurrence (Concus-Golub-O'Leary form, kernels_cgs.cu):
      // gamma' = mu'/nu', omega' = 1 / (1 - (gamma'/gamma) (mu'/mu) / omega)
      const double gnew = t[0] / t[2];
      const double om = 1.0 / (1.0 - (gnew / s->aux[4]) * (t[0] / s->rho) / s->aux[5]);
      if (bad(gnew) || !(fabs(om) < 1e300)) { s->status = 1; s->done = 1; break; }
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

// Reduction plumbing: every block writes K partial sums; the last block to
// finish (atomic ticket) sums the partials in fixed block order (deterministic)
// and either finalizes inline (single slab, single rank) or stores the slab
// total for a later cross-slab finalize.
struct RedArgs {
  double* part;          // [nblocks * 8]
  unsigned int* ticket;  // zeroed; reset by the last block
  double* tot;           // [nslabs_total * 8] slab totals (when !inline_fin)
  KScal* sc;
  FinCtx fc;
  int fin;
  int inline_fin;
  int slab;              // index of this slab in tot
  int pad;
};

template <int K>
__device__ __forceinline__ void block_reduce_finalize(double (&v)[K], const RedArgs& ra) {
  __shared__ double sm[32][K > 0 ? K : 1];
  __shared__ int am_last;
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  const int nw = (blockDim.x * blockDim.y + 31) >> 5;
  const int bid = blockIdx.x + blockIdx.y * gridDim.x;
  const int nb = gridDim.x * gridDim.y;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = warp_sum(v[k]);
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
      if (lane == 0) ra.part[(size_t)bid * 8 + k] = t;
    }
    if (lane == 0) {
      __threadfence();
      unsigned prev = atomicAdd(ra.ticket, 1u);
      am_last = (prev == (unsigned)(nb - 1));
    }
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // the last CTA sums the partials with all its warps (fixed partition and
  // order: deterministic), then one thread finalizes
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int b = wid * 32 + lane; b < nb; b += nw * 32) t += __ldcg(ra.part + (size_t)b * 8 + k);
    t = warp_sum(t);
    if (lane == 0) sm[wid][k] = t;
  }
  __syncthreads();
  if (wid != 0) return;
  double res[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sm[w][k];
    res[k] = t;
  }
  if (lane == 0) *ra.ticket = 0u;
  if (ra.inline_fin) {
    finalize_warp(ra.fin, res, ra.sc, ra.fc);
  } else if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) ra.tot[ra.slab * 8 + k] = res[k];
  }
}

// Cross-slab finalize: sums slab totals in slab order, then finalizes.
__global__ void k_finalize_slabs(const double* tot, int nslabs, int K, RedArgs ra);

}  // namespace chb
