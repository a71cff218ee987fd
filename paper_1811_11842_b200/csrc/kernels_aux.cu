// kernels_aux.cu -- once-per-solve kernels of the 5-point symmetric operator
// family (pressure Poisson, Eq. 20; intermediate velocity, Eq. 19; nutrient,
// Eq. 16) around the fused single-reduction CG sweep of kernels_cgs.cu:
//
//   y = a x + s * sum_faces k_f (x - x_nb) / h_f^2         (op5.cuh)
//
// Operator instances (OpKind):
//   POISSON_CONST  a = 0, s = 1, k = 1                      (rho_n == rho_s)
//   POISSON_VAR    a = 0, s = 1, k = 1/rho(face mean phi^{n+1})
//   NUTRIENT       a = a_c[], s = 1/2, k = D_s * face mean(phi_s^{1/2})
//   MOM_U          a = rho/dt[], s = theta_visc, k = face mean(eta), odd-reflection walls
//   MOM_V          a = rho/dt[], s = theta_visc, k = face mean(eta), Dirichlet wall faces,
//                  row 0 = identity          (eta = 1/Re_a at the unknown's points, R6)
//
// CG initialisation (r = b - A x, z = D^-1 r, three reductions), the plain
// operator apply of ch_apply_operator, the CG finish / null-space mean, and
// the cross-slab finalize.  Each thread owns one column and marches down a
// strip of rows keeping the three-row window in registers; x-neighbours come
// from warp shuffles (edge lanes and the periodic seam reload through L1).
#include "common.cuh"
#include "launch.h"
#include "op5.cuh"
#include "tma.cuh"

namespace chb {

// ---------------------------------------------------------------------------
// Column-marching helpers.  All threads of a block run the same row loop.
struct Col {
  int c, cc, cw, ce, lane;
  bool act, needW, needE;
  __device__ __forceinline__ Col(const Geom& g) {
    lane = threadIdx.x & 31;
    c = blockIdx.x * blockDim.x + threadIdx.x;
    act = c < g.nx;
    cc = act ? c : g.nx - 1;
    cw = wrapc(cc - 1, g.nx);
    ce = wrapc(cc + 1, g.nx);
    needW = (lane == 0) || (c == 0);
    needE = (lane == 31) || (c + 1 >= g.nx);
  }
};

#define CHB_SHFL_W(v) __shfl_up_sync(FULL, (v), 1)
#define CHB_SHFL_E(v) __shfl_down_sync(FULL, (v), 1)

// ------------------------------------------------------------------ CG init
// r = (b - shift) - A x;  z = r / d;  reduce ||b - shift||^2, (r, z), (r, r)
template <int BC, int AM, int KM>
__global__ void __launch_bounds__(128) k_cg5_init(Geom g, Op5T op, const double* __restrict__ x,
                                                  const double* __restrict__ b, int use_shift,
                                                  double* __restrict__ z, int strip, RedArgs ra) {
  const double shift = use_shift ? ra.sc->mean : 0.0;
  Col col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  int gj = g.j0 + jl0;
  double xm = ldf<BC>(x, g, gj - 1, col.cc), x0 = ldf<BC>(x, g, gj, col.cc);
  double wm = 0.0, w0 = 0.0;
  if (KM) {
    wm = ldf<BC_MIRROR>(op.w, g, gj - 1, col.cc);
    w0 = ldf<BC_MIRROR>(op.w, g, gj, col.cc);
  }
  for (int jl = jl0; jl < jl1; ++jl, ++gj) {
    const double xp = ldf<BC>(x, g, gj + 1, col.cc);
    double xw = CHB_SHFL_W(x0), xe = CHB_SHFL_E(x0);
    if (col.needW) xw = ldf<BC>(x, g, gj, col.cw);
    if (col.needE) xe = ldf<BC>(x, g, gj, col.ce);
    double wp = 0.0, ww = 0.0, we = 0.0;
    if (KM) {
      wp = ldf<BC_MIRROR>(op.w, g, gj + 1, col.cc);
      ww = CHB_SHFL_W(w0);
      we = CHB_SHFL_E(w0);
      if (col.needW) ww = ldf<BC_MIRROR>(op.w, g, gj, col.cw);
      if (col.needE) we = ldf<BC_MIRROR>(op.w, g, gj, col.ce);
    }
    const double ac = a_at<AM>(op, off(g, gj, col.cc));
    double y, d;
    eval5T<BC, AM, KM>(op, g, gj, ac, w0, ww, we, wm, wp, x0, xw, xe, xm, xp, y, d);
    if (col.act) {
      const size_t o = off(g, gj, col.c);
      const double bc = b[o] - ((BC == BC_VFACE && gj == 0) ? 0.0 : shift);
      const double r = bc - y;
      const double zz = r / d;
      z[o] = zz;
      s0 += bc * bc;
      s1 += r * zz;
      s2 += r * r;
    }
    xm = x0;
    x0 = xp;
    wm = w0;
    w0 = wp;
  }
  double v[3] = {s0, s1, s2};
  block_reduce_finalize<3>(v, ra);
}

// ------------------------------------------------- ring-staged plain apply
// y = A x for the isolated apply (ch_apply_operator; BASELINE configs[4]'s
// matvec sweeps).  Row marching like the CG sweep: one CTA of 128 threads per
// (<= 256-column chunk x row strip), one resident wave; x and (KM) w rows of
// the chunk plus a 2-column halo each side are streamed into an 8-deep
// shared-memory ring by 1-D bulk async copies (lane 0 of warp 0: x, of warp 1:
// w), each thread computes two adjacent columns with 16-B loads / stores.  Per
// cell: read x (+ w) (+ a), write y -- 16 / 24 / 32 B.
namespace {
constexpr int AP_T = 128;
constexpr int AP_CW = 2 * AP_T;       // columns per chunk (max)
constexpr int AP_SEG = AP_CW + 4;     // staged columns c0 - 2 .. c0 + wc + 1
constexpr int AP_NST = 8;

template <int BC>
__device__ __forceinline__ int ap_fold(const Geom& g, int gj) {
  if (BC == BC_VFACE) return gj < 0 ? 1 : (gj >= g.ny ? g.ny - 1 : gj);  // value zeroed below
  if (gj < 0) return -1 - gj;
  if (gj >= g.ny) return 2 * g.ny - 1 - gj;
  return gj;
}

template <int BC>
__device__ __forceinline__ double ap_scale(const Geom& g, int gj) {
  if (BC == BC_VFACE) return (gj <= 0 || gj >= g.ny) ? 0.0 : 1.0;
  if (BC == BC_ODD) return (gj < 0 || gj >= g.ny) ? -1.0 : 1.0;
  return 1.0;
}

__device__ __forceinline__ void ap_issue(const Geom& g, const double* base, int row, uint32_t dst,
                                         uint32_t bar, int c0, int wc) {
  const double* r = base + (size_t)(row - g.j0 + GH) * g.pitch;
  const int lo = c0 - 2, hi = c0 + wc + 2;
  const int mlo = lo < 0 ? 0 : lo, mhi = hi > g.nx ? g.nx : hi;
  uint32_t d = dst;
  if (lo < 0) {
    bulk_g2s_s(d, r + (lo + g.nx), (uint32_t)(-lo) * 8u, bar);
    d += (uint32_t)(-lo) * 8u;
  }
  bulk_g2s_s(d, r + mlo, (uint32_t)(mhi - mlo) * 8u, bar);
  d += (uint32_t)(mhi - mlo) * 8u;
  if (hi > g.nx) bulk_g2s_s(d, r, (uint32_t)(hi - g.nx) * 8u, bar);
}
}  // namespace

template <int BC, int AM, int KM>
__global__ void __launch_bounds__(AP_T) k_op5_rm(Geom g, Op5T op, const double* __restrict__ x,
                                               double* __restrict__ yout, int ncb, int cw) {
  constexpr int NA = KM ? 2 : 1;       // staged arrays
  constexpr int STAGE = NA * AP_SEG;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[AP_NST];
  const uint32_t ring_s = s_u32(smem), bars_s = s_u32(bars);
  // block -> (chunk, strip)
  const int nb = gridDim.x, b = blockIdx.x;
  const int q = nb / ncb, rem = nb % ncb;
  int chunk, k, sc;
  if (b < rem * (q + 1)) {
    chunk = b / (q + 1), k = b % (q + 1), sc = q + 1;
  } else {
    const int bb = b - rem * (q + 1);
    chunk = rem + bb / q, k = bb % q, sc = q;
  }
  const int jl0 = (int)(((long long)k * g.nyl) / sc), jl1 = (int)(((long long)(k + 1) * g.nyl) / sc);
  const int c0 = chunk * cw, wc = min(cw, g.nx - c0);
  const int n = jl1 - jl0, nq = n + 2;   // ring rows j0+jl0-1 .. j0+jl1
  const int rbase = g.j0 + jl0 - 1;
  const int t = threadIdx.x;
  const bool own = 2 * t < wc;
  const int ci = 2 * t + 2;
  if (t == 0) {
    for (int i = 0; i < AP_NST; ++i) mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int slot, int qq) {   // ring row qq into slot (thread 0 only)
    const uint32_t bar = bars_s + 8u * (uint32_t)slot;
    mbar_expect_tx_s(bar, (uint32_t)NA * (uint32_t)(wc + 4) * 8u);
    const int gq = rbase + qq;
    const uint32_t dst = ring_s + 8u * (uint32_t)(slot * STAGE);
    ap_issue(g, x, ap_fold<BC>(g, gq), dst, bar, c0, wc);
    if (KM) ap_issue(g, op.w, ap_fold<BC_MIRROR>(g, gq), dst + 8u * AP_SEG, bar, c0, wc);
  };
  if (t == 0)
    for (int qq = 0; qq < AP_NST && qq < nq; ++qq) issue(qq, qq);
  auto slot = [&](int qq) { return smem + (qq % AP_NST) * STAGE; };
  auto wait = [&](int qq) {
    mbar_wait_s(bars_s + 8u * (uint32_t)(qq % AP_NST), (uint32_t)((qq / AP_NST) & 1));
  };
  wait(0);
  wait(1);
  for (int r = 1; r <= n; ++r) {
    wait(r + 1);
    const int gj = rbase + r;
    if (own) {
      const double *sS = slot(r - 1), *sC = slot(r), *sN = slot(r + 1);
      const double scS = ap_scale<BC>(g, gj - 1), scN = ap_scale<BC>(g, gj + 1);
      const size_t o = off(g, gj, c0 + 2 * t);
      double y[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = ci + j;
        const double xc = sC[c], xw = sC[c - 1], xe = sC[c + 1];
        const double xs = scS * sS[c], xn = scN * sN[c];
        double wc_ = 0, ww = 0, we = 0, wS = 0, wN = 0;
        if (KM) {
          wc_ = sC[AP_SEG + c], ww = sC[AP_SEG + c - 1], we = sC[AP_SEG + c + 1];
          wS = sS[AP_SEG + c], wN = sN[AP_SEG + c];
        }
        const double ac = a_at<AM>(op, o + j);
        const Cf5 cf = coef5<BC, AM, KM>(op, g, gj, ac, wc_, ww, we, wS, wN);
        y[j] = apply5<BC>(cf, op, g, gj, xc, xw, xe, xs, xn);   // v wall row: identity
      }
      *reinterpret_cast<double2*>(yout + o) = make_double2(y[0], y[1]);
    }
    __syncthreads();   // ring row r - 1 consumed by every thread: refill its slot
    if (t == 0 && r - 1 + AP_NST < nq) {
      fence_proxy_async();
      issue((r - 1) % AP_NST, r - 1 + AP_NST);
    }
  }
}

// ---------------------------------------------------------------- CG finish
// x += alpha p (last iteration's update, deferred by the A kernel), or x = 0
// when b = 0; optional reduction of sum(x) for the null-space projection.
// mode 0: add the last alpha p; 1 (single-reduction CG, x over pairs of
// sweeps): only after an odd iteration count; 2 (deferred p/x blocks, already
// applied): no update, only the b = 0 case and the null-space sum.
__global__ void __launch_bounds__(256) k_cg5_finish(Geom g, double* __restrict__ x,
                                                    const double* __restrict__ p, int nullspace,
                                                    int odd_only, RedArgs ra) {
  const KScal* sc = ra.sc;
  const int zero = sc->zero;
  const int upd = (sc->iter >= 1) && !zero && sc->status == 0 && odd_only != 2 &&
                  (!odd_only || (sc->iter & 1));
  const double alpha = sc->alpha;
  double acc = 0.0;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  for (int jl = blockIdx.y; jl < g.nyl; jl += gridDim.y) {
    if (c < g.nx) {
      const size_t o = off(g, g.j0 + jl, c);
      double v = zero ? 0.0 : x[o];
      if (upd) v += alpha * p[o];
      x[o] = v;
      acc += v;
    }
  }
  if (nullspace) {
    double v[1] = {acc};
    block_reduce_finalize<1>(v, ra);
  }
}

__global__ void __launch_bounds__(256) k_sub_mean(Geom g, double* __restrict__ x, const KScal* sc) {
  const double m = sc->mean;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  for (int jl = blockIdx.y; jl < g.nyl; jl += gridDim.y)
    if (c < g.nx) x[off(g, g.j0 + jl, c)] -= m;
}

__global__ void k_finalize_slabs(const double* tot, int nslabs, int K, RedArgs ra) {
  // one warp (launch_finalize_slabs): lane 0 finalizes, the lanes share the
  // coefficient-table update
  // iteration-phase finalizers are no-ops once the solve is done (their slab
  // kernels returned early and the totals are stale); BiCGStab's omega phase
  // is skipped after a half-step convergence
  const int iter_phase = ra.fin == FIN_CG_A || ra.fin == FIN_CG_B || ra.fin == FIN_CGS ||
                         ra.fin == FIN_CGS_D0 || ra.fin == FIN_BI_ALPHA ||
                         ra.fin == FIN_BI_S || ra.fin == FIN_BI_OMEGA || ra.fin == FIN_BI_R;
  if (iter_phase && ra.sc->done) return;
  if (ra.fin == FIN_BI_OMEGA && ra.sc->half) return;
  double t[8];
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int i = 0; i < nslabs; ++i) s += tot[i * 8 + k];
    t[k] = s;
  }
  finalize_warp(ra.fin, t, ra.sc, ra.fc);
}

// ============================================================== launchers
static Op5T make_op(const OpDesc& d) {
  Op5T o;
  o.a = d.a;
  o.w = d.w;
  o.s = d.s;
  o.kscale = d.kscale;
  o.rho_n = d.rho_n;
  o.rho_s = d.rho_s;
  o.ascal = d.ascal;
  return o;
}

static dim3 grid5(const Geom& g, int strip) {
  return dim3((g.nx + 127) / 128, (g.nyl + strip - 1) / strip);
}

#define CHB_DISPATCH(KIND, CALL)                                        \
  switch (KIND) {                                                       \
    case OPK_POISSON_CONST: { constexpr int BC = BC_MIRROR, AM = 0, KM = 0; CALL; } break; \
    case OPK_POISSON_VAR:   { constexpr int BC = BC_MIRROR, AM = 0, KM = 2; CALL; } break; \
    case OPK_NUTRIENT:      { constexpr int BC = BC_MIRROR, AM = 1, KM = 1; CALL; } break; \
    case OPK_MOM_U:         { constexpr int BC = BC_ODD,    AM = 1, KM = 1; CALL; } break; \
    case OPK_MOM_V:         { constexpr int BC = BC_VFACE,  AM = 1, KM = 1; CALL; } break; \
    case OPK_MOM_U_C:       { constexpr int BC = BC_ODD,    AM = 2, KM = 1; CALL; } break; \
    case OPK_MOM_V_C:       { constexpr int BC = BC_VFACE,  AM = 2, KM = 1; CALL; } break; \
    default: break;                                                     \
  }

void launch_cg5_init(const OpDesc& d, const Geom& g, const double* x, const double* b,
                     int use_shift, double* z, const RedArgs& ra, cudaStream_t st) {
  const Op5T op = make_op(d);
  const int strip = d.strip;
  CHB_DISPATCH(d.kind, (k_cg5_init<BC, AM, KM><<<grid5(g, strip), 128, 0, st>>>(
                           g, op, x, b, use_shift, z, strip, ra)));
}

template <int BC, int AM, int KM>
static void launch_op5_rm(const OpDesc& d, const Geom& g, const double* x, double* y,
                          cudaStream_t st) {
  auto kern = k_op5_rm<BC, AM, KM>;
  constexpr size_t smem = (size_t)AP_NST * (KM ? 2 : 1) * AP_SEG * sizeof(double);
  static int per_sm = -1, nsm = 0;
  if (per_sm < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, AP_T, smem);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ncb = (g.nx + AP_CW - 1) / AP_CW;
  int cw = (g.nx + ncb - 1) / ncb;
  cw += cw & 1;
  long nb = (long)nsm * per_sm;
  if (d.strip2 > 0) nb = (long)ncb * ((g.nyl + d.strip2 - 1) / d.strip2);
  if (nb < ncb) nb = ncb;
  if (nb > (long)ncb * g.nyl) nb = (long)ncb * g.nyl;
  kern<<<(unsigned)nb, AP_T, smem, st>>>(g, make_op(d), x, y, ncb, cw);
}

void launch_op5_apply(const OpDesc& d, const Geom& g, const double* x, double* y,
                      cudaStream_t st) {
  CHB_DISPATCH(d.kind, (launch_op5_rm<BC, AM, KM>(d, g, x, y, st)));
}

static dim3 grid_pw(const Geom& g) {  // ~8 CTAs per SM (bounded reduction partials)
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int gx = (g.nx + 255) / 256;
  int gy = (nsm * 8 + gx - 1) / gx;
  if (gy > g.nyl) gy = g.nyl;
  if (gy < 1) gy = 1;
  return dim3(gx, gy);
}

void launch_cg5_finish(const Geom& g, double* x, const double* p, int nullspace, int odd_only,
                       const RedArgs& ra, cudaStream_t st) {
  k_cg5_finish<<<grid_pw(g), 256, 0, st>>>(g, x, p, nullspace, odd_only, ra);
}

void launch_sub_mean(const Geom& g, double* x, const KScal* sc, cudaStream_t st) {
  k_sub_mean<<<grid_pw(g), 256, 0, st>>>(g, x, sc);
}

void launch_finalize_slabs(const double* tot, int nslabs, int K, const RedArgs& ra,
                           cudaStream_t st) {
  k_finalize_slabs<<<1, 32, 0, st>>>(tot, nslabs, K, ra);
}

}  // namespace chb
