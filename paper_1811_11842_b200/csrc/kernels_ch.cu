// kernels_ch.cu -- the 13-point modified Cahn-Hilliard operator
//   y = x^/dt + th Gamma1 L_{M*} Delta_h x^ + ta Adv(x^; v^n),   x^ = D^{-1} x
// (right Jacobi; Eq. 16 4th line with §4's Crank-Nicolson, th = ta
// = 1/2, R5, R12, R23) and the BiCGStab / GMRES vector updates
// that run around it (PAPER.md:233-244 names GMRES + Jacobi; BiCGStab is the
// north_star's GPU choice, R14).  Even nx only (two columns per thread).
#include <stdlib.h>

#include "common.cuh"
#include "launch.h"
#include "tma.cuh"

namespace chb {

// --------------------------------------------------------------------------
// Row-marching apply: one CTA per (<= 256-column chunk x row strip), x, D^-1
// and phi* rows streamed into a 6-deep (CHB_RM_NST) shared-memory ring by 1-D bulk async
// copies (lane 0 of warps 0-2, one array each), two columns per thread,
// x^ = D^-1 x and w = Delta_h x^ kept in three-row register windows (w
// recomputed on the two neighbour columns each side instead of exchanged),
// y = x^/dt + th G1 L_M w + ta Adv(x^) one row behind.  The face velocities
// of the advection part (u on the cell's two x-faces, v on its two y-faces)
// come straight from global memory at the thread's own columns.  Per cell:
// read x, D^-1, phi* (+ u, v; + dot operands), write y.
#ifndef CHB_RM_NST
#define CHB_RM_NST 6    // ring depth (rows in flight per CTA): 6 x 18.7 KB x 5 CTAs fit one SM
#endif
namespace {
constexpr int RM_T = 128;             // threads (4 warps)
constexpr int RM_CW = 2 * RM_T;       // max columns per chunk
constexpr int RM_SEG = RM_CW + 4;     // staged columns c0 - 2 .. c0 + wc + 1
// the isolated apply (NDOT = 0) and the in-solver applies with fused dots
// (NDOT > 0: more live registers) take their own CTAs-per-SM / ring depth
#ifndef CHB_RM_NST_DOT
#define CHB_RM_NST_DOT 8
#endif
constexpr int rm_nst(int ndot) { return ndot == 0 ? CHB_RM_NST : CHB_RM_NST_DOT; }
constexpr int RM_STAGE = 3 * RM_SEG;  // x | dinv | phi*

__device__ __forceinline__ int rm_fold(const Geom& g, int gj) {
  if (gj < 0) return -1 - gj;
  if (gj >= g.ny) return 2 * g.ny - 1 - gj;
  return gj;
}

__device__ __forceinline__ void rm_issue(const Geom& g, const double* base, uint32_t ring_s,
                                         uint32_t bars_s, int slot, int gj, int c0, int wc,
                                         int stream, bool use) {
  const uint32_t bar = bars_s + 8u * (uint32_t)slot;
  mbar_expect_tx_s(bar, use ? (uint32_t)(wc + 4) * 8u : 0u);
  if (!use) return;
  const double* row = base + (size_t)(rm_fold(g, gj) - g.j0 + GH) * g.pitch;
  uint32_t d = ring_s + 8u * (uint32_t)(slot * RM_STAGE + stream * RM_SEG);
  const int lo = c0 - 2, hi = c0 + wc + 2;
  const int mlo = lo < 0 ? 0 : lo, mhi = hi > g.nx ? g.nx : hi;
  if (lo < 0) {
    bulk_g2s_s(d, row + (lo + g.nx), (uint32_t)(-lo) * 8u, bar);
    d += (uint32_t)(-lo) * 8u;
  }
  bulk_g2s_s(d, row + mlo, (uint32_t)(mhi - mlo) * 8u, bar);
  d += (uint32_t)(mhi - mlo) * 8u;
  if (hi > g.nx) bulk_g2s_s(d, row, (uint32_t)(hi - g.nx) * 8u, bar);
}

__device__ __forceinline__ void rm_tile(int b, int nb, int ncb, int nyl, int& chunk, int& jl0,
                                        int& jl1) {
  const int q = nb / ncb, rem = nb % ncb;
  int k, sc;
  if (b < rem * (q + 1)) {
    chunk = b / (q + 1);
    k = b % (q + 1);
    sc = q + 1;
  } else {
    const int bb = b - rem * (q + 1);
    chunk = rem + bb / q;
    k = bb % q;
    sc = q;
  }
  jl0 = (int)(((long long)k * nyl) / sc);
  jl1 = (int)(((long long)(k + 1) * nyl) / sc);
}
}  // namespace

#ifndef CHB_MINB_CH
#define CHB_MINB_CH 5   // resident CTAs per SM requested from ptxas (<= 102 registers,
                        // 8-48 B of spills): measured on the isolated apply 4 vs the
                        // unconstrained 3 (149 registers) +16 % (4096^2) / +25 % (16384^2);
                        // 5 (ring depth 6) vs 4 (depth 8) +4 % / +4 %; 6 (85 registers) -21 %
#endif
#ifndef CHB_MINB_CH_DOT
#define CHB_MINB_CH_DOT 4   // applies with fused dots: 5 CTAs/SM measured 15 % SLOWER in the
                            // BiCGStab solve (217.7 -> 251.3 us at 4096^2): 4 stays
#endif
constexpr int rm_minb(int ndot) { return ndot == 0 ? CHB_MINB_CH : CHB_MINB_CH_DOT; }
template <int NDOT, int PRE>
__global__ void __launch_bounds__(RM_T, rm_minb(NDOT)) k_ch_rm(Geom g, ChCoef cc, const double* __restrict__ x,
                                                double* __restrict__ y,
                                                const double* __restrict__ d1,
                                                const double* __restrict__ d2, int skip_done,
                                                int skip_half, int ncb, int cw, RedArgs ra) {
  if (skip_done && ra.sc->done) return;
  if (skip_half && ra.sc->half) return;
  constexpr int NST = NDOT == 0 ? CHB_RM_NST : CHB_RM_NST_DOT;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[NST];
  const uint32_t ring_s = s_u32(smem), bars_s = s_u32(bars);
  int chunk, jl0, jl1;
  rm_tile(blockIdx.x, gridDim.x, ncb, g.nyl, chunk, jl0, jl1);
  const int c0 = chunk * cw, wc = min(cw, g.nx - c0);
  const int n = jl1 - jl0, nq = n + 4;  // ring rows j0+jl0-2 .. j0+jl1+1
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool own = 2 * t < wc;
  const int ci = 2 * t + 2;  // staged index of the thread's first column
  const int rbase = g.j0 + jl0 - 2;
  const double* mysrc = warp == 0 ? x : (warp == 1 ? cc.dinv : cc.phis);
  const bool myuse = warp == 0 || warp == 2 || (warp == 1 && PRE);
  if (t == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(bars + i, RM_T / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (lane == 0)
    for (int q = 0; q < NST && q < nq; ++q)
      rm_issue(g, mysrc, ring_s, bars_s, q, rbase + q, c0, wc, warp, myuse);
  auto slot = [&](int q) { return smem + (q % NST) * RM_STAGE; };
  auto xh = [&](const double* st, int idx) -> double {  // x^ = D^-1 x at staged index idx
    const double v = st[idx];
    return PRE ? v * st[RM_SEG + idx] : v;
  };
  auto wait_row = [&](int q) {
    mbar_wait_s(bars_s + 8u * (uint32_t)(q % NST), (uint32_t)((q / NST) & 1));
  };
  // x^ rows (older -> newer) at columns c-1 .. c+2 of the thread's pair; w = Delta_h x^
  // at the pair's own columns in registers (wm, wc_, wp: rows k-1, k, k+1, indices
  // 1..2), the neighbours' from a 3-row shared buffer (each w computed once; the
  // chunk's halo columns by the first / last owning thread)
  __shared__ double wrow[3][RM_SEG];
  double xa[4], xb[4], wm[4], wc_[4], wp[4];
  const bool edgeL = own && t == 0, edgeR = own && 2 * t + 2 >= wc;
  wait_row(0);
  wait_row(1);
  for (int j = 0; j < 4; ++j) {
    xa[j] = xh(slot(0), ci - 1 + j);
    xb[j] = xh(slot(1), ci - 1 + j);
    wm[j] = wc_[j] = 0.0;
  }
  // face mobility Lambda max(0, (a + b)/2) = hL max(0, a + b), hL = Lambda/2 (exact: the
  // factor 1/2 is a power of two); x/dt as x * (1/dt)
  const double hL = 0.5 * cc.Lambda, idt = 1.0 / cc.dt;
  const bool adv = cc.u != nullptr;
  // face velocities of the advection part, prefetched two output rows ahead in
  // registers: u on the pair's three x-faces of row gj, v on its y-faces gj, gj + 1
  // (v = 0 on the wall faces)
  const int lastrow = rbase + n + 1;
  struct UF {
    double2 w;
    double e;
  };
  auto ldu = [&](int gj) -> UF {
    UF r{make_double2(0.0, 0.0), 0.0};
    if (!adv || !own || gj > lastrow) return r;
    const size_t o = off(g, gj, c0 + 2 * t);
    r.w = __ldg(reinterpret_cast<const double2*>(cc.u + o));
    const int ce = c0 + 2 * t + 2;
    r.e = __ldg(cc.u + off(g, gj, ce >= g.nx ? ce - g.nx : ce));
    return r;
  };
  auto ldv = [&](int gj) -> double2 {
    if (!adv || !own || gj <= 0 || gj >= g.ny || gj > lastrow + 1) return make_double2(0.0, 0.0);
    return __ldg(reinterpret_cast<const double2*>(cc.v + off(g, gj, c0 + 2 * t)));
  };
  UF uq0 = ldu(rbase + 2), uq1 = ldu(rbase + 3);
  double2 vS2 = ldv(rbase + 2), vq0 = ldv(rbase + 3), vq1 = ldv(rbase + 4);
  double s0 = 0.0, s1 = 0.0;
  for (int k = 0; k <= n + 1; ++k) {
    UF unew{make_double2(0.0, 0.0), 0.0};
    double2 vnew = make_double2(0.0, 0.0);
    if (k >= 2) {   // loads for output row rbase + k + 2 (two rows ahead)
      unew = ldu(rbase + k + 2);
      vnew = ldv(rbase + k + 3);
    }
    wait_row(k + 2);
    // w on ring row k + 1 (x^ rows k, k+1, k+2) at columns c-1 .. c+2
    const double* sc1 = slot(k + 1);
    const double* sc2 = slot(k + 2);
    double xn[4];
    for (int j = 0; j < 4; ++j) xn[j] = xh(sc2, ci - 1 + j);
    for (int j = 1; j <= 2; ++j)
      wp[j] = (xb[j + 1] - 2.0 * xb[j] + xb[j - 1]) * g.ihx2 +
              (xn[j] - 2.0 * xb[j] + xa[j]) * g.ihy2;
    if (own) {
      double* wr = wrow[(k + 1) % 3];
      wr[ci] = wp[1];
      wr[ci + 1] = wp[2];
      if (edgeL) {
        const double xl = xh(sc1, ci - 2);
        wr[ci - 1] = (xb[1] - 2.0 * xb[0] + xl) * g.ihx2 + (xn[0] - 2.0 * xb[0] + xa[0]) * g.ihy2;
      }
      if (edgeR) {
        const double xr = xh(sc1, ci + 3);
        wr[ci + 2] = (xr - 2.0 * xb[3] + xb[2]) * g.ihx2 + (xn[3] - 2.0 * xb[3] + xa[3]) * g.ihy2;
      }
    }
    // y on ring row k (owned rows 2 .. n+1): w rows k-1 (wm), k (wc_), k+1 (wp)
    if (k >= 2 && own) {
      const int gj = rbase + k;
      wc_[0] = wrow[k % 3][ci - 1];   // row k's w at the neighbour columns (previous iteration)
      wc_[3] = wrow[k % 3][ci + 2];
      const double* ps0 = slot(k - 1) + 2 * RM_SEG;
      const double* ps1 = slot(k) + 2 * RM_SEG;
      const double* ps2 = slot(k + 1) + 2 * RM_SEG;
      double yv[2];
      for (int j = 0; j < 2; ++j) {
        const int cc_ = ci + j;      // staged index of this column
        const double pc = ps1[cc_];
        const double mE = hL * fmax(0.0, pc + ps1[cc_ + 1]);
        const double mW = hL * fmax(0.0, pc + ps1[cc_ - 1]);
        const double mN = (gj == g.ny - 1) ? 0.0 : hL * fmax(0.0, pc + ps2[cc_]);
        const double mS = (gj == 0) ? 0.0 : hL * fmax(0.0, pc + ps0[cc_]);
        const double w0 = wc_[j + 1];
        const double div = (mE * (wc_[j + 2] - w0) - mW * (w0 - wc_[j])) * g.ihx2 +
                           (mN * (wp[j + 1] - w0) - mS * (w0 - wm[j + 1])) * g.ihy2;
        yv[j] = xa[j + 1] * idt + cc.g1t * div;
      }
      const size_t o = off(g, gj, c0 + 2 * t);
      if (adv) {
        // ta Adv(x^) = ta [ (uE (x+xE) - uW (xW+x)) / 2hx + (vN (x+xN) - vS (xS+x)) / 2hy ]
        const double2 uw = uq0.w;
        const double ue = uq0.e;
        const double2 vn = vq0;
        const double* xs0 = slot(k - 1);
        const double xS0 = xh(xs0, ci), xS1 = xh(xs0, ci + 1);
        const double hx = 0.5 * g.ihx, hy = 0.5 * g.ihy;
        const double a0 = (uw.y * (xa[1] + xa[2]) - uw.x * (xa[0] + xa[1])) * hx +
                          (vn.x * (xa[1] + xb[1]) - vS2.x * (xS0 + xa[1])) * hy;
        const double a1 = (ue * (xa[2] + xa[3]) - uw.y * (xa[1] + xa[2])) * hx +
                          (vn.y * (xa[2] + xb[2]) - vS2.y * (xS1 + xa[2])) * hy;
        yv[0] += cc.tha * a0;
        yv[1] += cc.tha * a1;
      }
      *reinterpret_cast<double2*>(y + o) = make_double2(yv[0], yv[1]);
      if (NDOT >= 1) {
        const double2 a = *reinterpret_cast<const double2*>(d1 + o);
        s0 += yv[0] * a.x + yv[1] * a.y;
      }
      if (NDOT >= 2) {
        if (d2) {
          const double2 b = *reinterpret_cast<const double2*>(d2 + o);
          s1 += yv[0] * b.x + yv[1] * b.y;
        } else {
          s1 += yv[0] * yv[0] + yv[1] * yv[1];
        }
      }
    }
    __syncthreads();  // ring row k - 1 consumed by every warp
    if (lane == 0 && k >= 1 && k - 1 + NST < nq) {
      fence_proxy_async();
      rm_issue(g, mysrc, ring_s, bars_s, (k - 1) % NST, rbase + k - 1 + NST, c0, wc, warp,
               myuse);
    }
    for (int j = 0; j < 4; ++j) {
      xa[j] = xb[j];
      xb[j] = xn[j];
    }
    for (int j = 1; j <= 2; ++j) {
      wm[j] = wc_[j];
      wc_[j] = wp[j];
    }
    if (k >= 2) {   // the velocity FIFO advances with the output row
      uq0 = uq1;
      uq1 = unew;
      vS2 = vq0;
      vq0 = vq1;
      vq1 = vnew;
    }
  }
  if (NDOT == 1) {
    double v[1] = {s0};
    block_reduce_finalize<1>(v, ra);
  } else if (NDOT == 2) {
    double v[2] = {s0, s1};
    block_reduce_finalize<2>(v, ra);
  }
}

namespace {
template <int NDOT, int PRE>
void launch_rm(const Geom& g, const ChCoef& cc, const double* x, double* y, const double* d1,
               const double* d2, int skip_done, int skip_half, const RedArgs& ra,
               cudaStream_t st) {
  auto kern = k_ch_rm<NDOT, PRE>;
  constexpr size_t smem = (size_t)rm_nst(NDOT) * RM_STAGE * sizeof(double);
  static int per_sm = -1;
  static int nsm = 0;
  if (per_sm < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RM_T, smem);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ncb = (g.nx + RM_CW - 1) / RM_CW;
  int cw = (g.nx + ncb - 1) / ncb;
  cw += cw & 1;
  long nb = (long)nsm * per_sm;
  if (cc.strip > 0) nb = (long)ncb * ((g.nyl + cc.strip - 1) / cc.strip);  // forced strip height
  if (nb < ncb) nb = ncb;
  if (nb > (long)ncb * g.nyl) nb = (long)ncb * g.nyl;
  kern<<<(unsigned)nb, RM_T, smem, st>>>(g, cc, x, y, d1, d2, skip_done, skip_half, ncb, cw, ra);
}
}  // namespace

void launch_ch_apply(const Geom& g, const ChCoef& cc, const double* x, double* y, int ndot,
                     const double* d1, const double* d2, int skip_if_done, int skip_if_half,
                     const RedArgs& ra, cudaStream_t st) {
  if (cc.dinv) {
    if (ndot == 0) launch_rm<0, 1>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
    else if (ndot == 1) launch_rm<1, 1>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
    else launch_rm<2, 1>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
  } else {
    if (ndot == 0) launch_rm<0, 0>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
    else if (ndot == 1) launch_rm<1, 0>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
    else launch_rm<2, 0>(g, cc, x, y, d1, d2, skip_if_done, skip_if_half, ra, st);
  }
}

// ------------------------------------------------------- BiCGStab updates
// Row-parallel pointwise kernels over the slab's own cells.
#define CHB_PW_LOOP(g)                                              \
  const int c_ = blockIdx.x * blockDim.x + threadIdx.x;             \
  for (int jl = blockIdx.y; jl < (g).nyl; jl += gridDim.y)          \
    if (c_ < (g).nx)

// ~8 CTAs per SM: enough bytes in flight, and few enough partial sums that the
// last CTA's fixed-order reduction stays short
static dim3 grid_pw(const Geom& g) {
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

__global__ void __launch_bounds__(256) k_bi_init(Geom g, const double* __restrict__ y,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ r, double* __restrict__ rh,
                                                 RedArgs ra) {
  double s0 = 0.0, s1 = 0.0;
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    const double bb = b[o], rr = bb - y[o];
    r[o] = rr;
    rh[o] = rr;
    s0 += bb * bb;
    s1 += rr * rr;
  }
  double v[2] = {s0, s1};
  block_reduce_finalize<2>(v, ra);
}

__global__ void __launch_bounds__(256) k_bi_p(Geom g, const double* __restrict__ r,
                                              double* __restrict__ p, const double* __restrict__ v,
                                              int first, const KScal* sc) {
  if (sc->done) return;
  const double beta = (sc->rho / sc->rho_prev) * (sc->alpha / sc->omega);
  const double om = sc->omega;
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    p[o] = first ? r[o] : r[o] + beta * (p[o] - om * v[o]);
  }
}

__global__ void __launch_bounds__(256) k_bi_s(Geom g, const double* __restrict__ r,
                                              const double* __restrict__ v, double* __restrict__ s,
                                              RedArgs ra) {
  if (ra.sc->done) return;
  const double al = ra.sc->alpha;
  double acc = 0.0;
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    const double ss = r[o] - al * v[o];
    s[o] = ss;
    acc += ss * ss;
  }
  double vv[1] = {acc};
  block_reduce_finalize<1>(vv, ra);
}

__global__ void __launch_bounds__(256) k_bi_xr(Geom g, double* __restrict__ x,
                                               const double* __restrict__ p,
                                               const double* __restrict__ s,
                                               const double* __restrict__ t,
                                               double* __restrict__ r,
                                               const double* __restrict__ rh,
                                               const double* __restrict__ dinv, RedArgs ra) {
  if (ra.sc->done) return;
  const double al = ra.sc->alpha, om = ra.sc->omega;
  const int half = ra.sc->half;
  double a0 = 0.0, a1 = 0.0;
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    const double di = dinv[o];
    if (half) {
      x[o] += al * (di * p[o]);
    } else {
      const double ss = s[o];
      x[o] += al * (di * p[o]) + om * (di * ss);
      const double rr = ss - om * t[o];
      r[o] = rr;
      a0 += rr * rr;
      a1 += rh[o] * rr;
    }
  }
  double vv[2] = {a0, a1};
  block_reduce_finalize<2>(vv, ra);
}

void launch_bi_init(const Geom& g, const double* y, const double* b, double* r, double* rhat,
                    const RedArgs& ra, cudaStream_t st) {
  k_bi_init<<<grid_pw(g), 256, 0, st>>>(g, y, b, r, rhat, ra);
}
void launch_bi_p(const Geom& g, const double* r, double* p, const double* v, int first,
                 const KScal* sc, cudaStream_t st) {
  k_bi_p<<<grid_pw(g), 256, 0, st>>>(g, r, p, v, first, sc);
}
void launch_bi_s(const Geom& g, const double* r, const double* v, double* s, const RedArgs& ra,
                 cudaStream_t st) {
  k_bi_s<<<grid_pw(g), 256, 0, st>>>(g, r, v, s, ra);
}
void launch_bi_xr(const Geom& g, double* x, const double* p, const double* s, const double* t,
                  double* r, const double* rhat, const double* dinv, const RedArgs& ra,
                  cudaStream_t st) {
  k_bi_xr<<<grid_pw(g), 256, 0, st>>>(g, x, p, s, t, r, rhat, dinv, ra);
}

}  // namespace chb

// ----------------------------------------------------------------- GMRES
namespace chb {

struct VPtrs {
  double* v[66];
};

constexpr int GM_STRIDE = 72;  // partial-sum stride per block (k <= 66)

// out[i] = sum_cells V_i * w  (i < k), deterministic: per-block partials in
// fixed order, the last block (ticket) reduces them in block order.
__global__ void __launch_bounds__(256) k_gm_dots(Geom g, VPtrs V, int k,
                                                 const double* __restrict__ w, double* out,
                                                 double* part, unsigned int* ticket) {
  __shared__ double sm[8];
  __shared__ int am_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int bid = blockIdx.x + blockIdx.y * gridDim.x, nb = gridDim.x * gridDim.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < k; ++i) {
    double acc = 0.0;
    if (c < g.nx)
      for (int jl = blockIdx.y; jl < g.nyl; jl += gridDim.y) {
        const size_t o = off(g, g.j0 + jl, c);
        acc += V.v[i][o] * w[o];
      }
    acc = warp_sum(acc);
    if (lane == 0) sm[wid] = acc;
    __syncthreads();
    if (wid == 0) {
      double t = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) part[(size_t)bid * GM_STRIDE + i] = t;
    }
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    am_last = (atomicAdd(ticket, 1u) == (unsigned)(nb - 1));
  }
  __syncthreads();
  if (!am_last || wid != 0) return;
  __threadfence();
  for (int i = 0; i < k; ++i) {
    double t = 0.0;
    for (int b = lane; b < nb; b += 32) t += __ldcg(part + (size_t)b * GM_STRIDE + i);
    t = warp_sum(t);
    if (lane == 0) out[i] = t;
  }
  if (lane == 0) *ticket = 0u;
}

__global__ void __launch_bounds__(256) k_gm_scale(Geom g, double* v, const double* coef) {
  const double s = coef[0];
  CHB_PW_LOOP(g) { v[off(g, g.j0 + jl, c_)] *= s; }
}

__global__ void __launch_bounds__(256) k_gm_axpy_multi(Geom g, VPtrs V, int k,
                                                       const double* __restrict__ coef,
                                                       double* __restrict__ w) {
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    double acc = w[o];
    for (int i = 0; i < k; ++i) acc -= coef[i] * V.v[i][o];
    w[o] = acc;
  }
}

__global__ void __launch_bounds__(256) k_gm_residual(Geom g, const double* __restrict__ y,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ v0) {
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    v0[o] = b[o] - y[o];
  }
}

__global__ void __launch_bounds__(256) k_gm_update_x(Geom g, VPtrs V, int k,
                                                     const double* __restrict__ coef,
                                                     const double* __restrict__ dinv,
                                                     double* __restrict__ x) {
  CHB_PW_LOOP(g) {
    const size_t o = off(g, g.j0 + jl, c_);
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc += coef[i] * V.v[i][o];
    x[o] += dinv[o] * acc;
  }
}

static VPtrs vptrs(double* const* V, int k) {
  VPtrs p;
  for (int i = 0; i < 66; ++i) p.v[i] = i < k ? V[i] : nullptr;
  return p;
}

static dim3 grid_gm(const Geom& g) {
  int gy = g.nyl < 512 ? g.nyl : 512;
  return dim3((g.nx + 255) / 256, gy);
}

void launch_gm_dots(const Geom& g, double* const* V, int k, const double* w, double* out,
                    double* part, unsigned int* ticket, cudaStream_t st) {
  k_gm_dots<<<grid_gm(g), 256, 0, st>>>(g, vptrs(V, k), k, w, out, part, ticket);
}
void launch_gm_scale(const Geom& g, double* v, const double* coef, cudaStream_t st) {
  k_gm_scale<<<grid_pw(g), 256, 0, st>>>(g, v, coef);
}
void launch_gm_axpy_multi(const Geom& g, double* const* V, int k, const double* coef, double* w,
                          cudaStream_t st) {
  k_gm_axpy_multi<<<grid_pw(g), 256, 0, st>>>(g, vptrs(V, k), k, coef, w);
}
void launch_gm_residual(const Geom& g, const double* y, const double* b, double* v0,
                        cudaStream_t st) {
  k_gm_residual<<<grid_pw(g), 256, 0, st>>>(g, y, b, v0);
}
void launch_gm_update_x(const Geom& g, double* const* V, int k, const double* coef,
                        const double* dinv, double* x, cudaStream_t st) {
  k_gm_update_x<<<grid_pw(g), 256, 0, st>>>(g, vptrs(V, k), k, coef, dinv, x);
}

}  // namespace chb
