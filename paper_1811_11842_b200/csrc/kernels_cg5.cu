// kernels_cg5.cu -- the 5-point symmetric operator family and its fused
// Jacobi-preconditioned CG half-iterations (the hot path of every step:
// pressure Poisson, Eq. 20; intermediate velocity, Eq. 19; nutrient, Eq. 16).
//
//   y = a x + s * sum_faces k_f (x - x_nb) / h_f^2
//
// Operator instances (OpKind):
//   POISSON_CONST  a = 0, s = 1, k = 1                      (rho_n == rho_s)
//   POISSON_VAR    a = 0, s = 1, k = 1/rho(face mean phi^{n+1})
//   NUTRIENT       a = a_c[], s = 1/2, k = D_s * face mean(phi_s^{1/2})
//   MOM_U          a = a_u[], s = 1/2, k = 1, odd-reflection walls
//   MOM_V          a = a_v[], s = 1/2, k = 1, Dirichlet wall faces, row 0 = identity
//
// Memory plan per CG iteration (z-form CG: z = D^{-1} r is stored, r = d z is
// re-formed in registers, so D^{-1} is never needed at a neighbour):
//   A: read z, p_old, x (+coef);  write p, x;   reduce (p, Ap)         40 B/cell
//   B: read p, z (+coef);         write z;      reduce (r, z), (r, r)  24 B/cell
// Each thread owns one column and marches down a strip of rows keeping the
// three-row window in registers; x-neighbours come from warp shuffles (edge
// lanes and the periodic seam reload through L1).
#include "common.cuh"
#include "launch.h"

namespace chb {

struct Op5 {
  const double* a;   // diagonal coefficient at the unknown's location (AM = 1)
  const double* w;   // cell-centred coefficient source (KM = 1, 2)
  double s;          // face-term scale
  double kscale;     // KM = 1: k = kscale * mean(w)
  double rho_n, rho_s;
};

template <int KM>
__device__ __forceinline__ double kface(const Op5& op, double w1, double w2) {
  if (KM == 0) return 1.0;
  const double m = 0.5 * (w1 + w2);
  if (KM == 1) return op.kscale * m;
  return 1.0 / (op.rho_s + m * (op.rho_n - op.rho_s));
}

// y = (A x) at one cell and its diagonal d.  Neighbour values are already
// ghost-folded for the unknown's BC; w values are mirror-folded.
template <int BC, int AM, int KM>
__device__ __forceinline__ void eval5(const Op5& op, const Geom& g, int gj, double ac, double wc,
                                      double ww, double we, double ws, double wn, double xc,
                                      double xw, double xe, double xs, double xn, double& y,
                                      double& d) {
  if (BC == BC_VFACE && gj == 0) {  // wall row: identity
    y = xc;
    d = 1.0;
    return;
  }
  const double kE = kface<KM>(op, wc, we), kW = kface<KM>(op, ww, wc);
  const double kN = kface<KM>(op, wc, wn), kS = kface<KM>(op, ws, wc);
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
__global__ void __launch_bounds__(128) k_cg5_init(Geom g, Op5 op, const double* __restrict__ x,
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
    const double ac = AM ? op.a[off(g, gj, col.cc)] : 0.0;
    double y, d;
    eval5<BC, AM, KM>(op, g, gj, ac, w0, ww, we, wm, wp, x0, xw, xe, xm, xp, y, d);
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

// --------------------------------------------------------------- CG half A
// p = z + beta p_old (p = z on the first iteration);  x += alpha_prev p_old;
// q = A p;  reduce (p, q)  -> alpha = rho / (p, q)
template <int BC, int AM, int KM>
__global__ void __launch_bounds__(128) k_cg5_A(Geom g, Op5 op, const double* __restrict__ z,
                                               const double* __restrict__ po,
                                               double* __restrict__ pn, double* __restrict__ x,
                                               int first, int strip, RedArgs ra) {
  if (ra.sc->done) return;
  const double beta = first ? 0.0 : ra.sc->beta;
  const double alpha = first ? 0.0 : ra.sc->alpha;
  Col col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  double acc = 0.0;
  int gj = g.j0 + jl0;
  auto P = [&](int r, int cidx) -> double {
    double v = ldf<BC>(z, g, r, cidx);
    if (!first) v += beta * ldf<BC>(po, g, r, cidx);
    return v;
  };
  double pm = P(gj - 1, col.cc), p0 = P(gj, col.cc);
  double wm = 0.0, w0 = 0.0;
  if (KM) {
    wm = ldf<BC_MIRROR>(op.w, g, gj - 1, col.cc);
    w0 = ldf<BC_MIRROR>(op.w, g, gj, col.cc);
  }
  for (int jl = jl0; jl < jl1; ++jl, ++gj) {
    const double pp = P(gj + 1, col.cc);
    double pw = CHB_SHFL_W(p0), pe = CHB_SHFL_E(p0);
    if (col.needW) pw = P(gj, col.cw);
    if (col.needE) pe = P(gj, col.ce);
    double wp = 0.0, ww = 0.0, we = 0.0;
    if (KM) {
      wp = ldf<BC_MIRROR>(op.w, g, gj + 1, col.cc);
      ww = CHB_SHFL_W(w0);
      we = CHB_SHFL_E(w0);
      if (col.needW) ww = ldf<BC_MIRROR>(op.w, g, gj, col.cw);
      if (col.needE) we = ldf<BC_MIRROR>(op.w, g, gj, col.ce);
    }
    const double ac = AM ? op.a[off(g, gj, col.cc)] : 0.0;
    double y, d;
    eval5<BC, AM, KM>(op, g, gj, ac, w0, ww, we, wm, wp, p0, pw, pe, pm, pp, y, d);
    if (col.act) {
      const size_t o = off(g, gj, col.c);
      pn[o] = p0;
      if (!first) x[o] += alpha * po[o];
      acc += p0 * y;
    }
    pm = p0;
    p0 = pp;
    wm = w0;
    w0 = wp;
  }
  double v[1] = {acc};
  block_reduce_finalize<1>(v, ra);
}

// --------------------------------------------------------------- CG half B
// r = d z - alpha A p;  z = r / d;  reduce (r, z), (r, r)
template <int BC, int AM, int KM>
__global__ void __launch_bounds__(128) k_cg5_B(Geom g, Op5 op, const double* __restrict__ p,
                                               double* __restrict__ z, int strip, RedArgs ra) {
  if (ra.sc->done) return;
  const double alpha = ra.sc->alpha;
  Col col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  double s0 = 0.0, s1 = 0.0;
  int gj = g.j0 + jl0;
  double pm = ldf<BC>(p, g, gj - 1, col.cc), p0 = ldf<BC>(p, g, gj, col.cc);
  double wm = 0.0, w0 = 0.0;
  if (KM) {
    wm = ldf<BC_MIRROR>(op.w, g, gj - 1, col.cc);
    w0 = ldf<BC_MIRROR>(op.w, g, gj, col.cc);
  }
  for (int jl = jl0; jl < jl1; ++jl, ++gj) {
    const double pp = ldf<BC>(p, g, gj + 1, col.cc);
    double pw = CHB_SHFL_W(p0), pe = CHB_SHFL_E(p0);
    if (col.needW) pw = ldf<BC>(p, g, gj, col.cw);
    if (col.needE) pe = ldf<BC>(p, g, gj, col.ce);
    double wp = 0.0, ww = 0.0, we = 0.0;
    if (KM) {
      wp = ldf<BC_MIRROR>(op.w, g, gj + 1, col.cc);
      ww = CHB_SHFL_W(w0);
      we = CHB_SHFL_E(w0);
      if (col.needW) ww = ldf<BC_MIRROR>(op.w, g, gj, col.cw);
      if (col.needE) we = ldf<BC_MIRROR>(op.w, g, gj, col.ce);
    }
    const double ac = AM ? op.a[off(g, gj, col.cc)] : 0.0;
    double y, d;
    eval5<BC, AM, KM>(op, g, gj, ac, w0, ww, we, wm, wp, p0, pw, pe, pm, pp, y, d);
    if (col.act) {
      const size_t o = off(g, gj, col.c);
      const double r = d * z[o] - alpha * y;
      const double zz = r / d;
      z[o] = zz;
      s0 += r * zz;
      s1 += r * r;
    }
    pm = p0;
    p0 = pp;
    wm = w0;
    w0 = wp;
  }
  double v[2] = {s0, s1};
  block_reduce_finalize<2>(v, ra);
}

// --------------------------------------------------------------- plain apply
template <int BC, int AM, int KM>
__global__ void __launch_bounds__(128) k_op5_apply(Geom g, Op5 op, const double* __restrict__ x,
                                                   double* __restrict__ yout, int strip) {
  Col col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
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
    const double ac = AM ? op.a[off(g, gj, col.cc)] : 0.0;
    double y, d;
    eval5<BC, AM, KM>(op, g, gj, ac, w0, ww, we, wm, wp, x0, xw, xe, xm, xp, y, d);
    if (col.act) yout[off(g, gj, col.c)] = y;
    xm = x0;
    x0 = xp;
    wm = w0;
    w0 = wp;
  }
}

// ===================================================================== v2
// Vectorised marching kernels (even nx): each thread owns two adjacent
// columns (16-B loads/stores), rows are prefetched two ahead so every warp
// keeps two rows of loads in flight, and the strip index can be traversed in
// reverse (B after A reverses, so B starts on the rows A touched last and
// finds them in L2).
template <int BC>
__device__ __forceinline__ double2 ld2(const double* __restrict__ a, const Geom& g, int gj, int c) {
  if (BC == BC_VFACE) {
    if (gj <= 0 || gj >= g.ny) return make_double2(0.0, 0.0);
    return *reinterpret_cast<const double2*>(a + off(g, gj, c));
  }
  double s = 1.0;
  if (gj < 0) {
    gj = -1 - gj;
    s = (BC == BC_ODD) ? -1.0 : 1.0;
  } else if (gj >= g.ny) {
    gj = 2 * g.ny - 1 - gj;
    s = (BC == BC_ODD) ? -1.0 : 1.0;
  }
  double2 v = *reinterpret_cast<const double2*>(a + off(g, gj, c));
  v.x *= s;
  v.y *= s;
  return v;
}

struct Col2 {
  int c0, cc, cw, ce, lane;
  bool act, needW, needE;
  __device__ __forceinline__ Col2(const Geom& g) {
    lane = threadIdx.x & 31;
    c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
    act = c0 < g.nx;
    cc = act ? c0 : g.nx - 2;
    cw = wrapc(cc - 1, g.nx);
    ce = wrapc(cc + 2, g.nx);
    needW = (lane == 0) || (c0 == 0);
    needE = (lane == 31) || (c0 + 2 >= g.nx);
  }
};

// One row of an unknown-type stream: own two columns + the two outer neighbours.
struct R2 {
  double2 v;
  double w, e;
};

template <int BC>
__device__ __forceinline__ R2 ldrow(const double* __restrict__ a, const Geom& g, const Col2& col,
                                    int gj) {
  R2 r;
  r.v = ld2<BC>(a, g, gj, col.cc);
  r.w = col.needW ? ldf<BC>(a, g, gj, col.cw) : 0.0;
  r.e = col.needE ? ldf<BC>(a, g, gj, col.ce) : 0.0;
  return r;
}

// fill the outer neighbours from the adjacent lanes where they live there
__device__ __forceinline__ void xnb(const Col2& col, double2 v, double& w, double& e) {
  const double sw = __shfl_up_sync(FULL, v.y, 1);
  const double se = __shfl_down_sync(FULL, v.x, 1);
  if (!col.needW) w = sw;
  if (!col.needE) e = se;
}

template <int BC, int AM, int KM>
__device__ __forceinline__ void eval_pair(const Op5& op, const Geom& g, int gj, double2 ac,
                                          double2 wc, double ww, double we, double2 ws, double2 wn,
                                          double2 xc, double xw, double xe, double2 xs, double2 xn,
                                          double2& y, double2& d) {
  eval5<BC, AM, KM>(op, g, gj, ac.x, wc.x, ww, wc.y, ws.x, wn.x, xc.x, xw, xc.y, xs.x, xn.x, y.x,
                    d.x);
  eval5<BC, AM, KM>(op, g, gj, ac.y, wc.y, wc.x, we, ws.y, wn.y, xc.y, xc.x, xe, xs.y, xn.y, y.y,
                    d.y);
}

// Raw loads of one row for the CG half-iterations.  Rows are consumed one
// iteration after they are issued (prefetch distance 2), so each warp keeps
// two rows of loads in flight.
struct RawA {
  R2 z, p, w;
  double2 x, a;
};

template <int BC, int AM, int KM>
__device__ __forceinline__ void load_rawA(RawA& r, const Geom& g, const Col2& col, const Op5& op,
                                          const double* __restrict__ z,
                                          const double* __restrict__ po,
                                          const double* __restrict__ x, int gj, bool first,
                                          bool centre) {
  r.z = ldrow<BC>(z, g, col, gj);
  if (!first) r.p = ldrow<BC>(po, g, col, gj);
  if (KM) r.w = ldrow<BC_MIRROR>(op.w, g, col, gj);
  if (centre) {
    const size_t o = off(g, gj, col.cc);
    if (!first) r.x = *reinterpret_cast<const double2*>(x + o);
    if (AM) r.a = *reinterpret_cast<const double2*>(op.a + o);
  }
}

// A: p = z + beta p_old; x += alpha p_old; q = A p; reduce (p, q).
// DIR = +1 marches a strip upward in j, -1 downward (alternated with B).
template <int BC, int AM, int KM, int DIR>
__global__ void __launch_bounds__(128) k_cg5_A3(Geom g, Op5 op, const double* __restrict__ z,
                                                const double* __restrict__ po,
                                                double* __restrict__ pn, double* __restrict__ x,
                                                int first, int strip, RedArgs ra) {
  if (ra.sc->done) return;
  const double beta = first ? 0.0 : ra.sc->beta;
  const double alpha = first ? 0.0 : ra.sc->alpha;
  const Col2 col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  const int jb = DIR > 0 ? jl0 : jl1 - 1;       // first row marched
  const int n = jl1 - jl0;
  auto comb = [&](const RawA& r) {
    if (first) return r.z;
    R2 o;
    o.v.x = r.z.v.x + beta * r.p.v.x;
    o.v.y = r.z.v.y + beta * r.p.v.y;
    o.w = r.z.w + beta * r.p.w;
    o.e = r.z.e + beta * r.p.e;
    return o;
  };
  RawA rb, r0, r1, r2;
  int gj = g.j0 + jb;
  load_rawA<BC, AM, KM>(rb, g, col, op, z, po, x, gj - DIR, first, false);
  load_rawA<BC, AM, KM>(r0, g, col, op, z, po, x, gj, first, true);
  load_rawA<BC, AM, KM>(r1, g, col, op, z, po, x, gj + DIR, first, n > 1);
  R2 Pb = comb(rb), P0 = comb(r0);
  R2 Wb = rb.w, W0 = r0.w;
  double acc = 0.0;
  for (int k = 0; k < n; ++k, gj += DIR) {
    if (k + 1 < n) load_rawA<BC, AM, KM>(r2, g, col, op, z, po, x, gj + 2 * DIR, first, k + 2 < n);
    const R2 Pa = comb(r1);
    double pw = P0.w, pe = P0.e;
    xnb(col, P0.v, pw, pe);
    double ww = 0.0, we = 0.0;
    if (KM) {
      ww = W0.w;
      we = W0.e;
      xnb(col, W0.v, ww, we);
    }
    const R2& Ps = DIR > 0 ? Pb : Pa;   // south (j-1), north (j+1)
    const R2& Pn = DIR > 0 ? Pa : Pb;
    const double2 ws = DIR > 0 ? Wb.v : r1.w.v;
    const double2 wn = DIR > 0 ? r1.w.v : Wb.v;
    double2 y, d;
    eval_pair<BC, AM, KM>(op, g, gj, r0.a, W0.v, ww, we, ws, wn, P0.v, pw, pe, Ps.v, Pn.v, y, d);
    if (col.act) {
      const size_t o = off(g, gj, col.cc);
      *reinterpret_cast<double2*>(pn + o) = P0.v;
      if (!first) {
        double2 xo = r0.x;
        xo.x += alpha * r0.p.v.x;
        xo.y += alpha * r0.p.v.y;
        *reinterpret_cast<double2*>(x + o) = xo;
      }
      acc += P0.v.x * y.x + P0.v.y * y.y;
    }
    Pb = P0;
    P0 = Pa;
    Wb = W0;
    W0 = r1.w;
    r0 = r1;
    r1 = r2;
  }
  double v[1] = {acc};
  block_reduce_finalize<1>(v, ra);
}

struct RawB {
  R2 p, w;
  double2 z, a;
};

template <int BC, int AM, int KM>
__device__ __forceinline__ void load_rawB(RawB& r, const Geom& g, const Col2& col, const Op5& op,
                                          const double* __restrict__ p,
                                          const double* __restrict__ z, int gj, bool centre) {
  r.p = ldrow<BC>(p, g, col, gj);
  if (KM) r.w = ldrow<BC_MIRROR>(op.w, g, col, gj);
  if (centre) {
    const size_t o = off(g, gj, col.cc);
    r.z = *reinterpret_cast<const double2*>(z + o);
    if (AM) r.a = *reinterpret_cast<const double2*>(op.a + o);
  }
}

// B: r = d z - alpha A p; z = r / d; reduce (r, z), (r, r)
template <int BC, int AM, int KM, int DIR>
__global__ void __launch_bounds__(128) k_cg5_B3(Geom g, Op5 op, const double* __restrict__ p,
                                                double* __restrict__ z, int strip, RedArgs ra) {
  if (ra.sc->done) return;
  const double alpha = ra.sc->alpha;
  const Col2 col(g);
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  const int jb = DIR > 0 ? jl0 : jl1 - 1;
  const int n = jl1 - jl0;
  RawB rb, r0, r1, r2;
  int gj = g.j0 + jb;
  load_rawB<BC, AM, KM>(rb, g, col, op, p, z, gj - DIR, false);
  load_rawB<BC, AM, KM>(r0, g, col, op, p, z, gj, true);
  load_rawB<BC, AM, KM>(r1, g, col, op, p, z, gj + DIR, n > 1);
  double s0 = 0.0, s1 = 0.0;
  for (int k = 0; k < n; ++k, gj += DIR) {
    if (k + 1 < n) load_rawB<BC, AM, KM>(r2, g, col, op, p, z, gj + 2 * DIR, k + 2 < n);
    double pw = r0.p.w, pe = r0.p.e;
    xnb(col, r0.p.v, pw, pe);
    double ww = 0.0, we = 0.0;
    if (KM) {
      ww = r0.w.w;
      we = r0.w.e;
      xnb(col, r0.w.v, ww, we);
    }
    const double2 ps = DIR > 0 ? rb.p.v : r1.p.v, pnn = DIR > 0 ? r1.p.v : rb.p.v;
    const double2 ws = DIR > 0 ? rb.w.v : r1.w.v, wn = DIR > 0 ? r1.w.v : rb.w.v;
    double2 y, d;
    eval_pair<BC, AM, KM>(op, g, gj, r0.a, r0.w.v, ww, we, ws, wn, r0.p.v, pw, pe, ps, pnn, y, d);
    if (col.act) {
      const size_t o = off(g, gj, col.cc);
      const double rx = d.x * r0.z.x - alpha * y.x, ry = d.y * r0.z.y - alpha * y.y;
      const double2 zn = make_double2(rx / d.x, ry / d.y);
      *reinterpret_cast<double2*>(z + o) = zn;
      s0 += rx * zn.x + ry * zn.y;
      s1 += rx * rx + ry * ry;
    }
    rb = r0;
    r0 = r1;
    r1 = r2;
  }
  double v[2] = {s0, s1};
  block_reduce_finalize<2>(v, ra);
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
static Op5 make_op(const OpDesc& d) {
  Op5 o;
  o.a = d.a;
  o.w = d.w;
  o.s = d.s;
  o.kscale = d.kscale;
  o.rho_n = d.rho_n;
  o.rho_s = d.rho_s;
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
    case OPK_MOM_U:         { constexpr int BC = BC_ODD,    AM = 1, KM = 0; CALL; } break; \
    case OPK_MOM_V:         { constexpr int BC = BC_VFACE,  AM = 1, KM = 0; CALL; } break; \
    default: break;                                                     \
  }

void launch_cg5_init(const OpDesc& d, const Geom& g, const double* x, const double* b,
                     int use_shift, double* z, const RedArgs& ra, cudaStream_t st) {
  const Op5 op = make_op(d);
  const int strip = d.strip;
  CHB_DISPATCH(d.kind, (k_cg5_init<BC, AM, KM><<<grid5(g, strip), 128, 0, st>>>(
                           g, op, x, b, use_shift, z, strip, ra)));
}

// One resident wave: strip height chosen so that (column blocks x strips)
// fits the occupancy of the kernel instance on this device.
template <typename K>
static int wave_strip(K kern, const Geom& g, int min_strip) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  if (per_sm < 1) per_sm = 1;
  const int cap = nsm * per_sm;
  const int ncb = (g.nx + 255) / 256;
  int nstrips = cap / ncb;
  if (nstrips < 1) nstrips = 1;
  int strip = (g.nyl + nstrips - 1) / nstrips;
  if (strip < min_strip) strip = min_strip;
  return strip;
}

static dim3 grid5v(const Geom& g, int strip) {
  return dim3((g.nx + 255) / 256, (g.nyl + strip - 1) / strip);
}

template <int BC, int AM, int KM>
static void launch_A3(const OpDesc& d, const Op5& op, const Geom& g, const double* z,
                      const double* po, double* pn, double* x, int first, const RedArgs& ra,
                      cudaStream_t st) {
  const int strip = d.strip2 > 0 ? d.strip2 : wave_strip(k_cg5_A3<BC, AM, KM, 1>, g, 2);
  k_cg5_A3<BC, AM, KM, 1><<<grid5v(g, strip), 128, 0, st>>>(g, op, z, po, pn, x, first, strip, ra);
}

template <int BC, int AM, int KM>
static void launch_B3(const OpDesc& d, const Op5& op, const Geom& g, const double* p, double* z,
                      const RedArgs& ra, cudaStream_t st) {
  const int strip = d.strip2 > 0 ? d.strip2 : wave_strip(k_cg5_A3<BC, AM, KM, 1>, g, 2);
  k_cg5_B3<BC, AM, KM, -1><<<grid5v(g, strip), 128, 0, st>>>(g, op, p, z, strip, ra);
}

void launch_cg5_A(const OpDesc& d, const Geom& g, const double* z, const double* po, double* pn,
                  double* x, int first, const RedArgs& ra, cudaStream_t st) {
  const Op5 op = make_op(d);
  if (d.vec == 2 && (g.nx % 2 == 0)) {
    launch_cg5_A_tma(d, g, z, po, pn, x, first, ra, st);
    return;
  }
  if (d.vec && (g.nx % 2 == 0)) {
    CHB_DISPATCH(d.kind, (launch_A3<BC, AM, KM>(d, op, g, z, po, pn, x, first, ra, st)));
    return;
  }
  const int strip = d.strip;
  CHB_DISPATCH(d.kind, (k_cg5_A<BC, AM, KM><<<grid5(g, strip), 128, 0, st>>>(
                           g, op, z, po, pn, x, first, strip, ra)));
}

void launch_cg5_B(const OpDesc& d, const Geom& g, const double* p, double* z, const RedArgs& ra,
                  cudaStream_t st) {
  const Op5 op = make_op(d);
  if (d.vec == 2 && (g.nx % 2 == 0)) {
    launch_cg5_B_tma(d, g, p, z, ra, st);
    return;
  }
  if (d.vec && (g.nx % 2 == 0)) {
    CHB_DISPATCH(d.kind, (launch_B3<BC, AM, KM>(d, op, g, p, z, ra, st)));
    return;
  }
  const int strip = d.strip;
  CHB_DISPATCH(d.kind, (k_cg5_B<BC, AM, KM><<<grid5(g, strip), 128, 0, st>>>(g, op, p, z, strip,
                                                                               ra)));
}

void launch_op5_apply(const OpDesc& d, const Geom& g, const double* x, double* y,
                      cudaStream_t st) {
  const Op5 op = make_op(d);
  const int strip = d.strip;
  CHB_DISPATCH(d.kind, (k_op5_apply<BC, AM, KM><<<grid5(g, strip), 128, 0, st>>>(g, op, x, y,
                                                                                   strip)));
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
