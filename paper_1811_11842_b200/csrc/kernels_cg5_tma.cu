// kernels_cg5_tma.cu -- TMA-staged (cp.async.bulk + mbarrier ring) versions
// of the fused CG half-iterations of kernels_cg5.cu.
//
// Each block owns a 256-column chunk of a row strip.  One elected thread
// streams whole row segments of every input array into an NST-deep shared
// memory ring with 1-D bulk async copies (TMA engine, no registers held while
// in flight); the four warps consume rows j-1, j, j+1 from shared memory
// (x-neighbours included: each staged segment carries two halo columns on
// each side, periodic wrap resolved by the producer).  So each SM keeps
// (NST - 3) rows x (staged arrays) in flight without any register cost --
// enough to cover HBM latency at full bandwidth -- and the 5-point evaluation
// reads shared memory only.  Arithmetic is identical to kernels_cg5.cu.
#include <stdint.h>

#include "common.cuh"
#include "launch.h"
#include "op5.cuh"
#include "tma.cuh"

namespace chb {

constexpr int TW = 256;   // columns per block (128 threads x 2)
constexpr int TSEG = TW + 4;
constexpr int NSTREAM = 5;

// Stream roles.  Halo streams are staged with 2 halo columns each side on
// every ring row (including the strip's two halo rows); centre streams only
// on the strip's own rows.
struct Streams {
  const double* g[NSTREAM];
  int halo[NSTREAM];
  int on[NSTREAM];
  int soff[NSTREAM];   // doubles from stage start
  int stage_doubles;
};

template <int BC>
__device__ __forceinline__ int fold_src_row(const Geom& g, int gj) {
  if (BC == BC_VFACE) return gj < 0 ? 1 : (gj >= g.ny ? g.ny - 1 : gj);  // ghosts: value ignored
  if (gj < 0) return -1 - gj;
  if (gj >= g.ny) return 2 * g.ny - 1 - gj;
  return gj;
}

// Issue ring row i (global row gj) into stage st.  Called by one thread.
template <int BC>
__device__ __forceinline__ void issue_row(const Geom& g, const Streams& S, double* ring,
                                          uint64_t* bars, int st, int gj, bool centre, int c0,
                                          int wc) {
  const int grow = fold_src_row<BC>(g, gj);
  const int crow = fold_src_row<BC_MIRROR>(g, gj);  // coefficient rows are mirror-folded
  const int cl = c0 - 2 < 0 ? c0 - 2 + g.nx : c0 - 2;
  const int cr = c0 + wc >= g.nx ? c0 + wc - g.nx : c0 + wc;
  uint32_t tx = 0;
#pragma unroll
  for (int s = 0; s < NSTREAM; ++s) {
    if (!S.on[s]) continue;
    if (S.halo[s]) tx += (uint32_t)(wc * 8 + 32);
    else if (centre) tx += (uint32_t)(wc * 8);
  }
  uint64_t* bar = bars + st;
  mbar_expect_tx(bar, tx);
  double* stage = ring + (size_t)st * S.stage_doubles;
#pragma unroll
  for (int s = 0; s < NSTREAM; ++s) {
    if (!S.on[s]) continue;
    const int r = (s == 2) ? crow : grow;   // stream 2 is always the cell coefficient w
    const double* row = S.g[s] + (size_t)(r - g.j0 + GH) * g.pitch;
    double* dst = stage + S.soff[s];
    if (S.halo[s]) {
      if (cl + 2 == c0 && cr == c0 + wc) {       // interior chunk: one contiguous segment
        bulk_g2s(dst, row + cl, wc * 8 + 32, bar);
      } else {                                   // periodic seam: main + wrapped halos
        bulk_g2s(dst + 2, row + c0, wc * 8, bar);
        bulk_g2s(dst, row + cl, 16, bar);
        bulk_g2s(dst + 2 + wc, row + cr, 16, bar);
      }
    } else if (centre) {
      bulk_g2s(dst, row + c0, wc * 8, bar);
    }
  }
}


// sign / zero of a staged unknown value at global row gj (BC at read time)
template <int BC>
__device__ __forceinline__ double bc_scale(const Geom& g, int gj) {
  if (BC == BC_VFACE) return (gj <= 0 || gj >= g.ny) ? 0.0 : 1.0;
  if (BC == BC_ODD) return (gj < 0 || gj >= g.ny) ? -1.0 : 1.0;
  return 1.0;
}

// ------------------------------------------------------------------- A
// p = z + beta p_old; x += alpha p_old; q = A p; reduce (p, q)
template <int BC, int AM, int KM, int NST>
__global__ void __launch_bounds__(128) k_cg5_A4(Geom g, Op5T op, const double* __restrict__ z,
                                                const double* __restrict__ po,
                                                double* __restrict__ pn, double* __restrict__ x,
                                                int first, int strip, int dir, RedArgs ra) {
  if (ra.sc->done) return;
  extern __shared__ __align__(128) double ring[];
  __shared__ uint64_t bars[NST];
  const double beta = first ? 0.0 : ra.sc->beta;
  const double alpha = first ? 0.0 : ra.sc->alpha;
  const int c0 = blockIdx.x * TW;
  const int wc = min(TW, g.nx - c0);
  const int t = threadIdx.x;
  const bool act = 2 * t < wc;
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  const int n = jl1 - jl0;
  const int jb = dir > 0 ? jl0 : jl1 - 1;
  Streams S;
  S.g[0] = z;  S.halo[0] = 1; S.on[0] = 1;
  S.g[1] = po; S.halo[1] = 1; S.on[1] = !first;
  S.g[2] = op.w; S.halo[2] = 1; S.on[2] = KM != 0;
  S.g[3] = x;  S.halo[3] = 0; S.on[3] = !first;
  S.g[4] = op.a; S.halo[4] = 0; S.on[4] = AM != 0;
  int o = 0;
  for (int s = 0; s < NSTREAM; ++s) {
    S.soff[s] = o;
    if (S.on[s]) o += S.halo[s] ? TSEG : TW;
  }
  S.stage_doubles = (o + 15) & ~15;
  ring_setup(bars, NST);
  const int nrow = n + 2;  // ring rows: halo, n strip rows, halo
  auto rowg = [&](int i) { return g.j0 + jb + (i - 1) * dir; };
  if (t == 0) {
    for (int i = 0; i < NST && i < nrow; ++i)
      issue_row<BC>(g, S, ring, bars, i, rowg(i), i >= 1 && i <= n, c0, wc);
  }
  const int ci = 2 * t + 2;  // index of own first column inside a halo segment
  // P at the 4 positions (w, c, c+1, e) of ring row i
  auto Pq = [&](int i, double& pw, double& p0, double& p1, double& pe) {
    const double* st = ring + (size_t)(i % NST) * S.stage_doubles;
    const double sc = bc_scale<BC>(g, rowg(i));
    const double* zs = st + S.soff[0];
    pw = zs[ci - 1]; p0 = zs[ci]; p1 = zs[ci + 1]; pe = zs[ci + 2];
    if (!first) {
      const double* ps = st + S.soff[1];
      pw += beta * ps[ci - 1]; p0 += beta * ps[ci]; p1 += beta * ps[ci + 1]; pe += beta * ps[ci + 2];
    }
    pw *= sc; p0 *= sc; p1 *= sc; pe *= sc;
  };
  mbar_wait(bars + 0, 0);
  mbar_wait(bars + 1, 0);
  double acc = 0.0;
  int gj = g.j0 + jb;
  for (int k = 0; k < n; ++k, gj += dir) {
    const int ib = k, ic = k + 1, ia = k + 2;   // behind, centre, ahead ring rows
    mbar_wait(bars + (ia % NST), (ia / NST) & 1);
    double bw, b0, b1, be, cw_, c0v, c1v, ce, aw, a0, a1, ae;
    Pq(ib, bw, b0, b1, be);
    Pq(ic, cw_, c0v, c1v, ce);
    Pq(ia, aw, a0, a1, ae);
    const double* stc = ring + (size_t)(ic % NST) * S.stage_doubles;
    double w_w = 0, w_0 = 0, w_1 = 0, w_e = 0, w_s0 = 0, w_s1 = 0, w_n0 = 0, w_n1 = 0;
    if (KM) {
      const double* wcs = stc + S.soff[2];
      const double* wbs = ring + (size_t)(ib % NST) * S.stage_doubles + S.soff[2];
      const double* was = ring + (size_t)(ia % NST) * S.stage_doubles + S.soff[2];
      w_w = wcs[ci - 1]; w_0 = wcs[ci]; w_1 = wcs[ci + 1]; w_e = wcs[ci + 2];
      const double* wsS = dir > 0 ? wbs : was;
      const double* wsN = dir > 0 ? was : wbs;
      w_s0 = wsS[ci]; w_s1 = wsS[ci + 1]; w_n0 = wsN[ci]; w_n1 = wsN[ci + 1];
    }
    double a_0 = 0.0, a_1 = 0.0;
    if (AM) {
      const double* as = stc + S.soff[4];
      a_0 = as[2 * t]; a_1 = as[2 * t + 1];
    }
    const double s0 = dir > 0 ? b0 : a0, s1 = dir > 0 ? b1 : a1;   // south row (j-1)
    const double n0 = dir > 0 ? a0 : b0, n1 = dir > 0 ? a1 : b1;   // north row (j+1)
    double y0, y1, d0, d1;
    eval5T<BC, AM, KM>(op, g, gj, a_0, w_0, w_w, w_1, w_s0, w_n0, c0v, cw_, c1v, s0, n0, y0, d0);
    eval5T<BC, AM, KM>(op, g, gj, a_1, w_1, w_0, w_e, w_s1, w_n1, c1v, c0v, ce, s1, n1, y1, d1);
    if (act) {
      const size_t go = off(g, gj, c0 + 2 * t);
      *reinterpret_cast<double2*>(pn + go) = make_double2(c0v, c1v);
      if (!first) {
        const double* xs = stc + S.soff[3];
        const double* ps = stc + S.soff[1];
        double2 xo = make_double2(xs[2 * t], xs[2 * t + 1]);
        xo.x += alpha * ps[ci];
        xo.y += alpha * ps[ci + 1];
        *reinterpret_cast<double2*>(x + go) = xo;
      }
      acc += c0v * y0 + c1v * y1;
    }
    __syncthreads();                                  // ring row ib is free
    if (t == 0 && ib + NST < nrow) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_row<BC>(g, S, ring, bars, ib % NST, rowg(ib + NST), ib + NST <= n, c0, wc);
    }
  }
  double v[1] = {acc};
  block_reduce_finalize<1>(v, ra);
}

// ------------------------------------------------------------------- B
// r = d z - alpha A p; z = r / d; reduce (r, z), (r, r)
template <int BC, int AM, int KM, int NST>
__global__ void __launch_bounds__(128) k_cg5_B4(Geom g, Op5T op, const double* __restrict__ p,
                                                double* __restrict__ z, int strip, int dir,
                                                RedArgs ra) {
  if (ra.sc->done) return;
  extern __shared__ __align__(128) double ring[];
  __shared__ uint64_t bars[NST];
  const double alpha = ra.sc->alpha;
  const int c0 = blockIdx.x * TW;
  const int wc = min(TW, g.nx - c0);
  const int t = threadIdx.x;
  const bool act = 2 * t < wc;
  const int jl0 = blockIdx.y * strip, jl1 = min(jl0 + strip, g.nyl);
  const int n = jl1 - jl0;
  const int jb = dir > 0 ? jl0 : jl1 - 1;
  Streams S;
  S.g[0] = p;  S.halo[0] = 1; S.on[0] = 1;
  S.g[1] = nullptr; S.halo[1] = 0; S.on[1] = 0;
  S.g[2] = op.w; S.halo[2] = 1; S.on[2] = KM != 0;
  S.g[3] = z;  S.halo[3] = 0; S.on[3] = 1;
  S.g[4] = op.a; S.halo[4] = 0; S.on[4] = AM != 0;
  int o = 0;
  for (int s = 0; s < NSTREAM; ++s) {
    S.soff[s] = o;
    if (S.on[s]) o += S.halo[s] ? TSEG : TW;
  }
  S.stage_doubles = (o + 15) & ~15;
  ring_setup(bars, NST);
  const int nrow = n + 2;
  auto rowg = [&](int i) { return g.j0 + jb + (i - 1) * dir; };
  if (t == 0) {
    for (int i = 0; i < NST && i < nrow; ++i)
      issue_row<BC>(g, S, ring, bars, i, rowg(i), i >= 1 && i <= n, c0, wc);
  }
  const int ci = 2 * t + 2;
  mbar_wait(bars + 0, 0);
  mbar_wait(bars + 1, 0);
  double s0acc = 0.0, s1acc = 0.0;
  int gj = g.j0 + jb;
  for (int k = 0; k < n; ++k, gj += dir) {
    const int ib = k, ic = k + 1, ia = k + 2;
    mbar_wait(bars + (ia % NST), (ia / NST) & 1);
    const double* stb = ring + (size_t)(ib % NST) * S.stage_doubles;
    const double* stc = ring + (size_t)(ic % NST) * S.stage_doubles;
    const double* sta = ring + (size_t)(ia % NST) * S.stage_doubles;
    const double sb = bc_scale<BC>(g, rowg(ib)), scc = bc_scale<BC>(g, rowg(ic)),
                 sa = bc_scale<BC>(g, rowg(ia));
    const double* pc = stc + S.soff[0];
    const double cw_ = scc * pc[ci - 1], c0v = scc * pc[ci], c1v = scc * pc[ci + 1],
                 ce = scc * pc[ci + 2];
    const double b0 = sb * stb[S.soff[0] + ci], b1 = sb * stb[S.soff[0] + ci + 1];
    const double a0 = sa * sta[S.soff[0] + ci], a1 = sa * sta[S.soff[0] + ci + 1];
    double w_w = 0, w_0 = 0, w_1 = 0, w_e = 0, w_s0 = 0, w_s1 = 0, w_n0 = 0, w_n1 = 0;
    if (KM) {
      const double* wcs = stc + S.soff[2];
      w_w = wcs[ci - 1]; w_0 = wcs[ci]; w_1 = wcs[ci + 1]; w_e = wcs[ci + 2];
      const double* wsS = (dir > 0 ? stb : sta) + S.soff[2];
      const double* wsN = (dir > 0 ? sta : stb) + S.soff[2];
      w_s0 = wsS[ci]; w_s1 = wsS[ci + 1]; w_n0 = wsN[ci]; w_n1 = wsN[ci + 1];
    }
    double a_0 = 0.0, a_1 = 0.0;
    if (AM) {
      const double* as = stc + S.soff[4];
      a_0 = as[2 * t]; a_1 = as[2 * t + 1];
    }
    const double s0 = dir > 0 ? b0 : a0, s1 = dir > 0 ? b1 : a1;
    const double n0 = dir > 0 ? a0 : b0, n1 = dir > 0 ? a1 : b1;
    double y0, y1, d0, d1;
    eval5T<BC, AM, KM>(op, g, gj, a_0, w_0, w_w, w_1, w_s0, w_n0, c0v, cw_, c1v, s0, n0, y0, d0);
    eval5T<BC, AM, KM>(op, g, gj, a_1, w_1, w_0, w_e, w_s1, w_n1, c1v, c0v, ce, s1, n1, y1, d1);
    if (act) {
      const double* zs = stc + S.soff[3];
      const double rx = d0 * zs[2 * t] - alpha * y0, ry = d1 * zs[2 * t + 1] - alpha * y1;
      const double2 zn = make_double2(rx / d0, ry / d1);
      *reinterpret_cast<double2*>(z + off(g, gj, c0 + 2 * t)) = zn;
      s0acc += rx * zn.x + ry * zn.y;
      s1acc += rx * rx + ry * ry;
    }
    __syncthreads();
    if (t == 0 && ib + NST < nrow) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_row<BC>(g, S, ring, bars, ib % NST, rowg(ib + NST), ib + NST <= n, c0, wc);
    }
  }
  double v[2] = {s0acc, s1acc};
  block_reduce_finalize<2>(v, ra);
}

// ============================================================== launchers
constexpr int RING = 8;

static Op5T make_opT(const OpDesc& d) {
  Op5T o;
  o.a = d.a;
  o.w = d.w;
  o.s = d.s;
  o.kscale = d.kscale;
  o.rho_n = d.rho_n;
  o.rho_s = d.rho_s;
  return o;
}

template <int AM, int KM>
static size_t ring_bytes_A(int first) {
  int o = TSEG + (first ? 0 : TSEG) + (KM ? TSEG : 0) + (first ? 0 : TW) + (AM ? TW : 0);
  return (size_t)RING * (size_t)((o + 15) & ~15) * sizeof(double);
}
template <int AM, int KM>
static size_t ring_bytes_B() {
  int o = TSEG + (KM ? TSEG : 0) + TW + (AM ? TW : 0);
  return (size_t)RING * (size_t)((o + 15) & ~15) * sizeof(double);
}

template <typename K>
static int strip_for(K kern, size_t smem, const Geom& g, int forced) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (forced > 0) return forced;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem);
  if (per_sm < 1) per_sm = 1;
  const int ncb = (g.nx + TW - 1) / TW;
  int nstrips = nsm * per_sm / ncb;
  if (nstrips < 1) nstrips = 1;
  int strip = (g.nyl + nstrips - 1) / nstrips;
  return strip < 2 ? 2 : strip;
}

template <int BC, int AM, int KM>
static void launch_A4(const OpDesc& d, const Geom& g, const double* z, const double* po,
                      double* pn, double* x, int first, const RedArgs& ra, cudaStream_t st) {
  const Op5T op = make_opT(d);
  // strips are sized from the (larger) non-first footprint so A and B share them
  const size_t smem_full = ring_bytes_A<AM, KM>(0);
  const int strip = strip_for(k_cg5_A4<BC, AM, KM, RING>, smem_full, g, d.strip2);
  const size_t smem = ring_bytes_A<AM, KM>(first);
  dim3 grid((g.nx + TW - 1) / TW, (g.nyl + strip - 1) / strip);
  k_cg5_A4<BC, AM, KM, RING><<<grid, 128, smem, st>>>(g, op, z, po, pn, x, first, strip, 1, ra);
}

template <int BC, int AM, int KM>
static void launch_B4(const OpDesc& d, const Geom& g, const double* p, double* z,
                      const RedArgs& ra, cudaStream_t st) {
  const Op5T op = make_opT(d);
  const int strip = strip_for(k_cg5_A4<BC, AM, KM, RING>, ring_bytes_A<AM, KM>(0), g, d.strip2);
  const size_t smem = ring_bytes_B<AM, KM>();
  cudaFuncSetAttribute(k_cg5_B4<BC, AM, KM, RING>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  dim3 grid((g.nx + TW - 1) / TW, (g.nyl + strip - 1) / strip);
  k_cg5_B4<BC, AM, KM, RING><<<grid, 128, smem, st>>>(g, op, p, z, strip, -1, ra);
}

#define CHB_DISPATCH_T(KIND, CALL)                                                        \
  switch (KIND) {                                                                         \
    case OPK_POISSON_CONST: { constexpr int BC = BC_MIRROR, AM = 0, KM = 0; CALL; } break; \
    case OPK_POISSON_VAR:   { constexpr int BC = BC_MIRROR, AM = 0, KM = 2; CALL; } break; \
    case OPK_NUTRIENT:      { constexpr int BC = BC_MIRROR, AM = 1, KM = 1; CALL; } break; \
    case OPK_MOM_U:         { constexpr int BC = BC_ODD,    AM = 1, KM = 0; CALL; } break; \
    case OPK_MOM_V:         { constexpr int BC = BC_VFACE,  AM = 1, KM = 0; CALL; } break; \
    default: break;                                                                       \
  }

void launch_cg5_A_tma(const OpDesc& d, const Geom& g, const double* z, const double* po,
                      double* pn, double* x, int first, const RedArgs& ra, cudaStream_t st) {
  CHB_DISPATCH_T(d.kind, (launch_A4<BC, AM, KM>(d, g, z, po, pn, x, first, ra, st)));
}

void launch_cg5_B_tma(const OpDesc& d, const Geom& g, const double* p, double* z,
                      const RedArgs& ra, cudaStream_t st) {
  CHB_DISPATCH_T(d.kind, (launch_B4<BC, AM, KM>(d, g, p, z, ra, st)));
}

}  // namespace chb
