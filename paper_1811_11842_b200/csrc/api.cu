// api.cu -- C ABI (include/ch_b200.h), handle/memory management, the Krylov
// drivers (device-side scalars, host polls convergence once per chunk) and the
// time-step orchestration of DESIGN.md §1.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <unistd.h>

#include <algorithm>
#include <string>
#include <vector>

#include "ch_b200.h"
#include "comm.h"
#include "common.cuh"
#include "launch.h"

using namespace chb;

namespace {

enum Arr {
  A_PHI = 0, A_PHIP, A_C, A_U, A_V, A_P,   // state (pointer-swapped)
  A_PHI1, A_C1, A_US, A_VS,                // next-level values
  A_PHIS, A_DINV, A_B, A_CA, A_CW,         // phi*, CH Jacobi, rhs, coefficients
  A_Z, A_PA, A_PB,                         // CG
  A_R, A_RH, A_BP, A_BV, A_BS, A_BT,       // BiCGStab
  A_TMP, A_TMP2,
  A_USG, A_VSG,                            // u*, v* of the last step: momentum guesses (R25)
  A_ZH0,                                   // z history of the deferred-p/x CG (CGM - 1 more)
  A_N = A_ZH0 + CGM - 1
};

constexpr size_t XR_TOT_BYTES = (size_t)2 * XS_MAX * 8 * sizeof(double);
constexpr size_t XR_BYTES = XR_TOT_BYTES + 256;   // totals + XR_MAX flags (padded)
constexpr int MAX_BLOCKS = 1 << 20;  // reduction partials (8 doubles each): covers 16384^2 grids
constexpr int NSC = CH_NSYS + 2;  // one KScal per system + apply + spare

struct Slab {
  Geom g;
  double* a[A_N];
  std::vector<double*> V;  // GMRES basis (m + 1 vectors) + work
  std::vector<void*> bases;  // cudaMalloc'd blocks behind a[]
};

struct Timer {
  int stride = 0;
  struct Rec {
    int kc;
    long iter;  // >= 0: Krylov iteration index of the launch (for useful filtering), -1: always
    double bytes;
    cudaEvent_t e0, e1;
    int n = 1;  // launches between the two events (sweep groups: TGRP)
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  long counter[CH_NKC] = {0};
};

}  // namespace

struct ch_handle {
  ch_grid grid;
  ch_params prm;
  int S = 1;                 // slabs in this process
  int nslabs_total = 1;
  std::vector<Slab> sl;
  int row0 = 0, nrows = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  KScal* sc = nullptr;       // device [NSC]
  KScal* sch = nullptr;      // pinned host [NSC]
  KScal* pollbuf = nullptr;  // pinned host [2]: pipelined CG convergence polls
  cudaEvent_t pollev[2] = {nullptr, nullptr};
  double* part = nullptr;
  unsigned int* ticket = nullptr;
  double* tot = nullptr;     // [nslabs_total * 8]
  double* tot_local = nullptr;
  ch_stats stats;
  std::string err;
  Timer tm;
  Comm* comm = nullptr;
  size_t arr_elems = 0;
  double* cgtab = nullptr;    // deferred-p/x CG coefficient tables, device [NSC][2][CGT]
  int cur_m = 0;              // block length of the solve in flight (0: cg_defer)
  int cg_defer = 64;          // block length m (2..64) of the deferred p/x CG (env CHB_DEFER);
                              // reduced at ch_create if the z history would not fit
  double* gm_dev = nullptr;   // GMRES dot results / coefficients (device, 192)
  double* gm_host = nullptr;  // pinned mirror (max(192, 72 * slabs) doubles)
  double* gm_red = nullptr;   // GMRES per-slab dot results, device [slabs + 1][72]
  int cg3 = 1;                // single-reduction CG: three-term z recurrence (env CHB_CG3)
  int strip2 = 0;             // rows per strip, 0 = one resident wave (env CHB_STRIP)
  int pdl = 1;                // programmatic dependent launch of the CG sweeps (env CHB_PDL)
  int ms = 1;                 // virtual slabs: one sweep launch over all slabs with in-kernel
                              // halo rows and cross-slab finalize (env CHB_MS=0: per-slab
                              // launches + halo copies + finalize kernel)
  int64_t tidx = 0;           // time index n of the state (ch_set_time_index; R23 start-up)
  // cross-rank / cross-slab combine of the multi-slab CG sweep (common.cuh XPeers)
  void* xr_mem = nullptr;     // this rank's totals area [2][XS_MAX][8] + flags [XR_MAX]
  XPeers* xp_dev = nullptr;   // device copy of the peer table
  unsigned epoch = 0;         // multi-slab sweep launches so far (same on every rank)
  int p2p = 0;                // ranks combine and exchange halo rows over NVLink peer memory
  double* nb_lo[A_N] = {};    // lower / upper neighbouring rank's boundary-slab arrays,
  double* nb_hi[A_N] = {};    // peer-mapped (ring arrays only; p2p)
  int nb_lo_j0 = 0, nb_hi_j0 = 0;
  std::vector<void*> ipc_open;  // peer mappings to close at ch_destroy
};

namespace {

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      h->err = std::string(#call) + ": " + cudaGetErrorName(e_) + " " +             \
               cudaGetErrorString(e_);                                               \
      return CH_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define TRY(x)               \
  do {                       \
    int s_ = (x);            \
    if (s_ != CH_OK) return s_; \
  } while (0)

// Parameters of the step at time index n: the CH and advection weights are 1
// during the backward-Euler start-up steps (R23).
Phys phys_at(const ch_params& p, int64_t n);

Phys phys(const ch_params& p) {
  Phys ph;
  ph.dt = p.dt; ph.Gamma1 = p.Gamma1; ph.Gamma2 = p.Gamma2; ph.Lambda = p.Lambda;
  ph.mu = p.mu; ph.Kc = p.Kc; ph.eps = p.eps; ph.A = p.A; ph.Ds = p.Ds;
  ph.Re_s = p.Re_s; ph.Re_n = p.Re_n; ph.rho_n = p.rho_n; ph.rho_s = p.rho_s;
  ph.lid_u = p.lid_u;
  ph.th_ch = p.theta_ch;
  ph.th_adv = p.theta_adv;
  ph.th_visc = p.theta_visc;
  return ph;
}

Phys phys_at(const ch_params& p, int64_t n) {
  Phys ph = phys(p);
  if (n < p.startup_be) ph.th_ch = ph.th_adv = 1.0;
  return ph;
}

StateP state(const Slab& s) {
  StateP p;
  p.phi = s.a[A_PHI]; p.phip = s.a[A_PHIP]; p.c = s.a[A_C];
  p.u = s.a[A_U]; p.v = s.a[A_V]; p.p = s.a[A_P];
  return p;
}

int check_launch(ch_handle* h, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->err = std::string("launch ") + what + ": " + cudaGetErrorName(e) + " " +
             cudaGetErrorString(e);
    return CH_ERR_CUDA;
  }
  return CH_OK;
}

// ------------------------------------------------------------- timing
cudaEvent_t ev_get(ch_handle* h) {
  if (!h->tm.pool.empty()) {
    cudaEvent_t e = h->tm.pool.back();
    h->tm.pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct KTime {
  ch_handle* h;
  int kc;
  long iter;
  double bytes;
  bool on = false;
  cudaEvent_t e0, e1;
  // bytes: algorithmic bytes of ONE slab launch; the timed region covers all slabs
  // count_only: launch accounting without events (the CG sweeps are timed in
  // groups by SweepTimer)
  KTime(ch_handle* hh, int k, double b, long it = -1, bool count_only = false)
      : h(hh), kc(k), iter(it), bytes(b * hh->S) {
    h->stats.launches += h->S;
    h->stats.kc_launches[kc] += h->S;
    if (!count_only && h->tm.stride > 0 && (h->tm.counter[kc]++ % h->tm.stride) == 0) {
      on = true;
      e0 = ev_get(h);
      e1 = ev_get(h);
      cudaEventRecord(e0, h->st);
    }
  }
  ~KTime() {
    if (on) {
      cudaEventRecord(e1, h->st);
      h->tm.pending.push_back({kc, iter, bytes, e0, e1, 1});
    }
  }
};

// CG sweeps are timed as groups of TGRP consecutive launches of one solve
// between ONE event pair: an event recorded between two sweeps keeps the
// second from starting under programmatic dependent launch, so a pair per
// launch times every sampled sweep without the overlap the chain runs with.
// A group never contains the deferred p/x launch or a convergence poll.
constexpr int TGRP = 8;
struct SweepTimer {
  ch_handle* h;
  int kc;
  int left = 0, n = 0;
  bool due = false;
  double bytes = 0.0;
  cudaEvent_t e0;
  SweepTimer(ch_handle* hh, int k) : h(hh), kc(k) {}
  // before sweep k (it-th of a chunk of `chunk` launches, p/x after every m-th)
  void before(long k, int it, int chunk, int m) {
    if (h->tm.stride <= 0 || left > 0) return;
    if ((h->tm.counter[kc]++ % h->tm.stride) == 0) due = true;
    const int G = m < TGRP ? m : TGRP;
    if (due && k > 0 && it + G <= chunk && (int)(k % m) + G <= m) {
      due = false;
      left = n = G;
      bytes = 0.0;
      e0 = ev_get(h);
      cudaEventRecord(e0, h->st);
    }
  }
  void after(long k, double b) {
    if (left == 0) return;
    bytes += b * h->S;
    if (--left == 0) {
      cudaEvent_t e1 = ev_get(h);
      cudaEventRecord(e1, h->st);
      h->tm.pending.push_back({kc, k + 1, bytes, e0, e1, n});
    }
  }
};

// Harvest timed launches.  Launches of Krylov iteration index > useful_iters
// (no-op launches after convergence) are discarded.
void harvest(ch_handle* h, long useful_iters) {
  for (auto& r : h->tm.pending) {
    if (r.iter < 0 || r.iter <= useful_iters) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, r.e0, r.e1) == cudaSuccess) {
        h->stats.kc_ms[r.kc] += ms;
        h->stats.kc_timed[r.kc] += r.n;
        h->stats.kc_bytes[r.kc] += r.bytes;
      }
    }
    h->tm.pool.push_back(r.e0);
    h->tm.pool.push_back(r.e1);
  }
  h->tm.pending.clear();
}

// ------------------------------------------------------ reductions / halos
RedArgs rargs(ch_handle* h, int fin, int sys, int slab) {
  RedArgs ra;
  ra.part = h->part;
  ra.ticket = h->ticket;
  ra.tot = h->tot_local;
  ra.sc = h->sc + sys;
  ra.fc.rtol2 = h->prm.rtol * h->prm.rtol;
  ra.fc.ncells = (double)h->grid.nx * (double)h->grid.ny;
  ra.fc.tab = h->cgtab ? h->cgtab + (size_t)sys * 2 * CGT : nullptr;
  ra.fc.m = h->cur_m > 0 ? h->cur_m : h->cg_defer;
  ra.fc.pad = 0;
  ra.fin = fin;
  ra.inline_fin = (h->nslabs_total == 1);
  ra.slab = slab;
  ra.pad = 0;
  ra.nbs = 0;
  ra.nslab = h->S;
  ra.ticket2 = h->ticket + MS_MAX;
  ra.xp = nullptr;
  ra.epoch = 0;
  ra.pad2 = 0;
  return ra;
}

// Combine slab totals (local slabs, then across ranks) and finalize.
int fin_slabs(ch_handle* h, int fin, int sys, int K) {
  if (h->nslabs_total == 1) return CH_OK;
  const double* tot = h->tot_local;
  if (h->comm) {
    if (comm_allgather(h->comm, h->tot_local, h->tot, h->S * 8, h->st) != 0) {
      h->err = "comm allgather failed";
      return CH_ERR_COMM;
    }
    tot = h->tot;
  }
  RedArgs ra = rargs(h, fin, sys, 0);
  launch_finalize_slabs(tot, h->nslabs_total, K, ra, h->st);
  h->stats.launches += 1;
  return check_launch(h, "finalize_slabs");
}

// Exchange `w` ghost rows of array `id` between the slabs of this process.
int halo_local(ch_handle* h, int id, int w) {
  for (int s = 0; s + 1 < h->S; ++s) {
    Slab& lo = h->sl[s];
    Slab& hi = h->sl[s + 1];
    const size_t pitch = lo.g.pitch;
    double* src = lo.a[id] + (size_t)(lo.g.nyl + GH - w) * pitch;
    double* dst = hi.a[id] + (size_t)(GH - w) * pitch;
    CK(cudaMemcpyAsync(dst, src, w * pitch * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    src = hi.a[id] + (size_t)GH * pitch;
    dst = lo.a[id] + (size_t)(lo.g.nyl + GH) * pitch;
    CK(cudaMemcpyAsync(dst, src, w * pitch * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
  }
  return CH_OK;
}

int halo(ch_handle* h, int id, int w);

// One CG iteration's communication: partial-sum combination (finalize) and
// the ghost rows of z' (2) and s (1; none for the three-term recurrence, sid < 0).
// Across processes the allgather and the halo rows go in ONE NCCL group.
int iter_exchange(ch_handle* h, int fin, int sys, int K, int zid, int sid) {
  if (h->nslabs_total == 1) return CH_OK;
  static int grouped = -1;  // env CHB_NCCL_GROUP=0: separate NCCL calls (safety valve)
  if (grouped < 0) {
    const char* e = getenv("CHB_NCCL_GROUP");
    grouped = e ? atoi(e) != 0 : 1;
  }
  if (!h->comm || !grouped) {
    TRY(fin_slabs(h, fin, sys, K));
    TRY(halo(h, zid, 2));
    return sid >= 0 ? halo(h, sid, 1) : CH_OK;
  }
  TRY(halo_local(h, zid, 2));
  if (sid >= 0) TRY(halo_local(h, sid, 1));
  const Slab& first = h->sl.front();
  const Slab& last = h->sl.back();
  HaloSpec hs[2] = {{first.a[zid], last.a[zid], last.g.nyl, 2},
                    {sid >= 0 ? first.a[sid] : nullptr, sid >= 0 ? last.a[sid] : nullptr,
                     last.g.nyl, 1}};
  if (comm_iter_exchange(h->comm, h->tot_local, h->tot, (size_t)h->S * 8, hs, sid >= 0 ? 2 : 1,
                         first.g.pitch, h->st) != 0) {
    h->err = "comm iteration exchange failed";
    return CH_ERR_COMM;
  }
  RedArgs ra = rargs(h, fin, sys, 0);
  launch_finalize_slabs(h->tot, h->nslabs_total, K, ra, h->st);
  h->stats.launches += 1;
  return check_launch(h, "finalize_slabs");
}

// Exchange `w` ghost rows of array `id` between neighbouring slabs.
int halo(ch_handle* h, int id, int w) {
  if (h->nslabs_total == 1) return CH_OK;
  for (int s = 0; s + 1 < h->S; ++s) {
    Slab& lo = h->sl[s];
    Slab& hi = h->sl[s + 1];
    const size_t pitch = lo.g.pitch;
    // lo's top rows -> hi's bottom ghost rows
    double* src = lo.a[id] + (size_t)(lo.g.nyl + GH - w) * pitch;
    double* dst = hi.a[id] + (size_t)(GH - w) * pitch;
    CK(cudaMemcpyAsync(dst, src, w * pitch * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    // hi's bottom rows -> lo's top ghost rows
    src = hi.a[id] + (size_t)GH * pitch;
    dst = lo.a[id] + (size_t)(lo.g.nyl + GH) * pitch;
    CK(cudaMemcpyAsync(dst, src, w * pitch * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
  }
  if (h->comm) {
    std::vector<double*> bufs(h->S);
    for (int s = 0; s < h->S; ++s) bufs[s] = h->sl[s].a[id];
    const Slab& first = h->sl.front();
    const Slab& last = h->sl.back();
    if (comm_halo(h->comm, first.a[id], first.g.nyl, last.a[id], last.g.nyl, first.g.pitch, w,
                  h->st) != 0) {
      h->err = "comm halo failed";
      return CH_ERR_COMM;
    }
  }
  return CH_OK;
}

int copy_arr(ch_handle* h, int src, int dst) {
  for (auto& s : h->sl)
    CK(cudaMemcpyAsync(s.a[dst], s.a[src], h->arr_elems * sizeof(double),
                       cudaMemcpyDeviceToDevice, h->st));
  return CH_OK;
}

int poll(ch_handle* h, int sys) {
  CK(cudaMemcpyAsync(h->sch + sys, h->sc + sys, sizeof(KScal), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int solve_status(ch_handle* h, int sys, const char* name) {
  const KScal& s = h->sch[sys];
  h->stats.iters_last[sys] = s.iter;
  h->stats.iters_total[sys] += s.iter;
  h->stats.resid_last[sys] = s.bb > 0 ? sqrt(s.rr / s.bb) : 0.0;
  if (s.status == KS_PEER_TIMEOUT) {
    char buf[200];
    snprintf(buf, sizeof buf, "%s: peer-memory combine timed out at iteration %d of step %lld "
             "(a rank's totals never arrived)", name, s.iter, (long long)h->tidx);
    h->err = buf;
    return CH_ERR_COMM;
  }
  if (s.status == 1 || s.status >= 3) {
    static const char* what[] = {
        "", "zero or non-finite inner product", "",
        "(r, z) <= 0 or non-finite (operator or preconditioner not SPD?)",
        "(A z, z) <= 0 or non-finite (operator not SPD?)",
        "CG step denominator delta - beta gamma/alpha <= 0",
        "three-term recurrence omega non-finite",
        "BiCGStab (r^, r) = 0 or non-finite",
        "BiCGStab (r^, v) = 0 or non-finite",
        "BiCGStab (t, t) = 0 or non-finite / omega = 0",
        "residual norm non-finite (NaN/Inf in the iterates)"};
    char buf[320];
    snprintf(buf, sizeof buf, "%s: Krylov breakdown at iteration %d of step %lld: %s "
             "[value %.6e, |r|^2 %.6e, |b|^2 %.6e]", name, s.iter, (long long)h->tidx,
             s.status <= 10 ? what[s.status] : "?", s.last, s.rr, s.bb);
    h->err = buf;
    return CH_ERR_BREAKDOWN;
  }
  if (s.status == 2) {
    char buf[160];
    snprintf(buf, sizeof buf, "%s: not converged in %d iterations (|r|/|b| = %.3e)", name,
             s.iter, h->stats.resid_last[sys]);
    h->err = buf;
    return CH_ERR_NOT_CONVERGED;
  }
  return CH_OK;
}

int set_maxit(ch_handle* h, int sys) {
  // maxit lives in the device scalars (read by the finalizers)
  int m = h->prm.maxit;
  CK(cudaMemcpyAsync(&h->sc[sys].maxit, &m, sizeof(int), cudaMemcpyHostToDevice, h->st));
  return CH_OK;
}

// ------------------------------------------------------------------- CG
OpDesc opdesc(ch_handle* h, int kind, const Slab& s) {
  OpDesc d;
  d.kind = kind;
  d.strip = 16;
  d.strip2 = h->strip2;
  d.pdl = h->pdl;
  d.a = nullptr;
  d.w = nullptr;
  d.s = 1.0;
  d.kscale = 1.0;
  d.ascal = 0.0;
  d.rho_n = h->prm.rho_n;
  d.rho_s = h->prm.rho_s;
  switch (kind) {
    case OPK_POISSON_CONST: d.s = 1.0 / h->prm.rho_s; break;
    case OPK_POISSON_VAR: d.w = s.a[A_PHI1]; break;
    case OPK_NUTRIENT: d.a = s.a[A_CA]; d.w = s.a[A_CW]; d.s = 0.5; d.kscale = h->prm.Ds; break;
    case OPK_MOM_U:
    case OPK_MOM_V:
      d.a = s.a[A_CA];
      d.w = s.a[A_CW];
      d.s = h->prm.theta_visc;
      if (h->prm.rho_n == h->prm.rho_s) {  // a = rho/dt is one number: no a[] stream
        d.kind = kind == OPK_MOM_U ? OPK_MOM_U_C : OPK_MOM_V_C;
        d.ascal = h->prm.rho_s / h->prm.dt;
      }
      break;
  }
  return d;
}

// ------------------------------------------- single-reduction CG (default)
// One fused sweep per iteration (kernels_cgs.cu).  Buffers: z ping-pong
// (A_Z, A_R), s ping-pong (A_RH, A_BP), p in place (A_PA) -- the BiCGStab
// work arrays are free while the symmetric systems are solved.
int cgs_solve(ch_handle* h, int sys, int kind, int xid, int bid, int nullspace, int use_shift,
              const char* name, int wid = -1) {
  TRY(set_maxit(h, sys));
  const int AM = (kind == OPK_NUTRIENT || kind == OPK_MOM_U || kind == OPK_MOM_V);
  if (wid >= 0) TRY(halo(h, wid, 2));
  if (AM) TRY(halo(h, A_CA, 1));
  TRY(halo(h, xid, 1));
  // z ring of m + 1 buffers (p/x deferred over blocks of m sweeps)
  const int m = h->cg_defer;
  const int NZ = m + 1;
  h->cur_m = m;
  int Zr[CGM + 1];
  Zr[0] = A_Z;
  Zr[1] = A_R;
  for (int k = 2; k < NZ; ++k) Zr[k] = A_ZH0 + (k - 2);
  const int S[2] = {A_RH, A_BP}, P = A_PA;
  const double cells = (double)h->grid.nx * (double)h->nrows / h->S;
  const int ekind = opdesc(h, kind, h->sl[0]).kind;  // kind the kernels run (bytes per cell)
  const double* tab = h->cgtab + (size_t)sys * 2 * CGT;
  auto px = [&](long k_last, int n, int write_p) -> int {
    // z_k of iterations k_last - n + 1 .. k_last
    const long k0 = k_last - n + 1;
    KTime kt(h, CH_KC_CG_PX, 8.0 * (n + 4) * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      ZList zl;
      for (int j = 0; j < CGM; ++j) zl.z[j] = j < n ? sl.a[Zr[(k0 + j) % NZ]] : nullptr;
      launch_cgs_px(sl.g, zl, n, k0 == 0, write_p, (int)(k_last + 1),
                    tab + ((k_last / m) & 1) * CGT, h->sc + sys, sl.a[P], sl.a[xid], h->st);
    }
    return check_launch(h, "cgs_px");
  };
  {
    KTime kt(h, CH_KC_CG_INIT, 40.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_cg5_init(opdesc(h, kind, sl), sl.g, sl.a[xid], sl.a[bid], use_shift, sl.a[Zr[0]],
                      rargs(h, FIN_CG_INIT, sys, s), h->st);
    }
  }
  TRY(check_launch(h, "cg5_init"));
  TRY(fin_slabs(h, FIN_CG_INIT, sys, 3));
  TRY(halo(h, Zr[0], 2));
  {
    KTime kt(h, CH_KC_CG_INIT, 16.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_cgs_delta0(opdesc(h, kind, sl), sl.g, sl.a[Zr[0]], rargs(h, FIN_CGS_D0, sys, s),
                        h->st);
    }
  }
  TRY(check_launch(h, "cgs_delta0"));
  TRY(fin_slabs(h, FIN_CGS_D0, sys, 1));
  const int kc_sys = sys == CH_SYS_U ? CH_KC_CG_FUSED_U
                   : sys == CH_SYS_V ? CH_KC_CG_FUSED_V
                   : sys == CH_SYS_P ? CH_KC_CG_FUSED_P : CH_KC_CG_FUSED;
  const int tt = h->cg3 && NZ >= 3;
  // one sweep launch over all local slabs with in-kernel halo rows and the
  // peer-memory combine: virtual slabs of one process, or ranks with P2P
  const bool ms_launch = h->ms && h->S <= MS_MAX && (h->p2p || (h->S > 1 && !h->comm));
  // neighbour array `id` of local slab s, offset to global rows (dir -1: below)
  auto nbp = [&](int s, int id, int dir) -> double* {
    const Slab& sl = h->sl[s];
    const double* base = nullptr;
    int j0 = 0;
    if (dir < 0 && s > 0) {
      base = h->sl[s - 1].a[id];
      j0 = h->sl[s - 1].g.j0;
    } else if (dir < 0 && h->p2p) {
      base = h->nb_lo[id];
      j0 = h->nb_lo_j0;
    } else if (dir > 0 && s + 1 < h->S) {
      base = h->sl[s + 1].a[id];
      j0 = h->sl[s + 1].g.j0;
    } else if (dir > 0 && h->p2p) {
      base = h->nb_hi[id];
      j0 = h->nb_hi_j0;
    }
    if (!base) return nullptr;
    return const_cast<double*>(base) + (long)(sl.g.j0 - j0) * (long)sl.g.pitch;
  };
  long k = 0;
  long npoll = 0;
  int chunk = 4;
  SweepTimer swt(h, kc_sys);
  for (;;) {
    for (int it = 0; it < chunk; ++it, ++k) {
      const int first = (k == 0), dir = (k & 1) ? -1 : 1;
      swt.before(k, it, chunk, m);
      const int zi = Zr[k % NZ], zo = Zr[(k + 1) % NZ];
      // three-term: the sweep reads z_{k-1} (still in the ring) instead of s_{k-1}
      // and writes no s
      const int si = tt ? Zr[(k + NZ - 1) % NZ] : S[(k + 1) & 1], so = tt ? -1 : S[k & 1];
      if (ms_launch) {
        // all local slabs in one launch: halo rows and the cross-slab finalize in-kernel
        MsArgs ma;
        memset(&ma, 0, sizeof ma);
        ma.S = h->S;
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          const OpDesc od = opdesc(h, kind, sl);
          ma.g[s] = sl.g;
          ma.zi[s] = sl.a[zi];
          ma.zo[s] = sl.a[zo];
          ma.si[s] = sl.a[si];
          ma.so[s] = so >= 0 ? sl.a[so] : nullptr;
          ma.w[s] = od.w;
          ma.a[s] = od.a;
          ma.zlo[s] = nbp(s, zo, -1);
          ma.zhi[s] = nbp(s, zo, 1);
          ma.slo[s] = so >= 0 ? nbp(s, so, -1) : nullptr;
          ma.shi[s] = so >= 0 ? nbp(s, so, 1) : nullptr;
        }
        ma.sysfence = h->p2p;
        RedArgs ra = rargs(h, FIN_CGS, sys, 0);
        ra.xp = h->xp_dev;
        ra.epoch = ++h->epoch;
        KTime kt(h, kc_sys, cgs_bytes(ekind, first, tt) * cells, k + 1, true);
        h->stats.launches -= h->S - 1;   // one launch for all slabs
        h->stats.kc_launches[kc_sys] -= h->S - 1;
        launch_cgs_iter_ms(opdesc(h, kind, h->sl[0]), ma, first, dir, tt, ra, h->st);
      } else {
        {
          KTime kt(h, kc_sys, cgs_bytes(ekind, first, tt) * cells, k + 1, true);
          for (int s = 0; s < h->S; ++s) {
            Slab& sl = h->sl[s];
            launch_cgs_iter(opdesc(h, kind, sl), sl.g, sl.a[zi], sl.a[zo], sl.a[si],
                            so >= 0 ? sl.a[so] : nullptr, first, dir, tt,
                            rargs(h, FIN_CGS, sys, s), h->st);
          }
        }
        TRY(iter_exchange(h, FIN_CGS, sys, 3, zo, so));
      }
      swt.after(k, cgs_bytes(ekind, first, tt) * cells);
      if ((k + 1) % m == 0) TRY(px(k, m, 1));
    }
    TRY(check_launch(h, "cgs iteration"));
    // pipelined convergence poll: this chunk's scalars go to a pinned slot
    // behind an event while the host waits only for the PREVIOUS chunk's --
    // the GPU always has the next chunk queued (after convergence the sweeps
    // of the chunk in flight exit on the device flag)
    const int slot = (int)(npoll & 1);
    CK(cudaMemcpyAsync(h->pollbuf + slot, h->sc + sys, sizeof(KScal), cudaMemcpyDeviceToHost,
                       h->st));
    CK(cudaEventRecord(h->pollev[slot], h->st));
    ++npoll;
    if (npoll >= 2) {
      CK(cudaEventSynchronize(h->pollev[slot ^ 1]));
      if (h->pollbuf[slot ^ 1].done) break;
    }
    if (chunk < 64) chunk *= 2;
  }
  TRY(poll(h, sys));
  const long K = h->sch[sys].iter;
  if (K > 0 && K % m != 0) TRY(px(K - 1, (int)(K % m), 0));
  {
    KTime kt(h, CH_KC_VEC, 24.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_cg5_finish(sl.g, sl.a[xid], sl.a[P], nullspace, 2,
                        rargs(h, FIN_MEAN, sys, s), h->st);
    }
  }
  TRY(check_launch(h, "cg5_finish"));
  if (nullspace) TRY(fin_slabs(h, FIN_MEAN, sys, 1));
  harvest(h, K);
  return solve_status(h, sys, name);
}

int cg_once(ch_handle* h, int sys, int kind, int xid, int bid, int nullspace, int use_shift,
            const char* name, int wid) {
  return cgs_solve(h, sys, kind, xid, bid, nullspace, use_shift, name, wid);
}

// CG with optional true-residual refinement (params.refine): each restart's
// initialisation computes b - A x from scratch, so a restart that reports 0
// iterations proves ||b - A x|| <= rtol ||b||.  Iterations of all passes are
// reported together.
int cg_any(ch_handle* h, int sys, int kind, int xid, int bid, int nullspace, int use_shift,
           const char* name, int wid = -1) {
  TRY(cg_once(h, sys, kind, xid, bid, nullspace, use_shift, name, wid));
  long total = h->sch[sys].iter;
  for (int pass = 0; pass < h->prm.refine && h->sch[sys].iter > 0; ++pass) {
    if (nullspace) {
      // the finish left mean(x) in the scalars: make x mean-free again and
      // restore the mean of b for the shifted initial residual
      for (auto& s : h->sl) launch_sub_mean(s.g, s.a[xid], h->sc + sys, h->st);
      for (int s = 0; s < h->S; ++s) {
        Slab& sl = h->sl[s];
        launch_sum(sl.g, sl.a[bid], rargs(h, FIN_MEAN, sys, s), h->st);
      }
      TRY(check_launch(h, "refine mean"));
      TRY(fin_slabs(h, FIN_MEAN, sys, 1));
    }
    h->stats.iters_total[sys] -= h->stats.iters_last[sys];  // re-counted below
    TRY(cg_once(h, sys, kind, xid, bid, nullspace, use_shift, name, wid));
    total += h->sch[sys].iter;
    h->stats.iters_total[sys] += total - h->sch[sys].iter;
    h->stats.iters_last[sys] = (int32_t)total;
  }
  return CH_OK;
}

// ------------------------------------------------------------ BiCGStab (CH)
ChCoef chcoef(ch_handle* h, const Slab& s, bool precond) {
  const Phys ph = phys_at(h->prm, h->tidx);
  ChCoef c;
  c.phis = s.a[A_PHIS];
  c.dinv = precond ? s.a[A_DINV] : nullptr;
  c.u = ph.th_adv != 0.0 ? s.a[A_U] : nullptr;
  c.v = s.a[A_V];
  c.dt = h->prm.dt;
  c.g1t = ph.th_ch * h->prm.Gamma1;
  c.Lambda = h->prm.Lambda;
  c.tha = ph.th_adv;
  c.strip = h->strip2;
  return c;
}

int bicgstab_solve(ch_handle* h, int sys, int xid, int bid) {
  TRY(set_maxit(h, sys));
  const double cells = (double)h->grid.nx * (double)h->nrows / h->S;
  TRY(halo(h, xid, 2));
  {
    KTime kt(h, CH_KC_CH_APPLY, 24.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_ch_apply(sl.g, chcoef(h, sl, false), sl.a[xid], sl.a[A_TMP], 0, nullptr, nullptr, 0,
                      0, rargs(h, FIN_NONE, sys, s), h->st);
    }
  }
  {
    KTime kt(h, CH_KC_VEC, 32.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_bi_init(sl.g, sl.a[A_TMP], sl.a[bid], sl.a[A_R], sl.a[A_RH],
                     rargs(h, FIN_BI_INIT, sys, s), h->st);
    }
  }
  TRY(fin_slabs(h, FIN_BI_INIT, sys, 2));
  TRY(check_launch(h, "bicgstab init"));
  long k = 1;
  int chunk = 2;
  for (;;) {
    for (int it = 0; it < chunk; ++it, ++k) {
      {
        KTime kt(h, CH_KC_VEC, 32.0 * cells, k);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          launch_bi_p(sl.g, sl.a[A_R], sl.a[A_BP], sl.a[A_BV], k == 1, h->sc + sys, h->st);
        }
      }
      TRY(halo(h, A_BP, 2));
      {
        KTime kt(h, CH_KC_CH_APPLY, 40.0 * cells, k);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          launch_ch_apply(sl.g, chcoef(h, sl, true), sl.a[A_BP], sl.a[A_BV], 1, sl.a[A_RH],
                          nullptr, 1, 0, rargs(h, FIN_BI_ALPHA, sys, s), h->st);
        }
      }
      TRY(fin_slabs(h, FIN_BI_ALPHA, sys, 1));
      {
        KTime kt(h, CH_KC_VEC, 24.0 * cells, k);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          launch_bi_s(sl.g, sl.a[A_R], sl.a[A_BV], sl.a[A_BS], rargs(h, FIN_BI_S, sys, s), h->st);
        }
      }
      TRY(fin_slabs(h, FIN_BI_S, sys, 1));
      TRY(halo(h, A_BS, 2));
      {
        KTime kt(h, CH_KC_CH_APPLY, 40.0 * cells, k);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          launch_ch_apply(sl.g, chcoef(h, sl, true), sl.a[A_BS], sl.a[A_BT], 2, sl.a[A_BS],
                          nullptr, 1, 1, rargs(h, FIN_BI_OMEGA, sys, s), h->st);
        }
      }
      TRY(fin_slabs(h, FIN_BI_OMEGA, sys, 2));
      {
        KTime kt(h, CH_KC_VEC, 64.0 * cells, k);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          launch_bi_xr(sl.g, sl.a[xid], sl.a[A_BP], sl.a[A_BS], sl.a[A_BT], sl.a[A_R],
                       sl.a[A_RH], sl.a[A_DINV], rargs(h, FIN_BI_R, sys, s), h->st);
        }
      }
      TRY(fin_slabs(h, FIN_BI_R, sys, 2));
    }
    TRY(check_launch(h, "bicgstab iteration"));
    TRY(poll(h, sys));
    if (h->sch[sys].done) break;
    if (chunk < 32) chunk *= 2;
  }
  if (h->sch[sys].zero) {
    for (auto& s : h->sl) CK(cudaMemsetAsync(s.a[xid], 0, h->arr_elems * sizeof(double), h->st));
  }
  harvest(h, h->sch[sys].iter);
  return solve_status(h, sys, "cahn-hilliard");
}

int gmres_solve(ch_handle* h, int sys, int xid, int bid);  // below

int bicgstab_or_gmres(ch_handle* h, int xid, int bid) {
  if (h->prm.ch_solver == CH_SOLVER_GMRES) return gmres_solve(h, CH_SYS_CH, xid, bid);
  return bicgstab_solve(h, CH_SYS_CH, xid, bid);
}

// ------------------------------------------------------------- one step
int step_once(ch_handle* h) {
  const Phys ph = phys_at(h->prm, h->tidx);
  const double cells = (double)h->grid.nx * (double)h->nrows / h->S;
  // 1. Cahn-Hilliard
  TRY(halo(h, A_PHI, 2));
  TRY(halo(h, A_PHIP, 2));
  TRY(halo(h, A_U, 1));
  TRY(halo(h, A_V, 1));
  TRY(halo(h, A_C, 1));
  {
    KTime kt(h, CH_KC_RHS, 72.0 * cells);
    for (auto& s : h->sl) launch_ch_rhs(s.g, ph, state(s), s.a[A_PHIS], s.a[A_DINV], s.a[A_B], h->st);
  }
  TRY(check_launch(h, "ch_rhs"));
  TRY(halo(h, A_PHIS, 2));
  TRY(halo(h, A_DINV, 2));
  TRY(copy_arr(h, A_PHIS, A_PHI1));
  TRY(bicgstab_or_gmres(h, A_PHI1, A_B));
  // 2. nutrient
  TRY(halo(h, A_PHI1, 1));
  {
    KTime kt(h, CH_KC_RHS, 64.0 * cells);
    for (auto& s : h->sl)
      launch_nut_rhs(s.g, ph, state(s), s.a[A_PHI1], s.a[A_CA], s.a[A_CW], s.a[A_B], h->st);
  }
  TRY(check_launch(h, "nut_rhs"));
  TRY(copy_arr(h, A_C, A_C1));
  TRY(cg_any(h, CH_SYS_NUTRIENT, OPK_NUTRIENT, A_C1, A_B, 0, 0, "nutrient", A_CW));
  // 3. intermediate velocity
  {
    KTime kt(h, CH_KC_RHS, 40.0 * cells);
    for (auto& s : h->sl)
      launch_mom_rhs_u(s.g, ph, state(s), s.a[A_PHIS], s.a[A_CA], s.a[A_CW], s.a[A_B], h->st);
  }
  TRY(check_launch(h, "mom_rhs_u"));
  TRY(copy_arr(h, A_USG, A_US));  // initial guess u* of the previous step (R25)
  TRY(cg_any(h, CH_SYS_U, OPK_MOM_U, A_US, A_B, 0, 0, "momentum-u", A_CW));
  {
    KTime kt(h, CH_KC_RHS, 40.0 * cells);
    for (auto& s : h->sl)
      launch_mom_rhs_v(s.g, ph, state(s), s.a[A_PHIS], s.a[A_CA], s.a[A_CW], s.a[A_B], h->st);
  }
  TRY(check_launch(h, "mom_rhs_v"));
  TRY(copy_arr(h, A_VSG, A_VS));
  TRY(cg_any(h, CH_SYS_V, OPK_MOM_V, A_VS, A_B, 0, 0, "momentum-v", A_CW));
  // 4. pressure Poisson with the constant null space
  TRY(halo(h, A_US, 1));
  TRY(halo(h, A_VS, 1));
  {
    KTime kt(h, CH_KC_RHS, 24.0 * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_div(sl.g, sl.a[A_US], sl.a[A_VS], sl.a[A_B], rargs(h, FIN_MEAN, CH_SYS_P, s), h->st);
    }
  }
  TRY(check_launch(h, "div"));
  TRY(fin_slabs(h, FIN_MEAN, CH_SYS_P, 1));
  const int pk = (h->prm.rho_n == h->prm.rho_s) ? OPK_POISSON_CONST : OPK_POISSON_VAR;
  // p^{n+1} into a work array (initial guess p^n), so that a failed solve leaves p^n
  TRY(copy_arr(h, A_P, A_TMP2));
  TRY(cg_any(h, CH_SYS_P, pk, A_TMP2, A_B, 1, 1, "pressure",
             pk == OPK_POISSON_VAR ? A_PHI1 : -1));
  {
    KTime kt(h, CH_KC_VEC, 16.0 * cells);
    for (auto& s : h->sl) launch_sub_mean(s.g, s.a[A_TMP2], h->sc + CH_SYS_P, h->st);
  }
  // 5. projection (every solve has succeeded: the state is updated from here on)
  TRY(halo(h, A_TMP2, 1));
  {
    KTime kt(h, CH_KC_RHS, 56.0 * cells);
    for (auto& s : h->sl)
      launch_project(s.g, ph, s.a[A_PHI1], s.a[A_US], s.a[A_VS], s.a[A_TMP2], s.a[A_U], s.a[A_V],
                     h->st);
  }
  TRY(check_launch(h, "project"));
  // rotate time levels
  for (auto& s : h->sl) {
    std::swap(s.a[A_PHIP], s.a[A_PHI]);   // phi_prev <- phi^n
    std::swap(s.a[A_PHI], s.a[A_PHI1]);   // phi <- phi^{n+1}
    std::swap(s.a[A_C], s.a[A_C1]);
    std::swap(s.a[A_P], s.a[A_TMP2]);     // p <- p^{n+1}
    std::swap(s.a[A_USG], s.a[A_US]);     // next step's momentum guesses <- u*, v* (R25)
    std::swap(s.a[A_VSG], s.a[A_VS]);
  }
  harvest(h, -1);
  h->stats.steps += 1;
  h->tidx += 1;
  return CH_OK;
}

// ------------------------------------------------------------ field copies
int field_arr(int field) {
  switch (field) {
    case CH_FIELD_PHI: return A_PHI;
    case CH_FIELD_PHI_PREV: return A_PHIP;
    case CH_FIELD_C: return A_C;
    case CH_FIELD_U: return A_U;
    case CH_FIELD_V: return A_V;
    case CH_FIELD_P: return A_P;
    case CH_FIELD_U_STAR: return A_USG;
    case CH_FIELD_V_STAR: return A_VSG;
  }
  return -1;
}

// Copy a user (nrows x nx, ld = nx) array into internal array `id` of all slabs.
int put(ch_handle* h, int id, const double* src, int where) {
  const cudaMemcpyKind k = where == CH_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  for (auto& s : h->sl) {
    const double* sp = src + (size_t)(s.g.j0 - h->row0) * h->grid.nx;
    double* dp = s.a[id] + (size_t)GH * s.g.pitch;
    CK(cudaMemcpy2DAsync(dp, s.g.pitch * sizeof(double), sp, h->grid.nx * sizeof(double),
                         h->grid.nx * sizeof(double), s.g.nyl, k, h->st));
  }
  if (where != CH_DEVICE) CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int get(ch_handle* h, int id, double* dst, int where) {
  const cudaMemcpyKind k = where == CH_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  for (auto& s : h->sl) {
    double* dp = dst + (size_t)(s.g.j0 - h->row0) * h->grid.nx;
    const double* sp = s.a[id] + (size_t)GH * s.g.pitch;
    CK(cudaMemcpy2DAsync(dp, h->grid.nx * sizeof(double), sp, s.g.pitch * sizeof(double),
                         h->grid.nx * sizeof(double), s.g.nyl, k, h->st));
  }
  if (where != CH_DEVICE) CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int zero_vrow0(ch_handle* h, int id = A_V) {
  if (h->row0 == 0) {
    Slab& s = h->sl.front();
    CK(cudaMemsetAsync(s.a[id] + (size_t)GH * s.g.pitch, 0, s.g.pitch * sizeof(double), h->st));
  }
  return CH_OK;
}

}  // namespace

// ======================================================================
// GMRES(m) with right Jacobi preconditioning (PAPER.md:238 KSPGMRES +
// PCJACOBI).  Arnoldi by classical Gram-Schmidt with one
// re-orthogonalisation (CGS2): every basis vector is read twice per step in
// fused multi-dot / multi-axpy sweeps instead of j+1 dependent passes.  The
// (m+1) x m Hessenberg least-squares problem (Givens rotations) is tiny and
// runs on the host from the reduced coefficients.
namespace {

int gm_dots(ch_handle* h, int k, int wvec, std::vector<double>& out) {
  // out[i] = (V_i, V_wvec) for i < k, summed over slabs in slab order, then over
  // ranks by one in-place device allreduce of all k values (one host round trip)
  out.assign(k, 0.0);
  for (int s = 0; s < h->S; ++s) {
    Slab& sl = h->sl[s];
    launch_gm_dots(sl.g, sl.V.data(), k, sl.V[wvec], h->gm_red + (size_t)s * 72, h->part,
                   h->ticket, h->st);
  }
  h->stats.launches += h->S;
  h->stats.kc_launches[CH_KC_GMRES] += h->S;
  TRY(check_launch(h, "gm_dots"));
  CK(cudaMemcpyAsync(h->gm_host, h->gm_red, (size_t)h->S * 72 * sizeof(double),
                     cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  for (int s = 0; s < h->S; ++s)
    for (int i = 0; i < k; ++i) out[i] += h->gm_host[(size_t)s * 72 + i];
  if (h->comm) {
    for (int i = 0; i < k; ++i) h->gm_host[i] = out[i];
    CK(cudaMemcpyAsync(h->gm_red, h->gm_host, k * sizeof(double), cudaMemcpyHostToDevice, h->st));
    double* sum = h->gm_red + (size_t)h->S * 72;  // distinct receive buffer
    if (comm_allreduce_sum(h->comm, h->gm_red, sum, (size_t)k, h->st) != 0) {
      h->err = "gmres: allreduce of the Gram-Schmidt dots failed";
      return CH_ERR_COMM;
    }
    CK(cudaMemcpyAsync(h->gm_host, sum, k * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    for (int i = 0; i < k; ++i) out[i] = h->gm_host[i];
  }
  return CH_OK;
}

int gm_set_coef(ch_handle* h, const double* v, int k) {
  CK(cudaMemcpyAsync(h->gm_dev + 96, v, k * sizeof(double), cudaMemcpyHostToDevice, h->st));
  return CH_OK;
}

int gmres_solve(ch_handle* h, int sys, int xid, int bid) {
  const int m = std::max(1, std::min(64, (int)h->prm.gmres_restart));
  const double cells = (double)h->grid.nx * (double)h->nrows / h->S;
  for (auto& s : h->sl)
    while ((int)s.V.size() < m + 1) {
      double* p = nullptr;
      CK(cudaMalloc(&p, h->arr_elems * sizeof(double)));
      CK(cudaMemsetAsync(p, 0, h->arr_elems * sizeof(double), h->st));
      s.V.push_back(p);
    }
  KScal& hs = h->sch[sys];
  memset(&hs, 0, sizeof(KScal));
  // ||b||^2: stage b in V[0]
  for (auto& s : h->sl)
    CK(cudaMemcpyAsync(s.V[0], s.a[bid], h->arr_elems * sizeof(double), cudaMemcpyDeviceToDevice,
                       h->st));
  std::vector<double> t;
  TRY(gm_dots(h, 1, 0, t));
  hs.bb = t[0];
  if (hs.bb == 0.0) {
    for (auto& s : h->sl) CK(cudaMemsetAsync(s.a[xid], 0, h->arr_elems * sizeof(double), h->st));
    return solve_status(h, sys, "cahn-hilliard (gmres)");
  }
  const double tol = h->prm.rtol * sqrt(hs.bb);
  long total = 0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gv(m + 1), y(m);
  for (;;) {
    // V0 = b - A x
    TRY(halo(h, xid, 2));
    {
      KTime kt(h, CH_KC_CH_APPLY, 24.0 * cells);
      for (int s = 0; s < h->S; ++s) {
        Slab& sl = h->sl[s];
        launch_ch_apply(sl.g, chcoef(h, sl, false), sl.a[xid], sl.a[A_TMP], 0, nullptr, nullptr,
                        0, 0, rargs(h, FIN_NONE, sys, s), h->st);
        launch_gm_residual(sl.g, sl.a[A_TMP], sl.a[bid], sl.V[0], h->st);
      }
    }
    TRY(check_launch(h, "gmres residual"));
    TRY(gm_dots(h, 1, 0, t));
    const double beta = sqrt(t[0]);
    if (beta <= tol) {
      hs.rr = t[0];
      break;
    }
    const double ib = 1.0 / beta;
    TRY(gm_set_coef(h, &ib, 1));
    for (auto& s : h->sl) launch_gm_scale(s.g, s.V[0], h->gm_dev + 96, h->st);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int k = 0;
    bool conv = false;
    for (int j = 0; j < m; ++j) {
      total++;
      // w = A D^{-1} V_j -> V_{j+1}   (multi-slab: V_j staged in TMP2 for its halo)
      if (h->nslabs_total > 1) {
        for (auto& s : h->sl)
          CK(cudaMemcpyAsync(s.a[A_TMP2], s.V[j], h->arr_elems * sizeof(double),
                             cudaMemcpyDeviceToDevice, h->st));
        TRY(halo(h, A_TMP2, 2));
      }
      {
        KTime kt(h, CH_KC_CH_APPLY, 32.0 * cells, total);
        for (int s = 0; s < h->S; ++s) {
          Slab& sl = h->sl[s];
          const double* src = h->nslabs_total > 1 ? sl.a[A_TMP2] : sl.V[j];
          launch_ch_apply(sl.g, chcoef(h, sl, true), src, sl.V[j + 1], 0, nullptr, nullptr, 0, 0,
                          rargs(h, FIN_NONE, sys, s), h->st);
        }
      }
      // CGS2: h = V^T w; w -= V h; twice
      std::vector<double> hc(j + 1, 0.0), hp;
      for (int pass = 0; pass < 2; ++pass) {
        TRY(gm_dots(h, j + 1, j + 1, hp));
        TRY(gm_set_coef(h, hp.data(), j + 1));
        {
          KTime kt(h, CH_KC_GMRES, 8.0 * (j + 3) * cells, total);
          for (auto& s : h->sl)
            launch_gm_axpy_multi(s.g, s.V.data(), j + 1, h->gm_dev + 96, s.V[j + 1], h->st);
        }
        for (int i = 0; i <= j; ++i) hc[i] += hp[i];
      }
      // ||w||: self dot of V_{j+1}
      {
        std::vector<double> all;
        // (V_i, V_{j+1}) for i <= j+1, last entry is the squared norm
        TRY(gm_dots(h, j + 2, j + 1, all));
        H[(size_t)(j + 1) * m + j] = sqrt(all[j + 1]);
      }
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hc[i];
      const double hn = H[(size_t)(j + 1) * m + j];
      if (hn != 0.0) {
        const double ihn = 1.0 / hn;
        TRY(gm_set_coef(h, &ihn, 1));
        for (auto& s : h->sl) launch_gm_scale(s.g, s.V[j + 1], h->gm_dev + 96, h->st);
      }
      for (int i = 0; i < j; ++i) {
        const double a0 = H[(size_t)i * m + j], a1 = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a0 + sn[i] * a1;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a0 + cs[i] * a1;
      }
      const double den = hypot(H[(size_t)j * m + j], hn);
      cs[j] = H[(size_t)j * m + j] / den;
      sn[j] = hn / den;
      H[(size_t)j * m + j] = den;
      H[(size_t)(j + 1) * m + j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      k = j + 1;
      if (fabs(gv[j + 1]) <= tol || total >= h->prm.maxit) {
        conv = fabs(gv[j + 1]) <= tol;
        break;
      }
    }
    for (int i = k - 1; i >= 0; --i) {
      double acc = gv[i];
      for (int l = i + 1; l < k; ++l) acc -= H[(size_t)i * m + l] * y[l];
      y[i] = acc / H[(size_t)i * m + i];
    }
    TRY(gm_set_coef(h, y.data(), k));
    {
      KTime kt(h, CH_KC_GMRES, 8.0 * (k + 3) * cells);
      for (auto& s : h->sl)
        launch_gm_update_x(s.g, s.V.data(), k, h->gm_dev + 96, s.a[A_DINV], s.a[xid], h->st);
    }
    TRY(check_launch(h, "gmres update"));
    hs.rr = gv[k] * gv[k];
    if (conv) break;
    if (total >= h->prm.maxit) {
      hs.status = 2;
      break;
    }
  }
  hs.iter = (int)total;
  CK(cudaStreamSynchronize(h->st));
  harvest(h, -1);
  return solve_status(h, sys, "cahn-hilliard (gmres)");
}

}  // namespace

// ======================================================================
// C ABI
extern "C" {

int ch_abi_version(void) { return CH_ABI_VERSION; }

// Host-only: the slab decomposition ch_create uses (balanced split of ny over
// nranks * virtual_slabs slabs, the first ny % total one row taller).
int ch_partition(int32_t ny, int32_t nranks, int32_t rank, int32_t virtual_slabs, int32_t* row0,
                 int32_t* nrows) {
  const int S = virtual_slabs < 1 ? 1 : virtual_slabs;
  if (ny < 4 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !nrows) return CH_ERR_ARG;
  const int total = nranks * S;
  if (ny < 2 * total) return CH_ERR_ARG;
  const int base = ny / total, rem = ny % total;
  auto slab_row0 = [&](int k) { return k * base + std::min(k, rem); };
  *row0 = slab_row0(rank * S);
  *nrows = slab_row0(rank * S + S) - *row0;
  return CH_OK;
}

const char* ch_last_error(const ch_handle* h) { return h ? h->err.c_str() : "null handle"; }

static void destroy_mem(ch_handle* h) {
  for (auto& s : h->sl) {
    for (void* p : s.bases) cudaFree(p);
    for (double* p : s.V) cudaFree(p);
  }
  h->sl.clear();
  if (h->sc) cudaFree(h->sc);
  if (h->sch) cudaFreeHost(h->sch);
  if (h->pollbuf) cudaFreeHost(h->pollbuf);
  for (auto& e : h->pollev)
    if (e) cudaEventDestroy(e);
  if (h->part) cudaFree(h->part);
  if (h->ticket) cudaFree(h->ticket);
  if (h->tot) cudaFree(h->tot);
  if (h->tot_local) cudaFree(h->tot_local);
  if (h->gm_dev) cudaFree(h->gm_dev);
  if (h->gm_red) cudaFree(h->gm_red);
  if (h->cgtab) cudaFree(h->cgtab);
  if (h->gm_host) cudaFreeHost(h->gm_host);
  for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
  h->ipc_open.clear();
  if (h->xr_mem) cudaFree(h->xr_mem);
  if (h->xp_dev) cudaFree(h->xp_dev);
  for (auto& r : h->tm.pending) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  for (auto e : h->tm.pool) cudaEventDestroy(e);
  h->tm.pending.clear();
  h->tm.pool.clear();
}

}  // extern "C"

namespace {

// The arrays of the CG z ring (and s ping-pong) in a fixed order, the same on
// every rank: the peer-mapped sweep stores its edge rows of z' into these.
constexpr int NRING_MAX = 4 + CGM - 1;
int ring_ids(const ch_handle* h, int* ids) {
  int n = 0;
  ids[n++] = A_Z;
  ids[n++] = A_R;
  ids[n++] = A_RH;
  ids[n++] = A_BP;
  for (int k = 0; k + 1 < h->cg_defer; ++k) ids[n++] = A_ZH0 + k;
  return n;
}

struct PeerInfo {
  int32_t pid, cg_defer, S, nring;
  int32_t j0_first, j0_last, ok, pad;
  char bus[16];                              // PCI bus id of the rank's device
  cudaIpcMemHandle_t xr;                     // totals area + flags
  cudaIpcMemHandle_t first[NRING_MAX], last[NRING_MAX];  // ring arrays, first / last slab
};

// After the NCCL clique exists: agree on the deferred-p/x block length (the
// z ring must index the same arrays on every rank), then try to map the
// neighbours' ring arrays and every rank's totals area through CUDA IPC
// (NVLink peer memory).  P2P is used only if every rank is a separate process
// on its own device with peer access to all the others (never two ranks on
// one GPU: their sweeps wait on one another) and CHB_P2P is not 0; otherwise
// the per-iteration NCCL group stays in use.
int peer_setup(ch_handle* h) {
  const int R = h->grid.nranks, me = h->grid.rank, S = h->S;
  CK(cudaSetDevice(h->grid.device));
  PeerInfo mine;
  memset(&mine, 0, sizeof mine);
  mine.pid = (int32_t)getpid();
  mine.cg_defer = h->cg_defer;
  mine.S = S;
  int ids[NRING_MAX];
  mine.nring = ring_ids(h, ids);
  mine.j0_first = h->sl.front().g.j0;
  mine.j0_last = h->sl.back().g.j0;
  int ok = 1;
  if (const char* e = getenv("CHB_P2P")) ok = atoi(e) != 0;
  if (R > XR_MAX || R * S > XS_MAX || S > MS_MAX || !h->ms) ok = 0;
  if (cudaDeviceGetPCIBusId(mine.bus, sizeof mine.bus, h->grid.device) != cudaSuccess) ok = 0;
  if (ok && cudaIpcGetMemHandle(&mine.xr, h->xr_mem) != cudaSuccess) ok = 0;
  for (int i = 0; ok && i < mine.nring; ++i)
    if (cudaIpcGetMemHandle(&mine.first[i], h->sl.front().a[ids[i]]) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.last[i], h->sl.back().a[ids[i]]) != cudaSuccess)
      ok = 0;
  cudaGetLastError();  // an IPC refusal is not a CUDA error of the step
  std::vector<PeerInfo> all(R);
  if (comm_allgather_host(h->comm, &mine, all.data(), sizeof(PeerInfo), h->st) != 0) {
    h->err = "peer setup: allgather failed";
    return CH_ERR_COMM;
  }
  for (const PeerInfo& q : all) h->cg_defer = std::min(h->cg_defer, (int)q.cg_defer);
  // local verdict: distinct processes on distinct devices with peer access
  for (int q = 0; q < R && ok; ++q) {
    if (q == me) continue;
    int dq = -1, can = 0;
    if (all[q].pid == mine.pid) ok = 0;
    if (ok && cudaDeviceGetByPCIBusId(&dq, all[q].bus) != cudaSuccess) ok = 0;
    if (ok && dq == h->grid.device) ok = 0;
    if (ok && (cudaDeviceCanAccessPeer(&can, h->grid.device, dq) != cudaSuccess || !can)) ok = 0;
  }
  cudaGetLastError();
  auto agree = [&](int v, int* all_ok) -> int {
    std::vector<int32_t> flags(R);
    int32_t x = v;
    if (comm_allgather_host(h->comm, &x, flags.data(), sizeof x, h->st) != 0) return CH_ERR_COMM;
    *all_ok = 1;
    for (int32_t f : flags) *all_ok &= f != 0;
    return CH_OK;
  };
  int all_ok = 0;
  if (agree(ok && mine.pid != 0, &all_ok) != CH_OK) {
    h->err = "peer setup: allgather failed";
    return CH_ERR_COMM;
  }
  if (!all_ok) return CH_OK;  // NCCL halos and allgather per iteration
  // map: every rank's totals area, the neighbours' boundary-slab ring arrays
  XPeers xp;
  memset(&xp, 0, sizeof xp);
  xp.R = R;
  xp.rank = me;
  xp.slab0 = me * S;
  xp.nslab_all = R * S;
  auto open = [&](const cudaIpcMemHandle_t& hd) -> void* {
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    h->ipc_open.push_back(p);
    return p;
  };
  int mapped = 1;
  for (int q = 0; q < R && mapped; ++q) {
    char* base = q == me ? static_cast<char*>(h->xr_mem) : static_cast<char*>(open(all[q].xr));
    if (!base) {
      mapped = 0;
      break;
    }
    xp.tot[q] = reinterpret_cast<double*>(base);
    xp.flag[q] = reinterpret_cast<unsigned*>(base + XR_TOT_BYTES);
  }
  const int nr = ring_ids(h, ids);  // the agreed block length
  for (int i = 0; i < nr && mapped; ++i) {
    if (me > 0) {
      h->nb_lo[ids[i]] = static_cast<double*>(open(all[me - 1].last[i]));
      mapped &= h->nb_lo[ids[i]] != nullptr;
    }
    if (me + 1 < R) {
      h->nb_hi[ids[i]] = static_cast<double*>(open(all[me + 1].first[i]));
      mapped &= h->nb_hi[ids[i]] != nullptr;
    }
  }
  if (me > 0) h->nb_lo_j0 = all[me - 1].j0_last;
  if (me + 1 < R) h->nb_hi_j0 = all[me + 1].j0_first;
  CK(cudaMemsetAsync(h->xr_mem, 0, XR_BYTES, h->st));
  h->epoch = 0;
  if (agree(mapped, &all_ok) != CH_OK) {
    h->err = "peer setup: allgather failed";
    return CH_ERR_COMM;
  }
  if (!all_ok) {
    for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
    h->ipc_open.clear();
    for (int i = 0; i < A_N; ++i) h->nb_lo[i] = h->nb_hi[i] = nullptr;
    cudaGetLastError();
    return CH_OK;
  }
  CK(cudaMemcpy(h->xp_dev, &xp, sizeof xp, cudaMemcpyHostToDevice));
  // probe the mapped clique with the stores and the combine of one sweep:
  // edge rows of A_Z into the neighbours' ghost rows, one cross-rank combine
  // (epoch 1); a rank whose ghost rows or sums come out wrong votes NCCL
  {
    const Slab& f = h->sl.front();
    const Slab& l = h->sl.back();
    const long P = f.g.pitch;
    double* lo = me > 0 ? h->nb_lo[A_Z] + (long)(f.g.j0 - h->nb_lo_j0) * P : nullptr;
    double* hi = me + 1 < R ? h->nb_hi[A_Z] + (long)(l.g.j0 - h->nb_hi_j0) * P : nullptr;
    h->epoch = 1;
    launch_peer_probe(h->xp_dev, h->epoch, h->tot_local, S, f.g, lo, l.g, hi, h->gm_dev, h->st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
    int ok_probe = 1;
    double sums[3];
    CK(cudaMemcpy(sums, h->gm_dev, sizeof sums, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 3; ++k) {
      double want = 0.0;
      for (int q = 0; q < R; ++q)
        for (int sl = 0; sl < S; ++sl) want += (q + 1.0) * (k + 1.0);
      ok_probe &= sums[k] == want;
    }
    std::vector<double> row((size_t)f.g.nx);
    auto check_rows = [&](const Slab& sb, int gq0) {
      for (int gq = gq0; gq < gq0 + 2; ++gq) {
        const double* src = sb.a[A_Z] + (size_t)(gq - sb.g.j0 + GH) * P;
        if (cudaMemcpy(row.data(), src, row.size() * sizeof(double), cudaMemcpyDeviceToHost) !=
            cudaSuccess)
          return 0;
        for (int c = 0; c < sb.g.nx; ++c)
          if (row[c] != gq * 1e6 + c + 0.25) return 0;
      }
      return 1;
    };
    if (me > 0) ok_probe &= check_rows(f, f.g.j0 - 2);
    if (me + 1 < R) ok_probe &= check_rows(l, l.g.j0 + l.g.nyl);
    if (agree(ok_probe, &all_ok) != CH_OK) {
      h->err = "peer setup: allgather failed";
      return CH_ERR_COMM;
    }
    for (auto& sb : h->sl) CK(cudaMemsetAsync(sb.a[A_Z], 0, h->arr_elems * sizeof(double), h->st));
    if (!all_ok) {
      fprintf(stderr, "ch_comm_init: peer-memory probe failed on some rank; using NCCL\n");
      for (void* q : h->ipc_open) cudaIpcCloseMemHandle(q);
      h->ipc_open.clear();
      for (int i = 0; i < A_N; ++i) h->nb_lo[i] = h->nb_hi[i] = nullptr;
      cudaGetLastError();
      return CH_OK;
    }
  }
  h->p2p = 1;
  return CH_OK;
}

}  // namespace

extern "C" {

ch_handle* ch_create(const ch_grid* grid, const ch_params* params, int* status) {
  auto fail = [&](int code, ch_handle* h, const char* msg) -> ch_handle* {
    if (status) *status = code;
    if (h) {
      fprintf(stderr, "ch_create: %s %s\n", msg, h->err.c_str());
      destroy_mem(h);
      delete h;
    } else {
      fprintf(stderr, "ch_create: %s\n", msg);
    }
    return nullptr;
  };
  if (!grid || !params) return fail(CH_ERR_ARG, nullptr, "null argument");
  const ch_grid G = *grid;
  if (G.nx < 4 || G.ny < 4 || (G.nx & 1) || G.nranks < 1 || G.rank < 0 || G.rank >= G.nranks)
    return fail(CH_ERR_ARG, nullptr, "bad grid (need even nx >= 4, ny >= 4, 0 <= rank < nranks)");
  const int S = G.virtual_slabs < 1 ? 1 : G.virtual_slabs;
  const int total = G.nranks * S;
  if (G.ny < 2 * total) return fail(CH_ERR_ARG, nullptr, "too many slabs for ny (>= 2 rows each)");
  if (!(params->dt > 0) || !(params->rtol > 0) || params->maxit < 1)
    return fail(CH_ERR_ARG, nullptr, "bad params (dt > 0, rtol > 0, maxit >= 1)");
  if (!(params->theta_ch >= 0 && params->theta_ch <= 1) ||
      !(params->theta_adv >= 0 && params->theta_adv <= 1) ||
      !(params->theta_visc > 0 && params->theta_visc <= 1) || params->startup_be < 0)
    return fail(CH_ERR_ARG, nullptr,
                "bad params (theta_ch, theta_adv in [0,1], theta_visc in (0,1], startup_be >= 0)");
  if (cudaSetDevice(G.device) != cudaSuccess) return fail(CH_ERR_CUDA, nullptr, "cudaSetDevice");
  ch_handle* h = new ch_handle();
  h->grid = G;
  h->prm = *params;
  h->S = S;
  h->nslabs_total = total;
  if (const char* e = getenv("CHB_CG3")) h->cg3 = atoi(e) != 0;
  if (const char* e = getenv("CHB_STRIP")) h->strip2 = std::max(0, atoi(e));
  if (const char* e = getenv("CHB_PDL")) h->pdl = atoi(e) != 0;
  if (const char* e = getenv("CHB_MS")) h->ms = atoi(e) != 0;
  if (const char* e = getenv("CHB_DEFER")) h->cg_defer = std::min(std::max(2, atoi(e)), CGM);
  memset(&h->stats, 0, sizeof(ch_stats));
  // rows: balanced split of ny over `total` slabs (first ny % total get one more)
  const int base = G.ny / total, rem = G.ny % total;
  auto slab_row0 = [&](int k) { return k * base + std::min(k, rem); };
  const int pitch = ((G.nx + 31) / 32) * 32;
  h->row0 = slab_row0(G.rank * S);
  h->nrows = slab_row0(G.rank * S + S) - h->row0;
  int maxrows = 0;
  for (int s = 0; s < S; ++s) {
    const int k = G.rank * S + s;
    maxrows = std::max(maxrows, slab_row0(k + 1) - slab_row0(k));
  }
  h->arr_elems = (size_t)(maxrows + 2 * GH) * pitch;
  {
    // the z history (m - 1 arrays beyond the fixed set) may use at most ~half of
    // the device memory left after the fixed arrays
    size_t freeb = 0, totb = 0;
    if (cudaMemGetInfo(&freeb, &totb) == cudaSuccess) {
      const double arr = (double)h->arr_elems * sizeof(double) * S;
      const double fixed = arr * A_ZH0;
      while (h->cg_defer > 2 && fixed + arr * (h->cg_defer - 1) > 0.8 * (double)freeb)
        h->cg_defer /= 2;
    }
  }
  h->sl.resize(S);
  for (int s = 0; s < S; ++s) {
    Slab& sl = h->sl[s];
    const int k = G.rank * S + s;
    sl.g.nx = G.nx;
    sl.g.ny = G.ny;
    sl.g.j0 = slab_row0(k);
    sl.g.nyl = slab_row0(k + 1) - sl.g.j0;
    sl.g.pitch = pitch;
    sl.g.pad = 0;
    sl.g.hx = 1.0 / G.nx;
    sl.g.hy = 1.0 / G.ny;
    sl.g.ihx = (double)G.nx;
    sl.g.ihy = (double)G.ny;
    sl.g.ihx2 = (double)G.nx * G.nx;
    sl.g.ihy2 = (double)G.ny * G.ny;
    for (int i = 0; i < A_N; ++i) sl.a[i] = nullptr;
    // z history: only the m - 1 buffers the chosen block length needs
    const int n_alloc = A_ZH0 + std::max(0, h->cg_defer - 1);
    for (int i = 0; i < n_alloc; ++i) {
      void* base = nullptr;
      if (cudaMalloc(&base, h->arr_elems * sizeof(double)) != cudaSuccess)
        return fail(CH_ERR_CUDA, h, "cudaMalloc (out of device memory?)");
      sl.bases.push_back(base);
      sl.a[i] = static_cast<double*>(base);
      cudaMemset(sl.a[i], 0, h->arr_elems * sizeof(double));
    }
  }
  if (cudaMalloc(&h->sc, NSC * sizeof(KScal)) != cudaSuccess ||
      cudaMallocHost(&h->sch, NSC * sizeof(KScal)) != cudaSuccess ||
      cudaMallocHost(&h->pollbuf, 2 * sizeof(KScal)) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->pollev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->pollev[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&h->part, (size_t)MAX_BLOCKS * 8 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->ticket, (MS_MAX + 1) * sizeof(unsigned int)) != cudaSuccess ||
      cudaMalloc(&h->tot, (size_t)total * 8 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->tot_local, (size_t)total * 8 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->gm_dev, 192 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->cgtab, (size_t)NSC * 2 * CGT * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&h->gm_red, (size_t)(S + 1) * 72 * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&h->gm_host, (size_t)std::max(192, 72 * S) * sizeof(double)) != cudaSuccess)
    return fail(CH_ERR_CUDA, h, "cudaMalloc (scalars)");
  if (cudaMalloc(&h->xr_mem, XR_BYTES) != cudaSuccess ||
      cudaMalloc(&h->xp_dev, sizeof(XPeers)) != cudaSuccess)
    return fail(CH_ERR_CUDA, h, "cudaMalloc (peer table)");
  cudaMemset(h->xr_mem, 0, XR_BYTES);
  {
    XPeers xp;
    memset(&xp, 0, sizeof xp);
    xp.R = 1;
    xp.rank = 0;
    xp.slab0 = 0;
    xp.nslab_all = S;
    xp.tot[0] = static_cast<double*>(h->xr_mem);
    xp.flag[0] = reinterpret_cast<unsigned*>(static_cast<char*>(h->xr_mem) + XR_TOT_BYTES);
    cudaMemcpy(h->xp_dev, &xp, sizeof xp, cudaMemcpyHostToDevice);
  }
  cudaMemset(h->sc, 0, NSC * sizeof(KScal));
  memset(h->sch, 0, NSC * sizeof(KScal));
  cudaMemset(h->ticket, 0, (MS_MAX + 1) * sizeof(unsigned int));
  h->st = nullptr;
  // c = 1 initially
  {
    std::vector<double> ones((size_t)h->arr_elems, 1.0);
    for (auto& s : h->sl) cudaMemcpy(s.a[A_C], ones.data(), h->arr_elems * sizeof(double),
                                     cudaMemcpyHostToDevice);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(CH_ERR_CUDA, h, "init sync");
  if (status) *status = CH_OK;
  return h;
}

int ch_comm_unique_id(void* id_out, size_t len) { return comm_unique_id(id_out, len); }

int ch_comm_init(ch_handle* h, const void* id, size_t len) {
  if (!h) return CH_ERR_ARG;
  if (h->grid.nranks == 1) return CH_OK;
  h->comm = comm_create(id, len, h->grid.rank, h->grid.nranks, h->grid.device, &h->err);
  if (!h->comm) return CH_ERR_COMM;
  return peer_setup(h);
}

int ch_comm_mode(const ch_handle* h) {
  if (!h) return -CH_ERR_ARG;
  return !h->comm ? 0 : (h->p2p ? 2 : 1);
}

int ch_local_rows(const ch_handle* h, int32_t* row0, int32_t* nrows) {
  if (!h) return CH_ERR_ARG;
  if (row0) *row0 = h->row0;
  if (nrows) *nrows = h->nrows;
  return CH_OK;
}

int ch_set_stream(ch_handle* h, void* stream) {
  if (!h) return CH_ERR_ARG;
  h->st = (cudaStream_t)stream;
  return CH_OK;
}

int ch_set_field(ch_handle* h, int field, const double* src, int where) {
  if (!h || !src) return CH_ERR_ARG;
  const int id = field_arr(field);
  if (id < 0) {
    h->err = "bad field id";
    return CH_ERR_ARG;
  }
  TRY(put(h, id, src, where));
  if (field == CH_FIELD_V) TRY(zero_vrow0(h));
  // a new velocity resets the momentum guess to it (R25; oracle initial_state)
  if (field == CH_FIELD_U) TRY(copy_arr(h, A_U, A_USG));
  if (field == CH_FIELD_V) TRY(copy_arr(h, A_V, A_VSG));
  if (field == CH_FIELD_V_STAR) TRY(zero_vrow0(h, A_VSG));
  if (where != CH_DEVICE) CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int ch_set_fields(ch_handle* h, const double* phi, const double* c, const double* u,
                  const double* v, const double* p, int where) {
  if (!h) return CH_ERR_ARG;
  if (phi) {
    TRY(put(h, A_PHI, phi, where));
    TRY(copy_arr(h, A_PHI, A_PHIP));
  }
  if (c) TRY(put(h, A_C, c, where));
  if (u) {
    TRY(put(h, A_U, u, where));
    TRY(copy_arr(h, A_U, A_USG));  // momentum guess := u (R25)
  }
  if (v) {
    TRY(put(h, A_V, v, where));
    TRY(zero_vrow0(h));
    TRY(copy_arr(h, A_V, A_VSG));
  }
  if (p) TRY(put(h, A_P, p, where));
  if (where != CH_DEVICE) CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int ch_get_field(ch_handle* h, int field, double* dst, int where) {
  if (!h || !dst) return CH_ERR_ARG;
  const int id = field_arr(field);
  if (id < 0) {
    h->err = "bad field id";
    return CH_ERR_ARG;
  }
  return get(h, id, dst, where);
}

int ch_get_fields(ch_handle* h, double* phi, double* c, double* u, double* v, double* p,
                  int where) {
  if (!h) return CH_ERR_ARG;
  if (phi) TRY(get(h, A_PHI, phi, where));
  if (c) TRY(get(h, A_C, c, where));
  if (u) TRY(get(h, A_U, u, where));
  if (v) TRY(get(h, A_V, v, where));
  if (p) TRY(get(h, A_P, p, where));
  return CH_OK;
}

int ch_set_time_index(ch_handle* h, int64_t n) {
  if (!h || n < 0) return CH_ERR_ARG;
  h->tidx = n;
  return CH_OK;
}

int ch_get_time_index(const ch_handle* h, int64_t* n) {
  if (!h || !n) return CH_ERR_ARG;
  *n = h->tidx;
  return CH_OK;
}

int ch_step(ch_handle* h, int nsteps) {
  if (!h || nsteps < 0) return CH_ERR_ARG;
  for (int n = 0; n < nsteps; ++n) TRY(step_once(h));
  return CH_OK;
}

namespace {
// Coefficients of operator `op` from the current state (what ch_step would
// use for its first solve of that kind); returns the 5-point kind or -1 (CH).
int prep_operator(ch_handle* h, int op, int* kind) {
  const Phys ph = phys_at(h->prm, h->tidx);
  TRY(halo(h, A_PHI, 2));
  TRY(halo(h, A_PHIP, 2));
  TRY(halo(h, A_U, 1));
  TRY(halo(h, A_V, 1));
  TRY(halo(h, A_C, 1));
  for (auto& s : h->sl) launch_ch_rhs(s.g, ph, state(s), s.a[A_PHIS], s.a[A_DINV], s.a[A_TMP2], h->st);
  TRY(halo(h, A_PHIS, 2));
  TRY(halo(h, A_DINV, 2));
  switch (op) {
    case CH_OP_CH:
      *kind = -1;
      break;
    case CH_OP_POISSON:
      TRY(copy_arr(h, A_PHI, A_PHI1));
      *kind = (h->prm.rho_n == h->prm.rho_s) ? OPK_POISSON_CONST : OPK_POISSON_VAR;
      break;
    case CH_OP_MOM_U:
    case CH_OP_MOM_V:
      for (auto& s : h->sl) {
        if (op == CH_OP_MOM_U)
          launch_mom_rhs_u(s.g, ph, state(s), s.a[A_PHIS], s.a[A_CA], s.a[A_CW], s.a[A_TMP2], h->st);
        else
          launch_mom_rhs_v(s.g, ph, state(s), s.a[A_PHIS], s.a[A_CA], s.a[A_CW], s.a[A_TMP2], h->st);
      }
      *kind = (op == CH_OP_MOM_U) ? OPK_MOM_U : OPK_MOM_V;
      break;
    case CH_OP_NUTRIENT:
      // the nutrient system of a step whose CH solve returned phi^{n+1} = phi^n
      TRY(copy_arr(h, A_PHI, A_PHI1));
      TRY(halo(h, A_PHI1, 1));
      for (auto& s : h->sl)
        launch_nut_rhs(s.g, ph, state(s), s.a[A_PHI1], s.a[A_CA], s.a[A_CW], s.a[A_TMP2], h->st);
      *kind = OPK_NUTRIENT;
      break;
    default:
      h->err = "bad operator id";
      return CH_ERR_ARG;
  }
  return check_launch(h, "prep_operator");
}
}  // namespace

int ch_apply_operator(ch_handle* h, int op, const double* x, double* y, int where) {
  if (!h || !x || !y) return CH_ERR_ARG;
  int kind = 0;
  TRY(prep_operator(h, op, &kind));
  TRY(put(h, A_TMP, x, where));
  const double cells = (double)h->grid.nx * (double)h->nrows / h->S;
  if (kind < 0) {
    TRY(halo(h, A_TMP, 2));
    // read x, phi* (+ u, v of the advection part); write y
    const bool adv = phys_at(h->prm, h->tidx).th_adv != 0.0;
    KTime kt(h, CH_KC_CH_APPLY, (adv ? 40.0 : 24.0) * cells);
    for (int s = 0; s < h->S; ++s) {
      Slab& sl = h->sl[s];
      launch_ch_apply(sl.g, chcoef(h, sl, false), sl.a[A_TMP], sl.a[A_B], 0, nullptr, nullptr, 0,
                      0, rargs(h, FIN_NONE, CH_NSYS, s), h->st);
    }
  } else {
    TRY(halo(h, A_TMP, 1));
    if (kind == OPK_MOM_U || kind == OPK_MOM_V || kind == OPK_NUTRIENT) TRY(halo(h, A_CW, 1));
    // x, y (+ w) (+ a[])
    const int ek = opdesc(h, kind, h->sl[0]).kind;
    const double bpc = ek == OPK_POISSON_CONST ? 16.0
                     : (ek == OPK_POISSON_VAR || ek == OPK_MOM_U_C || ek == OPK_MOM_V_C) ? 24.0
                     : 32.0;
    KTime kt(h, CH_KC_OP_APPLY, bpc * cells);
    for (auto& s : h->sl) launch_op5_apply(opdesc(h, kind, s), s.g, s.a[A_TMP], s.a[A_B], h->st);
  }
  TRY(check_launch(h, "apply_operator"));
  TRY(get(h, A_B, y, where));
  CK(cudaStreamSynchronize(h->st));
  harvest(h, -1);
  return CH_OK;
}

int ch_solve(ch_handle* h, int op, const double* b, double* x, int where) {
  if (!h || !b || !x) return CH_ERR_ARG;
  int kind = 0;
  TRY(prep_operator(h, op, &kind));
  TRY(put(h, A_B, b, where));
  TRY(put(h, A_US, x, where));
  int sys = CH_SYS_CH;
  if (kind < 0) {
    TRY(bicgstab_or_gmres(h, A_US, A_B));
  } else {
    sys = (op == CH_OP_POISSON) ? CH_SYS_P
        : (op == CH_OP_MOM_U) ? CH_SYS_U
        : (op == CH_OP_MOM_V) ? CH_SYS_V : CH_SYS_NUTRIENT;
    const int ns = (op == CH_OP_POISSON);
    if (ns) {
      for (int s = 0; s < h->S; ++s) {
        Slab& sl = h->sl[s];
        launch_sum(sl.g, sl.a[A_B], rargs(h, FIN_MEAN, sys, s), h->st);
      }
      TRY(check_launch(h, "sum"));
      TRY(fin_slabs(h, FIN_MEAN, sys, 1));
    }
    TRY(cg_any(h, sys, kind, A_US, A_B, ns, ns, "solve",
               kind == OPK_POISSON_VAR ? A_PHI1 : (ns ? -1 : A_CW)));
    if (ns)
      for (auto& s : h->sl) launch_sub_mean(s.g, s.a[A_US], h->sc + sys, h->st);
  }
  TRY(get(h, A_US, x, where));
  if (where == CH_DEVICE) CK(cudaStreamSynchronize(h->st));
  return CH_OK;
}

int ch_get_stats(const ch_handle* h, ch_stats* out) {
  if (!h || !out) return CH_ERR_ARG;
  *out = h->stats;
  return CH_OK;
}

int ch_reset_stats(ch_handle* h) {
  if (!h) return CH_ERR_ARG;
  const int64_t steps = h->stats.steps;
  memset(&h->stats, 0, sizeof(ch_stats));
  h->stats.steps = steps;
  return CH_OK;
}

int ch_enable_timing(ch_handle* h, int stride) {
  if (!h || stride < 0) return CH_ERR_ARG;
  h->tm.stride = stride;
  return CH_OK;
}

void ch_destroy(ch_handle* h) {
  if (!h) return;
  cudaSetDevice(h->grid.device);
  if (h->st) cudaStreamSynchronize(h->st);
  cudaDeviceSynchronize();
  if (h->comm) comm_destroy(h->comm);
  destroy_mem(h);
  delete h;
}

}  // extern "C"
