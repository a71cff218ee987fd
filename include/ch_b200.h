/*
 * ch_b200.h -- C ABI of the B200-native hot path of arxiv 1811.11842
 * ("2D parallel implementation of the modified Cahn-Hilliard equation for
 * the simulation of a biofilm", PAPER.md).
 *
 * One handle = one rank's slab of the nx x ny cell-centred MAC grid on
 * [0,1]^2 (periodic in x, walls at y = 0, 1).  ch_step()
 * advances the coupled model of PAPER.md Eq. 16 (lines 108-114) by the
 * semi-implicit scheme of §4 (lines 117-151): modified Cahn-Hilliard solve
 * (Eq. 4-5, GMRES/BiCGStab + Jacobi), nutrient solve,
 * Chorin projection (Eq. 19-21) with the constant null space of the pressure
 * operator removed (Listing 5).
 *
 * Conventions shared by every entry point:
 *  - Arrays are fp64, row-major (ny_rows, nx), row j = y index, x contiguous,
 *    leading dimension nx.  A rank's arrays hold its local rows
 *    [row0, row0 + nrows) (see ch_local_rows).
 *  - Staggering: phi, c, p at cell centres; u[j][i] on the x-face (i/nx,
 *    (j+1/2)/ny); v[j][i] on the y-face ((i+1/2)/nx, j/ny); v[0][*] is the
 *    bottom wall and must be 0.
 *  - `where` = CH_HOST: pointer is host memory (pageable or pinned; the call
 *    copies synchronously w.r.t. the library stream).  CH_DEVICE: pointer is
 *    device memory on the handle's device; the call is stream-ordered on the
 *    library stream (ch_set_stream) and does not synchronise.
 *  - Ownership: the caller owns every pointer it passes; the library never
 *    retains one past the call.  The handle owns all device memory it
 *    allocates; ch_destroy frees it.
 *  - Errors: every int-returning call returns CH_OK (0) or a CH_ERR_* code
 *    and records a message readable with ch_last_error(h).  No call aborts the
 *    process; a failed ch_step leaves the state at the last completed step.
 */
#ifndef CH_B200_H
#define CH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CH_ABI_VERSION 2

enum {
  CH_OK = 0,
  CH_ERR_ARG = 1,            /* invalid argument / size / state            */
  CH_ERR_CUDA = 2,           /* CUDA runtime error (message has the name)  */
  CH_ERR_NOT_CONVERGED = 3,  /* a Krylov solve hit maxit (stats say which) */
  CH_ERR_BREAKDOWN = 4,      /* Krylov breakdown (zero/NaN inner product)  */
  CH_ERR_COMM = 5            /* halo / reduction transport failure         */
};

/* Opaque handle: one rank's slab state + workspace on one device. */
typedef struct ch_handle ch_handle;

enum { CH_HOST = 0, CH_DEVICE = 1 };

/* Field ids for ch_set_field / ch_get_field. */
enum {
  CH_FIELD_PHI = 0,       /* phi_n^n  (network volume fraction, cells)   */
  CH_FIELD_PHI_PREV = 1,  /* phi_n^{n-1} (extrapolation history, R5)      */
  CH_FIELD_C = 2,         /* nutrient c (cells)                           */
  CH_FIELD_U = 3,         /* x-velocity (x-faces)                         */
  CH_FIELD_V = 4,         /* y-velocity (y-faces, row 0 = wall)           */
  CH_FIELD_P = 5,         /* pressure variable of Eq. 20 (cells, R15)     */
  CH_FIELD_U_STAR = 6,    /* u* of the last step = initial guess of the   */
  CH_FIELD_V_STAR = 7     /* next momentum solves (R25; x-/y-   */
                          /* faces); reset to u / v when u / v are set    */
};

/* Linear systems, in solve order within a step (also the stats index). */
enum { CH_SYS_CH = 0, CH_SYS_NUTRIENT = 1, CH_SYS_U = 2, CH_SYS_V = 3, CH_SYS_P = 4, CH_NSYS = 5 };

/* Operators for ch_apply_operator (isolated matrix-free stencil sweeps). */
enum {
  CH_OP_CH = 0,       /* y = [I/dt + th G1 L_{M*} Delta_h + ta Adv(.; v^n)] x, M* from phi, phi_prev */
  CH_OP_POISSON = 1,  /* y = -D_h beta G_h x, beta = 1/rho(current phi) on faces (Eq. 20 LHS)      */
  CH_OP_MOM_U = 2,    /* y = [a - theta_visc Delta_h^0] x on x-faces, a = 1/(nu(phi*) dt)          */
  CH_OP_MOM_V = 3,    /* same on y-faces, wall row identity                                       */
  CH_OP_NUTRIENT = 4  /* y = [diag(f_s/dt + A/2 f) - 1/2 div(K grad)] x, the nutrient system of   */
                      /* Eq. 16 (3rd line) with phi^{n+1} = phi^{n} = the current phi (R11, R24)  */
};

/* Krylov method for the (nonsymmetric) Cahn-Hilliard system. */
enum { CH_SOLVER_BICGSTAB = 0, CH_SOLVER_GMRES = 1 };

typedef struct ch_grid {
  int32_t nx, ny;        /* global cells; nx even and >= 4, ny >= 4                     */
  int32_t rank, nranks;  /* slab decomposition in y over processes (1 GPU each)          */
  int32_t device;        /* CUDA device ordinal for this handle                          */
  int32_t virtual_slabs; /* >= 1: split this rank's rows into that many slabs with halo   */
                         /* exchange between them on the same device (tests the           */
                         /* decomposition on one GPU); 1 = off                            */
} ch_grid;

typedef struct ch_params {
  /* PAPER.md §5 dimensionless parameters (lines 271-274) and Eq. 5, 7, 15. */
  double dt;       /* time step                                    */
  double Gamma1;   /* conformation-entropy strength  (33.467)      */
  double Gamma2;   /* bulk free-energy strength      (1.25e6)      */
  double Lambda;   /* mobility                       (1e-10)       */
  double mu;       /* max production rate            (0.14)        */
  double Kc;       /* half-saturation constant       (0.15)        */
  double eps;      /* production scaling (Eq. 5)     (1, R8)       */
  double A;        /* consumption rate (Eq. 7)       (100)         */
  double Ds;       /* nutrient diffusion             (2.3)         */
  double Re_s;     /* solvent Reynolds number        (9.98e-4)     */
  double Re_n;     /* network Reynolds number        (2.33e-9)     */
  double rho_n;    /* rho_n / rho_0                  (1)           */
  double rho_s;    /* rho_s / rho_0                  (1)           */
  double lid_u;    /* top-wall tangential velocity U0 (1, R10)     */
  double rtol;     /* Krylov relative residual ||r||/||b|| (1e-10) */
  /* Implicit weights of the time discretisation (R5, R7, R12, R23). */
  double theta_ch;   /* Gamma1 fourth-order CH term: 0.5 = Crank-Nicolson       */
                     /* ("Crank-Nicholson ... in R and f"), [0,1]  */
  double theta_adv;  /* advection div(phi v^n) in the CH system: 0.5 = CN, [0,1] */
  double theta_visc; /* viscous term of Eq. 19: 1 = at u^{n+1} (the BVP "for    */
                     /* u^{n+1}"), (0,1]                       */
  int32_t maxit;   /* iteration cap per solve                      */
  int32_t ch_solver;      /* CH_SOLVER_*                           */
  int32_t gmres_restart;  /* m of GMRES(m), 1..64                  */
  int32_t refine;  /* symmetric (CG) solves: up to `refine` restarts  */
                   /* from the converged x until the TRUE residual   */
                   /* ||b - A x|| <= rtol ||b|| (0 = stop on the     */
                   /* method's recursive residual, PETSc's default)  */
  int32_t startup_be; /* steps with time index n < startup_be take theta_ch =  */
                      /* theta_adv = 1 (backward-Euler start-up, R23), >= 0    */
} ch_params;

typedef struct ch_stats {
  int64_t steps;                      /* completed time steps                       */
  int32_t iters_last[CH_NSYS];        /* Krylov iterations of the last step          */
  int64_t iters_total[CH_NSYS];
  double resid_last[CH_NSYS];         /* method's final ||r||/||b|| of the last step */
  int64_t launches;                   /* CUDA kernels launched by the library        */
  /* per kernel class (CH_KC_*), filled while timing is enabled: sampled launches */
  int64_t kc_launches[16];            /* launches of that class                      */
  int64_t kc_timed[16];               /* how many of them were event-timed           */
  double kc_ms[16];                   /* summed event time of the timed ones (ms)    */
  double kc_bytes[16];                /* algorithmic bytes of the timed launches (§6) */
} ch_stats;

/* Kernel classes for ch_stats.kc_* */
enum {
  CH_KC_CG_A = 0,     /* CG half-iteration 1: p = z + beta p, x += alpha p, q = A p, (p,q)  */
  CH_KC_CG_B = 1,     /* CG half-iteration 2: r -= alpha A p, z = D^-1 r, (r,z), (r,r)       */
  CH_KC_CG_INIT = 2,
  CH_KC_CH_APPLY = 3, /* 13-point CH apply fused with D^-1 and dots                          */
  CH_KC_VEC = 4,      /* fused BLAS-1 + reductions (BiCGStab / GMRES updates)                */
  CH_KC_RHS = 5,      /* explicit right-hand sides, coefficients, projection                 */
  CH_KC_GMRES = 6,    /* GMRES orthogonalisation                                            */
  CH_KC_CG_FUSED = 7, /* single-reduction CG sweep, nutrient system (default CG path)         */
  CH_KC_CG_FUSED_U = 8,  /* ... momentum u                                                   */
  CH_KC_CG_FUSED_V = 9,  /* ... momentum v                                                   */
  CH_KC_CG_FUSED_P = 10, /* ... pressure Poisson                                             */
  CH_KC_CG_PX = 11,      /* deferred p / x update of the single-reduction CG                 */
  CH_KC_OP_APPLY = 12,   /* isolated 5-point operator apply (ch_apply_operator)              */
  CH_NKC = 13
};

/* Create a handle: allocates the rank's slab state and workspace on
 * grid->device (28 fields + the m - 1 = 63 z-history buffers of the
 * deferred-p/x CG, each (nrows + 4) x pitch doubles: ~12 GB at 4096^2; m is
 * halved automatically while the history would not fit in 80 % of the free
 * device memory).
 * Fields start zero except c = 1.  Parameters are copied (the caller keeps
 * ownership of *grid and *params).  Returns NULL on error with *status set
 * (status may be NULL): CH_ERR_ARG for an invalid grid / parameter set,
 * CH_ERR_CUDA if the device cannot be used or memory runs out. */
ch_handle* ch_create(const ch_grid* grid, const ch_params* params, int* status);

/* Multi-process runs (grid->nranks > 1): join the NCCL clique.  `id` is the
 * 128-byte ncclUniqueId produced by rank 0 with ch_comm_unique_id and
 * broadcast by the caller (e.g. torch.distributed).  Collective.  Then, if
 * every rank is its own process on its own device with peer access to all
 * the others (and env CHB_P2P is not 0), maps the neighbours' CG ring arrays
 * and every rank's reduction area through CUDA IPC: each CG iteration is then
 * ONE kernel per rank that stores its edge rows of z' into the neighbours'
 * ghost rows and combines the iteration's inner products over NVLink peer
 * memory ("MPI is used to communicate ghost points"; DESIGN.md
 * §7).  Also makes the deferred-p/x block length the minimum over ranks. */
int ch_comm_unique_id(void* id_out, size_t len);
int ch_comm_init(ch_handle* h, const void* id, size_t len);
/* 0: single process; 1: NCCL halo rows + allgather per CG iteration;
 * 2: peer-memory CG iterations (NCCL for the rest of the step). */
int ch_comm_mode(const ch_handle* h);

/* Rows owned by this handle: [*row0, *row0 + *nrows). */
int ch_local_rows(const ch_handle* h, int32_t* row0, int32_t* nrows);

/* Host-only (no device work, callable without a GPU): the 1-D slab
 * decomposition in y that ch_create applies -- ny rows split over
 * nranks * virtual_slabs slabs as evenly as possible, the first
 * (ny mod total) slabs one row taller, each >= 2 rows; rank r owns slabs
 * r*virtual_slabs .. (r+1)*virtual_slabs - 1.  Returns CH_ERR_ARG for an
 * invalid decomposition (the same condition ch_create rejects). */
int ch_partition(int32_t ny, int32_t nranks, int32_t rank, int32_t virtual_slabs, int32_t* row0,
                 int32_t* nrows);

/* Use `stream` (a cudaStream_t, may be NULL = legacy default) for all work. */
int ch_set_stream(ch_handle* h, void* stream);

/* Time index n of the state (0 after ch_create; +1 per completed step).  It
 * selects the backward-Euler start-up steps (params.startup_be, R23); a caller
 * restoring a saved state sets it back with ch_set_time_index.  n >= 0. */
int ch_set_time_index(ch_handle* h, int64_t n);
int ch_get_time_index(const ch_handle* h, int64_t* n);

/* Set the state (any pointer may be NULL = leave unchanged).  Each array is
 * the local slab, nrows x nx, ld = nx.  Setting phi also sets phi_prev = phi
 * (first step extrapolates to phi* = phi^0, R5); setting u (v) also
 * sets the momentum guess u* (v*) to it (R25).  ch_set_field sets one field
 * (CH_FIELD_*): the same side effects except for phi (PHI_PREV is its own
 * field); U_STAR / V_STAR restore a saved guess and must follow u / v. */
int ch_set_fields(ch_handle* h, const double* phi, const double* c, const double* u,
                  const double* v, const double* p, int where);
int ch_set_field(ch_handle* h, int field, const double* src, int where);

/* Advance nsteps time steps of the semi-implicit scheme (§4, lines
 * 117-151; splitting order DESIGN.md R1), each step:
 *   1. phi* = (3 phi^n - phi^{n-1}) / 2; Cahn-Hilliard system (Eq. 16 4th
 *      line with Eq. 4-5; theta-weighted Gamma1 term and advection, CN by
 *      default) solved by BiCGStab / GMRES(m) with Jacobi;
 *   2. nutrient c^{n+1} (Eq. 16 3rd line, Eq. 7), Jacobi-PCG;
 *   3. intermediate velocity u*, v* (Eq. 18-19, R6-R7), Jacobi-PCG each,
 *      initial guesses the previous step's u*, v* (R25);
 *   4. pressure -div(1/rho grad p) = div u* (Eq. 20) with the constant null
 *      space removed (Listing 5), Jacobi-PCG;
 *   5. projection v^{n+1} = u* + (1/rho) grad p (Eq. 21).
 * Every solve stops at ||r|| <= rtol ||b|| (R13, R21 for params.refine).
 * All device work is ordered on the library stream; the call returns when
 * the last step is complete.  On error (CH_ERR_NOT_CONVERGED,
 * CH_ERR_BREAKDOWN, CH_ERR_CUDA, CH_ERR_COMM) ch_last_error names the
 * system and the steps completed before it remain in the state; stats say
 * which system failed (iters_last / resid_last). */
int ch_step(ch_handle* h, int nsteps);

/* Copy the state out (NULL pointers skipped).  CH_HOST copies synchronise. */
int ch_get_fields(ch_handle* h, double* phi, double* c, double* u, double* v, double* p,
                  int where);
int ch_get_field(ch_handle* h, int field, double* dst, int where);

/* Isolated matrix-free apply y = Op x on the local slab (halo exchange
 * included for multi-slab handles), coefficients from the current state. */
int ch_apply_operator(ch_handle* h, int op, const double* x, double* y, int where);

/* Isolated solve Op x = b on the local slab with the operator's coefficients
 * from the current state and the step's Krylov method for that operator
 * (CH_OP_CH: BiCGStab or GMRES(m) per params.ch_solver, PAPER.md:233-244;
 * the 5-point operators: Jacobi-preconditioned CG; for
 * CH_OP_POISSON b is projected to mean zero and x returned with mean zero,
 * Listing 5).  x: initial guess in, solution out (nrows x nx, same `where`
 * as b).  Stops at ||r||_2 <= rtol ||b||_2 (R13); the iteration count and
 * final residual land in ch_stats.{iters_last,resid_last}[system]
 * (CH_SYS_CH, CH_SYS_P, CH_SYS_U, CH_SYS_V, CH_SYS_NUTRIENT).  Returns CH_ERR_NOT_CONVERGED /
 * CH_ERR_BREAKDOWN like ch_step.  Does not advance the state. */
int ch_solve(ch_handle* h, int op, const double* b, double* x, int where);

int ch_get_stats(const ch_handle* h, ch_stats* out);
int ch_reset_stats(ch_handle* h);
/* Sample every `stride`-th launch of each kernel class with a CUDA event pair
 * on the library stream (0 = off).  The CG sweeps are sampled as groups of up
 * to 8 consecutive launches of one solve between ONE pair (kc_timed counts
 * every launch of the group): an event between two sweeps would keep the
 * second from starting under programmatic dependent launch, so a group times
 * the sweeps as the chain runs them.  A group holds no p/x launch and no
 * convergence poll. */
int ch_enable_timing(ch_handle* h, int stride);

/* Self-test of the peer-memory combine of the CG sweep on one
 * device: `nranks` groups of `nloc` CTAs play the ranks of a clique inside ONE
 * cooperative launch (the way blocks that wait on one another may share a
 * GPU), each with its own totals area and flags, for `epochs` iterations with
 * randomised arrival order; at epoch `absent_epoch` (0 = never) the last rank
 * does not arrive and every other rank must time out (~2 s) instead of
 * hanging.  Returns the number of mismatches (0: every rank computed the
 * bit-exact slab-ordered sums, every timeout was reported) or -CH_ERR_*.
 * last (may be NULL): [nranks][8] combined totals of the last epoch.
 * nranks <= 8, nloc <= 8. */
int ch_selftest_xrank(int device, int nranks, int nloc, int epochs, int absent_epoch,
                      double* last);

const char* ch_last_error(const ch_handle* h);
int ch_abi_version(void);
void ch_destroy(ch_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* CH_B200_H */
