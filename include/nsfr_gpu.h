/*
 * nsfr_gpu.h — C ABI of the B200-native NSFR residual path (libnsfr_b200.so).
 *
 * This is the drop-in boundary for the reference's MISSING solver layer
 * (proj/CMakeLists.txt:26 lists src/solver.cpp, which is absent; its contract
 * is SPEC.md:422-518 and PAPER.md:869-929). Each entry point names the
 * reference interface it replaces:
 *
 *   nsfr_gpu_create        build_reference_operators (fr_operators.cpp:89-113)
 *                          + warp_grid_3d (geometry.cpp:62-73)
 *                          + build_metrics_conservative_curl (geometry.cpp:86-266),
 *                          or adopts caller-built tables/metrics (setup fields)
 *   nsfr_gpu_set_state     ConservativeField upload (layout sumfac.hpp:46,86-87)
 *   nsfr_gpu_init_case     CaseSpec::initial at the solution nodes (cases.cpp:78-101)
 *   nsfr_gpu_rhs           nsfr_residual / assemble_rhs: entropy
 *                          projection + hadamard_sumfac_volume
 *                          (sumfac.hpp:48-94) + hadamard_sumfac_surface
 *                          (sumfac.hpp:110-157) + EC/Roe face flux (euler.cpp:142-162,
 *                          229-301) + weight_adjusted_inverse_apply (fr_operators.cpp:280-309)
 *   nsfr_gpu_rk4_step      rk4_step + adaptive_dt
 *   nsfr_gpu_advance       run_simulation's stepping loop
 *   nsfr_gpu_l2_error      l2_error
 *   nsfr_gpu_entropy_change discrete_entropy_change
 *
 * Conventions: every call returns int (NSFR_OK or an NSFR_E_* code); no C++
 * exception crosses the ABI; nsfr_gpu_last_error() describes the last failure.
 * Host pointers are borrowed for the duration of the call and copied. A
 * context is single-threaded and stream-ordered; one context per GPU.
 * Layouts: state [e_local][5][(p+1)^3] (modal = nodal values at the LGL
 * solution nodes), jac [e_local][nq^3], cof [e_local][nq^3][9] with
 * cof[3*n_phys + i_ref] exactly as ElementMetrics::cof_vol (geometry.hpp:66-80).
 * Elements are numbered e = i + m*(j + m*k) (geometry.hpp:16-22); a rank owns
 * the z-slab k in [k0, k1).
 */
#ifndef NSFR_GPU_H
#define NSFR_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSFR_OK 0
#define NSFR_E_DIM 1          /* DimensionError (defs.hpp:12-14) */
#define NSFR_E_MESH 2         /* InvalidMeshError (defs.hpp:16-18) */
#define NSFR_E_INADMISSIBLE 3 /* InadmissibleStateError / StepFailureError{t} (defs.hpp:20-28) */
#define NSFR_E_CUDA 4
#define NSFR_E_NCCL 5
#define NSFR_E_CONFIG 6       /* ConfigError (defs.hpp:30-32) */

#define NSFR_CASE_VORTEX 0     /* isentropic_vortex_exact, cases.cpp:36-56 */
#define NSFR_CASE_TGV 1        /* tgv_initial, cases.cpp:7-14 */
#define NSFR_CASE_FREESTREAM 2 /* CaseSpec free stream, cases.hpp:24-28 */

typedef struct nsfr_gpu_ctx nsfr_gpu_ctx;

/* Optional caller-built 1D tables (ReferenceOperators, fr_operators.hpp:40-57),
 * row-major. When `interp` is NULL the library builds them natively.
 * interp and fr_proj must be centrosymmetric (A[n-1-r][n-1-c] = A[r][c], true of
 * every symmetric node set and basis: GL / LGL, the reference's own tables):
 * the NSFR update kernel applies them through their even / odd halves, and
 * nsfr_gpu_create returns NSFR_E_CONFIG otherwise. */
typedef struct nsfr_gpu_tables {
  const double* interp;     /* basis.interp  chi(xi_v)   nq x np */
  const double* proj;       /* proj          Pi          np x nq */
  const double* fr_proj;    /* fr_proj       Pi~         np x nq */
  const double* skew;       /* skew   W Dq - Dq^T W      nq x nq */
  const double* bound_flux; /* bound_flux                2 x nq  */
  const double* bound_sol;  /* bound_sol                 2 x np  */
  const double* wq;         /* wq                        nq      */
} nsfr_gpu_tables;

typedef struct nsfr_gpu_setup {
  int p;               /* polynomial degree; np = nq = p+1 (no overintegration) */
  int quad_kind;       /* 0 Gauss-Legendre, 1 Gauss-Lobatto-Legendre */
  double c1d;          /* ESFR parameter, this code's convention (fr_operators.cpp:17-46) */
  double gamma;        /* EulerGas::gamma (euler.hpp:14-16) */
  int roe;             /* 1: EC + Roe surface flux, 0: EC only */
  int m;               /* elements per direction of the periodic m^3 box */
  int k0, k1;          /* this rank's z-slab [k0,k1) */
  double x_left, x_right;
  double beta;         /* warp amplitude (warp_grid_3d) */
  double length_scale; /* <= 0: (x_right-x_left)/(2 pi) */
  int grid_degree;     /* mapping degree, reference default p+1 (geometry.hpp:50-51) */
  int device;          /* CUDA device ordinal */
  int entropy_diag;    /* keep v_hat for nsfr_gpu_entropy_change */
  /* optional caller-built data (copied): tables and/or metrics of the slab */
  const nsfr_gpu_tables* tables;
  const double* jac_vol;  /* [e_local][nq^3]     or NULL: built on the device */
  const double* cof_vol;  /* [e_local][nq^3][9]  or NULL */
  /* multi-GPU: an NCCL unique id from nsfr_gpu_nccl_unique_id on rank 0,
   * broadcast by the caller; NULL for a single rank, or with nranks > 1 for
   * external halo transport (see nsfr_gpu_halo_buffers) */
  const void* nccl_id;
  int rank, nranks;
  /* scheme (SolverConfig.scheme): NSFR_SCHEME_NSFR (the hot
   * path) or NSFR_SCHEME_DG, the conservative strong-form DG residual with the
   * Roe surface flux (roe = 1) or the central flux (roe = 0), weight-adjusted
   * inverse (exact for overint = 0). overint: extra volume
   * quadrature nodes, n_q = p+1+overint (DG only; p in [3,5], overint in [0,2]). */
  int scheme;
  int overint;
} nsfr_gpu_setup;

#define NSFR_SCHEME_NSFR 0
#define NSFR_SCHEME_DG 1

int nsfr_gpu_create(const nsfr_gpu_setup* setup, nsfr_gpu_ctx** out);
int nsfr_gpu_destroy(nsfr_gpu_ctx* ctx);
const char* nsfr_gpu_last_error(const nsfr_gpu_ctx* ctx);
/* Last error of a failed nsfr_gpu_create (no context exists then). */
const char* nsfr_gpu_create_error(void);

/* 128-byte NCCL unique id (call on rank 0, broadcast to the others). */
int nsfr_gpu_nccl_unique_id(void* out128);

/* The NCCL communicator a context exchanges over, as NCCL itself reports it
 * (ncclCommCount / ncclCommUserRank / ncclCommCuDevice): a multi-GPU launch
 * prints these per rank so the world size can be checked. A context without
 * a communicator (single rank, external halos) reports 0 / -1 / its device. */
int nsfr_gpu_comm_info(nsfr_gpu_ctx* ctx, int* nccl_nranks, int* nccl_rank, int* cuda_device);

/* Halo plan of a z-slab decomposition (pure host logic, no GPU needed):
 * the slab of `rank`, the peers it exchanges face traces with, and the
 * message size in doubles. */
typedef struct nsfr_gpu_halo_plan {
  int k0, k1;        /* z planes owned */
  int peer_lo;       /* rank owning plane k0-1 (periodic) */
  int peer_hi;       /* rank owning plane k1 (periodic) */
  long long count;   /* doubles per message: m*m*6*nq*nq (6 values per face node, see below) */
} nsfr_gpu_halo_plan;
int nsfr_gpu_halo_plan_for(int m, int p, int rank, int nranks, nsfr_gpu_halo_plan* out);

/* Tables actually used (for parity checks): packed like nsfr_gpu_tables. */
int nsfr_gpu_get_tables(nsfr_gpu_ctx* ctx, double* out, int cap);
int nsfr_gpu_get_metrics(nsfr_gpu_ctx* ctx, double* jac, double* cof);

int nsfr_gpu_set_state(nsfr_gpu_ctx* ctx, const double* u);
int nsfr_gpu_get_state(nsfr_gpu_ctx* ctx, double* u);
/* The solver's own representation, u at the volume quadrature nodes
 * (u_q = chi^3 u_hat, same [e][5][nq^3] layout), copied without conversion:
 * a bit-exact restart (checkpoints) where set/get_state round trips to ~1 ulp. */
int nsfr_gpu_set_state_q(nsfr_gpu_ctx* ctx, const double* uq);
int nsfr_gpu_get_state_q(nsfr_gpu_ctx* ctx, double* uq);
int nsfr_gpu_init_case(nsfr_gpu_ctx* ctx, int case_kind);
int nsfr_gpu_set_time(nsfr_gpu_ctx* ctx, double t);
int nsfr_gpu_get_time(nsfr_gpu_ctx* ctx, double* t);

/* One residual dU/dt of the current state; dudt may be NULL (kept on device).
 * entropy_change may be NULL; else receives -sum v_hat . R (allreduced). */
int nsfr_gpu_rhs(nsfr_gpu_ctx* ctx, double* dudt, double* entropy_change);
/* Entropy-projected face traces of the local elements, conservative,
 * [e][6 faces][5][nq^2] (converted from the device's primitive form). */
int nsfr_gpu_get_traces(nsfr_gpu_ctx* ctx, double* traces);

/* One classical RK4 step; dt = cfl*dx/lambda_max (allreduced) from u_n,
 * dx = (x_right-x_left)/(m(p+1)), clipped to t_final - t (t_final <= 0: no clip). */
int nsfr_gpu_rk4_step(nsfr_gpu_ctx* ctx, double cfl, double t_final, double* dt_used);
/* nsteps RK4 steps without host synchronisation between them (CUDA graph). */
int nsfr_gpu_advance(nsfr_gpu_ctx* ctx, int nsteps, double cfl, double t_final, double* t_out);
/* Fixed dt variant (no wavespeed reduction): used by the parity tests. */
int nsfr_gpu_rk4_step_dt(nsfr_gpu_ctx* ctx, double dt);
/* One RK4 step on HOST buffers (replaces rk4_step(field, dt) on the caller's
 * std::span state, and adaptive_dt(field, cfl),
 * SPEC.md:475-483): the same result as set_state(u_in); dt > 0 ?
 * rk4_step_dt(dt) : rk4_step(cfl, t_final); get_state(u_out), bitwise, with
 * the host->device copy, the compute and the device->host copy pipelined over
 * element chunks (pinned buffers overlap; pageable ones work without
 * overlap). u_out may alias u_in. dt_next (may be NULL) receives
 * adaptive_dt(u_out, cfl) clipped to t_final, computed on the way out, so a
 * reference-style loop `dt = adaptive_dt(u); u = rk4_step(u, dt)` runs as
 * rk4_step_host(u, u, dt, cfl, t_final, NULL, &dt) with no global reduction
 * inside the step (dt <= 0 takes lambda_max of u_in first: one barrier).
 * NSFR contexts stream: a single rank, and a z-slab with an NCCL
 * communicator (its end chunks take the per-stage halo planes). External-halo
 * slab contexts (no NCCL id: the caller moves the planes between stages) and
 * DG contexts run the same calls in sequence. */
int nsfr_gpu_rk4_step_host(nsfr_gpu_ctx* ctx, const double* u_in, double* u_out, double dt,
                           double cfl, double t_final, double* dt_used, double* dt_next);
int nsfr_gpu_max_wavespeed(nsfr_gpu_ctx* ctx, double* lam);

/* L2 density/pressure error against the case's exact solution at the
 * context time (allreduced sums; returns the square roots). */
int nsfr_gpu_l2_error(nsfr_gpu_ctx* ctx, int case_kind, double out2[2]);
/* -sum v_hat . R of the last RHS of the current state (allreduced). */
int nsfr_gpu_entropy_change(nsfr_gpu_ctx* ctx, double* out);
/* Conserved totals sum_e sum_q w_q J_q u_q of the current state: mass,
 * x/y/z momentum, energy (DiagnosticRecord totals; Thm 3 drift
 * check SPEC.md:650), allreduced in a fixed order. */
int nsfr_gpu_conserved_totals(nsfr_gpu_ctx* ctx, double out5[5]);
/* sum_e sum_q w_q J_q U(u_q), U = -rho s/(gamma-1): the entropy total that
 * normalises the entropy change. */
int nsfr_gpu_entropy_total(nsfr_gpu_ctx* ctx, double* out);
/* Kinetic-energy volume term of the current state (kinetic_energy_change's
 * volume_term): sum_s v_KE,s . S6 rows of
 * the EC flux minus the pressure work P~_ij = 1/2 (p_i + p_j) I_d 1/2 (C_i + C_j),
 * v_KE = (-|v|^2/2, v, 0) at the volume nodes. Round-off for the KEP flux. */
int nsfr_gpu_ke_volume(nsfr_gpu_ctx* ctx, double* out);
/* Kinetic-energy change minus pressure work (kinetic_energy_change's
 * total_minus_pressure_work):
 * -sum v_hat_KE . R with R the pre-inverse residual rows (volume, hybrid
 * surface, face; chi^T lifted) of the EC flux minus the pressure work and no
 * Roe term, v_hat_KE = Pi^3 v_KE(u_q). Round-off for LGL, not for GL (Lemma 1). */
int nsfr_gpu_ke_total(nsfr_gpu_ctx* ctx, double* out);

/* Bench helper: time nsteps RK4 steps (t_final unbounded) with CUDA events on
 * the context stream; inputs stay resident in HBM. kernel_ms (optional, [3])
 * receives the summed durations of the K1 (projection prologue), K2 (pair
 * and face fluxes) and K3 (lift, mass inverse, RK update, next projection)
 * launches, each bracketed by its own events (disables the step graph). */
int nsfr_gpu_time_steps(nsfr_gpu_ctx* ctx, int nsteps, double cfl, double* step_ms, double* kernel_ms);

/* FP64 pipe peak of `device` in TFLOP/s (DFMA loop; roofline denominator). */
int nsfr_gpu_measure_fp64_peak(int device, double* tflops);
/* Same, plus the SM clock (MHz) the loop ran at, from the CTAs' clock64 spans
 * over the event-timed launch (nominal peak = SMs x 128 flop/clk x clock). */
int nsfr_gpu_measure_fp64_peak_ex(int device, double* tflops, double* sm_mhz);

/* ---- Stage-level driving and external halo transport ----------------------
 * A context created with nranks > 1 but nccl_id == NULL exchanges no data
 * itself: the caller moves the z-halo planes (e.g. over MPI, or between two
 * contexts in a test). Each plane is an opaque block of halo_plan.count doubles,
 * [m*m][6][nq^2]: the NSFR kernels keep face traces as the six primitives
 * (rho, u, v, w, p, rho/p) of u(v~); the DG scheme uses the first 5/6 of the
 * block for its conservative face states. Move the block as it is:
 * rank r's send_lo goes to rank r-1's recv_hi and its send_hi to rank r+1's
 * recv_lo (periodic). The driving sequence is
 *   nsfr_gpu_project;  [swap];  nsfr_gpu_residual            (one RHS), or
 *   nsfr_gpu_project;  for s = 1..4: { [swap]; nsfr_gpu_stage(s, dt) }
 * with dt = cfl dx / max over ranks of nsfr_gpu_max_wavespeed. Stage 4 leaves
 * the projection (and send planes) of u_{n+1}, so the next step starts with a
 * swap. In NCCL mode the same calls exchange internally. */
int nsfr_gpu_halo_buffers(nsfr_gpu_ctx* ctx, double** send_lo, double** send_hi, double** recv_lo,
                          double** recv_hi);
int nsfr_gpu_halo_get(nsfr_gpu_ctx* ctx, double* send_lo, double* send_hi);
int nsfr_gpu_halo_set(nsfr_gpu_ctx* ctx, const double* recv_lo, const double* recv_hi);
/* Entropy projection of the current state (faces, volume primitives, send planes, lambda). */
int nsfr_gpu_project(nsfr_gpu_ctx* ctx);
/* dU/dt of the projected state (after nsfr_gpu_project and the halo swap). */
int nsfr_gpu_residual(nsfr_gpu_ctx* ctx, double* dudt, double* entropy_change);
/* One RK4 stage (1..4) with the given dt (read at stage 1). */
int nsfr_gpu_stage(nsfr_gpu_ctx* ctx, int stage, double dt);

/* Device pointers (for callers that keep inputs resident in HBM). The device
 * state holds u at the volume quadrature nodes, u_q = chi^3 u_hat ([e][5][n^3]);
 * nsfr_gpu_set_state / nsfr_gpu_get_state convert from / to u_hat. A caller
 * writing through this pointer must call nsfr_gpu_set_time (or set_state)
 * before the next step so the cached projection is rebuilt. */
double* nsfr_gpu_state_device_ptr(nsfr_gpu_ctx* ctx);
size_t nsfr_gpu_state_count(const nsfr_gpu_ctx* ctx);
/* Synchronise and report a pending device error (NSFR_E_INADMISSIBLE...). */
int nsfr_gpu_sync(nsfr_gpu_ctx* ctx);
/* Kernel launches issued so far by this context (for the bench's claim). */
long long nsfr_gpu_launch_count(const nsfr_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
