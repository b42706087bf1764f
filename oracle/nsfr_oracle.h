/*
 * nsfr_oracle.h — CPU checker ABI (TEST INFRASTRUCTURE ONLY).
 *
 * Two CPU libraries export this ABI, differing only in the symbol prefix:
 *   - oracle/libnsfr_oracle.so  (prefix nsfr_oracle_): the plain-C restatement
 *     in oracle/nsfr_oracle.c of the reference path (every function cites the
 *     /root/reference/proj file:line it follows) plus the residual glue that
 *     the reference only specifies.
 *   - oracle/_ref/libnsfr_ref.so (prefix nsfr_ref_): the reference's OWN
 *     compiled primitives (the .cpp files of /root/reference/proj/src, built by
 *     oracle/Makefile) driven by the same glue in oracle/ref_driver.cpp.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load these.
 * The product (paper_2312_07725_b200/libnsfr_b200.so) never links them.
 *
 * Layouts (all row-major, xi fastest; SURVEY.md §8 notation):
 *   state / dudt      [e_local][5][np^3]        modal = nodal values at LGL nodes
 *   jac               [e_local][nq^3]
 *   cof               [e_local][nq^3][9]        cof[3*n_phys + i_ref]
 *   traces            [e_local][6][5][nq^2]     entropy-projected conservative (DG: chi u_hat)
 *   halo_lo / halo_hi [m*m][5][nq^2]            face 5 of plane k0-1 / face 4 of plane k1
 */
#ifndef NSFR_ORACLE_H
#define NSFR_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nsfr_cfg {
  int p;              /* polynomial degree, n_p = p+1 */
  int quad_kind;      /* 0 = Gauss-Legendre, 1 = Gauss-Lobatto-Legendre */
  int overint;        /* extra quadrature nodes (only 0 is supported by the GPU path) */
  double c1d;         /* ESFR correction parameter (this code's convention) */
  int m;              /* elements per direction of the periodic m^3 box */
  int k0, k1;         /* local z-slab [k0,k1) (k0=0,k1=m for the whole box) */
  double x_left, x_right;
  double beta;        /* warp amplitude */
  double length_scale;/* warp length l; <=0 -> (xR-xL)/(2 pi) */
  int grid_degree;    /* mapping degree (reference default p+1) */
  double gamma;
  int roe;            /* 1: EC + Roe surface flux, 0: EC only (DG: central + Roe / central) */
  int workers;        /* element-parallel threads (<=1 serial) */
  int scheme;         /* 0: NSFR-EC; 1: conservative strong-form DG
                         (SPEC.md:457-465), overintegration allowed */
} nsfr_cfg;

#define NSFR_SCHEME_NSFR 0
#define NSFR_SCHEME_DG 1

#define NSFR_CASE_VORTEX 0
#define NSFR_CASE_TGV 1
#define NSFR_CASE_FREESTREAM 2

/* Return codes (shared with include/nsfr_gpu.h). */
#define NSFR_OK 0
#define NSFR_E_DIM 1
#define NSFR_E_MESH 2
#define NSFR_E_INADMISSIBLE 3

#define NSFR_CAT2(a, b) a##b
#define NSFR_CAT(a, b) NSFR_CAT2(a, b)
#define NSFR_CPU_API(name) NSFR_CAT(NSFR_CPU_PREFIX, name)

#ifdef NSFR_CPU_PREFIX
void* NSFR_CPU_API(create)(const nsfr_cfg* cfg, char* err, int errlen);
void NSFR_CPU_API(destroy)(void* ctx);
const char* NSFR_CPU_API(last_error)(void* ctx);
/* Packed 1D tables: interp(nq*np) proj(np*nq) fr_proj(np*nq) skew(nq*nq)
 * bound_flux(2*nq) bound_sol(2*np) wq(nq) quad_nodes(nq) sol_nodes(np)
 * mmass1d(np*np) quad_diff(nq*nq). Returns the number of doubles. */
int NSFR_CPU_API(tables)(void* ctx, double* out, int cap);
int NSFR_CPU_API(metrics)(void* ctx, double* jac, double* cof);
int NSFR_CPU_API(x_sol)(void* ctx, double* x);  /* [e][np^3][3] */
int NSFR_CPU_API(x_vol)(void* ctx, double* x);  /* [e][nq^3][3] */
int NSFR_CPU_API(initial_state)(void* ctx, int case_kind, double* u);
/* Entropy-projected face traces of all local elements [e][6][5][nq^2]. */
int NSFR_CPU_API(traces)(void* ctx, const double* u, double* traces);
/* Face traces of the plane-boundary elements for a halo exchange. */
int NSFR_CPU_API(boundary_traces)(void* ctx, const double* u, double* send_lo, double* send_hi);
/* Full residual; halo pointers may be NULL only when the slab is the box. */
int NSFR_CPU_API(rhs)(void* ctx, const double* u, const double* halo_lo, const double* halo_hi,
                      double* dudt, double* entropy_change);
int NSFR_CPU_API(max_wavespeed)(void* ctx, const double* u, double* lam);
int NSFR_CPU_API(rk4_step)(void* ctx, double* u, double dt);
int NSFR_CPU_API(l2_error)(void* ctx, const double* u, double t, int case_kind, double out2[2]);
int NSFR_CPU_API(entropy_total)(void* ctx, const double* u, double* out);
/* conserved totals sum w J u_q: mass, momentum x3, energy */
int NSFR_CPU_API(conserved_totals)(void* ctx, const double* u, double out5[5]);
/* kinetic-energy volume term sum v_KE . S6 rows of (EC flux - pressure work)
 * (SPEC.md:602-609); ~0 for the KEP flux */
int NSFR_CPU_API(ke_volume)(void* ctx, const double* u, double* out);
/* kinetic-energy change minus pressure work: -sum v_hat_KE . R with every
 * two-point flux minus the pressure work, no Roe; whole box */
int NSFR_CPU_API(ke_total)(void* ctx, const double* u, double* out);
#endif

#ifdef __cplusplus
}
#endif
#endif
