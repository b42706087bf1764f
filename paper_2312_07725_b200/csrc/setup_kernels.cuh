// Setup-side kernels and shared device helpers of the NSFR path:
//   k_metrics   device build of J and the conservative-curl cofactors
//               (geometry.cpp:86-266) from the closed-form warp (geometry.cpp:62-73)
//   k_init      initial state at the LGL solution nodes (cases.cpp)
//   k_l2        L2 error partials; k_reduce deterministic sums
//   k_step_*    adaptive-dt bookkeeping
// Layout in HBM (element-contiguous blocks, xi fastest):
//   state u_q/acc [E][5][N^3] at the volume quadrature nodes; ut_vol [E][6][N^3] node
//   primitives; traces [E][6][5][N^2]; vol [E][5][N^3] and facc [E][3][5][2][N^2] (K2 -> K3);
//   cof [E][9][N^3] = 0.5 C
//   (component 3*n_phys + i_ref major); wj [E][N^3] = 1/(w_i w_j w_k J).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "physics.cuh"

namespace nsfr_b200 {

constexpr int MAXN = 8;
constexpr int MAXG = 9;

// 1D tables on the device (row-major).
struct DevTables {
  int np, nq, g;
  double interp[MAXN * MAXN];     // nq x np
  double interp_t[MAXN * MAXN];   // np x nq
  double proj[MAXN * MAXN];       // np x nq
  double frproj[MAXN * MAXN];     // np x nq
  double frproj_t[MAXN * MAXN];   // nq x np
  double qskew[MAXN * MAXN];      // q(a,b) - q(b,a) with q = 0.5*skew  (== skew(a,b))
  double bflux[2 * MAXN];
  double bsol[2 * MAXN];
  double wq[MAXN];
  double quad_diff[MAXN * MAXN];
  double gnodes[MAXG];
  double ig[MAXN * MAXG];         // nq x g
  double is[MAXN * MAXG];         // np x g
  double dg[MAXG * MAXG];         // g x g
};

enum ErrBits : unsigned { ERR_STATE = 1u, ERR_ROE = 2u, ERR_MESH = 4u };

__device__ __forceinline__ unsigned long long dbl_bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

// ---------------------------------------------------------------------------
// Directional tensor pass on shared memory: out = op along direction D.
// `nb` batches of an (E0,E1,E2) tensor (xi fastest); op is ROWS x COLS
// row-major with COLS == extent D. Same accumulation order as
// apply_operator_dir (sumfac.cpp:7-55): fma chain over the contracted index.
template <int D, int E0, int E1, int E2, int ROWS>
__device__ __forceinline__ void tp_pass(const double* __restrict__ op, const double* in,
                                        double* out, int nb, int tid, int nthr) {
  constexpr int IN_SZ = E0 * E1 * E2;
  constexpr int O0 = D == 0 ? ROWS : E0, O1 = D == 1 ? ROWS : E1, O2 = D == 2 ? ROWS : E2;
  constexpr int OUT_SZ = O0 * O1 * O2;
  constexpr int COLS = D == 0 ? E0 : (D == 1 ? E1 : E2);
  for (int it = tid; it < nb * OUT_SZ; it += nthr) {
    const int b = it / OUT_SZ, r = it - b * OUT_SZ;
    const int i = r % O0, j = (r / O0) % O1, k = r / (O0 * O1);
    const int row = D == 0 ? i : (D == 1 ? j : k);
    const double* src = in + b * IN_SZ;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < COLS; ++a) {
      const int ii = D == 0 ? a : i, jj = D == 1 ? a : j, kk = D == 2 ? a : k;
      acc = fma(op[row * COLS + a], src[ii + E0 * (jj + E1 * kk)], acc);
    }
    out[b * OUT_SZ + r] = acc;
  }
}

// ---------------------------------------------------------------------------
// Metric build (one CTA per element). Control points follow
// mapping_from_function (geometry.cpp:29-60) on the warp of geometry.cpp:62-73.
struct MetricParams {
  const DevTables* tab;
  double* jac;   // [E][N^3]
  double* cof;   // [E][9][N^3]
  double* wj;    // [E][N^3]
  int E, m, k0;
  double x_left, h, beta, l;
  unsigned* err;
};

__device__ __forceinline__ void d_warp(double beta, double l, const double* a, double* x) {
  x[0] = a[0] + beta * sin(a[0] / l) * sin(a[1] / l) * sin(2.0 * a[2] / l);
  x[1] = a[1] + beta * sin(4.0 * a[0] / l) * sin(a[1] / l) * sin(3.0 * a[2] / l);
  x[2] = a[2] + beta * sin(2.0 * a[0] / l) * sin(5.0 * a[1] / l) * sin(a[2] / l);
}

// control point (grid node) of element (ei,ej,ek) at grid indices (i,j,k)
__device__ __forceinline__ void d_control_point(const DevTables& T, int ei, int ej, int ek, int i,
                                                int j, int k, double x_left, double h,
                                                double beta, double l, double* x) {
  const double a[3] = {x_left + (ei + 0.5 * (T.gnodes[i] + 1.0)) * h,
                       x_left + (ej + 0.5 * (T.gnodes[j] + 1.0)) * h,
                       x_left + (ek + 0.5 * (T.gnodes[k] + 1.0)) * h};
  d_warp(beta, l, a, x);
}

// generic (runtime-extent) directional pass for the setup kernels
__device__ __forceinline__ void tp_pass_rt(const double* op, int rows, int D, const double* in,
                                           int e0, int e1, int e2, double* out, int tid,
                                           int nthr) {
  const int o0 = D == 0 ? rows : e0, o1 = D == 1 ? rows : e1, o2 = D == 2 ? rows : e2;
  const int cols = D == 0 ? e0 : (D == 1 ? e1 : e2);
  for (int r = tid; r < o0 * o1 * o2; r += nthr) {
    const int i = r % o0, j = (r / o0) % o1, k = r / (o0 * o1);
    const int row = D == 0 ? i : (D == 1 ? j : k);
    double acc = 0.0;
    for (int a = 0; a < cols; ++a) {
      const int ii = D == 0 ? a : i, jj = D == 1 ? a : j, kk = D == 2 ? a : k;
      acc = fma(op[row * cols + a], in[ii + e0 * (jj + e1 * kk)], acc);
    }
    out[r] = acc;
  }
}

// out = (A (x) A (x) A) in, extents g^3 -> rows^3, via scratch t1/t2
__device__ __forceinline__ void tp3_rt(const double* A, int rows, int g, const double* in,
                                       double* t1, double* t2, double* out, int tid, int nthr) {
  tp_pass_rt(A, rows, 0, in, g, g, g, t1, tid, nthr);
  __syncthreads();
  tp_pass_rt(A, rows, 1, t1, rows, g, g, t2, tid, nthr);
  __syncthreads();
  tp_pass_rt(A, rows, 2, t2, rows, rows, g, out, tid, nthr);
  __syncthreads();
}

__global__ void k_metrics(MetricParams P) {
  extern __shared__ double sm[];
  dbg_kernel_entry(sm);
  const DevTables& T = *P.tab;
  const int e = NSFR_BID;
  if (e >= P.E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int g = T.g, nq = T.nq, G3 = g * g * g, N3 = nq * nq * nq;
  const int M = g > nq ? g : nq, M3 = M * M * M;
  double* xg = sm;                 // 3 * G3
  double* dxg = xg + 3 * G3;       // 9 * G3   [m][k]
  double* t1 = dxg + 9 * G3;       // M3
  double* t2 = t1 + M3;            // M3
  double* dxq = t2 + M3;           // 9 * N3   [m][k]
  double* aq = dxq + 9 * N3;       // 9 * N3   [n][k]
  double* ag = aq + 9 * N3;        // G3
  double* d1 = ag + G3;            // N3
  double* d2 = d1 + N3;            // N3
  const int m = P.m;
  const int ei = e % m, ej = (e / m) % m, ek = e / (m * m) + P.k0;
  for (int node = tid; node < G3; node += nthr) {
    const int i = node % g, j = (node / g) % g, k = node / (g * g);
    double x[3];
    d_control_point(T, ei, ej, ek, i, j, k, P.x_left, P.h, P.beta, P.l, x);
    xg[node] = x[0];
    xg[G3 + node] = x[1];
    xg[2 * G3 + node] = x[2];
  }
  __syncthreads();
  // dx_m/dxi_k at grid nodes (geometry.cpp:129-137)
  for (int mm = 0; mm < 3; ++mm)
    for (int k = 0; k < 3; ++k) tp_pass_rt(T.dg, g, k, xg + mm * G3, g, g, g, dxg + (3 * mm + k) * G3, tid, nthr);
  __syncthreads();
  for (int q = 0; q < 9; ++q) tp3_rt(T.ig, nq, g, dxg + q * G3, t1, t2, dxq + q * N3, tid, nthr);
  // Jacobian determinant (geometry.cpp:139-149)
  for (int q = tid; q < N3; q += nthr) {
    const double a11 = dxq[0 * N3 + q], a12 = dxq[1 * N3 + q], a13 = dxq[2 * N3 + q];
    const double a21 = dxq[3 * N3 + q], a22 = dxq[4 * N3 + q], a23 = dxq[5 * N3 + q];
    const double a31 = dxq[6 * N3 + q], a32 = dxq[7 * N3 + q], a33 = dxq[8 * N3 + q];
    const double J = a11 * (a22 * a33 - a23 * a32) - a12 * (a21 * a33 - a23 * a31) +
                     a13 * (a21 * a32 - a22 * a31);
    if (!(J > 0.0)) atomicOr(P.err, ERR_MESH);
    P.jac[(size_t)e * N3 + q] = J;
    const int i = q % nq, j = (q / nq) % nq, k = q / (nq * nq);
    double w = T.wq[i];
    w *= T.wq[j];
    w *= T.wq[k];
    P.wj[(size_t)e * N3 + q] = 1.0 / (w * J);  // the WA inverse multiplies by 1/(w J)
  }
  // conservative curl (geometry.cpp:174-199)
  for (int n = 0; n < 3; ++n) {
    const int mm = (n + 1) % 3, ll = (n + 2) % 3;
    for (int k = 0; k < 3; ++k) {
      __syncthreads();
      for (int node = tid; node < G3; node += nthr)
        ag[node] = 0.5 * (xg[ll * G3 + node] * dxg[(3 * mm + k) * G3 + node] -
                          xg[mm * G3 + node] * dxg[(3 * ll + k) * G3 + node]);
      __syncthreads();
      tp3_rt(T.ig, nq, g, ag, t1, t2, aq + (3 * n + k) * N3, tid, nthr);
    }
  }
  double* C = P.cof + (size_t)e * 9 * N3;
  for (int n = 0; n < 3; ++n)
    for (int i = 0; i < 3; ++i) {
      const int j = (i + 1) % 3, k = (i + 2) % 3;
      __syncthreads();
      tp_pass_rt(T.quad_diff, nq, k, aq + (3 * n + j) * N3, nq, nq, nq, d1, tid, nthr);
      tp_pass_rt(T.quad_diff, nq, j, aq + (3 * n + k) * N3, nq, nq, nq, d2, tid, nthr);
      __syncthreads();
      // stored pre-halved: K2 uses 0.5 (C_i + C_j) = Ch_i + Ch_j exactly
      for (int q = tid; q < N3; q += nthr) C[(3 * n + i) * N3 + q] = 0.5 * (d1[q] - d2[q]);
    }
  __syncthreads();
  // face normals must be nondegenerate (geometry.cpp:227-233)
  for (int it = tid; it < 6 * nq * nq; it += nthr) {
    const int f = it / (nq * nq), node = it % (nq * nq), dir = f / 2, side = f % 2;
    const int t1i = node % nq, t2i = node / nq;
    double v2 = 0.0;
    for (int n = 0; n < 3; ++n) {
      double cf = 0.0;
      for (int a = 0; a < nq; ++a) {
        const int q = dir == 0 ? a + nq * (t1i + nq * t2i)
                               : (dir == 1 ? t1i + nq * (a + nq * t2i) : t1i + nq * (t2i + nq * a));
        cf = fma(T.bflux[side * nq + a], 2.0 * C[(3 * n + dir) * N3 + q], cf);
      }
      v2 += cf * cf;
    }
    if (!(sqrt(v2) > 0.0)) atomicOr(P.err, ERR_MESH);
  }
}

// ---------------------------------------------------------------------------
// Initial state at the solution nodes: u_hat = IC(x_sol), x_sol = is^3 xg.
struct InitParams {
  const DevTables* tab;
  double* u;
  int E, m, k0, kind;
  double x_left, h, beta, l, gamma;
};

__global__ void k_init(InitParams P) {
  extern __shared__ double sm[];
  dbg_kernel_entry(sm);
  const DevTables& T = *P.tab;
  const int e = NSFR_BID;
  if (e >= P.E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int g = T.g, np = T.np, G3 = g * g * g, S3 = np * np * np;
  const int M = g > np ? g : np, M3 = M * M * M;
  double* xg = sm;
  double* t1 = xg + 3 * G3;
  double* t2 = t1 + M3;
  double* xs = t2 + M3;  // 3 * S3
  const int m = P.m;
  const int ei = e % m, ej = (e / m) % m, ek = e / (m * m) + P.k0;
  for (int node = tid; node < G3; node += nthr) {
    const int i = node % g, j = (node / g) % g, k = node / (g * g);
    double x[3];
    d_control_point(T, ei, ej, ek, i, j, k, P.x_left, P.h, P.beta, P.l, x);
    xg[node] = x[0];
    xg[G3 + node] = x[1];
    xg[2 * G3 + node] = x[2];
  }
  __syncthreads();
  for (int d = 0; d < 3; ++d) tp3_rt(T.is, np, g, xg + d * G3, t1, t2, xs + d * S3, tid, nthr);
  for (int q = tid; q < S3; q += nthr) {
    double st[NS];
    d_case_state(P.kind, P.gamma, xs[q], xs[S3 + q], xs[2 * S3 + q], 0.0, st);
#pragma unroll
    for (int s = 0; s < NS; ++s) P.u[((size_t)e * NS + s) * S3 + q] = st[s];
  }
}


// ---------------------------------------------------------------------------
// State representation change at the API boundary: the solver carries u at the
// volume quadrature nodes, u_q = chi^3 u_hat (the reference's S1); the API
// speaks the reference's solution-node coefficients u_hat = Pi^3 u_q (Pi = chi^-1
// for n_q = n_p). One CTA per element, 5 states.
__global__ void k_convert(const DevTables* tab, const double* in, double* out, int E, int to_quad) {
  extern __shared__ double sm[];
  dbg_kernel_entry(sm);
  const DevTables& T = *tab;
  const int e = NSFR_BID;
  if (e >= E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int np = T.np, nq = T.nq;
  const int nin = to_quad ? np : nq, nout = to_quad ? nq : np;  // chi: nq x np, Pi: np x nq
  const int IN3 = nin * nin * nin, OUT3 = nout * nout * nout;
  const int M = np > nq ? np : nq, M3 = M * M * M;
  double* src = sm;
  double* t1 = src + M3;
  double* t2 = t1 + M3;
  double* dst = t2 + M3;
  for (int s = 0; s < NS; ++s) {
    for (int i = tid; i < IN3; i += nthr) src[i] = in[((size_t)e * NS + s) * IN3 + i];
    __syncthreads();
    tp3_rt(to_quad ? T.interp : T.proj, nout, nin, src, t1, t2, dst, tid, nthr);
    for (int i = tid; i < OUT3; i += nthr) out[((size_t)e * NS + s) * OUT3 + i] = dst[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// L2 error partials: per element sum w J (rho - rho_ex)^2 and (p - p_ex)^2.
struct L2Params {
  const DevTables* tab;
  const double* u;
  const double* jac;
  double* part;  // [E][2]
  int E, m, k0, kind;
  double x_left, h, beta, l, gamma, t;
};

__global__ void k_l2(L2Params P) {
  extern __shared__ double sm[];
  dbg_kernel_entry(sm);
  const DevTables& T = *P.tab;
  const int e = NSFR_BID;
  if (e >= P.E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int g = T.g, n = T.nq, G3 = g * g * g, N3 = n * n * n;
  const int M = g > n ? g : n, M3 = M * M * M;
  double* xg = sm;
  double* t1 = xg + 3 * G3;
  double* t2 = t1 + M3;
  double* xv = t2 + M3;   // 3*N3
  double* uq = xv + 3 * N3;  // 5*N3
  double* pr = uq + 5 * N3;  // 2*N3
  const int m = P.m;
  const int ei = e % m, ej = (e / m) % m, ek = e / (m * m) + P.k0;
  for (int node = tid; node < G3; node += nthr) {
    const int i = node % g, j = (node / g) % g, k = node / (g * g);
    double x[3];
    d_control_point(T, ei, ej, ek, i, j, k, P.x_left, P.h, P.beta, P.l, x);
    xg[node] = x[0];
    xg[G3 + node] = x[1];
    xg[2 * G3 + node] = x[2];
  }
  __syncthreads();
  for (int d = 0; d < 3; ++d) tp3_rt(T.ig, n, g, xg + d * G3, t1, t2, xv + d * N3, tid, nthr);
  // the device state already holds u at the volume quadrature nodes (chi^3 u_hat)
  for (int i = tid; i < NS * N3; i += nthr) uq[i] = P.u[(size_t)e * NS * N3 + i];
  __syncthreads();
  for (int q = tid; q < N3; q += nthr) {
    const int i = q % n, j = (q / n) % n, k = q / (n * n);
    double w = T.wq[i];
    w *= T.wq[j];
    w *= T.wq[k];
    const double wj = w * P.jac[(size_t)e * N3 + q];
    double uu[NS], ex[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] = uq[s * N3 + q];
    d_case_state(P.kind, P.gamma, xv[q], xv[N3 + q], xv[2 * N3 + q], P.t, ex);
    const double dr = uu[0] - ex[0];
    const double dp = d_pressure(P.gamma, uu) - d_pressure(P.gamma, ex);
    pr[q] = wj * dr * dr;
    pr[N3 + q] = wj * dp * dp;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < N3; ++q) {
      a += pr[q];
      b += pr[N3 + q];
    }
    P.part[2 * (size_t)e] = a;
    P.part[2 * (size_t)e + 1] = b;
  }
}

// Deterministic two-level sum of `ncomp` interleaved components over n items.
__global__ void k_reduce(const double* in, int n, int ncomp, double* out) {
  __shared__ double sh[1024];
  for (int c = 0; c < ncomp; ++c) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += in[(size_t)i * ncomp + c];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = sh[0];
    __syncthreads();
  }
}

// Totals per element: sum_q w J u_q[s] (mass, momentum, energy; SPEC.md:587
// DiagnosticRecord, Thm 3 drift SPEC.md:650) and sum_q w J U(u_q) with the
// entropy function U = -rho s/(gamma-1) (the |U_total| normaliser of
// SPEC.md:654). part[E][6]; fixed-order sums.
constexpr int NTOT = NS + 1;
__global__ void k_totals(const DevTables* tab, const double* u, const double* jac, double gamma,
                         double* part, int E) {
  __shared__ double red[NTOT][128];
  const DevTables& T = *tab;
  const int e = NSFR_BID;
  if (e >= E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;  // nthr <= 128
  const int n = T.nq, N3 = n * n * n;
  double acc[NTOT] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int q = tid; q < N3; q += nthr) {
    const int i = q % n, j = (q / n) % n, k = q / (n * n);
    double w = T.wq[i];
    w *= T.wq[j];
    w *= T.wq[k];
    const double wj = w * jac[(size_t)e * N3 + q];
    double uu[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uu[s] = u[((size_t)e * NS + s) * N3 + q];
      acc[s] += wj * uu[s];
    }
    const double sp = log(d_pressure(gamma, uu)) - gamma * log(uu[0]);
    acc[NS] += wj * (-uu[0] * sp / (gamma - 1.0));
  }
#pragma unroll
  for (int s = 0; s < NTOT; ++s) red[s][tid] = acc[s];
  __syncthreads();
  if (tid < NTOT) {
    double t = 0.0;
    for (int r = 0; r < nthr; ++r) t += red[tid][r];
    part[(size_t)e * NTOT + tid] = t;
  }
}

// Kinetic-energy volume term per element: sum_q v_KE(u_q) . vol_q with the
// volume rows of k_residual<N, true> (flux minus pressure work, S6 only) and
// v_KE = (-|v|^2/2, v_x, v_y, v_z, 0). Fixed-order sums.
__global__ void k_ke_dot(const double* u, const double* vol, int N3, double* part, int E) {
  __shared__ double red[128];
  const int e = NSFR_BID;
  if (e >= E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;  // nthr <= 128
  const double* ue = u + (size_t)e * NS * N3;
  const double* ve = vol + (size_t)e * NS * N3;
  double acc = 0.0;
  for (int q = tid; q < N3; q += nthr) {
    const double iu = 1.0 / ue[q];  // kinetic_energy_variables, euler.cpp:83-87
    const double vx = ue[N3 + q] * iu, vy = ue[2 * N3 + q] * iu, vz = ue[3 * N3 + q] * iu;
    const double vk0 = -0.5 * (vx * vx + vy * vy + vz * vz);
    acc += vk0 * ve[q] + vx * ve[N3 + q] + vy * ve[2 * N3 + q] + vz * ve[3 * N3 + q];
  }
  red[tid] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < nthr; ++i) t += red[i];
    part[e] = t;
  }
}

// Kinetic-energy variables projected to the solution nodes: v_hat_KE =
// Pi^3 v_KE(u_q), v_KE = (-|v|^2/2, v, 0) (kinetic_energy_variables,
// euler.cpp:83-87), for the KE change diagnostic. One CTA per element.
__global__ void k_ke_vars(const DevTables* tab, const double* uq, double* vhat, int E) {
  extern __shared__ double sm[];
  dbg_kernel_entry(sm);
  const DevTables& T = *tab;
  const int e = NSFR_BID;
  if (e >= E) return;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int n = T.nq, N3 = n * n * n;  // n_q = n_p
  double* vk = sm;
  double* t1 = vk + N3;
  double* t2 = t1 + N3;
  double* dst = t2 + N3;
  const double* ue = uq + (size_t)e * NS * N3;
  for (int s = 0; s < NS; ++s) {
    for (int q = tid; q < N3; q += nthr) {
      const double iu = 1.0 / ue[q];
      const double vx = ue[N3 + q] * iu, vy = ue[2 * N3 + q] * iu, vz = ue[3 * N3 + q] * iu;
      vk[q] = s == 0 ? -0.5 * (vx * vx + vy * vy + vz * vz) : (s == 1 ? vx : (s == 2 ? vy : (s == 3 ? vz : 0.0)));
    }
    __syncthreads();
    tp3_rt(T.proj, n, n, vk, t1, t2, dst, tid, nthr);
    for (int i = tid; i < N3; i += nthr) vhat[((size_t)e * NS + s) * N3 + i] = dst[i];
    __syncthreads();
  }
}

// Step bookkeeping: reset lambda, compute dt from lambda.
struct StepState {
  double t, dt, t_final, cfl, dx;
  unsigned long long lam_bits;
  int active;
  unsigned long long lam_out_bits;  // streamed step: lambda_max of the state handed back
  double dt_next;                   // adaptive_dt of that state
};

__global__ void k_step_begin(StepState* S) {
  S->lam_bits = 0ull;
  S->lam_out_bits = 0ull;
}

// adaptive_dt: cfl dx / lambda_max, clipped to t_final - t
__device__ __forceinline__ double step_dt_of(const StepState* S, unsigned long long bits) {
  const double lam = __longlong_as_double(static_cast<long long>(bits));
  double dt = lam > 0.0 ? S->cfl * S->dx / lam : S->cfl * S->dx;
  if (S->t_final > 0.0) {
    if (S->t >= S->t_final)
      dt = 0.0;
    else
      dt = fmin(dt, S->t_final - S->t);
  }
  return dt;
}

__global__ void k_step_dt(StepState* S) {
  S->dt = step_dt_of(S, S->lam_bits);
  S->lam_bits = 0ull;  // K3 of the last stage accumulates the next step's lambda
}

__global__ void k_step_end(StepState* S) { S->t += S->dt; }

// after k_step_end: the dt the next step would take from the output state
__global__ void k_step_next(StepState* S) { S->dt_next = step_dt_of(S, S->lam_out_bits); }

}  // namespace nsfr_b200
