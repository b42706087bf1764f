// sm_100a fp64 kernels of the NSFR per-stage residual.
//
//   k_metrics   device build of J and the conservative-curl cofactors
//               (geometry.cpp:86-266) from the closed-form warp (geometry.cpp:62-73)
//   k_init      initial state at the LGL solution nodes (cases.cpp)
//   k_project   K1: entropy projection S1-S5, face traces,
//               optional lambda_max for adaptive dt
//   k_residual  K2: volume Hadamard (sumfac.hpp:48-94), hybrid surface Hadamard
//               (sumfac.hpp:110-157), EC+Roe face flux (euler.cpp:142-162,229-301),
//               chi^T lifting, weight-adjusted inverse (fr_operators.cpp:280-309),
//               fused RK4 stage update
//   k_l2        L2 error partials
//
// Layout in HBM (element-contiguous blocks, xi fastest):
//   state/us/acc/ut_vol [E][5][N^3]; traces [E][6][5][N^2]; cof [E][9][N^3]
//   (component 3*n_phys + i_ref major); wj [E][N^3] = w_i w_j w_k J.
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
  const DevTables& T = *P.tab;
  const int e = blockIdx.x;
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
    P.wj[(size_t)e * N3 + q] = w * J;
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
      for (int q = tid; q < N3; q += nthr) C[(3 * n + i) * N3 + q] = d1[q] - d2[q];
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
        cf = fma(T.bflux[side * nq + a], C[(3 * n + dir) * N3 + q], cf);
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
  const DevTables& T = *P.tab;
  const int e = blockIdx.x;
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
// K1: entropy projection. EPB elements per CTA, threads over nodes.
struct ProjParams {
  const DevTables* tab;
  const double* u;       // [E][5][N^3] stage input
  double* ut_vol;        // [E][5][N^3] entropy-projected conservative (volume)
  double* traces;        // [E][6][5][N^2]
  double* vhat;          // [E][5][N^3] or nullptr
  double* send_lo;       // [m*m][5][N^2] face 4 of plane 0, or nullptr
  double* send_hi;       // [m*m][5][N^2] face 5 of plane nz-1, or nullptr
  unsigned long long* lam;  // lambda_max bits or nullptr
  unsigned* err;
  int E, m, nz;
  double gamma;
};

template <int N>
struct ProjCfg {
  static constexpr int N2 = N * N, N3 = N * N * N;
  static constexpr int EPB = N3 <= 32 ? 8 : (N3 <= 64 ? 4 : (N3 <= 128 ? 2 : 1));
  static constexpr int THREADS = ((EPB * N3 + 31) / 32) * 32;
  // smem doubles: tables + A,B,V,C4 (5N^3 each) + T0,T0b,T1 (10N^2 each) + F (30N^2)
  static constexpr int TAB = 2 * N2 + 2 * N;
  static constexpr int PER_EL = 20 * N3 + 60 * N2;
  static constexpr int SMEM = (TAB + EPB * PER_EL) * 8;
};

template <int N>
__global__ void __launch_bounds__(ProjCfg<N>::THREADS) k_project(ProjParams P) {
  using Cfg = ProjCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, EPB = Cfg::EPB;
  extern __shared__ double sm[];
  double* s_interp = sm;            // N x N
  double* s_proj = s_interp + N2;   // N x N
  double* s_bsol = s_proj + N2;     // 2 x N
  double* base = sm + Cfg::TAB;
  double* A = base;
  double* B = A + EPB * 5 * N3;
  double* V = B + EPB * 5 * N3;
  double* C4 = V + EPB * 5 * N3;
  double* T0 = C4 + EPB * 5 * N3;   // [EPB][2][5][N2]  dir0: bs_xi v_hat
  double* T0b = T0 + EPB * 10 * N2; // [EPB][2][5][N2]
  double* T1 = T0b + EPB * 10 * N2; // [EPB][2][5][N2]  dir1: bs_eta X
  double* F = T1 + EPB * 10 * N2;   // [EPB][6][5][N2]  final face v~
  const DevTables& T = *P.tab;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int e0 = blockIdx.x * EPB;
  const int nb = min(EPB, P.E - e0);
  const double g = P.gamma;
  for (int i = tid; i < N2; i += nthr) {
    s_interp[i] = T.interp[i];
    s_proj[i] = T.proj[i];
  }
  for (int i = tid; i < 2 * N; i += nthr) s_bsol[i] = T.bsol[i];
  {
    const double* src = P.u + (size_t)e0 * 5 * N3;
    for (int i = tid; i < nb * 5 * N3; i += nthr) A[i] = src[i];
  }
  __syncthreads();
  const int nbs = nb * 5;
  // S1 u_q = chi^3 u_hat
  tp_pass<0, N, N, N, N>(s_interp, A, B, nbs, tid, nthr);
  __syncthreads();
  tp_pass<1, N, N, N, N>(s_interp, B, A, nbs, tid, nthr);
  __syncthreads();
  tp_pass<2, N, N, N, N>(s_interp, A, B, nbs, tid, nthr);
  __syncthreads();
  // S2 v(u_q), and the wavespeed for adaptive dt
  double lam = 0.0;
  for (int it = tid; it < nb * N3; it += nthr) {
    const int b = it / N3, q = it - b * N3;
    double uu[NS], vv[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] = B[(b * 5 + s) * N3 + q];
    if (!d_entropy_vars(g, uu, vv)) {
      atomicOr(P.err, ERR_STATE);
#pragma unroll
      for (int s = 0; s < NS; ++s) vv[s] = (s == 4) ? -1.0 : 0.0;
    } else if (P.lam) {
      const double vx = uu[1] / uu[0], vy = uu[2] / uu[0], vz = uu[3] / uu[0];
      const double speed = sqrt(vx * vx + vy * vy + vz * vz);
      const double a = sqrt(g * d_pressure(g, uu) / uu[0]);
      lam = fmax(lam, speed + a);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) B[(b * 5 + s) * N3 + q] = vv[s];
  }
  if (P.lam) {
    for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
    if ((tid & 31) == 0 && lam > 0.0) atomicMax(P.lam, dbl_bits(lam));
  }
  __syncthreads();
  // S3 v_hat = Pi^3 v_q
  tp_pass<0, N, N, N, N>(s_proj, B, A, nbs, tid, nthr);
  __syncthreads();
  tp_pass<1, N, N, N, N>(s_proj, A, B, nbs, tid, nthr);
  __syncthreads();
  tp_pass<2, N, N, N, N>(s_proj, B, V, nbs, tid, nthr);
  __syncthreads();
  if (P.vhat) {
    double* dst = P.vhat + (size_t)e0 * 5 * N3;
    for (int i = tid; i < nb * 5 * N3; i += nthr) dst[i] = V[i];
  }
  // S4: X = chi_xi V (A), XY = chi_eta X (B); dir0 faces contract V along xi
  tp_pass<0, N, N, N, N>(s_interp, V, A, nbs, tid, nthr);
  for (int it = tid; it < nbs * 2 * N2; it += nthr) {  // T0[b][side][s][j,k]
    const int bs5 = it / (2 * N2), r = it - bs5 * 2 * N2, side = r / N2, jk = r - side * N2;
    const double* src = V + bs5 * N3 + jk * N;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) acc = fma(s_bsol[side * N + a], src[a], acc);
    const int b = bs5 / 5, s = bs5 - b * 5;
    T0[((b * 2 + side) * 5 + s) * N2 + jk] = acc;
  }
  __syncthreads();
  tp_pass<1, N, N, N, N>(s_interp, A, B, nbs, tid, nthr);
  for (int it = tid; it < nbs * 2 * N2; it += nthr) {  // T1[b][side][s][i,k] = bs_eta X
    const int bs5 = it / (2 * N2), r = it - bs5 * 2 * N2, side = r / N2, ik = r - side * N2;
    const int i = ik % N, k = ik / N;
    const double* src = A + bs5 * N3 + i + N2 * k;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) acc = fma(s_bsol[side * N + a], src[a * N], acc);
    const int b = bs5 / 5, s = bs5 - b * 5;
    T1[((b * 2 + side) * 5 + s) * N2 + ik] = acc;
  }
  for (int it = tid; it < nbs * 2 * N2; it += nthr) {  // T0b = chi_eta T0
    const int bs5 = it / (2 * N2), r = it - bs5 * 2 * N2, side = r / N2, jk = r - side * N2;
    const int j = jk % N, k = jk / N;
    const int b = bs5 / 5, s = bs5 - b * 5;
    const double* src = T0 + ((b * 2 + side) * 5 + s) * N2 + k * N;
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) acc = fma(s_interp[j * N + a], src[a], acc);
    T0b[((b * 2 + side) * 5 + s) * N2 + jk] = acc;
  }
  __syncthreads();
  // v~ volume (C4 = chi_zeta XY); dir2 faces bs_zeta XY; dir1 faces chi_zeta T1;
  // dir0 faces chi_zeta T0b
  tp_pass<2, N, N, N, N>(s_interp, B, C4, nbs, tid, nthr);
  for (int it = tid; it < nbs * 2 * N2; it += nthr) {
    const int bs5 = it / (2 * N2), r = it - bs5 * 2 * N2, side = r / N2, ij = r - side * N2;
    const int b = bs5 / 5, s = bs5 - b * 5;
    {  // dir 2: F[b][4+side][s][i,j]
      const double* src = B + bs5 * N3 + ij;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_bsol[side * N + a], src[a * N2], acc);
      F[((b * 6 + 4 + side) * 5 + s) * N2 + ij] = acc;
    }
    {  // dir 1: F[b][2+side][s][i,k'] = sum_k chi(k',k) T1[i,k]
      const int i = ij % N, kp = ij / N;
      const double* src = T1 + ((b * 2 + side) * 5 + s) * N2 + i;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp[kp * N + a], src[a * N], acc);
      F[((b * 6 + 2 + side) * 5 + s) * N2 + ij] = acc;
    }
    {  // dir 0: F[b][side][s][j',k'] = sum_k chi(k',k) T0b[j',k]
      const int jp = ij % N, kp = ij / N;
      const double* src = T0b + ((b * 2 + side) * 5 + s) * N2 + jp;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp[kp * N + a], src[a * N], acc);
      F[((b * 6 + side) * 5 + s) * N2 + ij] = acc;
    }
  }
  __syncthreads();
  // S5 u~ = u(v~) at volume and face nodes
  for (int it = tid; it < nb * N3; it += nthr) {
    const int b = it / N3, q = it - b * N3;
    double vv[NS], uu[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) vv[s] = C4[(b * 5 + s) * N3 + q];
    if (!d_entropy_to_cons(g, vv, uu)) atomicOr(P.err, ERR_STATE);
    double* dst = P.ut_vol + (size_t)(e0 + b) * 5 * N3 + q;
#pragma unroll
    for (int s = 0; s < NS; ++s) dst[s * N3] = uu[s];
  }
  for (int it = tid; it < nb * 6 * N2; it += nthr) {
    const int b = it / (6 * N2), r = it - b * 6 * N2, f = r / N2, k = r - f * N2;
    double vv[NS], uu[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) vv[s] = F[((b * 6 + f) * 5 + s) * N2 + k];
    if (!d_entropy_to_cons(g, vv, uu)) atomicOr(P.err, ERR_STATE);
    const int e = e0 + b;
    double* dst = P.traces + ((size_t)e * 6 + f) * 5 * N2 + k;
#pragma unroll
    for (int s = 0; s < NS; ++s) dst[s * N2] = uu[s];
    // boundary planes also go to the halo send buffers
    const int mm = P.m * P.m, kl = e / mm, plane = e - kl * mm;
    if (P.send_lo && f == 4 && kl == 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) P.send_lo[((size_t)plane * 5 + s) * N2 + k] = uu[s];
    }
    if (P.send_hi && f == 5 && kl == P.nz - 1) {
#pragma unroll
      for (int s = 0; s < NS; ++s) P.send_hi[((size_t)plane * 5 + s) * N2 + k] = uu[s];
    }
  }
}

// ---------------------------------------------------------------------------
// K2: residual + lifting + weight-adjusted inverse + RK stage update.
struct ResParams {
  const DevTables* tab;
  const double* ut_vol;   // [E][5][N^3]
  const double* traces;   // [E][6][5][N^2]
  const double* halo_lo;  // [m*m][5][N^2] face 5 of plane k0-1 (nullptr: wrap locally)
  const double* halo_hi;  // [m*m][5][N^2] face 4 of plane k1
  const double* cof;      // [E][9][N^3]
  const double* wj;       // [E][N^3]
  const double* vhat;     // [E][5][N^3] or nullptr
  double* dS;             // [E] or nullptr
  double* un;             // RK base state (stage 4 writes it)
  double* us;             // next stage state
  double* acc;            // RK accumulator
  double* out;            // stage 0: dU/dt
  const double* dt;       // device scalar
  unsigned* err;
  int stage, E, m, nz;
  double gamma;
  int roe;
};

template <int N>
struct ResCfg {
  static constexpr int N2 = N * N, N3 = N * N * N;
  static constexpr int LINES = 3 * N2;
  static constexpr int EPB = LINES <= 32 ? 6 : (LINES <= 64 ? 4 : 2);
  static constexpr int THREADS = ((EPB * LINES + 31) / 32) * 32;
  static constexpr int TAB = 4 * N2 + 5 * N + N2;  // interp_t, frproj, frproj_t, qskew, bflux, bsol, wq, pad
  static constexpr int WORK = (15 * N3 > 10 * N3 + 30 * N2) ? 15 * N3 : 10 * N3 + 30 * N2;
  static constexpr int PER_EL = 15 * N3 + 30 * N2 + WORK;
  static constexpr int SMEM = (TAB + EPB * PER_EL) * 8;
  static constexpr int MINB = SMEM <= 56 * 1024 ? 4 : (SMEM <= 75 * 1024 ? 3 : (SMEM <= 112 * 1024 ? 2 : 1));
};

template <int N>
__global__ void __launch_bounds__(ResCfg<N>::THREADS, ResCfg<N>::MINB) k_residual(ResParams P) {
  using Cfg = ResCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, EPB = Cfg::EPB, LINES = Cfg::LINES;
  extern __shared__ double sm[];
  double* s_interp_t = sm;              // N x N  (chi^T)
  double* s_fr = s_interp_t + N2;       // N x N  (Pi~)
  double* s_fr_t = s_fr + N2;           // N x N  (Pi~^T)
  double* s_q = s_fr_t + N2;            // N x N  skew(a,b)
  double* s_bflux = s_q + N2;           // 2N
  double* s_bsol = s_bflux + 2 * N;     // 2N
  double* s_wq = s_bsol + 2 * N;        // N
  double* base = sm + Cfg::TAB;
  double* ACCV = base;                          // [EPB][3][5][N3]
  double* FACC = ACCV + EPB * 15 * N3;          // [EPB][6][5][N2]
  double* WORK = FACC + EPB * 30 * N2;          // [EPB][WORK]
  const DevTables& T = *P.tab;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int e0 = blockIdx.x * EPB;
  const int nb = min(EPB, P.E - e0);
  const double g = P.gamma;
  const Gas G{g, g - 1.0, 1.0 / (g - 1.0)};
  for (int i = tid; i < N2; i += nthr) {
    s_interp_t[i] = T.interp_t[i];
    s_fr[i] = T.frproj[i];
    s_fr_t[i] = T.frproj_t[i];
    s_q[i] = T.qskew[i];
  }
  for (int i = tid; i < 2 * N; i += nthr) {
    s_bflux[i] = T.bflux[i];
    s_bsol[i] = T.bsol[i];
  }
  for (int i = tid; i < N; i += nthr) s_wq[i] = T.wq[i];
  // stage element data: primitives of u~ and 0.5*C
  for (int it = tid; it < nb * N3; it += nthr) {
    const int b = it / N3, q = it - b * N3;
    const double* src = P.ut_vol + (size_t)(e0 + b) * 5 * N3 + q;
    double uc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uc[s] = src[s * N3];
    const Prim pr = d_prim(g, uc);
    double* Pd = WORK + b * Cfg::WORK;
    Pd[0 * N3 + q] = pr.rho;
    Pd[1 * N3 + q] = pr.u;
    Pd[2 * N3 + q] = pr.v;
    Pd[3 * N3 + q] = pr.w;
    Pd[4 * N3 + q] = pr.p;
    Pd[5 * N3 + q] = pr.rp;
  }
  for (int it = tid; it < nb * 9 * N3; it += nthr) {
    const int b = it / (9 * N3), r = it - b * 9 * N3;
    WORK[b * Cfg::WORK + 6 * N3 + r] = 0.5 * P.cof[(size_t)(e0 + b) * 9 * N3 + r];
  }
  __syncthreads();

  // ---- line phase: one thread owns one 1D line (dir, t1, t2) ----
  {
    const int b = tid / LINES;
    const int l = tid - b * LINES;
    if (b < nb) {
      const int e = e0 + b;
      const int dir = l / N2, rem = l - dir * N2, t1 = rem % N, t2 = rem / N;
      const int stride = dir == 0 ? 1 : (dir == 1 ? N : N2);
      const int lbase = dir == 0 ? N * (t1 + N * t2) : (dir == 1 ? t1 + N2 * t2 : t1 + N * t2);
      const double* Pd = WORK + b * Cfg::WORK;
      const double* Ch = Pd + 6 * N3;
      double* acc = ACCV + (b * 3 + dir) * 5 * N3;
      const double wt = s_wq[t1] * s_wq[t2];
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int s = 0; s < NS; ++s) acc[s * N3 + lbase + a * stride] = 0.0;
      // S6 volume pairs a<b
#pragma unroll 1
      for (int a = 0; a < N - 1; ++a) {
        const int ia = lbase + a * stride;
        const Prim pa{Pd[ia], Pd[N3 + ia], Pd[2 * N3 + ia], Pd[3 * N3 + ia], Pd[4 * N3 + ia], Pd[5 * N3 + ia]};
        const double ca0 = Ch[(0 + dir) * N3 + ia], ca1 = Ch[(3 + dir) * N3 + ia],
                     ca2 = Ch[(6 + dir) * N3 + ia];
        double fa[NS] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
        for (int bb = a + 1; bb < N; ++bb) {
          const int ib = lbase + bb * stride;
          const Prim pb{Pd[ib], Pd[N3 + ib], Pd[2 * N3 + ib], Pd[3 * N3 + ib], Pd[4 * N3 + ib], Pd[5 * N3 + ib]};
          double f[NS];
          d_flux_contract(G, pa, pb, ca0 + Ch[(0 + dir) * N3 + ib], ca1 + Ch[(3 + dir) * N3 + ib],
                          ca2 + Ch[(6 + dir) * N3 + ib], f);
          const double c = wt * s_q[a * N + bb];
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            fa[s] = fma(c, f[s], fa[s]);
            acc[s * N3 + ib] = fma(-c, f[s], acc[s * N3 + ib]);
          }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) acc[s * N3 + ia] += fa[s];
      }
      // S7 + S8 for the two faces this line pierces
#pragma unroll 1
      for (int side = 0; side < 2; ++side) {
        const int f = 2 * dir + side;
        const double sign = side ? 1.0 : -1.0;
        const int k = t1 + N * t2;
        double uf[NS], un[NS];
        const double* tr = P.traces + ((size_t)e * 6 + f) * 5 * N2 + k;
#pragma unroll
        for (int s = 0; s < NS; ++s) uf[s] = tr[s * N2];
        // neighbour across face f (geometry.hpp:24-29), its face f^1, same node k
        {
          const int mm = P.m;
          int i = e % mm, j = (e / mm) % mm, kl = e / (mm * mm);
          const int step = side ? 1 : -1;
          const double* nt = nullptr;
          if (dir == 0) i = (i + step + mm) % mm;
          if (dir == 1) j = (j + step + mm) % mm;
          if (dir == 2) {
            kl += step;
            if (kl < 0 || kl >= P.nz) {
              const double* halo = kl < 0 ? P.halo_lo : P.halo_hi;
              if (halo) nt = halo + (size_t)(i + mm * j) * 5 * N2 + k;
              kl = (kl + P.nz) % P.nz;
            }
          }
          if (!nt) nt = P.traces + (((size_t)(i + mm * (j + mm * kl))) * 6 + (f ^ 1)) * 5 * N2 + k;
#pragma unroll
          for (int s = 0; s < NS; ++s) un[s] = nt[s * N2];
        }
        const Prim pf = d_prim(g, uf);
        // own face cofactor column C_f[:,dir] = sum_a bound_flux(side,a) C_a (geometry.cpp:218-226)
        double cf0 = 0.0, cf1 = 0.0, cf2 = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const int ia = lbase + a * stride;
          const double w = s_bflux[side * N + a];
          cf0 = fma(w, 2.0 * Ch[(0 + dir) * N3 + ia], cf0);
          cf1 = fma(w, 2.0 * Ch[(3 + dir) * N3 + ia], cf1);
          cf2 = fma(w, 2.0 * Ch[(6 + dir) * N3 + ia], cf2);
        }
        const double ch0 = 0.5 * cf0, ch1 = 0.5 * cf1, ch2 = 0.5 * cf2;
        double ff[NS] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
        for (int a = 0; a < N; ++a) {
          const int ia = lbase + a * stride;
          const Prim pa{Pd[ia], Pd[N3 + ia], Pd[2 * N3 + ia], Pd[3 * N3 + ia], Pd[4 * N3 + ia], Pd[5 * N3 + ia]};
          double fl[NS];
          d_flux_contract(G, pa, pf, Ch[(0 + dir) * N3 + ia] + ch0, Ch[(3 + dir) * N3 + ia] + ch1,
                          Ch[(6 + dir) * N3 + ia] + ch2, fl);
          const double c = sign * s_bflux[side * N + a] * wt;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            acc[s * N3 + ia] = fma(c, fl[s], acc[s * N3 + ia]);
            ff[s] = fma(-c, fl[s], ff[s]);
          }
        }
        // S8 f*.n with the own unit normal and J^Gamma (geometry.cpp:227-236)
        const double v0 = sign * cf0, v1 = sign * cf1, v2 = sign * cf2;
        const double jg = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
        const double nrm[3] = {v0 / jg, v1 / jg, v2 / jg};
        const Prim pn = d_prim(g, un);
        double fn[NS];
        d_flux_contract(G, pf, pn, nrm[0], nrm[1], nrm[2], fn);
        if (P.roe) {
          double d[NS];
          if (!d_roe(g, uf, un, nrm, d)) atomicOr(P.err, ERR_ROE);
#pragma unroll
          for (int s = 0; s < NS; ++s) fn[s] -= d[s];
        }
        const double cc = wt * jg;
        double* fo = FACC + (b * 6 + f) * 5 * N2 + k;
#pragma unroll
        for (int s = 0; s < NS; ++s) fo[s * N2] = fma(cc, fn[s], ff[s]);
      }
    }
  }
  __syncthreads();

  // ---- S9 lifting: R = chi^T^3 vol + sum_f (bs^T chi^T chi^T) facc ----
  const int nbs = nb * 5;
  for (int it = tid; it < nbs * N3; it += nthr) {  // vol = sum over the 3 directions -> ACCV[b][0]
    const int b = it / (5 * N3), r = it - b * 5 * N3;
    double* a0 = ACCV + b * 15 * N3;
    a0[r] = a0[r] + a0[5 * N3 + r] + a0[10 * N3 + r];
  }
  __syncthreads();
  // vol lift passes use WORK[0:5N3] and WORK[5N3:10N3]; face lift uses WORK[10N3:10N3+30N2]
  {
    // pass xi: vol (ACCV[b][0]) -> WORK[b][0:5N3]
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, jk = q / N;
      const double* src = ACCV + b * 15 * N3 + s * N3 + jk * N;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp_t[i * N + a], src[a], acc);
      WORK[b * Cfg::WORK + r] = acc;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // eta: WORK[0] -> WORK[5N3]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, j = (q / N) % N, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + s * N3 + i + N2 * k;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp_t[j * N + a], src[a * N], acc);
      WORK[b * Cfg::WORK + 5 * N3 + r] = acc;
    }
    // face lifting stage 1: G[b][f][s][t1',t2] = sum_t1 chi^T(t1',t1) facc[f][s][t1,t2]
    for (int it = tid; it < nb * 30 * N2; it += nthr) {
      const int b = it / (30 * N2), r = it - b * 30 * N2, fs = r / N2, k = r - fs * N2;
      const int t1p = k % N, t2 = k / N;
      const double* src = FACC + b * 30 * N2 + fs * N2 + t2 * N;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp_t[t1p * N + a], src[a], acc);
      WORK[b * Cfg::WORK + 10 * N3 + r] = acc;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // zeta: WORK[5N3] -> ACCV[b][1]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int ij = q % N2, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + 5 * N3 + s * N3 + ij;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp_t[k * N + a], src[a * N2], acc);
      ACCV[b * 15 * N3 + 5 * N3 + r] = acc;
    }
    // face lifting stage 2: H[b][f][s][t1',t2'] = sum_t2 chi^T(t2',t2) G[..][t1',t2] -> FACC
    for (int it = tid; it < nb * 30 * N2; it += nthr) {
      const int b = it / (30 * N2), r = it - b * 30 * N2, fs = r / N2, k = r - fs * N2;
      const int t1p = k % N, t2p = k / N;
      const double* src = WORK + b * Cfg::WORK + 10 * N3 + fs * N2 + t1p;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_interp_t[t2p * N + a], src[a * N], acc);
      FACC[b * 30 * N2 + r] = acc;
    }
    __syncthreads();
    // R += sum_f bs(side, a_dir) H_f  (R in ACCV[b][1])
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, j = (q / N) % N, k = q / N2;
      const double* H = FACC + b * 30 * N2;
      double R = ACCV[b * 15 * N3 + 5 * N3 + r];
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        const int dir = f / 2, side = f % 2;
        const int a = dir == 0 ? i : (dir == 1 ? j : k);
        const int fk = dir == 0 ? j + N * k : (dir == 1 ? i + N * k : i + N * j);
        R = fma(s_bsol[side * N + a], H[(f * 5 + s) * N2 + fk], R);
      }
      ACCV[b * 15 * N3 + 5 * N3 + r] = R;
    }
    __syncthreads();
  }
  // D9 entropy change partial: -sum v_hat . R (deterministic per element)
  if (P.dS) {
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int b = it / (5 * N3), r = it - b * 5 * N3;
      WORK[b * Cfg::WORK + r] = P.vhat[(size_t)(e0 + b) * 5 * N3 + r] * ACCV[b * 15 * N3 + 5 * N3 + r];
    }
    __syncthreads();
    if (tid < nb) {
      double acc = 0.0;
      for (int r = 0; r < 5 * N3; ++r) acc += WORK[tid * Cfg::WORK + r];
      P.dS[e0 + tid] = -acc;
    }
    __syncthreads();
  }
  // ---- S10 weight-adjusted inverse: -Pi~ (W J)^-1 Pi~^T R ----
  {
    double* R = ACCV + 5 * N3;  // per element at stride 15*N3
    // Pi~^T along xi: R -> WORK[0]
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, jk = q / N;
      const double* src = R + b * 15 * N3 + s * N3 + jk * N;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr_t[i * N + a], src[a], acc);
      WORK[b * Cfg::WORK + r] = acc;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // eta: WORK[0] -> WORK[5N3]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, j = (q / N) % N, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + s * N3 + i + N2 * k;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr_t[j * N + a], src[a * N], acc);
      WORK[b * Cfg::WORK + 5 * N3 + r] = acc;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // zeta + divide by w J -> ACCV[b][2]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int ij = q % N2, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + 5 * N3 + s * N3 + ij;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr_t[k * N + a], src[a * N2], acc);
      const double wjq = P.wj[(size_t)(e0 + b) * N3 + q];
      if (!(wjq > 0.0)) atomicOr(P.err, ERR_MESH);
      ACCV[b * 15 * N3 + 10 * N3 + r] = acc / wjq;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // Pi~ xi: ACCV[b][2] -> WORK[0]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, jk = q / N;
      const double* src = ACCV + b * 15 * N3 + 10 * N3 + s * N3 + jk * N;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr[i * N + a], src[a], acc);
      WORK[b * Cfg::WORK + r] = acc;
    }
    __syncthreads();
    for (int it = tid; it < nbs * N3; it += nthr) {  // eta: WORK[0] -> WORK[5N3]
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int i = q % N, j = (q / N) % N, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + s * N3 + i + N2 * k;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr[j * N + a], src[a * N], acc);
      WORK[b * Cfg::WORK + 5 * N3 + r] = acc;
    }
    __syncthreads();
    // zeta + negate + RK stage epilogue (coalesced global I/O)
    const double dt = P.stage ? *P.dt : 0.0;
    const double hdt = 0.5 * dt, sdt = dt / 6.0;
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int b = it / (5 * N3), r = it - b * 5 * N3, s = r / N3, q = r - s * N3;
      const int ij = q % N2, k = q / N2;
      const double* src = WORK + b * Cfg::WORK + 5 * N3 + s * N3 + ij;
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(s_fr[k * N + a], src[a * N2], acc);
      const double kv = -acc;
      const size_t gi = (size_t)(e0 + b) * 5 * N3 + r;
      switch (P.stage) {
        case 0: P.out[gi] = kv; break;
        case 1:
          P.acc[gi] = kv;
          P.us[gi] = fma(hdt, kv, P.un[gi]);
          break;
        case 2:
          P.acc[gi] = fma(2.0, kv, P.acc[gi]);
          P.us[gi] = fma(hdt, kv, P.un[gi]);
          break;
        case 3:
          P.acc[gi] = fma(2.0, kv, P.acc[gi]);
          P.us[gi] = fma(dt, kv, P.un[gi]);
          break;
        default: {
          const double a4 = P.acc[gi] + kv;
          P.un[gi] = fma(sdt, a4, P.un[gi]);
        }
      }
    }
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
  const DevTables& T = *P.tab;
  const int e = blockIdx.x;
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
  for (int s = 0; s < NS; ++s) {
    const double* src = P.u + ((size_t)e * NS + s) * N3;
    for (int i = tid; i < N3; i += nthr) t2[i] = src[i];
    __syncthreads();
    tp3_rt(T.interp, n, n, t2, t1, xg, uq + s * N3, tid, nthr);
  }
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

// Step bookkeeping: reset lambda, compute dt from lambda.
struct StepState {
  double t, dt, t_final, cfl, dx;
  unsigned long long lam_bits;
  int active;
};

__global__ void k_step_begin(StepState* S) { S->lam_bits = 0ull; }

__global__ void k_step_dt(StepState* S) {
  const double lam = __longlong_as_double(static_cast<long long>(S->lam_bits));
  double dt = lam > 0.0 ? S->cfl * S->dx / lam : S->cfl * S->dx;
  if (S->t_final > 0.0) {
    if (S->t >= S->t_final)
      dt = 0.0;
    else
      dt = fmin(dt, S->t_final - S->t);
  }
  S->dt = dt;
}

__global__ void k_step_end(StepState* S) { S->t += S->dt; }

}  // namespace nsfr_b200
