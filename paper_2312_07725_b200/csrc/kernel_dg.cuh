// Conservative strong-form DG residual (SPEC.md:457-465,
// PAPER.md:695-701 "cons DG strong"), the paper's cost-comparison baseline:
//
//   M du/dt = -[ chi^T W div^r(f^r) + sum_f (bs_f (x) chi^T (x) chi^T) W_f (J^G f*.n - n^r.phi(xi_f) f^r) ]
//
// on n_q = n_p + overint quadrature nodes per direction (collocated flux basis,
// f^r_dir = sum_k C[k][dir] f_k), f*.n = 1/2 (f(u-) + f(u+)).n minus the Roe
// dissipation (the paper's Roe surface flux for DG), own face
// metrics (D1) and the weight-adjusted inverse (D6; exact for n_q = n_p).
//   KD1 k_dg_states:   face states (bs (x) chi (x) chi) u_hat of every element
//                      (+ halo send planes, + lambda_max over the quadrature nodes)
//   KD2 k_dg_residual: u_q = chi^3 u_hat, f^r at the nodes, W div^r f^r by
//                      quad_diff line passes, the face terms per line, then the
//                      K3 tail (lift + WA inverse) and the RK stage update in
//                      u_hat space.
// The state stays at the solution nodes (u_hat): chi is not invertible when
// overintegrated.
#pragma once
#include "kernel_update.cuh"
#include "physics.cuh"

namespace nsfr_b200 {

// euler.cpp:30-40 physical_flux: f[k][s] for physical direction k
__device__ __forceinline__ bool d_physical_flux(double g, const double* u, double (&f)[3][NS]) {
  if (!d_admissible(g, u)) return false;
  const double p = d_pressure(g, u);
  const double ir = 1.0 / u[0];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double vk = u[1 + k] * ir;
    f[k][0] = u[0] * vk;
    f[k][1] = u[1] * vk;
    f[k][2] = u[2] * vk;
    f[k][3] = u[3] * vk;
    f[k][4] = (u[4] + p) * vk;
    f[k][1 + k] += p;
  }
  return true;
}

// Rectangular line pass along D of [nbat][E0 x E1 x E2] (xi fastest) with an
// NO x E_D operator: out extents replace E_D by NO. One thread per line; the
// fma chain runs over the contracted index (apply_operator_dir, sumfac.cpp:7-55).
template <int E0, int E1, int E2, int D, int NO>
__device__ __forceinline__ void rpass(const double (&op)[NO * (D == 0 ? E0 : (D == 1 ? E1 : E2))],
                                      const double* in, double* out, int nbat, int tid, int nthr) {
  constexpr int ED = D == 0 ? E0 : (D == 1 ? E1 : E2);
  constexpr int O0 = D == 0 ? NO : E0, O1 = D == 1 ? NO : E1;
  constexpr int IN_SZ = E0 * E1 * E2, OUT_SZ = (IN_SZ / ED) * NO;
  constexpr int LINES = IN_SZ / ED;
  constexpr int si = D == 0 ? 1 : (D == 1 ? E0 : E0 * E1);
  constexpr int so = D == 0 ? 1 : (D == 1 ? O0 : O0 * O1);
  for (int it = tid; it < nbat * LINES; it += nthr) {
    const int b = it / LINES, l = it - b * LINES;
    int ib, ob;
    if (D == 0) {
      ib = l * E0;
      ob = l * O0;
    } else if (D == 1) {
      const int i = l % E0, k = l / E0;
      ib = i + E0 * E1 * k;
      ob = i + O0 * O1 * k;
    } else {
      ib = l;
      ob = l;
    }
    const double* src = in + b * IN_SZ + ib;
    double x[ED];
#pragma unroll
    for (int a = 0; a < ED; ++a) x[a] = src[a * si];
    double* dst = out + b * OUT_SZ + ob;
#pragma unroll
    for (int r = 0; r < NO; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < ED; ++a) acc = fma(op[r * ED + a], x[a], acc);
      dst[r * so] = acc;
    }
  }
}

struct DgStateParams {
  const double* u;      // [E][5][NP^3] u_hat
  double* traces;       // [E][6][5][NQ^2] face states
  double* send_lo;      // [m*m][5][NQ^2] or nullptr
  double* send_hi;
  unsigned long long* lam;  // lambda_max bits or nullptr
  unsigned* err;
  int E, m, nz;
  double gamma;
};

template <int NP, int NQ>
struct DgOps {
  double chi[NQ * NP];    // interp (nq x np)
  double bs[2 * NP];      // bound_sol
  double D[NQ * NQ];      // quad_diff
  double bflux[2 * NQ];   // flux basis at -1, +1
  double wq[NQ];
  double M[NQ * NQ];      // Pi~^T chi^T
  double bm[2 * NQ];      // Pi~^T bound_sol_side
  double fr[NP * NQ];     // Pi~
};

template <int NP, int NQ>
struct DgCfg {
  static constexpr int P3 = NP * NP * NP, Q3 = NQ * NQ * NQ, Q2 = NQ * NQ;
  static constexpr int THREADS = 256;
  // KD2 per-element shared memory (doubles), see below; elements per CTA fill
  // the 256 threads in the pointwise phases within ~112 KB (2 CTAs per SM)
  static constexpr int R_EL = 5 * P3 + 9 * Q3 + Q3 + 5 * Q3 + 15 * Q3 + 5 * Q3 + 60 * Q2;
  static constexpr int E_FILL = 256 / Q3 > 1 ? 256 / Q3 : 1;
  static constexpr int E_SMEM = (112 * 1024) / (R_EL * 8) > 1 ? (112 * 1024) / (R_EL * 8) : 1;
  static constexpr int EPB = E_FILL < E_SMEM ? E_FILL : E_SMEM;
  // KD1 smem: U (5 P3), T1 (5 NQ NP^2), T2 (5 NQ^2 NP), six face buffers of
  // 5 x 2 NQ^2 (A1, A2, B1 intermediates; F0, F1, F2 results), UQ (5 Q3)
  static constexpr int S_PER_EL = 5 * P3 + 5 * NQ * NP * NP + 5 * NQ * NQ * NP + 60 * Q2 + 5 * Q3;
  static constexpr int S_SMEM = EPB * S_PER_EL * 8;
  // KD2 smem: U, CH (9 Q3), WJ (Q3), Q (5 Q3), FR (15 Q3, also S1/S2 and tail R1/R2),
  // VOL (5 Q3), FACC (30 Q2), G (30 Q2)
  static constexpr int R_SMEM = EPB * R_EL * 8;
};

// KD1: face states and lambda
template <int NP, int NQ>
__global__ void __launch_bounds__(256) k_dg_states(DgStateParams P, DgOps<NP, NQ> O) {
  using Cfg = DgCfg<NP, NQ>;
  constexpr int P3 = Cfg::P3, Q2 = Cfg::Q2, Q3 = Cfg::Q3, EPB = Cfg::EPB;
  extern __shared__ __align__(128) double sm[];
  dbg_kernel_entry(sm);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int e0 = NSFR_BID * EPB, nb = min(EPB, P.E - e0), nbs = nb * 5;
  double* U = sm;                            // [EPB*5][P3]
  double* T1 = U + EPB * 5 * P3;             // [EPB*5][NQ NP NP]
  double* T2 = T1 + EPB * 5 * NQ * NP * NP;  // [EPB*5][NQ NQ NP]
  double* A1 = T2 + EPB * 5 * NQ * NQ * NP;  // face buffers, [EPB*5][2 NQ^2] each
  double* A2 = A1 + EPB * 10 * Q2;
  double* B1 = A2 + EPB * 10 * Q2;
  double* F0 = B1 + EPB * 10 * Q2;
  double* F1 = F0 + EPB * 10 * Q2;
  double* F2 = F1 + EPB * 10 * Q2;
  double* UQ = F2 + EPB * 10 * Q2;           // [EPB*5][Q3]
  __shared__ unsigned long long bar;
  {
    const StageBlock blk[1] = {{U, P.u + (size_t)e0 * 5 * P3, nb * 5 * P3}};
    stage_issue<1>(blk, &bar);
  }
  __syncthreads();
  stage_wait(&bar);
  __syncthreads();
  const double g = P.gamma;
  // apply_tensor_product order (x, y, z) of each face's (bs (x) chi (x) chi):
  // A1 = bs_x U, T1 = chi_x U
  rpass<NP, NP, NP, 0, 2>(O.bs, U, A1, nbs, tid, nthr);
  rpass<NP, NP, NP, 0, NQ>(O.chi, U, T1, nbs, tid, nthr);
  __syncthreads();
  // A2 = chi_y A1 [2 NQ NP], B1 = bs_y T1 [NQ 2 NP], T2 = chi_y T1 [NQ NQ NP]
  rpass<2, NP, NP, 1, NQ>(O.chi, A1, A2, nbs, tid, nthr);
  rpass<NQ, NP, NP, 1, 2>(O.bs, T1, B1, nbs, tid, nthr);
  rpass<NQ, NP, NP, 1, NQ>(O.chi, T1, T2, nbs, tid, nthr);
  __syncthreads();
  // F0 = chi_z A2 [2 NQ NQ], F1 = chi_z B1 [NQ 2 NQ], F2 = bs_z T2 [NQ NQ 2], u_q = chi_z T2
  rpass<2, NQ, NP, 2, NQ>(O.chi, A2, F0, nbs, tid, nthr);
  rpass<NQ, 2, NP, 2, NQ>(O.chi, B1, F1, nbs, tid, nthr);
  rpass<NQ, NQ, NP, 2, 2>(O.bs, T2, F2, nbs, tid, nthr);
  if (P.lam) rpass<NQ, NQ, NP, 2, NQ>(O.chi, T2, UQ, nbs, tid, nthr);
  __syncthreads();
  // face states -> traces [e][f][s][k] (+ halo send planes)
  for (int it = tid; it < nb * 6 * Q2; it += nthr) {
    const int b = it / (6 * Q2), r = it - b * 6 * Q2, f = r / Q2, k = r - f * Q2;
    const int dir = f >> 1, side = f & 1, i = k % NQ, jk = k / NQ;
    double uu[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int o = (b * 5 + s) * 2 * Q2;
      uu[s] = dir == 0 ? F0[o + side + 2 * k]
                       : (dir == 1 ? F1[o + i + NQ * (side + 2 * jk)] : F2[o + k + Q2 * side]);
    }
    if (!d_admissible(g, uu)) atomicOr(P.err, ERR_STATE);
    const int e = e0 + b;
    double* dst = P.traces + ((size_t)e * 6 + f) * 5 * Q2 + k;
#pragma unroll
    for (int s = 0; s < NS; ++s) dst[s * Q2] = uu[s];
    const int mm = P.m * P.m, kl = e / mm, plane = e - kl * mm;
    if (P.send_lo && f == 4 && kl == 0) {
#pragma unroll
      for (int s = 0; s < NS; ++s) P.send_lo[((size_t)plane * 5 + s) * Q2 + k] = uu[s];
    }
    if (P.send_hi && f == 5 && kl == P.nz - 1) {
#pragma unroll
      for (int s = 0; s < NS; ++s) P.send_hi[((size_t)plane * 5 + s) * Q2 + k] = uu[s];
    }
  }
  if (P.lam) {
    double lam = 0.0;
    for (int it = tid; it < nb * Q3; it += nthr) {
      const int b = it / Q3, q = it - b * Q3;
      double uu[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) uu[s] = UQ[(b * 5 + s) * Q3 + q];
      if (!d_admissible(g, uu)) {
        atomicOr(P.err, ERR_STATE);
        continue;
      }
      lam = fmax(lam, d_node_wavespeed(g, uu));
    }
    for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
    if ((tid & 31) == 0 && lam > 0.0) atomicMax(P.lam, dbl_bits(lam));
  }
}

struct DgResParams {
  const double* us;      // [E][5][NP^3] stage state u_hat
  const double* traces;  // [E][6][5][NQ^2]
  const double* halo_lo;
  const double* halo_hi;
  const double* cof;     // [E][9][NQ^3] = 0.5 C
  const double* wj;      // [E][NQ^3] = 1/(w J)
  double* un;            // RK base (stage 4 writes it)
  double* uo;            // next stage state (stages 1-3)
  double* acc;
  double* out;           // stage 0: dU/dt
  const double* dt;
  unsigned* err;
  int stage, E, m, nz;
  double gamma;
  int roe;
};

// KD2: residual + WA inverse + RK stage
template <int NP, int NQ>
__global__ void __launch_bounds__(256, 2) k_dg_residual(DgResParams P, DgOps<NP, NQ> O) {
  using Cfg = DgCfg<NP, NQ>;
  constexpr int P3 = Cfg::P3, Q2 = Cfg::Q2, Q3 = Cfg::Q3, EPB = Cfg::EPB;
  constexpr int VS = 5 * Q3, FS = 30 * Q2;
  extern __shared__ __align__(128) double sm[];
  dbg_kernel_entry(sm);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int e0 = NSFR_BID * EPB, nb = min(EPB, P.E - e0), nbs = nb * 5;
  double* U = sm;                    // [EPB*5][P3]
  double* CH = U + EPB * 5 * P3;     // [EPB][9][Q3]
  double* WJ = CH + EPB * 9 * Q3;    // [EPB][Q3]
  double* Q = WJ + EPB * Q3;         // [EPB*5][Q3]
  double* FR = Q + EPB * VS;         // [EPB*15][Q3]; S1/S2 before, tail R1/R2 after
  double* VOL = FR + EPB * 15 * Q3;  // [EPB*5][Q3]
  double* FACC = VOL + EPB * VS;     // [EPB][3][5][2][Q2]
  double* G = FACC + EPB * FS;       // [EPB][30 Q2]
  const double g = P.gamma;
  const GasC gas = GasC::make(g);
  __shared__ unsigned long long bar;
  {
    const StageBlock blk[3] = {{U, P.us + (size_t)e0 * 5 * P3, nb * 5 * P3},
                               {CH, P.cof + (size_t)e0 * 9 * Q3, nb * 9 * Q3},
                               {WJ, P.wj + (size_t)e0 * Q3, nb * Q3}};
    stage_issue<3>(blk, &bar);
  }
  // the RK operands of the epilogue, into L2 meanwhile
  if (P.stage >= 1 && tid == 32) l2_prefetch(P.un + (size_t)e0 * 5 * P3, (size_t)nb * 5 * P3 * 8);
  if (P.stage >= 2 && tid == 64) l2_prefetch(P.acc + (size_t)e0 * 5 * P3, (size_t)nb * 5 * P3 * 8);
  __syncthreads();
  stage_wait(&bar);
  __syncthreads();
  // u_q = chi^3 u_hat (apply_tensor_product order)
  double* S1 = FR;
  double* S2 = FR + EPB * 5 * NQ * NP * NP;
  rpass<NP, NP, NP, 0, NQ>(O.chi, U, S1, nbs, tid, nthr);
  __syncthreads();
  rpass<NQ, NP, NP, 1, NQ>(O.chi, S1, S2, nbs, tid, nthr);
  __syncthreads();
  rpass<NQ, NQ, NP, 2, NQ>(O.chi, S2, Q, nbs, tid, nthr);
  __syncthreads();
  // contravariant flux f^r_dir = sum_k C[k][dir] f_k at every quadrature node
  for (int it = tid; it < nb * Q3; it += nthr) {
    const int b = it / Q3, q = it - b * Q3;
    double uu[NS], f[3][NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] = Q[(b * 5 + s) * Q3 + q];
    if (!d_physical_flux(g, uu, f)) {
      atomicOr(P.err, ERR_STATE);
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int s = 0; s < NS; ++s) f[k][s] = 0.0;
    }
    const double* Cb = CH + b * 9 * Q3 + q;
#pragma unroll
    for (int dir = 0; dir < 3; ++dir) {
      const double c0 = 2.0 * Cb[(0 + dir) * Q3], c1 = 2.0 * Cb[(3 + dir) * Q3], c2 = 2.0 * Cb[(6 + dir) * Q3];
#pragma unroll
      for (int s = 0; s < NS; ++s) FR[((b * 15) + dir * 5 + s) * Q3 + q] = f[0][s] * c0 + f[1][s] * c1 + f[2][s] * c2;
    }
  }
  __syncthreads();
  // W div^r f^r: quad_diff along x into VOL, += along y, += along z then * w
  for (int it = tid; it < nbs * Q2; it += nthr) {  // x lines
    const int bs_ = it / Q2, l = it - bs_ * Q2, b = bs_ / 5, s = bs_ - 5 * b;
    const double* src = FR + ((b * 15) + 0 + s) * Q3 + l * NQ;
    double x[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) x[a] = src[a];
    double* dst = VOL + bs_ * Q3 + l * NQ;
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a) acc = fma(O.D[r * NQ + a], x[a], acc);
      dst[r] = acc;
    }
  }
  __syncthreads();
  for (int it = tid; it < nbs * Q2; it += nthr) {  // y lines
    const int bs_ = it / Q2, l = it - bs_ * Q2, b = bs_ / 5, s = bs_ - 5 * b;
    const int i = l % NQ, k = l / NQ, base = i + Q2 * k;
    const double* src = FR + ((b * 15) + 5 + s) * Q3 + base;
    double x[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) x[a] = src[a * NQ];
    double* dst = VOL + bs_ * Q3 + base;
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a) acc = fma(O.D[r * NQ + a], x[a], acc);
      dst[r * NQ] += acc;
    }
  }
  __syncthreads();
  for (int it = tid; it < nbs * Q2; it += nthr) {  // z lines, then the weights
    const int bs_ = it / Q2, l = it - bs_ * Q2, b = bs_ / 5, s = bs_ - 5 * b;
    const int i = l % NQ, j = l / NQ;
    const double* src = FR + ((b * 15) + 10 + s) * Q3 + l;
    double x[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) x[a] = src[a * Q2];
    double* dst = VOL + bs_ * Q3 + l;
    const double wij = O.wq[i] * O.wq[j];
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a) acc = fma(O.D[r * NQ + a], x[a], acc);
      dst[r * Q2] = (dst[r * Q2] + acc) * (wij * O.wq[r]);
    }
  }
  // face terms: one thread per (b, face f = 2 dir + side, node k) at the end of line k
  for (int it = tid; it < nb * 6 * Q2; it += nthr) {
    const int b = it / (6 * Q2), r = it - b * 6 * Q2, f = r / Q2, k = r - f * Q2;
    const int dir = f >> 1, side = f & 1;
    const int t1 = k % NQ, t2 = k / NQ, e = e0 + b;
    const int stride = dir == 0 ? 1 : (dir == 1 ? NQ : Q2);
    const int base = dir == 0 ? NQ * (t1 + NQ * t2) : (dir == 1 ? t1 + Q2 * t2 : t1 + NQ * t2);
    const double wt = O.wq[t1] * O.wq[t2];
    const double* Cb = CH + b * 9 * Q3;
    {
      const double sign = side ? 1.0 : -1.0;
      double fi[NS], cf0 = 0.0, cf1 = 0.0, cf2 = 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s) fi[s] = 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a) {
        const double w = O.bflux[side * NQ + a];
        const int ia = base + a * stride;
#pragma unroll
        for (int s = 0; s < NS; ++s) fi[s] += w * FR[((b * 15) + dir * 5 + s) * Q3 + ia];
        cf0 = fma(w, 2.0 * Cb[(0 + dir) * Q3 + ia], cf0);
        cf1 = fma(w, 2.0 * Cb[(3 + dir) * Q3 + ia], cf1);
        cf2 = fma(w, 2.0 * Cb[(6 + dir) * Q3 + ia], cf2);
      }
      const double v0 = sign * cf0, v1 = sign * cf1, v2 = sign * cf2;
      const double jg = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
      const double ijg = 1.0 / jg;
      const double nrm[3] = {v0 * ijg, v1 * ijg, v2 * ijg};
      double ul[NS], ur[NS];
      const double* tr = P.traces + ((size_t)e * 6 + f) * 5 * Q2 + k;
#pragma unroll
      for (int s = 0; s < NS; ++s) ul[s] = tr[s * Q2];
      {  // neighbour across face f (geometry.hpp:24-29), its face f^1, same node k
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
            if (halo) nt = halo + (size_t)(i + mm * j) * 5 * Q2 + k;
            kl = (kl + P.nz) % P.nz;
          }
        }
        if (!nt) nt = P.traces + (((size_t)(i + mm * (j + mm * kl))) * 6 + (f ^ 1)) * 5 * Q2 + k;
#pragma unroll
        for (int s = 0; s < NS; ++s) ur[s] = nt[s * Q2];
      }
      double fl[3][NS], fr2[3][NS], fn[NS];
      if (!d_physical_flux(g, ul, fl) || !d_physical_flux(g, ur, fr2)) atomicOr(P.err, ERR_STATE);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        // CentralConservative two-point flux (euler.cpp:205-211), contracted with n
        const double a0 = 0.5 * (fl[0][s] + fr2[0][s]), a1 = 0.5 * (fl[1][s] + fr2[1][s]),
                     a2 = 0.5 * (fl[2][s] + fr2[2][s]);
        fn[s] = a0 * nrm[0] + a1 * nrm[1] + a2 * nrm[2];
      }
      if (P.roe) {
        double d[NS];
        const PrimX pl = d_primx(g, ul), pr = d_primx(g, ur);
        if (!d_roe_prim(gas, pl, pr, nrm, d)) atomicOr(P.err, ERR_ROE);
#pragma unroll
        for (int s = 0; s < NS; ++s) fn[s] -= d[s];
      }
      double* fa = FACC + b * FS + dir * 10 * Q2;
#pragma unroll
      for (int s = 0; s < NS; ++s) fa[(s * 2 + side) * Q2 + k] = wt * (jg * fn[s] - sign * fi[s]);
    }
  }
  __syncthreads();
  // lift + first half of the WA inverse (the K3 tail), 1/(w J) fused
  double* R1 = FR;
  double* R2 = FR + EPB * VS;
  tail_pass<NQ, 0, true, false>(O.M, O.bm, FACC, FS, VOL, VS, R1, VS, WJ, nbs, tid, nthr);
  tail_face_pass<NQ, 0>(O.M, FACC + 10 * Q2, FS, G, FS, nb, face_vt<NQ>(tid, nthr, 0), nthr);
  tail_face_pass<NQ, 0>(O.M, FACC + 20 * Q2, FS, G + 10 * Q2, FS, nb, face_vt<NQ>(tid, nthr, nb * 10 * NQ), nthr);
  __syncthreads();
  tail_pass<NQ, 1, true, false>(O.M, O.bm, G, FS, R1, VS, R2, VS, WJ, nbs, tid, nthr);
  tail_face_pass<NQ, 1>(O.M, G + 10 * Q2, FS, G + 20 * Q2, FS, nb, face_vt<NQ>(tid, nthr, 0), nthr);
  __syncthreads();
  tail_pass<NQ, 2, true, true>(O.M, O.bm, G + 20 * Q2, FS, R2, VS, VOL, VS, WJ, nbs, tid, nthr);
  __syncthreads();
  // second half: Pi~ (np x nq) along xi, eta, then zeta with the RK update
  rpass<NQ, NQ, NQ, 0, NP>(O.fr, VOL, R1, nbs, tid, nthr);
  __syncthreads();
  rpass<NP, NQ, NQ, 1, NP>(O.fr, R1, R2, nbs, tid, nthr);
  __syncthreads();
  const double dt = P.stage ? *P.dt : 0.0;
  const double hdt = 0.5 * dt, sdt = dt / 6.0;
  constexpr int PP = NP * NP;
  for (int it = tid; it < nbs * PP; it += nthr) {
    const int bs_ = it / PP, l = it - bs_ * PP;
    const double* src = R2 + bs_ * PP * NQ + l;
    double x[NQ];
#pragma unroll
    for (int a = 0; a < NQ; ++a) x[a] = src[a * PP];
    const size_t gb = (size_t)e0 * 5 * P3 + (size_t)bs_ * P3 + l;
#pragma unroll
    for (int c = 0; c < NP; ++c) {
      double z = 0.0;
#pragma unroll
      for (int a = 0; a < NQ; ++a) z = fma(O.fr[c * NQ + a], x[a], z);
      const double kv = -z;
      const size_t gi = gb + c * PP;
      switch (P.stage) {
        case 0: P.out[gi] = kv; break;
        case 1:
          P.acc[gi] = kv;
          P.uo[gi] = fma(hdt, kv, P.un[gi]);
          break;
        case 2:
          P.acc[gi] = fma(2.0, kv, P.acc[gi]);
          P.uo[gi] = fma(hdt, kv, P.un[gi]);
          break;
        case 3:
          P.acc[gi] = fma(2.0, kv, P.acc[gi]);
          P.uo[gi] = fma(dt, kv, P.un[gi]);
          break;
        default: P.un[gi] = fma(sdt, P.acc[gi] + kv, P.un[gi]);
      }
    }
  }
}

}  // namespace nsfr_b200
