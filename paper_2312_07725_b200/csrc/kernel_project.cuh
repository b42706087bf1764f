// K1: entropy projection S1-S5.
//
//   u_q = chi^3 u_hat (the solver's state representation);  v_q = v(u_q);  v_hat = Pi^3 v_q;
//   v~ = chi^3 v_hat at the volume, (bs_side (x) chi (x) chi) v_hat at each face;
//   u~ = u(v~)                                   (euler.cpp:46-71)
// plus lambda_max = max(|u| + a) over the volume nodes for adaptive dt.
//
// EPB elements per CTA, element blocks staged in shared memory. Every
// directional contraction is a LINE pass: one thread per 1D line loads its N
// inputs once and writes N outputs (fma chain in the reference's order,
// apply_operator_dir sumfac.cpp:7-55). The 1D operators travel in the kernel
// parameter (constant) bank, so each FMA takes its coefficient as an operand.
#pragma once
#include "kernel_convert.cuh"
#include "physics.cuh"
#include "setup_kernels.cuh"

namespace nsfr_b200 {

struct ProjParams {
  const double* u;       // [E][5][N^3] stage input u_q at the volume quadrature nodes
  double* ut_vol;        // [E][6][N^3] rho,u,v,w,p,rho/p of the entropy-projected volume state
  double* traces;        // [E][6 faces][NTR][N^2] primitives rho,u,v,w,p,rho/p of u(v~) (physics.cuh)
  double* vhat;          // [E][5][N^3] or nullptr
  double* send_lo;       // [m*m][NTR][N^2] face 4 of plane 0, or nullptr
  double* send_hi;       // [m*m][NTR][N^2] face 5 of plane nz-1, or nullptr
  unsigned long long* lam;  // lambda_max bits or nullptr
  unsigned* err;
  int E, m, nz;          // E: end of the launched element range [e_begin, E) (the slab by default)
  double gamma;
  int e_begin;           // first element of the launched range (a multiple of 8)
  double* uq_out;        // K1 from u_hat (streamed host step): u is u_hat, chi^3 u goes here
};

template <int N>
struct ProjOps {
  double proj[N * N];    // Pi    (np x nq)
  double bsol[2 * N];    // bound_sol rows at xi = -1, +1
  double bp[2 * N];      // bound_sol_side Pi: face trace rows applied to nodal v (chi Pi = I)
  double c35;            // gm1^(1/gm1) when gamma/(gamma-1) == 7/2 (closed-form u(v)), else 0
  double chi[N * N];     // chi (nq x np): K1 from u_hat, K3's outgoing lambda
};

template <int N>
__device__ __forceinline__ bool prim_of_v(const ProjOps<N>& O, double g, const double* v, double* q) {
  return O.c35 > 0.0 ? d_entropy_to_prim_35(g, O.c35, v, q) : d_entropy_to_prim(g, v, q);
}

template <int N>
struct ProjCfg {
  static constexpr int N2 = N * N, N3 = N * N * N;
  static constexpr int EPB = N3 <= 32 ? 8 : (N3 <= 64 ? 4 : (N3 <= 128 ? 2 : 1));
  static constexpr int THREADS = ((EPB * N3 + 31) / 32) * 32;
  // smem doubles per element: A, B, V (5 N3 each) + F0, F1, F2 (10 N2 each)
  static constexpr int PER_EL = 15 * N3 + 30 * N2;
  static constexpr int SMEM = EPB * PER_EL * 8;
};

// One thread per 1D line along D of a [batch][N^3] tensor; out[r] = sum_a op[r][a] x[a].
// FACE: also contract the same line with the two boundary rows into fo[batch][side][N2].
template <int N, int D, bool FACE>
__device__ __forceinline__ void line_pass(const double (&op)[N * N], const double* in, double* out,
                                          const double (&bs)[2 * N], double* fo, int nbs, int tid,
                                          int nthr) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N : N2);
  for (int it = tid; it < nbs * N2; it += nthr) {
    const int bsi = it / N2, l = it - bsi * N2;
    const int l0 = l % N, l1 = l / N;
    const int base = D == 0 ? N * (l0 + N * l1) : (D == 1 ? l0 + N2 * l1 : l0 + N * l1);
    const double* src = in + bsi * N3 + base;
    double x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = src[a * stride];
    double* dst = out + bsi * N3 + base;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(op[r * N + a], x[a], acc);
      dst[r * stride] = acc;
    }
    if (FACE) {
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) acc = fma(bs[side * N + a], x[a], acc);
        fo[(bsi * 2 + side) * N2 + l] = acc;
      }
    }
  }
}

// Face traces: one thread per 1D line contracts it with the two boundary rows
// bp[side] into fo[batch][side][N2] (line index l).
// The three directions in one loop: a line index (tensor bsi, l0 + N l1) names one
// line per direction, so its index arithmetic is done once (same sums, same bits).
template <int N, int D>
__device__ __forceinline__ void face_contract_line(const double (&bp)[2 * N], const double* in, double* fo,
                                                   int bsi, int l, int l0, int l1) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N : N2);
  const int base = D == 0 ? N * (l0 + N * l1) : (D == 1 ? l0 + N2 * l1 : l0 + N * l1);
  const double* src = in + bsi * N3 + base;
  double x[N];
#pragma unroll
  for (int a = 0; a < N; ++a) x[a] = src[a * stride];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a) acc = fma(bp[side * N + a], x[a], acc);
    fo[(bsi * 2 + side) * N2 + l] = acc;
  }
}
template <int N>
__device__ __forceinline__ void face_contract_all(const double (&bp)[2 * N], const double* in, double* F0,
                                                  double* F1, double* F2, int nbs, int tid, int nthr) {
  constexpr int N2 = N * N;
  for (int it = tid; it < nbs * N2; it += nthr) {
    const int bsi = it / N2, l = it - bsi * N2;
    const int l0 = l % N, l1 = l / N;
    face_contract_line<N, 0>(bp, in, F0, bsi, l, l0, l1);
    face_contract_line<N, 1>(bp, in, F1, bsi, l, l0, l1);
    face_contract_line<N, 2>(bp, in, F2, bsi, l, l0, l1);
  }
}

// S2-S5 for the nb elements whose state u_q (volume quadrature nodes) sits in
// shared memory A ([EPB*5][N3], synchronised by the caller). B, V: [EPB*5][N3] scratch;
// F: [3][EPB*5][2][N2] face scratch. Shared by K1 and the fused K3 (kernel_update.cuh).
template <int N, int EPB = ProjCfg<N>::EPB, class Team = CtaTeam>
__device__ __forceinline__ void proj_core(const ProjParams& P, const ProjOps<N>& O, int e0, int nb,
                                          double* A, double* B, double* V, double* F, const Team& tm = Team{}) {
  using Cfg = ProjCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3;
  double* F0 = F;                   // [EPB*5][2][N2] dir-0 face v~ (index j + N k)
  double* F1 = F0 + EPB * 10 * N2;  // [EPB*5][2][N2] dir-1 face v~ (index i + N k)
  double* F2 = F1 + EPB * 10 * N2;  // [EPB*5][2][N2] dir-2 face v~ (index i + N j)
  const int tid = tm.tid(), nthr = tm.nthr();
  const double g = P.gamma;
  const int nbs = nb * 5;
  PHASE_START();
  // S1 u_q = chi^3 u_hat is where the state lives: the solver carries u_q
  // (k_convert at the API boundary), so A already holds it.
  // S2 v(u_q) -> V, the wavespeed for adaptive dt, and the
  // volume state K2 consumes. With n_q = n_p (GL or LGL, no overintegration)
  // Pi = chi^-1, so the reference's volume round trip u(chi^3 Pi^3 v(u_q))
  // is u_q in exact arithmetic: K2 gets the primitives of u_q directly
  // (the RHS moves by ~1x the reference's own 1-ulp floor).
  double lam = 0.0;
  for (int it = tid; it < nb * N3; it += nthr) {
    const int b = it / N3, q = it - b * N3;
    double uu[NS], vv[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] = A[(b * 5 + s) * N3 + q];
    // primitives once (1/rho, 1/p): the entropy variables and K2's bundle share them
    const PrimX px = d_primx(g, uu);
    if (!d_admissible(g, uu)) {
      atomicOr(P.err, ERR_STATE);
#pragma unroll
      for (int s = 0; s < NS; ++s) vv[s] = (s == 4) ? -1.0 : 0.0;
    } else {
      d_entropy_vars_x(g, uu, px, vv);
      if (P.lam) lam = fmax(lam, d_node_wavespeed(g, uu));
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) V[(b * 5 + s) * N3 + q] = vv[s];
    // half-scaled primitive bundle for K2's pair fluxes (prim(), euler.cpp:109-115)
    const PrimH ph = to_half(g - 1.0, px);
    double* dst = P.ut_vol + (size_t)(e0 + b) * 6 * N3 + q;
    dst[0 * N3] = ph.hr;
    dst[1 * N3] = ph.hu;
    dst[2 * N3] = ph.hv;
    dst[3 * N3] = ph.hw;
    dst[4 * N3] = ph.hp;
    dst[5 * N3] = ph.grp;
  }
  if (P.lam) {
    for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
    if ((tid & 31) == 0 && lam > 0.0) atomicMax(P.lam, dbl_bits(lam));
  }
  tm.sync();
  // S3 v_hat = Pi^3 v_q: only the entropy diagnostic (-v_hat . R) needs it
  if (P.vhat) {
    line_pass<N, 0, false>(O.proj, V, A, O.bsol, nullptr, nbs, tid, nthr);
    tm.sync();
    line_pass<N, 1, false>(O.proj, A, B, O.bsol, nullptr, nbs, tid, nthr);
    tm.sync();
    line_pass<N, 2, false>(O.proj, B, A, O.bsol, nullptr, nbs, tid, nthr);
    tm.sync();
    double* dst = P.vhat + (size_t)e0 * 5 * N3;
    for (int i = tid; i < nb * 5 * N3; i += nthr) dst[i] = A[i];
  }
  PHASE_MARK(11);
  // S4 faces: v~_f = (bs_side (x) chi (x) chi) Pi^3 v_q = (bs_side Pi) along the
  // normal applied to v_q (chi Pi = I tangentially): one contraction per line
  face_contract_all<N>(O.bp, V, F0, F1, F2, nbs, tid, nthr);
  tm.sync();
  PHASE_MARK(12);
  // S5 u~ = u(v~) at the face nodes, kept as primitives (NTR values per node)
  for (int it = tid; it < nb * 6 * N2; it += nthr) {
    const int b = it / (6 * N2), r = it - b * 6 * N2, f = r / N2, k = r - f * N2;
    const int dir = f / 2, side = f % 2;
    const double* Fd = dir == 0 ? F0 : (dir == 1 ? F1 : F2);
    double vv[NS], qq[NTR];
#pragma unroll
    for (int s = 0; s < NS; ++s) vv[s] = Fd[((b * 5 + s) * 2 + side) * N2 + k];
    if (!prim_of_v<N>(O, g, vv, qq)) atomicOr(P.err, ERR_STATE);
    const int e = e0 + b;
    double* dst = P.traces + ((size_t)e * 6 + f) * NTR * N2 + k;
#pragma unroll
    for (int s = 0; s < NTR; ++s) dst[s * N2] = qq[s];
    // boundary planes also go to the halo send buffers (z faces of slab contexts only)
    if ((P.send_lo && f == 4) || (P.send_hi && f == 5)) {
      const int mm = P.m * P.m, kl = e / mm, plane = e - kl * mm;
      if (f == 4 && kl == 0) {
#pragma unroll
        for (int s = 0; s < NTR; ++s) P.send_lo[((size_t)plane * NTR + s) * N2 + k] = qq[s];
      }
      if (f == 5 && kl == P.nz - 1) {
#pragma unroll
        for (int s = 0; s < NTR; ++s) P.send_hi[((size_t)plane * NTR + s) * N2 + k] = qq[s];
      }
    }
  }
  PHASE_MARK(13);
}

template <int N, bool HAT>
__device__ __forceinline__ void proj_batch(const ProjParams& P, const ProjOps<N>& O, int e0, double* sm) {
  using Cfg = ProjCfg<N>;
  constexpr int N3 = Cfg::N3, EPB = Cfg::EPB;
  double* A = sm;
  double* B = A + EPB * 5 * N3;
  double* V = B + EPB * 5 * N3;
  const int nb = min(EPB, P.E - e0);
  __shared__ unsigned long long bar;
  {
    const StageBlock blk[1] = {{A, P.u + (size_t)e0 * 5 * N3, nb * 5 * N3}};
    stage_issue<1>(blk, &bar);
  }
  __syncthreads();
  stage_wait(&bar);
  __syncthreads();
  // HAT: the block is u_hat (just uploaded): u_q = chi^3 u_hat in place, also
  // to P.uq_out (kernel_convert's passes: the bits of k_convert_lines)
  if constexpr (HAT) conv_passes<N, true, true>(O.chi, A, P.uq_out, e0, nb);
  proj_core<N>(P, O, e0, nb, A, B, V, V + EPB * 5 * N3);
}

// One batch per CTA; L2 prefetch of the input block of the CTA `ahead`
// (= #resident CTAs) later (see k_residual).
template <int N, bool HAT = false>
__global__ void __launch_bounds__(ProjCfg<N>::THREADS) k_project(ProjParams P, ProjOps<N> O, int ahead) {
  extern __shared__ __align__(128) double sm[];
  dbg_kernel_entry(sm);
  constexpr int EPB = ProjCfg<N>::EPB, N3 = N * N * N;
  const int nbatch = (P.E - P.e_begin + EPB - 1) / EPB;
  const long long pb = static_cast<long long>(NSFR_BID) + ahead;
  if (threadIdx.x == 0 && pb < nbatch) {
    const int e0 = P.e_begin + pb * EPB, nb = min(EPB, P.E - e0);
    l2_prefetch(P.u + (size_t)e0 * 5 * N3, (size_t)nb * 5 * N3 * sizeof(double));
  }
  proj_batch<N, HAT>(P, O, P.e_begin + NSFR_BID * EPB, sm);
}

}  // namespace nsfr_b200
