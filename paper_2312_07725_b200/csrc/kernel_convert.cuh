// u_hat <-> u_q state conversion (chi^3 on the way in, Pi^3 on the way out;
// SPEC S1 / sumfac.cpp:57-78 apply_tensor_product) for n_q = n_p: the host
// transfers of set_state / get_state and the streamed host step run it once
// per element on the critical path, so it is a line-pass kernel at the HBM
// roofline instead of one element per CTA. Same arithmetic as k_convert
// (passes xi, eta, zeta; each output an fma chain from 0 in column order), so
// the two are bitwise interchangeable.
#pragma once
#include "setup_kernels.cuh"

namespace nsfr_b200 {

template <int N>
struct ConvOps {
  double A[N * N];  // chi (to_quad) or Pi, row-major N x N
  double B[N * N];  // MODE 2: chi, applied after A to what A wrote out
};

template <int N>
struct ConvCfg {
  static constexpr int N2 = N * N, N3 = N * N * N, LINES = 5 * N2;
  static constexpr int EPB = N <= 5 ? 4 : 2;
  static constexpr int THREADS = 256;
  static constexpr int SMEM = EPB * 5 * N3 * 8;
};

// The three passes of op over the staged block S (in place); the zeta pass
// also writes its results to out when WRITE (consecutive threads, consecutive
// nodes), and keeps them in S when KEEP.
template <int N, bool WRITE, bool KEEP, class Team = CtaTeam>
__device__ __forceinline__ void conv_passes(const double (&op)[N * N], double* S, double* __restrict__ out,
                                            int e0, int nb, const Team& tm = Team{}) {
  using Cfg = ConvCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, LINES = Cfg::LINES;
  const int tid = tm.tid(), nthr = tm.nthr();
#pragma unroll
  for (int D = 0; D < 3; ++D) {
    const int stride = D == 0 ? 1 : (D == 1 ? N : N2);
    for (int l = tid; l < nb * LINES; l += nthr) {
      const int b = l / LINES, r = l - b * LINES, s = r / N2, t = r - s * N2;
      const int t1 = t % N, t2 = t / N;
      const int base = D == 0 ? N * t1 + N2 * t2 : (D == 1 ? t1 + N2 * t2 : t1 + N * t2);
      double* x = S + (b * 5 + s) * N3 + base;
      double v[N];
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = x[a * stride];
#pragma unroll
      for (int row = 0; row < N; ++row) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) acc = fma(op[row * N + a], v[a], acc);
        if (D < 2 || KEEP) x[row * stride] = acc;
        if (D == 2 && WRITE) out[((size_t)(e0 + b) * 5 + s) * N3 + base + row * N2] = acc;
      }
    }
    if (D < 2 || KEEP) tm.sync();
  }
}

// lambda_max = max(|u| + a) over the admissible nodes of the [nb][5][N3]
// block S (synchronised by the caller) into *lam (atomicMax on the bits);
// every thread of the CTA calls it
template <int N, class Team = CtaTeam>
__device__ __forceinline__ void conv_lambda(const double* S, int nb, double gamma, unsigned long long* lam,
                                            const Team& tm = Team{}) {
  constexpr int N3 = N * N * N;
  double lm = 0.0;
  for (int it = tm.tid(); it < nb * N3; it += tm.nthr()) {
    const int b = it / N3, q = it - b * N3;
    double uu[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) uu[s] = S[(b * 5 + s) * N3 + q];
    if (d_admissible(gamma, uu)) lm = fmax(lm, d_node_wavespeed(gamma, uu));
  }
  for (int o = 16; o > 0; o >>= 1) lm = fmax(lm, __shfl_xor_sync(0xffffffffu, lm, o));
  if ((threadIdx.x & 31) == 0 && lm > 0.0) atomicMax(lam, dbl_bits(lm));
}

// elements [e_begin, e_end): one CTA per EPB elements; each thread owns whole
// lines, so a pass updates its lines in place (no other thread touches them).
// MODE 0: out = A^3 in. MODE 1 (LAM): no output; lambda_max = max(|u| + a)
// over the admissible nodes of A^3 in (A = chi: u_q = chi^3 u_hat, the node set
// and formula of K1, so adaptive_dt of a state about to leave the device
// equals what K1 finds when it comes back) into *lam (atomicMax on the bits).
// MODE 2: out = A^3 in (A = Pi) and lambda_max of B^3 out (B = chi) from the
// same bytes, in one pass over HBM.
template <int N, int MODE = 0>
__global__ void __launch_bounds__(ConvCfg<N>::THREADS)
    k_convert_lines(ConvOps<N> O, const double* __restrict__ in, double* __restrict__ out, int e_begin,
                    int e_end, double gamma = 0.0, unsigned long long* lam = nullptr) {
  using Cfg = ConvCfg<N>;
  constexpr int N3 = Cfg::N3, EPB = Cfg::EPB;
  constexpr bool LAM = MODE != 0;
  extern __shared__ __align__(128) double S[];
  dbg_kernel_entry(S);
  const int e0 = e_begin + NSFR_BID * EPB;
  const int nb = min(EPB, e_end - e0);
  __shared__ unsigned long long bar;
  {
    const StageBlock blk[1] = {{S, in + (size_t)e0 * 5 * N3, nb * 5 * N3}};
    stage_issue<1>(blk, &bar);
  }
  __syncthreads();
  stage_wait(&bar);
  __syncthreads();
  if constexpr (MODE == 0) {
    conv_passes<N, true, false>(O.A, S, out, e0, nb);
  } else if constexpr (MODE == 1) {
    conv_passes<N, false, true>(O.A, S, out, e0, nb);
  } else {
    conv_passes<N, true, true>(O.A, S, out, e0, nb);
    conv_passes<N, false, true>(O.B, S, out, e0, nb);
  }
  if (LAM) conv_lambda<N>(S, nb, gamma, lam);
}

}  // namespace nsfr_b200
