// K3: the rest of the residual, the RK4 stage update and the NEXT stage's
// entropy projection, fused:
//   S9  chi^T lifting of the volume rows (K2's vol; its face rows are already in
//       them for n = 4..7, fuse_face, else K2's facc is lifted here too)
//   S10 weight-adjusted inverse -Pi~ (W J)^-1 Pi~^T R (fr_operators.cpp:280-309, D6)
//   RK  classical RK4 stage update (D4)
//   S1-S5 of u_{s+1} (kernel_project.cuh::proj_core) straight from shared memory,
//       so the stage state never round-trips through HBM; lambda_max of the
//       new u_n after the last stage (adaptive dt of the next step).
//
// S9 and the first half of S10 are both tensor products, so
//   Pi~^T^3 R = M^3 vol + sum_f (b_f (x) M (x) M) facc_f,  M = Pi~^T chi^T, b_f = Pi~^T bs_f
// runs as three LINE passes (fused: M^3 of K2's vol + sum_f l_f (x) facc_f,
// b_f = M l_f; else the face lifts injected into the pass of their normal
// direction), the 1/(w J) scaling fused into the last one, then
// three Pi~ passes with the RK update fused into the last. (The entropy
// diagnostic needs R itself: that path lifts with chi^T first.)
//
// Stage 0 is a plain residual (dU/dt into `out`, optional -v_hat . R); stages
// 1-3 accumulate acc and project u_{s+1}; stage 4 writes u_{n+1} and projects it.
#pragma once
#include "kernel_convert.cuh"
#include "kernel_project.cuh"
#include "physics.cuh"

namespace nsfr_b200 {

struct UpdParams {
  const double* vol;   // [E][5][N^3] volume rows (K2)
  const double* facc;  // [E][3][5][2][N^2] face rows (K2)
  const double* wj;    // [E][N^3] 1/(w J)
  const double* vhat;  // [E][5][N^3] or nullptr (entropy diagnostic, stage 0)
  double* dS;          // [E] or nullptr
  double* un;          // RK base state (stage 4 writes it)
  double* acc;         // RK accumulator
  double* out;         // stage 0: dU/dt
  const double* dt;    // device scalar
  int stage;
  ProjParams pj;       // projection of u_{s+1} (pj.u unused); pj.err, pj.E shared
  double* uhat_out;    // OUT (stage 4 of the streamed host step): Pi^3 u_{n+1} instead of the projection
  unsigned long long* lam_out;  // OUT: adaptive_dt's lambda_max of chi^3 of that u_hat, or nullptr
};

// A centrosymmetric 1D operator (M = J M J, J the flip: every operator built
// from a symmetric node set and basis is one) applied through its even / odd
// halves: with se = x + Jx, so = x - Jx (first halves),
//   y[r], y[N-1-r] = e[r] +- o[r],  e = E se (ceil(N/2) square), o = O so (floor(N/2) square),
// E[r][a] = (M[r][a] + M[r][N-1-a]) / 2 (the middle column of an odd N as it is),
// O[r][a] = (M[r][a] - M[r][N-1-a]) / 2. At N = 5: 13 multiply-adds + 8 additions
// and 13 constant operands instead of 25 + 25 (each constant is a uniform load
// in the SASS, and K3 is issue-bound).
template <int N>
struct SymOp {
  static constexpr int H = N / 2, C = (N + 1) / 2;
  double e[C * C];
  double o[H * H];
  // largest |M - J M J| over |M|: the caller refuses an operator that is not centrosymmetric
  static double asymmetry(const double* M) {
    double d = 0.0, m = 0.0;
    for (int r = 0; r < N; ++r)
      for (int a = 0; a < N; ++a) {
        const double x = M[r * N + a], y = M[(N - 1 - r) * N + (N - 1 - a)];
        d = d < (x > y ? x - y : y - x) ? (x > y ? x - y : y - x) : d;
        m = m < (x < 0 ? -x : x) ? (x < 0 ? -x : x) : m;
      }
    return m > 0.0 ? d / m : 0.0;
  }
  static SymOp fold(const double* M) {
    SymOp S{};
    for (int r = 0; r < C; ++r)
      for (int a = 0; a < C; ++a)
        S.e[r * C + a] = (a < H) ? 0.5 * (M[r * N + a] + M[r * N + (N - 1 - a)]) : M[r * N + a];
    for (int r = 0; r < H; ++r)
      for (int a = 0; a < H; ++a) S.o[r * H + a] = 0.5 * (M[r * N + a] - M[r * N + (N - 1 - a)]);
    return S;
  }
  __device__ __forceinline__ void apply(const double (&x)[N], double (&y)[N]) const {
    double se[C], so[H > 0 ? H : 1];
#pragma unroll
    for (int a = 0; a < H; ++a) {
      se[a] = x[a] + x[N - 1 - a];
      so[a] = x[a] - x[N - 1 - a];
    }
    if (C > H) se[H] = x[H];
#pragma unroll
    for (int r = 0; r < C; ++r) {
      double ev = 0.0;
#pragma unroll
      for (int a = 0; a < C; ++a) ev = fma(e[r * C + a], se[a], ev);
      if (r < H) {
        double ov = 0.0;
#pragma unroll
        for (int a = 0; a < H; ++a) ov = fma(o[r * H + a], so[a], ov);
        y[r] = ev + ov;
        y[N - 1 - r] = ev - ov;
      } else {
        y[r] = ev;
      }
    }
  }
};

template <int N>
struct TailOps {
  SymOp<N> Ms, frs;      // M and fr folded (the hot path without face injection)
  double M[N * N];       // Pi~^T chi^T          (lift + project, hot path)
  double bm[2 * N];      // Pi~^T bound_sol_side
  double fr[N * N];      // final passes: Pi~ (stage 0, u_hat space) or chi Pi~ (RK stages, u_q space)
  double frt[N * N];     // Pi~^T                (entropy-diagnostic path)
  double it[N * N];      // chi^T                (entropy-diagnostic path)
  double bs[2 * N];      // bound_sol            (entropy-diagnostic path)
};

template <int N>
struct UpdOps {
  TailOps<N> t;
  ProjOps<N> p;          // p.chi: OUT's lambda of the outgoing state
};

template <int N>
struct UpdCfg {
  static constexpr int N2 = N * N, N3 = N * N * N;
  // elements per CTA: proj_core's batch (at n = 5 two; one measured K3 +6.5%)
  static constexpr int EPB = ProjCfg<N>::EPB;
  // Threads per CTA: proj_core's (one per volume node of the batch), except at
  // n >= 6 (one element per CTA, 216 / 343 nodes) where fewer threads with
  // more line items each keep the per-item constant loads (LDCU, the 1D
  // operators) in uniform registers across items. Measured K3 (A/B, one
  // session): p=5 224 -> 128 threads -13% (96: -8%, 160: +5%); p=6 352 -> 160
  // threads -8% (128: -4%); the same change costs +3% at p=4 and +16% at p=3.
  // (re-swept with the round-2 kernels: n = 6 96 / 128 / 192 / 224 threads ->
  // K3 3.18 / 3.08 / 3.41 / 3.61 ms at 64^3; n = 7 128 / 160 / 256 threads ->
  // 1.31 / 1.30 / 1.21 ms at 40^3 with c_DG, 1.57 / 1.56 / 1.53 ms with a c > 0)
#ifndef NSFR_UPD_T6
#define NSFR_UPD_T6 128
#endif
#ifndef NSFR_UPD_T7
#define NSFR_UPD_T7 256
#endif
  static constexpr int THREADS = N == 6 ? NSFR_UPD_T6 : (N == 7 ? NSFR_UPD_T7 : ((EPB * N3 + 31) / 32) * 32);
  // R0 vol/u_{s+1}, R1, R2 pass buffers (5 N3 each), R3 facc / face scratch,
  // R4 face-lift buffers (30 N2 each), R5 1/(w J) (N3)
  // fuse_face: K2 lifted the face rows into vol, no facc staging, no face-lift buffers R4
  static constexpr int PER_EL = 16 * N3 + (fuse_face(N) ? 30 : 60) * N2;
  static constexpr int SMEM = EPB * PER_EL * 8;
  // CTAs per SM: what shared memory allows, but keep >= RMIN registers per thread
  static constexpr int RMIN = N <= 5 ? 64 : 80;
  static constexpr int FIT_S = (228 * 1024) / (SMEM + 1024), FIT_R = 65536 / (THREADS * RMIN);
  static constexpr int FIT = FIT_S < FIT_R ? FIT_S : FIT_R;
  static constexpr int MINB = FIT < 1 ? 1 : (FIT > 8 ? 8 : FIT);
  static constexpr int LPT = (EPB * 5 * N2 + THREADS - 1) / THREADS;  // epilogue lines per thread
};

// Line pass along D over nbs = nb*5 tensors [N^3] with element strides; optional
// injection of a face array (two sides, [s][side][N2] per element) through the
// boundary vectors bvec[side][r], and optional scaling by 1/(w J) (smem).
template <int N, int D, bool INJ, bool DIV>
__device__ __forceinline__ void tail_pass(const double (&op)[N * N], const double (&bvec)[2 * N],
                                          const double* inj, int inj_es, const double* in, int in_es,
                                          double* out, int out_es, const double* wj, int nbs,
                                          int tid, int nthr) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N : N2);
  for (int it = tid; it < nbs * N2; it += nthr) {
    const int bsi = it / N2, l = it - bsi * N2;
    const int b = bsi / 5, s = bsi - 5 * b;
    const int l0 = l % N, l1 = l / N;
    const int base = D == 0 ? N * (l0 + N * l1) : (D == 1 ? l0 + N2 * l1 : l0 + N * l1);
    const double* src = in + b * in_es + s * N3 + base;
    double x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = src[a * stride];
    double f0 = 0.0, f1 = 0.0;
    if (INJ) {
      f0 = inj[b * inj_es + (s * 2 + 0) * N2 + l];
      f1 = inj[b * inj_es + (s * 2 + 1) * N2 + l];
    }
    double* dst = out + b * out_es + s * N3 + base;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(op[r * N + a], x[a], acc);
      if (INJ) {
        acc = fma(bvec[r], f0, acc);
        acc = fma(bvec[N + r], f1, acc);
      }
      if (DIV) acc = acc * wj[b * N3 + base + r * stride];  // wj holds 1/(w J)
      dst[r * stride] = acc;
    }
  }
}

// The same line pass through a folded centrosymmetric operator (no injection).
template <int N, int D, bool DIV>
__device__ __forceinline__ void tail_pass_sym(const SymOp<N>& op, const double* in, int in_es, double* out,
                                              int out_es, const double* wj, int nbs, int tid, int nthr) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N : N2);
  for (int it = tid; it < nbs * N2; it += nthr) {
    const int bsi = it / N2, l = it - bsi * N2;
    const int b = bsi / 5, s = bsi - 5 * b;
    const int l0 = l % N, l1 = l / N;
    const int base = D == 0 ? N * (l0 + N * l1) : (D == 1 ? l0 + N2 * l1 : l0 + N * l1);
    const double* src = in + b * in_es + s * N3 + base;
    double x[N], y[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = src[a * stride];
    op.apply(x, y);
    double* dst = out + b * out_es + s * N3 + base;
#pragma unroll
    for (int r = 0; r < N; ++r) dst[r * stride] = DIV ? y[r] * wj[b * N3 + base + r * stride] : y[r];
  }
}

#ifndef NSFR_UPD_HOIST_MAX
#define NSFR_UPD_HOIST_MAX 2
#endif
#define NSFR_UPD_LINES(j) _Pragma("unroll") for (int j = 0; j < LPT; ++j)
// One line of that pass for a thread whose (tensor bsi, line l0 + N l1) was
// worked out once per batch: the index arithmetic of the five passes (two
// divisions by constants each) is done once for the thread's one or two lines
// (measured K3: n = 5 -3.5%, n = 4 -6.7%, n = 6 -1.8%).
template <int N, int D, bool DIV>
__device__ __forceinline__ void tail_line_sym(const SymOp<N>& op, const double* in, double* out,
                                              const double* wjb, int bsi, int l0, int l1) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int stride = D == 0 ? 1 : (D == 1 ? N : N2);
  const int base = D == 0 ? N * (l0 + N * l1) : (D == 1 ? l0 + N2 * l1 : l0 + N * l1);
  const double* src = in + bsi * N3 + base;
  double x[N], y[N];
#pragma unroll
  for (int a = 0; a < N; ++a) x[a] = src[a * stride];
  op.apply(x, y);
  double* dst = out + bsi * N3 + base;
#pragma unroll
  for (int r = 0; r < N; ++r) dst[r * stride] = DIV ? y[r] * wjb[base + r * stride] : y[r];
}

// Face-array pass (10 arrays [s][side] of N2 per element) along t1 (T=0) or t2 (T=1).
// Callers pass a virtual thread index from face_vt. At n >= 6 the face items
// fill the threads counted from the top of the block, i.e. those the volume
// tail_pass of the same phase leaves idle (phase 1 at p=5: at most 2 line items
// per thread instead of 3; K3 -3.5%). At p=3/4 the same remap measured +1.6% /
// +0.3%, so there the face items start at thread 0.
template <int N>
__device__ __forceinline__ int face_vt(int tid, int nthr, int off) {
  if constexpr (N < 6) return tid;
  return (((nthr - 1 - tid - off) % nthr) + nthr) % nthr;
}

template <int N, int T>
__device__ __forceinline__ void tail_face_pass(const double (&op)[N * N], const double* in, int in_es,
                                               double* out, int out_es, int nb, int tid, int nthr) {
  constexpr int N2 = N * N;
  constexpr int stride = T == 0 ? 1 : N;
  for (int it = tid; it < nb * 10 * N; it += nthr) {
    const int b = it / (10 * N), r = it - b * 10 * N, bi = r / N, l = r - bi * N;
    const int base = T == 0 ? N * l : l;
    const double* src = in + b * in_es + bi * N2 + base;
    double x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = src[a * stride];
    double* dst = out + b * out_es + bi * N2 + base;
#pragma unroll
    for (int rr = 0; rr < N; ++rr) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(op[rr * N + a], x[a], acc);
      dst[rr * stride] = acc;
    }
  }
}

template <int N>
__device__ __forceinline__ void upd_prefetch(const UpdParams& P, int e0, int tid) {
  using Cfg = UpdCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, EPB = Cfg::EPB;
  if (e0 >= P.pj.E || tid >= 6) return;
  const size_t nb = min(EPB, P.pj.E - e0), b8 = sizeof(double);
  switch (tid) {
    case 0: l2_prefetch(P.vol + (size_t)e0 * 5 * N3, nb * 5 * N3 * b8); break;
    case 1: if (!fuse_face(N)) l2_prefetch(P.facc + (size_t)e0 * 30 * N2, nb * 30 * N2 * b8); break;
    case 2: l2_prefetch(P.wj + (size_t)e0 * N3, nb * N3 * b8); break;
    case 3: if (P.stage >= 1) l2_prefetch(P.un + (size_t)e0 * 5 * N3, nb * 5 * N3 * b8); break;
    case 4: if (P.stage >= 2) l2_prefetch(P.acc + (size_t)e0 * 5 * N3, nb * 5 * N3 * b8); break;
    default: if (P.vhat) l2_prefetch(P.vhat + (size_t)e0 * 5 * N3, nb * 5 * N3 * b8);
  }
}

// chi Pi~ = I (c_DG, where Pi~ = Pi = chi^-1; the host decides, round-off-level
// change): IDM: M = Pi~^T chi^T = I as well, so lift + first half of the WA
// inverse reduce to the pointwise face injection and 1/(w J) (same fma order);
// IDF: the RK stages also skip the final three (chi Pi~) passes.
// One team (the CTA; team-generic so a warp could own an element) runs the tail for its nb <=
// EPB elements e0.. in its shared region sm, with its own staging barrier bar.
// NT: threads per team (compile time: the RK-operand preload depth).
template <int N, int EPB, int NT, class Team, bool IDM, bool IDF, bool OUT>
__device__ __forceinline__ void upd_batch(const UpdParams& P, const UpdOps<N>& O, int e0, int nb, double* sm,
                                          unsigned long long* bar_p, const Team& tm, long long pe = -1) {
  constexpr int N2 = N * N, N3 = N * N * N;
  constexpr int LPT = (EPB * 5 * N2 + NT - 1) / NT;  // epilogue lines per thread
  constexpr int VS = 5 * N3, FS = 30 * N2;  // element strides of the volume / face regions
  double* R0 = sm;                 // vol, then Pi~^T R, then u_{s+1}
  double* R1 = R0 + EPB * VS;
  double* R2 = R1 + EPB * VS;
  double* R3 = R2 + EPB * VS;      // facc [b][dir][s][side][N2], later proj_core face scratch
  constexpr bool INJ = !fuse_face(N);  // fused: the face lifts are already in vol (K2)
  double* R4 = INJ ? R3 + EPB * FS : R3;  // [b][G1 | G2 | H2] (10 N2 each); unused when fused
  double* WJ = R4 + EPB * FS;
  const TailOps<N>& T = O.t;
  const int tid = tm.tid(), nthr = tm.nthr();
  const int nbs = nb * 5;
  // a thread's line(s) of every pass: the indices once per batch (tail_line_sym)
  constexpr bool ONE = !INJ && NSFR_UPD_HOIST_MAX >= LPT;
  bool on1[LPT];
  int bsi1[LPT], q0[LPT], q1[LPT];
  const double* wjb1[LPT];
#pragma unroll
  for (int j = 0; j < LPT; ++j) {
    const int it = tid + j * NT;
    on1[j] = it < nbs * N2;
    bsi1[j] = it / N2;
    q0[j] = (it - bsi1[j] * N2) % N;
    q1[j] = (it - bsi1[j] * N2) / N;
    wjb1[j] = WJ + (bsi1[j] / 5) * N3;
  }
  PHASE_START();
  // the team syncs on the barrier's initialisation alone; thread 0 then issues
  // the TMA copies (and the look-ahead L2 prefetch of batch `pe`) while the
  // others already load their RK operands (see k_residual's res_batch)
  if (tid == 0) mbar_init(bar_p, 1);
  tm.sync();
  {
    const StageBlock blk[3] = {{R0, P.vol + (size_t)e0 * VS, nb * VS},
                               {R3, P.facc + (size_t)e0 * FS, INJ ? nb * FS : 0},
                               {WJ, P.wj + (size_t)e0 * N3, nb * N3}};
    stage_copy<3>(blk, bar_p, tm);
  }
  if (pe >= 0 && pe < P.pj.E) upd_prefetch<N>(P, static_cast<int>(pe), tid);
  // RK operands of the final pass (zeta lines, same mapping), loaded ahead so
  // their latency hides behind the passes in between
  double pre_un[LPT][N], pre_acc[LPT][N];
  auto preload = [&]() {
#pragma unroll
    for (int j = 0; j < LPT; ++j) {
      const int it = tid + j * nthr;
#pragma unroll
      for (int c = 0; c < N; ++c) pre_un[j][c] = pre_acc[j][c] = 0.0;
      if (it < nbs * N2 && P.stage >= 1) {
        const int bsi = it / N2, l = it - bsi * N2;
        const size_t gb = (size_t)e0 * VS + (size_t)bsi * N3 + l;
#pragma unroll
        for (int c = 0; c < N; ++c) {
          pre_un[j][c] = P.un[gb + c * N2];
          if (P.stage >= 2) pre_acc[j][c] = P.acc[gb + c * N2];
        }
      }
    }
  };
  // p >= 5: loaded after the first-half passes instead (registers free through
  // them; measured K3 -7.6% at p=5, +0.5% at p=4)
  constexpr bool LATE = N >= 6;
  if constexpr (!LATE) preload();
  stage_wait(bar_p);
  tm.sync();
  PHASE_MARK(8);

  if (IDM && !P.dS) {
    // M = I: vol + b_f (x) facc_f injected per node (x, y, z faces in the pass
    // order), times 1/(w J)
    for (int it = tid; it < nbs * N3; it += nthr) {
      const int bsi = it / N3, q = it - bsi * N3, b = bsi / 5;
      double v = R0[it];
      if constexpr (INJ) {
        const int s = bsi - 5 * b;
        const int i = q % N, j = (q / N) % N, k = q / N2;
        const double* fb = R3 + b * FS + (s * 2) * N2;
        v = fma(T.bm[i], fb[j + N * k], v);
        v = fma(T.bm[N + i], fb[N2 + j + N * k], v);
        v = fma(T.bm[j], fb[10 * N2 + i + N * k], v);
        v = fma(T.bm[N + j], fb[10 * N2 + N2 + i + N * k], v);
        v = fma(T.bm[k], fb[20 * N2 + i + N * j], v);
        v = fma(T.bm[N + k], fb[20 * N2 + N2 + i + N * j], v);
      }
      R0[it] = v * WJ[b * N3 + q];
    }
    tm.sync();
  } else if (!P.dS) {
    // Pi~^T S9 in three fused passes; 1/(w J) in the last
    if constexpr (INJ) {
      tail_pass<N, 0, true, false>(T.M, T.bm, R3, FS, R0, VS, R1, VS, WJ, nbs, tid, nthr);
      tail_face_pass<N, 0>(T.M, R3 + 10 * N2, FS, R4, FS, nb, face_vt<N>(tid, nthr, 0), nthr);
      tail_face_pass<N, 0>(T.M, R3 + 20 * N2, FS, R4 + 10 * N2, FS, nb, face_vt<N>(tid, nthr, nb * 10 * N), nthr);
      tm.sync();
      tail_pass<N, 1, true, false>(T.M, T.bm, R4, FS, R1, VS, R2, VS, WJ, nbs, tid, nthr);
      tail_face_pass<N, 1>(T.M, R4 + 10 * N2, FS, R4 + 20 * N2, FS, nb, face_vt<N>(tid, nthr, 0), nthr);
      tm.sync();
      tail_pass<N, 2, true, true>(T.M, T.bm, R4 + 20 * N2, FS, R2, VS, R0, VS, WJ, nbs, tid, nthr);
    } else {
      if constexpr (ONE) {
        NSFR_UPD_LINES(j) if (on1[j]) tail_line_sym<N, 0, false>(T.Ms, R0, R1, wjb1[j], bsi1[j], q0[j], q1[j]);
        tm.sync();
        NSFR_UPD_LINES(j) if (on1[j]) tail_line_sym<N, 1, false>(T.Ms, R1, R2, wjb1[j], bsi1[j], q0[j], q1[j]);
        tm.sync();
        NSFR_UPD_LINES(j) if (on1[j]) tail_line_sym<N, 2, true>(T.Ms, R2, R0, wjb1[j], bsi1[j], q0[j], q1[j]);
      } else {
        tail_pass_sym<N, 0, false>(T.Ms, R0, VS, R1, VS, WJ, nbs, tid, nthr);
        tm.sync();
        tail_pass_sym<N, 1, false>(T.Ms, R1, VS, R2, VS, WJ, nbs, tid, nthr);
        tm.sync();
        tail_pass_sym<N, 2, true>(T.Ms, R2, VS, R0, VS, WJ, nbs, tid, nthr);
      }
    }
    tm.sync();
  } else {
    // entropy diagnostic: R = S9 explicitly (chi^T, bound_sol), -v_hat . R, then Pi~^T
    tail_pass<N, 0, INJ, false>(T.it, T.bs, R3, FS, R0, VS, R1, VS, WJ, nbs, tid, nthr);
    if constexpr (INJ) {
      tail_face_pass<N, 0>(T.it, R3 + 10 * N2, FS, R4, FS, nb, face_vt<N>(tid, nthr, 0), nthr);
      tail_face_pass<N, 0>(T.it, R3 + 20 * N2, FS, R4 + 10 * N2, FS, nb, face_vt<N>(tid, nthr, nb * 10 * N), nthr);
    }
    tm.sync();
    tail_pass<N, 1, INJ, false>(T.it, T.bs, R4, FS, R1, VS, R2, VS, WJ, nbs, tid, nthr);
    if constexpr (INJ)
      tail_face_pass<N, 1>(T.it, R4 + 10 * N2, FS, R4 + 20 * N2, FS, nb, face_vt<N>(tid, nthr, 0), nthr);
    tm.sync();
    tail_pass<N, 2, INJ, false>(T.it, T.bs, R4 + 20 * N2, FS, R2, VS, R0, VS, WJ, nbs, tid, nthr);
    tm.sync();
    for (int it = tid; it < nbs * N3; it += nthr) R1[it] = P.vhat[(size_t)e0 * VS + it] * R0[it];
    tm.sync();
    if (tid < nb) {
      double s = 0.0;
      for (int r = 0; r < VS; ++r) s += R1[tid * VS + r];
      P.dS[e0 + tid] = -s;
    }
    tm.sync();
    tail_pass<N, 0, false, false>(T.frt, T.bs, nullptr, 0, R0, VS, R1, VS, WJ, nbs, tid, nthr);
    tm.sync();
    tail_pass<N, 1, false, false>(T.frt, T.bs, nullptr, 0, R1, VS, R2, VS, WJ, nbs, tid, nthr);
    tm.sync();
    tail_pass<N, 2, false, true>(T.frt, T.bs, nullptr, 0, R2, VS, R0, VS, WJ, nbs, tid, nthr);
    tm.sync();
  }
  PHASE_MARK(9);
  if constexpr (LATE) preload();
  // second half of S10: Pi~ along xi, eta
  if constexpr (!IDF) {
    if constexpr (ONE) {
      NSFR_UPD_LINES(j) if (on1[j]) tail_line_sym<N, 0, false>(T.frs, R0, R1, wjb1[j], bsi1[j], q0[j], q1[j]);
      tm.sync();
      NSFR_UPD_LINES(j) if (on1[j]) tail_line_sym<N, 1, false>(T.frs, R1, R2, wjb1[j], bsi1[j], q0[j], q1[j]);
      tm.sync();
    } else {
      tail_pass_sym<N, 0, false>(T.frs, R0, VS, R1, VS, WJ, nbs, tid, nthr);
      tm.sync();
      tail_pass_sym<N, 1, false>(T.frs, R1, VS, R2, VS, WJ, nbs, tid, nthr);
      tm.sync();
    }
  }
  // Pi~ along zeta, negate, RK stage epilogue (zeta lines: coalesced across the
  // warp); u_{s+1} also lands in R0 for the projection below
  const double dt = P.stage ? *P.dt : 0.0;
  const double hdt = 0.5 * dt, sdt = dt / 6.0;
#pragma unroll
  for (int j = 0; j < LPT; ++j) {
    const int it = tid + j * nthr;
    if (it >= nbs * N2) break;
    const int bsi = it / N2, l = it - bsi * N2;
    const double* src = (IDF ? R0 : R2) + bsi * N3 + l;  // IDF: each thread rewrites only its own line
    double x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = src[a * N2];
    const size_t gb = (size_t)e0 * VS + (size_t)bsi * N3 + l;
    double* nxt = R0 + bsi * N3 + l;
    double kv[N];
    if constexpr (IDF) {
#pragma unroll
      for (int c = 0; c < N; ++c) kv[c] = -x[c];
    } else {
      T.frs.apply(x, kv);
#pragma unroll
      for (int c = 0; c < N; ++c) kv[c] = -kv[c];
    }
    // one (warp-uniform) stage dispatch per line, not per node
    switch (P.stage) {
      case 0:
#pragma unroll
        for (int c = 0; c < N; ++c) P.out[gb + c * N2] = kv[c];
        break;
      case 1:
#pragma unroll
        for (int c = 0; c < N; ++c) {
          P.acc[gb + c * N2] = kv[c];
          nxt[c * N2] = fma(hdt, kv[c], pre_un[j][c]);
        }
        break;
      case 2:
      case 3: {
        const double cdt = P.stage == 2 ? hdt : dt;
#pragma unroll
        for (int c = 0; c < N; ++c) {
          P.acc[gb + c * N2] = fma(2.0, kv[c], pre_acc[j][c]);
          nxt[c * N2] = fma(cdt, kv[c], pre_un[j][c]);
        }
        break;
      }
      default:
#pragma unroll
        for (int c = 0; c < N; ++c) {
          const double u1 = fma(sdt, pre_acc[j][c] + kv[c], pre_un[j][c]);
          P.un[gb + c * N2] = u1;
          nxt[c * N2] = u1;
        }
    }
  }
  if (P.stage == 0) return;
  tm.sync();
  PHASE_MARK(10);
  if constexpr (OUT) {
    // the state leaves for the host: u_hat = Pi^3 u_{n+1} (kernel_convert's
    // passes, same bits as k_convert_lines) and adaptive_dt's lambda of it,
    // instead of a projection the next (uploaded) state would replace
    conv_passes<N, true, true, Team>(O.p.proj, R0, P.uhat_out, e0, nb, tm);
    if (P.lam_out) {
      conv_passes<N, false, true, Team>(O.p.chi, R0, nullptr, e0, nb, tm);
      conv_lambda<N, Team>(R0, nb, P.pj.gamma, P.lam_out, tm);
    }
    return;
  }
  proj_core<N, EPB, Team>(P.pj, O.p, e0, nb, R0, R1, R2, R3, tm);
}

// One batch per CTA with look-ahead L2 prefetch (see k_residual).
template <int N, bool IDM = false, bool IDF = false, bool OUT = false>
__global__ void __launch_bounds__(UpdCfg<N>::THREADS, UpdCfg<N>::MINB)
    k_update(UpdParams P, UpdOps<N> O, int ahead) {
  extern __shared__ __align__(128) double sm[];
  dbg_kernel_entry(sm);
  constexpr int EPB = UpdCfg<N>::EPB;
  __shared__ unsigned long long bar;
  const long long pe = P.pj.e_begin + (static_cast<long long>(NSFR_BID) + ahead) * EPB;
  const int e0 = P.pj.e_begin + NSFR_BID * EPB;
  upd_batch<N, EPB, UpdCfg<N>::THREADS, CtaTeam, IDM, IDF, OUT>(P, O, e0, min(EPB, P.pj.E - e0), sm, &bar,
                                                                 CtaTeam{}, pe);
}

}  // namespace nsfr_b200
