// K2: residual rows S6-S8 for one RK stage:
//   S6  volume Hadamard flux differencing   (sumfac.hpp:48-94, 0.5*skew -> skew(a,b), D2)
//   S7  hybrid surface-volume Hadamard      (sumfac.hpp:110-157, own face cofactor, D1)
//   S8  EC + Roe face flux vs the neighbour's trace (euler.cpp:142-162, 229-301; D3)
// Output: the volume rows vol = sum over directions [E][5][N^3], with the face
// rows already lifted onto their lines (fuse_face, n = 4..7: vol + sum_f l_f (x)
// facc_f); at n = 3 the face rows facc [E][3 dir][5][2 side][N^2] separately.
// The rest of S9, S10 and the RK update run in K3 (kernel_update.cuh), fused
// with the next stage's entropy projection.
//
// Thread mapping. One thread per 1D line (dir, t1, t2) of an element does
// every two-point evaluation touching that line: the n(n-1)/2 volume pairs,
// the 2n hybrid pairs with the two faces it pierces and the two face fluxes.
// Each node belongs to exactly one line per direction, so the per-direction
// accumulators need no atomics (deterministic).
// All 1D operators travel in the kernel parameter (constant) bank.
#pragma once
#include "physics.cuh"

namespace nsfr_b200 {


// S6 volume pairs a < b of one line (sumfac.hpp:76-89): node a's row in
// registers, node b's in the line's shared accumulator. UNR: fully unrolled
// (compile-time indices and coefficients; p=3 K2 -1.6%), used for n <= 4;
// rolled above (the unrolled code outgrows the instruction cache: p=4 +4%,
// p=5 +1.5%; measured).
// Running pointers (node a / node b of PRIM, their cofactor column, the line's
// accumulator) advance by the line stride: the rolled loops carry three
// addresses instead of rebuilding each from (lbase, stride, index) and the
// shared window base every pair (S2R + LEA + 5 IMAD per pair in the SASS).
#define NSFR_VOL_PAIRS_BODY                                                                    \
  {                                                                                            \
    const PrimH pa{pa_p[0], pa_p[N3], pa_p[2 * N3], pa_p[3 * N3], pa_p[4 * N3], pa_p[5 * N3]}; \
    const double ca0 = ca_p[0], ca1 = ca_p[3 * N3], ca2 = ca_p[6 * N3];                        \
    double fa[NS] = {0.0, 0.0, 0.0, 0.0, 0.0};                                                 \
    const double* __restrict__ pb_p = pa_p + stride;                                           \
    const double* __restrict__ cb_p = ca_p + stride;                                           \
    double* __restrict__ ab_p = aa_p + stride;                                                 \
    NSFR_INNER_UNROLL                                                                          \
    for (int bb = a + 1; bb < N; ++bb) {                                                       \
      const PrimH pb{pb_p[0], pb_p[N3], pb_p[2 * N3], pb_p[3 * N3], pb_p[4 * N3], pb_p[5 * N3]}; \
      double f[NS];                                                                            \
      d_flux_h<KE>(pa, pb, ca0 + cb_p[0], ca1 + cb_p[3 * N3], ca2 + cb_p[6 * N3], f);          \
      const double c = wt * q[a * N + bb];                                                     \
      _Pragma("unroll") for (int s = 0; s < NS; ++s) {                                         \
        fa[s] = fma(c, f[s], fa[s]);                                                           \
        ab_p[s * N3] = fma(-c, f[s], ab_p[s * N3]);                                            \
      }                                                                                        \
      pb_p += stride;                                                                          \
      cb_p += stride;                                                                          \
      ab_p += stride;                                                                          \
    }                                                                                          \
    _Pragma("unroll") for (int s = 0; s < NS; ++s) aa_p[s * N3] += fa[s];                      \
    pa_p += stride;                                                                            \
    ca_p += stride;                                                                            \
    aa_p += stride;                                                                            \
  }

#ifndef NSFR_UNROLL_MAXN
#define NSFR_UNROLL_MAXN 4
#endif
__device__ __forceinline__ PrimH load_prim(const double* __restrict__ Pd, int N3, int i) {
  return PrimH{Pd[i], Pd[N3 + i], Pd[2 * N3 + i], Pd[3 * N3 + i], Pd[4 * N3 + i], Pd[5 * N3 + i]};
}

template <int N, bool KE>
__device__ __forceinline__ void vol_pairs(const double* __restrict__ Pd, const double* __restrict__ Ch,
                                          double* __restrict__ acc,
                                          const double (&q)[N * N], double wt, int lbase,
                                          int stride, int dir) {
  constexpr int N3 = N * N * N;
  const double* __restrict__ pa_p = Pd + lbase;
  const double* __restrict__ ca_p = Ch + dir * N3 + lbase;
  double* __restrict__ aa_p = acc + lbase;
  if constexpr (N <= NSFR_UNROLL_MAXN) {
#define NSFR_INNER_UNROLL _Pragma("unroll")
#pragma unroll
    for (int a = 0; a < N - 1; ++a) NSFR_VOL_PAIRS_BODY
#undef NSFR_INNER_UNROLL
  } else {
#define NSFR_INNER_UNROLL _Pragma("unroll 1")
#pragma unroll 1
    for (int a = 0; a < N - 1; ++a) NSFR_VOL_PAIRS_BODY
#undef NSFR_INNER_UNROLL
  }
}
#undef NSFR_VOL_PAIRS_BODY

// n / d for a run-time d by one high multiply: M = ceil(2^64 / d) gives the
// exact quotient for every 32-bit n (n (M d - 2^64) < 2^64). K2 took three
// hardware-less integer divisions per thread to place its batch in the box
// (2.5% of its instructions, their latency ahead of the face loop).
struct DivMagic {
  unsigned long long M;  // 0: d = 1
  int d;
  static DivMagic make(int d) { return DivMagic{d <= 1 ? 0ull : ~0ull / static_cast<unsigned>(d) + 1ull, d}; }
  __device__ __forceinline__ int div(int n) const {
    return M ? static_cast<int>(__umul64hi(static_cast<unsigned long long>(static_cast<unsigned>(n)), M)) : n;
  }
};

struct ResParams {
  const double* ut_vol;   // [E][6][N^3] half-scaled primitives of u~ (K1 / K3)
  const double* traces;   // [E][6 faces][NTR][N^2] primitives of u(v~) (physics.cuh)
  const double* halo_lo;  // [m*m][NTR][N^2] face 5 of plane k0-1 (nullptr: wrap locally)
  const double* halo_hi;  // [m*m][NTR][N^2] face 4 of plane k1
  const double* cof;      // [E][9][N^3] = 0.5 C
  double* vol;            // [E][5][N^3] volume rows
  double* facc;           // [E][3][5][2][N^2] face rows
  unsigned* err;
  int E, m, nz;           // E: end of the launched element range [e_begin, E)
  double gamma;
  int roe;
  int e_begin;            // first element of the launched range (a multiple of 8)
  DivMagic dm, dmm;       // division by m and by m^2 (host-formed multipliers)
  GasC gas;               // gamma and its reciprocals (host-formed)
};

template <int N>
struct ResOps {
  double q[N * N];       // skew(a,b) = q(a,b) - q(b,a), q = 0.5 skew
  double bflux[2 * N];   // flux basis at -1, +1
  double wq[N];          // quadrature weights
};

template <int N>
struct ResCfg {
  static constexpr int N2 = N * N, N3 = N * N * N;
  static constexpr int LINES = 3 * N2;
// n >= 6: one element per CTA (108 / 147 lines in 128 / 160 threads, 4 CTAs
// per SM at p=5) beats two (224 / 320 threads, 2 CTAs): K2 p=5 -1.6%, p=6 -7%.
#ifndef NSFR_RES_EPB_HI
#define NSFR_RES_EPB_HI 1
#endif
  static constexpr int EPB = LINES <= 32 ? 6 : (LINES <= 64 ? 4 : (N >= 6 ? NSFR_RES_EPB_HI : 2));
  static constexpr int THREADS = ((EPB * LINES + 31) / 32) * 32;
  // The element's own face traces (6 NTR N2) are staged with the rest where that
  // helps (N <= 4; measured K2 p=3 -2.4%, p=4 +1.7%): the face loop starts from shared
  // memory instead of waiting on a global load (K2's largest long-scoreboard
  // stall); at N = 5 the longer staging wait costs more, at N >= 6 a CTA per SM.
  static constexpr bool STR = N <= 4;
  // The line phase is bound by the shared-memory data pipe (ncu: l1tex data-pipe
  // wavefronts at 93% of peak), and with the natural thread -> line order its
  // 64-bit accesses cost 1.65 wavefronts per ideal one (bank conflicts between
  // the lines of a half-warp). MAPPED: the lines are dealt to the lanes by a
  // table and the direction accumulators are padded (element stride AS,
  // direction offsets DOFF) so that the same accesses cost ~1.2x
  // (tools/k2_bankmap.c anneals both against the bank model, which reproduces
  // the measured 1.65x). Results are bitwise unchanged: which lane runs a line
  // does not enter its arithmetic. Measured K2 (A/B, one session): n = 4 -12%
  // (model 3.00x -> 2.26x: the power-of-two strides leave 4-way conflicts no
  // lane order removes), n = 5 -3.7% (1.65x -> 1.20x), n = 6 -4.8% (1.90x ->
  // 1.56x), n = 7 -14% (1.70x -> 1.30x).
#ifndef NSFR_RES_MAPMASK
#define NSFR_RES_MAPMASK 0xf0
#endif
  static constexpr bool MAPPED = N >= 4 && N <= 7 && ((NSFR_RES_MAPMASK >> N) & 1);
  // paddings per degree: the smallest offsets >= the dense ones with the
  // annealed residues mod 16 (N = 4: 0, 12, element stride 3; N = 5: 7, 0, 13;
  // N = 6: 5, 6; N = 7: 0, 5)
  static constexpr int DOFF1 = !MAPPED ? 5 * N3 : (N == 4 ? 320 : (N == 5 ? 631 : (N == 6 ? 1093 : 1728)));
  static constexpr int DOFF2 = !MAPPED ? 10 * N3 : (N == 4 ? 652 : (N == 5 ? 1264 : (N == 6 ? 2182 : 3445)));
  // doubles per element of ACCV
  static constexpr int AS = !MAPPED ? 15 * N3 : (N == 4 ? 979 : (N == 5 ? 1901 : (N == 6 ? 3262 : 5160)));
  static constexpr int ACC_ALL = (EPB * AS + 1) / 2 * 2;  // ACCV region (even: PRIM stays 16-byte aligned)
  // ACCV (3 directions x 5 N3, padded) + node primitives (6 N3) + half cofactors (9 N3)
  // [+ own traces 6 NTR N2]
  static constexpr int SMEM = (ACC_ALL + EPB * (15 * N3 + (STR ? 6 * NTR * N2 : 0))) * 8;
#ifdef NSFR_RES_MINB
  static constexpr int MINB = NSFR_RES_MINB;
#else
  // what shared memory allows, except p <= 3: 2 CTAs/SM with the registers the
  // fully unrolled pair loops want beat 3-4 CTAs with spills (measured K2:
  // p=3 -6.2%, p=2 -12%; p=4 keeps 3: 2 is +23%)
  static constexpr int MINB_S = SMEM <= 56 * 1024 ? 4 : (SMEM <= 75 * 1024 ? 3 : (SMEM <= 112 * 1024 ? 2 : 1));
  static constexpr int MINB = N <= 4 && MINB_S > 2 ? 2 : MINB_S;
#endif
};

// L2 prefetch of everything batch `e0` will read (issued one batch ahead) by the
// first lanes of warp 0: the three element blocks and the 2 nb z-neighbour face
// blocks. (Dealing the items to every warp instead measured no gain at p=4 and
// +8% at p=3.)
template <int N>
__device__ __forceinline__ void res_prefetch(const ResParams& P, int e0, int tid) {
  using Cfg = ResCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, EPB = Cfg::EPB;
  if (e0 >= P.E || tid >= 32) return;
  const int nb = min(EPB, P.E - e0);
  const size_t b8 = sizeof(double);
  switch (tid) {
    case 0: l2_prefetch(P.ut_vol + (size_t)e0 * 6 * N3, nb * 6 * N3 * b8); break;
    case 1: l2_prefetch(P.cof + (size_t)e0 * 9 * N3, nb * 9 * N3 * b8); break;
    case 2: l2_prefetch(P.traces + (size_t)e0 * 6 * NTR * N2, nb * 6 * NTR * N2 * b8); break;
    default: {  // neighbour face blocks (geometry.hpp:24-29), lanes 3.. : (element, face)
      // z neighbours only: the x and y neighbours' own blocks are inside the
      // look-ahead window of the CTAs already running (K2 -0.6%)
      const int j = tid - 3;
      if (j >= 2 * nb) break;
      const int e = e0 + j / 2, f = 4 + (j & 1), dir = 2, step = (f & 1) ? 1 : -1;
      const int mm = P.m;
      int kl = P.dmm.div(e);
      const int pl = e - kl * mm * mm;
      int jj = P.dm.div(pl), i = pl - jj * mm;
      if (dir == 0) i = (i + step + mm) % mm;
      if (dir == 1) jj = (jj + step + mm) % mm;
      if (dir == 2) {
        kl += step;
        if (kl < 0 || kl >= P.nz) {
          const double* halo = kl < 0 ? P.halo_lo : P.halo_hi;
          if (halo) {
            l2_prefetch(halo + (size_t)(i + mm * jj) * NTR * N2, NTR * N2 * b8);
            break;
          }
          kl = (kl + P.nz) % P.nz;
        }
      }
      l2_prefetch(P.traces + ((size_t)(i + mm * (jj + mm * kl)) * 6 + (f ^ 1)) * NTR * N2, NTR * N2 * b8);
    }
  }
}

// KM (kinetic-energy diagnostics; every two-point flux minus the pressure work):
//   0 the residual; 1 volume rows only (S6); 2 all rows (S6-S8) without Roe.

// Shared-memory carve-up of one batch: ACCV [EPB][3][5][N3] direction
// accumulators (element stride AS, direction offsets 0 / DOFF1 / DOFF2), PRIM [EPB][6][N3] half-scaled primitives, COF [EPB][9][N3] 0.5 C.
template <int N>
struct ResSmem {
  static constexpr int N3 = N * N * N, EPB = ResCfg<N>::EPB, ACC_ALL = ResCfg<N>::ACC_ALL;
  double *ACCV, *PRIM, *COF, *TRC;  // TRC [EPB][6][NTR][N2] (ResCfg::STR), else nullptr
  __device__ __forceinline__ explicit ResSmem(double* sm)
      : ACCV(sm), PRIM(sm + ACC_ALL), COF(sm + ACC_ALL + EPB * 6 * N3),
        TRC(ResCfg<N>::STR ? sm + ACC_ALL + EPB * 15 * N3 : nullptr) {}
};

// the staging blocks of batch e0 (pure copies: node primitives of u~ and 0.5 C)
template <int N>
__device__ __forceinline__ void res_stage_blocks(const ResParams& P, const ResSmem<N>& S, int e0, int nb,
                                                 StageBlock (&blk)[3]) {
  constexpr int N2 = N * N, N3 = N * N * N;
  blk[0] = {S.PRIM, P.ut_vol + (size_t)e0 * 6 * N3, nb * 6 * N3};
  blk[1] = {S.COF, P.cof + (size_t)e0 * 9 * N3, nb * 9 * N3};
  blk[2] = {S.TRC, P.traces + (size_t)e0 * 6 * NTR * N2, ResCfg<N>::STR ? nb * 6 * NTR * N2 : 0};
}

// Thread -> line table of the MAPPED configurations (tools/k2_bankmap.c; code =
// b << 12 | dir << 8 | t2 << 4 | t1, 0xffff = idle lane). N = 5, two elements
// per CTA: 1.197 wavefronts per ideal one in the bank model (natural order 1.656).
__device__ const unsigned short g_res_map5[160] = {
    0x0013, 0x0004, 0x0210, 0x0214, 0x0201, 0x0212, 0xffff, 0x0033, 0x0031, 0x0203, 0x0230, 0x0042, 0x0022, 0x0024, 0x0020, 0x0223,
    0xffff, 0x1212, 0x0140, 0x1103, 0xffff, 0x0244, 0x0131, 0x1130, 0x0211, 0x1114, 0x0233, 0x0231, 0xffff, 0x0220, 0x1141, 0x0224,
    0x0141, 0x0114, 0x1231, 0x1120, 0x0221, 0x0243, 0x1140, 0x1124, 0x1111, 0x1213, 0xffff, 0x0232, 0x1113, 0x1133, 0x0234, 0xffff,
    0x0204, 0x0041, 0x0023, 0x0014, 0x0012, 0xffff, 0x0222, 0x0213, 0x0001, 0xffff, 0x0242, 0x0202, 0x0200, 0x0030, 0x0003, 0x0021,
    0x1100, 0x1134, 0x1123, 0x1142, 0x1131, 0x1101, 0xffff, 0x1102, 0x1121, 0x1112, 0x1144, 0x1110, 0x1132, 0x1143, 0xffff, 0x1122,
    0x1033, 0x1031, 0x1023, 0x1010, 0x1014, 0x1012, 0x1020, 0x1011, 0x1004, 0x1013, 0x1022, 0x1034, 0x1030, 0x1024, 0x1021, 0x1032,
    0x0113, 0x0130, 0x0123, 0x0132, 0x0122, 0x0133, 0x0144, 0x0110, 0x0134, 0x0143, 0x0101, 0x0120, 0x0111, 0x0103, 0x0100, 0x0142,
    0x0112, 0x1232, 0x1104, 0x0032, 0x1233, 0x1204, 0x0102, 0x0241, 0x0240, 0x1043, 0x0104, 0x1242, 0x0124, 0x0121, 0x1203, 0x1241,
    0x0040, 0x0002, 0x0043, 0x0034, 0x0010, 0x1044, 0x0000, 0x1042, 0x1000, 0x1003, 0x0011, 0x0044, 0x1040, 0x1002, 0x1001, 0x1041,
    0x1211, 0x1240, 0x1234, 0x1224, 0x1221, 0x1220, 0x1244, 0x1222, 0x1200, 0x1214, 0x1201, 0x1202, 0x1243, 0x1210, 0x1230, 0x1223};
// N = 4, four elements per CTA: 2.26 wavefronts per ideal one (natural order 3.00)
__device__ const unsigned short g_res_map4[192] = {
    0x3113, 0x2122, 0x2130, 0x2133, 0x0100, 0x1100, 0x2111, 0x0030, 0x0121, 0x1101, 0x1132, 0x3013, 0x0001, 0x1020, 0x3012, 0x0022,
    0x2121, 0x1021, 0x3020, 0x2132, 0x1010, 0x3110, 0x1113, 0x3123, 0x1012, 0x1131, 0x3132, 0x0123, 0x2002, 0x2011, 0x0002, 0x2020,
    0x0200, 0x0201, 0x0202, 0x0203, 0x0210, 0x0211, 0x0212, 0x0213, 0x0220, 0x0221, 0x0222, 0x0223, 0x0230, 0x0231, 0x0232, 0x0233,
    0x0021, 0x0112, 0x2033, 0x2000, 0x0103, 0x0130, 0x2100, 0x1033, 0x3112, 0x0023, 0x3133, 0x1122, 0x3121, 0x3010, 0x2123, 0x3111,
    0x1022, 0x3033, 0x3031, 0x3002, 0x2013, 0x0011, 0x2012, 0x3030, 0x1023, 0x1031, 0x0020, 0x2030, 0x0032, 0x0013, 0x2031, 0x1000,
    0x1200, 0x1201, 0x1202, 0x1203, 0x1210, 0x1211, 0x1212, 0x1213, 0x1220, 0x1221, 0x1222, 0x1223, 0x1230, 0x1231, 0x1232, 0x1233,
    0x2010, 0x2102, 0x2023, 0x1112, 0x0132, 0x3120, 0x3022, 0x1123, 0x3101, 0x1030, 0x2131, 0x0113, 0x0031, 0x0111, 0x2021, 0x3023,
    0x2120, 0x3000, 0x3011, 0x0120, 0x2112, 0x2001, 0x0003, 0x3103, 0x3102, 0x3001, 0x1013, 0x2113, 0x2003, 0x1130, 0x0010, 0x1032,
    0x2200, 0x2201, 0x2202, 0x2203, 0x2210, 0x2211, 0x2212, 0x2213, 0x2220, 0x2221, 0x2222, 0x2223, 0x2230, 0x2231, 0x2232, 0x2233,
    0x0012, 0x3021, 0x0033, 0x2110, 0x3122, 0x0122, 0x3003, 0x1111, 0x3131, 0x3130, 0x0133, 0x0110, 0x1001, 0x0101, 0x2032, 0x1003,
    0x0102, 0x2101, 0x1110, 0x1120, 0x1133, 0x1103, 0x3100, 0x1102, 0x0131, 0x1121, 0x1011, 0x2022, 0x0000, 0x1002, 0x2103, 0x3032,
    0x3200, 0x3201, 0x3202, 0x3203, 0x3210, 0x3211, 0x3212, 0x3213, 0x3220, 0x3221, 0x3222, 0x3223, 0x3230, 0x3231, 0x3232, 0x3233};
// N = 6, one element per CTA: 1.56 (natural order 1.90)
__device__ const unsigned short g_res_map6[128] = {
    0x0020, 0x0114, 0x0033, 0x0140, 0x0034, 0x0101, 0x0054, 0x0105, 0x0041, 0x0125, 0x0035, 0x0015, 0x0121, 0x0144, 0x0052, 0x0230,
    0x0005, 0x0224, 0x0145, 0x0253, 0x0143, 0x0012, 0x0055, 0x0151, 0x0104, 0x0042, 0x0115, 0x0135, 0x0153, 0x0025, 0x0202, 0x0203,
    0x0004, 0x0040, 0xffff, 0x0023, 0x0134, 0x0050, 0x0003, 0x0152, 0x0124, 0x0122, 0x0102, 0x0002, 0x0120, 0xffff, 0x0110, 0x0013,
    0x0132, 0x0021, 0x0044, 0x0022, 0x0000, 0x0100, 0x0112, 0x0130, 0x0154, 0x0142, 0x0053, 0x0150, 0xffff, 0x0030, 0x0051, 0x0031,
    0x0045, 0x0010, 0x0011, 0x0141, 0x0032, 0x0014, 0x0133, 0x0043, 0x0113, 0x0131, 0x0103, 0x0024, 0x0001, 0x0123, 0x0155, 0x0111,
    0x0243, 0x0235, 0x0254, 0x0244, 0x0231, 0x0232, 0x0214, 0x0225, 0x0200, 0x0240, 0x0210, 0x0222, 0x0241, 0x0233, 0x0223, 0x0245,
    0x0204, 0x0215, 0x0255, 0x0221, 0x0201, 0x0250, 0x0213, 0x0242, 0x0252, 0xffff, 0x0220, 0x0251, 0x0211, 0x0205, 0x0212, 0x0234,
    0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff, 0xffff};
// N = 7, one element per CTA: 1.30 (natural order 1.70)
__device__ const unsigned short g_res_map7[160] = {
    0x0036, 0x0060, 0x0043, 0xffff, 0x0024, 0x0032, 0x0066, 0x0011, 0x0052, 0x0026, 0x0056, 0x0041, 0x0025, 0x0053, 0x0040, 0x0064,
    0x0021, 0x0051, 0x0002, 0x0050, 0x0044, 0x0016, 0x0035, 0x0061, 0x0034, 0x0054, 0x0030, 0x0020, 0x0033, 0x0045, 0x0062, 0x0031,
    0x0015, 0x0022, 0x0001, 0x0005, 0x0003, 0x0065, 0x0013, 0x0063, 0x0010, 0x0006, 0x0055, 0x0014, 0x0042, 0x0012, 0x0004, 0x0046,
    0x0142, 0x0140, 0x0110, 0x0166, 0x0100, 0x0120, 0x0150, 0x0156, 0x0163, 0x0162, 0x0121, 0x0164, 0xffff, 0x0116, 0xffff, 0xffff,
    0x0122, 0x0141, 0x0153, 0x0133, 0x0136, 0x0102, 0x0161, 0xffff, 0x0131, 0x0135, 0x0155, 0x0112, 0x0132, 0x0146, 0x0152, 0x0160,
    0x0023, 0x0101, 0xffff, 0x0130, 0xffff, 0x0000, 0x0145, 0xffff, 0x0123, 0x0143, 0x0222, 0x0151, 0x0115, 0xffff, 0x0165, 0xffff,
    0x0104, 0xffff, 0x0114, 0x0111, 0x0125, 0x0154, 0x0113, 0xffff, 0x0124, 0x0106, 0x0105, 0x0144, 0x0103, 0xffff, 0x0134, 0x0126,
    0x0255, 0x0201, 0x0200, 0x0246, 0x0241, 0x0264, 0x0252, 0x0253, 0x0243, 0x0256, 0x0260, 0x0236, 0x0203, 0x0204, 0x0240, 0x0210,
    0x0261, 0x0206, 0x0266, 0x0263, 0x0251, 0x0232, 0x0242, 0x0235, 0x0205, 0x0223, 0x0250, 0x0221, 0x0215, 0x0211, 0x0202, 0x0212,
    0x0234, 0x0226, 0x0244, 0x0265, 0x0214, 0x0245, 0x0220, 0x0230, 0x0213, 0x0254, 0x0233, 0x0225, 0x0262, 0x0216, 0x0231, 0x0224};
// A global (L1-cached) table, not a __constant__ one: every lane reads its own
// entry, which the constant cache would serialise 32 ways.
template <int N>
__device__ __forceinline__ unsigned res_line_map(int tid) {
  static_assert(N >= 4 && N <= 7, "no line map for this degree");
  if constexpr (N == 4) return __ldg(&g_res_map4[tid]);
  if constexpr (N == 5) return __ldg(&g_res_map5[tid]);
  if constexpr (N == 6) return __ldg(&g_res_map6[tid]);
  return __ldg(&g_res_map7[tid]);
}

template <int N, int KM>
__device__ __forceinline__ void res_lines(const ResParams& P, const ResOps<N>& O, int e0, int nb,
                                          const ResSmem<N>& S);
template <int N>
__device__ __forceinline__ void res_writeout(const ResParams& P, int e0, int nb, const double* ACCV);

// Order of a batch. Thread 0 initialises the staging barrier and issues the TMA
// copies at once, so the data is in flight from the first instructions on (its
// ~3000-cycle flight is the one wait a CTA cannot avoid); meanwhile every thread
// clears the direction accumulators. One CTA barrier publishes both. Then warp
// 0 issues the look-ahead L2 prefetch of batch `pe`, and each thread waits on
// the mbarrier ITSELF: no second CTA barrier, so no warp waits for warp 0's
// prefetch before its lines (only the per-thread cp.async fallback of a
// misaligned block still needs one). History: with one barrier behind the
// prefetch and the TMA issue, four warps spent 9.7% of the kernel's warp time
// waiting for warp 0 (K2 -9% when it moved ahead of the issue).
template <int N, int KM>
__device__ __forceinline__ void res_batch(const ResParams& P, const ResOps<N>& O, int e0, long long pe,
                                          double* sm) {
  using Cfg = ResCfg<N>;
  constexpr int EPB = Cfg::EPB;
  const ResSmem<N> S(sm);
  const int nb = min(EPB, P.E - e0);
  PHASE_START();
  __shared__ unsigned long long bar;
  bool all_bulk = true;
  {
    StageBlock blk[3];
    res_stage_blocks<N>(P, S, e0, nb, blk);
    stage_issue<3>(blk, &bar);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      all_bulk = all_bulk && (blk[i].count == 0 || bulk_ok(blk[i].src, blk[i].dst, blk[i].count * sizeof(double)));
  }
  {  // ACCV (an even number of doubles, 16-byte aligned) = 0
    double2* z = reinterpret_cast<double2*>(S.ACCV);
    constexpr int NZ = Cfg::ACC_ALL / 2;
    for (int i = threadIdx.x; i < NZ; i += Cfg::THREADS) z[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (pe < P.E) res_prefetch<N>(P, static_cast<int>(pe), threadIdx.x);
  stage_wait(&bar);
  if (!all_bulk) __syncthreads();
  PHASE_MARK(0);
  res_lines<N, KM>(P, O, e0, nb, S);
  __syncthreads();
  PHASE_MARK(1);
  res_writeout<N>(P, e0, nb, S.ACCV);
  PHASE_MARK(2);
}

template <int N, int KM>
__device__ __forceinline__ void res_lines(const ResParams& P, const ResOps<N>& O, int e0, int nb,
                                          const ResSmem<N>& S) {
  using Cfg = ResCfg<N>;
  constexpr int N2 = Cfg::N2, N3 = Cfg::N3, LINES = Cfg::LINES;
  constexpr int AS = Cfg::AS;     // element stride of ACCV
  double* ACCV = S.ACCV;
  const double* PRIM = S.PRIM;
  const double* COF = S.COF;
  const int tid = threadIdx.x;
  const double g = P.gamma, gm1 = g - 1.0;
  // box coordinates of the batch's first element (block-uniform)
  const int ek0 = P.dmm.div(e0), epl = e0 - ek0 * P.m * P.m, ej0 = P.dm.div(epl), ei0 = epl - ej0 * P.m;

  // ---- line phase: one thread owns one 1D line (b, dir, t1, t2) ----
  int lb, ldir, lt1, lt2;
  if constexpr (Cfg::MAPPED) {
    const unsigned code = res_line_map<N>(tid);  // 0xffff: idle lane
    lb = code >> 12;                             // 15 for an idle lane (>= nb)
    ldir = (code >> 8) & 3;
    lt2 = (code >> 4) & 15;
    lt1 = code & 15;
    // opaque from here on: under register pressure the compiler otherwise
    // re-reads the table inside the pair loops to rebuild dir
    asm volatile("" : "+r"(lb), "+r"(ldir), "+r"(lt1), "+r"(lt2));
  } else {
    lb = tid / LINES;
    const int ll = tid - lb * LINES;
    ldir = ll / N2;
    const int lrem = ll - ldir * N2;
    lt1 = lrem % N;
    lt2 = lrem / N;
  }
  if (lb < nb) {
    const int b = lb, e = e0 + b, dir = ldir, t1 = lt1, t2 = lt2;
    const int stride = dir == 0 ? 1 : (dir == 1 ? N : N2);
    const int lbase = dir == 0 ? N * (t1 + N * t2) : (dir == 1 ? t1 + N2 * t2 : t1 + N * t2);
    // disjoint shared-memory regions: lets the next pair's loads pass this pair's stores
    const double* __restrict__ Pd = PRIM + b * 6 * N3;
    const double* __restrict__ Ch = COF + b * 9 * N3;
    double* __restrict__ acc = ACCV + b * AS + (dir == 0 ? 0 : (dir == 1 ? Cfg::DOFF1 : Cfg::DOFF2));
    const double wt = O.wq[t1] * O.wq[t2];
    vol_pairs<N, (KM != 0)>(Pd, Ch, acc, O.q, wt, lbase, stride, dir);
    // S7 hybrid surface pairs + S8 face flux for the two faces this line pierces
#pragma unroll 1
    for (int side = 0; side < (KM == 1 ? 0 : 2); ++side) {
      const int f = 2 * dir + side;
      const double sign = side ? 1.0 : -1.0;
      const int k = t1 + N * t2;
      // Through the hybrid loop only the two traces, the face's half-scaled
      // bundle and its halved cofactor column stay live (the primitives are
      // recomputed after it), which keeps the flux chains out of local memory.
      const double* tr = ResCfg<N>::STR ? S.TRC + (b * 6 + f) * NTR * N2 + k
                                        : P.traces + ((size_t)e * 6 + f) * NTR * N2 + k;
      const double* nt = nullptr;
      {  // neighbour across face f (geometry.hpp:24-29), its face f^1, same node k.
        // The element's box coordinates come from the batch's first element
        // (uniform divisions, once per CTA) by stepping b elements along x:
        // no per-thread division by the run-time m.
        const int mm = P.m;
        int i = ei0 + b, j = ej0, kl = ek0;
        while (i >= mm) {
          i -= mm;
          if (++j >= mm) {
            j = 0;
            ++kl;
          }
        }
        const int step = side ? 1 : -1;
        if (dir == 0) {
          i += step;
          i = i < 0 ? i + mm : (i >= mm ? i - mm : i);
        }
        if (dir == 1) {
          j += step;
          j = j < 0 ? j + mm : (j >= mm ? j - mm : j);
        }
        if (dir == 2) {
          kl += step;
          if (kl < 0 || kl >= P.nz) {
            const double* halo = kl < 0 ? P.halo_lo : P.halo_hi;
            if (halo) nt = halo + (size_t)(i + mm * j) * NTR * N2 + k;
            kl = kl < 0 ? kl + P.nz : kl - P.nz;
          }
        }
        NSFR_DASSERT(i >= 0 && i < mm && j >= 0 && j < mm && kl >= 0 && kl < P.nz && e < P.E);
        if (!nt) nt = P.traces + (((size_t)(i + mm * (j + mm * kl))) * 6 + (f ^ 1)) * NTR * N2 + k;
      }
      // the own and the neighbour's face state (primitives), loaded now: the
      // neighbour's latency hides behind the hybrid loop
      double qn[NTR];
      PrimH pfh;
      double rp_own;
      {
        double qf[NTR];
#pragma unroll
        for (int s = 0; s < NTR; ++s) {
          qf[s] = tr[s * N2];
          qn[s] = nt[s * N2];
        }
        pfh = PrimH{0.5 * qf[0], 0.5 * qf[1], 0.5 * qf[2], 0.5 * qf[3], 0.5 * qf[4], (0.5 * gm1) * qf[5]};
        rp_own = qf[5];
      }
      // own face cofactor column C_f[:,dir] = sum_a bound_flux(side,a) C_a (geometry.cpp:218-226),
      // kept halved (ch = C_f/2; doubling it back is exact): the same fma chain
      // on the stored halves gives exactly half of the chain on C itself
      double ch0 = 0.0, ch1 = 0.0, ch2 = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const int ia = lbase + a * stride;
        const double w = O.bflux[side * N + a];
        ch0 = fma(w, Ch[(0 + dir) * N3 + ia], ch0);
        ch1 = fma(w, Ch[(3 + dir) * N3 + ia], ch1);
        ch2 = fma(w, Ch[(6 + dir) * N3 + ia], ch2);
      }
      double ff[NS] = {0.0, 0.0, 0.0, 0.0, 0.0};
      {
        // running pointers along the line (see vol_pairs)
        const double* __restrict__ pa_p = Pd + lbase;
        const double* __restrict__ ca_p = Ch + dir * N3 + lbase;
        double* __restrict__ aa_p = acc + lbase;
        const double swt = sign * wt;
#pragma unroll 1
        for (int a = 0; a < N; ++a) {
          const PrimH pa = load_prim(pa_p, N3, 0);
          double fl[NS];
          d_flux_h<(KM != 0)>(pa, pfh, ca_p[0] + ch0, ca_p[3 * N3] + ch1, ca_p[6 * N3] + ch2, fl);
          const double c = swt * O.bflux[side * N + a];
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            aa_p[s * N3] = fma(c, fl[s], aa_p[s * N3]);
            ff[s] = fma(-c, fl[s], ff[s]);
          }
          pa_p += stride;
          ca_p += stride;
          aa_p += stride;
        }
      }
      // S8 f*.n with the own unit normal and J^Gamma (geometry.cpp:227-236)
      const double v0 = sign * (2.0 * ch0), v1 = sign * (2.0 * ch1), v2 = sign * (2.0 * ch2);
      const double j2 = v0 * v0 + v1 * v1 + v2 * v2;
      const double ijg = rsqrt(j2), jg = j2 * ijg;
      const double nrm[3] = {v0 * ijg, v1 * ijg, v2 * ijg};
      // the own primitives back from the half-scaled bundle (doubling is exact);
      // rho/p is kept as loaded: rebuilt from the scaled grp it carries a rounding
      // the neighbour's does not, a one-sided bias in Roe's entropy-variable jump
      // that drifts a long run (configs[2] p=4 to t=2: L2 off by 2.6e-10 instead
      // of 3e-11 relative)
      const PrimX pf{2.0 * pfh.hr, 2.0 * pfh.hu, 2.0 * pfh.hv, 2.0 * pfh.hw, 2.0 * pfh.hp, rp_own, 0.0, 0.0};
      const PrimX pn{qn[0], qn[1], qn[2], qn[3], qn[4], qn[5], 0.0, 0.0};
      double fn[NS];
      d_flux_h<(KM != 0)>(pfh, to_half(gm1, pn), nrm[0], nrm[1], nrm[2], fn);
      if (P.roe && KM == 0) {
        double d[NS];
        if (!d_roe_prim(P.gas, pf, pn, nrm, d)) atomicOr(P.err, ERR_ROE);
#pragma unroll
        for (int s = 0; s < NS; ++s) fn[s] -= d[s];
      }
      const double cc = wt * jg;
      if constexpr (fuse_face(N)) {
        // S9's face lift, done here: in the collocated flux basis the lift of this
        // face row onto its own line is l_f(a) = bound_flux(side, a) (chi^T l_f =
        // bound_sol_f, so (M l_f (x) M (x) M) facc = M^3 (l_f (x) facc): the rows K3
        // lifts are vol + sum_f l_f (x) facc_f). The line's nodes belong to this
        // thread in its direction accumulator, so the face row never leaves the
        // SM: no facc array in HBM (12 KB per element and stage at p=4), no face
        // passes in K3.
        double fr[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) fr[s] = fma(cc, fn[s], ff[s]);
        {
          double* __restrict__ aa_p = acc + lbase;
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const double w = O.bflux[side * N + a];
#pragma unroll
            for (int s = 0; s < NS; ++s) aa_p[s * N3 + a * stride] = fma(w, fr[s], aa_p[s * N3 + a * stride]);
          }
        }
      } else {
        // this face's row leaves registers now (facc[e][dir][s][side][k]): nothing
        // of side 0 stays live through side 1
        double* fa = P.facc + ((size_t)e * 3 + dir) * 10 * N2 + k + side * N2;
#pragma unroll
        for (int s = 0; s < NS; ++s) fa[s * 2 * N2] = fma(cc, fn[s], ff[s]);
      }
    }
  }
}

// volume rows: sum of the three direction accumulators
template <int N>
__device__ __forceinline__ void res_writeout(const ResParams& P, int e0, int nb, const double* ACCV) {
  constexpr int N3 = N * N * N, AS = ResCfg<N>::AS, D1 = ResCfg<N>::DOFF1, D2 = ResCfg<N>::DOFF2;
  // compile-time trip count: every thread's shared loads issue before its sums
  constexpr int T = ResCfg<N>::THREADS, ITS = (ResCfg<N>::EPB * 5 * N3 + T - 1) / T;
  const int lim = nb * 5 * N3;
  double v[ITS];
#pragma unroll
  for (int j = 0; j < ITS; ++j) {
    const int it = threadIdx.x + j * T;
    const int b = it / (5 * N3), r = it - b * 5 * N3;
    const double* a0 = ACCV + b * AS;
    v[j] = it < lim ? a0[r] + a0[D1 + r] + a0[D2 + r] : 0.0;
  }
#pragma unroll
  for (int j = 0; j < ITS; ++j) {
    const int it = threadIdx.x + j * T;
    if (it < lim) P.vol[(size_t)e0 * 5 * N3 + it] = v[j];
  }
}

// One batch per CTA (CTAs retire at staggered times, so their staging and
// line phases overlap on each SM — a persistent grid that walks batches in
// lockstep measured slower). Each CTA prefetches into L2 the batch of the CTA
// `ahead` = #resident CTAs later, which the block scheduler starts about when
// this one retires, so that CTA's staging loads hit L2.
template <int N, int KM = 0>
__global__ void __launch_bounds__(ResCfg<N>::THREADS, ResCfg<N>::MINB)
    k_residual(ResParams P, ResOps<N> O, int ahead) {
  extern __shared__ __align__(128) double sm[];
  dbg_kernel_entry(sm);
  constexpr int EPB = ResCfg<N>::EPB;
  const long long pe = P.e_begin + (static_cast<long long>(NSFR_BID) + ahead) * EPB;
  res_batch<N, KM>(P, O, P.e_begin + NSFR_BID * EPB, pe, sm);
}

}  // namespace nsfr_b200
