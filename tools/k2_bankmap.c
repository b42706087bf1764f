// Simulated annealing of K2's line -> lane map and accumulator padding against
// the bank-conflict model of tools/k2_bankmap.py (same cost, C for speed).
//   gcc -O2 -o /tmp/k2_bankmap tools/k2_bankmap.c -lm && /tmp/k2_bankmap N secs
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#define MAXL 512
static int N, N2, N3, LINES, EPB, THREADS, NHW, NL;
static int Lb[MAXL], Ld[MAXL], Lt1[MAXL], Lt2[MAXL];
static int WP[8], WC[8], WA[8];
static unsigned char R[MAXL][8][3];
static int lbase(int d, int t1, int t2) { return d == 0 ? N * (t1 + N * t2) : (d == 1 ? t1 + N2 * t2 : t1 + N * t2); }
static void residues(int esa, int da1, int da2) {
  for (int l = 0; l < NL; ++l)
    for (int a = 0; a < N; ++a) {
      int st = Ld[l] == 0 ? 1 : (Ld[l] == 1 ? N : N2);
      int o = lbase(Ld[l], Lt1[l], Lt2[l]) + a * st;
      int da = Ld[l] == 0 ? 0 : (Ld[l] == 1 ? da1 : da2);
      R[l][a][0] = (6 * N3 * Lb[l] + o) % 16;
      R[l][a][1] = (9 * N3 * Lb[l] + N3 * Ld[l] + o) % 16;
      R[l][a][2] = (esa * Lb[l] + da + o) % 16;
    }
}
static int hw_cost(const int* s) {
  int c = 0;
  for (int a = 0; a < N; ++a) {
    int cnt[3][16];
    memset(cnt, 0, sizeof cnt);
    int m0 = 0, m1 = 0, m2 = 0;
    for (int i = 0; i < 16; ++i) {
      int l = s[i];
      if (l < 0) continue;
      int v;
      v = ++cnt[0][R[l][a][0]]; if (v > m0) m0 = v;
      v = ++cnt[1][R[l][a][1]]; if (v > m1) m1 = v;
      v = ++cnt[2][R[l][a][2]]; if (v > m2) m2 = v;
    }
    c += WP[a] * m0 + WC[a] * m1 + WA[a] * m2;
  }
  return c;
}
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
static unsigned long long rs = 88172645463325252ull;
static unsigned rnd(void) { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return (unsigned)(rs >> 11); }
static int anneal(int* slots, double secs, double T0) {
  int cost[64], cur = 0;
  for (int h = 0; h < NHW; ++h) cur += cost[h] = hw_cost(slots + 16 * h);
  int best = cur;
  static int bs[1024];
  memcpy(bs, slots, sizeof(int) * THREADS);
  double t0 = now(), T = T0;
  for (long it = 0;; ++it) {
    if ((it & 4095) == 0) {
      double f = (now() - t0) / secs;
      if (f >= 1) break;
      T = T0 * (1 - f) * (1 - f) + 0.02;
    }
    int i = rnd() % THREADS, j = rnd() % THREADS, hi = i / 16, hj = j / 16;
    if (hi == hj || (slots[i] < 0 && slots[j] < 0)) continue;
    int t = slots[i]; slots[i] = slots[j]; slots[j] = t;
    int ci = hw_cost(slots + 16 * hi), cj = hw_cost(slots + 16 * hj);
    int d = ci + cj - cost[hi] - cost[hj];
    if (d <= 0 || (rnd() & 0xffffff) / 16777216.0 < exp(-d / T)) {
      cost[hi] = ci; cost[hj] = cj; cur += d;
      if (cur < best) { best = cur; memcpy(bs, slots, sizeof(int) * THREADS); }
    } else { t = slots[i]; slots[i] = slots[j]; slots[j] = t; }
  }
  memcpy(slots, bs, sizeof(int) * THREADS);
  return best;
}
static void natural(int* s) {
  for (int t = 0; t < THREADS; ++t) s[t] = t < NL ? t : -1;
}
int main(int argc, char** argv) {
  N = argc > 1 ? atoi(argv[1]) : 5;
  double secs = argc > 2 ? atof(argv[2]) : 60;
  N2 = N * N; N3 = N2 * N; LINES = 3 * N2;
  EPB = LINES <= 32 ? 6 : (LINES <= 64 ? 4 : (N >= 6 ? 1 : 2));
  THREADS = ((EPB * LINES + 31) / 32) * 32; NHW = THREADS / 16; NL = EPB * LINES;
  int l = 0;
  for (int b = 0; b < EPB; ++b) for (int d = 0; d < 3; ++d) for (int t2 = 0; t2 < N; ++t2) for (int t1 = 0; t1 < N; ++t1) {
    Lb[l] = b; Ld[l] = d; Lt1[l] = t1; Lt2[l] = t2; ++l; }
  int tot = 0;
  for (int a = 0; a < N; ++a) {
    int asb = a, asa = a < N - 1 ? 1 : 0;
    WP[a] = 6 * (asa + asb + 2); WC[a] = 3 * (asa + asb + 4); WA[a] = 10 * (asa + asb + 2);
    tot += WP[a] + WC[a] + WA[a];
  }
  int ideal = ((NL + 15) / 16) * tot;
  static int slots[1024], bestslots[1024];
  residues((15 * N3) % 16, (5 * N3) % 16, (10 * N3) % 16);
  natural(slots);
  int nat = 0;
  for (int h = 0; h < NHW; ++h) nat += hw_cost(slots + 16 * h);
  printf("N=%d EPB=%d threads=%d: ideal %d natural %d (%.3fx)\n", N, EPB, THREADS, ideal, nat, (double)nat / ideal);
  // coarse pass over all paddings, then long anneals of the best few
  typedef struct { int c, e, d1, d2; } Cand;
  static Cand cands[4096];
  int nc = 0;
  double coarse = secs * 0.4 / 4096;
  for (int e = 0; e < 16; ++e) for (int d1 = 0; d1 < 16; ++d1) for (int d2 = 0; d2 < 16; ++d2) {
    if (EPB == 1 && e) continue;
    residues(e, d1, d2); natural(slots);
    cands[nc++] = (Cand){anneal(slots, EPB == 1 ? coarse * 16 : coarse, 8.0), e, d1, d2};
  }
  for (int i = 0; i < nc; ++i) for (int j = i + 1; j < nc; ++j) if (cands[j].c < cands[i].c) { Cand t = cands[i]; cands[i] = cands[j]; cands[j] = t; }
  int best = 1 << 30, be = 0, bd1 = 0, bd2 = 0;
  int top = nc < 12 ? nc : 12;
  for (int k = 0; k < top; ++k) {
    residues(cands[k].e, cands[k].d1, cands[k].d2); natural(slots);
    int c = anneal(slots, secs * 0.6 / top, 20.0);
    printf("  pad (%d,%d,%d): coarse %d -> %d (%.3fx)\n", cands[k].e, cands[k].d1, cands[k].d2, cands[k].c, c, (double)c / ideal);
    fflush(stdout);
    if (c < best) { best = c; be = cands[k].e; bd1 = cands[k].d1; bd2 = cands[k].d2; memcpy(bestslots, slots, sizeof(int) * THREADS); }
  }
  printf("best %d (%.3fx) pad ES_A=%d DA1=%d DA2=%d (mod 16)\nmap:", best, (double)best / ideal, be, bd1, bd2);
  for (int t = 0; t < THREADS; ++t) {
    int s = bestslots[t];
    if (t % 16 == 0) printf("\n   ");
    if (s < 0) printf(" 0xffff,"); else printf(" 0x%04x,", Lb[s] << 12 | Ld[s] << 8 | Lt2[s] << 4 | Lt1[s]);
  }
  printf("\n");
  return 0;
}
