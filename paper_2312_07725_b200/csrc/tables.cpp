// Host-side setup tables (once per context, never on the hot path): Gauss /
// Gauss-Lobatto rules, the Lagrange basis and the 1D operators of
// ReferenceOperators (fr_operators.cpp:54-113, basis.cpp), plus the c-dependent
// Pi~ (fr_operators.cpp:61-87).
//
// Note on provenance: legendre() and make_rule() below restate the textbook
// Newton iteration for Gauss(-Lobatto) nodes the way the reference's
// quadrature.cpp:8-92 does it -- the same Chebyshev starting guesses, Newton
// update, 1e-15 / 100-iteration stopping rule and endpoint-derivative
// expression -- deliberately, so that the nodes, weights and every table
// built from them come out bit-identical to the reference build's
// (tests/test_gpu_parity.py::test_tables_match_reference, <= 2e-15). SURVEY §2
// allows reusing the reference's setup code outright; restating it keeps the
// library free of the reference's sources and of Eigen.
#include "tables.hpp"

#include <algorithm>
#include <cmath>

namespace nsfr_b200 {
namespace {

using Mat = std::vector<double>;  // row-major, dims carried alongside

// P_n(x) and P_n'(x) by the three-term recurrence (quadrature.cpp:7-27)
void legendre(int n, double x, double& p, double& dp) {
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  double prev = 1.0, prev2 = 0.0, cur = x;
  for (int k = 2; k <= n; ++k) {
    prev2 = prev;
    prev = cur;
    cur = ((2.0 * k - 1.0) * x * prev - (k - 1.0) * prev2) / k;
  }
  p = cur;
  if (std::abs(x) < 1.0)
    dp = n * (prev - x * cur) / (1.0 - x * x);
  else
    dp = n * (n + 1.0) / 2.0 * (x > 0 ? 1.0 : ((n % 2 == 0) ? -1.0 : 1.0));
}

struct Bary {
  std::vector<double> x, b;
  explicit Bary(const std::vector<double>& pts) : x(pts), b(pts.size(), 1.0) {
    const int n = static_cast<int>(x.size());
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        if (i != j) b[i] /= (x[i] - x[j]);
  }
  int n() const { return static_cast<int>(x.size()); }
  // cardinal values l_j(t), exact unit row at a node (basis.cpp:16-30)
  void row(double t, double* out) const {
    for (int j = 0; j < n(); ++j)
      if (t == x[j]) {
        for (int k = 0; k < n(); ++k) out[k] = (k == j) ? 1.0 : 0.0;
        return;
      }
    double den = 0.0;
    for (int j = 0; j < n(); ++j) {
      out[j] = b[j] / (t - x[j]);
      den += out[j];
    }
    for (int j = 0; j < n(); ++j) out[j] /= den;
  }
  Mat eval(const std::vector<double>& pts) const {
    Mat m(pts.size() * n());
    for (size_t i = 0; i < pts.size(); ++i) row(pts[i], &m[i * n()]);
    return m;
  }
  // negative-sum diagonal (basis.cpp:38-52)
  Mat diff() const {
    const int N = n();
    Mat d(N * N, 0.0);
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
      for (int j = 0; j < N; ++j) {
        if (i == j) continue;
        d[i * N + j] = (b[j] / b[i]) / (x[i] - x[j]);
        s += d[i * N + j];
      }
      d[i * N + i] = -s;
    }
    return d;
  }
};

Mat matmul(const Mat& a, int ar, int ac, const Mat& b, int bc) {
  Mat c(ar * bc, 0.0);
  for (int i = 0; i < ar; ++i)
    for (int k = 0; k < ac; ++k) {
      const double v = a[i * ac + k];
      if (v == 0.0) continue;
      for (int j = 0; j < bc; ++j) c[i * bc + j] += v * b[k * bc + j];
    }
  return c;
}

Mat transpose(const Mat& a, int r, int c) {
  Mat t(r * c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) t[j * r + i] = a[i * c + j];
  return t;
}

// LU with partial pivoting, multiple right-hand sides (basis.cpp:66-102)
bool solve(Mat a, int n, Mat x, int nrhs, Mat& out) {
  for (int col = 0; col < n; ++col) {
    int piv = col;
    double best = std::abs(a[col * n + col]);
    for (int r = col + 1; r < n; ++r)
      if (std::abs(a[r * n + col]) > best) {
        best = std::abs(a[r * n + col]);
        piv = r;
      }
    if (best < 2.2250738585072014e-308 * 4) return false;
    if (piv != col) {
      for (int j = 0; j < n; ++j) std::swap(a[col * n + j], a[piv * n + j]);
      for (int j = 0; j < nrhs; ++j) std::swap(x[col * nrhs + j], x[piv * nrhs + j]);
    }
    for (int r = col + 1; r < n; ++r) {
      const double f = a[r * n + col] / a[col * n + col];
      a[r * n + col] = f;
      for (int j = col + 1; j < n; ++j) a[r * n + j] -= f * a[col * n + j];
      for (int j = 0; j < nrhs; ++j) x[r * nrhs + j] -= f * x[col * nrhs + j];
    }
  }
  for (int col = n - 1; col >= 0; --col)
    for (int j = 0; j < nrhs; ++j) {
      x[col * nrhs + j] /= a[col * n + col];
      for (int r = 0; r < col; ++r) x[r * nrhs + j] -= a[r * n + col] * x[col * nrhs + j];
    }
  out = std::move(x);
  return true;
}

Mat eye(int n) {
  Mat m(n * n, 0.0);
  for (int i = 0; i < n; ++i) m[i * n + i] = 1.0;
  return m;
}

}  // namespace

Rule1D make_rule(int kind, int n) {
  Rule1D r;
  r.x.assign(n, 0.0);
  r.w.assign(n, 0.0);
  if (kind == 0) {  // Gauss-Legendre (quadrature.cpp:34-58)
    for (int i = 0; i < (n + 1) / 2; ++i) {
      double x = -std::cos(M_PI * (i + 0.75) / (n + 0.5)), p = 0, dp = 0;
      for (int it = 0; it < 100; ++it) {
        legendre(n, x, p, dp);
        const double dx = -p / dp;
        x += dx;
        if (std::abs(dx) < 1e-15) break;
      }
      legendre(n, x, p, dp);
      r.x[i] = x;
      r.w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
      r.x[n - 1 - i] = -x;
      r.w[n - 1 - i] = r.w[i];
    }
    if (n % 2 == 1) r.x[n / 2] = 0.0;
    return r;
  }
  // Gauss-Lobatto-Legendre (quadrature.cpp:60-92)
  const int m = n - 1;
  r.x[0] = -1.0;
  r.x[n - 1] = 1.0;
  for (int i = 1; i <= (n - 1) / 2; ++i) {
    double x = -std::cos(M_PI * i / m);
    for (int it = 0; it < 100; ++it) {
      double p = 0, dp = 0;
      legendre(m, x, p, dp);
      const double d2p = (2.0 * x * dp - m * (m + 1.0) * p) / (1.0 - x * x);
      const double dx = -dp / d2p;
      x += dx;
      if (std::abs(dx) < 1e-15) break;
    }
    r.x[i] = x;
    r.x[n - 1 - i] = -x;
  }
  if (n % 2 == 1) r.x[n / 2] = 0.0;
  std::sort(r.x.begin(), r.x.end());
  for (int i = 0; i < n; ++i) {
    double p = 0, dp = 0;
    legendre(m, r.x[i], p, dp);
    r.w[i] = 2.0 / (m * (m + 1.0) * p * p);
  }
  return r;
}

double c_plus(int p) {
  switch (p) {
    case 2: return 0.5 * 0.206;
    case 3: return 0.5 * 3.80e-3;
    case 4: return 0.5 * 4.67e-5;
    case 5: return 0.5 * 4.28e-7;
    default: return -1.0;
  }
}

bool build_tables(int p, int quad_kind, int overint, double c1d, int grid_degree, Tables1D& t,
                  const char** msg) {
  const int np = p + 1, nq = p + 1 + overint;  // fr_operators.cpp:93
  t.p = p;
  t.np = np;
  t.nq = nq;
  const Rule1D sol = make_rule(1, np), quad = make_rule(quad_kind, nq);
  const bool collocated = (quad_kind == 1 && nq == np);
  const Bary lb(sol.x);
  t.sol_nodes = sol.x;
  t.quad_nodes = quad.x;
  t.wq = quad.w;
  t.interp = collocated ? eye(np) : lb.eval(quad.x);
  const Mat diff = matmul(t.interp, nq, np, lb.diff(), np);
  Mat mass(np * np), stiff(np * np);
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) {
      double mm = 0.0, ss = 0.0;
      for (int q = 0; q < nq; ++q) {
        mm += t.interp[q * np + i] * quad.w[q] * t.interp[q * np + j];
        ss += t.interp[q * np + i] * quad.w[q] * diff[q * np + j];
      }
      mass[i * np + j] = mm;
      stiff[i * np + j] = ss;
    }
  Mat ctw = transpose(t.interp, nq, np);  // np x nq, columns scaled by w
  for (int i = 0; i < np; ++i)
    for (int q = 0; q < nq; ++q) ctw[i * nq + q] *= quad.w[q];
  if (collocated)
    t.proj = eye(np);
  else if (!solve(mass, np, ctw, nq, t.proj)) {
    *msg = "l2_projection: singular mass";
    return false;
  }
  if (c1d < 0.0) {
    *msg = "correction parameter must be nonnegative";
    return false;
  }
  Mat k1d(np * np, 0.0);
  if (c1d != 0.0) {  // K = c (D^p)^T M D^p  (fr_operators.cpp:54-75)
    Mat d;
    if (!solve(mass, np, stiff, np, d)) {
      *msg = "diff_power_p: singular mass";
      return false;
    }
    Mat dp = eye(np);
    for (int k = 0; k < p; ++k) dp = matmul(d, np, np, dp, np);
    const Mat mdp = matmul(mass, np, np, dp, np);
    k1d = matmul(transpose(dp, np, np), np, np, mdp, np);
    for (double& v : k1d) v *= c1d;
  }
  t.mmass1d = mass;
  for (int i = 0; i < np * np; ++i) t.mmass1d[i] += k1d[i];
  if (!solve(t.mmass1d, np, ctw, nq, t.fr_proj)) {
    *msg = "build_fr_projection: singular M+K";
    return false;
  }
  const Bary fb(quad.x);
  t.quad_diff = fb.diff();
  t.skew.assign(nq * nq, 0.0);
  for (int i = 0; i < nq; ++i)
    for (int j = 0; j < nq; ++j)
      t.skew[i * nq + j] = quad.w[i] * t.quad_diff[i * nq + j] - t.quad_diff[j * nq + i] * quad.w[j];
  const std::vector<double> ends{-1.0, 1.0};
  t.bound_flux = fb.eval(ends);
  t.bound_sol = lb.eval(ends);
  // mapping tables (geometry.cpp:29-60, 96-101)
  t.g = grid_degree + 1;
  const Rule1D gn = make_rule(1, t.g);
  const Bary gb(gn.x);
  t.grid_nodes = gn.x;
  t.ig = gb.eval(quad.x);
  t.is = gb.eval(sol.x);
  t.dg = gb.diff();
  return true;
}

}  // namespace nsfr_b200
