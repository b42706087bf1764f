// Host construction of the 1D operator tables the device kernels consume.
// Product code (no oracle / reference linkage). The algorithms restate:
//   quadrature_rule           proj/src/quadrature.cpp:7-103  (Newton on Legendre)
//   LagrangeBasis             proj/src/basis.cpp:8-52        (barycentric)
//   lagrange_matrices, l2_projection, mat_solve  proj/src/basis.cpp:66-149
//   build_reference_operators proj/src/fr_operators.cpp:48-113 (c, M+K, Pi~, skew)
#pragma once
#include <vector>

namespace nsfr_b200 {

struct Rule1D {
  std::vector<double> x, w;
};

// kind 0 = Gauss-Legendre, 1 = Gauss-Lobatto-Legendre
Rule1D make_rule(int kind, int n);

struct Tables1D {
  int p = 0, np = 0, nq = 0, g = 0;
  std::vector<double> interp;      // nq x np   chi(xi_v)
  std::vector<double> proj;        // np x nq   Pi
  std::vector<double> fr_proj;     // np x nq   Pi~ = (M+K)^-1 chi^T W
  std::vector<double> skew;        // nq x nq   W Dq - Dq^T W
  std::vector<double> bound_flux;  // 2 x nq
  std::vector<double> bound_sol;   // 2 x np
  std::vector<double> wq;          // nq
  std::vector<double> quad_nodes;  // nq
  std::vector<double> sol_nodes;   // np
  std::vector<double> mmass1d;     // np x np
  std::vector<double> quad_diff;   // nq x nq
  // mapping (grid) tables for the device metric build, g = grid_degree + 1
  std::vector<double> grid_nodes;  // g   (LGL)
  std::vector<double> ig;          // nq x g  grid basis at quadrature nodes
  std::vector<double> is;          // np x g  grid basis at solution nodes
  std::vector<double> dg;          // g x g   grid differentiation
};

// Returns false (with msg) on a singular system or a negative c.
// n_q = p + 1 + overint volume quadrature nodes per direction (fr_operators.cpp:89-113)
bool build_tables(int p, int quad_kind, int overint, double c1d, int grid_degree, Tables1D& t,
                  const char** msg);

double c_plus(int p);  // fr_operators.cpp:36-46 (halved von Neumann values); <0 if absent

}  // namespace nsfr_b200
