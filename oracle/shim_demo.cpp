// TEST INFRASTRUCTURE: the drop-in boundary exercised from the reference's
// side. Builds operators, warped mapping and conservative-curl metrics with
// the reference's OWN setup code (fr_operators.cpp, geometry.cpp), hands them
// to libnsfr_b200.so through the C++ shim of INTEGRATION.md
// (integration/gpu_solver.hpp), and checks the GPU's assemble_rhs and
// rk4_step(field, dt) / adaptive_dt loop against the reference build under the
// residual glue (oracle/ref_driver.cpp, same process). Prints one JSON line;
// exit code 0 when every gate holds. Built by oracle/Makefile (needs the
// reference headers), run by tests/test_gpu_shim.py on the GPU box.
//   shim_demo [p] [m] [c_plus 0|1]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "gpu_solver.hpp"
#define NSFR_CPU_PREFIX nsfr_ref_
#include "nsfr_oracle.h"

namespace {

double norm_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::fmax(num, std::fabs(a[i] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return num / den;
}

}  // namespace

int main(int argc, char** argv) {
  const int p = argc > 1 ? std::atoi(argv[1]) : 3;
  const int m = argc > 2 ? std::atoi(argv[2]) : 4;
  const bool cplus = argc > 3 ? std::atoi(argv[3]) != 0 : true;
  const double beta = 0.05, xl = 0.0, xr = 10.0, gamma = 1.4, cfl = 0.1;
  try {
    // reference setup objects
    const double c1d = cplus ? nsfr::correction_c_plus(p) : 0.0;
    const nsfr::ReferenceOperators ops = nsfr::build_reference_operators(p, nsfr::QuadKind::GaussLegendre, 0, c1d);
    const nsfr::CurvilinearMapping map = nsfr::warp_grid_3d(m, beta, xl, xr, p + 1);
    const nsfr::MetricData md = nsfr::build_metrics_conservative_curl(map, ops);
    nsfr::GpuSolver gpu(ops, map, md, gamma, /*roe=*/true);

    // the reference build under the residual glue, same configuration
    nsfr_cfg cfg{p, 0, 0, c1d, m, 0, m, xl, xr, beta, 0.0, p + 1, gamma, 1, 8, 0};
    char err[256] = {0};
    void* ref = nsfr_ref_create(&cfg, err, sizeof err);
    if (!ref) {
      std::printf("{\"ok\": false, \"error\": \"%s\"}\n", err);
      return 2;
    }
    const size_t n = static_cast<size_t>(m) * m * m * 5 * (p + 1) * (p + 1) * (p + 1);
    std::vector<double> u(n), r_gpu(n), r_ref(n), r_pert(n);
    nsfr_ref_initial_state(ref, NSFR_CASE_VORTEX, u.data());
    std::mt19937_64 rng(20231207);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (auto& x : u) x *= 1.0 + 1e-3 * uni(rng);

    // assemble_rhs through the shim vs the reference build; the parity floor is
    // the reference's own RHS change under a 1-ulp perturbation of its input
    gpu.assemble_rhs(u, r_gpu);
    nsfr_ref_rhs(ref, u.data(), nullptr, nullptr, r_ref.data(), nullptr);
    std::vector<double> up(u);
    for (auto& x : up) x *= 1.0 + 0x1p-52 * (uni(rng) < 0 ? -1.0 : 1.0);
    nsfr_ref_rhs(ref, up.data(), nullptr, nullptr, r_pert.data(), nullptr);
    const double rhs_err = norm_rel(r_gpu, r_ref), floor = norm_rel(r_pert, r_ref);
    const double gate = std::fmin(1e-8, std::fmax(1e-12, 4.0 * floor));

    // the reference loop dt = adaptive_dt(u); u = rk4_step(u, dt) through the
    // shim, next to the reference build stepping with the same dt sequence
    std::vector<double> ug(u), ur(u);
    double dt = gpu.adaptive_dt(ug, cfl);
    double lam = 0.0;
    nsfr_ref_max_wavespeed(ref, ur.data(), &lam);
    const double dx = (xr - xl) / (m * (p + 1));
    const double dt_ref0 = cfl * dx / lam;
    for (int s = 0; s < 3; ++s) {
      nsfr_ref_rk4_step(ref, ur.data(), dt);
      dt = gpu.rk4_step(ug, dt, cfl);
    }
    std::vector<double> dg(n), dr(n);
    for (size_t i = 0; i < n; ++i) {
      dg[i] = ug[i] - u[i];
      dr[i] = ur[i] - u[i];
    }
    const double step_err = norm_rel(dg, dr);
    const double dt_err = std::fabs(gpu.adaptive_dt(u, cfl) - dt_ref0) / dt_ref0;
    const bool ok = rhs_err <= gate && step_err <= 1e-10 && dt_err <= 1e-14;
    std::printf(
        "{\"ok\": %s, \"p\": %d, \"m\": %d, \"c1d\": %.6g, \"rhs_err\": %.3e, \"floor\": %.3e, "
        "\"gate\": %.3e, \"step_increment_err\": %.3e, \"adaptive_dt_err\": %.3e}\n",
        ok ? "true" : "false", p, m, c1d, rhs_err, floor, gate, step_err, dt_err);
    nsfr_ref_destroy(ref);
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 3;
  }
}
