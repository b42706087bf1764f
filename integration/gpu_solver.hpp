// Reference-side shim: binds the reference's missing solver
// surface (proj/CMakeLists.txt:26 src/solver.cpp) to libnsfr_b200.so.
#pragma once
#include <array>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>
#include "nsfr/fr_operators.hpp"   // ReferenceOperators
#include "nsfr/geometry.hpp"       // MetricData, CurvilinearMapping
#include "nsfr_gpu.h"               // libnsfr_b200.so

namespace nsfr {

// Replaces the missing src/solver.cpp surface with the B200 path.
class GpuSolver {
 public:
  GpuSolver(const ReferenceOperators& ops, const CurvilinearMapping& map, const MetricData& md,
            double gamma, bool roe, int device = 0) {
    const int np = ops.np(), nq = ops.nq(), nv = nq * nq * nq;
    if (np != nq) throw DimensionError("GpuSolver: overintegration not supported");
    // ElementMetrics (geometry.hpp:66-80) -> flat [e][q], [e][q][9]
    jac_.reserve(md.elem.size() * nv);
    cof_.reserve(md.elem.size() * nv * 9);
    for (const auto& em : md.elem) {
      jac_.insert(jac_.end(), em.jac_vol.begin(), em.jac_vol.end());
      cof_.insert(cof_.end(), em.cof_vol.begin(), em.cof_vol.end());
    }
    nsfr_gpu_tables t{ops.basis.interp.a.data(), ops.proj.a.data(), ops.fr_proj.a.data(),
                      ops.skew.a.data(), ops.bound_flux.a.data(), ops.bound_sol.a.data(),
                      ops.wq.data()};
    nsfr_gpu_setup s{};
    s.p = ops.basis.p; s.quad_kind = ops.basis.eval_rule.kind == QuadKind::GaussLegendre ? 0 : 1;
    s.c1d = ops.c1d; s.gamma = gamma; s.roe = roe ? 1 : 0;
    s.m = map.mesh.m; s.k0 = 0; s.k1 = map.mesh.m;
    s.x_left = map.mesh.x_left; s.x_right = map.mesh.x_right;
    s.grid_degree = map.grid_degree; s.device = device; s.entropy_diag = 1;
    s.tables = &t; s.jac_vol = jac_.data(); s.cof_vol = cof_.data();
    s.nranks = 1;
    check(nsfr_gpu_create(&s, &ctx_));
    dx_ = (s.x_right - s.x_left) / (s.m * (s.p + 1));
  }
  ~GpuSolver() { nsfr_gpu_destroy(ctx_); }

  // assemble_rhs: dU/dt of `u` ([e][5][np^3]); returns -sum v_hat . R
  double assemble_rhs(std::span<const double> u, std::span<double> dudt) {
    check(nsfr_gpu_set_state(ctx_, u.data()));
    double ds = 0.0;
    check(nsfr_gpu_rhs(ctx_, dudt.data(), &ds));
    return ds;
  }
  // rk4_step(field, dt) on the caller's host field: upload,
  // step and download pipelined on the device. Returns adaptive_dt(u, cfl)
  // of the new field, so the reference loop
  //   dt = adaptive_dt(u, cfl); while (...) dt = rk4_step(u, dt, cfl, t_final);
  // runs without a global reduction inside the step. dt <= 0: take
  // adaptive_dt of the incoming field first.
  double rk4_step(std::span<double> u, double dt, double cfl, double t_final = 0.0) {
    double used = 0.0, next = 0.0;
    check(nsfr_gpu_rk4_step_host(ctx_, u.data(), u.data(), dt, cfl, t_final, &used, &next));
    return next;
  }
  // adaptive_dt(field, cfl) of a host field
  double adaptive_dt(std::span<const double> u, double cfl) {
    double lam = 0.0;
    check(nsfr_gpu_set_state(ctx_, u.data()));
    check(nsfr_gpu_max_wavespeed(ctx_, &lam));
    return lam > 0.0 ? cfl * dx_ / lam : cfl * dx_;
  }
  std::array<double, 2> l2_error(int case_kind) {
    std::array<double, 2> e{};
    check(nsfr_gpu_l2_error(ctx_, case_kind, e.data()));
    return e;
  }

 private:
  void check(int rc) {
    if (rc == NSFR_OK) return;
    const std::string what = ctx_ ? nsfr_gpu_last_error(ctx_) : nsfr_gpu_create_error();
    double t = 0.0;
    switch (rc) {
      case NSFR_E_DIM: throw DimensionError(what);
      case NSFR_E_MESH: throw InvalidMeshError(what);
      case NSFR_E_INADMISSIBLE: nsfr_gpu_get_time(ctx_, &t); throw StepFailureError(what, t);
      case NSFR_E_CONFIG: throw ConfigError(what);
      default: throw std::runtime_error(what);
    }
  }
  nsfr_gpu_ctx* ctx_ = nullptr;
  double dx_ = 0.0;  // l/(M(p+1))
  std::vector<double> jac_, cof_;
};

}  // namespace nsfr
