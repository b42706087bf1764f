// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Drives the reference's OWN compiled primitives (/root/reference/proj, built
// from its sources by oracle/Makefile into oracle/_ref/libnsfr_ref.so) through
// the residual glue that the reference specifies but does not ship
// (CMakeLists.txt:26 src/solver.cpp is absent). The glue is the same one the
// C oracle (oracle/nsfr_oracle.c) restates; conventions D1-D10 of SURVEY.md
// §8(c). Exports the nsfr_ref_* flavour of oracle/nsfr_oracle.h.
//
// Everything on the path is a reference call:
//   build_reference_operators      fr_operators.cpp:89-113
//   warp_grid_3d                   geometry.cpp:62-73
//   build_metrics_conservative_curl geometry.cpp:86-266
//   apply_tensor_product           sumfac.cpp:57-69
//   entropy_variables / entropy_to_conservative  euler.cpp:46-71
//   hadamard_sumfac_volume         sumfac.hpp:48-94 (called with 0.5*skew, D2)
//   hadamard_sumfac_surface        sumfac.hpp:110-157
//   two_point_flux(ChandrashekarRanochaFix)  euler.cpp:194-214
//   roe_dissipation                euler.cpp:229-301
//   weight_adjusted_inverse_apply  fr_operators.cpp:280-309
//   isentropic_vortex_exact / tgv_initial    cases.cpp:7-56
//   parallel_for                   defs.hpp:36-50
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "nsfr/cases.hpp"
#include "nsfr/euler.hpp"
#include "nsfr/fr_operators.hpp"
#include "nsfr/geometry.hpp"
#include "nsfr/sumfac.hpp"

#define NSFR_CPU_PREFIX nsfr_ref_
#include "nsfr_oracle.h"

using namespace nsfr;

namespace {

struct RefCtx {
  nsfr_cfg cfg{};
  EulerGas gas;
  ReferenceOperators ops;
  Operator1D half_skew, interp_t, bs_row[2], bs_col[2];
  CurvilinearMapping mapping;
  MetricData md;
  int md_base = 0;  // md.elem[i] holds global element md_base + i
  int np = 0, nq = 0, nv = 0, nsol = 0, nf = 0, ne = 0;
  std::vector<double> ut_vol, ut_f, vhat;
  std::string msg;
};

int global_elem(const RefCtx& c, int e) { return e + c.cfg.m * c.cfg.m * c.cfg.k0; }
int md_index(const RefCtx& c, int e) { return global_elem(c, e) - c.md_base; }

// Metrics of the slab's elements only. build_metrics_conservative_curl
// (geometry.cpp:86-266) is element-local: it reads mapping.point(e, .) and the
// shared 1D operators, nothing of the neighbours or of the mesh. So it runs on
// chunks of the slab in parallel (parallel_for, defs.hpp:36-50), each chunk a
// sub-mapping whose stand-in mesh has >= chunk elements (padded by repeating
// the chunk's last element); element i of a chunk gets exactly the metrics the
// whole-box build gives it. A 128x128x16 slab then needs 1/8 of the whole
// box's metric memory and the build runs on every core.
MetricData build_metrics_slab(const CurvilinearMapping& full, const ReferenceOperators& ops, int e0,
                              int ne, int workers) {
  MetricData md;
  md.elem.resize(ne);
  const int nchunks = std::max(1, std::min(ne, 4 * std::max(1, workers)));
  const size_t per = static_cast<size_t>(full.nodes_per_element()) * 3;
  std::vector<MetricData> heads(1);
  parallel_for(nchunks, workers, [&](int ch) {
    const int a = static_cast<int>(static_cast<long long>(ne) * ch / nchunks);
    const int b = static_cast<int>(static_cast<long long>(ne) * (ch + 1) / nchunks);
    const int cnt = b - a;
    if (cnt <= 0) return;
    int mf = 1;
    while (mf * mf * mf < cnt) ++mf;
    CurvilinearMapping sub;
    sub.mesh = StructuredMesh{mf, full.mesh.x_left, full.mesh.x_right};
    sub.grid_degree = full.grid_degree;
    sub.grid_basis = full.grid_basis;
    sub.grid_ext = full.grid_ext;
    sub.control_points.resize(static_cast<size_t>(mf) * mf * mf * per);
    for (int i = 0; i < mf * mf * mf; ++i) {
      const size_t src = static_cast<size_t>(e0 + a + std::min(i, cnt - 1)) * per;
      std::copy(full.control_points.begin() + src, full.control_points.begin() + src + per,
                sub.control_points.begin() + static_cast<size_t>(i) * per);
    }
    MetricData part = build_metrics_conservative_curl(sub, ops);
    for (int i = 0; i < cnt; ++i) md.elem[a + i] = std::move(part.elem[i]);
    if (ch == 0) {
      heads[0].vol_ext = part.vol_ext;
      heads[0].sol_ext = part.sol_ext;
    }
  });
  md.vol_ext = heads[0].vol_ext;
  md.sol_ext = heads[0].sol_ext;
  return md;
}

void case_state(const RefCtx& c, int kind, const double* x, double t, double* u) {
  State st;
  if (kind == NSFR_CASE_TGV)
    st = tgv_initial(c.gas, x[0], x[1], x[2]);
  else if (kind == NSFR_CASE_VORTEX)
    st = isentropic_vortex_exact(c.gas, x[0], x[1], x[2], t, 0.4);
  else
    st = make_case(CaseKind::FreeStream, c.gas).initial({x[0], x[1], x[2]});
  for (int s = 0; s < kStates; ++s) u[s] = st[s];
}

State load(const double* base, int stride, int idx) {
  State s;
  for (int k = 0; k < kStates; ++k) s[k] = base[k * stride + idx];
  return s;
}

// S1-S5 with reference primitives
void project_elem(RefCtx& c, const double* u, int e) {
  const auto& o = c.ops;
  const Extents me{c.np, c.np, c.np}, qe{c.nq, c.nq, c.nq};
  std::vector<double> work(4096), uq(kStates * c.nv), vq(kStates * c.nv), vt(kStates * c.nv);
  const double* ue = u + static_cast<size_t>(e) * kStates * c.nsol;
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                         std::span<const double>(ue + s * c.nsol, c.nsol), me,
                         std::span<double>(&uq[s * c.nv], c.nv), work);
  for (int q = 0; q < c.nv; ++q) {
    State v = entropy_variables(c.gas, load(uq.data(), c.nv, q));
    for (int s = 0; s < kStates; ++s) vq[s * c.nv + q] = v[s];
  }
  double* vh = &c.vhat[static_cast<size_t>(e) * kStates * c.nsol];
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(o.proj, o.proj, o.proj, std::span<const double>(&vq[s * c.nv], c.nv), qe,
                         std::span<double>(vh + s * c.nsol, c.nsol), work);
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                         std::span<const double>(vh + s * c.nsol, c.nsol), me,
                         std::span<double>(&vt[s * c.nv], c.nv), work);
  double* utv = &c.ut_vol[static_cast<size_t>(e) * kStates * c.nv];
  for (int q = 0; q < c.nv; ++q) {
    State uu = entropy_to_conservative(c.gas, load(vt.data(), c.nv, q));
    for (int s = 0; s < kStates; ++s) utv[s * c.nv + q] = uu[s];
  }
  std::vector<double> vf(kStates * c.nf);
  for (int dir = 0; dir < 3; ++dir)
    for (int side = 0; side < 2; ++side) {
      const int f = 2 * dir + side;
      const Operator1D& a0 = dir == 0 ? c.bs_row[side] : o.basis.interp;
      const Operator1D& a1 = dir == 1 ? c.bs_row[side] : o.basis.interp;
      const Operator1D& a2 = dir == 2 ? c.bs_row[side] : o.basis.interp;
      for (int s = 0; s < kStates; ++s)
        apply_tensor_product(a0, a1, a2, std::span<const double>(vh + s * c.nsol, c.nsol), me,
                             std::span<double>(&vf[s * c.nf], c.nf), work);
      double* utf = &c.ut_f[(static_cast<size_t>(e) * 6 + f) * kStates * c.nf];
      for (int k = 0; k < c.nf; ++k) {
        State uu = entropy_to_conservative(c.gas, load(vf.data(), c.nf, k));
        for (int s = 0; s < kStates; ++s) utf[s * c.nf + k] = uu[s];
      }
    }
}

// conservative DG: chi u_hat at volume and face nodes (no entropy projection)
void dg_states_elem(RefCtx& c, const double* u, int e) {
  const auto& o = c.ops;
  const Extents me{c.np, c.np, c.np};
  std::vector<double> work(8192);
  const double* ue = u + static_cast<size_t>(e) * kStates * c.nsol;
  double* utv = &c.ut_vol[static_cast<size_t>(e) * kStates * c.nv];
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                         std::span<const double>(ue + s * c.nsol, c.nsol), me,
                         std::span<double>(utv + s * c.nv, c.nv), work);
  for (int q = 0; q < c.nv; ++q)
    if (!admissible(c.gas, load(utv, c.nv, q))) throw InadmissibleStateError("dg: volume state");
  for (int dir = 0; dir < 3; ++dir)
    for (int side = 0; side < 2; ++side) {
      const int f = 2 * dir + side;
      const Operator1D& a0 = dir == 0 ? c.bs_row[side] : o.basis.interp;
      const Operator1D& a1 = dir == 1 ? c.bs_row[side] : o.basis.interp;
      const Operator1D& a2 = dir == 2 ? c.bs_row[side] : o.basis.interp;
      double* utf = &c.ut_f[(static_cast<size_t>(e) * 6 + f) * kStates * c.nf];
      for (int s = 0; s < kStates; ++s)
        apply_tensor_product(a0, a1, a2, std::span<const double>(ue + s * c.nsol, c.nsol), me,
                             std::span<double>(utf + s * c.nf, c.nf), work);
      for (int k = 0; k < c.nf; ++k)
        if (!admissible(c.gas, load(utf, c.nf, k))) throw InadmissibleStateError("dg: face state");
    }
}

int project_all(RefCtx& c, const double* u) {
  std::atomic<int> bad{-1};
  std::string what;
  parallel_for(c.ne, c.cfg.workers, [&](int e) {
    try {
      if (c.cfg.scheme == NSFR_SCHEME_DG)
        dg_states_elem(c, u, e);
      else
        project_elem(c, u, e);
    } catch (const std::exception& ex) {
      bad = e;
    }
  });
  if (bad >= 0) {
    c.msg = "entropy projection: inadmissible state in element " + std::to_string(bad.load());
    return NSFR_E_INADMISSIBLE;
  }
  return NSFR_OK;
}

const double* nbr_trace(const RefCtx& c, int e, int f, const double* halo_lo,
                        const double* halo_hi) {
  const int m = c.cfg.m, nz = c.cfg.k1 - c.cfg.k0, blk = kStates * c.nf;
  const StructuredMesh& mesh = c.mapping.mesh;
  const int eg = global_elem(c, e);
  const int en = mesh.neighbor(eg, f);  // geometry.hpp:24-29
  const int kl = e / (m * m);
  const bool whole = (c.cfg.k0 == 0 && c.cfg.k1 == m);
  if (!whole && f / 2 == 2) {
    if (f == 4 && kl == 0) return halo_lo + static_cast<size_t>(e % (m * m)) * blk;
    if (f == 5 && kl == nz - 1) return halo_hi + static_cast<size_t>(e % (m * m)) * blk;
  }
  const int el = en - m * m * c.cfg.k0;
  return &c.ut_f[(static_cast<size_t>(el) * 6 + (f ^ 1)) * blk];
}

// S6-S10
// F~ - P~ (kinetic-energy diagnostics)
void strip_pressure(const RefCtx& c, const State& ui, const State& uj, Flux& F) {
  const double pbar = 0.5 * (pressure(c.gas, ui) + pressure(c.gas, uj));
  for (int k = 0; k < 3; ++k) F[k][1 + k] -= pbar;
}

void rhs_elem(RefCtx& c, int e, const double* halo_lo, const double* halo_hi, double* dudt,
              double* dS, const double* uke = nullptr, double* keS = nullptr) {
  const auto& o = c.ops;
  const int nv = c.nv, nf = c.nf, nsol = c.nsol, nq = c.nq;
  const Extents qe{nq, nq, nq}, me{c.np, c.np, c.np};
  const ElementMetrics& em = c.md.elem[md_index(c, e)];
  const double* utv = &c.ut_vol[static_cast<size_t>(e) * kStates * nv];
  const double* utf_all = &c.ut_f[static_cast<size_t>(e) * 6 * kStates * nf];
  std::vector<double> vol(kStates * nv, 0.0);
  std::array<std::vector<double>, 6> facc;
  for (auto& fa : facc) fa.assign(kStates * nf, 0.0);
  const std::array<const Operator1D*, 3> hs{&c.half_skew, &c.half_skew, &c.half_skew};
  const std::span<const double> w(o.wq);
  const std::array<std::span<const double>, 3> w3{w, w, w};
  auto vol_provider = [&](int i, int j, int dir, double* out) {
    Flux F = two_point_flux(c.gas, TwoPointFluxKind::ChandrashekarRanochaFix,
                            load(utv, nv, i), load(utv, nv, j));
    if (keS) strip_pressure(c, load(utv, nv, i), load(utv, nv, j), F);
    const double* Ci = em.cof_at(i);
    const double* Cj = em.cof_at(j);
    const double cm0 = 0.5 * (Ci[0 + dir] + Cj[0 + dir]);
    const double cm1 = 0.5 * (Ci[3 + dir] + Cj[3 + dir]);
    const double cm2 = 0.5 * (Ci[6 + dir] + Cj[6 + dir]);
    for (int s = 0; s < kStates; ++s) out[s] = F[0][s] * cm0 + F[1][s] * cm1 + F[2][s] * cm2;
  };
  hadamard_sumfac_volume(hs, w3, qe, kStates, vol_provider, vol, nullptr);
  const std::array<const Operator1D*, 3> bf{&o.bound_flux, &o.bound_flux, &o.bound_flux};
  auto surf_provider = [&](int i, int fid, int k, int dir, double* out) {
    const double* utf = utf_all + static_cast<size_t>(fid) * kStates * nf;
    Flux F = two_point_flux(c.gas, TwoPointFluxKind::ChandrashekarRanochaFix,
                            load(utv, nv, i), load(utf, nf, k));
    if (keS) strip_pressure(c, load(utv, nv, i), load(utf, nf, k), F);
    const double* Ci = em.cof_at(i);
    const double* Cf = em.cof_face_at(fid, k);
    const double cm0 = 0.5 * (Ci[0 + dir] + Cf[0 + dir]);
    const double cm1 = 0.5 * (Ci[3 + dir] + Cf[3 + dir]);
    const double cm2 = 0.5 * (Ci[6 + dir] + Cf[6 + dir]);
    for (int s = 0; s < kStates; ++s) out[s] = F[0][s] * cm0 + F[1][s] * cm1 + F[2][s] * cm2;
  };
  auto sink = [&](int fid, int s, int k) -> double& { return facc[fid][s * nf + k]; };
  hadamard_sumfac_surface(bf, w3, qe, kStates, surf_provider, vol, sink, nullptr);
  // S8 surface numerical flux (D3)
  for (int fid = 0; fid < 6; ++fid) {
    const double* utf = utf_all + static_cast<size_t>(fid) * kStates * nf;
    const double* utn = nbr_trace(c, e, fid, halo_lo, halo_hi);
    const FaceNormals fnrm = physical_normals(c.md, md_index(c, e), fid);
    for (int t2 = 0; t2 < nq; ++t2)
      for (int t1 = 0; t1 < nq; ++t1) {
        const int k = t1 + nq * t2;
        const State ul = load(utf, nf, k), ur = load(utn, nf, k);
        const std::array<double, 3> nr{fnrm.unit_normals[3 * k], fnrm.unit_normals[3 * k + 1],
                                       fnrm.unit_normals[3 * k + 2]};
        Flux F = two_point_flux(c.gas, TwoPointFluxKind::ChandrashekarRanochaFix, ul, ur);
        if (keS) strip_pressure(c, ul, ur, F);
        double fn[kStates];
        for (int s = 0; s < kStates; ++s) fn[s] = F[0][s] * nr[0] + F[1][s] * nr[1] + F[2][s] * nr[2];
        if (c.cfg.roe && !keS) {
          const State d = roe_dissipation(c.gas, ul, ur, nr);
          for (int s = 0; s < kStates; ++s) fn[s] -= d[s];
        }
        const double cc = o.wq[t1] * o.wq[t2] * fnrm.surface_jacobian[k];
        for (int s = 0; s < kStates; ++s) facc[fid][s * nf + k] += cc * fn[s];
      }
  }
  // S9 lifting
  std::vector<double> work(4096), R(kStates * nsol), tmp(nsol);
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(c.interp_t, c.interp_t, c.interp_t,
                         std::span<const double>(&vol[s * nv], nv), qe,
                         std::span<double>(&R[s * nsol], nsol), work);
  for (int dir = 0; dir < 3; ++dir)
    for (int side = 0; side < 2; ++side) {
      const int fid = 2 * dir + side;
      const Operator1D& a0 = dir == 0 ? c.bs_col[side] : c.interp_t;
      const Operator1D& a1 = dir == 1 ? c.bs_col[side] : c.interp_t;
      const Operator1D& a2 = dir == 2 ? c.bs_col[side] : c.interp_t;
      const Extents fe{dir == 0 ? 1 : nq, dir == 1 ? 1 : nq, dir == 2 ? 1 : nq};
      for (int s = 0; s < kStates; ++s) {
        apply_tensor_product(a0, a1, a2, std::span<const double>(&facc[fid][s * nf], nf), fe, tmp,
                             work);
        for (int i = 0; i < nsol; ++i) R[s * nsol + i] += tmp[i];
      }
    }
  if (keS) {  // -sum v_hat_KE . R, v_hat_KE = Pi^3 kinetic_energy_variables(chi^3 u_hat)
    std::vector<double> uq(kStates * nv), vk(4 * nv), vkh(nsol);
    for (int s = 0; s < kStates; ++s)
      apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                           std::span<const double>(uke + (static_cast<size_t>(e) * kStates + s) * nsol, nsol),
                           me, std::span<double>(&uq[s * nv], nv), work);
    for (int q = 0; q < nv; ++q) {
      const State v = kinetic_energy_variables(load(uq.data(), nv, q));
      for (int s = 0; s < 4; ++s) vk[s * nv + q] = v[s];
    }
    double acc = 0.0;
    for (int s = 0; s < 4; ++s) {
      apply_tensor_product(o.proj, o.proj, o.proj, std::span<const double>(&vk[s * nv], nv), qe, vkh, work);
      for (int i = 0; i < nsol; ++i) acc += vkh[i] * R[s * nsol + i];
    }
    keS[e] = -acc;
    return;
  }
  if (dS) {
    const double* vh = &c.vhat[static_cast<size_t>(e) * kStates * nsol];
    double acc = 0.0;
    for (int s = 0; s < kStates; ++s)
      for (int i = 0; i < nsol; ++i) acc += vh[s * nsol + i] * R[s * nsol + i];
    dS[e] = -acc;
  }
  // S10 weight-adjusted inverse
  std::vector<double> wa(wa_work_size(o, 3));
  double* out = dudt + static_cast<size_t>(e) * kStates * nsol;
  for (int s = 0; s < kStates; ++s) {
    weight_adjusted_inverse_apply(o, 3, em.jac_vol, std::span<const double>(&R[s * nsol], nsol),
                                  std::span<double>(out + s * nsol, nsol), wa);
    for (int i = 0; i < nsol; ++i) out[s * nsol + i] = -out[s * nsol + i];
  }
  (void)me;
}

// conservative strong-form DG with the reference primitives
void dg_rhs_elem(RefCtx& c, int e, const double* halo_lo, const double* halo_hi, double* dudt) {
  const auto& o = c.ops;
  const int nv = c.nv, nf = c.nf, nsol = c.nsol, nq = c.nq;
  const Extents qe{nq, nq, nq};
  const ElementMetrics& em = c.md.elem[md_index(c, e)];
  const double* utv = &c.ut_vol[static_cast<size_t>(e) * kStates * nv];
  const double* utf_all = &c.ut_f[static_cast<size_t>(e) * 6 * kStates * nf];
  std::vector<double> fr(3 * kStates * nv), vol(kStates * nv), tmpv(nv);
  for (int q = 0; q < nv; ++q) {
    const Flux F = physical_flux(c.gas, load(utv, nv, q));  // euler.cpp:30-40
    const double* Cq = em.cof_at(q);
    for (int dir = 0; dir < 3; ++dir)
      for (int s = 0; s < kStates; ++s)
        fr[(dir * kStates + s) * nv + q] =
            F[0][s] * Cq[0 + dir] + F[1][s] * Cq[3 + dir] + F[2][s] * Cq[6 + dir];
  }
  for (int s = 0; s < kStates; ++s) {
    std::span<double> vs(&vol[s * nv], nv);
    apply_operator_dir(o.quad_diff, 0, std::span<const double>(&fr[(0 * kStates + s) * nv], nv), qe, vs);
    for (int dir = 1; dir < 3; ++dir) {
      apply_operator_dir(o.quad_diff, dir, std::span<const double>(&fr[(dir * kStates + s) * nv], nv), qe,
                         tmpv);
      for (int q = 0; q < nv; ++q) vs[q] += tmpv[q];
    }
  }
  for (int k = 0; k < nq; ++k)
    for (int j = 0; j < nq; ++j)
      for (int i = 0; i < nq; ++i) {
        const int q = i + nq * (j + nq * k);
        double w = o.wq[i];
        w *= o.wq[j];
        w *= o.wq[k];
        for (int s = 0; s < kStates; ++s) vol[s * nv + q] *= w;
      }
  std::array<std::vector<double>, 6> facc;
  for (int dir = 0; dir < 3; ++dir) {
    const int stride = (dir == 0) ? 1 : (dir == 1 ? nq : nq * nq);
    for (int side = 0; side < 2; ++side) {
      const int fid = 2 * dir + side;
      const double sign = side ? 1.0 : -1.0;
      facc[fid].assign(kStates * nf, 0.0);
      const double* utf = utf_all + static_cast<size_t>(fid) * kStates * nf;
      const double* utn = nbr_trace(c, e, fid, halo_lo, halo_hi);
      const FaceNormals fnrm = physical_normals(c.md, md_index(c, e), fid);
      for (int t2 = 0; t2 < nq; ++t2)
        for (int t1 = 0; t1 < nq; ++t1) {
          const int k = t1 + nq * t2;
          const int base = (dir == 0) ? nq * (t1 + nq * t2) : (dir == 1 ? t1 + nq * nq * t2 : t1 + nq * t2);
          const State ul = load(utf, nf, k), ur = load(utn, nf, k);
          const std::array<double, 3> nr{fnrm.unit_normals[3 * k], fnrm.unit_normals[3 * k + 1],
                                         fnrm.unit_normals[3 * k + 2]};
          const Flux F = two_point_flux(c.gas, TwoPointFluxKind::CentralConservative, ul, ur);
          double fn[kStates];
          for (int s = 0; s < kStates; ++s) fn[s] = F[0][s] * nr[0] + F[1][s] * nr[1] + F[2][s] * nr[2];
          if (c.cfg.roe) {
            const State d = roe_dissipation(c.gas, ul, ur, nr);
            for (int s = 0; s < kStates; ++s) fn[s] -= d[s];
          }
          const double jg = fnrm.surface_jacobian[k];
          const double wt = o.wq[t1] * o.wq[t2];
          for (int s = 0; s < kStates; ++s) {
            double fi = 0.0;
            for (int a = 0; a < nq; ++a)
              fi += o.bound_flux(side, a) * fr[(dir * kStates + s) * nv + base + a * stride];
            facc[fid][s * nf + k] = wt * (jg * fn[s] - sign * fi);
          }
        }
    }
  }
  std::vector<double> work(8192), R(kStates * nsol), tmp(nsol);
  for (int s = 0; s < kStates; ++s)
    apply_tensor_product(c.interp_t, c.interp_t, c.interp_t, std::span<const double>(&vol[s * nv], nv), qe,
                         std::span<double>(&R[s * nsol], nsol), work);
  for (int dir = 0; dir < 3; ++dir)
    for (int side = 0; side < 2; ++side) {
      const int fid = 2 * dir + side;
      const Operator1D& a0 = dir == 0 ? c.bs_col[side] : c.interp_t;
      const Operator1D& a1 = dir == 1 ? c.bs_col[side] : c.interp_t;
      const Operator1D& a2 = dir == 2 ? c.bs_col[side] : c.interp_t;
      const Extents fe{dir == 0 ? 1 : nq, dir == 1 ? 1 : nq, dir == 2 ? 1 : nq};
      for (int s = 0; s < kStates; ++s) {
        apply_tensor_product(a0, a1, a2, std::span<const double>(&facc[fid][s * nf], nf), fe, tmp, work);
        for (int i = 0; i < nsol; ++i) R[s * nsol + i] += tmp[i];
      }
    }
  std::vector<double> wa(wa_work_size(o, 3));
  double* out = dudt + static_cast<size_t>(e) * kStates * nsol;
  for (int s = 0; s < kStates; ++s) {
    weight_adjusted_inverse_apply(o, 3, em.jac_vol, std::span<const double>(&R[s * nsol], nsol),
                                  std::span<double>(out + s * nsol, nsol), wa);
    for (int i = 0; i < nsol; ++i) out[s * nsol + i] = -out[s * nsol + i];
  }
}

int do_rhs(RefCtx& c, const double* u, const double* halo_lo, const double* halo_hi, double* dudt,
           double* dS_total) {
  if (dS_total && c.cfg.scheme == NSFR_SCHEME_DG) {
    c.msg = "rhs: the entropy diagnostic is defined for NSFR only";
    return NSFR_E_DIM;
  }
  int rc = project_all(c, u);
  if (rc) return rc;
  std::vector<double> dS(dS_total ? c.ne : 0);
  std::atomic<int> bad{-1};
  parallel_for(c.ne, c.cfg.workers, [&](int e) {
    try {
      if (c.cfg.scheme == NSFR_SCHEME_DG)
        dg_rhs_elem(c, e, halo_lo, halo_hi, dudt);
      else
        rhs_elem(c, e, halo_lo, halo_hi, dudt, dS_total ? dS.data() : nullptr);
    } catch (const std::exception&) {
      bad = e;
    }
  });
  if (bad >= 0) {
    c.msg = "rhs: inadmissible state in element " + std::to_string(bad.load());
    return NSFR_E_INADMISSIBLE;
  }
  if (dS_total) {
    double acc = 0.0;
    for (int e = 0; e < c.ne; ++e) acc += dS[e];
    *dS_total = acc;
  }
  return NSFR_OK;
}

}  // namespace

extern "C" {

void* nsfr_ref_create(const nsfr_cfg* cfg, char* err, int errlen) {
  try {
    auto c = std::make_unique<RefCtx>();
    c->cfg = *cfg;
    c->gas.gamma = cfg->gamma;
    c->ops = build_reference_operators(cfg->p, cfg->quad_kind == 0 ? QuadKind::GaussLegendre
                                                                   : QuadKind::GaussLobattoLegendre,
                                       cfg->overint, cfg->c1d);
    c->np = c->ops.np();
    c->nq = c->ops.nq();
    c->nv = c->nq * c->nq * c->nq;
    c->nsol = c->np * c->np * c->np;
    c->nf = c->nq * c->nq;
    c->ne = cfg->m * cfg->m * (cfg->k1 - cfg->k0);
    c->half_skew = c->ops.skew;
    for (double& v : c->half_skew.a) v *= 0.5;
    c->interp_t = c->ops.basis.interp.transposed();
    for (int side = 0; side < 2; ++side) {
      c->bs_row[side] = Operator1D(1, c->np);
      c->bs_col[side] = Operator1D(c->np, 1);
      for (int a = 0; a < c->np; ++a) {
        c->bs_row[side](0, a) = c->ops.bound_sol(side, a);
        c->bs_col[side](a, 0) = c->ops.bound_sol(side, a);
      }
    }
    c->mapping = warp_grid_3d(cfg->m, cfg->beta, cfg->x_left, cfg->x_right, cfg->grid_degree,
                              cfg->length_scale);
    if (cfg->k0 == 0 && cfg->k1 == cfg->m) {
      c->md = build_metrics_conservative_curl(c->mapping, c->ops);
    } else {  // a z-slab: its own elements only
      c->md_base = cfg->m * cfg->m * cfg->k0;
      c->md = build_metrics_slab(c->mapping, c->ops, c->md_base, c->ne, cfg->workers);
      std::vector<double>().swap(c->mapping.control_points);  // the mesh (neighbours) stays
    }
    c->ut_vol.resize(static_cast<size_t>(c->ne) * kStates * c->nv);
    c->ut_f.resize(static_cast<size_t>(c->ne) * 6 * kStates * c->nf);
    c->vhat.resize(static_cast<size_t>(c->ne) * kStates * c->nsol);
    return c.release();
  } catch (const std::exception& ex) {
    std::snprintf(err, errlen, "%s", ex.what());
    return nullptr;
  }
}

void nsfr_ref_destroy(void* ctx) { delete static_cast<RefCtx*>(ctx); }

const char* nsfr_ref_last_error(void* ctx) { return static_cast<RefCtx*>(ctx)->msg.c_str(); }

int nsfr_ref_tables(void* ctx, double* out, int cap) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  const auto& o = c.ops;
  int pos = 0;
  auto put = [&](const double* a, size_t n) {
    for (size_t i = 0; i < n; ++i)
      if (pos + static_cast<int>(i) < cap) out[pos + i] = a[i];
    pos += static_cast<int>(n);
  };
  put(o.basis.interp.a.data(), o.basis.interp.a.size());
  put(o.proj.a.data(), o.proj.a.size());
  put(o.fr_proj.a.data(), o.fr_proj.a.size());
  put(o.skew.a.data(), o.skew.a.size());
  put(o.bound_flux.a.data(), o.bound_flux.a.size());
  put(o.bound_sol.a.data(), o.bound_sol.a.size());
  put(o.wq.data(), o.wq.size());
  put(o.basis.eval_rule.nodes.data(), o.basis.eval_rule.nodes.size());
  put(o.basis.solution_rule.nodes.data(), o.basis.solution_rule.nodes.size());
  put(o.mmass1d.a.data(), o.mmass1d.a.size());
  put(o.quad_diff.a.data(), o.quad_diff.a.size());
  return pos;
}

int nsfr_ref_metrics(void* ctx, double* jac, double* cof) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  for (int e = 0; e < c.ne; ++e) {
    const ElementMetrics& em = c.md.elem[md_index(c, e)];
    if (jac) std::memcpy(jac + static_cast<size_t>(e) * c.nv, em.jac_vol.data(), sizeof(double) * c.nv);
    if (cof)
      std::memcpy(cof + static_cast<size_t>(e) * c.nv * 9, em.cof_vol.data(),
                  sizeof(double) * c.nv * 9);
  }
  return NSFR_OK;
}

int nsfr_ref_x_sol(void* ctx, double* x) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  for (int e = 0; e < c.ne; ++e)
    std::memcpy(x + static_cast<size_t>(e) * c.nsol * 3, c.md.elem[md_index(c, e)].x_sol.data(),
                sizeof(double) * c.nsol * 3);
  return NSFR_OK;
}

int nsfr_ref_x_vol(void* ctx, double* x) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  for (int e = 0; e < c.ne; ++e)
    std::memcpy(x + static_cast<size_t>(e) * c.nv * 3, c.md.elem[md_index(c, e)].x_vol.data(),
                sizeof(double) * c.nv * 3);
  return NSFR_OK;
}

int nsfr_ref_initial_state(void* ctx, int kind, double* u) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  for (int e = 0; e < c.ne; ++e) {
    const auto& xs = c.md.elem[md_index(c, e)].x_sol;
    for (int q = 0; q < c.nsol; ++q) {
      double st[kStates];
      case_state(c, kind, &xs[3 * static_cast<size_t>(q)], 0.0, st);
      for (int s = 0; s < kStates; ++s) u[(static_cast<size_t>(e) * kStates + s) * c.nsol + q] = st[s];
    }
  }
  return NSFR_OK;
}

int nsfr_ref_traces(void* ctx, const double* u, double* traces) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  int rc = project_all(c, u);
  if (rc) return rc;
  std::memcpy(traces, c.ut_f.data(), sizeof(double) * c.ut_f.size());
  return NSFR_OK;
}

int nsfr_ref_boundary_traces(void* ctx, const double* u, double* send_lo, double* send_hi) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  int rc = project_all(c, u);
  if (rc) return rc;
  const int m = c.cfg.m, nz = c.cfg.k1 - c.cfg.k0, blk = kStates * c.nf;
  for (int plane = 0; plane < m * m; ++plane) {
    const int e_lo = plane, e_hi = plane + m * m * (nz - 1);
    std::memcpy(send_lo + static_cast<size_t>(plane) * blk,
                &c.ut_f[(static_cast<size_t>(e_lo) * 6 + 4) * blk], sizeof(double) * blk);
    std::memcpy(send_hi + static_cast<size_t>(plane) * blk,
                &c.ut_f[(static_cast<size_t>(e_hi) * 6 + 5) * blk], sizeof(double) * blk);
  }
  return NSFR_OK;
}

int nsfr_ref_rhs(void* ctx, const double* u, const double* halo_lo, const double* halo_hi,
                 double* dudt, double* entropy_change) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const bool whole = (c.cfg.k0 == 0 && c.cfg.k1 == c.cfg.m);
  if (!whole && (!halo_lo || !halo_hi)) {
    c.msg = "rhs: halo traces required for a partial slab";
    return NSFR_E_DIM;
  }
  return do_rhs(c, u, halo_lo, halo_hi, dudt, entropy_change);
}

// kinetic-energy volume term: hadamard_sumfac_volume (sumfac.hpp:48-94, 0.5 skew)
// of the reference flux minus the pressure work, dotted with v_KE
int nsfr_ref_ke_volume(void* ctx, const double* u, double* out) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  if (int rc = project_all(c, u)) return rc;
  const int nv = c.nv, nq = c.nq;
  const Extents qe{nq, nq, nq};
  const std::array<const Operator1D*, 3> hs{&c.half_skew, &c.half_skew, &c.half_skew};
  const std::span<const double> w(c.ops.wq);
  const std::array<std::span<const double>, 3> w3{w, w, w};
  std::vector<double> part(c.ne, 0.0);
  std::atomic<int> bad{-1};
  parallel_for(c.ne, c.cfg.workers, [&](int e) {
    const ElementMetrics& em = c.md.elem[md_index(c, e)];
    const double* utv = &c.ut_vol[static_cast<size_t>(e) * kStates * nv];
    std::vector<double> vol(kStates * nv, 0.0);
    auto provider = [&](int i, int j, int dir, double* o5) {
      const State ui = load(utv, nv, i), uj = load(utv, nv, j);
      Flux F = two_point_flux(c.gas, TwoPointFluxKind::ChandrashekarRanochaFix, ui, uj);
      const double pbar = 0.5 * (pressure(c.gas, ui) + pressure(c.gas, uj));
      for (int k = 0; k < 3; ++k) F[k][1 + k] -= pbar;
      const double* Ci = em.cof_at(i);
      const double* Cj = em.cof_at(j);
      const double cm0 = 0.5 * (Ci[0 + dir] + Cj[0 + dir]);
      const double cm1 = 0.5 * (Ci[3 + dir] + Cj[3 + dir]);
      const double cm2 = 0.5 * (Ci[6 + dir] + Cj[6 + dir]);
      for (int s = 0; s < kStates; ++s) o5[s] = F[0][s] * cm0 + F[1][s] * cm1 + F[2][s] * cm2;
    };
    try {
      hadamard_sumfac_volume(hs, w3, qe, kStates, provider, vol, nullptr);
    } catch (const std::exception&) {
      bad = e;
      return;
    }
    double acc = 0.0;
    for (int q = 0; q < nv; ++q) {
      const State vk = kinetic_energy_variables(load(utv, nv, q));  // euler.cpp:83-87
      acc += vk[0] * vol[q] + vk[1] * vol[nv + q] + vk[2] * vol[2 * nv + q] + vk[3] * vol[3 * nv + q];
    }
    part[e] = acc;
  });
  if (bad >= 0) {
    c.msg = "ke_volume: inadmissible state";
    return NSFR_E_INADMISSIBLE;
  }
  double acc = 0.0;
  for (int e = 0; e < c.ne; ++e) acc += part[e];
  *out = acc;
  return NSFR_OK;
}

int nsfr_ref_ke_total(void* ctx, const double* u, double* out) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  if (c.cfg.scheme != NSFR_SCHEME_NSFR || !(c.cfg.k0 == 0 && c.cfg.k1 == c.cfg.m)) {
    c.msg = "ke_total: NSFR on the whole box only";
    return NSFR_E_DIM;
  }
  if (int rc = project_all(c, u)) return rc;
  std::vector<double> keS(c.ne, 0.0);
  std::atomic<int> bad{-1};
  parallel_for(c.ne, c.cfg.workers, [&](int e) {
    try {
      rhs_elem(c, e, nullptr, nullptr, nullptr, nullptr, u, keS.data());
    } catch (const std::exception&) {
      bad = e;
    }
  });
  if (bad >= 0) {
    c.msg = "ke_total: inadmissible state";
    return NSFR_E_INADMISSIBLE;
  }
  double acc = 0.0;
  for (int e = 0; e < c.ne; ++e) acc += keS[e];
  *out = acc;
  return NSFR_OK;
}

int nsfr_ref_max_wavespeed(void* ctx, const double* u, double* lam) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const auto& o = c.ops;
  const Extents me{c.np, c.np, c.np};
  std::vector<double> work(4096), uq(kStates * c.nv);
  double best = 0.0;
  for (int e = 0; e < c.ne; ++e) {
    for (int s = 0; s < kStates; ++s)
      apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                           std::span<const double>(u + (static_cast<size_t>(e) * kStates + s) * c.nsol, c.nsol),
                           me, std::span<double>(&uq[s * c.nv], c.nv), work);
    for (int q = 0; q < c.nv; ++q) {
      const State uu = load(uq.data(), c.nv, q);
      if (!admissible(c.gas, uu)) {
        c.msg = "max_wavespeed: inadmissible state";
        return NSFR_E_INADMISSIBLE;
      }
      const double vx = uu[1] / uu[0], vy = uu[2] / uu[0], vz = uu[3] / uu[0];
      const double speed = std::sqrt(vx * vx + vy * vy + vz * vz);
      const double lm = speed + sound_speed(c.gas, uu);
      if (lm > best) best = lm;
    }
  }
  *lam = best;
  return NSFR_OK;
}

int nsfr_ref_rk4_step(void* ctx, double* u, double dt) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const size_t N = static_cast<size_t>(c.ne) * kStates * c.nsol;
  std::vector<double> us(N), k(N), acc(N);
  const double hdt = 0.5 * dt, sdt = dt / 6.0;
  int rc = do_rhs(c, u, nullptr, nullptr, k.data(), nullptr);
  if (rc) return rc;
  for (size_t i = 0; i < N; ++i) {
    acc[i] = k[i];
    us[i] = std::fma(hdt, k[i], u[i]);
  }
  if ((rc = do_rhs(c, us.data(), nullptr, nullptr, k.data(), nullptr))) return rc;
  for (size_t i = 0; i < N; ++i) {
    acc[i] = std::fma(2.0, k[i], acc[i]);
    us[i] = std::fma(hdt, k[i], u[i]);
  }
  if ((rc = do_rhs(c, us.data(), nullptr, nullptr, k.data(), nullptr))) return rc;
  for (size_t i = 0; i < N; ++i) {
    acc[i] = std::fma(2.0, k[i], acc[i]);
    us[i] = std::fma(dt, k[i], u[i]);
  }
  if ((rc = do_rhs(c, us.data(), nullptr, nullptr, k.data(), nullptr))) return rc;
  for (size_t i = 0; i < N; ++i) {
    acc[i] = acc[i] + k[i];
    u[i] = std::fma(sdt, acc[i], u[i]);
  }
  return NSFR_OK;
}

int nsfr_ref_l2_error(void* ctx, const double* u, double t, int kind, double out2[2]) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const auto& o = c.ops;
  const int nq = c.nq;
  const Extents me{c.np, c.np, c.np};
  std::vector<double> work(4096), uq(kStates * c.nv);
  double er = 0.0, ep = 0.0;
  for (int e = 0; e < c.ne; ++e) {
    const ElementMetrics& em = c.md.elem[md_index(c, e)];
    for (int s = 0; s < kStates; ++s)
      apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                           std::span<const double>(u + (static_cast<size_t>(e) * kStates + s) * c.nsol, c.nsol),
                           me, std::span<double>(&uq[s * c.nv], c.nv), work);
    double pr = 0.0, pp = 0.0;
    for (int k = 0; k < nq; ++k)
      for (int j = 0; j < nq; ++j)
        for (int i = 0; i < nq; ++i) {
          const int q = i + nq * (j + nq * k);
          double w = o.wq[i];
          w *= o.wq[j];
          w *= o.wq[k];
          const double wj = w * em.jac_vol[q];
          const State uu = load(uq.data(), c.nv, q);
          double ex[kStates];
          case_state(c, kind, &em.x_vol[3 * static_cast<size_t>(q)], t, ex);
          State exs{ex[0], ex[1], ex[2], ex[3], ex[4]};
          const double dr = uu[0] - ex[0];
          const double dp = pressure(c.gas, uu) - pressure(c.gas, exs);
          pr += wj * dr * dr;
          pp += wj * dp * dp;
        }
    er += pr;
    ep += pp;
  }
  out2[0] = er;
  out2[1] = ep;
  return NSFR_OK;
}

int nsfr_ref_entropy_total(void* ctx, const double* u, double* out) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const auto& o = c.ops;
  const int nq = c.nq;
  const Extents me{c.np, c.np, c.np};
  std::vector<double> work(4096), uq(kStates * c.nv);
  double tot = 0.0;
  for (int e = 0; e < c.ne; ++e) {
    const ElementMetrics& em = c.md.elem[md_index(c, e)];
    for (int s = 0; s < kStates; ++s)
      apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                           std::span<const double>(u + (static_cast<size_t>(e) * kStates + s) * c.nsol, c.nsol),
                           me, std::span<double>(&uq[s * c.nv], c.nv), work);
    double pe = 0.0;
    for (int k = 0; k < nq; ++k)
      for (int j = 0; j < nq; ++j)
        for (int i = 0; i < nq; ++i) {
          const int q = i + nq * (j + nq * k);
          double w = o.wq[i];
          w *= o.wq[j];
          w *= o.wq[k];
          pe += w * em.jac_vol[q] * entropy_function(c.gas, load(uq.data(), c.nv, q));
        }
    tot += pe;
  }
  *out = tot;
  return NSFR_OK;
}

int nsfr_ref_conserved_totals(void* ctx, const double* u, double out5[5]) {
  RefCtx& c = *static_cast<RefCtx*>(ctx);
  const auto& o = c.ops;
  const int nq = c.nq;
  const Extents me{c.np, c.np, c.np};
  std::vector<double> work(4096), uq(kStates * c.nv);
  double tot[kStates] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int e = 0; e < c.ne; ++e) {
    const ElementMetrics& em = c.md.elem[md_index(c, e)];
    for (int s = 0; s < kStates; ++s)
      apply_tensor_product(o.basis.interp, o.basis.interp, o.basis.interp,
                           std::span<const double>(u + (static_cast<size_t>(e) * kStates + s) * c.nsol, c.nsol),
                           me, std::span<double>(&uq[s * c.nv], c.nv), work);
    double pe[kStates] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < nq; ++k)
      for (int j = 0; j < nq; ++j)
        for (int i = 0; i < nq; ++i) {
          const int q = i + nq * (j + nq * k);
          double w = o.wq[i];
          w *= o.wq[j];
          w *= o.wq[k];
          const double wj = w * em.jac_vol[q];
          for (int s = 0; s < kStates; ++s) pe[s] += wj * uq[s * c.nv + q];
        }
    for (int s = 0; s < kStates; ++s) tot[s] += pe[s];
  }
  for (int s = 0; s < kStates; ++s) out5[s] = tot[s];
  return NSFR_OK;
}

// primitive probes (golden-vector generation)
double nsfr_ref_log_mean(double a, double b) { return log_mean(a, b); }
int nsfr_ref_flux_ec(double g, const double* ul, const double* ur, double* f15) {
  try {
    EulerGas gas{g};
    const Flux F = two_point_flux(gas, TwoPointFluxKind::ChandrashekarRanochaFix,
                                  State{ul[0], ul[1], ul[2], ul[3], ul[4]},
                                  State{ur[0], ur[1], ur[2], ur[3], ur[4]});
    for (int k = 0; k < 3; ++k)
      for (int s = 0; s < kStates; ++s) f15[k * kStates + s] = F[k][s];
    return NSFR_OK;
  } catch (const std::exception&) {
    return NSFR_E_INADMISSIBLE;
  }
}
int nsfr_ref_roe(double g, const double* ul, const double* ur, const double* n, double* out) {
  try {
    EulerGas gas{g};
    const State d = roe_dissipation(gas, State{ul[0], ul[1], ul[2], ul[3], ul[4]},
                                    State{ur[0], ur[1], ur[2], ur[3], ur[4]}, {n[0], n[1], n[2]});
    for (int s = 0; s < kStates; ++s) out[s] = d[s];
    return NSFR_OK;
  } catch (const std::exception&) {
    return NSFR_E_INADMISSIBLE;
  }
}
int nsfr_ref_entropy_vars(double g, const double* u, double* v) {
  try {
    const State r = entropy_variables(EulerGas{g}, State{u[0], u[1], u[2], u[3], u[4]});
    for (int s = 0; s < kStates; ++s) v[s] = r[s];
    return NSFR_OK;
  } catch (const std::exception&) {
    return NSFR_E_INADMISSIBLE;
  }
}
int nsfr_ref_entropy_to_cons(double g, const double* v, double* u) {
  try {
    const State r = entropy_to_conservative(EulerGas{g}, State{v[0], v[1], v[2], v[3], v[4]});
    for (int s = 0; s < kStates; ++s) u[s] = r[s];
    return NSFR_OK;
  } catch (const std::exception&) {
    return NSFR_E_INADMISSIBLE;
  }
}
double nsfr_ref_c_plus(int p) {
  return correction_c_plus_available(p) ? correction_c_plus(p) : -1.0;
}
double nsfr_ref_c_hu(int p) { return correction_c_hu(p); }
double nsfr_ref_gcl_residual(void* ctx) {
  const RefCtx& c = *static_cast<RefCtx*>(ctx);
  return gcl_residual(c.md, c.ops);
}

}  // extern "C"
