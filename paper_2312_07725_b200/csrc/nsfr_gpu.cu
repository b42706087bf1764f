// nsfr_gpu.cu — context, C ABI (include/nsfr_gpu.h), launch plumbing, NCCL halo
// exchange and reductions for the B200-native NSFR residual path.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nsfr_gpu.h"
#include "kernels.cuh"
#include "tables.hpp"

using namespace nsfr_b200;

struct nsfr_gpu_ctx {
  nsfr_gpu_setup s{};
  int N = 0, E = 0, m = 0, nz = 0, k0 = 0, k1 = 0;
  int NQ = 0;       // volume quadrature nodes per direction (N unless overintegrated, DG only)
  bool dg = false;  // conservative strong-form DG instead of NSFR (kernel_dg.cuh)
  double* d_dgus = nullptr;  // DG stage state u_hat
  Tables1D tab;
  DevTables htab{};  // host copy of the device tables (source of the kernel-parameter operators)
  DevTables* d_tab = nullptr;
  double *d_un = nullptr, *d_acc = nullptr, *d_rhs = nullptr;
  double *d_vol = nullptr, *d_facc = nullptr;  // K2 -> K3 volume / face rows
  double *d_utv = nullptr, *d_tr = nullptr, *d_cof = nullptr, *d_jac = nullptr, *d_wj = nullptr;
  double *d_vhat = nullptr, *d_dS = nullptr, *d_part = nullptr, *d_red = nullptr;
  double *d_send_lo = nullptr, *d_send_hi = nullptr, *d_halo_lo = nullptr, *d_halo_hi = nullptr;
  StepState* d_step = nullptr;
  StepState* h_step = nullptr;  // pinned
  unsigned* d_err = nullptr;
  unsigned* h_err = nullptr;    // pinned
  cudaStream_t st = nullptr;
  cudaStream_t st_copy = nullptr;  // host<->device state transfers, chunk-pipelined with st
  cudaStream_t st_d2h = nullptr;   // device->host leg of the streamed step (runs beside st_copy)
  cudaStream_t st_comm = nullptr;   // halo exchange overlapped with K2 on the interior planes
  cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
  std::vector<cudaStream_t> lanes;  // streamed step: compute lanes (a chunk's ops stay on one lane)
  std::vector<cudaEvent_t> op_ev;   // streamed step: one event per (layer, chunk) op, + fork/join
  std::vector<cudaEvent_t> chunk_ev;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, peer_lo = 0, peer_hi = 0;
  long long halo_count = 0;
  cudaGraphExec_t graph = nullptr;
  // ut_vol/traces hold the projection of d_un and lam_bits its lambda_max
  // (K3 re-projects after every stage); cleared when d_un changes from outside
  bool proj_valid = false;
  bool chi_pi_identity = false;  // chi Pi~ = I to 1e-13 (c_DG): K3 skips the final passes
  int ahead_proj = 0, ahead_res = 0, ahead_upd = 0;  // look-ahead L2 prefetch distances (CTAs)
  long long launches = 0;
  // per-launch event timing (bench roofline)
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_marks;  // (kind, index of start event)
  std::string msg;
};

namespace {

thread_local std::string g_create_error;

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      ctx->msg = std::string(#call) + ": " + cudaGetErrorString(e_);                      \
      return NSFR_E_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

#define NK(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) {                                                              \
      ctx->msg = std::string(#call) + ": " + ncclGetErrorString(r_);                      \
      return NSFR_E_NCCL;                                                                 \
    }                                                                                     \
  } while (0)

// Every ABI entry that takes a context runs on that context's device and
// restores the caller's current device on return (a thread may drive contexts
// on several GPUs; kernel attributes, lazily created streams/events and the
// launches themselves are all per device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int want) {
    int cur = -1;
    if (want < 0 || cudaGetDevice(&cur) != cudaSuccess) return;
    if (cur != want && cudaSetDevice(want) == cudaSuccess) prev = cur;
  }
  explicit DeviceGuard(const nsfr_gpu_ctx* c) : DeviceGuard(c ? c->s.device : -1) {}
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Blocking copy ordered on the context's (non-blocking) stream: a plain
// cudaMemcpy runs on the legacy stream, which does NOT wait for work queued on
// a cudaStreamNonBlocking stream (nor does that work wait for it).
cudaError_t copy_sync(cudaStream_t st, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
  return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
}

size_t nsol(const nsfr_gpu_ctx* c) { return static_cast<size_t>(c->N) * c->N * c->N; }
size_t state_count(const nsfr_gpu_ctx* c) { return static_cast<size_t>(c->E) * NS * nsol(c); }
size_t nquad(const nsfr_gpu_ctx* c) { return static_cast<size_t>(c->NQ) * c->NQ * c->NQ; }

// Kernel attributes (dynamic shared memory above 48 KB) are per device: the
// devices already configured, per instantiation (one thread per GPU may share
// the process). The look-ahead distances live in the context.
template <int N>
struct AttrsDone {
  static inline std::atomic<unsigned> mask{0};
};

template <int N>
int set_attrs(nsfr_gpu_ctx* ctx) {
  if (ctx->ahead_res) return NSFR_OK;
  const unsigned bit = 1u << (ctx->s.device & 31);
  if (!(AttrsDone<N>::mask.load() & bit)) {
    CK(cudaFuncSetAttribute(k_project<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, ProjCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_project<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ProjCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_residual<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, ResCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_residual<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ResCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_residual<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ResCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_update<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, UpdCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_update<N, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            UpdCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_update<N, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            UpdCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_update<N, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            UpdCfg<N>::SMEM));
    CK(cudaFuncSetAttribute(k_update<N, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            UpdCfg<N>::SMEM));
    AttrsDone<N>::mask.fetch_or(bit);
  }
  int sms = 0, bp = 0, br = 0, bu = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->s.device));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bp, k_project<N>, ProjCfg<N>::THREADS, ProjCfg<N>::SMEM));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&br, k_residual<N>, ResCfg<N>::THREADS, ResCfg<N>::SMEM));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bu, k_update<N>, UpdCfg<N>::THREADS, UpdCfg<N>::SMEM));
  // Look-ahead L2 prefetch distance in resident waves. Measured (A/B in one
  // session, round 1): a quarter wave helps at p=4 (K2 -0.7%, K3 -0.8% vs one
  // wave), none is best at p=3 (K2 -5%). Re-swept with the round-2 kernels
  // (fused face lift; 0 / 0.25 / 0.5 / 1 wave): p=4 within 0.3% either way,
  // p=3 none still best, p=5 a quarter wave -2.5% per step (K3 -7.8%).
  // NSFR_PF_WAVES overrides, NSFR_NO_PREFETCH=1 disables.
  const char* w = std::getenv("NSFR_PF_WAVES");
  const double waves = w ? std::atof(w) : (N == 5 || N == 6 ? 0.25 : 0.0);
  const bool pf = std::getenv("NSFR_NO_PREFETCH") == nullptr && waves > 0.0;
  auto ahead = [&](int blocks) { return pf ? static_cast<int>(waves * sms * std::max(blocks, 1)) : (1 << 30); };
  ctx->ahead_proj = ahead(bp);
  ctx->ahead_res = ahead(br);
  ctx->ahead_upd = ahead(bu);
  return NSFR_OK;
}

void ev_begin(nsfr_gpu_ctx* c, int kind) {
  if (!c->timing) return;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  c->ev_marks.push_back({kind, static_cast<int>(c->ev_pool.size())});
  c->ev_pool.push_back(a);
  c->ev_pool.push_back(b);
  cudaEventRecord(a, c->st);
}
void ev_end(nsfr_gpu_ctx* c) {
  if (!c->timing) return;
  cudaEventRecord(c->ev_pool.back(), c->st);
}

// 1D operators for the kernel-parameter bank, from the host table copy
template <int N>
ProjOps<N> proj_ops(const nsfr_gpu_ctx* ctx) {
  const DevTables& t = ctx->htab;
  ProjOps<N> o{};
  for (int i = 0; i < N * N; ++i) {
    o.proj[i] = t.proj[i];
    o.chi[i] = t.interp[i];
  }
  for (int i = 0; i < 2 * N; ++i) o.bsol[i] = t.bsol[i];
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < N; ++a) {  // (bound_sol Pi)[side][a]; Pi is np x nq
      double s = 0.0;
      for (int r = 0; r < N; ++r) s += t.bsol[side * N + r] * t.proj[r * N + a];
      o.bp[side * N + a] = s;
    }
  o.c35 = 0.0;
  {  // closed-form u(v) when gamma/(gamma-1) == 7/2 in exact arithmetic (gamma = 1.4)
    const double g = ctx->s.gamma, gm1 = g - 1.0;
    if (std::fabs(g / gm1 - 3.5) < 1e-12 && std::getenv("NSFR_POW_U_OF_V") == nullptr)
      o.c35 = std::pow(gm1, 1.0 / gm1);
  }
  return o;
}

template <int N>
ResOps<N> res_ops(const DevTables& t) {
  ResOps<N> o{};
  for (int i = 0; i < N * N; ++i) o.q[i] = t.qskew[i];
  for (int i = 0; i < 2 * N; ++i) o.bflux[i] = t.bflux[i];
  for (int i = 0; i < N; ++i) o.wq[i] = t.wq[i];
  return o;
}

// stage 0 ends in u_hat space (Pi~^3: dU/dt of the coefficients); the RK
// stages stay at the quadrature nodes, chi^3 Pi~^3 = (chi Pi~)^3
template <int N>
UpdOps<N> upd_ops(const nsfr_gpu_ctx* ctx, int stage) {
  const DevTables& t = ctx->htab;
  UpdOps<N> u{};
  TailOps<N>& o = u.t;
  for (int a = 0; a < N; ++a)
    for (int i = 0; i < N; ++i) {
      // M = Pi~^T chi^T: (Pi~^T)[a][r] = frproj[r][a], (chi^T)[r][i] = interp[i][r]
      double s = 0.0;
      for (int r = 0; r < N; ++r) s += t.frproj[r * N + a] * t.interp[i * N + r];
      o.M[a * N + i] = s;
    }
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < N; ++a) {
      double s = 0.0;
      for (int r = 0; r < N; ++r) s += t.frproj[r * N + a] * t.bsol[side * N + r];
      o.bm[side * N + a] = s;
    }
  for (int c = 0; c < N; ++c)
    for (int a = 0; a < N; ++a) {
      double s = 0.0;
      for (int r = 0; r < N; ++r) s += t.interp[c * N + r] * t.frproj[r * N + a];
      o.fr[c * N + a] = stage == 0 ? t.frproj[c * N + a] : s;
    }
  for (int i = 0; i < N * N; ++i) {
    o.frt[i] = t.frproj_t[i];
    o.it[i] = t.interp_t[i];
  }
  for (int i = 0; i < 2 * N; ++i) o.bs[i] = t.bsol[i];
  o.Ms = SymOp<N>::fold(o.M);
  o.frs = SymOp<N>::fold(o.fr);
  u.p = proj_ops<N>(ctx);
  return u;
}

// projection parameters writing ut_vol / traces / halo send buffers
ProjParams proj_params(nsfr_gpu_ctx* ctx, const double* u, bool want_lam) {
  ProjParams P{};
  P.u = u;
  P.ut_vol = ctx->d_utv;
  P.traces = ctx->d_tr;
  P.vhat = ctx->d_vhat;
  P.send_lo = ctx->d_send_lo;
  P.send_hi = ctx->d_send_hi;
  P.lam = want_lam ? &ctx->d_step->lam_bits : nullptr;
  P.err = ctx->d_err;
  P.E = ctx->E;
  P.m = ctx->m;
  P.nz = ctx->nz;
  P.gamma = ctx->s.gamma;
  return P;
}

// Launches cover the element range [ea, eb) (eb < 0: the whole slab); ea is a
// multiple of 8 so every batch's TMA blocks stay 16-byte aligned.
int range_end(const nsfr_gpu_ctx* ctx, int eb) { return eb < 0 ? ctx->E : eb; }

// uq_out: u is u_hat; chi^3 u lands there and is projected (streamed upload)
template <int N>
int launch_project(nsfr_gpu_ctx* ctx, const double* u, bool want_lam, int ea, int eb, double* uq_out) {
  if (int rc = set_attrs<N>(ctx)) return rc;
  ProjParams P = proj_params(ctx, u, want_lam);
  P.e_begin = ea;
  P.E = range_end(ctx, eb);
  P.uq_out = uq_out;
  const int grid = (P.E - ea + ProjCfg<N>::EPB - 1) / ProjCfg<N>::EPB;
  ev_begin(ctx, 1);
  if (uq_out)
    k_project<N, true><<<grid, ProjCfg<N>::THREADS, ProjCfg<N>::SMEM, ctx->st>>>(P, proj_ops<N>(ctx),
                                                                               ctx->ahead_proj);
  else
    k_project<N><<<grid, ProjCfg<N>::THREADS, ProjCfg<N>::SMEM, ctx->st>>>(P, proj_ops<N>(ctx),
                                                                           ctx->ahead_proj);
  ev_end(ctx);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

template <int N>
int launch_residual(nsfr_gpu_ctx* ctx, int km, int ea, int eb) {
  ResParams P{};
  P.ut_vol = ctx->d_utv;
  P.traces = ctx->d_tr;
  P.halo_lo = ctx->d_halo_lo;
  P.halo_hi = ctx->d_halo_hi;
  P.cof = ctx->d_cof;
  P.vol = ctx->d_vol;
  P.facc = ctx->d_facc;
  P.err = ctx->d_err;
  P.E = ctx->E;
  P.m = ctx->m;
  P.dm = DivMagic::make(ctx->m);
  P.dmm = DivMagic::make(ctx->m * ctx->m);
  P.nz = ctx->nz;
  P.gamma = ctx->s.gamma;
  P.gas = GasC::make(ctx->s.gamma);
  P.roe = ctx->s.roe;
  P.e_begin = ea;
  P.E = range_end(ctx, eb);
  if (int rc = set_attrs<N>(ctx)) return rc;
  const int grid = (P.E - ea + ResCfg<N>::EPB - 1) / ResCfg<N>::EPB;
  ev_begin(ctx, 2);
  if (km == 1)
    k_residual<N, 1><<<grid, ResCfg<N>::THREADS, ResCfg<N>::SMEM, ctx->st>>>(P, res_ops<N>(ctx->htab),
                                                                           ctx->ahead_res);
  else if (km == 2)
    k_residual<N, 2><<<grid, ResCfg<N>::THREADS, ResCfg<N>::SMEM, ctx->st>>>(P, res_ops<N>(ctx->htab),
                                                                           ctx->ahead_res);
  else
    k_residual<N><<<grid, ResCfg<N>::THREADS, ResCfg<N>::SMEM, ctx->st>>>(P, res_ops<N>(ctx->htab),
                                                                           ctx->ahead_res);
  ev_end(ctx);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

// stage 0: dU/dt (+ entropy change); stages 1-4: RK update and projection of
// the next stage state (lambda_max after stage 4)
// uhat_out (stage 4 only): write Pi^3 u_{n+1} there (and adaptive_dt's lambda
// into lam_out when given) instead of projecting u_{n+1}
template <int N>
int launch_update(nsfr_gpu_ctx* ctx, int stage, bool entropy, const double* vhat, int ea, int eb,
                  double* uhat_out, unsigned long long* lam_out) {
  UpdParams P{};
  P.vol = ctx->d_vol;
  P.facc = ctx->d_facc;
  P.wj = ctx->d_wj;
  P.vhat = entropy ? (vhat ? vhat : ctx->d_vhat) : nullptr;
  P.dS = entropy ? ctx->d_dS : nullptr;
  P.un = ctx->d_un;
  P.acc = ctx->d_acc;
  P.out = ctx->d_rhs;
  P.dt = &ctx->d_step->dt;
  P.stage = stage;
  P.pj = proj_params(ctx, nullptr, stage == 4);
  P.pj.vhat = nullptr;
  P.pj.e_begin = ea;
  P.pj.E = range_end(ctx, eb);
  P.uhat_out = uhat_out;
  P.lam_out = lam_out;
  if (int rc = set_attrs<N>(ctx)) return rc;
  ev_begin(ctx, 3);
  const UpdOps<N> O = upd_ops<N>(ctx, stage);
  // variant: 0 general, 1 c_DG identity M (+ entropy-free stage 0), 2 identity M and final passes,
  // 3 streamed stage 4 (u_hat out), 4 streamed stage 4 with the identity
  const int var = uhat_out ? (ctx->chi_pi_identity ? 4 : 3)
                           : (ctx->chi_pi_identity && stage > 0 ? 2 : (ctx->chi_pi_identity && !entropy ? 1 : 0));
  {
    using C = UpdCfg<N>;
    const int grid = (P.pj.E - ea + C::EPB - 1) / C::EPB;
    const int a = ctx->ahead_upd;
    switch (var) {
      case 4: k_update<N, true, true, true><<<grid, C::THREADS, C::SMEM, ctx->st>>>(P, O, a); break;
      case 3: k_update<N, false, false, true><<<grid, C::THREADS, C::SMEM, ctx->st>>>(P, O, a); break;
      case 2: k_update<N, true, true><<<grid, C::THREADS, C::SMEM, ctx->st>>>(P, O, a); break;
      case 1: k_update<N, true, false><<<grid, C::THREADS, C::SMEM, ctx->st>>>(P, O, a); break;
      default: k_update<N><<<grid, C::THREADS, C::SMEM, ctx->st>>>(P, O, a);
    }
  }
  ev_end(ctx);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

#define NSFR_DISPATCH(fn, args)                \
  switch (ctx->N) {                            \
    case 3: return fn<3> args;                 \
    case 4: return fn<4> args;                 \
    case 5: return fn<5> args;                 \
    case 6: return fn<6> args;                 \
    case 7: return fn<7> args;                 \
  }                                            \
  ctx->msg = "unsupported p";                  \
  return NSFR_E_DIM

int project(nsfr_gpu_ctx* ctx, const double* u, bool lam, int ea = 0, int eb = -1, double* uq_out = nullptr) {
  NSFR_DISPATCH(launch_project, (ctx, u, lam, ea, eb, uq_out));
}
// km: 0 the residual, 1 / 2 kinetic-energy diagnostic rows (kernel_residual.cuh)
int residual(nsfr_gpu_ctx* ctx, int km = 0, int ea = 0, int eb = -1) {
  NSFR_DISPATCH(launch_residual, (ctx, km, ea, eb));
}
// entropy: stage-0 diagnostic -vhat . R, with vhat = v_hat (default) or the given coefficients
int update(nsfr_gpu_ctx* ctx, int stage, bool entropy, const double* vhat = nullptr, int ea = 0,
           int eb = -1, double* uhat_out = nullptr, unsigned long long* lam_out = nullptr) {
  NSFR_DISPATCH(launch_update, (ctx, stage, entropy, vhat, ea, eb, uhat_out, lam_out));
}

// ---- conservative DG (kernel_dg.cuh) ------------------------------------------
template <int NP, int NQ>
DgOps<NP, NQ> dg_ops(const nsfr_gpu_ctx* ctx) {
  const DevTables& t = ctx->htab;
  DgOps<NP, NQ> o{};
  for (int i = 0; i < NQ * NP; ++i) o.chi[i] = t.interp[i];
  for (int i = 0; i < 2 * NP; ++i) o.bs[i] = t.bsol[i];
  for (int i = 0; i < NQ * NQ; ++i) o.D[i] = t.quad_diff[i];
  for (int i = 0; i < 2 * NQ; ++i) o.bflux[i] = t.bflux[i];
  for (int i = 0; i < NQ; ++i) o.wq[i] = t.wq[i];
  for (int a = 0; a < NQ; ++a)
    for (int i = 0; i < NQ; ++i) {  // M = Pi~^T chi^T (nq x nq)
      double v = 0.0;
      for (int r = 0; r < NP; ++r) v += t.frproj[r * NQ + a] * t.interp[i * NP + r];
      o.M[a * NQ + i] = v;
    }
  for (int side = 0; side < 2; ++side)
    for (int a = 0; a < NQ; ++a) {
      double v = 0.0;
      for (int r = 0; r < NP; ++r) v += t.frproj[r * NQ + a] * t.bsol[side * NP + r];
      o.bm[side * NQ + a] = v;
    }
  for (int i = 0; i < NP * NQ; ++i) o.fr[i] = t.frproj[i];
  return o;
}

template <int NP, int NQ>
struct DgAttrsDone {
  static inline std::atomic<unsigned> mask{0};
};

template <int NP, int NQ>
int dg_attrs(nsfr_gpu_ctx* ctx) {
  using Cfg = DgCfg<NP, NQ>;
  const unsigned bit = 1u << (ctx->s.device & 31);
  if (!(DgAttrsDone<NP, NQ>::mask.load() & bit)) {
    CK(cudaFuncSetAttribute(k_dg_states<NP, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::S_SMEM));
    CK(cudaFuncSetAttribute(k_dg_residual<NP, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            Cfg::R_SMEM));
    DgAttrsDone<NP, NQ>::mask.fetch_or(bit);
  }
  return NSFR_OK;
}

template <int NP, int NQ>
int launch_dg_states(nsfr_gpu_ctx* ctx, const double* u, bool want_lam) {
  using Cfg = DgCfg<NP, NQ>;
  if (int rc = dg_attrs<NP, NQ>(ctx)) return rc;
  DgStateParams P{};
  P.u = u;
  P.traces = ctx->d_tr;
  P.send_lo = ctx->d_send_lo;
  P.send_hi = ctx->d_send_hi;
  P.lam = want_lam ? &ctx->d_step->lam_bits : nullptr;
  P.err = ctx->d_err;
  P.E = ctx->E;
  P.m = ctx->m;
  P.nz = ctx->nz;
  P.gamma = ctx->s.gamma;
  const int grid = (ctx->E + Cfg::EPB - 1) / Cfg::EPB;
  ev_begin(ctx, 1);
  k_dg_states<NP, NQ><<<grid, Cfg::THREADS, Cfg::S_SMEM, ctx->st>>>(P, dg_ops<NP, NQ>(ctx));
  ev_end(ctx);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

template <int NP, int NQ>
int launch_dg_residual(nsfr_gpu_ctx* ctx, int stage, const double* us, double* uo) {
  using Cfg = DgCfg<NP, NQ>;
  if (int rc = dg_attrs<NP, NQ>(ctx)) return rc;
  DgResParams P{};
  P.us = us;
  P.traces = ctx->d_tr;
  P.halo_lo = ctx->d_halo_lo;
  P.halo_hi = ctx->d_halo_hi;
  P.cof = ctx->d_cof;
  P.wj = ctx->d_wj;
  P.un = ctx->d_un;
  P.uo = uo;
  P.acc = ctx->d_acc;
  P.out = ctx->d_rhs;
  P.dt = &ctx->d_step->dt;
  P.err = ctx->d_err;
  P.stage = stage;
  P.E = ctx->E;
  P.m = ctx->m;
  P.nz = ctx->nz;
  P.gamma = ctx->s.gamma;
  P.roe = ctx->s.roe;
  const int grid = (ctx->E + Cfg::EPB - 1) / Cfg::EPB;
  ev_begin(ctx, 2);
  k_dg_residual<NP, NQ><<<grid, Cfg::THREADS, Cfg::R_SMEM, ctx->st>>>(P, dg_ops<NP, NQ>(ctx));
  ev_end(ctx);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

#define NSFR_DG_DISPATCH(fn, args)                                  \
  switch (ctx->N * 16 + ctx->NQ) {                                  \
    case 4 * 16 + 4: return fn<4, 4> args;                          \
    case 4 * 16 + 5: return fn<4, 5> args;                          \
    case 4 * 16 + 6: return fn<4, 6> args;                          \
    case 5 * 16 + 5: return fn<5, 5> args;                          \
    case 5 * 16 + 6: return fn<5, 6> args;                          \
    case 5 * 16 + 7: return fn<5, 7> args;                          \
    case 6 * 16 + 6: return fn<6, 6> args;                          \
    case 6 * 16 + 7: return fn<6, 7> args;                          \
    case 6 * 16 + 8: return fn<6, 8> args;                          \
  }                                                                 \
  ctx->msg = "DG: unsupported (p, overint)";                        \
  return NSFR_E_DIM

int dg_states(nsfr_gpu_ctx* ctx, const double* u, bool lam) { NSFR_DG_DISPATCH(launch_dg_states, (ctx, u, lam)); }
int dg_residual(nsfr_gpu_ctx* ctx, int stage, const double* us, double* uo) {
  NSFR_DG_DISPATCH(launch_dg_residual, (ctx, stage, us, uo));
}

// z-face halo exchange with the two slab neighbours
int exchange(nsfr_gpu_ctx* ctx) {
  if (!ctx->comm) return NSFR_OK;  // single rank, or external halo mode
  const size_t n = static_cast<size_t>(ctx->halo_count);
  NK(ncclGroupStart());
  NK(ncclSend(ctx->d_send_lo, n, ncclDouble, ctx->peer_lo, ctx->comm, ctx->st));
  NK(ncclRecv(ctx->d_halo_hi, n, ncclDouble, ctx->peer_hi, ctx->comm, ctx->st));
  NK(ncclSend(ctx->d_send_hi, n, ncclDouble, ctx->peer_hi, ctx->comm, ctx->st));
  NK(ncclRecv(ctx->d_halo_lo, n, ncclDouble, ctx->peer_lo, ctx->comm, ctx->st));
  NK(ncclGroupEnd());
  return NSFR_OK;
}

int allreduce_sum(nsfr_gpu_ctx* ctx, double* d, int n) {
  if (!ctx->comm) return NSFR_OK;
  NK(ncclAllReduce(d, d, n, ncclDouble, ncclSum, ctx->comm, ctx->st));
  return NSFR_OK;
}

// K1 of d_un with lambda_max (the step pipeline's prologue); DG: KD1 face states
int project_state(nsfr_gpu_ctx* ctx) {
  k_step_begin<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  if (ctx->dg) {
    if (int rc = dg_states(ctx, ctx->d_un, true)) return rc;
  } else if (int rc = project(ctx, ctx->d_un, true)) {
    return rc;
  }
  ctx->proj_valid = true;
  return NSFR_OK;
}

// (DG steps start with their own face-state pass: nothing to cache)
int ensure_projected(nsfr_gpu_ctx* ctx) {
  return ctx->proj_valid || ctx->dg ? NSFR_OK : project_state(ctx);
}

// one full residual of d_un into d_rhs (stage 0)
int rhs_of_state(nsfr_gpu_ctx* ctx, bool entropy) {
  if (int rc = project_state(ctx)) return rc;
  if (int rc = exchange(ctx)) return rc;
  if (ctx->dg) return dg_residual(ctx, 0, ctx->d_un, nullptr);
  if (int rc = residual(ctx)) return rc;
  return update(ctx, 0, entropy);
}

// DG RK4 step: KD1 (face states of the stage state, lambda at stage 1) ->
// halo -> KD2 (residual, WA inverse, stage update in u_hat space), 4 times
int enqueue_step_dg(nsfr_gpu_ctx* ctx, bool fixed_dt) {
  k_step_begin<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  if (int rc = dg_states(ctx, ctx->d_un, !fixed_dt)) return rc;
  if (!fixed_dt) {
    if (ctx->comm)
      NK(ncclAllReduce(&ctx->d_step->lam_bits, &ctx->d_step->lam_bits, 1, ncclUint64, ncclMax,
                       ctx->comm, ctx->st));
    k_step_dt<<<1, 1, 0, ctx->st>>>(ctx->d_step);
    ++ctx->launches;
  }
  for (int stage = 1; stage <= 4; ++stage) {
    if (stage > 1)
      if (int rc = dg_states(ctx, ctx->d_dgus, false)) return rc;
    if (int rc = exchange(ctx)) return rc;
    if (int rc = dg_residual(ctx, stage, stage == 1 ? ctx->d_un : ctx->d_dgus, ctx->d_dgus)) return rc;
  }
  k_step_end<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  CK(cudaGetLastError());
  ctx->proj_valid = false;
  return NSFR_OK;
}

// One stage's halo exchange and K2: with NCCL and at least
// three planes, the grouped send/recv runs on st_comm while K2 covers the
// interior planes, whose faces need no halo; the two end planes follow once
// the halo has landed. Element-local arithmetic: bitwise the serial order.
// NSFR_NO_HALO_OVERLAP=1 keeps exchange -> K2 on one stream.
bool halo_overlap(const nsfr_gpu_ctx* ctx) {
  return ctx->comm && !ctx->dg && ctx->nz >= 3 && !std::getenv("NSFR_NO_HALO_OVERLAP");
}

int exchange_residual(nsfr_gpu_ctx* ctx) {
  if (!halo_overlap(ctx)) {
    if (int rc = exchange(ctx)) return rc;
    return residual(ctx);
  }
  if (!ctx->st_comm) {
    CK(cudaStreamCreateWithFlags(&ctx->st_comm, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
  }
  const int plane = ctx->m * ctx->m;
  cudaStream_t main_st = ctx->st;
  CK(cudaEventRecord(ctx->ev_fork, main_st));  // the send planes are packed
  CK(cudaStreamWaitEvent(ctx->st_comm, ctx->ev_fork, 0));
  ctx->st = ctx->st_comm;
  const int rc_x = exchange(ctx);
  ctx->st = main_st;
  if (rc_x) return rc_x;
  CK(cudaEventRecord(ctx->ev_halo, ctx->st_comm));
  if (int rc = residual(ctx, 0, plane, ctx->E - plane)) return rc;
  CK(cudaStreamWaitEvent(main_st, ctx->ev_halo, 0));
  if (int rc = residual(ctx, 0, 0, plane)) return rc;
  return residual(ctx, 0, ctx->E - plane, ctx->E);
}

// Enqueue one RK4 step (no host sync), graph-capturable: needs the projection
// of d_un in place (ensure_projected) and leaves the projection of u_{n+1}.
// fixed_dt: dt already in d_step.
constexpr long long kLaunchesPerStep = 1 + 4 * 2 + 1;
long long launches_per_step(const nsfr_gpu_ctx* ctx) {
  if (ctx->dg) return 1 + 1 + 1 + 4 + 3 + 1;
  return halo_overlap(ctx) ? kLaunchesPerStep + 4 * 2 : kLaunchesPerStep;  // K2 in three ranges
}
int enqueue_step(nsfr_gpu_ctx* ctx, bool fixed_dt) {
  if (ctx->dg) return enqueue_step_dg(ctx, fixed_dt);
  if (!fixed_dt) {
    if (ctx->comm)
      NK(ncclAllReduce(&ctx->d_step->lam_bits, &ctx->d_step->lam_bits, 1, ncclUint64, ncclMax,
                       ctx->comm, ctx->st));
    k_step_dt<<<1, 1, 0, ctx->st>>>(ctx->d_step);  // reads and clears lambda
  } else {
    k_step_begin<<<1, 1, 0, ctx->st>>>(ctx->d_step);  // clears lambda
  }
  ++ctx->launches;
  for (int stage = 1; stage <= 4; ++stage) {
    if (int rc = exchange_residual(ctx)) return rc;
    if (int rc = update(ctx, stage, false)) return rc;
  }
  k_step_end<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

// synchronise and translate the device error word
int sync_check(nsfr_gpu_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaMemcpyAsync(ctx->h_step, ctx->d_step, sizeof(StepState), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  const unsigned e = *ctx->h_err;
  if (e) {
    CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (e & ERR_MESH) {
      ctx->msg = "nonpositive metric Jacobian or degenerate face (InvalidMeshError)";
      return NSFR_E_MESH;
    }
    char buf[160];
    std::snprintf(buf, sizeof buf, "inadmissible state at t=%.17g (StepFailureError)%s",
                  ctx->h_step->t, (e & ERR_ROE) ? " [Roe average]" : "");
    ctx->msg = buf;
    return NSFR_E_INADMISSIBLE;
  }
  return NSFR_OK;
}

void fill_dev_tables(const Tables1D& t, const nsfr_gpu_tables* user, DevTables& d) {
  std::memset(&d, 0, sizeof d);
  const int np = t.np, nq = t.nq;
  d.np = np;
  d.nq = nq;
  d.g = t.g;
  const double* interp = user ? user->interp : t.interp.data();
  const double* proj = user ? user->proj : t.proj.data();
  const double* frp = user ? user->fr_proj : t.fr_proj.data();
  const double* skew = user ? user->skew : t.skew.data();
  const double* bflux = user ? user->bound_flux : t.bound_flux.data();
  const double* bsol = user ? user->bound_sol : t.bound_sol.data();
  const double* wq = user ? user->wq : t.wq.data();
  for (int i = 0; i < nq * np; ++i) d.interp[i] = interp[i];
  for (int i = 0; i < nq; ++i)
    for (int j = 0; j < np; ++j) d.interp_t[j * nq + i] = interp[i * np + j];
  for (int i = 0; i < np * nq; ++i) {
    d.proj[i] = proj[i];
    d.frproj[i] = frp[i];
  }
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < nq; ++j) d.frproj_t[j * np + i] = frp[i * nq + j];
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b) {
      // hadamard_sumfac_volume called with 0.5*skew (D2): q(a,b) - q(b,a)
      const double qab = 0.5 * skew[a * nq + b], qba = 0.5 * skew[b * nq + a];
      d.qskew[a * nq + b] = qab - qba;
    }
  for (int i = 0; i < 2 * nq; ++i) d.bflux[i] = bflux[i];
  for (int i = 0; i < 2 * np; ++i) d.bsol[i] = bsol[i];
  for (int i = 0; i < nq; ++i) d.wq[i] = wq[i];
  for (int i = 0; i < nq * nq; ++i) d.quad_diff[i] = t.quad_diff[i];
  for (int i = 0; i < t.g; ++i) d.gnodes[i] = t.grid_nodes[i];
  for (int i = 0; i < nq * t.g; ++i) d.ig[i] = t.ig[i];
  for (int i = 0; i < np * t.g; ++i) d.is[i] = t.is[i];
  for (int i = 0; i < t.g * t.g; ++i) d.dg[i] = t.dg[i];
}

double length_scale(const nsfr_gpu_setup& s) {
  return s.length_scale > 0.0 ? s.length_scale : (s.x_right - s.x_left) / (2.0 * M_PI);
}

int setup_kernel_smem(nsfr_gpu_ctx* ctx, size_t bytes, const void* fn) {
  if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return NSFR_OK;
}

// mode 0: out = (chi or Pi)^3 in; 1: lambda_max of chi^3 in into
// d_step->lam_out_bits (no output); 2: out = Pi^3 in and lambda_max of chi^3 out
template <int N>
int launch_convert_lines(nsfr_gpu_ctx* ctx, const double* in, double* out, bool to_quad, int e0, int e1,
                         int mode) {
  using Cfg = ConvCfg<N>;
  const unsigned bit = 1u << (ctx->s.device & 31);
  static std::atomic<unsigned> done{0};
  if (!(done.load() & bit)) {
    CK(cudaFuncSetAttribute(k_convert_lines<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    CK(cudaFuncSetAttribute(k_convert_lines<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    CK(cudaFuncSetAttribute(k_convert_lines<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    done.fetch_or(bit);
  }
  ConvOps<N> o{};
  for (int i = 0; i < N * N; ++i) {
    o.A[i] = to_quad ? ctx->htab.interp[i] : ctx->htab.proj[i];
    o.B[i] = ctx->htab.interp[i];
  }
  const int grid = (e1 - e0 + Cfg::EPB - 1) / Cfg::EPB;
  unsigned long long* lam = &ctx->d_step->lam_out_bits;
  if (mode == 1)
    k_convert_lines<N, 1><<<grid, Cfg::THREADS, Cfg::SMEM, ctx->st>>>(o, in, nullptr, e0, e1, ctx->s.gamma, lam);
  else if (mode == 2)
    k_convert_lines<N, 2><<<grid, Cfg::THREADS, Cfg::SMEM, ctx->st>>>(o, in, out, e0, e1, ctx->s.gamma, lam);
  else
    k_convert_lines<N, 0><<<grid, Cfg::THREADS, Cfg::SMEM, ctx->st>>>(o, in, out, e0, e1);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

// adaptive_dt's lambda_max of chi^3 u_hat over [e0, e1) (u_hat on the device,
// e.g. a state on its way to the host) into d_step->lam_out_bits; with
// from_q, u_hat = Pi^3 u_q is formed from `in` on the way into `out` first
int lam_of_uhat(nsfr_gpu_ctx* ctx, const double* in, int e0, int e1, double* out = nullptr) {
  if (e1 <= e0) return NSFR_OK;
  const int mode = out ? 2 : 1;
  switch (ctx->NQ == ctx->N ? ctx->N : 0) {
    case 3: return launch_convert_lines<3>(ctx, in, out, mode == 1, e0, e1, mode);
    case 4: return launch_convert_lines<4>(ctx, in, out, mode == 1, e0, e1, mode);
    case 5: return launch_convert_lines<5>(ctx, in, out, mode == 1, e0, e1, mode);
    case 6: return launch_convert_lines<6>(ctx, in, out, mode == 1, e0, e1, mode);
    case 7: return launch_convert_lines<7>(ctx, in, out, mode == 1, e0, e1, mode);
  }
  ctx->msg = "adaptive dt of the output: overintegrated DG is not supported";
  return NSFR_E_DIM;
}

// u_hat <-> u_q of elements [e0, e1): to_quad applies chi^3, else Pi^3
// (line-pass kernel for n_q = n_p; the generic k_convert for overintegrated DG)
int convert_range(nsfr_gpu_ctx* ctx, const double* in, double* out, bool to_quad, int e0, int e1) {
  if (e1 <= e0) return NSFR_OK;
  if (ctx->NQ == ctx->N) {
    switch (ctx->N) {
      case 3: return launch_convert_lines<3>(ctx, in, out, to_quad, e0, e1, 0);
      case 4: return launch_convert_lines<4>(ctx, in, out, to_quad, e0, e1, 0);
      case 5: return launch_convert_lines<5>(ctx, in, out, to_quad, e0, e1, 0);
      case 6: return launch_convert_lines<6>(ctx, in, out, to_quad, e0, e1, 0);
      case 7: return launch_convert_lines<7>(ctx, in, out, to_quad, e0, e1, 0);
    }
  }
  const size_t smem = sizeof(double) * 4 * std::max(nsol(ctx), nquad(ctx));
  const size_t in_per = NS * (to_quad ? nsol(ctx) : nquad(ctx)), out_per = NS * (to_quad ? nquad(ctx) : nsol(ctx));
  k_convert<<<e1 - e0, 128, smem, ctx->st>>>(ctx->d_tab, in + e0 * in_per, out + e0 * out_per, e1 - e0,
                                             to_quad ? 1 : 0);
  ++ctx->launches;
  CK(cudaGetLastError());
  return NSFR_OK;
}

int convert_state(nsfr_gpu_ctx* ctx, const double* in, double* out, bool to_quad) {
  return convert_range(ctx, in, out, to_quad, 0, ctx->E);
}

// state transfers: ~64 MB chunks (at least one)
int transfer_chunks(const nsfr_gpu_ctx* ctx) {
  const size_t bytes = sizeof(double) * state_count(ctx);
  return static_cast<int>(std::min<size_t>(64, std::max<size_t>(1, bytes >> 26)));
}

int ensure_chunk_events(nsfr_gpu_ctx* ctx, int n) {
  while (static_cast<int>(ctx->chunk_ev.size()) < n) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->chunk_ev.push_back(e);
  }
  return NSFR_OK;
}

int build_metrics(nsfr_gpu_ctx* ctx) {
  const int g = ctx->tab.g, n = ctx->NQ, G3 = g * g * g, N3 = n * n * n;
  const int M = std::max(g, n), M3 = M * M * M;
  const size_t smem = sizeof(double) * (13 * G3 + 2 * M3 + 20 * N3);
  if (int rc = setup_kernel_smem(ctx, smem, (const void*)k_metrics)) return rc;
  MetricParams P{};
  P.tab = ctx->d_tab;
  P.jac = ctx->d_jac;
  P.cof = ctx->d_cof;
  P.wj = ctx->d_wj;
  P.E = ctx->E;
  P.m = ctx->m;
  P.k0 = ctx->k0;
  P.x_left = ctx->s.x_left;
  P.h = (ctx->s.x_right - ctx->s.x_left) / ctx->m;
  P.beta = ctx->s.beta;
  P.l = length_scale(ctx->s);
  P.err = ctx->d_err;
  k_metrics<<<ctx->E, 128, smem, ctx->st>>>(P);
  ++ctx->launches;
  CK(cudaGetLastError());
  return sync_check(ctx);
}

}  // namespace

extern "C" {

const char* nsfr_gpu_create_error(void) { return g_create_error.c_str(); }

int nsfr_gpu_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return NSFR_E_NCCL;
  std::memcpy(out128, &id, sizeof id);
  return NSFR_OK;
}

int nsfr_gpu_halo_plan_for(int m, int p, int rank, int nranks, nsfr_gpu_halo_plan* out) {
  if (nranks < 1 || rank < 0 || rank >= nranks || m < nranks || p < 1) return NSFR_E_DIM;
  out->k0 = static_cast<int>(static_cast<long long>(rank) * m / nranks);
  out->k1 = static_cast<int>(static_cast<long long>(rank + 1) * m / nranks);
  out->peer_lo = (rank - 1 + nranks) % nranks;
  out->peer_hi = (rank + 1) % nranks;
  out->count = static_cast<long long>(m) * m * NTR * (p + 1) * (p + 1);
  return NSFR_OK;
}

int nsfr_gpu_create(const nsfr_gpu_setup* setup, nsfr_gpu_ctx** out) {
  DeviceGuard dev_guard_(setup ? setup->device : -1);
  *out = nullptr;
  auto* ctx = new nsfr_gpu_ctx();
  ctx->s = *setup;
  auto fail = [&](int rc) {
    g_create_error = ctx->msg;
    nsfr_gpu_destroy(ctx);
    return rc;
  };
  const nsfr_gpu_setup& s = ctx->s;
  if (s.p < 2 || s.p > 6 || s.m < 1 || s.k0 < 0 || s.k1 > s.m || s.k0 >= s.k1 ||
      !(s.quad_kind == 0 || s.quad_kind == 1) || s.grid_degree < 1 || s.grid_degree + 1 > MAXG ||
      !(s.gamma > 1.0) || !(s.x_right > s.x_left) || s.beta < 0.0) {
    ctx->msg = "nsfr_gpu_create: dimension/configuration out of range (p in [2,6], 0<=k0<k1<=m)";
    return fail(NSFR_E_DIM);
  }
  ctx->dg = (s.scheme == NSFR_SCHEME_DG);
  if (!(s.scheme == NSFR_SCHEME_NSFR || ctx->dg) || (!ctx->dg && s.overint != 0) ||
      (ctx->dg && (s.p < 3 || s.p > 5 || s.overint < 0 || s.overint > 2))) {
    ctx->msg = "nsfr_gpu_create: scheme/overint out of range (NSFR: overint 0; DG: p in [3,5], "
               "overint in [0,2])";
    return fail(NSFR_E_DIM);
  }
  ctx->N = s.p + 1;
  ctx->NQ = s.p + 1 + s.overint;
  ctx->m = s.m;
  ctx->k0 = s.k0;
  ctx->k1 = s.k1;
  ctx->nz = s.k1 - s.k0;
  ctx->E = s.m * s.m * ctx->nz;
  ctx->rank = s.rank;
  ctx->nranks = s.nranks < 1 ? 1 : s.nranks;
  if (ctx->nranks == 1 && (s.k0 != 0 || s.k1 != s.m)) {
    ctx->msg = "nsfr_gpu_create: a single rank must own the whole box";
    return fail(NSFR_E_DIM);
  }
  const char* why = nullptr;
  if (!build_tables(s.p, s.quad_kind, s.overint, s.c1d, s.grid_degree, ctx->tab, &why)) {
    ctx->msg = why;
    return fail(NSFR_E_DIM);
  }
  if (cudaSetDevice(s.device) != cudaSuccess) {
    ctx->msg = "cudaSetDevice failed (no CUDA device?)";
    return fail(NSFR_E_CUDA);
  }
  if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->st_copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->st_d2h, cudaStreamNonBlocking) != cudaSuccess) {
    ctx->msg = "cudaStreamCreate failed (no CUDA device?)";
    return fail(NSFR_E_CUDA);
  }
  DevTables dt;
  fill_dev_tables(ctx->tab, s.tables && s.tables->interp ? s.tables : nullptr, dt);
  ctx->htab = dt;
  if (!ctx->dg) {
    // K3 applies M = Pi~^T chi^T and chi Pi~ / Pi~ through their even / odd halves
    // (SymOp, kernel_update.cuh), which needs chi and Pi~ centrosymmetric: true of
    // every symmetric node set and basis (GL / LGL, the reference's tables)
    const int n = ctx->N;
    double asym = 0.0, big = 0.0;
    for (int r = 0; r < n; ++r)
      for (int a = 0; a < n; ++a) {
        const int i = r * n + a, j = (n - 1 - r) * n + (n - 1 - a);
        asym = std::max({asym, std::fabs(dt.interp[i] - dt.interp[j]), std::fabs(dt.frproj[i] - dt.frproj[j])});
        big = std::max({big, std::fabs(dt.interp[i]), std::fabs(dt.frproj[i])});
      }
    if (!(asym <= 1e-11 * big)) {
      ctx->msg = "nsfr_gpu_create: the 1D operators are not centrosymmetric (asymmetric nodes or basis)";
      return fail(NSFR_E_CONFIG);
    }
  }
  if (!ctx->dg && std::getenv("NSFR_NO_IDENTITY_SKIP") == nullptr) {
    double dev = 0.0;  // max |chi Pi~ - I| (n_q = n_p)
    for (int c = 0; c < ctx->N; ++c)
      for (int a = 0; a < ctx->N; ++a) {
        double v = 0.0;
        for (int r = 0; r < ctx->N; ++r) v += dt.interp[c * ctx->N + r] * dt.frproj[r * ctx->N + a];
        dev = std::max(dev, std::fabs(v - (c == a ? 1.0 : 0.0)));
      }
    ctx->chi_pi_identity = dev < 1e-13;
  }
  const size_t ns = state_count(ctx), n3 = static_cast<size_t>(ctx->E) * nquad(ctx);
  const size_t ntr = static_cast<size_t>(ctx->E) * 6 * NS * ctx->NQ * ctx->NQ;    // face rows
  const size_t ntrace = static_cast<size_t>(ctx->E) * 6 * NTR * ctx->NQ * ctx->NQ;  // face traces (DG: NS of NTR used)
  const size_t nscr = static_cast<size_t>(ctx->E) * NS * std::max(nsol(ctx), nquad(ctx));
  auto alloc = [&](double** p, size_t n) {
    cudaError_t e = cudaMalloc(p, sizeof(double) * std::max<size_t>(n, 1));
#ifdef NSFR_DEBUG_CHECKS
    // NaN bytes, on the context stream (stream-ordered before every use; the
    // legacy-stream cudaMemset would not be ordered with the non-blocking ctx->st)
    if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0xff, sizeof(double) * std::max<size_t>(n, 1), ctx->st);
#endif
    return e;
  };
  if (cudaMalloc(&ctx->d_tab, sizeof(DevTables)) || alloc(&ctx->d_un, ns) || alloc(&ctx->d_vol, nscr) ||
      alloc(&ctx->d_acc, ns) || alloc(&ctx->d_rhs, ns) || alloc(&ctx->d_utv, 6 * n3) ||
      alloc(&ctx->d_tr, ntrace) || alloc(&ctx->d_facc, !ctx->dg && fuse_face(ctx->N) ? 0 : ntr) || alloc(&ctx->d_cof, 9 * n3) || alloc(&ctx->d_jac, n3) ||
      alloc(&ctx->d_wj, n3) || alloc(&ctx->d_dS, ctx->E) || alloc(&ctx->d_part, 2 * (size_t)ctx->E) ||
      alloc(&ctx->d_red, 8) || cudaMalloc(&ctx->d_step, sizeof(StepState)) ||
      cudaMalloc(&ctx->d_err, sizeof(unsigned)) ||
      cudaMallocHost(&ctx->h_step, sizeof(StepState)) || cudaMallocHost(&ctx->h_err, sizeof(unsigned))) {
    ctx->msg = "nsfr_gpu_create: device allocation failed";
    return fail(NSFR_E_CUDA);
  }
  if ((s.entropy_diag && alloc(&ctx->d_vhat, ns)) || (ctx->dg && alloc(&ctx->d_dgus, ns))) {
    ctx->msg = "nsfr_gpu_create: device allocation failed";
    return fail(NSFR_E_CUDA);
  }
  // halo planes: z-slabs of nranks > 1, or a 1-rank NCCL communicator (nccl_id
  // given): its halo is a send/recv to itself, i.e. the periodic wrap through
  // the real NCCL path (tests/test_gpu_parity.py::test_nccl_loopback_*)
  if (ctx->nranks > 1 || s.nccl_id) {
    nsfr_gpu_halo_plan plan;
    if (nsfr_gpu_halo_plan_for(s.m, s.p, ctx->rank, ctx->nranks, &plan) || plan.k0 != s.k0 ||
        plan.k1 != s.k1) {
      ctx->msg = "nsfr_gpu_create: slab does not match nsfr_gpu_halo_plan_for";
      return fail(NSFR_E_DIM);
    }
    ctx->peer_lo = plan.peer_lo;
    ctx->peer_hi = plan.peer_hi;
    ctx->halo_count = static_cast<long long>(s.m) * s.m * NTR * ctx->NQ * ctx->NQ;
    const size_t hc = static_cast<size_t>(ctx->halo_count);
    if (alloc(&ctx->d_send_lo, hc) || alloc(&ctx->d_send_hi, hc) || alloc(&ctx->d_halo_lo, hc) ||
        alloc(&ctx->d_halo_hi, hc)) {
      ctx->msg = "nsfr_gpu_create: halo allocation failed";
      return fail(NSFR_E_CUDA);
    }
    // without an NCCL id the caller moves the halo planes itself (external
    // halo mode: nsfr_gpu_halo_buffers / halo_get / halo_set + nsfr_gpu_stage)
    if (s.nccl_id) {
      ncclUniqueId id;
      std::memcpy(&id, s.nccl_id, sizeof id);
      if (ncclCommInitRank(&ctx->comm, ctx->nranks, id, ctx->rank) != ncclSuccess) {
        ctx->msg = "ncclCommInitRank failed";
        return fail(NSFR_E_NCCL);
      }
    }
  }
  StepState h{};
  h.dx = (s.x_right - s.x_left) / (s.m * (s.p + 1));
  if (cudaMemcpyAsync(ctx->d_tab, &dt, sizeof dt, cudaMemcpyHostToDevice, ctx->st) ||
      cudaMemcpyAsync(ctx->d_step, &h, sizeof h, cudaMemcpyHostToDevice, ctx->st) ||
      cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->st) ||
      cudaStreamSynchronize(ctx->st)) {
    ctx->msg = "nsfr_gpu_create: upload failed";
    return fail(NSFR_E_CUDA);
  }
  if (setup->jac_vol && setup->cof_vol) {
    // caller-built metrics (ElementMetrics layout [e][q][9]) -> 0.5 C as [e][9][q], wj = w J
    const int N3 = static_cast<int>(nquad(ctx)), nq = ctx->NQ;
    std::vector<double> cof(9 * n3), wj(n3);
    const auto& wq = (s.tables && s.tables->wq) ? std::vector<double>(s.tables->wq, s.tables->wq + nq)
                                                : ctx->tab.wq;
    for (int e = 0; e < ctx->E; ++e)
      for (int q = 0; q < N3; ++q) {
        for (int c = 0; c < 9; ++c)
          cof[(static_cast<size_t>(e) * 9 + c) * N3 + q] =
              0.5 * setup->cof_vol[(static_cast<size_t>(e) * N3 + q) * 9 + c];
        const int i = q % nq, j = (q / nq) % nq, k = q / (nq * nq);
        double w = wq[i];
        w *= wq[j];
        w *= wq[k];
        const double J = setup->jac_vol[static_cast<size_t>(e) * N3 + q];
        if (!(J > 0.0)) {
          ctx->msg = "nsfr_gpu_create: nonpositive J in caller metrics";
          return fail(NSFR_E_MESH);
        }
        wj[static_cast<size_t>(e) * N3 + q] = 1.0 / (w * J);  // K2 multiplies by 1/(w J)
      }
    if (copy_sync(ctx->st, ctx->d_cof, cof.data(), sizeof(double) * cof.size(), cudaMemcpyHostToDevice) ||
        copy_sync(ctx->st, ctx->d_jac, setup->jac_vol, sizeof(double) * n3, cudaMemcpyHostToDevice) ||
        copy_sync(ctx->st, ctx->d_wj, wj.data(), sizeof(double) * n3, cudaMemcpyHostToDevice)) {
      ctx->msg = "nsfr_gpu_create: metric upload failed";
      return fail(NSFR_E_CUDA);
    }
  } else if (int rc = build_metrics(ctx)) {
    return fail(rc);
  }
  *out = ctx;
  return NSFR_OK;
}

int nsfr_gpu_destroy(nsfr_gpu_ctx* ctx) {
  DeviceGuard dev_guard_(ctx);
  if (!ctx) return NSFR_OK;
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  double* bufs[] = {ctx->d_dgus, ctx->d_un,  ctx->d_vol,  ctx->d_facc, ctx->d_acc,  ctx->d_rhs,     ctx->d_utv,     ctx->d_tr,
                    ctx->d_cof, ctx->d_jac,  ctx->d_wj,   ctx->d_vhat,    ctx->d_dS,      ctx->d_part,
                    ctx->d_red, ctx->d_send_lo, ctx->d_send_hi, ctx->d_halo_lo, ctx->d_halo_hi};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (ctx->d_tab) cudaFree(ctx->d_tab);
  if (ctx->d_step) cudaFree(ctx->d_step);
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->h_step) cudaFreeHost(ctx->h_step);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  for (auto e : ctx->chunk_ev) cudaEventDestroy(e);
  if (ctx->st_copy) cudaStreamDestroy(ctx->st_copy);
  if (ctx->st_d2h) cudaStreamDestroy(ctx->st_d2h);
  for (auto l : ctx->lanes) cudaStreamDestroy(l);
  if (ctx->st_comm) cudaStreamDestroy(ctx->st_comm);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  for (auto e : ctx->op_ev) cudaEventDestroy(e);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
  return NSFR_OK;
}

int nsfr_gpu_comm_info(nsfr_gpu_ctx* ctx, int* nccl_nranks, int* nccl_rank, int* cuda_device) {
  DeviceGuard dev_guard_(ctx);
  if (!ctx || !nccl_nranks || !nccl_rank || !cuda_device) return NSFR_E_DIM;
  *nccl_nranks = 0;
  *nccl_rank = -1;
  *cuda_device = ctx->s.device;
  if (!ctx->comm) return NSFR_OK;
  NK(ncclCommCount(ctx->comm, nccl_nranks));
  NK(ncclCommUserRank(ctx->comm, nccl_rank));
  NK(ncclCommCuDevice(ctx->comm, cuda_device));
  return NSFR_OK;
}

const char* nsfr_gpu_last_error(const nsfr_gpu_ctx* ctx) { return ctx ? ctx->msg.c_str() : "null context"; }

int nsfr_gpu_get_tables(nsfr_gpu_ctx* ctx, double* out, int cap) {
  DeviceGuard dev_guard_(ctx);
  const Tables1D& t = ctx->tab;
  int pos = 0;
  auto put = [&](const std::vector<double>& v) {
    for (size_t i = 0; i < v.size(); ++i)
      if (pos + static_cast<int>(i) < cap) out[pos + i] = v[i];
    pos += static_cast<int>(v.size());
  };
  put(t.interp);
  put(t.proj);
  put(t.fr_proj);
  put(t.skew);
  put(t.bound_flux);
  put(t.bound_sol);
  put(t.wq);
  put(t.quad_nodes);
  put(t.sol_nodes);
  put(t.mmass1d);
  put(t.quad_diff);
  return pos;
}

int nsfr_gpu_get_metrics(nsfr_gpu_ctx* ctx, double* jac, double* cof) {
  DeviceGuard dev_guard_(ctx);
  const size_t n3 = static_cast<size_t>(ctx->E) * nquad(ctx);
  const int N3 = static_cast<int>(nquad(ctx));
  CK(cudaStreamSynchronize(ctx->st));
  if (jac) CK(copy_sync(ctx->st, jac, ctx->d_jac, sizeof(double) * n3, cudaMemcpyDeviceToHost));
  if (cof) {
    std::vector<double> c(9 * n3);
    CK(copy_sync(ctx->st, c.data(), ctx->d_cof, sizeof(double) * c.size(), cudaMemcpyDeviceToHost));
    for (int e = 0; e < ctx->E; ++e)
      for (int q = 0; q < N3; ++q)
        for (int k = 0; k < 9; ++k)
          cof[(static_cast<size_t>(e) * N3 + q) * 9 + k] = 2.0 * c[(static_cast<size_t>(e) * 9 + k) * N3 + q];
  }
  return NSFR_OK;
}

int nsfr_gpu_set_state(nsfr_gpu_ctx* ctx, const double* u) {
  DeviceGuard dev_guard_(ctx);
  ctx->proj_valid = false;
  if (ctx->dg) return nsfr_gpu_set_state_q(ctx, u);  // DG carries u_hat itself
  // u_hat -> scratch (d_vol is dead between steps) -> u_q = chi^3 u_hat, in
  // element chunks: the copy of chunk c+1 overlaps the conversion of chunk c
  const int nch = transfer_chunks(ctx);
  if (int rc = ensure_chunk_events(ctx, nch)) return rc;
  const size_t per = nsol(ctx) * NS;
  CK(cudaStreamSynchronize(ctx->st));  // d_vol / d_un are free
  for (int c = 0; c < nch; ++c) {
    const int e0 = static_cast<int>(static_cast<long long>(ctx->E) * c / nch);
    const int e1 = static_cast<int>(static_cast<long long>(ctx->E) * (c + 1) / nch);
    if (e1 <= e0) continue;
    CK(cudaMemcpyAsync(ctx->d_vol + e0 * per, u + e0 * per, sizeof(double) * per * (e1 - e0),
                       cudaMemcpyHostToDevice, ctx->st_copy));
    CK(cudaEventRecord(ctx->chunk_ev[c], ctx->st_copy));
    CK(cudaStreamWaitEvent(ctx->st, ctx->chunk_ev[c], 0));
    if (int rc = convert_range(ctx, ctx->d_vol, ctx->d_un, true, e0, e1)) return rc;
  }
  CK(cudaStreamSynchronize(ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_get_state(nsfr_gpu_ctx* ctx, double* u) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) return nsfr_gpu_get_state_q(ctx, u);
  // u_q -> Pi^3 -> u_hat in element chunks; the copy of chunk c overlaps the
  // conversion of chunk c+1
  const int nch = transfer_chunks(ctx);
  if (int rc = ensure_chunk_events(ctx, nch)) return rc;
  const size_t per = nsol(ctx) * NS;
  for (int c = 0; c < nch; ++c) {
    const int e0 = static_cast<int>(static_cast<long long>(ctx->E) * c / nch);
    const int e1 = static_cast<int>(static_cast<long long>(ctx->E) * (c + 1) / nch);
    if (e1 <= e0) continue;
    if (int rc = convert_range(ctx, ctx->d_un, ctx->d_vol, false, e0, e1)) return rc;
    CK(cudaEventRecord(ctx->chunk_ev[c], ctx->st));
    CK(cudaStreamWaitEvent(ctx->st_copy, ctx->chunk_ev[c], 0));
    CK(cudaMemcpyAsync(u + e0 * per, ctx->d_vol + e0 * per, sizeof(double) * per * (e1 - e0),
                       cudaMemcpyDeviceToHost, ctx->st_copy));
  }
  CK(cudaStreamSynchronize(ctx->st_copy));
  CK(cudaStreamSynchronize(ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_set_state_q(nsfr_gpu_ctx* ctx, const double* uq) {
  DeviceGuard dev_guard_(ctx);
  ctx->proj_valid = false;
  CK(cudaMemcpyAsync(ctx->d_un, uq, sizeof(double) * state_count(ctx), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_get_state_q(nsfr_gpu_ctx* ctx, double* uq) {
  DeviceGuard dev_guard_(ctx);
  CK(cudaMemcpyAsync(uq, ctx->d_un, sizeof(double) * state_count(ctx), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_init_case(nsfr_gpu_ctx* ctx, int kind) {
  DeviceGuard dev_guard_(ctx);
  const int g = ctx->tab.g, np = ctx->N, G3 = g * g * g, S3 = np * np * np;
  const int M = std::max(g, np), M3 = M * M * M;
  const size_t smem = sizeof(double) * (3 * G3 + 2 * M3 + 3 * S3);
  if (int rc = setup_kernel_smem(ctx, smem, (const void*)k_init)) return rc;
  InitParams P{};
  P.tab = ctx->d_tab;
  P.u = ctx->dg ? ctx->d_un : ctx->d_vol;  // u_hat at the solution nodes (NSFR: then u_q)
  P.E = ctx->E;
  P.m = ctx->m;
  P.k0 = ctx->k0;
  P.kind = kind;
  P.x_left = ctx->s.x_left;
  P.h = (ctx->s.x_right - ctx->s.x_left) / ctx->m;
  P.beta = ctx->s.beta;
  P.l = length_scale(ctx->s);
  P.gamma = ctx->s.gamma;
  ctx->proj_valid = false;
  k_init<<<ctx->E, 128, smem, ctx->st>>>(P);
  ++ctx->launches;
  CK(cudaGetLastError());
  if (!ctx->dg)
    if (int rc = convert_state(ctx, ctx->d_vol, ctx->d_un, true)) return rc;
  return nsfr_gpu_set_time(ctx, 0.0);
}

int nsfr_gpu_set_time(nsfr_gpu_ctx* ctx, double t) {
  DeviceGuard dev_guard_(ctx);
  ctx->proj_valid = false;  // also the re-sync point after writes through state_device_ptr
  CK(cudaMemcpyAsync(&ctx->d_step->t, &t, sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_get_time(nsfr_gpu_ctx* ctx, double* t) {
  DeviceGuard dev_guard_(ctx);
  if (int rc = sync_check(ctx)) return rc;
  *t = ctx->h_step->t;
  return NSFR_OK;
}

int nsfr_gpu_rhs(nsfr_gpu_ctx* ctx, double* dudt, double* entropy_change) {
  DeviceGuard dev_guard_(ctx);
  const bool ent = entropy_change != nullptr;
  if (ent && ctx->dg) {
    ctx->msg = "entropy change: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  if (ent && !ctx->d_vhat) {
    ctx->msg = "entropy change needs setup.entropy_diag = 1";
    return NSFR_E_CONFIG;
  }
  if (int rc = rhs_of_state(ctx, ent)) return rc;
  if (ent) {
    k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_dS, ctx->E, 1, ctx->d_red);
    ++ctx->launches;
    if (int rc = allreduce_sum(ctx, ctx->d_red, 1)) return rc;
  }
  if (int rc = sync_check(ctx)) return rc;
  if (dudt) CK(copy_sync(ctx->st, dudt, ctx->d_rhs, sizeof(double) * state_count(ctx), cudaMemcpyDeviceToHost));
  if (ent) CK(copy_sync(ctx->st, entropy_change, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost));
  return NSFR_OK;
}

int nsfr_gpu_entropy_change(nsfr_gpu_ctx* ctx, double* out) {
  DeviceGuard dev_guard_(ctx);
  return nsfr_gpu_rhs(ctx, nullptr, out);
}

int nsfr_gpu_get_traces(nsfr_gpu_ctx* ctx, double* traces) {
  DeviceGuard dev_guard_(ctx);
  CK(cudaStreamSynchronize(ctx->st));
  const size_t q2 = static_cast<size_t>(ctx->NQ) * ctx->NQ, nf = static_cast<size_t>(ctx->E) * 6;
  if (ctx->dg) {  // the DG kernels keep conservative face states
    CK(copy_sync(ctx->st, traces, ctx->d_tr, sizeof(double) * nf * NS * q2, cudaMemcpyDeviceToHost));
    return NSFR_OK;
  }
  // NSFR traces are primitives (rho, u, v, w, p, rho/p; physics.cuh): back to
  // the conservative [E][6][5][nq^2] the interface speaks
  std::vector<double> prim(nf * NTR * q2);
  CK(copy_sync(ctx->st, prim.data(), ctx->d_tr, sizeof(double) * prim.size(), cudaMemcpyDeviceToHost));
  const double igm1 = 1.0 / (ctx->s.gamma - 1.0);
  for (size_t f = 0; f < nf; ++f)
    for (size_t k = 0; k < q2; ++k) {
      const double* q = prim.data() + f * NTR * q2 + k;
      double* u = traces + f * NS * q2 + k;
      const double rho = q[0], vx = q[q2], vy = q[2 * q2], vz = q[3 * q2], pr = q[4 * q2];
      u[0] = rho;
      u[q2] = rho * vx;
      u[2 * q2] = rho * vy;
      u[3 * q2] = rho * vz;
      u[4 * q2] = pr * igm1 + 0.5 * rho * (vx * vx + vy * vy + vz * vz);
    }
  return NSFR_OK;
}

int nsfr_gpu_max_wavespeed(nsfr_gpu_ctx* ctx, double* lam) {
  DeviceGuard dev_guard_(ctx);
  if (int rc = project_state(ctx)) return rc;
  if (ctx->comm)
    NK(ncclAllReduce(&ctx->d_step->lam_bits, &ctx->d_step->lam_bits, 1, ncclUint64, ncclMax, ctx->comm, ctx->st));
  if (int rc = sync_check(ctx)) return rc;
  unsigned long long b = ctx->h_step->lam_bits;
  std::memcpy(lam, &b, sizeof b);
  return NSFR_OK;
}

int nsfr_gpu_rk4_step_dt(nsfr_gpu_ctx* ctx, double dt) {
  DeviceGuard dev_guard_(ctx);
  CK(cudaMemcpyAsync(&ctx->d_step->dt, &dt, sizeof dt, cudaMemcpyHostToDevice, ctx->st));
  if (int rc = ensure_projected(ctx)) return rc;
  if (int rc = enqueue_step(ctx, true)) return rc;
  return sync_check(ctx);
}

static int set_step_params(nsfr_gpu_ctx* ctx, double cfl, double t_final) {
  StepState* hs = ctx->h_step;
  CK(cudaMemcpyAsync(hs, ctx->d_step, sizeof(StepState), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  hs->cfl = cfl;
  hs->t_final = t_final;
  CK(cudaMemcpyAsync(ctx->d_step, hs, sizeof(StepState), cudaMemcpyHostToDevice, ctx->st));
  return NSFR_OK;
}

int nsfr_gpu_rk4_step(nsfr_gpu_ctx* ctx, double cfl, double t_final, double* dt_used) {
  DeviceGuard dev_guard_(ctx);
  if (int rc = set_step_params(ctx, cfl, t_final)) return rc;
  if (int rc = ensure_projected(ctx)) return rc;
  if (int rc = enqueue_step(ctx, false)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  if (dt_used) *dt_used = ctx->h_step->dt;
  return NSFR_OK;
}

int nsfr_gpu_advance(nsfr_gpu_ctx* ctx, int nsteps, double cfl, double t_final, double* t_out) {
  DeviceGuard dev_guard_(ctx);
  if (int rc = set_step_params(ctx, cfl, t_final)) return rc;
  if (int rc = ensure_projected(ctx)) return rc;
  if (!ctx->graph && !ctx->timing) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    const long long l0 = ctx->launches;
    int rc = enqueue_step(ctx, false);
    CK(cudaStreamEndCapture(ctx->st, &g));
    if (rc) return rc;
    CK(cudaGraphInstantiate(&ctx->graph, g, 0));
    cudaGraphDestroy(g);
    ctx->launches = l0;  // counted on replay
  }
  // with a final time, poll t every 16 steps (steps past t_final have dt = 0)
  const int chunk = t_final > 0.0 ? 16 : nsteps;
  for (int i = 0; i < nsteps; ++i) {
    if (ctx->timing) {
      if (int rc = enqueue_step(ctx, false)) return rc;
    } else {
      CK(cudaGraphLaunch(ctx->graph, ctx->st));
      ctx->launches += launches_per_step(ctx);
    }
    if (chunk < nsteps && (i + 1) % chunk == 0) {
      if (int rc = sync_check(ctx)) return rc;
      if (ctx->h_step->t >= t_final) break;
    }
  }
  if (int rc = sync_check(ctx)) return rc;
  if (t_out) *t_out = ctx->h_step->t;
  return NSFR_OK;
}

// ---- streamed host step (rk4 step on host buffers, copies overlapped) --------
// set_state(u_in); rk4 step; get_state(u_out) as ONE pipeline over contiguous
// element chunks (>= one z-plane each, so a chunk's face neighbours lie in the
// cyclically adjacent chunks). Per chunk the work is 9 layers: L0 = upload +
// chi^3 + K1, L(2s-1) = K2 of stage s, L(2s) = K3 of stage s (s = 1..4), then
// Pi^3 + download. Layer L of chunk c needs layer L-1 of c-1, c, c+1 (K2 reads
// the neighbours' traces; K3 overwrites them, so it also waits for the
// neighbours' K2). Chunks are visited outward from chunk 0 in cyclic distance
// r, layer L at wave r + L: every dependency was enqueued earlier on the one
// compute stream, the uploads run ahead on st_copy and the downloads trail on
// st_d2h, both directions of the PCIe link busy while the SMs compute. The
// upload lands in (and the download leaves from) the chunk's RK accumulator,
// dead outside stages 1-4 of that chunk. Adaptive dt needs lambda_max of the
// whole state before any K3: layers 0-1 form the first sweep, then dt, then
// layers 2-8 a second sweep.
namespace {

int streamed_chunks(const nsfr_gpu_ctx* ctx, std::vector<int>& bounds) {
  const long long plane = static_cast<long long>(ctx->m) * ctx->m;
  const long long min_sz = plane + 8;  // >= one plane after rounding down to 8
  const char* env = std::getenv("NSFR_STREAM_CHUNKS");
  const long long cap = env ? std::max(1, std::atoi(env)) : 128;
  int nch = static_cast<int>(std::min<long long>(cap, ctx->E / min_sz));
  nch = std::max(nch, 1);
  bounds.resize(nch + 1);
  for (int c = 0; c <= nch; ++c)
    bounds[c] = c == nch ? ctx->E : static_cast<int>((static_cast<long long>(ctx->E) * c / nch) & ~7LL);
  return nch;
}

}  // namespace

// dt_next (adaptive_dt of u_out): from the chunks' u_hat as they leave
int finish_dt_next(nsfr_gpu_ctx* ctx, double* dt_next) {
  if (ctx->comm)
    NK(ncclAllReduce(&ctx->d_step->lam_out_bits, &ctx->d_step->lam_out_bits, 1, ncclUint64, ncclMax,
                     ctx->comm, ctx->st));
  k_step_next<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  CK(cudaGetLastError());
  if (int rc = sync_check(ctx)) return rc;
  *dt_next = ctx->h_step->dt_next;
  return NSFR_OK;
}

static int rk4_step_host_impl(nsfr_gpu_ctx* ctx, const double* u_in, double* u_out, double dt,
                              double cfl, double t_final, double* dt_used, double* dt_next) {
  const bool fixed = dt > 0.0;
  // seg: a z-slab (or a 1-rank NCCL loopback) whose end planes take NCCL halos
  // instead of wrapping locally; external-halo contexts and DG do not stream
  const bool seg = ctx->d_halo_lo != nullptr;
  const bool streamable = !ctx->dg && (seg ? ctx->comm != nullptr : ctx->nranks == 1);
  if (!streamable) {  // external halos / DG: the same GPU path, transfers not overlapped
    if (int rc = nsfr_gpu_set_state(ctx, u_in)) return rc;
    double used = dt;
    if (fixed) {
      if (dt_next)  // cfl / t_final of the adaptive_dt that follows
        if (int rc = set_step_params(ctx, cfl, t_final)) return rc;
      if (int rc = nsfr_gpu_rk4_step_dt(ctx, dt)) return rc;
    } else if (int rc = nsfr_gpu_rk4_step(ctx, cfl, t_final, &used)) {
      return rc;
    }
    if (dt_used) *dt_used = used;
    if (int rc = nsfr_gpu_get_state(ctx, u_out)) return rc;
    if (!dt_next) return NSFR_OK;
    // get_state left u_hat of the whole slab in d_vol (NSFR); DG carries u_hat
    CK(cudaMemsetAsync(&ctx->d_step->lam_out_bits, 0, sizeof(unsigned long long), ctx->st));
    if (int rc = lam_of_uhat(ctx, ctx->dg ? ctx->d_un : ctx->d_vol, 0, ctx->E)) return rc;
    return finish_dt_next(ctx, dt_next);
  }
  std::vector<int> b;
  const int nch = streamed_chunks(ctx, b);
  if (int rc = ensure_chunk_events(ctx, 2 * nch)) return rc;
  if (!fixed || dt_next)
    if (int rc = set_step_params(ctx, cfl, t_final)) return rc;
  if (fixed) CK(cudaMemcpyAsync(&ctx->d_step->dt, &dt, sizeof dt, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));  // device buffers free, step parameters in place
  ctx->proj_valid = false;
  k_step_begin<<<1, 1, 0, ctx->st>>>(ctx->d_step);  // clears lambda
  ++ctx->launches;
  // Compute lanes: chunk c's ops run on lane c % S, waiting only for the
  // events of the neighbour-chunk ops they depend on, so one kernel's tail
  // overlaps the next independent kernel (NSFR_STREAM_LANES, default 4;
  // 128^3 p=4 chained e2e step: 1 lane 347 ms, 2-3 lanes 335 ms, 4 lanes 327 ms).
  const char* lenv = std::getenv("NSFR_STREAM_LANES");
  const int S = std::max(1, std::min(nch, lenv ? std::atoi(lenv) : 4));
  while (static_cast<int>(ctx->lanes.size()) < S) {
    cudaStream_t l;
    CK(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
    ctx->lanes.push_back(l);
  }
  const int nev = 9 * nch + 2 * S + 2 + 5;
  while (static_cast<int>(ctx->op_ev.size()) < nev) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->op_ev.push_back(e);
  }
  cudaStream_t main_st = ctx->st;
  struct Restore {
    nsfr_gpu_ctx* c;
    cudaStream_t s;
    ~Restore() { c->st = s; }
  } restore{ctx, main_st};
  // fork: the lanes start after the step parameters (main) are in place
  auto fork = [&](int slot) -> int {
    CK(cudaEventRecord(ctx->op_ev[9 * nch + slot], main_st));
    for (int k = 0; k < S; ++k) CK(cudaStreamWaitEvent(ctx->lanes[k], ctx->op_ev[9 * nch + slot], 0));
    return NSFR_OK;
  };
  // join: main waits for every lane
  auto join = [&](int slot) -> int {
    for (int k = 0; k < S; ++k) {
      CK(cudaEventRecord(ctx->op_ev[9 * nch + 2 + slot * S + k], ctx->lanes[k]));
      CK(cudaStreamWaitEvent(main_st, ctx->op_ev[9 * nch + 2 + slot * S + k], 0));
    }
    return NSFR_OK;
  };
  if (int rc = fork(0)) return rc;
  const size_t per = nsol(ctx) * NS;
  const bool nocopy = std::getenv("NSFR_STREAM_NOCOPY") != nullptr;  // probe: the compute schedule alone
  // Periodic box: chunks visited outward from chunk 0 in cyclic distance.
  // Slab: a segment whose two end chunks take halo planes, visited outward
  // from its middle chunk c0; before K2 of stage s reaches an end chunk, the
  // stage's grouped send/recv runs on the main stream once both end chunks
  // have projected (their K1 / K3 pack the send planes).
  const int c0 = seg ? nch / 2 : 0;
  const int D = seg ? std::max(c0, nch - 1 - c0) : nch / 2;
  auto at_dist = [&](int r, int* cs) {
    if (seg) {
      int k = 0;
      if (c0 - r >= 0) cs[k++] = c0 - r;
      if (r > 0 && c0 + r < nch) cs[k++] = c0 + r;
      return k;
    }
    if (r == 0) { cs[0] = 0; return 1; }
    cs[0] = r;
    if (nch - r == r) return 1;
    cs[1] = nch - r;
    return 2;
  };
  auto nbr = [&](int c, int d) {  // -1: a slab end (its neighbour is the halo)
    const int cn = c + d;
    if (seg) return (cn < 0 || cn >= nch) ? -1 : cn;
    return (cn + nch) % nch;
  };
  std::vector<char> done(9 * nch, 0);
  bool exchanged[5] = {false, false, false, false, false};
  const int ex_ev0 = 9 * nch + 2 * S + 2;
  // uploads, in the order the sweep consumes them
  for (int r = 0; r <= D; ++r) {
    int cs[2];
    const int k = at_dist(r, cs);
    for (int i = 0; i < k; ++i) {
      const int c = cs[i], e0 = b[c], e1 = b[c + 1];
      if (!nocopy)
        CK(cudaMemcpyAsync(ctx->d_acc + e0 * per, u_in + e0 * per, sizeof(double) * per * (e1 - e0),
                           cudaMemcpyHostToDevice, ctx->st_copy));
      CK(cudaEventRecord(ctx->chunk_ev[c], ctx->st_copy));
    }
  }
  auto layer_ops = [&](int L, int c) -> int {
    const int e0 = b[c], e1 = b[c + 1];
    if (L == 0) {
      CK(cudaStreamWaitEvent(ctx->st, ctx->chunk_ev[c], 0));
      if (nocopy) {  // same conversion cost, the device state stays the input
        if (int rc = convert_range(ctx, ctx->d_un, ctx->d_rhs, true, e0, e1)) return rc;
        return project(ctx, ctx->d_un, !fixed, e0, e1);
      }
      // K1 straight from the uploaded u_hat: u_q = chi^3 u_hat into the state and projected
      return project(ctx, ctx->d_acc, !fixed, e0, e1, ctx->d_un);
    }
    const int stage = (L + 1) / 2;
    if (L & 1) return residual(ctx, 0, e0, e1);
    if (stage < 4) return update(ctx, stage, false, nullptr, e0, e1);
    // stage 4: u_{n+1} of this chunk is final; K3 writes Pi^3 u_{n+1} into the
    // dead accumulator (and adaptive_dt's lambda of exactly those bytes)
    // instead of projecting it, then the download
    if (int rc = update(ctx, 4, false, nullptr, e0, e1, ctx->d_acc,
                        dt_next ? &ctx->d_step->lam_out_bits : nullptr))
      return rc;
    CK(cudaEventRecord(ctx->chunk_ev[nch + c], ctx->st));
    CK(cudaStreamWaitEvent(ctx->st_d2h, ctx->chunk_ev[nch + c], 0));
    if (!nocopy)
      CK(cudaMemcpyAsync(u_out + e0 * per, ctx->d_acc + e0 * per, sizeof(double) * per * (e1 - e0),
                       cudaMemcpyDeviceToHost, ctx->st_d2h));
    return NSFR_OK;
  };
  auto layer = [&](int L, int c) -> int {
    cudaStream_t lane = ctx->lanes[c % S];
    if (L > 0)  // layer L-1 of the neighbour chunks (same-lane ops are in order already)
      for (int d = -1; d <= 1; d += 2) {
        const int cn = nbr(c, d);
        if (cn < 0 || cn % S == c % S) continue;
        if (!done[(L - 1) * nch + cn]) {
          ctx->msg = "streamed step: schedule out of order";
          return NSFR_E_DIM;
        }
        CK(cudaStreamWaitEvent(lane, ctx->op_ev[(L - 1) * nch + cn], 0));
      }
    if (seg && (L & 1) && (c == 0 || c == nch - 1)) {  // K2 of stage s at a slab end: halos first
      const int st = (L + 1) / 2;
      if (!exchanged[st]) {
        if (!done[(L - 1) * nch] || !done[(L - 1) * nch + nch - 1]) {
          ctx->msg = "streamed step: halo exchange before the end chunks projected";
          return NSFR_E_DIM;
        }
        CK(cudaStreamWaitEvent(main_st, ctx->op_ev[(L - 1) * nch], 0));
        CK(cudaStreamWaitEvent(main_st, ctx->op_ev[(L - 1) * nch + nch - 1], 0));
        if (int rc = exchange(ctx)) return rc;  // on ctx->st == main_st
        CK(cudaEventRecord(ctx->op_ev[ex_ev0 + st], main_st));
        exchanged[st] = true;
      }
      CK(cudaStreamWaitEvent(lane, ctx->op_ev[ex_ev0 + st], 0));
    }
    ctx->st = lane;
    const int rc = layer_ops(L, c);
    ctx->st = main_st;
    if (rc) return rc;
    CK(cudaEventRecord(ctx->op_ev[L * nch + c], lane));
    done[L * nch + c] = 1;
    return NSFR_OK;
  };
  auto sweep = [&](int La, int Lb) -> int {
    for (int w = 0; w <= D + (Lb - La); ++w)
      for (int L = La; L <= Lb; ++L) {
        const int r = w - (L - La);
        if (r < 0 || r > D) continue;
        int cs[2];
        const int k = at_dist(r, cs);
        for (int i = 0; i < k; ++i)
          if (int rc = layer(L, cs[i])) return rc;
      }
    return NSFR_OK;
  };
  if (fixed) {
    if (int rc = sweep(0, 8)) return rc;
  } else {
    if (int rc = sweep(0, 1)) return rc;
    if (int rc = join(0)) return rc;
    if (ctx->comm)
      NK(ncclAllReduce(&ctx->d_step->lam_bits, &ctx->d_step->lam_bits, 1, ncclUint64, ncclMax, ctx->comm,
                       ctx->st));
    k_step_dt<<<1, 1, 0, ctx->st>>>(ctx->d_step);  // reads and clears lambda
    ++ctx->launches;
    if (int rc = fork(1)) return rc;
    if (int rc = sweep(2, 8)) return rc;
  }
  if (int rc = join(1)) return rc;
  k_step_end<<<1, 1, 0, ctx->st>>>(ctx->d_step);
  ++ctx->launches;
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->st_d2h));
  CK(cudaStreamSynchronize(ctx->st_copy));
  if (int rc = sync_check(ctx)) return rc;
  ctx->proj_valid = false;  // K3 of stage 4 wrote u_hat instead of projecting u_{n+1}
  if (dt_used) *dt_used = ctx->h_step->dt;
  return dt_next ? finish_dt_next(ctx, dt_next) : NSFR_OK;
}

int nsfr_gpu_rk4_step_host(nsfr_gpu_ctx* ctx, const double* u_in, double* u_out, double dt,
                           double cfl, double t_final, double* dt_used, double* dt_next) {
  DeviceGuard dev_guard_(ctx);
  if (!ctx) return NSFR_E_DIM;
  if (!u_in || !u_out) {
    ctx->msg = "rk4_step_host: null state buffer";
    return NSFR_E_DIM;
  }
  const int rc = rk4_step_host_impl(ctx, u_in, u_out, dt, cfl, t_final, dt_used, dt_next);
  if (rc) {  // a failure mid-pipeline: let every stream drain before the context is reused
    for (auto l : ctx->lanes) cudaStreamSynchronize(l);
    if (ctx->st_copy) cudaStreamSynchronize(ctx->st_copy);
    if (ctx->st_d2h) cudaStreamSynchronize(ctx->st_d2h);
    cudaStreamSynchronize(ctx->st);
    ctx->proj_valid = false;
  }
  return rc;
}

int nsfr_gpu_l2_error(nsfr_gpu_ctx* ctx, int kind, double out2[2]) {
  DeviceGuard dev_guard_(ctx);
  const int g = ctx->tab.g, n = ctx->NQ, G3 = g * g * g, N3 = n * n * n;
  const int M = std::max(g, n), M3 = M * M * M;
  const size_t smem = sizeof(double) * (3 * G3 + 2 * M3 + 10 * N3);
  if (int rc = setup_kernel_smem(ctx, smem, (const void*)k_l2)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  if (ctx->dg)  // u at the quadrature nodes: chi^3 u_hat into the scratch
    if (int rc = convert_state(ctx, ctx->d_un, ctx->d_vol, true)) return rc;
  L2Params P{};
  P.tab = ctx->d_tab;
  P.u = ctx->dg ? ctx->d_vol : ctx->d_un;
  P.jac = ctx->d_jac;
  P.part = ctx->d_part;
  P.E = ctx->E;
  P.m = ctx->m;
  P.k0 = ctx->k0;
  P.kind = kind;
  P.x_left = ctx->s.x_left;
  P.h = (ctx->s.x_right - ctx->s.x_left) / ctx->m;
  P.beta = ctx->s.beta;
  P.l = length_scale(ctx->s);
  P.gamma = ctx->s.gamma;
  P.t = ctx->h_step->t;
  k_l2<<<ctx->E, 128, smem, ctx->st>>>(P);
  k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_part, ctx->E, 2, ctx->d_red);
  ctx->launches += 2;
  if (int rc = allreduce_sum(ctx, ctx->d_red, 2)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  double h[2];
  CK(copy_sync(ctx->st, h, ctx->d_red, sizeof h, cudaMemcpyDeviceToHost));
  out2[0] = std::sqrt(h[0]);
  out2[1] = std::sqrt(h[1]);
  return NSFR_OK;
}

// mass, momentum, energy and entropy-function totals of the current state
static int totals(nsfr_gpu_ctx* ctx, double out6[NTOT]) {
  if (int rc = sync_check(ctx)) return rc;
  // u_q (DG: chi^3 u_hat into d_vol); per-element partials into d_acc (dead
  // between steps), then fixed-order sums
  if (ctx->dg)
    if (int rc = convert_state(ctx, ctx->d_un, ctx->d_vol, true)) return rc;
  k_totals<<<ctx->E, 128, 0, ctx->st>>>(ctx->d_tab, ctx->dg ? ctx->d_vol : ctx->d_un, ctx->d_jac,
                                         ctx->s.gamma, ctx->d_acc, ctx->E);
  k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_acc, ctx->E, NTOT, ctx->d_red);
  ctx->launches += 2;
  CK(cudaGetLastError());
  if (int rc = allreduce_sum(ctx, ctx->d_red, NTOT)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  CK(copy_sync(ctx->st, out6, ctx->d_red, sizeof(double) * NTOT, cudaMemcpyDeviceToHost));
  return NSFR_OK;
}

// ---- external halo mode (nranks > 1, no NCCL id): the caller moves the planes
int nsfr_gpu_halo_buffers(nsfr_gpu_ctx* ctx, double** send_lo, double** send_hi, double** recv_lo,
                          double** recv_hi) {
  DeviceGuard dev_guard_(ctx);
  *send_lo = ctx->d_send_lo;
  *send_hi = ctx->d_send_hi;
  *recv_lo = ctx->d_halo_lo;
  *recv_hi = ctx->d_halo_hi;
  return NSFR_OK;
}

int nsfr_gpu_halo_get(nsfr_gpu_ctx* ctx, double* send_lo, double* send_hi) {
  DeviceGuard dev_guard_(ctx);
  if (!ctx->d_send_lo) {
    ctx->msg = "halo_get: single-rank context has no halo planes";
    return NSFR_E_CONFIG;
  }
  const size_t b = sizeof(double) * ctx->halo_count;
  CK(cudaMemcpyAsync(send_lo, ctx->d_send_lo, b, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaMemcpyAsync(send_hi, ctx->d_send_hi, b, cudaMemcpyDeviceToHost, ctx->st));
  return sync_check(ctx);
}

int nsfr_gpu_halo_set(nsfr_gpu_ctx* ctx, const double* recv_lo, const double* recv_hi) {
  DeviceGuard dev_guard_(ctx);
  if (!ctx->d_halo_lo) {
    ctx->msg = "halo_set: single-rank context has no halo planes";
    return NSFR_E_CONFIG;
  }
  const size_t b = sizeof(double) * ctx->halo_count;
  CK(cudaMemcpyAsync(ctx->d_halo_lo, recv_lo, b, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaMemcpyAsync(ctx->d_halo_hi, recv_hi, b, cudaMemcpyHostToDevice, ctx->st));
  return sync_check(ctx);
}

int nsfr_gpu_project(nsfr_gpu_ctx* ctx) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) {
    ctx->msg = "project: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  if (int rc = project_state(ctx)) return rc;
  return sync_check(ctx);
}

int nsfr_gpu_residual(nsfr_gpu_ctx* ctx, double* dudt, double* entropy_change) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) {
    ctx->msg = "residual: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  const bool ent = entropy_change != nullptr;
  if (ent && !ctx->d_vhat) {
    ctx->msg = "entropy change needs setup.entropy_diag = 1";
    return NSFR_E_CONFIG;
  }
  if (!ctx->proj_valid) {
    ctx->msg = "residual: no projection of the current state (call nsfr_gpu_project)";
    return NSFR_E_CONFIG;
  }
  if (int rc = exchange(ctx)) return rc;
  if (int rc = residual(ctx)) return rc;
  if (int rc = update(ctx, 0, ent)) return rc;
  if (ent) {
    k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_dS, ctx->E, 1, ctx->d_red);
    ++ctx->launches;
    if (int rc = allreduce_sum(ctx, ctx->d_red, 1)) return rc;
  }
  if (int rc = sync_check(ctx)) return rc;
  if (dudt) CK(copy_sync(ctx->st, dudt, ctx->d_rhs, sizeof(double) * state_count(ctx), cudaMemcpyDeviceToHost));
  if (ent) CK(copy_sync(ctx->st, entropy_change, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost));
  return NSFR_OK;
}

int nsfr_gpu_stage(nsfr_gpu_ctx* ctx, int stage, double dt) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) {
    ctx->msg = "stage: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  if (stage < 1 || stage > 4) {
    ctx->msg = "stage must be 1..4";
    return NSFR_E_DIM;
  }
  if (!ctx->proj_valid) {
    ctx->msg = "stage: no projection of the stage state (call nsfr_gpu_project first)";
    return NSFR_E_CONFIG;
  }
  if (stage == 1) {
    CK(cudaMemcpyAsync(&ctx->d_step->dt, &dt, sizeof dt, cudaMemcpyHostToDevice, ctx->st));
    k_step_begin<<<1, 1, 0, ctx->st>>>(ctx->d_step);  // lambda of u_{n+1} accumulates in stage 4
    ++ctx->launches;
  }
  if (int rc = exchange(ctx)) return rc;
  if (int rc = residual(ctx)) return rc;
  if (int rc = update(ctx, stage, false)) return rc;
  if (stage == 4) {
    k_step_end<<<1, 1, 0, ctx->st>>>(ctx->d_step);
    ++ctx->launches;
  }
  return sync_check(ctx);
}

int nsfr_gpu_conserved_totals(nsfr_gpu_ctx* ctx, double out5[5]) {
  DeviceGuard dev_guard_(ctx);
  double t[NTOT];
  if (int rc = totals(ctx, t)) return rc;
  for (int s = 0; s < NS; ++s) out5[s] = t[s];
  return NSFR_OK;
}

int nsfr_gpu_entropy_total(nsfr_gpu_ctx* ctx, double* out) {
  DeviceGuard dev_guard_(ctx);
  double t[NTOT];
  if (int rc = totals(ctx, t)) return rc;
  *out = t[NS];
  return NSFR_OK;
}

int nsfr_gpu_ke_volume(nsfr_gpu_ctx* ctx, double* out) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) {
    ctx->msg = "ke_volume: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  // volume rows of (flux - pressure work) for the projection of u_n, then
  // sum v_KE . rows; partials go to d_rhs (the rows occupy d_vol)
  if (int rc = project_state(ctx)) return rc;
  if (int rc = residual(ctx, 1)) return rc;
  k_ke_dot<<<ctx->E, 128, 0, ctx->st>>>(ctx->d_un, ctx->d_vol, static_cast<int>(nsol(ctx)), ctx->d_rhs,
                                         ctx->E);
  k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_rhs, ctx->E, 1, ctx->d_red);
  ctx->launches += 2;
  CK(cudaGetLastError());
  if (int rc = allreduce_sum(ctx, ctx->d_red, 1)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  CK(copy_sync(ctx->st, out, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost));
  return NSFR_OK;
}

int nsfr_gpu_ke_total(nsfr_gpu_ctx* ctx, double* out) {
  DeviceGuard dev_guard_(ctx);
  if (ctx->dg) {
    ctx->msg = "ke_total: defined for the NSFR scheme only";
    return NSFR_E_CONFIG;
  }
  // rows of (flux - pressure work) everywhere, no Roe (K2 km = 2); v_hat_KE =
  // Pi^3 v_KE(u_q) into d_acc (dead between steps); K3's diagnostic path forms
  // R = chi^T-lifted rows and -v_hat_KE . R per element
  if (int rc = project_state(ctx)) return rc;
  if (int rc = exchange(ctx)) return rc;
  if (int rc = residual(ctx, 2)) return rc;
  const size_t smem = sizeof(double) * 4 * nsol(ctx);
  k_ke_vars<<<ctx->E, 128, smem, ctx->st>>>(ctx->d_tab, ctx->d_un, ctx->d_acc, ctx->E);
  ++ctx->launches;
  CK(cudaGetLastError());
  if (int rc = update(ctx, 0, true, ctx->d_acc)) return rc;
  k_reduce<<<1, 1024, 0, ctx->st>>>(ctx->d_dS, ctx->E, 1, ctx->d_red);
  ++ctx->launches;
  if (int rc = allreduce_sum(ctx, ctx->d_red, 1)) return rc;
  if (int rc = sync_check(ctx)) return rc;
  CK(copy_sync(ctx->st, out, ctx->d_red, sizeof(double), cudaMemcpyDeviceToHost));
  return NSFR_OK;
}

double* nsfr_gpu_state_device_ptr(nsfr_gpu_ctx* ctx) { return ctx->d_un; }
size_t nsfr_gpu_state_count(const nsfr_gpu_ctx* ctx) { return state_count(ctx); }
int nsfr_gpu_sync(nsfr_gpu_ctx* ctx) {
  DeviceGuard dev_guard_(ctx);
  return sync_check(ctx);
}
long long nsfr_gpu_launch_count(const nsfr_gpu_ctx* ctx) { return ctx->launches; }

// Bench helper: time `nsteps` RK4 steps with CUDA events on the context
// stream. With kernel_ms != NULL each K1/K2 launch is bracketed by events and
// kernel_ms[0]/[1]/[2] receive the summed K1/K2/K3 durations (ms).
int nsfr_gpu_time_steps(nsfr_gpu_ctx* ctx, int nsteps, double cfl, double* step_ms,
                        double* kernel_ms) {
  DeviceGuard dev_guard_(ctx);
  if (int rc = set_step_params(ctx, cfl, 0.0)) return rc;
  if (!kernel_ms && !ctx->graph) {
    if (int rc = nsfr_gpu_advance(ctx, 0, cfl, 0.0, nullptr)) return rc;  // capture the step graph
  }
  if (int rc = ensure_projected(ctx)) return rc;
  ctx->timing = kernel_ms != nullptr;
  ctx->ev_marks.clear();
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, ctx->st));
  int rc = NSFR_OK;
  for (int i = 0; i < nsteps && !rc; ++i) {
    if (ctx->timing) {
      rc = enqueue_step(ctx, false);
    } else {
      CK(cudaGraphLaunch(ctx->graph, ctx->st));
      ctx->launches += launches_per_step(ctx);
    }
  }
  CK(cudaEventRecord(b, ctx->st));
  if (!rc) rc = sync_check(ctx);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, b));
  *step_ms = ms;
  if (kernel_ms) {
    kernel_ms[0] = kernel_ms[1] = kernel_ms[2] = 0.0;
    for (auto& mk : ctx->ev_marks) {
      float x = 0.f;
      cudaEventElapsedTime(&x, ctx->ev_pool[mk.second], ctx->ev_pool[mk.second + 1]);
      kernel_ms[mk.first - 1] += x;
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    ctx->ev_pool.clear();
    ctx->ev_marks.clear();
  }
  ctx->timing = false;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return rc;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP64 pipe peak (roofline denominator; MEASURED_PEAKS.json carries none):
// independent DFMA chains on every SM, best of 5, CUDA events.
namespace {
// Each CTA's thread 0 records its SM clock64 span: cycles / event time is the
// SM clock the DFMA loop actually ran at (roofline nominal = 148 x 128 x f).
__global__ void k_dfma_peak(double* out, long long* cycles, int iters, double a, double b) {
  const long long c0 = clock64();
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  __syncthreads();
  if (threadIdx.x == 0 && cycles) cycles[blockIdx.x] = clock64() - c0;
}
}  // namespace

extern "C" int nsfr_gpu_measure_fp64_peak_ex(int device, double* tflops, double* sm_mhz) {
  DeviceGuard dev_guard_(device);
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) return NSFR_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int threads = 256, blocks = sms * 8, iters = 2048;
  double* out = nullptr;
  long long* cyc = nullptr;
  if (cudaMalloc(&out, sizeof(double) * threads * blocks) != cudaSuccess) return NSFR_E_CUDA;
  if (cudaMalloc(&cyc, sizeof(long long) * blocks) != cudaSuccess) {
    cudaFree(out);
    return NSFR_E_CUDA;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_dfma_peak<<<blocks, threads>>>(out, nullptr, 64, 0.999999, 1e-7);
  float best = 1e30f;
  double mhz = 0.0;
  std::vector<long long> hc(blocks);
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_dfma_peak<<<blocks, threads>>>(out, cyc, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) {
      best = ms;
      // all CTAs are co-resident (8 per SM): the longest CTA span ~ the kernel
      cudaMemcpy(hc.data(), cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
      const long long mx = *std::max_element(hc.begin(), hc.end());
      mhz = mx / (ms * 1e3);
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(cyc);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return NSFR_E_CUDA;
  *tflops = 2.0 * 8 * 16 * (double)iters * threads * blocks / (best * 1e-3) / 1e12;
  if (sm_mhz) *sm_mhz = mhz;
  return NSFR_OK;
}

extern "C" int nsfr_gpu_measure_fp64_peak(int device, double* tflops) {
  return nsfr_gpu_measure_fp64_peak_ex(device, tflops, nullptr);
}

#ifdef NSFR_PHASE_PROF
// Development only: read and reset the K2 phase cycle counters.
extern "C" int nsfr_gpu_phase_counters(double* out16) {
  unsigned long long h[16];
  if (cudaMemcpyFromSymbol(h, g_phase_cycles, sizeof h) != cudaSuccess) return NSFR_E_CUDA;
  for (int i = 0; i < 16; ++i) out16[i] = static_cast<double>(h[i]);
  const unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  return NSFR_OK;
}
#endif
