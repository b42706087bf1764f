// sm_100a fp64 kernels of the NSFR per-stage residual (umbrella header).
//   setup_kernels.cuh   metric build, initial state, L2 partials, reductions, step bookkeeping
//   kernel_project.cuh  K1: entropy projection + face traces (+ lambda_max); prologue only
//   kernel_residual.cuh K2: Hadamard volume/surface pairs, EC+Roe faces -> volume/face rows
//   kernel_update.cuh   K3: lift, WA inverse, RK stage update + projection of the next stage
//   kernel_dg.cuh       conservative strong-form DG: KD1 face states, KD2 residual
//   kernel_convert.cuh  u_hat <-> u_q conversion of the host transfers (line passes)
#pragma once
#include "kernel_project.cuh"
#include "kernel_residual.cuh"
#include "kernel_update.cuh"
#include "kernel_dg.cuh"
#include "kernel_convert.cuh"
