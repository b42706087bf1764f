// sm_100a fp64 kernels of the NSFR per-stage residual (umbrella header).
//   setup_kernels.cuh   metric build, initial state, L2 partials, reductions, step bookkeeping
//   kernel_project.cuh  K1: entropy projection + face traces (+ lambda_max)
//   kernel_residual.cuh K2: Hadamard volume/surface, EC+Roe faces, lift, WA inverse, RK stage
#pragma once
#include "kernel_residual.cuh"
