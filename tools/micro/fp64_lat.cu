// FP64 pipe latency / throughput microbenchmarks on sm_100a (dev tool):
// dependent-chain latency of DFMA, DMUL, DADD, MUFU.RCP64H (rcp.approx.ftz.f64),
// LDS.64, and DFMA issue throughput vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcpa(double y) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  return r;
}

template <int OP>
__global__ void k_lat(double* out, long long* cyc, int n, double a, double b) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = 0.0;
  __syncthreads();
  double x = a + threadIdx.x * 1e-300;
  int idx = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = fma(x, a, b);
      if (OP == 1) x = x * a;
      if (OP == 2) x = x + b;
      if (OP == 3) x = rcpa(x);
      if (OP == 4) { idx = (int)sm[idx & 63]; }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + idx;
}

__global__ void k_tput(double* out, long long* cyc, int n, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <int ILP>
__global__ void k_ilp(double* out, long long* cyc, int n, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int j = 0; j < ILP; ++j) x[j] = fma(x[j], a, b);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  long long h[1024];
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RCP64H", "LDS.64(dep)"};
  const int n = 4096;
  for (int op = 0; op < 5; ++op) {
    void (*k)(double*, long long*, int, double, double) =
        op == 0 ? k_lat<0> : op == 1 ? k_lat<1> : op == 2 ? k_lat<2> : op == 3 ? k_lat<3> : k_lat<4>;
    k<<<1, 32>>>(out, cyc, 16, 0.999999, 1e-7);
    k<<<1, 32>>>(out, cyc, n, 0.999999, 1e-7);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"op\": \"%s\", \"latency_cycles\": %.2f}\n", names[op], h[0] / (16.0 * n));
  }
  // DFMA issue throughput: warps per SM 1..32, one block per SM (148 blocks)
  for (int w : {1, 2, 4, 8, 12, 16, 24, 32}) {
    k_tput<<<148, 32 * w>>>(out, cyc, 16, 0.999999, 1e-7);
    k_tput<<<148, 32 * w>>>(out, cyc, 1024, 0.999999, 1e-7);
    cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double dfma_per_sm = 8.0 * 8 * 1024 * 32 * w;
    printf("{\"warps_per_sm\": %d, \"ilp\": 8, \"dfma_lanes_per_clk_per_sm\": %.2f}\n", w, dfma_per_sm / mx);
  }
  // DFMA throughput vs warps per SM at ILP 1 / 2 / 4 (dependent chains per thread)
  for (int ilp : {1, 2, 4}) {
    for (int w : {4, 8, 12, 16, 20, 24, 32}) {
      auto k = ilp == 1 ? k_ilp<1> : ilp == 2 ? k_ilp<2> : k_ilp<4>;
      k<<<148, 32 * w>>>(out, cyc, 16, 0.999999, 1e-7);
      k<<<148, 32 * w>>>(out, cyc, 512, 0.999999, 1e-7);
      cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("{\"warps_per_sm\": %d, \"ilp\": %d, \"dfma_lanes_per_clk_per_sm\": %.2f}\n", w, ilp,
             16.0 * 512 * ilp * 32 * w / mx);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
