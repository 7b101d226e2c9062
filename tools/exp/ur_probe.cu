#include <cuda_runtime.h>
#include <cstdio>
// Which code shapes make ptxas feed a warp-uniform multiplier to DFMA from a uniform register?
extern "C" __global__ void k_lds(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 c = sm[(b & 31) * 16 + i];
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
extern "C" __global__ void k_ldg(double* out, const double2* __restrict__ g, int n) {
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 c = __ldg(&g[(b & 31) * 16 + i]);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
__constant__ double2 cc[2048];
extern "C" __global__ void k_const(double* out, int n) {
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 c = cc[(b & 31) * 16 + i];
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
__device__ __forceinline__ double bcast(double v) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  lo = __shfl_sync(0xffffffffu, lo, 0); hi = __shfl_sync(0xffffffffu, hi, 0);
  return __hiloint2double(hi, lo);
}
extern "C" __global__ void k_shfl(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double2 c = sm[(b & 31) * 16 + i];
      c.x = bcast(c.x); c.y = bcast(c.y);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
