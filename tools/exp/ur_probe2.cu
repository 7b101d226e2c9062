#include <cuda_runtime.h>
__device__ __forceinline__ double ldu64(const double* p) {
  double v; asm volatile("ldu.global.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}
extern "C" __global__ void k_ldu(double* out, const double2* __restrict__ g, int n) {
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double* p = (const double*)&g[(b & 31) * 16 + i];
      double2 c; c.x = ldu64(p); c.y = ldu64(p + 1);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
__device__ __forceinline__ double red64(double v) {
  unsigned lo = __double2loint(v), hi = __double2hiint(v);
  lo = __reduce_or_sync(0xffffffffu, lo); hi = __reduce_or_sync(0xffffffffu, hi);
  return __hiloint2double(hi, lo);
}
extern "C" __global__ void k_redux(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double2 c = sm[(b & 31) * 16 + i];
      c.x = red64(c.x); c.y = red64(c.y);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
__device__ __forceinline__ unsigned vshfl(unsigned v) {
  unsigned r; asm volatile("shfl.sync.idx.b32 %0, %1, 0, 31, 0xffffffff;" : "=r"(r) : "r"(v)); return r;
}
extern "C" __global__ void k_vshfl(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double2 c = sm[((b & 31) * 16 + i) * 32 + (threadIdx.x & 31)];
      c.x = __hiloint2double(vshfl(__double2hiint(c.x)), vshfl(__double2loint(c.x)));
      c.y = __hiloint2double(vshfl(__double2hiint(c.y)), vshfl(__double2loint(c.y)));
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
