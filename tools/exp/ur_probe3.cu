#include <cuda_runtime.h>
__device__ __forceinline__ double red64(double v) {
  unsigned long long b = __double_as_longlong(v);
  unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)b), hi = __reduce_or_sync(0xffffffffu, (unsigned)(b >> 32));
  unsigned long long o = ((unsigned long long)hi << 32) | lo;
  return __longlong_as_double(o);
}
extern "C" __global__ void __launch_bounds__(384, 1) k_redux(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double2 c = sm[(b & 31) * 16 + i];
      c.x = red64(c.x); c.y = red64(c.y);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
