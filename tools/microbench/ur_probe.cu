// Which code shapes make ptxas feed the rotation's warp-uniform multiplier to DFMA from a
// uniform register (DFMA R, R, UR, R issues at the full FP64 rate; three vector-register
// operands cap it at 2/3, dfma_operands.cu)? Compile-only probe:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -cubin -o ur_probe.cubin ur_probe.cu
//   cuobjdump -sass -fun k_const ur_probe.cubin | grep -E "DFMA|LDCU|LDS|REDUX|R2UR|SHFL|MOV"
// Findings (CUDA 12.9): only constant-bank data (k_const: LDCU.64 -> DFMA R, R, UR, R) gets
// there. Shared / global loads with a uniform address stay in vector registers (k_lds,
// k_ldg, k_ldu); a shfl broadcast of such a value is elided (k_shfl) or, when volatile,
// stays a vector SHFL (k_vshfl); __reduce_or_sync does produce REDUX.OR UR, R but ptxas
// copies the uniform registers back to vector ones before the DFMAs (k_redux, k_redux64).
#include <cuda_runtime.h>
#include <cstdio>
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
__device__ __forceinline__ double red64b(double v) {
  unsigned long long b = __double_as_longlong(v);
  unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)b), hi = __reduce_or_sync(0xffffffffu, (unsigned)(b >> 32));
  unsigned long long o = ((unsigned long long)hi << 32) | lo;
  return __longlong_as_double(o);
}
extern "C" __global__ void __launch_bounds__(384, 1) k_redux64(double* out, int n) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double x0 = threadIdx.x, y0 = 1.0, x1 = 2.0 * threadIdx.x, y1 = 3.0;
  for (int b = 0; b < n; ++b) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double2 c = sm[(b & 31) * 16 + i];
      c.x = red64b(c.x); c.y = red64b(c.y);
      double xo = x0; x0 = fma(c.x, y0, x0); y0 = fma(c.y, xo, y0);
      xo = x1; x1 = fma(c.x, y1, x1); y1 = fma(c.y, xo, y1);
    }
  }
  out[threadIdx.x] = x0 + y0 + x1 + y1;
}
