// FP64 / FP32 pipe microbenchmarks for the roofline denominators (DFMA, FFMA peaks).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void fma_tput(T* out, int iters, T a, T b) {
  T acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == (T)12345.678) out[0] = s;
}
template <typename T>
__global__ void fma_lat(T* out, int iters, T a, T b, long long* cyc) {
  T x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
template <typename T, int CH>
double run_tput(int blocks, int threads, int iters) {
  T* o; cudaMalloc(&o, 64);
  fma_tput<T, CH><<<blocks, threads>>>(o, iters, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_tput<T, CH><<<blocks, threads>>>(o, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * CH * (double)iters * blocks * threads;
  cudaFree(o);
  return flops / (ms * 1e-3) / 1e12;
}
int main(int argc, char** argv) {
  if (argc > 1) {  // sustained: back-to-back launches for ~N seconds
    double* o; cudaMalloc(&o, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = atoi(argv[1]);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) fma_tput<double, 8><<<148 * 8, 256>>>(o, 20000, 0.999, 0.001);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("sustained DFMA over %.1f ms: %.2f TF/s\n", ms, 2.0 * 8 * 20000.0 * 148 * 8 * 256 * reps / (ms * 1e-3) / 1e12);
    return 0;
  }
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sms = p.multiProcessorCount;
  for (int occ : {1, 2, 4, 8}) {
    printf("f64 DFMA tput occ=%d threads=256 ch=8: %.2f TF/s\n", occ, run_tput<double, 8>(sms * occ, 256, 20000));
  }
  printf("f64 DFMA tput occ=4 ch=4: %.2f TF/s\n", run_tput<double, 4>(sms * 4, 256, 20000));
  printf("f64 DFMA tput occ=2 ch=16 t=128: %.2f TF/s\n", run_tput<double, 16>(sms * 2, 128, 20000));
  printf("f64 DFMA tput 1 warp/SMSP ch=8: %.2f TF/s\n", run_tput<double, 8>(sms, 128, 20000));
  printf("f64 DFMA tput 1 warp/SMSP ch=16: %.2f TF/s\n", run_tput<double, 16>(sms, 128, 20000));
  for (int occ : {2, 4, 8})
    printf("f32 FFMA tput occ=%d ch=8: %.2f TF/s\n", occ, run_tput<float, 8>(sms * occ, 256, 40000));
  double* od; long long* cy; cudaMalloc(&od, 64); cudaMalloc(&cy, 8);
  fma_lat<double><<<1, 32>>>(od, 100000, 0.999, 0.001, cy); cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", c / 100000.0);
  float* of; cudaMalloc(&of, 64);
  fma_lat<float><<<1, 32>>>(of, 100000, 0.999f, 0.001f, cy); cudaDeviceSynchronize();
  cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", c / 100000.0);
  return 0;
}
