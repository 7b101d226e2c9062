// Prototype: one band of K sweeps, register window of K+1 columns per row, R rows per thread.
// Measures steady-state rotation throughput (triangle lanes use identity coefs; timing only).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
template <int K, int R, int CMODE>
__global__ void __launch_bounds__(128) proto(double* __restrict__ A, int m, int n, long lda,
                                             const double2* __restrict__ coef, int nwaves) {
  __shared__ double2 sc[2][32 * K];
  const int lane = threadIdx.x & 31;
  const long rbase = ((long)blockIdx.x * blockDim.x / 32 + threadIdx.x / 32) * 32 * R + lane;
  double w[R][K + 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int s = 0; s < K + 1; ++s) w[r][s] = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) w[r][0] = A[rbase + r * 32];
  for (int t0 = 0; t0 < nwaves; t0 += K + 1) {
    if (CMODE == 1) {
      // stage 32 waves... simple: each warp stages K+1 waves of coefs into its own smem (warp-private)
      __syncwarp();
      for (int i = lane; i < (K + 1) * K; i += 32) sc[0][(threadIdx.x / 32) * 0 + i] = coef[(long)t0 * K + i];
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < K + 1; ++u) {
      const int t = t0 + u;
      const int cin = t + 1;
      const int sin_ = (u + 1) % (K + 1);
#pragma unroll
      for (int r = 0; r < R; ++r) w[r][sin_] = (cin < n) ? A[rbase + r * 32 + (long)cin * lda] : 0.0;
#pragma unroll
      for (int l = 0; l < K; ++l) {
        double2 cs = (CMODE == 0) ? __ldg(&coef[(long)t * K + l]) : sc[0][u * K + l];
        const int sx = ((u - l) % (K + 1) + (K + 1)) % (K + 1);
        const int sy = (sx + 1) % (K + 1);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double x = w[r][sx], y = w[r][sy];
          double cx = cs.x * x, sx_ = cs.y * x;
          w[r][sx] = fma(cs.y, y, cx);
          w[r][sy] = fma(cs.x, y, -sx_);
        }
      }
      const int cout = t - K + 1;
      const int sout = ((u - K + 1) % (K + 1) + (K + 1)) % (K + 1);
      if (cout >= 0 && cout < n) {
#pragma unroll
        for (int r = 0; r < R; ++r) A[rbase + r * 32 + (long)cout * lda] = w[r][sout];
      }
    }
  }
}
template <int K, int R, int CMODE>
void run(int m, int n) {
  long lda = m;
  double* A; cudaMalloc(&A, sizeof(double) * lda * n);
  cudaMemset(A, 0, sizeof(double) * lda * n);
  int nwaves = n + K - 1;
  int nwp = ((nwaves + K) / (K + 1)) * (K + 1);
  std::vector<double2> h((size_t)nwp * K);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(0.6, 0.8);
  double2* c; cudaMalloc(&c, h.size() * 16);
  cudaMemcpy(c, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  int threads = 128;
  int blocks = m / (R * threads);
  proto<K, R, CMODE><<<blocks, threads>>>(A, m, n, lda, c, nwaves);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  int reps = 5;
  for (int i = 0; i < reps; ++i) proto<K, R, CMODE><<<blocks, threads>>>(A, m, n, lda, c, nwaves);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  double fl = 6.0 * m * (n - 1.0) * K;
  printf("K=%2d R=%d cmode=%d m=%d n=%d: %.3f ms  %.2f TF/s  err=%s\n", K, R, CMODE, m, n, ms, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(A); cudaFree(c);
}
int main() {
  const int m = 148 * 4 * 128 * 2, n = 2048;  // ~151k rows: plenty of parallelism
  run<4, 1, 0>(m, n); run<8, 1, 0>(m, n); run<16, 1, 0>(m, n);
  run<8, 2, 0>(m, n); run<16, 2, 0>(m, n); run<8, 4, 0>(m, n);
  run<4, 1, 1>(m, n); run<8, 1, 1>(m, n); run<16, 1, 1>(m, n);
  run<8, 2, 1>(m, n); run<16, 2, 1>(m, n); run<8, 4, 1>(m, n);
  return 0;
}
