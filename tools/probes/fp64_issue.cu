// Micro-probe: FP64 latency / throughput and the register-FFT core's IPC vs warps per SM.
//   chain:   dependent DFMA chain (latency)
//   indep:   8 independent DFMA chains per thread, W warps per SM (throughput vs occupancy)
//   fft32:   the 32-point register DFT of fft4.cuh in a loop, W warps per SM
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2304_14021_b200/csrc fp64_issue.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fft4.cuh"

__global__ void chain(double* out, int iters) {
  double a = threadIdx.x * 1e-3;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0) / iters;
  if (a == 12345.0) out[1] = a;
}

__global__ void indep(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.0) out[0] = s;
}

template <int R>
__global__ void fftk(double* out, int iters) {
  double2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = make_double2(threadIdx.x * 1e-3 + i, i * 0.5);
  for (int it = 0; it < iters; ++it) {
    pd::dft_reg<R, -1>(v);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = make_double2(v[i].x * 0.03125, v[i].y * 0.03125);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) s += v[i].x + v[i].y;
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  chain<<<1, 32>>>(out, 10000);
  cudaDeviceSynchronize();
  double lat;
  cudaMemcpy(&lat, out, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", lat);
  const int nsm = 148;
  for (int w : {4, 8, 16, 32}) {
    const int iters = 20000;
    indep<<<nsm, 32 * w>>>(out, 100);
    cudaEventRecord(e0);
    indep<<<nsm, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double wi = (double)nsm * w * iters * 8;   // warp-instructions
    printf("indep DFMA  warps/SM=%2d: %.3f warp-instr/clk/SM at 1.92 GHz (%.1f TFLOP/s)\n", w,
           wi / (ms * 1e-3) / nsm / 1.92e9, wi * 32 * 2 / (ms * 1e-3) / 1e12);
  }
  for (int w : {4, 8, 12, 16}) {
    const int iters = 2000;
    fftk<32><<<nsm, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    fftk<32><<<nsm, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dft32 warps/SM=%2d: %.2f us per 1000 DFTs/warp -> %.3f Gpoint/s/SM\n", w, ms * 1e3 / iters * 1000 / 1000,
           (double)w * 32 * 32 * iters / (ms * 1e-3) / nsm / 1e9);
  }
  for (int w : {8, 16, 24, 32}) {
    const int iters = 2000;
    fftk<16><<<nsm, 32 * w>>>(out, 10);
    cudaEventRecord(e0);
    fftk<16><<<nsm, 32 * w>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dft16 warps/SM=%2d: -> %.3f Gpoint/s/SM\n", w, (double)w * 32 * 16 * iters / (ms * 1e-3) / nsm / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
