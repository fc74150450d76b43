// Micro-probe: HBM read / write bandwidth vs contiguous segment size for the time-pencil access
// pattern (S consecutive doubles from each of NT slices, slice stride = NS doubles), with high
// memory-level parallelism (every warp keeps UNR 16-byte loads in flight per lane).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a seg_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 512;
constexpr size_t NS = 2049ull * 2049ull + 1;   // even slice stride (16-B aligned rows)

// each warp: tiles of S points x NT slices; lane reads 16 B (2 doubles); a row segment of S doubles
// needs S/2 lanes; warp covers 64/S rows per instruction.
template <int S, int UNR>
__global__ void __launch_bounds__(256) seg_read(const double* __restrict__ in, double* __restrict__ out, size_t ntiles) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int LPR = S / 2;               // lanes per row
  constexpr int RPI = 32 / LPR;            // rows per instruction
  const int lr = lane / LPR, lc = lane % LPR;
  double acc = 0.0;
  for (size_t tile = (size_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (size_t)gridDim.x * 8) {
    const double* base = in + tile * S + 2 * lc;
    for (int t0 = 0; t0 < NT; t0 += RPI * UNR) {
      double2 v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) v[u] = __ldg(reinterpret_cast<const double2*>(base + (size_t)(t0 + u * RPI + lr) * NS));
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc += v[u].x + v[u].y;
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int S, int UNR>
__global__ void __launch_bounds__(256) seg_write(double* __restrict__ outp, size_t ntiles) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int LPR = S / 2;
  constexpr int RPI = 32 / LPR;
  const int lr = lane / LPR, lc = lane % LPR;
  for (size_t tile = (size_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (size_t)gridDim.x * 8) {
    double* base = outp + tile * S + 2 * lc;
    for (int t0 = 0; t0 < NT; t0 += RPI * UNR) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        *reinterpret_cast<double2*>(base + (size_t)(t0 + u * RPI + lr) * NS) = make_double2(1.0, 2.0);
    }
  }
}

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const size_t n = NS * NT;
  double *a, *o;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&o, 64);
  cudaMemset(a, 0, n * 8);
  const size_t usable = (NS / 128) * 128;   // points covered
  for (int cps : {1, 2, 4}) {
#define R(S)                                                                                        \
  {                                                                                                 \
    const size_t ntiles = usable / S;                                                               \
    float ms = timeit([&] { seg_read<S, 8><<<148 * cps, 256>>>(a, o, ntiles); });                   \
    float ms2 = timeit([&] { seg_write<S, 8><<<148 * cps, 256>>>(a, ntiles); });                    \
    const double gb = (double)ntiles * S * NT * 8 / 1e9;                                            \
    printf("S=%3d (%4d B) CTAs/SM=%d  read %7.1f GB/s  write %7.1f GB/s\n", S, S * 8, cps, gb / ms * 1e3, gb / ms2 * 1e3); \
  }
    R(2) R(4) R(8) R(16) R(32) R(64)
  }
  // contiguous reference
  {
    const size_t ntiles = n / 64;
    float ms = timeit([&] { seg_read<64, 8><<<148 * 4, 256>>>(a, o, 0); });
    (void)ms;
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
