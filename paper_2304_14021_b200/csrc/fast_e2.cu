// fast_e2.cu — register-FFT pass instantiations for E = 2 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(2)
}  // namespace pd
