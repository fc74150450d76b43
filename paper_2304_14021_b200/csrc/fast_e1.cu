// fast_e1.cu — register-FFT pass instantiations for E = 1 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(1)
}  // namespace pd
