// fast_e4.cu — register-FFT pass instantiations for E = 4 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(4)
}  // namespace pd
