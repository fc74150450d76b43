// fast_e16.cu — register-FFT pass instantiations for E = 16 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(16)
}  // namespace pd
