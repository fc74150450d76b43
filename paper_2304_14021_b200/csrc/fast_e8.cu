// fast_e8.cu — register-FFT pass instantiations for E = 8 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(8)
}  // namespace pd
