// fast_e32.cu — register-FFT pass instantiations for E = 32 (fast_launch.cuh).
#define PD_FAST_DEFINE
#include "fast_launch.cuh"
namespace pd {
PD_FAST_INSTANTIATE(32)
}  // namespace pd
