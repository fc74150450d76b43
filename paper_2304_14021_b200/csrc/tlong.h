// tlong.h — the long-window time pass (k_tlong.cuh) as seen by the engine.
#pragma once
#include <cuda_runtime.h>

#include "k_tlong.cuh"

namespace pd {

// N = 2^log2N split as N1 = 2^⌈log2N/2⌉ (pass A) × N2 (pass B)
void tlong_split(int log2N, int* log2N1, int* log2N2);
cudaError_t tlong_attrs();
// stage 0: pass A forward (real in → Y), 1: pass B forward (Y → X), 2: divide (X in place, `out`),
// 3: pass B inverse (X → Y), 4: pass A inverse (Y → real out).  false: unsupported factor length.
bool tlong_launch(int stage, const void* in, void* out, const TlongParams& Q, cudaStream_t s);

}  // namespace pd
