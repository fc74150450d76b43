// tlong.h — the long-window time pass (k_tlong.cuh) as seen by the engine.
#pragma once
#include <cuda_runtime.h>

#include "k_tlong.cuh"

namespace pd {

// N = 2^log2N split as N1 (pass A) × N2 (pass B): N2 = 1024 from N = 2^15 on, else balanced
void tlong_split(int log2N, int* log2N1, int* log2N2);
cudaError_t tlong_attrs();
// N = N1·N2 for the mixed-radix passes (k_tmix.cuh): N has only the factors 2 and 5, N1 the
// largest divisor ≤ √N with N1, N2 ≤ kMixMaxL; plans = radices (8, 4, 2, then 5s).  false: no split.
constexpr int kMixMaxL = 1024;          // staged tile [L][8 pairs] of kTlSmem bytes
bool mixed_split(int N, int* N1, int* N2, int8_t* plan1, int* ns1, int8_t* plan2, int* ns2);
// pass B forward + divide + pass B inverse fused (stage 5) applies: N2 = 1024
bool tlong_fusable(const TlongParams& Q);
// stage 0: pass A forward (real in → Y), 1: pass B forward (Y → X), 2: divide (X in place, `out`),
// 3: pass B inverse (X → Y), 4: pass A inverse (Y → real out), 5: fused pass B with the divide
// (Y in place, `out`).  false: unsupported factor length.
bool tlong_launch(int stage, const void* in, void* out, const TlongParams& Q, cudaStream_t s);

}  // namespace pd
