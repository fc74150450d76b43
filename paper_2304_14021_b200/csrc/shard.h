// shard.h — internal interface between the C ABI (paradiag.cu) and the sharded multi-rank engine
// (shard.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/paradiag.h"

struct pd_shard;

extern "C" {   // (the definitions in paradiag.cu sit inside its extern "C" block; not exported)

// accessors into pd_handle (paradiag.cu)
pd_shard*& pd_handle_shard(pd_handle* h);
cudaStream_t pd_handle_stream(const pd_handle* h);
unsigned long long* pd_handle_stats_dev(pd_handle* h);     // {‖δ‖∞ bits, ‖U‖∞ bits} on the device
int pd_set_error(int code, const char* msg);                // records paradiag_last_error, returns code

// sharded engine (shard.cu): one rank of a slab-sharded 2D linear problem
int shard_init(const pd_problem* p, int device, void* cuda_stream, const unsigned char* nccl_id, int rank,
               int nranks, pd_handle** out);
int shard_apply_precond(pd_handle* h, const double* r, double* delta);
int shard_iterate(pd_handle* h, const double* u0_l, double* U_l, pd_iter_info* info);
int shard_solve(pd_handle* h, const double* u0_l, double* U_l, pd_solve_info* info);
int shard_local_rows(const pd_handle* h, int64_t* y0, int64_t* nyl);
void shard_destroy(pd_shard* s);
int shard_unique_id(unsigned char id[128]);

}  // extern "C"
