// tma.cuh — Tensor Memory Accelerator (cp.async.bulk.tensor) helpers for the fp64 passes, sm_100a.
//
// A tiled TMA box must start on a 16-byte boundary (measured on B200: a box whose first fp64
// element has an odd inner coordinate is an illegal instruction, tools/probes/tma_probe3.cu), and
// tensor-map strides must be multiples of 16 bytes.  The iterate arrays have odd line and slice
// lengths (2049, 2049², 511², 257²), so the TMA-staged time pass runs on a workspace whose slice
// pitch is rounded up to even (paradiag.cu, pd_handle::wt).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "common.cuh"

namespace pd {

PD_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

PD_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PD_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
PD_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
PD_DEV void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!done);
}
// generic-proxy shared-memory accesses before this point are ordered before later async-proxy
// (TMA) accesses of the same memory
PD_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

PD_DEV void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
PD_DEV void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
PD_DEV void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
// at most N of this thread's bulk groups still reading their shared-memory source
template <int N>
PD_DEV void tma_wait_read_le() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
PD_DEV void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
PD_DEV void tma_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
PD_DEV void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
PD_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Byte offset of double (row r, column c) inside a box of 16-double (128-byte) rows written with
// CU_TENSOR_MAP_SWIZZLE_128B: 16-byte chunk j of row r lives at chunk j ^ (r & 7) (box base
// 1024-byte aligned).  A double2 at an even column is one conflict-free 16-byte access per lane for
// eight consecutive rows.
PD_DEV unsigned sw128(int r, int c) {
  return (unsigned)(r * 128 + ((((c >> 1) ^ (r & 7)) << 4) | ((c & 1) << 3)));
}

}  // namespace pd
