// stage.cuh — shared-memory residency of a kernel's small per-block arrays.
//
// The dependent searches of the hot path (reaching-definition searches,
// waitcnt chain enumeration) walk the CFG one block at a time; from global
// memory every step is an L2 round trip.  When the arrays a search touches fit
// in shared memory, each CTA stages them once with 1-D TMA bulk copies
// (cp.async.bulk global -> shared, completion counted on an mbarrier) and the
// search runs at shared-memory latency.
//
// Protocol (all threads of the CTA call every function):
//   StageBar sb; sb.init();                 // thread 0 inits the mbarrier
//   sb.begin();                             // proxy fence before re-staging
//   sb.copy(dst, src, bytes);  ...          // thread 0 issues bulk parts;
//                                           // every thread helps with tails
//   sb.commit_and_wait();                   // expect_tx + wait on the phase
#pragma once
#include "common.cuh"

namespace leo {

LEO_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

LEO_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LEO_DEV uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster
LEO_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct StageBar {
  uint64_t* bar;
  uint16_t mc_mask;            // != 0: cluster multicast (rank 0 issues, every CTA receives)
  uint32_t mc_rank;
  uint32_t phase;
  uint32_t tx;                 // bytes in flight this phase (thread 0's view)
  // bulk copies queued by thread 0 (issued after expect_tx)
  const void* src[8];
  void* dst[8];
  uint32_t len[8];
  int n;

  // multicast: the CTAs of a thread-block cluster stage the same image; CTA
  // rank 0 issues each bulk copy once with .multicast::cluster and it lands at
  // the same offset in every CTA's shared memory, completing on every CTA's
  // own mbarrier (one L2 / HBM fetch per cluster instead of one per CTA).
  LEO_DEV void init(uint64_t* b, bool multicast = false) {
    bar = b; phase = 0; tx = 0; n = 0; mc_mask = 0; mc_rank = 0;
    if (multicast) {
      const uint32_t nc = cluster_nctarank();
      if (nc > 1) { mc_mask = (uint16_t)((1u << nc) - 1u); mc_rank = cluster_ctarank(); }
    }
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // every CTA's barrier exists before the leader's copies can signal it
    if (mc_mask) cluster_sync_all();
  }
  // Generic-proxy writes to the destination (previous round) must be ordered
  // before the async-proxy (TMA) writes of the next round.
  LEO_DEV void begin() {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tx = 0; n = 0;
  }
  // dst must be 16-byte aligned shared memory.
  LEO_DEV void copy(void* d, const void* s, size_t bytes) {
    if (bytes == 0) return;
    const bool aligned = (((uintptr_t)s) & 15) == 0 && (((uintptr_t)d) & 15) == 0;
    size_t bulk = aligned ? (bytes & ~(size_t)15) : 0;
    if (bulk > 0 && n == 8) bulk = 0;
    if (bulk > 0 && threadIdx.x == 0) {
      src[n] = s; dst[n] = d; len[n] = (uint32_t)bulk; n++;
      tx += (uint32_t)bulk;
    } else if (bulk > 0) {
      n++;
    }
    // tail (or whole unaligned segment) with plain loads by all threads
    const unsigned char* s8 = (const unsigned char*)s;
    unsigned char* d8 = (unsigned char*)d;
    if (!aligned || bulk == 0) {
      if ((((uintptr_t)s | (uintptr_t)d | bytes) & 3) == 0) {
        const uint32_t* s4 = (const uint32_t*)s;
        uint32_t* d4 = (uint32_t*)d;
        for (size_t x = threadIdx.x; x < bytes / 4; x += blockDim.x) d4[x] = s4[x];
      } else {
        for (size_t x = threadIdx.x; x < bytes; x += blockDim.x) d8[x] = s8[x];
      }
    } else {
      for (size_t x = bulk + threadIdx.x; x < bytes; x += blockDim.x) d8[x] = s8[x];
    }
  }
  LEO_DEV void commit_and_wait() {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   :: "r"(smem_addr(bar)), "r"(tx) : "memory");
      if (!mc_mask) {
        for (int i = 0; i < n; i++)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(smem_addr(dst[i])), "l"(src[i]), "r"(len[i]), "r"(smem_addr(bar)) : "memory");
      } else if (mc_rank == 0) {
        for (int i = 0; i < n; i++)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                       " [%0], [%1], %2, [%3], %4;"
                       :: "r"(smem_addr(dst[i])), "l"(src[i]), "r"(len[i]), "r"(smem_addr(bar)), "h"(mc_mask)
                       : "memory");
      }
    }
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_addr(bar)), "r"(phase) : "memory");
    }
    phase ^= 1;
    __syncthreads();            // plain-load tails visible to every thread
  }
};

// 16-byte aligned carve-out of dynamic shared memory
struct SmemCarve {
  unsigned char* p;
  template <typename T> LEO_DEV T* take(size_t n) {
    T* r = (T*)p;
    p += (n * sizeof(T) + 15) & ~(size_t)15;
    return r;
  }
};
__host__ __device__ inline size_t carve_bytes(size_t n, size_t elem) { return (n * elem + 15) & ~(size_t)15; }

}  // namespace leo
