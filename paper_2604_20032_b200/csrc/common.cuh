// common.cuh — shared device helpers for the LEO B200 hot path (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>
#include <utility>

#include "../../include/leo_b200.h"

#define LEO_DEV __device__ __forceinline__

#define BIT(c) (1u << (c))
constexpr uint32_t kMemoryProducer = BIT(LEO_OC_GLOBAL_LOAD) | BIT(LEO_OC_LOCAL_LOAD) |
    BIT(LEO_OC_SCALAR_LOAD) | BIT(LEO_OC_CONSTANT_LOAD) | BIT(LEO_OC_ATOMIC) | BIT(LEO_OC_SEND);
constexpr uint32_t kMemoryClasses = kMemoryProducer | BIT(LEO_OC_GLOBAL_STORE) | BIT(LEO_OC_LOCAL_STORE);
constexpr uint32_t kCompute = BIT(LEO_OC_FP_ARITH) | BIT(LEO_OC_INT_ARITH) | BIT(LEO_OC_CONVERSION);
constexpr uint32_t kVmcnt = BIT(LEO_OC_GLOBAL_LOAD) | BIT(LEO_OC_GLOBAL_STORE) | BIT(LEO_OC_ATOMIC);
constexpr uint32_t kLgkmcnt = BIT(LEO_OC_LOCAL_LOAD) | BIT(LEO_OC_LOCAL_STORE) |
    BIT(LEO_OC_SCALAR_LOAD) | BIT(LEO_OC_CONSTANT_LOAD);

// RegClass rank in `.value` string order (depgraph.py:514-516 sort key)
__constant__ static const int kRcRank[8] = {6, 2, 1, 0, 5, 3, 4, 7};

LEO_DEV int op_index(uint32_t r) { return (int)(r & 0xFFFF); }
LEO_DEV int op_span(uint32_t r) { return (int)((r >> 16) & 0xFF); }
LEO_DEV int op_class(uint32_t r) { return (int)((r >> 24) & 7); }
LEO_DEV int op_role(uint32_t r) { return (int)((r >> 27) & 3); }

LEO_DEV int dep_class_of(uint32_t producer_oc, int kind) {   // depgraph.py:63-68
  if (kind >= LEO_EK_MEM_WAITCNT) return LEO_DC_MEMORY;
  if (kMemoryProducer & BIT(producer_oc)) return LEO_DC_MEMORY;
  if (producer_oc == LEO_OC_BARRIER_ALL) return LEO_DC_SYNCHRONIZATION;
  return LEO_DC_EXECUTION;
}

// Kernel struct passed by value to kernels (pointers are device pointers).
struct KView {
  int32_t N, B, U, dialect;
  int32_t unit_base[8];
  const uint8_t* __restrict__ opclass;
  const int32_t* __restrict__ block_of;
  const int32_t* __restrict__ opnd_ptr;
  const uint32_t* __restrict__ opnd;
  const uint8_t* __restrict__ sync_kind;
  const uint32_t* __restrict__ sync_a;
  const uint32_t* __restrict__ sync_b;
  const int32_t* __restrict__ blk_first;
  const int32_t* __restrict__ blk_last;
  const int32_t* __restrict__ succ_ptr;
  const int32_t* __restrict__ succ;
  const int32_t* __restrict__ pred_ptr;
  const int32_t* __restrict__ pred;
};

inline KView make_kview(const LeoKernel* k) {
  // (LeoKernel.n_segments / seg_block are read by the segment-aware tiers)
  KView v;
  v.N = k->n_instr; v.B = k->n_blocks; v.U = k->n_units; v.dialect = k->dialect;
  for (int c = 0; c < 8; c++) v.unit_base[c] = k->unit_base[c];
  v.opclass = k->opclass; v.block_of = k->block_of; v.opnd_ptr = k->opnd_ptr; v.opnd = k->opnd;
  v.sync_kind = k->sync_kind; v.sync_a = k->sync_a; v.sync_b = k->sync_b;
  v.blk_first = k->blk_first; v.blk_last = k->blk_last; v.succ_ptr = k->succ_ptr;
  v.succ = k->succ; v.pred_ptr = k->pred_ptr; v.pred = k->pred;
  return v;
}

// consumer ownership under stalled-PC sharding (LeoConfig.consumer_lo/hi)
struct Range {
  int lo, hi;
  LEO_DEV bool has(int j) const { return hi <= 0 || (j >= lo && j < hi); }
};

LEO_DEV int unit_of(const KView& k, uint32_t r) { return k.unit_base[op_class(r)] + op_index(r); }

// ---- diagnostics ------------------------------------------------------------
LEO_DEV void diag_push(LeoDiags d, uint32_t* status, int code, int instr, int a0, int a1, int a2, int seq) {
  int slot = atomicAdd(d.count, 1);
  if (slot < d.capacity) {
    LeoDiag r; r.code = code; r.instr = instr; r.a0 = a0; r.a1 = a1; r.a2 = a2; r.seq = seq;
    d.rec[slot] = r;
  } else {
    atomicOr(status, (uint32_t)LEO_ST_DIAG_OVERFLOW);
  }
}

// ---- CPython >= 3.12 builtins.sum over floats (Neumaier), analysis.py:464,472
struct PySum {
  double s, c; int n;
  LEO_DEV PySum() : s(0.0), c(0.0), n(0) {}
  LEO_DEV void add(double x) {
    if (n++ == 0) { s = __dadd_rn(0.0, x); c = 0.0; return; }
    double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
    s = t;
  }
  LEO_DEV double value() const {
    if (c != 0.0 && isfinite(c)) return __dadd_rn(s, c);
    return s;
  }
};

// ---- profiling aid: per-CTA phase marks (LEO_DBG_PHASES) ----------------------
__device__ long long g_phase_ts[4][1024][8];
__device__ long long g_item_cycles[16384];     // per-item cycles: waitcnt tier [0, 8192), reach tier 0 [8192, 16384)
__device__ int g_reach_item_ctr;
__device__ int g_tier_counts[16];              // build_graph counters (LEO_DBG_PHASES)
__global__ void k_copy_counts(const int32_t* ctr, int n) {
  for (int i = threadIdx.x; i < n && i < 16; i += blockDim.x) g_tier_counts[i] = ctr[i];
}
struct PhaseMarks {
  int on; long long t0;
  LEO_DEV PhaseMarks(int dbg) {
#ifdef __CUDA_ARCH__
    on = (dbg & LEO_DBG_PHASES) && blockIdx.x < 1024;
    t0 = clock64();
#endif
  }
  LEO_DEV void mark(int slot, int ph) const {
#ifdef __CUDA_ARCH__
    if (on && threadIdx.x == 0) g_phase_ts[slot][blockIdx.x][ph] = clock64() - t0;
#endif
  }
};

// ---- programmatic dependent launch ------------------------------------------
// Every pipeline kernel is launched with programmatic stream serialization
// (leo_launch) and starts with pdl_wait(): the kernel may be scheduled while
// its predecessor drains, and waits here until the predecessor grid has
// completed and its memory is visible (a no-op without the attribute).
LEO_DEV void pdl_wait() {
#ifdef __CUDA_ARCH__
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// ---- launch helpers ---------------------------------------------------------
// dynamic shared memory a shared-memory-resident tier may request per CTA
constexpr int kSmemResidentMax = 200 * 1024;
inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

// LEO_NO_PDL=1 launches without the programmatic-serialization attribute
inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("LEO_NO_PDL"); v = (e && e[0] == '1') ? 0 : 1; }
  return v == 1;
}

// Scheduling priority of the launches issued by this host thread: the
// register-dataflow chain (the step's critical path) runs at the device's
// greatest priority, the side branches that only need to finish before their
// join (vendor sync tracing, binning, the addressing test) at the least, so
// their CTAs fill the SMs the critical chain leaves free instead of
// displacing it.  LEO_NO_PRIO=1 launches everything at the default priority.
struct LaunchPrio {
  // 1 = greatest, 0 = least, -1 = no priority attribute (the default)
  static int& current() { static thread_local int p = -1; return p; }
};
struct HighPriority {
  int saved;
  explicit HighPriority(bool on) : saved(LaunchPrio::current()) { if (on) LaunchPrio::current() = 1; }
  ~HighPriority() { LaunchPrio::current() = saved; }
};
struct LowPriority {
  int saved;
  explicit LowPriority(bool on = true) : saved(LaunchPrio::current()) {
    if (on && saved >= 0) LaunchPrio::current() = 0;   // only inside a prioritised call
  }
  ~LowPriority() { LaunchPrio::current() = saved; }
};
inline int prio_value(bool high) {
  static int least = 0, greatest = 0, init = 0, off = 0;
  if (!init) {
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const char* e = getenv("LEO_NO_PRIO");
    off = (e && e[0] == '1') ? 1 : 0;
    init = 1;
  }
  if (off) return least;
  return high ? greatest : least;
}

template <typename... KArgs, typename... Args>
inline void leo_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  if (LaunchPrio::current() >= 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = prio_value(LaunchPrio::current() != 0);
    na++;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// leo_launch with a thread-block cluster of `csize` CTAs along x (grid % csize == 0)
template <typename... KArgs, typename... Args>
inline void leo_launch_cluster(void (*kern)(KArgs...), int grid, int csize, dim3 block, size_t smem,
                               cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = csize;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  na++;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    na++;
  }
  if (LaunchPrio::current() >= 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = prio_value(LaunchPrio::current() != 0);
    na++;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define LEO_CUDA_CHECK(x)                                      \
  do {                                                         \
    cudaError_t _e = (x);                                      \
    if (_e != cudaSuccess) return -1000 - (int)_e;             \
  } while (0)
