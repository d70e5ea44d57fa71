// prims.cuh — scan / segmented sort primitives with device-resident counts.
//
// Every variable-size stage of the pipeline writes a device counter; the
// kernels below take the element count from device memory (`n_dev`) and an
// upper bound (`cap`) for launch sizing, so the whole pipeline runs without a
// host round trip (and can be captured in a CUDA graph).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace leo {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
// one CTA walks arrays up to this size (its latency grows with n / 1024
// elements per thread); larger arrays take the two-launch tiled scan
constexpr int64_t kScanSingleMax = 1 << 14;

LEO_DEV int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix,
// writes the block total to *total.
LEO_DEV int block_excl_scan(int v, int* smem_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = warp_incl_scan(v);
  if (lane == 31) smem_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? smem_warp[lane] : 0;
    int wi = warp_incl_scan(w);
    if (lane < nw) smem_warp[lane] = wi - w;
    if (lane == nw - 1) smem_warp[32] = wi;
  }
  __syncthreads();
  int r = inc - v + smem_warp[warp];
  *total = smem_warp[32];
  __syncthreads();
  return r;
}

__global__ void scan_tile_sums(const int32_t* __restrict__ in, const int32_t* n_dev, int64_t n_cap,
                               int32_t* __restrict__ tile_sums) {
  pdl_wait();
  __shared__ int sw[33];
  int64_t n = n_dev ? (int64_t)*n_dev : n_cap;
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) s += in[i];
  }
  int total;
  block_excl_scan(s, sw, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// tile_sums are raw per-tile sums: each CTA adds up the sums of the tiles
// before it (a few hundred L2-resident ints) instead of a separate prefix launch
__global__ void scan_tile_apply(const int32_t* __restrict__ in, const int32_t* n_dev, int64_t n_cap,
                                const int32_t* __restrict__ tile_sums, int32_t* __restrict__ out,
                                int32_t* total_out) {
  pdl_wait();
  __shared__ int sw[33];
  __shared__ int tile_base;
  int64_t n = n_dev ? (int64_t)*n_dev : n_cap;
  {
    int acc = 0;
    for (int t = threadIdx.x; t < (int)blockIdx.x; t += blockDim.x) acc += tile_sums[t];
    int tot;
    block_excl_scan(acc, sw, &tot);
    if (threadIdx.x == 0) tile_base = tot;
    __syncthreads();
  }
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    v[k] = i < n ? in[i] : 0;
    s += v[k];
  }
  int total;
  int ex = block_excl_scan(s, sw, &total) + tile_base;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    if (i < n) out[i] = ex;
    ex += v[k];
  }
  // out[n] = total (CSR end) written by the last tile owner
  const int64_t last_tile = n > 0 ? (n - 1) / kScanTile : 0;
  if ((int64_t)blockIdx.x == last_tile && threadIdx.x == 0) {
    out[n] = tile_base + total;
    if (total_out) *total_out = tile_base + total;
  }
}

// one CTA scans the whole array tile by tile (small arrays: one launch)
// Single CTA, thread-contiguous chunks: pass 1 sums each thread's chunk
// (independent 16-byte loads), one block scan of the chunk sums, pass 2
// writes the running prefix.  Two reads of the input (L2-resident), one
// block-wide barrier phase instead of one per 8K-element tile.
LEO_DEV void scan_one_cta(const int32_t* __restrict__ in, int n, int32_t* __restrict__ out, int32_t* total_out) {
  __shared__ int sw[33];
  const int per = ((n + blockDim.x - 1) / blockDim.x + 3) & ~3;   // multiple of 4
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  const bool vec = ((((uintptr_t)in) & 15) == 0);
  int s = 0;
  if (vec) {
    int x = lo;
    for (; x + 4 <= hi; x += 4) {
      const int4 v = *reinterpret_cast<const int4*>(in + x);
      s += v.x + v.y + v.z + v.w;
    }
    for (; x < hi; x++) s += in[x];
  } else {
    for (int x = lo; x < hi; x++) s += in[x];
  }
  int tot;
  int run = block_excl_scan(s, sw, &tot);
  if (vec && ((((uintptr_t)out) & 15) == 0)) {
    int x = lo;
    for (; x + 4 <= hi; x += 4) {
      const int4 v = *reinterpret_cast<const int4*>(in + x);
      int4 o;
      o.x = run; run += v.x; o.y = run; run += v.y; o.z = run; run += v.z; o.w = run; run += v.w;
      *reinterpret_cast<int4*>(out + x) = o;
    }
    for (; x < hi; x++) { const int v = in[x]; out[x] = run; run += v; }
  } else {
    for (int x = lo; x < hi; x++) { const int v = in[x]; out[x] = run; run += v; }
  }
  if (threadIdx.x == 0) { out[n] = tot; if (total_out) *total_out = tot; }
}

__global__ void __launch_bounds__(1024) scan_single_cta(const int32_t* __restrict__ in, const int32_t* n_dev,
                                                        int64_t n_cap, int32_t* __restrict__ out,
                                                        int32_t* total_out) {
  pdl_wait();
  scan_one_cta(in, (int)(n_dev ? (int64_t)*n_dev : n_cap), out, total_out);
}

// two independent scans of n elements in one launch (CTA 0: a, CTA 1: b)
__global__ void __launch_bounds__(1024) scan_single_cta_pair(const int32_t* __restrict__ a_in, int32_t* __restrict__ a_out,
                                                             const int32_t* __restrict__ b_in, int32_t* __restrict__ b_out,
                                                             int n) {
  pdl_wait();
  if (blockIdx.x == 0) scan_one_cta(a_in, n, a_out, nullptr);
  else scan_one_cta(b_in, n, b_out, nullptr);
}

// ---- one-launch scan: co-resident CTAs (cooperative launch), tile sums, one
// grid barrier, then each tile adds the sums before it and writes its prefix.
// A CTA that owns one tile keeps it in registers across the barrier (one read
// of the input).  Replaces the tile-sum + apply launch pair (two launches and a
// dependent drain on the critical chain per scan).
constexpr int kCsThreads = 512, kCsItems = 16, kCsTile = kCsThreads * kCsItems;

LEO_DEV int block_reduce_sum(int v, int* sw) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sw[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nw ? sw[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0) sw[32] = w;
  }
  __syncthreads();
  const int r = sw[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kCsThreads) scan_coop(const int32_t* __restrict__ in, const int32_t* n_dev,
                                                        int64_t n_cap, int32_t* __restrict__ tsum,
                                                        int32_t* __restrict__ out, int32_t* total_out) {
  __shared__ int sw[33];
  const int64_t n = n_dev ? (int64_t)*n_dev : n_cap;
  const int64_t ntiles = n > 0 ? (n + kCsTile - 1) / kCsTile : 1;
  const bool one = ntiles <= (int64_t)gridDim.x;
  const int tid = threadIdx.x;
  int v[kCsItems];
  auto load = [&](int64_t t) {
    const int64_t base = t * kCsTile + (int64_t)tid * kCsItems;
    if (base + kCsItems <= n) {
      const int4* p = reinterpret_cast<const int4*>(in + base);
#pragma unroll
      for (int q = 0; q < kCsItems / 4; q++) {
        const int4 x = p[q];
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kCsItems; k++) v[k] = base + k < n ? in[base + k] : 0;
    }
  };
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    load(t);
    int s = 0;
#pragma unroll
    for (int k = 0; k < kCsItems; k++) s += v[k];
    const int tot = block_reduce_sum(s, sw);
    if (tid == 0) tsum[t] = tot;
  }
  cooperative_groups::this_grid().sync();
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (!one) load(t);
    int acc = 0;
    for (int64_t x = tid; x < t; x += kCsThreads) acc += tsum[x];
    const int prefix = block_reduce_sum(acc, sw);
    int s = 0;
#pragma unroll
    for (int k = 0; k < kCsItems; k++) s += v[k];
    int tile_total;
    int ex = block_excl_scan(s, sw, &tile_total) + prefix;
    const int64_t base = t * kCsTile + (int64_t)tid * kCsItems;
    if (base + kCsItems <= n) {
      int4* p = reinterpret_cast<int4*>(out + base);
#pragma unroll
      for (int q = 0; q < kCsItems / 4; q++) {
        int4 o;
        o.x = ex; ex += v[4 * q]; o.y = ex; ex += v[4 * q + 1];
        o.z = ex; ex += v[4 * q + 2]; o.w = ex; ex += v[4 * q + 3];
        p[q] = o;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kCsItems; k++) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
      }
    }
    if (t == ntiles - 1 && tid == 0) {
      out[n] = prefix + tile_total;
      if (total_out) *total_out = prefix + tile_total;
    }
  }
}

int scan_coop_grid();   // co-resident CTAs of scan_coop on the current device (leo_b200.cu)

// exclusive scan of in[0..n) into out[0..n] (out[n] = total); n from n_dev if
// given else n_cap.  scratch: >= tiles(n_cap) ints.  total_out optional.
// in / out must be 16-byte aligned (arena allocations are 256-byte aligned).
inline void scan_exclusive(const int32_t* in, int32_t* out, const int32_t* n_dev, int64_t n_cap,
                           int32_t* scratch, int32_t* total_out, cudaStream_t st) {
  if (n_cap <= kScanSingleMax) {
    leo_launch(scan_single_cta, 1, 1024, 0, st, in, n_dev, n_cap, out, total_out);
    return;
  }
  if (!getenv("LEO_SCAN_TILED")) {     // one launch: -2..-15 us per step on C2/C3/C5 (measured A/B)
    const int64_t ntiles = (n_cap + kCsTile - 1) / kCsTile;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, scan_coop_grid()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCsThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    na++;
    if (LaunchPrio::current() >= 0) {
      attr[na].id = cudaLaunchAttributePriority;
      attr[na].val.priority = prio_value(LaunchPrio::current() != 0);
      na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, scan_coop, in, n_dev, n_cap, scratch, out, total_out);
    return;
  }
  int64_t ntiles = (n_cap + kScanTile - 1) / kScanTile;
  if (ntiles < 1) ntiles = 1;
  leo_launch(scan_tile_sums, (unsigned)ntiles, kScanThreads, 0, st, in, n_dev, n_cap, scratch);
  leo_launch(scan_tile_apply, (unsigned)ntiles, kScanThreads, 0, st, in, n_dev, n_cap, scratch, out, total_out);
}
inline int64_t scan_scratch_ints(int64_t n_cap) { return (n_cap + kScanTile - 1) / kScanTile + 1; }

// ---- segmented sort + unique (thread per segment) --------------------------
LEO_DEV void sort_small_u64(uint64_t* a, int n) {
  for (int i = 1; i < n; i++) {
    uint64_t x = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; j--; }
    a[j + 1] = x;
  }
}
LEO_DEV void shell_sort_u64(uint64_t* a, int n) {
  int gap = 1;
  while (gap < n / 3) gap = gap * 3 + 1;
  for (; gap > 0; gap /= 3)
    for (int i = gap; i < n; i++) {
      uint64_t x = a[i];
      int j = i;
      while (j >= gap && a[j - gap] > x) { a[j] = a[j - gap]; j -= gap; }
      a[j] = x;
    }
}

// Sort keys[begin[s] .. begin[s]+len[s]) ascending, drop duplicates in place,
// write the unique count to uniq[s].  Segments reaching past `cap` (the
// producer overflowed its buffer and flagged it) are left empty.
// Lane per segment for short segments (register network / insertion sort);
// segments of 25..kSegWarpMax keys are sorted by the whole warp (bitonic sort
// in shared memory, ballot compaction), longer ones fall back to a shell sort.
constexpr int kSegWarpMax = 256, kSegThreads = 128;

__global__ void __launch_bounds__(kSegThreads) segsort_unique_u64(uint64_t* __restrict__ keys,
                                                                  const int32_t* __restrict__ begin,
                                                                  const int32_t* __restrict__ len,
                                                                  const int32_t* nseg_dev, int nseg_cap,
                                                                  int32_t* __restrict__ uniq, int64_t cap) {
  pdl_wait();
  __shared__ uint64_t wbuf[kSegThreads / 32][kSegWarpMax];
  uint64_t* buf = wbuf[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int nseg = nseg_dev ? *nseg_dev : nseg_cap;
  // whole warps iterate together (the cooperative path needs every lane)
  for (int s0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); s0 < nseg; s0 += gridDim.x * blockDim.x) {
    const int s = s0 + lane;
    int n = 0, b = 0;
    bool mine = false;
    if (s < nseg) {
      n = len[s];
      b = begin[s];
      if ((int64_t)b + n > cap) { uniq[s] = 0; n = 0; }
      else mine = true;
    }
    uint64_t* a = keys + b;
    if (mine && n <= 1) { uniq[s] = n; mine = false; }
    if (mine && n <= 4) {
      // register sorting network (no local-memory array): the common case
      uint64_t r0 = a[0], r1 = a[1], r2 = n > 2 ? a[2] : ~0ull, r3 = n > 3 ? a[3] : ~0ull;
      auto cs = [](uint64_t& x, uint64_t& y) { const uint64_t lo = x < y ? x : y; y = x < y ? y : x; x = lo; };
      cs(r0, r1); cs(r2, r3); cs(r0, r2); cs(r1, r3); cs(r1, r2);
      int u = 0;
      a[u++] = r0;
      if (r1 != r0) a[u++] = r1;
      if (n > 2 && r2 != r1) a[u++] = r2;
      if (n > 3 && r3 != r2) a[u++] = r3;
      uniq[s] = u;
      mine = false;
    } else if (mine && n <= 8) {
      // 8-key register network (Batcher odd-even merge sort, 19 exchanges)
      uint64_t r[8];
#pragma unroll
      for (int i = 0; i < 8; i++) r[i] = i < n ? a[i] : ~0ull;
      auto cs = [&](int x, int y) { const uint64_t lo = r[x] < r[y] ? r[x] : r[y]; r[y] = r[x] < r[y] ? r[y] : r[x]; r[x] = lo; };
      cs(0, 1); cs(2, 3); cs(4, 5); cs(6, 7);
      cs(0, 2); cs(1, 3); cs(4, 6); cs(5, 7);
      cs(1, 2); cs(5, 6);
      cs(0, 4); cs(1, 5); cs(2, 6); cs(3, 7);
      cs(2, 4); cs(3, 5);
      cs(1, 2); cs(3, 4); cs(5, 6);
      int u = 0;
#pragma unroll
      for (int i = 0; i < 8; i++)
        if (i < n && (i == 0 || r[i] != r[i - 1])) a[u++] = r[i];
      uniq[s] = u;
      mine = false;
    } else if (mine && n <= 24) {
      uint64_t r[24];
      for (int i = 0; i < n; i++) r[i] = a[i];
      sort_small_u64(r, n);
      int u = 0;
      for (int i = 0; i < n; i++)
        if (i == 0 || r[i] != r[i - 1]) a[u++] = r[i];
      uniq[s] = u;
      mine = false;
    } else if (mine && n > kSegWarpMax) {
      shell_sort_u64(a, n);
      int u = 0;
      for (int i = 0; i < n; i++) {
        const uint64_t x = a[i];
        if (i == 0 || x != a[u - 1]) a[u++] = x;
      }
      uniq[s] = u;
      mine = false;
    }
    unsigned big = __ballot_sync(0xffffffffu, mine);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int sn = __shfl_sync(0xffffffffu, n, src), sb = __shfl_sync(0xffffffffu, b, src);
      uint64_t* sa = keys + sb;
      int P = 32;
      while (P < sn) P <<= 1;
      for (int i = lane; i < P; i += 32) buf[i] = i < sn ? sa[i] : ~0ull;
      __syncwarp();
      for (int k2 = 2; k2 <= P; k2 <<= 1)
        for (int jj = k2 >> 1; jj > 0; jj >>= 1) {
          for (int i = lane; i < P; i += 32) {
            const int ixj = i ^ jj;
            if (ixj > i) {
              const uint64_t x = buf[i], y = buf[ixj];
              if ((x > y) == ((i & k2) == 0)) { buf[i] = y; buf[ixj] = x; }
            }
          }
          __syncwarp();
        }
      int base = 0;
      for (int i0 = 0; i0 < sn; i0 += 32) {
        const int i = i0 + lane;
        const bool keep = i < sn && (i == 0 || buf[i] != buf[i - 1]);
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const uint64_t v = i < sn ? buf[i] : 0;
        __syncwarp();
        if (keep) sa[base + __popc(m & ((1u << lane) - 1))] = v;
        base += __popc(m);
      }
      if (lane == src) uniq[s] = base;
      __syncwarp();
    }
  }
}

}  // namespace leo
