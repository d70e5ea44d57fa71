// report.cu — report assembly on the device outputs.
//
//   single_dep_coverage (analysis.py:547-561) before (base graph minus sync
//   edges, report.py:135-137) and after (pruned graph):  per consumer, the set
//   of dependency classes of its incoming edges and their number; a node
//   qualifies when it has one class or every class appears once.  Edge-parallel
//   atomics into [N] masks/counts, then a node-parallel reduction.
//
//   rank_hotspots (report.py:96-109):  instructions with stall cycles > 0 by
//   (-S_j, offset); offsets strictly increase with the instruction index
//   (disasm.py:391-392), so the key is (-lat_j, j).  One CTA: binary search of
//   the top_n-th largest latency count, ordered compaction of the selection,
//   bitonic sort in shared memory; zero-stall instructions follow in index
//   order when include_unsampled.
//
//   per hotspot (warp each):  its blame entries (contiguous: entries are
//   grouped by stalled instruction in increasing order) sorted by
//   (-blame_cycles, cause index, self first) as report.py:160-163 orders
//   causes, and trace_chain (analysis.py:499-538): greedy walk along the entry
//   minimising (-blame_cycles, cause offset, self last), first minimum in
//   entry order, stopping at self-blame, a revisit, missing entries or
//   chain_depth hops.
#include "prims.cuh"

namespace leo {

__global__ void k_cov_edges(const int32_t* __restrict__ cons, const uint32_t* __restrict__ meta,
                            const int32_t* n_dev, int32_t cap, int32_t* __restrict__ mask,
                            int32_t* __restrict__ cnt) {
  pdl_wait();
  const int n = min(*n_dev, cap);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int c = cons[e];
    atomicOr(&mask[c], 1 << ((meta[e] >> 30) & 3));
    atomicAdd(&cnt[c], 1);
  }
}

__global__ void k_cov_nodes(int N, const int32_t* __restrict__ mask, const int32_t* __restrict__ cnt,
                            int32_t* __restrict__ out) {
  pdl_wait();
  __shared__ int sw[33];
  int nodes = 0, qual = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    const int c = cnt[j];
    if (c == 0) continue;
    nodes++;
    const int d = __popc(mask[j]);
    if (d == 1 || d == c) qual++;
  }
  int t0, t1;
  block_excl_scan(nodes, sw, &t0);
  block_excl_scan(qual, sw, &t1);
  if (threadIdx.x == 0) { atomicAdd(&out[0], t0); atomicAdd(&out[1], t1); }
}

constexpr int kRankMax = 4096;      // device ranking capacity (top_n)

LEO_DEV int cta_count(int N, const int32_t* lat, int lo_inclusive, int* sw) {
  int c = 0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) c += lat[j] >= lo_inclusive;
  int tot;
  block_excl_scan(c, sw, &tot);
  return tot;
}

// ordered compaction of j with pred(lat[j]) into out[base ..], at most `limit`
template <class Pred>
LEO_DEV int cta_compact(int N, const int32_t* lat, Pred pred, int32_t* out, int limit, int* sw) {
  const int per = (N + blockDim.x - 1) / blockDim.x;
  const int lo = min(N, (int)threadIdx.x * per), hi = min(N, lo + per);
  int c = 0;
  for (int j = lo; j < hi; j++) c += pred(lat[j]);
  int tot;
  int pos = block_excl_scan(c, sw, &tot);
  for (int j = lo; j < hi && pos < limit; j++)
    if (pred(lat[j])) out[pos++] = j;
  return min(tot, limit);
}

__global__ void __launch_bounds__(1024) k_report_rank(int N, const int32_t* __restrict__ lat, int top_n,
                                                      int include_unsampled, int32_t* __restrict__ hot,
                                                      int32_t* __restrict__ n_hot) {
  pdl_wait();
  __shared__ int sw[33];
  __shared__ unsigned long long key[kRankMax];
  int32_t* sel = hot;                    // the selection is staged in the output
  top_n = min(top_n, kRankMax);
  int mx = 0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) mx = max(mx, lat[j]);
  // block max: warp shuffles, then across warps
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = threadIdx.x < (blockDim.x >> 5) ? sw[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) sw[32] = v;
  }
  __syncthreads();
  mx = sw[32];
  __syncthreads();
  const int n_st = mx > 0 ? cta_count(N, lat, 1, sw) : 0;
  const int K = min(top_n, n_st);
  int k = 0;
  if (K > 0) {
    // T = largest v with |{lat >= v}| >= K
    int lo = 1, hi = mx;
    while (lo < hi) {
      const int mid = lo + (hi - lo + 1) / 2;
      if (cta_count(N, lat, mid, sw) >= K) lo = mid; else hi = mid - 1;
    }
    const int T = lo;
    const int above = cta_compact(N, lat, [T](int v) { return v > T; }, sel, K, sw);
    __syncthreads();
    cta_compact(N, lat, [T](int v) { return v == T; }, sel + above, K - above, sw);
    __syncthreads();
    int P = 1;
    while (P < K) P <<= 1;
    __syncthreads();
    for (int x = threadIdx.x; x < P; x += blockDim.x)
      key[x] = x < K ? ((unsigned long long)(0x7fffffff - lat[sel[x]]) << 32) | (unsigned)sel[x] : ~0ull;
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int x = threadIdx.x; x < P; x += blockDim.x) {
          const int y = x ^ stride;
          if (y > x) {
            const bool up = (x & size) == 0;
            const unsigned long long a = key[x], b = key[y];
            if ((a > b) == up) { key[x] = b; key[y] = a; }
          }
        }
        __syncthreads();
      }
    __syncthreads();
    for (int x = threadIdx.x; x < K; x += blockDim.x) hot[x] = (int32_t)(key[x] & 0xffffffffu);
    k = K;
  }
  __syncthreads();
  if (include_unsampled && k < top_n)
    k += cta_compact(N, lat, [](int v) { return v == 0; }, hot + k, top_n - k, sw);
  if (threadIdx.x == 0) *n_hot = k;
}

struct ReportArgs {
  const int32_t* n_hot;
  const int32_t* hot;
  const int32_t* b_stalled;
  const int32_t* b_edge;
  const double* b_blame;
  const int32_t* b_count;
  int32_t b_cap;
  const int32_t* pprod;
  int32_t max_causes;
  int32_t chain_depth;
  int32_t* n_causes;
  int32_t* causes;
  int32_t* chain_len;
  int32_t* chain_node;
  int32_t* chain_entry;
  int32_t* chain_self;
  uint32_t* status;
};

// first entry index with stalled >= j (entries are sorted by stalled)
LEO_DEV int lower_entry(const int32_t* st, int n, int j) {
  int lo = 0, hi = n;
  while (lo < hi) { const int m = (lo + hi) >> 1; if (st[m] < j) lo = m + 1; else hi = m; }
  return lo;
}

// cause order key pieces: report.py:160-163 (self = -1 first on ties);
// trace_chain analysis.py:520-522 (self = +inf last on ties)
__global__ void k_report_hot(ReportArgs a) {
  pdl_wait();
  const int h = blockIdx.x;
  if (h >= *a.n_hot || threadIdx.x != 0) return;
  const int nb = *a.b_count <= a.b_cap ? *a.b_count : 0;
  const int j = a.hot[h];
  // causes: entries of j sorted by (-blame, cause index, self first)
  const int b0 = lower_entry(a.b_stalled, nb, j), b1 = lower_entry(a.b_stalled, nb, j + 1);
  const int cnt = b1 - b0;
  a.n_causes[h] = cnt;
  if (cnt > a.max_causes) atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
  int32_t* out = a.causes + (size_t)h * a.max_causes;
  int m = 0;
  for (int x = b0; x < b1 && m < a.max_causes; x++) {
    const double bl = a.b_blame[x];
    const int cz = a.b_edge[x] < 0 ? -1 : a.pprod[a.b_edge[x]];
    int y = m - 1;
    while (y >= 0) {                               // stable insertion
      const double by = a.b_blame[out[y]];
      const int cy = a.b_edge[out[y]] < 0 ? -1 : a.pprod[a.b_edge[out[y]]];
      if (by < bl || (by == bl && cy > cz)) { out[y + 1] = out[y]; y--; } else break;
    }
    out[y + 1] = x;
    m++;
  }
  // trace_chain
  int32_t* cn = a.chain_node + (size_t)h * a.chain_depth;
  int32_t* ce = a.chain_entry + (size_t)h * a.chain_depth;
  int len = 0, self = -1;
  if (a.chain_depth > 0) { cn[0] = j; ce[0] = -1; len = 1; }
  int node = j;
  while (len > 0 && len < a.chain_depth) {
    const int e0 = lower_entry(a.b_stalled, nb, node), e1 = lower_entry(a.b_stalled, nb, node + 1);
    if (e0 == e1) break;
    int best = -1;
    double bb = 0.0;
    int bc = 0;
    for (int x = e0; x < e1; x++) {
      const double bl = a.b_blame[x];
      const int cz = a.b_edge[x] < 0 ? 0x7fffffff : a.pprod[a.b_edge[x]];
      if (best < 0 || bl > bb || (bl == bb && cz < bc)) { best = x; bb = bl; bc = cz; }
    }
    if (a.b_edge[best] < 0) { self = best; break; }
    const int cause = bc;
    bool seen = false;
    for (int t = 0; t < len; t++) if (cn[t] == cause) { seen = true; break; }
    if (seen) break;
    cn[len] = cause; ce[len] = best; len++;
    node = cause;
  }
  a.chain_len[h] = len;
  a.chain_self[h] = self;
}

}  // namespace leo
