// sync.cu — vendor synchronization edges (depgraph.py:296-501).
//
//   amd    s_waitcnt:  exact chain enumeration (_scan_backward :312-348 with the
//          _WaitcntState visitor :365-399): one thread per waiting instruction
//          walks every simple backward block path (b0 pre-visited, forks inherit
//          the remaining 4096-instruction budget); member operations appended at
//          pending index >= level become edges; best_m drives the diagnostic.
//   nvidia barrier / intel SWSB setter search (_trace_setter :431-443): closed
//          form — nearest setter before the wait in its own block, otherwise a
//          node-weighted Dijkstra over setter-free predecessor blocks (b0
//          excluded): a setter block p yields its last setter iff the cheapest
//          path reaches it within the budget.  (Shortest paths are simple, so
//          this equals the union over the reference's per-chain simple paths.)
//
// Raw (producer, wait) keys are appended to a buffer; k_sync_* then group them
// by producer, sort + dedup per producer and append them after the raw/guard
// edges in (producer, consumer) order (_materialize_sync :485-492).
#include "prims.cuh"

namespace leo {

constexpr int kSyncBudget = 4096;   // SYNC_SCAN_BUDGET depgraph.py:43

struct SyncArgs {
  uint64_t* keys;            // raw (producer << 32 | consumer)
  int64_t key_cap;
  int32_t* key_count;
  int32_t* slow_list;        // (instr << 6 | sub-item) items re-run on global scratch
  int32_t* slow_count;
  int64_t slow_cap;
  LeoDiags diags;
  uint32_t* status;
};

LEO_DEV void sync_emit(const SyncArgs& a, int producer, int wait) {
  int s = atomicAdd(a.key_count, 1);
  if (s < a.key_cap) a.keys[s] = ((uint64_t)(uint32_t)producer << 32) | (uint32_t)wait;
  else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
}

struct Frame { int blk, q, m, a, budget; };

// waitcnt visitor (depgraph.py:368-384); returns false to stop the chain
LEO_DEV bool wc_visit(const KView& k, int x, int counter, uint32_t members, int level, int wait,
                      int& m, int& a, const SyncArgs& sa, int32_t* seen, int& nseen, int seen_cap) {
  if (k.sync_kind[x] == LEO_SYNC_WAITCNT) {
    uint32_t v = counter == 0 ? k.sync_a[x] : k.sync_b[x];
    if (v != LEO_NONE_U32) {
      a = (a < 0) ? (int)v : min(a, (int)v);
      if (a == 0) return false;
    }
  } else if (members & BIT(k.opclass[x])) {
    if (a != 0) {
      if (m >= level) {   // pending[level:] -> edge (emitted once per wait when possible)
        bool dup = false;
        for (int t = 0; t < nseen; t++) if (seen[t] == x) { dup = true; break; }
        if (!dup) {
          if (nseen < seen_cap) seen[nseen++] = x;
          sync_emit(sa, x, wait);
        }
      }
      m++;
      if (a > 0) { a--; if (a == 0) return false; }
    }
  }
  return true;
}

LEO_DEV bool on_path(const Frame* fr, int top, int blk) {
  for (int t = 0; t < top; t++) if (fr[t].blk == blk) return true;
  return false;
}

// Enumerate all chains of one (wait, counter).  Returns false on frame overflow.
LEO_DEV bool trace_waitcnt_one(const KView& k, int wait, int counter, int level, uint32_t members,
                               const SyncArgs& sa, Frame* fr, int fcap, int& best_m) {
  int32_t seen[16];
  int nseen = 0;
  const int b0 = k.block_of[wait];
  int m = 0, a = -1, budget = kSyncBudget;
  bool stopped = false;
  for (int x = wait - 1; x >= k.blk_first[b0]; x--) {
    if (budget == 0) { stopped = true; break; }
    budget--;
    if (!wc_visit(k, x, counter, members, level, wait, m, a, sa, seen, nseen, 16)) { stopped = true; break; }
  }
  best_m = 0;
  if (stopped) { best_m = m; return true; }
  int top = 0;
  fr[top++] = Frame{b0, k.pred_ptr[b0], m, a, budget};
  {
    bool any = false;
    for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) if (k.pred[q] != b0) any = true;
    if (!any) { best_m = m; return true; }
  }
  while (top > 0) {
    Frame& f = fr[top - 1];
    int p = -1;
    while (f.q < k.pred_ptr[f.blk + 1]) {
      int c = k.pred[f.q++];
      if (!on_path(fr, top, c)) { p = c; break; }
    }
    if (p < 0) { top--; continue; }
    m = f.m; a = f.a; budget = f.budget; stopped = false;
    for (int x = k.blk_last[p]; x >= k.blk_first[p]; x--) {
      if (budget == 0) { stopped = true; break; }
      budget--;
      if (!wc_visit(k, x, counter, members, level, wait, m, a, sa, seen, nseen, 16)) { stopped = true; break; }
    }
    if (stopped) { best_m = max(best_m, m); continue; }
    if (top == fcap) return false;
    fr[top++] = Frame{p, k.pred_ptr[p], m, a, budget};
    bool any = false;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1] && !any; q++)
      if (!on_path(fr, top, k.pred[q])) any = true;
    if (!any) { best_m = max(best_m, m); top--; }
  }
  return true;
}

LEO_DEV bool is_setter(const KView& k, int x, int kind, int id) {
  if (kind == LEO_EK_MEM_BARRIER)
    return k.sync_kind[x] == LEO_SYNC_BARRIER && (((k.sync_a[x] | (k.sync_a[x] >> 8)) >> id) & 1);
  return k.sync_kind[x] == LEO_SYNC_SWSB && k.sync_a[x] == (uint32_t)id;
}

// Setter search for one (wait, id).  Dijkstra state in (node, dist, done)
// arrays of capacity ncap.  Returns -1 on overflow, else found (0/1).
LEO_DEV int setter_search(const KView& k, int wait, int kind, int id, const SyncArgs& sa,
                          int32_t* node, int32_t* dist, uint8_t* done, int ncap) {
  const int b0 = k.block_of[wait];
  const int first0 = k.blk_first[b0];
  int lim = min(wait - first0, kSyncBudget);
  for (int x = wait - 1; x >= wait - lim; x--)
    if (is_setter(k, x, kind, id)) { sync_emit(sa, x, wait); return 1; }
  const int cost0 = wait - first0;
  if (cost0 >= kSyncBudget) return 0;
  int n = 0, found = 0;
  auto relax = [&](int blk, int d) -> bool {
    if (blk == b0) return true;
    for (int t = 0; t < n; t++)
      if (node[t] == blk) { if (!done[t] && d < dist[t]) dist[t] = d; return true; }
    if (n == ncap) return false;
    node[n] = blk; dist[n] = d; done[n] = 0; n++;
    return true;
  };
  for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++)
    if (!relax(k.pred[q], cost0)) return -1;
  while (true) {
    int best = -1;
    for (int t = 0; t < n; t++)
      if (!done[t] && (best < 0 || dist[t] < dist[best])) best = t;
    if (best < 0) break;
    done[best] = 1;
    const int p = node[best], d = dist[best];
    if (d >= kSyncBudget) break;                       // entering with no budget left
    int s = -1;
    for (int x = k.blk_last[p]; x >= k.blk_first[p]; x--)
      if (is_setter(k, x, kind, id)) { s = x; break; }
    if (s >= 0) {
      if (d + (k.blk_last[p] - s + 1) <= kSyncBudget) { sync_emit(sa, s, wait); found = 1; }
      continue;
    }
    const int nd = d + (k.blk_last[p] - k.blk_first[p] + 1);
    if (nd >= kSyncBudget) continue;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1]; q++)
      if (!relax(k.pred[q], nd)) return -1;
  }
  return found;
}

constexpr int kFrames = 24, kDij = 64;

__host__ __device__ inline size_t sync_slow_bytes_per_worker(int B) {
  return (((size_t)(B + 2) * (sizeof(Frame) + 9)) + 15) & ~(size_t)15;
}

// One thread per instruction; sub-items: amd counters 0/1, nvidia barriers
// 1..6, intel tokens 0..31.  Overflowing items go to the slow list.
template <bool SLOW>
__global__ void k_sync(KView k, SyncArgs a, int32_t* scratch, int nworkers) {
  const int dialect = k.dialect;
  int n_items, stride, start;
  if (SLOW) {
    n_items = min((int64_t)*a.slow_count, a.slow_cap);
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = nworkers;
    if (start >= nworkers) return;
  } else {
    n_items = k.N;
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = gridDim.x * blockDim.x;
  }
  Frame lfr[SLOW ? 1 : kFrames];
  int32_t lnode[SLOW ? 1 : kDij], ldist[SLOW ? 1 : kDij];
  uint8_t ldone[SLOW ? 1 : kDij];
  Frame* fr = lfr;
  int32_t *node = lnode, *dist = ldist;
  uint8_t* done = ldone;
  int fcap = kFrames, ncap = kDij;
  if (SLOW) {
    const size_t per = sync_slow_bytes_per_worker(k.B);
    char* base = (char*)scratch + (size_t)start * per;
    fr = (Frame*)base;
    node = (int32_t*)(base + (size_t)(k.B + 2) * sizeof(Frame));
    dist = node + (k.B + 2);
    done = (uint8_t*)(dist + (k.B + 2));
    fcap = k.B + 2; ncap = k.B + 2;
  }
  for (int t = start; t < n_items; t += stride) {
    int i, only = -1;
    if (SLOW) { int it = a.slow_list[t]; i = it >> 6; only = it & 63; }
    else i = t;
    if (dialect == LEO_AMD) {
      if (k.sync_kind[i] != LEO_SYNC_WAITCNT) continue;
      for (int counter = 0; counter < 2; counter++) {   // vmcnt before lgkmcnt (:410-415)
        if (only >= 0 && only != counter) continue;
        uint32_t lv = counter == 0 ? k.sync_a[i] : k.sync_b[i];
        if (lv == LEO_NONE_U32) continue;
        int best_m = 0;
        if (!trace_waitcnt_one(k, i, counter, (int)lv, counter == 0 ? kVmcnt : kLgkmcnt, a, fr, fcap, best_m)) {
          int s = atomicAdd(a.slow_count, 1);
          if (s < a.slow_cap) a.slow_list[s] = (i << 6) | counter;
          else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
          continue;
        }
        if (best_m < (int)lv) diag_push(a.diags, a.status, LEO_DIAG_WAITCNT, i, counter, (int)lv, best_m, counter);
      }
    } else {
      uint32_t mask;
      int kind;
      if (dialect == LEO_NVIDIA) {
        if (k.sync_kind[i] != LEO_SYNC_BARRIER) continue;
        mask = (k.sync_a[i] >> 16) & 0x7E;
        kind = LEO_EK_MEM_BARRIER;
      } else {
        if (k.sync_kind[i] != LEO_SYNC_SWSB) continue;
        mask = k.sync_b[i];
        kind = LEO_EK_MEM_SWSB;
      }
      while (mask) {
        int id = __ffs(mask) - 1;
        mask &= mask - 1;
        if (only >= 0 && only != id) continue;
        int f = setter_search(k, i, kind, id, a, node, dist, done, ncap);
        if (f < 0) {
          int s = atomicAdd(a.slow_count, 1);
          if (s < a.slow_cap) a.slow_list[s] = (i << 6) | id;
          else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
          continue;
        }
        if (!f) diag_push(a.diags, a.status, LEO_DIAG_NO_SETTER, i, id, 0, 0, id);
      }
    }
  }
}

template __global__ void k_sync<false>(KView, SyncArgs, int32_t*, int);
template __global__ void k_sync<true>(KView, SyncArgs, int32_t*, int);

// ---- group raw keys by producer, dedup, append after the raw/guard edges ----
__global__ void k_key_hist(const uint64_t* __restrict__ keys, const int32_t* n_dev, int64_t cap,
                           int32_t* __restrict__ cnt) {
  int64_t n = min((int64_t)*n_dev, cap);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[(int)(keys[x] >> 32)], 1);
}
__global__ void k_key_scatter(const uint64_t* __restrict__ keys, const int32_t* n_dev, int64_t cap,
                              const int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                              uint64_t* __restrict__ out) {
  int64_t n = min((int64_t)*n_dev, cap);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(keys[x] >> 32);
    out[off[p] + atomicAdd(&cursor[p], 1)] = keys[x];
  }
}
__global__ void k_sync_emit(int N, int kind, const uint64_t* __restrict__ sorted,
                            const int32_t* __restrict__ off, const int32_t* __restrict__ uniq,
                            const int32_t* __restrict__ uoff, const int32_t* n_regular,
                            LeoEdges out, uint32_t* status) {
  const int base = *n_regular;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    int n = uniq[p], o = base + uoff[p];
    if (o + n > out.capacity) { if (n) atomicOr(status, (uint32_t)LEO_ST_EDGE_OVERFLOW); continue; }
    for (int x = 0; x < n; x++) {
      uint64_t key = sorted[off[p] + x];
      out.prod[o + x] = p;
      out.cons[o + x] = (int)(uint32_t)key;
      out.meta[o + x] = LEO_META(kind, LEO_DC_MEMORY, 0);
    }
  }
}
// counts are clamped to the capacity so downstream kernels never read past the
// buffers; an overflow is signalled in the status word and the host re-runs.
__global__ void k_edge_totals(const int32_t* n_regular, const int32_t* n_sync, LeoEdges out, uint32_t* status) {
  int r = *n_regular, t = *n_regular + *n_sync;
  if (t > out.capacity) atomicOr(status, (uint32_t)LEO_ST_EDGE_OVERFLOW);
  *out.n_regular = min(r, out.capacity);
  *out.count = min(t, out.capacity);
}

}  // namespace leo
