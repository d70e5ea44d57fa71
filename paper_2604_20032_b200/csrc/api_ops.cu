// api_ops.cu — device ops behind the reference-compatible stage functions of
// api.py that run outside the fused pipeline (the drop-in boundary for the
// reference's own call patterns: chained stages, hand-built graphs, the
// dataflow sub-steps, self_blame of any instruction).
//
//   k_gather_edges    arbitrary-order edge list -> consumer-sorted copy (stable):
//                     the base graph's RAW CSR for the indirect-addressing
//                     test (analysis.py:390-411) of a hand-built base graph
//   k_copy_pool       prune of an already-pruned graph: the input valid_paths
//                     pool is carried to the output (kept edges keep their
//                     PathRecords, analysis.py:143-299)
//   k_edge_dist       _edge_distance (analysis.py:371-376) of any edge list
//   k_self_entries    self_blame (analysis.py:414-428) of given instructions
//   k_live_*          liveness (depgraph.py:235-271) as a bit-parallel
//                     backward fixed point, one thread per 32-unit word, and
//                     liveness_filter (:274-293) thread per link
//   k_reach_claim_all reaching_definitions (:135-177) for every (block, unit):
//                     the production query search run on all pairs, exported
//                     as a CSR of reach-in sets
//   k_line_flag / k_line_scatter  the per-line totals as a sparse list (the
//                     lines a kernel touches), stable order, for read-back
#include "prims.cuh"

namespace leo {

__global__ void k_line_flag(int n, const double* __restrict__ lb, const double* __restrict__ ls,
                            int32_t* __restrict__ flag) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    flag[x] = (lb[x] != 0.0 || ls[x] != 0.0) ? 1 : 0;
}

__global__ void k_line_scatter(int n, const double* __restrict__ lb, const double* __restrict__ ls,
                               const int32_t* __restrict__ off, int32_t cap, int32_t* __restrict__ ids,
                               double* __restrict__ lb_out, double* __restrict__ ls_out, int32_t* count) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int o = off[x];
    if (off[x + 1] != o && o < cap) { ids[o] = x; lb_out[o] = lb[x]; ls_out[o] = ls[x]; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = off[n];
}

__global__ void k_gather_edges(const int32_t* __restrict__ n_dev, const uint64_t* __restrict__ idx,
                               const int32_t* __restrict__ prod, const int32_t* __restrict__ cons,
                               const uint32_t* __restrict__ meta, LeoEdges out) {
  pdl_wait();
  const int n = min(*n_dev, out.capacity);
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int e = (int)idx[x];
    out.prod[x] = prod[e];
    out.cons[x] = cons[e];
    out.meta[x] = meta[e];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { *out.count = n; *out.n_regular = n; }
}

__global__ void k_copy_pool(LeoPaths in, LeoPaths out, uint32_t* status) {
  pdl_wait();
  const int n = *in.count;
  const int m = min(n, out.capacity);
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) {
    out.len[x] = in.len[x];
    out.accum[x] = in.accum[x];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out.count = n;                       // new records are reserved after the carried ones
    if (n > out.capacity) atomicOr(status, (uint32_t)LEO_ST_PATH_OVERFLOW);
  }
}

// mean valid-path length, else max(1, |consumer - producer|)
__global__ void k_edge_dist(const int32_t* __restrict__ n_dev, int32_t cap, const int32_t* __restrict__ prod,
                            const int32_t* __restrict__ cons, LeoPaths paths, double* __restrict__ dist) {
  pdl_wait();
  const int n = min(*n_dev, cap);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int np = paths.npaths ? paths.npaths[e] : 0;
    if (np > 0) {
      const int f = paths.first[e];
      int64_t s = 0;
      for (int q = 0; q < np; q++) s += paths.len[f + q];
      dist[e] = __ddiv_rn((double)s, (double)np);
    } else {
      int d = cons[e] - prod[e];
      if (d < 0) d = -d;
      dist[e] = (double)(d < 1 ? 1 : d);
    }
  }
}

__global__ void k_self_entries(KView k, PView p, const uint8_t* __restrict__ mp_ok, int n,
                               const int32_t* __restrict__ idx, uint8_t* __restrict__ sub,
                               double* __restrict__ cycles) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int j = idx[x];
    int s = dominant_self(p, j);
    if (s == LEO_SB_MEMORY_LATENCY && (kMemoryClasses & BIT(k.opclass[j])) && mp_ok && mp_ok[j])
      s = LEO_SB_INDIRECT_ADDRESSING;
    sub[x] = (uint8_t)s;
    cycles[x] = (double)((int64_t)p.lat[j] * p.period);
  }
}

// ---- liveness ------------------------------------------------------------------
// gen[b] = units used before any in-block definition, kill[b] = units defined
// in the block (depgraph.py:239-251); rows of W words per block.
__global__ void k_live_genkill(KView k, int W, uint32_t* __restrict__ gen, uint32_t* __restrict__ kill) {
  pdl_wait();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < k.B; b += gridDim.x * blockDim.x) {
    uint32_t* g = gen + (size_t)b * W;
    uint32_t* kl = kill + (size_t)b * W;
    for (int w = 0; w < W; w++) { g[w] = 0u; kl[w] = 0u; }
    for (int i = k.blk_first[b]; i <= k.blk_last[b]; i++) {
      const int q0 = k.opnd_ptr[i], q1 = k.opnd_ptr[i + 1];
      for (int q = q0; q < q1; q++) {                 // uses (srcs, guard) first
        const uint32_t r = k.opnd[q];
        if (op_role(r) == LEO_ROLE_DST) continue;
        const int u0 = unit_of(k, r);
        for (int u = u0; u < u0 + op_span(r); u++)
          if (!(kl[u >> 5] & (1u << (u & 31)))) g[u >> 5] |= 1u << (u & 31);
      }
      for (int q = q0; q < q1; q++) {                 // then the instruction's defs
        const uint32_t r = k.opnd[q];
        if (op_role(r) != LEO_ROLE_DST) continue;
        const int u0 = unit_of(k, r);
        for (int u = u0; u < u0 + op_span(r); u++) kl[u >> 5] |= 1u << (u & 31);
      }
    }
  }
}

// Least fixed point of live_in = gen | (live_out & ~kill), live_out = OR of
// the successors' live_in: every 32-unit word is an independent bit-parallel
// problem; its thread sweeps the blocks in reverse layout order (in place,
// Gauss-Seidel) until a sweep changes nothing.  Monotone from all-zero, so the
// result is the same least fixed point the reference's worklist reaches.
__global__ void k_live_solve(KView k, int W, const uint32_t* __restrict__ gen, const uint32_t* __restrict__ kill,
                             uint32_t* __restrict__ live_in, uint32_t* __restrict__ live_out) {
  pdl_wait();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  for (int b = 0; b < k.B; b++) { live_in[(size_t)b * W + w] = 0u; live_out[(size_t)b * W + w] = 0u; }
  bool changed = true;
  while (changed) {
    changed = false;
    for (int b = k.B - 1; b >= 0; b--) {
      uint32_t out = 0u;
      for (int q = k.succ_ptr[b]; q < k.succ_ptr[b + 1]; q++) out |= live_in[(size_t)k.succ[q] * W + w];
      live_out[(size_t)b * W + w] = out;
      const uint32_t nin = gen[(size_t)b * W + w] | (out & ~kill[(size_t)b * W + w]);
      if (nin != live_in[(size_t)b * W + w]) { live_in[(size_t)b * W + w] = nin; changed = true; }
    }
  }
}

// keep a link iff same block, or (use ∩ written, else use) meets live_out[pb]
__global__ void k_live_filter(KView k, int W, const uint32_t* __restrict__ live_out, const int32_t* __restrict__ n_dev,
                              int32_t cap, const int32_t* __restrict__ prod, const int32_t* __restrict__ cons,
                              const uint32_t* __restrict__ meta, uint8_t* __restrict__ keep) {
  pdl_wait();
  const int n = min(*n_dev, cap);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int p = prod[e], c = cons[e];
    const int pb = k.block_of[p], cb = k.block_of[c];
    if (pb == cb) { keep[e] = 1; continue; }
    const uint32_t ref = meta[e] & 0x07FFFFFFu;
    const int u0 = unit_of(k, ref), sp = op_span(ref);
    // written = units of the producer's destination operands
    bool any_written = false;
    for (int u = u0; u < u0 + sp && !any_written; u++)
      for (int q = k.opnd_ptr[p]; q < k.opnd_ptr[p + 1]; q++) {
        const uint32_t r = k.opnd[q];
        if (op_role(r) != LEO_ROLE_DST) continue;
        const int d0 = unit_of(k, r);
        if (u >= d0 && u < d0 + op_span(r)) { any_written = true; break; }
      }
    const uint32_t* lo = live_out + (size_t)pb * W;
    bool live = false;
    for (int u = u0; u < u0 + sp && !live; u++) {
      bool in_link = true;
      if (any_written) {
        in_link = false;
        for (int q = k.opnd_ptr[p]; q < k.opnd_ptr[p + 1]; q++) {
          const uint32_t r = k.opnd[q];
          if (op_role(r) != LEO_ROLE_DST) continue;
          const int d0 = unit_of(k, r);
          if (u >= d0 && u < d0 + op_span(r)) { in_link = true; break; }
        }
      }
      if (in_link && (lo[u >> 5] & (1u << (u & 31)))) live = true;
    }
    keep[e] = live ? 1 : 0;
  }
}

// ---- reaching_definitions for every (block, unit) --------------------------------
// After the block walk: every (b, u) pair without an upward-exposed query gets
// one (slot NU + b*U + u), so the production reach tiers answer all pairs.
__global__ void k_reach_claim_all(KView k, int Bp, int64_t nu, int32_t* __restrict__ qtab,
                                  int32_t* __restrict__ q_block, int32_t* __restrict__ q_unit,
                                  int32_t* __restrict__ q_list, int32_t* __restrict__ q_count) {
  pdl_wait();
  const int64_t n = (int64_t)k.B * k.U;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(x / k.U), u = (int)(x % k.U);
    int32_t* cell = qtab + (size_t)u * Bp + b;
    if (*cell >= 0) continue;
    const int slot = (int)(nu + x);
    *cell = slot;
    q_block[slot] = b;
    q_unit[slot] = u;
    if (q_list) q_list[atomicAdd(q_count, 1)] = slot;
  }
}

__global__ void k_reach_export_count(KView k, int Bp, const int32_t* __restrict__ qtab,
                                     const int32_t* __restrict__ q_len, int32_t* __restrict__ cnt) {
  pdl_wait();
  const int64_t n = (int64_t)k.B * k.U;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(x / k.U), u = (int)(x % k.U);
    const int slot = qtab[(size_t)u * Bp + b];
    cnt[x] = slot >= 0 ? q_len[slot] : 0;
  }
}

__global__ void k_reach_export_fill(KView k, int Bp, const int32_t* __restrict__ qtab,
                                    const int32_t* __restrict__ q_off, const int32_t* __restrict__ q_len,
                                    const int32_t* __restrict__ qres, LeoReachIn out, uint32_t* status) {
  pdl_wait();
  const int64_t n = (int64_t)k.B * k.U;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(x / k.U), u = (int)(x % k.U);
    const int slot = qtab[(size_t)u * Bp + b];
    if (slot < 0) continue;
    const int o = out.set_off[x], m = q_len[slot], s = q_off[slot];
    if ((int64_t)o + m > out.capacity) { atomicOr(status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); continue; }
    for (int t = 0; t < m; t++) out.defs[o + t] = qres[s + t];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out.count = out.set_off[n];
}

}  // namespace leo

namespace leo {
// ---- trace_chain over an arbitrary blame-entry list (analysis.py:499-538) -------
__global__ void k_chain_prep(int start, int n_entries, int32_t* one, int32_t* ncount, int32_t* zero4) {
  if (threadIdx.x == 0) {
    one[0] = 1; one[1] = start;
    *ncount = n_entries;
    zero4[0] = 0; zero4[1] = 0; zero4[2] = 0; zero4[3] = 0;
  }
}
// entries in stalled-grouped order: x-th sorted entry = input entry perm[x];
// its "edge" is itself (-1 for a self entry), its producer the cause
__global__ void k_chain_gather(int n, const uint64_t* __restrict__ perm, const int32_t* __restrict__ stalled,
                               const int32_t* __restrict__ cause, const double* __restrict__ blame,
                               int32_t* __restrict__ sst, int32_t* __restrict__ sedge, int32_t* __restrict__ sprod,
                               double* __restrict__ sbl) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int e = (int)perm[x];
    sst[x] = stalled[e];
    sprod[x] = cause[e];
    sedge[x] = cause[e] < 0 ? -1 : x;
    sbl[x] = blame[e];
  }
}
__global__ void k_chain_unperm(const uint64_t* __restrict__ perm, const int32_t* __restrict__ len,
                               const int32_t* __restrict__ ent, const int32_t* __restrict__ self,
                               int32_t* __restrict__ chain_entry, int32_t* __restrict__ chain_self) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  for (int t = 0; t < *len; t++) chain_entry[t] = ent[t] < 0 ? -1 : (int)perm[ent[t]];
  *chain_self = *self >= 0 ? (int)perm[*self] : -1;
}
}  // namespace leo

namespace leo {
// per-line rollup of an arbitrary blame-entry list: entry x's "edge" is itself
__global__ void k_entry_edges(int n, const int32_t* __restrict__ cause, int32_t* __restrict__ edge, int32_t* count) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
    edge[x] = cause[x] < 0 ? -1 : x;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = n;
}
}  // namespace leo
