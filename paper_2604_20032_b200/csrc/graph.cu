// graph.cu — register dependency edges (reaching definitions + per-use link).
//
// Replaces depgraph.reaching_definitions (depgraph.py:135-177), per_use_link
// (:188-223), liveness_filter (:274-293; identity on pipeline output, see
// DESIGN.md) and the raw/guard half of build_graph (:510-524).
//
// Device algorithm
//   G0 k_unit_counts   thread/instr: use-unit and def-unit counts -> scans
//   G1 k_block_walk    warp/basic block: every use-unit event resolves to its
//                      in-block reaching def, or to the upward-exposed (block,
//                      unit) query led by the block's first use of the unit.
//                      Blocks of <= 32 instructions are staged and resolved in
//                      parallel (one lane per use event against the staged def
//                      list); longer blocks walk in order over a per-warp unit
//                      table.  Writes the block's last defs and led queries
//                      into the -1-initialised [U][B] unit columns (sparse:
//                      one write per last def / query, not per unit).
//   G2 k_reach         thread/query: backward search over predecessor blocks
//                      through blocks transparent to the unit; the union of the
//                      last defs of the defining blocks reached is exactly the
//                      least fixed point reach_in(b)[u] of the reference's
//                      worklist.  Overflowing searches re-run on global scratch.
//   G3/G4 k_link_*     thread/consumer: count, then write candidate keys
//                      (producer, kind, class rank, index, span)
//   G5 segsort_unique  per consumer: reference sort order + dedup on the full key
//   G6 k_link_emit     edges in (consumer, producer, kind, class, index, span) order
#include "prims.cuh"
#include "stage.cuh"

namespace leo {

LEO_DEV int warp_incl_max(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, t);
  }
  return v;
}

// Per-instruction use/def unit counts, and in the same launch the
// fallthrough-run records of the blocks (both only read the kernel SoA).
//
// Fallthrough runs: runhead(b) = first block of the maximal run ending at b in
// which every block but the first has exactly one predecessor, the previous
// block.  A backward search entering the run at y can only leave it through
// preds(runhead(y)), so a run is resolved with independent loads of the dense
// last-def table instead of one search level per block.  runhead is an
// inclusive max-scan of (b starts a run ? b : -1) over the CTA's blocks; only
// the run entering the CTA's range from below is walked serially (one thread).
//
// Block record (one 16-byte load per search step):
//   rec[y] = {h = runhead(y), np = |preds(h)|, p0, p1}
//   np <= 2: p0/p1 are the predecessors of h; np > 2: p0 = pred_ptr[h].
__global__ void k_unit_counts(KView k, int32_t* __restrict__ ucnt, int32_t* __restrict__ dcnt,
                              int4* __restrict__ rec, int32_t* __restrict__ rh) {
  pdl_wait();
  __shared__ int sw[33];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k.N; i += gridDim.x * blockDim.x) {
    int u = 0, d = 0;
    for (int q = k.opnd_ptr[i]; q < k.opnd_ptr[i + 1]; q++) {
      uint32_t r = k.opnd[q];
      if (op_role(r) == LEO_ROLE_DST) d += op_span(r); else u += op_span(r);
    }
    ucnt[i] = u;
    dcnt[i] = d;
  }
  if (!rec) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b0 = blockIdx.x * blockDim.x; b0 < k.B; b0 += gridDim.x * blockDim.x) {
    const int b = b0 + threadIdx.x;
    bool cont = false;
    if (b < k.B && b > 0) {
      const int q0 = k.pred_ptr[b];
      cont = k.pred_ptr[b + 1] - q0 == 1 && k.pred[q0] == b - 1;
    }
    int h = warp_incl_max(cont || b >= k.B ? -1 : b);
    if (lane == 31) sw[warp] = h;
    __syncthreads();
    if (warp == 0) {
      const int w = warp_incl_max(lane < nw ? sw[lane] : -1);
      if (lane < nw) sw[lane] = w;
    }
    if (threadIdx.x == 0) {
      // head of the run entering from below b0
      int x = b0;
      if (cont)
        while (x > 0 && k.pred_ptr[x + 1] - k.pred_ptr[x] == 1 && k.pred[k.pred_ptr[x]] == x - 1) x--;
      sw[32] = x;
    }
    __syncthreads();
    if (warp > 0) h = max(h, sw[warp - 1]);
    if (h < 0) h = sw[32];
    if (b < k.B) {
      const int q0 = k.pred_ptr[h], np = k.pred_ptr[h + 1] - q0;
      int4 r;
      r.x = h; r.y = np;
      if (np <= 2) { r.z = np > 0 ? k.pred[q0] : -1; r.w = np > 1 ? k.pred[q0 + 1] : -1; }
      else { r.z = q0; r.w = -1; }
      rec[b] = r;
      rh[b] = h;
    }
    __syncthreads();
  }
}

// unit of the x-th use-unit (or def-unit when `defs`) event of instruction i
LEO_DEV int event_unit(const KView& k, int i, int x, bool defs, int* opos, uint32_t* oref) {
  for (int q = k.opnd_ptr[i]; q < k.opnd_ptr[i + 1]; q++) {
    uint32_t r = k.opnd[q];
    bool is_def = op_role(r) == LEO_ROLE_DST;
    if (is_def != defs) continue;
    int s = op_span(r);
    if (x < s) { *opos = q - k.opnd_ptr[i]; *oref = r; return unit_of(k, r) + x; }
    x -= s;
  }
  return -1;
}

struct WalkArgs {
  const int32_t* use_ptr;    // [N+1]
  const int32_t* def_ptr;    // [N+1]
  int32_t* ev_res;           // [use units] def (>=0) or -(query slot+1)
  int32_t* q_block;          // [use units]
  int32_t* q_unit;           // [use units]
  int32_t* q_list;           // [use units]
  int32_t* q_count;          // scalar
  int32_t* ldtab;            // [U * Bp] column-major: last def of unit u in block b, -1 if none
  int32_t* qtab;             // [U * Bp] column-major: query slot of (b, u), -1 if none
  int32_t Bp;                // column stride (B rounded up to 4: 16-byte aligned columns)
  int32_t* gtab;             // global per-warp tables (when U too large for smem) or null
};

// per-warp staging of a window of <= 32 instructions' unit events
constexpr int kWalkUse = 384, kWalkDef = 192, kWalkLeads = 64;
constexpr int kWalkStage = 2 * kWalkUse + 2 * kWalkDef + kWalkLeads;   // units + their instructions

// warp per block; blocks visited in increasing order per warp so that stale
// table entries (from earlier blocks) are recognisable by index comparison.
// The block's instructions are taken 32 at a time: one lane per instruction
// loads its event offsets and expands its operands into per-warp unit lists
// (independent loads), then the in-order walk runs on shared memory only.
// New query slots are buffered per warp and published with one atomic.
__global__ void k_block_walk(KView k, WalkArgs a, int warps_per_cta) {
  pdl_wait();
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * warps_per_cta + wid, nw = gridDim.x * warps_per_cta;
  const int U = k.U;
  int32_t* wsm = smem + (size_t)wid * ((a.gtab ? 0 : 4 * U) + kWalkStage);
  int32_t* last = a.gtab ? a.gtab + (size_t)gw * 2 * U : wsm;
  int32_t* qtab = last + U;
  // parallel path (shared-memory tables only): per unit, the mask of the
  // block's instructions defining it and its first use event in the block
  uint32_t* dmask = a.gtab ? nullptr : reinterpret_cast<uint32_t*>(wsm + 2 * U);
  int32_t* fuse = a.gtab ? nullptr : wsm + 3 * U;
  int32_t* evu = a.gtab ? wsm : wsm + 4 * U;
  int32_t* evd = evu + kWalkUse;
  int32_t* evui = evd + kWalkDef;                  // instruction of each staged use / def unit
  int32_t* evdi = evui + kWalkUse;
  int32_t* leads = evdi + kWalkDef;
  int nlead = 0;                                   // warp-uniform
  const unsigned lt = (1u << lane) - 1;
  auto publish = [&]() {
    int qbase = 0;
    if (lane == 0) qbase = atomicAdd(a.q_count, nlead);
    qbase = __shfl_sync(0xffffffffu, qbase, 0);
    for (int x = lane; x < nlead; x += 32) a.q_list[qbase + x] = leads[x];
    nlead = 0;
    __syncwarp();
  };
  for (int u = lane; u < U; u += 32) { last[u] = -1; qtab[u] = -1; }
  if (dmask)
    for (int u = lane; u < U; u += 32) { dmask[u] = 0u; fuse[u] = INT_MAX; }
  __syncwarp();
  for (int b = gw; b < k.B; b += nw) {
    const int first = k.blk_first[b], lastI = k.blk_last[b];
    const int ev_block = a.use_ptr[first];
    bool par = false;                              // block resolved by the parallel path
    for (int w0 = first; w0 <= lastI; w0 += 32) {
      const int i = w0 + lane, nin = min(32, lastI - w0 + 1);
      const bool in = lane < nin;
      int u0 = 0, u1 = 0, d0 = 0, d1 = 0, q0 = 0, q1 = 0;
      if (in) {
        u0 = a.use_ptr[i]; u1 = a.use_ptr[i + 1];
        d0 = a.def_ptr[i]; d1 = a.def_ptr[i + 1];
        q0 = k.opnd_ptr[i]; q1 = k.opnd_ptr[i + 1];
      }
      const int ub = __shfl_sync(0xffffffffu, u0, 0), ue = __shfl_sync(0xffffffffu, u1, nin - 1);
      const int db = __shfl_sync(0xffffffffu, d0, 0), de = __shfl_sync(0xffffffffu, d1, nin - 1);
      const bool staged = ue - ub <= kWalkUse && de - db <= kWalkDef;
      if (staged && in) {
        int pu = u0 - ub, pd = d0 - db;
        for (int q = q0; q < q1; q++) {
          const uint32_t r = k.opnd[q];
          const int s = op_span(r), base = unit_of(k, r);
          if (op_role(r) == LEO_ROLE_DST) { for (int x = 0; x < s; x++) { evdi[pd] = i; evd[pd++] = base + x; } }
          else { for (int x = 0; x < s; x++) { evui[pu] = i; evu[pu++] = base + x; } }
        }
      }
      __syncwarp();
      if (dmask && staged && w0 == first && lastI - first < 32) {
        // The whole block is staged: every use event is resolved in parallel.
        // dmask[u] = the block's instructions defining u (bit i - first);
        // fuse[u] = u's first use event.  A use at i reads the highest def bit
        // below i (uses read before the same instruction's defs); with none it
        // joins the (block, unit) query led by u's first use, which is then
        // upward-exposed too.  Last defs and led queries are written sparsely.
        par = true;
        const int nu = ue - ub, nd = de - db;
        for (int y = lane; y < nd; y += 32) atomicOr(&dmask[evd[y]], 1u << (evdi[y] - first));
        for (int x = lane; x < nu; x += 32) atomicMin(&fuse[evu[x]], x);
        __syncwarp();
        for (int x0 = 0; x0 < nu; x0 += 32) {
          const int x = x0 + lane;
          bool lead = false;
          if (x < nu) {
            const int u = evu[x], i = evui[x];
            const uint32_t m = dmask[u] & ((1u << (i - first)) - 1u);
            int res;
            if (m) {
              res = first + 31 - __clz(m);
            } else {
              const int l = fuse[u];
              lead = l == x;
              res = -(ub + l + 1);
              if (lead) {
                a.q_block[ub + x] = b;
                a.q_unit[ub + x] = u;
                a.qtab[(size_t)u * a.Bp + b] = ub + x;
              }
            }
            a.ev_res[ub + x] = res;
          }
          if (a.q_list) {
            const unsigned lm = __ballot_sync(0xffffffffu, lead);
            if (lm) {
              if (nlead + __popc(lm) > kWalkLeads) publish();
              if (lead) leads[nlead + __popc(lm & lt)] = ub + x;
              nlead += __popc(lm);
            }
          }
        }
        for (int y = lane; y < nd; y += 32) {
          const int u = evd[y], i = evdi[y];
          if (first + 31 - __clz(dmask[u]) == i) a.ldtab[(size_t)u * a.Bp + b] = i;
        }
        __syncwarp();
        for (int y = lane; y < nd; y += 32) dmask[evd[y]] = 0u;
        for (int x = lane; x < nu; x += 32) fuse[evu[x]] = INT_MAX;
        __syncwarp();
        continue;
      }
      for (int j = 0; j < nin; j++) {
        const int ii = w0 + j;
        const int e0 = __shfl_sync(0xffffffffu, u0, j), e1 = __shfl_sync(0xffffffffu, u1, j);
        for (int base = e0; base < e1; base += 32) {
          const int e = base + lane;
          const bool valid = e < e1;
          int u = -1, res = 0;
          bool fresh = false;
          if (valid) {
            if (staged) u = evu[e - ub];
            else { int opos; uint32_t oref; u = event_unit(k, ii, e - e0, false, &opos, &oref); }
            const int ld = last[u];
            if (ld >= first) res = ld;
            else if (qtab[u] >= ev_block) res = -(qtab[u] + 1);
            else fresh = true;
          }
          // first claimant of (block, unit) creates the query: qtab[u] still
          // holds a stale slot (< ev_block) until one lane's CAS replaces it
          bool lead = false;
          if (fresh) {
            const int seen = qtab[u];
            const int prev = atomicCAS(&qtab[u], seen, e);
            if (prev == seen) { lead = true; res = -(e + 1); }
            else res = -(prev + 1);          // another lane of this chunk claimed it
          }
          if (a.q_list) {                  // the query list feeds tier 1 only
            const unsigned lm = __ballot_sync(0xffffffffu, lead);
            if (lm) {
              if (nlead + __popc(lm) > kWalkLeads) publish();
              if (lead) leads[nlead + __popc(lm & lt)] = e;
              nlead += __popc(lm);
            }
          }
          if (lead) {
            a.q_block[e] = b;
            a.q_unit[e] = u;
          }
          if (valid) a.ev_res[e] = res;
          __syncwarp();
        }
        const int f0 = __shfl_sync(0xffffffffu, d0, j), f1 = __shfl_sync(0xffffffffu, d1, j);
        for (int d = f0 + lane; d < f1; d += 32) {
          int u;
          if (staged) u = evd[d - db];
          else { int opos; uint32_t oref; u = event_unit(k, ii, d - f0, true, &opos, &oref); }
          last[u] = ii;
        }
        __syncwarp();
      }
    }
    // the block's last definitions (block_defs depgraph.py:143-149) and its
    // upward-exposed queries into the (-1 initialised) unit columns
    if (!par) {
      for (int u = lane; u < U; u += 32) {
        const int ld = last[u], qs = qtab[u];
        if (ld >= first) a.ldtab[(size_t)u * a.Bp + b] = ld;
        if (qs >= ev_block) a.qtab[(size_t)u * a.Bp + b] = qs;
      }
    }
    __syncwarp();
  }
  if (a.q_list && nlead) publish();
}

struct ReachArgs {
  int32_t dbg;               // LEO_DBG_* routing (testing)
  const int32_t* ldtab;      // [U * Bp] column-major
  const int4* rec;           // [B]
  int32_t U;
  int32_t Bp;
  const int32_t* q_block;
  const int32_t* q_unit;
  int32_t* q_off;            // [use units] result offset per query slot
  int32_t* q_len;            // [use units]
  int32_t* qres;             // results pool
  int64_t qres_cap;
  int32_t* qres_count;
  int32_t* slow_list;
  int32_t* slow_count;
  int64_t slow_cap;
  uint32_t* status;
};

// Entering block y backward: the nearest definition of u in y, y-1, ...,
// runhead(y) (loads issued four at a time), or -1.
LEO_DEV int run_lookup(const ReachArgs& a, int y, int h, int u) {
  const int32_t* col = a.ldtab + (size_t)u * a.Bp;
  for (int x = y; x >= h; x -= 4) {
    int v0 = col[x];
    int v1 = x - 1 >= h ? col[x - 1] : -1;
    int v2 = x - 2 >= h ? col[x - 2] : -1;
    int v3 = x - 3 >= h ? col[x - 3] : -1;
    if (v0 >= 0) return v0;
    if (v1 >= 0) return v1;
    if (v2 >= 0) return v2;
    if (v3 >= 0) return v3;
  }
  return -1;
}

// Visited-set policies for the search: a private open-addressing hash
// (shared memory, strided per thread) or a stamp array in global scratch.
struct SmemHash {
  int32_t* h; int stride, cap, n, limit;
  LEO_DEV void clear() { for (int s = 0; s < cap; s++) h[s * stride] = -1; n = 0; }
  LEO_DEV int insert(int key) {            // 1 new, 0 seen, -1 overflow
    int s = (int)(((uint32_t)key * 2654435761u) >> 26) & (cap - 1);
    for (int probe = 0; probe < cap; probe++) {
      int v = h[s * stride];
      if (v == key) return 0;
      if (v == -1) {
        if (n == limit) return -1;
        h[s * stride] = key; n++;
        return 1;
      }
      s = (s + 1) & (cap - 1);
    }
    return -1;
  }
};
struct StampSet {
  int32_t* stamp; int val;
  LEO_DEV int insert(int key) { if (stamp[key] == val) return 0; stamp[key] = val; return 1; }
};

// Backward search for query (b, u) over run-contracted blocks.  Returns false
// when a buffer overflowed (the caller re-runs the query on a larger tier).
template <class Visited>
LEO_DEV bool reach_search(const KView& k, const ReachArgs& a, int b, int u, Visited& vis,
                          int32_t* stk, int scap, int32_t* res, int rcap, int* nres_out) {
  int sp = 0, nres = 0;
  for (int q = k.pred_ptr[b]; q < k.pred_ptr[b + 1]; q++) {
    int p = k.pred[q];
    int v = vis.insert(p);
    if (v < 0) return false;
    if (v) { if (sp == scap) return false; stk[sp++] = p; }
  }
  while (sp > 0) {
    const int y = stk[--sp];
    const int4 r = a.rec[y];
    const int ld = run_lookup(a, y, r.x, u);
    if (ld >= 0) {
      if (nres == rcap) return false;
      res[nres++] = ld;
      continue;
    }
    const int np = r.y;
    for (int t = 0; t < np; t++) {
      const int pp = np <= 2 ? (t == 0 ? r.z : r.w) : k.pred[r.z + t];
      int v = vis.insert(pp);
      if (v < 0) return false;
      if (v) { if (sp == scap) return false; stk[sp++] = pp; }
    }
  }
  *nres_out = nres;
  return true;
}

LEO_DEV void reach_commit(const ReachArgs& a, int e, const int32_t* res, int nres) {
  int off = atomicAdd(a.qres_count, nres);
  if ((int64_t)off + nres > a.qres_cap) {
    atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
    a.q_off[e] = 0; a.q_len[e] = 0;
    return;
  }
  for (int x = 0; x < nres; x++) a.qres[off + x] = res[x];
  a.q_off[e] = off;
  a.q_len[e] = nres;
}

// Tier 0 (shared-memory resident): one CTA per register unit.  The CTA stages
// the unit's last-def and query columns plus the block -> run-head map and the
// predecessor CSR with TMA bulk copies, turns the last-def column into
// near[y] = nearest def of u in [runhead(y), y] (or -(runhead + 1) when that
// stretch of the run is transparent), and resolves every (b, u) query of the
// unit by a thread-private DFS whose visited set is a bitmap over blocks in
// shared memory.  Every search step is a shared-memory access.  Queries whose
// stack or result list overflows go to tier 2.
#ifndef LEO_RU_STACK
#define LEO_RU_STACK 16          // per-thread DFS stack / results of tier 0: 2 CTAs per SM at C4 members (-11 %)
#endif
constexpr int kRUStack = LEO_RU_STACK, kRURes = LEO_RU_STACK;

__host__ __device__ inline size_t reach_unit_smem(int B, int threads) {
  const size_t Bp = (size_t)((B + 3) & ~3);
  const size_t W = (size_t)((B + 31) >> 5);
  return 16 + carve_bytes(Bp, 4) * 4                                    // rh, cell, qs, qlist
         + carve_bytes(B + 1, 4) + carve_bytes(2 * (size_t)B + 4, 4)    // pred_ptr, pred (<= 2 per block)
         + carve_bytes(W * threads, 4)                                  // visited bitmaps
         + carve_bytes((size_t)kRUStack * threads, 4) + carve_bytes((size_t)kRURes * threads, 4);
}

// `parts` CTAs share one unit (each takes every parts-th query) so that
// kernels with few register units still fill the chip.
// Segments (LeoKernel.seg_block): a concatenated batch of independent
// kernels is staged one member kernel at a time (per_seg CTAs per segment,
// block ids rebased to the segment); bcap = largest segment's block count.
__global__ void k_reach_unit(KView k, ReachArgs a, const int32_t* __restrict__ qtab,
                             const int32_t* __restrict__ rh_g, int parts,
                             const int32_t* __restrict__ seg_block, int per_seg, int bcap) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  __shared__ int nq, rbase;
  __shared__ int swarp[33];
  __shared__ long long wmax[32];
  const int Bp = a.Bp, T = blockDim.x, tid = threadIdx.x;
  const int seg = blockIdx.x / per_seg, lcta = blockIdx.x % per_seg;
  const int sb0 = seg_block ? seg_block[seg] : 0, sb1 = seg_block ? seg_block[seg + 1] : k.B;
  const int B = sb1 - sb0, W = (B + 31) >> 5;
  const int Bcp = (bcap + 3) & ~3, Wc = (bcap + 31) >> 5;
  const int P0 = k.pred_ptr[sb0], P1 = k.pred_ptr[sb1];
  SmemCarve cv{sm_raw};
  uint64_t* bar = cv.take<uint64_t>(2);
  int32_t* rh = cv.take<int32_t>(Bcp);
  int32_t* cell = cv.take<int32_t>(Bcp);
  int32_t* qs = cv.take<int32_t>(Bcp);
  int32_t* ql = cv.take<int32_t>(Bcp);
  int32_t* pptr = cv.take<int32_t>(bcap + 1);
  int32_t* pred = cv.take<int32_t>(2 * (size_t)bcap + 4);
  uint32_t* vis = cv.take<uint32_t>((size_t)Wc * T);
  int32_t* stk = cv.take<int32_t>((size_t)kRUStack * T);
  int32_t* res = cv.take<int32_t>((size_t)kRURes * T);
  PhaseMarks pm(a.dbg);
  StageBar sb;
  sb.init(bar);
  bool first = true, rebase = false;
  const int part = lcta % parts;
  for (int u = lcta / parts; u < k.U; u += per_seg / parts) {
    sb.begin();
    if (first) {
      // <= 2 predecessors per block ([target, fallthrough]); none leaves the segment
      sb.copy(rh, rh_g + sb0, (size_t)B * 4);
      sb.copy(pptr, k.pred_ptr + sb0, (size_t)(B + 1) * 4);
      sb.copy(pred, k.pred + P0, (size_t)(P1 - P0) * 4);
      first = false;
      rebase = sb0 != 0;
    }
    sb.copy(cell, a.ldtab + (size_t)u * Bp + sb0, (size_t)B * 4);
    sb.copy(qs, qtab + (size_t)u * Bp + sb0, (size_t)B * 4);
    if (tid == 0) nq = 0;
    sb.commit_and_wait();
    if (rebase) {                            // segment-local block ids
      for (int y = tid; y < B; y += T) rh[y] -= sb0;
      for (int y = tid; y <= B; y += T) pptr[y] -= P0;
      for (int q = tid; q < P1 - P0; q += T) pred[q] -= sb0;
      rebase = false;
      __syncthreads();
    }
    pm.mark(0, 1);
    // near[y] = last def of u in [runhead(y), y]: an inclusive max-scan of
    // key(x) = runhead(x) << 32 | (def(x) + 1).  Run heads never decrease, so
    // the running max carries y's own run head and the latest def inside the
    // run.  Thread-contiguous chunks, shuffle scan of chunk maxima.
    {
      const int per = (B + T - 1) / T, lo = tid * per, hi = min(B, lo + per);
      long long run = -1;
#pragma unroll 8
      for (int y = lo; y < hi; y++) run = max(run, ((long long)rh[y] << 32) | (long long)(cell[y] + 1));
      long long inc = run;
      for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, inc, o);
        if ((tid & 31) >= o) inc = max(inc, v);
      }
      if ((tid & 31) == 31) wmax[tid >> 5] = inc;
      __syncthreads();
      long long carry = -1;
      for (int w = 0; w < (tid >> 5); w++) carry = max(carry, wmax[w]);
      const long long prev = __shfl_up_sync(0xffffffffu, inc, 1);
      if ((tid & 31) > 0) carry = max(carry, prev);
#pragma unroll 8
      for (int y = lo; y < hi; y++) {
        carry = max(carry, ((long long)rh[y] << 32) | (long long)(cell[y] + 1));
        const int d = (int)(carry & 0xffffffffLL) - 1;
        cell[y] = ((int)(carry >> 32) == rh[y] && d >= 0) ? d : -(rh[y] + 1);
      }
    }
    __syncthreads();
    pm.mark(0, 2);
    // ordered compaction of the unit's query blocks (every CTA sharing the
    // unit derives the same list, then takes its share of it)
    {
      const int per = (B + T - 1) / T, lo = min(B, tid * per), hi = min(B, lo + per);
      int cnt = 0;
#pragma unroll 8
      for (int y = lo; y < hi; y++) cnt += qs[y] >= 0;
      int tot;
      int pos = block_excl_scan(cnt, swarp, &tot);
      for (int y = lo; y < hi; y++) if (qs[y] >= 0) ql[pos++] = y;
      if (tid == 0) nq = tot;
    }
    __syncthreads();
    pm.mark(0, 3);
    const int n = nq;
    // rounds of T queries; one global reservation per CTA per round
    for (int base = part * T; base < n; base += T * parts) {
      const int t = base + tid;
      int e = -1, nres = 0;
      bool ovf = false;
      if (t < n) {
        const int b = ql[t];
        e = qs[b];
        ovf = (a.dbg & (LEO_DBG_REACH_T2 | LEO_DBG_REACH_T3)) != 0;
        int sp = 0, nvis = 0;
        const long long qc0 = clock64();
        if (!ovf) {
          for (int w = 0; w < W; w++) vis[w * T + tid] = 0u;
          // Entering block p backward either ends at its nearest def (a result)
          // or crosses the transparent stretch to run head h, whose expansion is
          // shared by every entry of the run: the bitmap marks result blocks
          // (cell >= 0) and expanded heads (cell < 0), which are disjoint.
          auto visit = [&](int p) {
            const int c = cell[p];
            const int key = c >= 0 ? p : -c - 1;
            uint32_t* word = &vis[(key >> 5) * T + tid];
            const uint32_t m = 1u << (key & 31);
            if (*word & m) return;
            *word |= m;
            nvis++;
            if (c >= 0) {
              if (nres == kRURes) ovf = true;
              else res[(nres++) * T + tid] = c;
            } else if (sp == kRUStack) {
              ovf = true;
            } else {
              stk[(sp++) * T + tid] = key;
            }
          };
          for (int q = pptr[b]; q < pptr[b + 1]; q++) visit(pred[q]);
          while (sp > 0 && !ovf) {
            const int h = stk[(--sp) * T + tid];
            for (int q = pptr[h]; q < pptr[h + 1]; q++) visit(pred[q]);
          }
        }
        if ((a.dbg & LEO_DBG_PHASES) && clock64() - qc0 > 14000) {   // per-query tail record (profiling)
          const int slot = atomicAdd(&g_reach_item_ctr, 1);
          if (slot < 8192) g_item_cycles[8192 + slot] = ((clock64() - qc0) << 24) | min(nvis, 0xFFFFFF);
        }
        if (ovf) {                                 // tier 2 re-runs the query
          const int s2 = atomicAdd(a.slow_count, 1);
          if (s2 < a.slow_cap) a.slow_list[s2] = e;
          else { a.q_off[e] = 0; a.q_len[e] = 0; atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); }
        }
      }
      const int cnt = (t < n && !ovf) ? nres : 0;
      int tot;
      const int ex = block_excl_scan(cnt, swarp, &tot);
      if (tid == 0) rbase = tot > 0 ? atomicAdd(a.qres_count, tot) : 0;
      __syncthreads();
      if (t < n && !ovf) {
        const int off = rbase + ex;
        if ((int64_t)off + nres > a.qres_cap) {
          atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
          a.q_off[e] = 0; a.q_len[e] = 0;
        } else {
          for (int x = 0; x < nres; x++) a.qres[off + x] = res[x * T + tid];
          a.q_off[e] = off;
          a.q_len[e] = nres;
        }
      }
      __syncthreads();
    }
    __syncthreads();
    pm.mark(0, 4);
  }
}

// Tier 1: lockstep per-lane state machine.  Every lane owns one query at a
// time and advances it by one search step per loop iteration; a lane whose
// query finished takes the next from a warp-private batch of the query list
// (one global atomic per kT1Fetch queries), so lanes never idle behind the
// warp's longest query.  Finished queries reserve their result slots from a
// warp-private chunk of the results pool (one global atomic per kT1Chunk
// results): on C5 (~1 M queries) a per-query atomic on the one pool counter
// was 40 % of the kernel's stall samples.  The visited set is a private
// open-addressing hash in shared memory (strided per thread), cleared through
// the list of slots it used.
constexpr int kT1Hash = 128, kT1Limit = 96, kT1Stack = 96, kT1Res = 32, kT1Threads = 128;
#ifndef LEO_T1_STEPS
#define LEO_T1_STEPS 2          // search steps (blocks' loads in flight) per lane per round
#endif
constexpr int kT1Fetch = 64, kT1Chunk = 512;

// KT: hash key type (uint16_t when every block id < 0xFFFF: half the shared
// memory per thread, twice the resident warps); HASH slots, LIMIT visits.
template <typename KT, int HASH, int LIMIT>
__global__ void __launch_bounds__(kT1Threads) k_reach_fast(KView k, ReachArgs a,
                                                           const int32_t* __restrict__ q_list,
                                                           const int32_t* q_count, int32_t* q_head) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char hsm_raw[];
  constexpr KT kEmpty = (KT)~(KT)0;
  const int nq = *q_count;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  KT* H = reinterpret_cast<KT*>(hsm_raw) + threadIdx.x;   // slot s at H[s * blockDim.x]
  const int stride = blockDim.x;
  for (int s2 = 0; s2 < HASH; s2++) H[s2 * stride] = kEmpty;
  int32_t stk[kT1Stack], res[kT1Res];
  int e = -1, u = 0, sp = 0, nres = 0, nused = 0;
  bool drained = false, ovf = false;
  // warp-uniform: the warp's current batch of the query list, and chunk of the pool
  int fb = 0, fleft = 0, cb = 0, cleft = 0;

  auto insert = [&](int key) -> int {              // 1 new, 0 seen, -1 overflow
    int x = (int)(((uint32_t)key * 2654435761u) >> (32 - __popc(HASH - 1)));
    for (int probe = 0; probe < HASH; probe++) {
      const KT v = H[x * stride];
      if (v == (KT)key) return 0;
      if (v == kEmpty) {
        if (nused == LIMIT) return -1;
        H[x * stride] = (KT)key;
        nused++;
        return 1;
      }
      x = (x + 1) & (HASH - 1);
    }
    return -1;
  };
  auto release = [&]() {
    // clear the whole table: HASH shared stores beat replaying a list of used
    // slots kept in local memory (its loads were 15 % of the stall samples)
    if (nused)
#pragma unroll 8
      for (int t = 0; t < HASH; t++) H[t * stride] = kEmpty;
    nused = 0; sp = 0; nres = 0; ovf = false; e = -1;
  };

  while (true) {
    // lanes without a query take one from the warp's batch (refilled with one atomic)
    const bool need = e < 0 && !drained;
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (m) {
      const int nm = __popc(m);
      // ranks [0, fleft) take the rest of the current batch, the others a new one
      int nb = 0;
      if (fleft < nm) {
        int g = 0;
        if (lane == 0) g = atomicAdd(q_head, kT1Fetch);
        nb = __shfl_sync(0xffffffffu, g, 0);
      }
      if (need) {
        const int rk = __popc(m & lt);
        const int t = rk < fleft ? fb + rk : nb + (rk - fleft);
        if (t >= nq) {
          drained = true;
        } else {
          e = q_list[t];
          u = a.q_unit[e];
          const int b = a.q_block[e];
          if (a.dbg & (LEO_DBG_REACH_T2 | LEO_DBG_REACH_T3)) ovf = true;
          for (int q = k.pred_ptr[b]; q < k.pred_ptr[b + 1] && !ovf; q++) {
            const int p = k.pred[q];
            const int v = insert(p);
            if (v < 0 || (v && sp == kT1Stack)) ovf = true;
            else if (v) stk[sp++] = p;
          }
        }
      }
      if (fleft < nm) { fb = nb + (nm - fleft); fleft = kT1Fetch - (nm - fleft); }
      else { fb += nm; fleft -= nm; }
    }
    if (!__any_sync(0xffffffffu, e >= 0)) {
      if (__all_sync(0xffffffffu, drained)) break;
      continue;
    }
    if (e >= 0 && !ovf && sp > 0) {
      // up to two search steps per round: both blocks' last-def and record
      // loads are issued before either is used (twice the loads in flight per
      // lane, half the round overhead per visit; the visited set makes the
      // result set independent of the order)
      auto step = [&](int y, int own, int4 r) {
        const int ld = own >= 0 ? own : (r.x < y ? run_lookup(a, y - 1, r.x, u) : -1);
        if (ld >= 0) {
          if (nres == kT1Res) ovf = true; else res[nres++] = ld;
        } else {
          for (int t = 0; t < r.y && !ovf; t++) {
            const int pp = r.y <= 2 ? (t == 0 ? r.z : r.w) : k.pred[r.z + t];
            const int v = insert(pp);
            if (v < 0 || (v && sp == kT1Stack)) ovf = true;
            else if (v) stk[sp++] = pp;
          }
        }
      };
      int ys[LEO_T1_STEPS], owns[LEO_T1_STEPS];
      int4 rs[LEO_T1_STEPS];
      int ns = 0;
#pragma unroll
      for (int x = 0; x < LEO_T1_STEPS; x++)
        if (sp > 0) { ys[x] = stk[--sp]; ns = x + 1; } else ys[x] = -1;
#pragma unroll
      for (int x = 0; x < LEO_T1_STEPS; x++) {
        owns[x] = ys[x] >= 0 ? a.ldtab[(size_t)u * a.Bp + ys[x]] : -1;
        rs[x] = ys[x] >= 0 ? a.rec[ys[x]] : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int x = 0; x < LEO_T1_STEPS; x++)
        if (x < ns && !ovf) step(ys[x], owns[x], rs[x]);
    }
    if (e >= 0 && ovf) {                           // hand the query to tier 2
      const int s2 = atomicAdd(a.slow_count, 1);
      if (s2 < a.slow_cap) a.slow_list[s2] = e;
      else { a.q_off[e] = 0; a.q_len[e] = 0; atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); }
      release();
    }
    // finished queries: result slots from the warp's chunk of the pool
    const bool done = e >= 0 && sp == 0;
    if (__ballot_sync(0xffffffffu, done)) {
      const int cnt = done ? nres : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tot > cleft) {
        const int want = max(tot, kT1Chunk);
        int g = 0;
        if (lane == 0) g = atomicAdd(a.qres_count, want);
        cb = __shfl_sync(0xffffffffu, g, 0);
        cleft = want;
      }
      if (done) {
        const int off = cb + incl - cnt;
        if ((int64_t)off + nres > a.qres_cap) {
          atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
          a.q_off[e] = 0; a.q_len[e] = 0;
        } else {
          for (int x = 0; x < nres; x++) a.qres[off + x] = res[x];
          a.q_off[e] = off;
          a.q_len[e] = nres;
        }
        release();
      }
      cb += tot;
      cleft -= tot;
    }
  }
}

// Tier 2: one warp per query, BFS level by level; visited set = open-addressing
// hash in shared memory, frontiers + results in shared memory.
constexpr int kWHash = 1024, kWFront = 512, kWRes = 128;
constexpr int kWarpSmemInts = kWHash + 2 * kWFront + kWRes + 8;

LEO_DEV bool hash_insert(int32_t* h, int key, int* count) {
  uint32_t x = ((uint32_t)key * 2654435761u) >> 22;   // 10 bits
  for (int probe = 0; probe < kWHash; probe++) {
    int32_t prev = atomicCAS(&h[x], -1, key);
    if (prev == -1) { atomicAdd(count, 1); return true; }
    if (prev == key) return false;
    x = (x + 1) & (kWHash - 1);
  }
  return false;
}

__global__ void k_reach_warp(KView k, ReachArgs a, const int32_t* __restrict__ list,
                             const int32_t* count, int64_t list_cap, int32_t* slow_list,
                             int32_t* slow_count) {
  pdl_wait();
  extern __shared__ int32_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  int32_t* base = smem + (size_t)wid * kWarpSmemInts;
  int32_t* hash = base;
  int32_t* fa = hash + kWHash;
  int32_t* fb = fa + kWFront;
  int32_t* res = fb + kWFront;
  int32_t* c = res + kWRes;   // 0 nres, 1 ncur, 2 nnext, 3 ovf, 4 nhash
  const int n = (int)min((int64_t)*count, list_cap);
  for (int t = blockIdx.x * wpc + wid; t < n; t += gridDim.x * wpc) {
    const int e = list[t];
    const int b = a.q_block[e], u = a.q_unit[e];
    for (int x = lane; x < kWHash; x += 32) hash[x] = -1;
    if (lane < 8) c[lane] = 0;
    __syncwarp();
    for (int q = k.pred_ptr[b] + lane; q < k.pred_ptr[b + 1]; q += 32) {
      int p = k.pred[q];
      if (hash_insert(hash, p, &c[4])) {
        int pos = atomicAdd(&c[1], 1);
        if (pos < kWFront) fa[pos] = p; else c[3] = 1;
      }
    }
    if ((a.dbg & LEO_DBG_REACH_T3) && lane == 0) c[3] = 1;
    __syncwarp();
    int32_t *cur = fa, *nxt = fb;
    while (true) {
      // every lane reads the loop control before any lane can modify it
      const int ncur = c[1];
      const bool stop = ncur == 0 || c[3];
      __syncwarp();
      if (stop) break;
      for (int x = lane; x < ncur; x += 32) {
        const int y = cur[x];
        const int4 r = a.rec[y];
        const int ld = run_lookup(a, y, r.x, u);
        if (ld >= 0) {
          int rr = atomicAdd(&c[0], 1);
          if (rr < kWRes) res[rr] = ld; else c[3] = 1;
          continue;
        }
        for (int t2 = 0; t2 < r.y; t2++) {
          const int pp = r.y <= 2 ? (t2 == 0 ? r.z : r.w) : k.pred[r.z + t2];
          if (hash_insert(hash, pp, &c[4])) {
            int pos = atomicAdd(&c[2], 1);
            if (pos < kWFront) nxt[pos] = pp; else c[3] = 1;
          }
        }
      }
      __syncwarp();
      if (c[4] > kWHash / 2) c[3] = 1;          // keep probing short
      if (lane == 0) { c[1] = c[2]; c[2] = 0; }
      __syncwarp();
      int32_t* tmp = cur; cur = nxt; nxt = tmp;
    }
    __syncwarp();
    if (c[3]) {
      if (lane == 0) {
        int s = atomicAdd(slow_count, 1);
        if (s < a.slow_cap) slow_list[s] = e;
        else { a.q_off[e] = 0; a.q_len[e] = 0; atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); }
      }
    } else {
      const int nres = c[0];
      int off = 0;
      if (lane == 0) off = atomicAdd(a.qres_count, nres);
      off = __shfl_sync(0xffffffffu, off, 0);
      if ((int64_t)off + nres > a.qres_cap) {
        if (lane == 0) { atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); a.q_off[e] = 0; a.q_len[e] = 0; }
      } else {
        for (int x = lane; x < nres; x += 32) a.qres[off + x] = res[x];
        if (lane == 0) { a.q_off[e] = off; a.q_len[e] = nres; }
      }
    }
    __syncwarp();
  }
}

// Tier 3: one worker thread per slot of global scratch (stamp / stack / results
// of B entries each); stamps are query slot + 1, so no clearing between queries.
__global__ void k_reach_slow(KView k, ReachArgs a, const int32_t* list, const int32_t* count,
                             int32_t* scratch, int nworkers) {
  pdl_wait();
  const int ns = (int)min((int64_t)*count, a.slow_cap);
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nworkers) return;
  const int B = k.B;
  int32_t* stamp = scratch + (size_t)w * 3 * (B + 1);
  int32_t* stk = stamp + (B + 1);
  int32_t* res = stk + (B + 1);
  // a worker with items clears its own stamps (no memset node ahead of the
  // build for a tier that usually has nothing to do)
  if (w < ns)
    for (int x = 0; x <= B; x++) stamp[x] = 0;
  for (int t = w; t < ns; t += nworkers) {
    int e = list[t];
    int nres = 0;
    StampSet vis{stamp, e + 1};
    reach_search(k, a, a.q_block[e], a.q_unit[e], vis, stk, B + 1, res, B + 1, &nres);
    reach_commit(a, e, res, nres);
  }
}

struct LinkArgs {
  const int32_t* use_ptr;
  const int32_t* ev_res;
  const int32_t* q_off;
  const int32_t* q_len;
  const int32_t* qres;
  int32_t* cand_cnt;         // [N]
  const int32_t* cand_off;   // [N+1]
  uint64_t* cand;            // keys
  int64_t cand_cap;
  LeoDiags diags;
  uint32_t* status;
  Range own;
};

LEO_DEV uint64_t link_key(int producer, int kind, uint32_t r) {
  uint64_t ref = ((uint64_t)kRcRank[op_class(r)] << 24) | ((uint64_t)op_index(r) << 8) | (uint64_t)op_span(r);
  return ((uint64_t)producer << 28) | ((uint64_t)(kind == LEO_EK_RAW ? 1 : 0) << 27) | ref;
}

// mode 0: count candidates + unresolved diagnostics; mode 1: write keys
template <int MODE>
__global__ void k_link(KView k, LinkArgs a) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k.N; i += gridDim.x * blockDim.x) {
    int e = a.use_ptr[i];
    int cnt = 0;
    int64_t w = MODE ? a.cand_off[i] : 0;
    if (MODE && (int64_t)a.cand_off[i + 1] > a.cand_cap) { atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW); continue; }
    for (int q = k.opnd_ptr[i]; q < k.opnd_ptr[i + 1]; q++) {
      uint32_t r = k.opnd[q];
      int role = op_role(r);
      if (role == LEO_ROLE_DST) continue;
      int kind = role == LEO_ROLE_GUARD ? LEO_EK_GUARD : LEO_EK_RAW;
      bool found = false;
      for (int s = 0; s < op_span(r); s++, e++) {
        int res = a.ev_res[e];
        if (res >= 0) {
          found = true;
          if (MODE) a.cand[w++] = link_key(res, kind, r); else cnt++;
        } else {
          int qs = -(res + 1);
          int L = a.q_len[qs], off = a.q_off[qs];
          if (L > 0) found = true;
          if (MODE) { for (int x = 0; x < L; x++) a.cand[w++] = link_key(a.qres[off + x], kind, r); }
          else cnt += L;
        }
      }
      if (!MODE && !found && a.own.has(i))   // depgraph.py:208-210 — no unit of the ref has a def
        diag_push(a.diags, a.status, LEO_DIAG_UNRESOLVED, i, (int)r, 0, 0, q - k.opnd_ptr[i]);
    }
    if (!MODE) a.cand_cnt[i] = cnt;
  }
}

__constant__ static const int kRankToClass[8] = {3, 2, 1, 5, 6, 4, 0, 7};

__global__ void k_link_emit(KView k, const int32_t* __restrict__ cand_off, const uint64_t* __restrict__ cand,
                            const int32_t* __restrict__ uniq, const int32_t* __restrict__ eoff,
                            LeoEdges out, uint32_t* status) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k.N; i += gridDim.x * blockDim.x) {
    int n = uniq[i], o = eoff[i];
    if (o + n > out.capacity) { if (n) atomicOr(status, (uint32_t)LEO_ST_EDGE_OVERFLOW); continue; }
    const uint64_t* c = cand + cand_off[i];
    for (int x = 0; x < n; x++) {
      uint64_t key = c[x];
      int prod = (int)(key >> 28);
      int kind = ((key >> 27) & 1) ? LEO_EK_RAW : LEO_EK_GUARD;
      int cls = kRankToClass[(key >> 24) & 7];
      uint32_t ref27 = (uint32_t)((key >> 8) & 0xFFFF) | ((uint32_t)(key & 0xFF) << 16) | ((uint32_t)cls << 24);
      out.prod[o + x] = prod;
      out.cons[o + x] = i;
      out.meta[o + x] = LEO_META(kind, dep_class_of(k.opclass[prod], kind), ref27);
    }
  }
}

}  // namespace leo
