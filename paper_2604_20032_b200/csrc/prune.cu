// prune.cu — the four pruning stages (analysis.py:130-314) as one per-edge map
// plus a stable stream compaction.
//
// run_pruning applies stages 1 -> 2 -> 3 -> 4 to the whole edge list, but every
// stage decides each edge from that edge alone (plus instruction and profile
// data), so  keep(e) = s1(e) & s2(e) & s3(e) & s4(e)  with stage-3 run only
// on edges that survive 1 and 2 (its diagnostics are emitted for exactly those
// edges, in edge order after the host sorts them by edge index).
//
//   k_prune_edges   thread/edge: stage-1 opcode rule, stage-2 barrier rule,
//                   stage-3 exact LIFO path DFS (_enumerate_paths :210-253,
//                   budget 65,536 pops, max_paths, max_depth, layout back edges
//                   at most once per path), stage-4 exec-count rule; surviving
//                   paths reserved in the path pool, sorted (len, accum);
//                   _edge_distance (:371-376) precomputed for blame.
//   k_prune_slow    same DFS on global scratch for edges whose stack / back-
//                   edge arena / path buffer overflowed the register budget.
//   scan + k_compact  order-preserving compaction.
#include "prims.cuh"
#include "stage.cuh"

namespace leo {

struct PView {
  int64_t period;
  const int32_t* __restrict__ lat;
  const int32_t* __restrict__ cls_cnt;
  const int64_t* __restrict__ exec_cnt;
  const int32_t* __restrict__ total;
  const double* __restrict__ eff;
  const uint8_t* __restrict__ sampled;
};
inline PView make_pview(const LeoProfile* p) {
  PView v;
  v.period = p->period; v.lat = p->lat; v.cls_cnt = p->cls_cnt; v.exec_cnt = p->exec_cnt;
  v.total = p->total; v.eff = p->eff; v.sampled = p->sampled;
  return v;
}

LEO_DEV bool only_class(const PView& p, int j, int cls) {   // _only_class :134-140
  if (p.lat[j] == 0) return false;
  const int4* row = reinterpret_cast<const int4*>(p.cls_cnt + (size_t)j * 8);
  int4 a = row[0], b = row[1];
  int v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int c = 0; c < 8; c++) if (c != cls && v[c] > 0) return false;
  return true;
}

LEO_DEV double issue_weight(const KView& k, int i) {   // _issue_weights :188-199
  if (k.dialect == LEO_NVIDIA && k.sync_kind[i] == LEO_SYNC_BARRIER && k.sync_b[i] != LEO_NONE_U32)
    return (double)k.sync_b[i];
  return 1.0;
}

struct DfsEnt { int32_t node, len, back, pad; double acc; };
struct BackNode { int32_t nb, cb, parent; };

enum { DFS_OK = 0, DFS_TRUNC = 1, DFS_OVERFLOW = 2 };

// Exact emulation of _enumerate_paths.  Returns DFS_OK / DFS_TRUNC, or
// DFS_OVERFLOW when a caller buffer was too small (caller re-runs elsewhere).
// `wpre` (nvidia, may be null): per-instruction prefix sums of the issue
// weights within each block (wpre[i] = w[first(b)] + ... + w[i]), so straight
// runs resolve in closed form with weights too (integer-valued doubles: the
// differences are exact, as the step-by-step sums are).
LEO_DEV int enumerate_paths(const KView& k, int producer, int consumer, double thr, int max_paths,
                            int max_depth, DfsEnt* stk, int scap, BackNode* arena, int acap,
                            int32_t* vlen, double* vacc, int vcap, int* nvalid_out,
                            const double* __restrict__ wpre = nullptr) {
  int budget = 65536, truncated = 0, sp = 0, na = 0, nv = 0;
  *nvalid_out = 0;
  const double w0 = issue_weight(k, producer);
  if (w0 > thr) return DFS_OK;
  stk[sp++] = DfsEnt{producer, 1, -1, 0, w0};
  const bool unit_w = k.dialect != LEO_NVIDIA;     // every issue weight is 1.0
  while (sp > 0) {
    DfsEnt e = stk[--sp];
    if (budget <= 0 || nv >= max_paths) { truncated = 1; break; }
    budget--;
    const int nb = k.block_of[e.node];
    if ((unit_w || wpre) && e.node < k.blk_last[nb]) {
      // Straight run e.node+1 .. blk_last: each step pushes its successor and
      // the LIFO pops it right back, so the run is a sequence of consecutive
      // pops that can be resolved in closed form.  Step i reaches node
      // x+i with len+i, acc+i; the first of {consumer reached, acc > thr,
      // len >= max_depth} ends the run (checked in that order), each step
      // before it costs one pop of budget.
      const int x = e.node, L = k.blk_last[nb];
      const int i_end = L - x;
      const int i_c = (consumer > x && consumer <= L) ? consumer - x : 0x7fffffff;
      int i_thr;
      if (unit_w) {
        const double f = thr - e.acc;
        i_thr = f < 0.0 ? 1 : (f > 1e9 ? 0x3fffffff : (int)floor(f) + 1);
        while (i_thr > 1 && __dadd_rn(e.acc, (double)(i_thr - 1)) > thr) i_thr--;
        while (i_thr < 0x3fffffff && !(__dadd_rn(e.acc, (double)i_thr) > thr)) i_thr++;
      } else {
        // first step i in [1, i_end] whose accumulation exceeds thr (weights
        // are >= 0: monotone), else past the run.  One load decides the common
        // cases: the run's end (or the step before the consumer) within thr
        // means no step up to there exceeds it; only otherwise binary search.
        const double w0 = wpre[x];
        const int probe = i_c <= i_end ? i_c - 1 : i_end;
        int lo = 1, hi = i_end + 1;
        if (probe >= 1 && !(__dadd_rn(e.acc, __dsub_rn(wpre[x + probe], w0)) > thr)) {
          // consumer in the run and reached within thr: i_thr >= i_c, and any
          // such value stops the run at the same step (i_stop = min(i_c, i_dep))
          lo = i_c <= i_end ? i_c : probe + 1;
          if (i_c <= i_end) hi = lo;
        } else if (probe >= 1) {
          hi = probe;
        }
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__dadd_rn(e.acc, __dsub_rn(wpre[x + mid], w0)) > thr) hi = mid; else lo = mid + 1;
        }
        i_thr = lo <= i_end ? lo : 0x3fffffff;
      }
      const double wrun = unit_w ? 0.0 : wpre[x];
      const int i_dep = max(1, max_depth - e.len);
      const int i_stop = min(i_c, min(i_thr, i_dep));
      if (i_stop <= i_end) {
        const int need = i_stop - 1;
        if (budget < need) { budget = 0; truncated = 1; break; }
        budget -= need;
        if (i_stop == i_c) {
          if (nv == vcap) return DFS_OVERFLOW;
          vlen[nv] = e.len + i_c - 1;
          vacc[nv] = __dadd_rn(e.acc, unit_w ? (double)(i_c - 1) : __dsub_rn(wpre[x + i_c - 1], wrun));
          nv++;
          if (nv >= max_paths) truncated = 1;
        } else if (i_stop != i_thr) {
          truncated = 1;                              // max_depth
        }
        continue;
      }
      if (budget < i_end) { budget = 0; truncated = 1; break; }
      budget -= i_end;
      e.node = L; e.len += i_end;
      e.acc = __dadd_rn(e.acc, unit_w ? (double)i_end : __dsub_rn(wpre[L], wrun));
    }
    int succ_n, s0 = -1, s1 = -1;
    if (e.node < k.blk_last[nb]) { succ_n = 1; s0 = e.node + 1; }
    else {
      const int q0 = k.succ_ptr[nb];
      succ_n = k.succ_ptr[nb + 1] - q0;
      if (succ_n > 0) s0 = k.blk_first[k.succ[q0]];
      if (succ_n > 1) s1 = k.blk_first[k.succ[q0 + 1]];
      if (succ_n > 2) return DFS_OVERFLOW;
    }
    for (int t = 0; t < succ_n; t++) {
      const int nxt = t == 0 ? s0 : s1;
      if (nxt == consumer) {
        if (nv == vcap) return DFS_OVERFLOW;
        vlen[nv] = e.len; vacc[nv] = e.acc; nv++;
        if (nv >= max_paths) truncated = 1;
        continue;
      }
      const int cb = k.block_of[nxt];
      int nback = e.back;
      if (nb != cb && k.blk_first[cb] <= k.blk_first[nb]) {
        bool hit = false;
        for (int x = e.back; x >= 0; x = arena[x].parent)
          if (arena[x].nb == nb && arena[x].cb == cb) { hit = true; break; }
        if (hit) continue;
        if (na == acap) return DFS_OVERFLOW;
        arena[na] = BackNode{nb, cb, e.back};
        nback = na++;
      }
      const int nlen = e.len + 1;
      const double nacc = __dadd_rn(e.acc, issue_weight(k, nxt));
      if (nacc > thr) continue;
      if (nlen >= max_depth) { truncated = 1; continue; }
      if (sp == scap) return DFS_OVERFLOW;
      stk[sp++] = DfsEnt{nxt, nlen, nback, 0, nacc};
    }
  }
  // valid.sort(key=(length, accum))
  for (int i = 1; i < nv; i++) {
    int l = vlen[i]; double a = vacc[i];
    int j = i - 1;
    while (j >= 0 && (vlen[j] > l || (vlen[j] == l && vacc[j] > a))) { vlen[j + 1] = vlen[j]; vacc[j + 1] = vacc[j]; j--; }
    vlen[j + 1] = l; vacc[j + 1] = a;
  }
  *nvalid_out = nv;
  return truncated ? DFS_TRUNC : DFS_OK;
}

// wpre[i] = issue weights of first(block_of(i)) .. i (thread per block)
__global__ void k_weight_prefix(KView k, double* __restrict__ wpre) {
  pdl_wait();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < k.B; b += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int i = k.blk_first[b]; i <= k.blk_last[b]; i++) { s = __dadd_rn(s, issue_weight(k, i)); wpre[i] = s; }
  }
}

struct PruneArgs {
  int32_t dbg;
  LeoConfig cfg;
  const int32_t* prod;
  const int32_t* cons;
  const uint32_t* meta;
  const int32_t* n_in;       // device count of input edges
  int32_t cap_in;
  int32_t* keep;             // [cap_in] 0/1
  int32_t* npaths;           // [cap_in]
  int32_t* pfirst;           // [cap_in]
  double* dist;              // [cap_in]
  LeoPaths paths;            // pool (len / accum / count)
  const double* wpre;        // nvidia: per-block prefix sums of the issue weights (null: unit weights)
  LeoPaths in_paths;         // valid_paths of the input edges (first == null: none); their
                             // records were copied to the front of `paths` (k_copy_pool)
  int32_t* slow_list;
  int32_t* slow_count;
  int64_t slow_cap;
  LeoDiags diags;
  uint32_t* status;
};

// stage 1/2/4 predicates + stage-3 DFS for edge e.  Returns false when the
// DFS needs the slow path.
// `deferred` (optional): do not reserve path-pool space here; report the
// valid-path count and leave vlen/vacc + pfirst[e] to the caller, which
// reserves pool space for a whole CTA round with one atomic.
LEO_DEV bool prune_one(const KView& k, const PView& p, const PruneArgs& a, int e, DfsEnt* stk, int scap,
                       BackNode* arena, int acap, int32_t* vlen, double* vacc, int vcap,
                       int* deferred = nullptr) {
  const uint32_t m = a.meta[e];
  const int kind = (m >> 27) & 7;
  const int pr = a.prod[e], cn = a.cons[e];
  int keep = 1, nv = 0;
  if (a.cfg.consumer_hi > 0 && (cn < a.cfg.consumer_lo || cn >= a.cfg.consumer_hi)) {
    a.keep[e] = 0; a.npaths[e] = 0; a.pfirst[e] = -1; a.dist[e] = 1.0;   // not owned (sharding)
    return true;
  }
  const uint32_t mask = a.cfg.stage_mask;
  double dist;
  {
    int d = cn - pr; if (d < 0) d = -d; if (d < 1) d = 1;
    dist = (double)d;
  }
  // the edge keeps its input valid_paths unless stage 3 replaces them (a raw /
  // guard edge with valid paths): sync edges, stages 1/2/4 and a truncated
  // enumeration without valid paths keep `e` as it was (analysis.py:143-299)
  bool carry = true;
  if (kind < LEO_EK_MEM_WAITCNT) {                       // sync edges are exempt
    const uint32_t poc = k.opclass[pr];
    if ((mask & 1) && ((only_class(p, cn, LEO_CS_MEMORY_DEP) && (kCompute & BIT(poc))) ||
                       (only_class(p, cn, LEO_CS_EXECUTION_DEP) && poc == LEO_OC_GLOBAL_LOAD)))
      keep = 0;                                          // prune_opcode :143-162
    if (keep && (mask & 2) && k.dialect == LEO_NVIDIA) {   // prune_barrier :165-185
      uint32_t sets = 0, waits = 0;
      if (k.sync_kind[pr] == LEO_SYNC_BARRIER) sets = (k.sync_a[pr] | (k.sync_a[pr] >> 8)) & 0xFF;
      if (sets) {
        if (k.sync_kind[cn] == LEO_SYNC_BARRIER) waits = (k.sync_a[cn] >> 16) & 0xFF;
        if (!(sets & waits)) keep = 0;
      }
    }
    if (keep && (mask & 4)) {                            // prune_latency :256-286
      int r = enumerate_paths(k, pr, cn, a.cfg.threshold[poc], a.cfg.max_paths, a.cfg.max_depth,
                              stk, scap, arena, acap, vlen, vacc, vcap, &nv, a.wpre);
      if (r == DFS_OVERFLOW) return false;
      if (nv > 0) carry = false;
      if (nv > 0 && deferred) {
        *deferred = nv;
        int64_t s = 0;
        for (int x = 0; x < nv; x++) s += vlen[x];
        dist = __ddiv_rn((double)s, (double)nv);
        if (r == DFS_TRUNC) diag_push(a.diags, a.status, LEO_DIAG_PATH_CAPPED, pr, cn, 1, 0, e);
      } else if (nv > 0) {
        int off = atomicAdd(a.paths.count, nv);
        if (off + nv > a.paths.capacity) {
          atomicOr(a.status, (uint32_t)LEO_ST_PATH_OVERFLOW);
          off = -1;
          nv = 0;                                        // keep readers in bounds
        } else {
          for (int x = 0; x < nv; x++) { a.paths.len[off + x] = vlen[x]; a.paths.accum[off + x] = vacc[x]; }
        }
        int64_t s = 0;
        for (int x = 0; x < nv; x++) s += vlen[x];
        dist = nv > 0 ? __ddiv_rn((double)s, (double)nv) : dist;
        a.pfirst[e] = off;
        if (r == DFS_TRUNC) diag_push(a.diags, a.status, LEO_DIAG_PATH_CAPPED, pr, cn, 1, 0, e);
      } else if (r == DFS_TRUNC) {
        diag_push(a.diags, a.status, LEO_DIAG_PATH_CAPPED, pr, cn, 0, 0, e);
      } else {
        keep = 0;
      }
    }
    if (keep && (mask & 8) && a.cfg.prune_exec && p.exec_cnt[pr] == 0) keep = 0;   // :289-299
  }
  a.keep[e] = keep;
  if (carry && a.in_paths.first && a.in_paths.npaths[e] > 0) {
    const int np = a.in_paths.npaths[e], f = a.in_paths.first[e];
    if ((int64_t)f + np > a.paths.capacity) {             // carried pool did not fit (flagged)
      a.npaths[e] = 0; a.pfirst[e] = -1; a.dist[e] = dist;
      return true;
    }
    int64_t s = 0;
    for (int q = 0; q < np; q++) s += a.paths.len[f + q];   // (copied to the same slots)
    a.npaths[e] = np;
    a.pfirst[e] = f;
    a.dist[e] = __ddiv_rn((double)s, (double)np);
    return true;
  }
  a.npaths[e] = nv;
  if (nv == 0) a.pfirst[e] = -1;
  a.dist[e] = dist;
  return true;
}

#ifndef LEO_DFS_PATHS
#define LEO_DFS_PATHS 64
#endif
constexpr int kDfsStack = 20, kDfsArena = 24, kDfsPaths = LEO_DFS_PATHS;

__global__ void __launch_bounds__(128) k_prune_edges(KView k, PView p, PruneArgs a) {
  pdl_wait();
  const int n = *a.n_in;
  DfsEnt stk[kDfsStack];
  BackNode arena[kDfsArena];
  int32_t vlen[kDfsPaths];
  double vacc[kDfsPaths];
  // an edge whose valid paths outgrow the local buffer overflows to the slow
  // tier on its own (enumerate_paths returns DFS_OVERFLOW at vcap)
  const bool big_paths = (a.dbg & LEO_DBG_PRUNE_SLOW) || (LEO_DFS_PATHS >= 64 && a.cfg.max_paths > kDfsPaths);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    bool ok = !big_paths && prune_one(k, p, a, e, stk, kDfsStack, arena, kDfsArena, vlen, vacc, kDfsPaths);
    if (!ok) {
      int s = atomicAdd(a.slow_count, 1);
      if (s < a.slow_cap) {
        a.slow_list[s] = e;
      } else {
        // no room: leave safe outputs (dropped edge, no paths); the host sees
        // the status bit and re-runs with a larger slow list
        a.keep[e] = 0; a.npaths[e] = 0; a.pfirst[e] = -1; a.dist[e] = 1.0;
        atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      }
    }
  }
}

// Shared-memory tier: the per-thread DFS state (stack, back-edge arena, valid
// paths) lives in shared memory instead of local memory (which thrashes L1 at
// ~1.5 KB per thread), and when the instruction -> block map and the block /
// successor tables fit, every CTA stages them with TMA bulk copies so each
// DFS pop is a shared-memory access.  Persistent CTAs, edges grid-strided.
// Overflowing edges take the global-scratch worker (k_prune_slow).
constexpr int kPSStack = 16, kPSArena = 16, kPSPaths = 8;
constexpr int kPSThreadBytes = ((kPSStack * (int)sizeof(DfsEnt) + kPSArena * (int)sizeof(BackNode) +
                                 kPSPaths * 12 + 7) & ~7) + 8;   // 8-byte pad: 2-way bank spread

__host__ __device__ inline size_t prune_image_bytes(int N, int B) {
  return carve_bytes(N, 4) + carve_bytes(B, 4) * 2 + carve_bytes(B + 1, 4) + carve_bytes(2 * (size_t)B + 4, 4);
}
__host__ __device__ inline size_t prune_smem_bytes(int N, int B, int threads, bool stage) {
  return 16 + (stage ? prune_image_bytes(N, B) : 0) + (size_t)kPSThreadBytes * threads;
}

template <bool STAGE>
__global__ void k_prune_edges_smem(KView k, PView p, PruneArgs a) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  SmemCarve cv{sm_raw};
  uint64_t* bar = cv.take<uint64_t>(2);
  PhaseMarks pm(a.dbg);
  KView ks = k;
  if (STAGE) {
    const int N = k.N, B = k.B;
    int32_t* bo = cv.take<int32_t>(N);
    int32_t* bf = cv.take<int32_t>(B);
    int32_t* bl = cv.take<int32_t>(B);
    int32_t* sp = cv.take<int32_t>(B + 1);
    int32_t* su = cv.take<int32_t>(2 * (size_t)B + 4);
    StageBar sb;
    sb.init(bar);
    sb.begin();
    sb.copy(bo, k.block_of, (size_t)N * 4);
    sb.copy(bf, k.blk_first, (size_t)B * 4);
    sb.copy(bl, k.blk_last, (size_t)B * 4);
    sb.copy(sp, k.succ_ptr, (size_t)(B + 1) * 4);
    sb.copy(su, k.succ, (size_t)min(k.succ_ptr[B], 2 * B + 4) * 4);
    sb.commit_and_wait();
    ks.block_of = bo; ks.blk_first = bf; ks.blk_last = bl; ks.succ_ptr = sp; ks.succ = su;
  }
  pm.mark(2, 1);
  unsigned char* mine = cv.p + (size_t)threadIdx.x * kPSThreadBytes;
  DfsEnt* stk = (DfsEnt*)mine;
  BackNode* arena = (BackNode*)(mine + kPSStack * sizeof(DfsEnt));
  double* vacc = (double*)(((uintptr_t)(arena + kPSArena) + 7) & ~(uintptr_t)7);
  int32_t* vlen = (int32_t*)(vacc + kPSPaths);
  __shared__ int swarp[33];
  __shared__ int rbase;
  const int n = *a.n_in;
  const bool big_paths = a.cfg.max_paths > 64 || (a.dbg & LEO_DBG_PRUNE_SLOW);
  // rounds of one edge per thread; valid paths reserved once per CTA round
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const int e = base + threadIdx.x;
    int nvd = 0;
    if (e < n) {
      bool ok = !big_paths && prune_one(ks, p, a, e, stk, kPSStack, arena, kPSArena, vlen, vacc, kPSPaths, &nvd);
      if (!ok) {
        nvd = 0;
        int s2 = atomicAdd(a.slow_count, 1);
        if (s2 < a.slow_cap) {
          a.slow_list[s2] = e;
        } else {
          a.keep[e] = 0; a.npaths[e] = 0; a.pfirst[e] = -1; a.dist[e] = 1.0;
          atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
        }
      }
    }
    int tot;
    const int ex = block_excl_scan(nvd, swarp, &tot);
    if (threadIdx.x == 0) rbase = tot > 0 ? atomicAdd(a.paths.count, tot) : 0;
    __syncthreads();
    if (nvd > 0) {
      const int off = rbase + ex;
      if (off + nvd > a.paths.capacity) {
        atomicOr(a.status, (uint32_t)LEO_ST_PATH_OVERFLOW);
        a.npaths[e] = 0; a.pfirst[e] = -1;
      } else {
        for (int x = 0; x < nvd; x++) { a.paths.len[off + x] = vlen[x]; a.paths.accum[off + x] = vacc[x]; }
        a.pfirst[e] = off;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  pm.mark(2, 2);
}

__host__ __device__ inline size_t prune_slow_bytes(int max_depth, int max_paths) {
  size_t scap = (size_t)max_depth + 8, acap = 2 * 65536 + 8, vcap = (size_t)max_paths + 2;
  return ((scap * sizeof(DfsEnt) + acap * sizeof(BackNode) + vcap * 12) + 255) & ~(size_t)255;
}

__global__ void k_prune_slow(KView k, PView p, PruneArgs a, char* scratch, int nworkers) {
  pdl_wait();
  const int ns = (int)min((int64_t)*a.slow_count, a.slow_cap);
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nworkers) return;
  const int scap = a.cfg.max_depth + 8, acap = 2 * 65536 + 8, vcap = a.cfg.max_paths + 2;
  char* base = scratch + (size_t)w * prune_slow_bytes(a.cfg.max_depth, a.cfg.max_paths);
  DfsEnt* stk = (DfsEnt*)base;
  BackNode* arena = (BackNode*)(stk + scap);
  double* vacc = (double*)(((uintptr_t)(arena + acap) + 7) & ~(uintptr_t)7);
  int32_t* vlen = (int32_t*)(vacc + vcap);
  for (int t = w; t < ns; t += nworkers) {
    int e = a.slow_list[t];
    if (!prune_one(k, p, a, e, stk, scap, arena, acap, vlen, vacc, vcap))
      atomicOr(a.status, (uint32_t)LEO_ST_BAD_INPUT);   // > 2 successors: malformed CFG
  }
}

// `zero` (optional): four int arrays of zn elements the next stage expects
// zeroed (the pruned graph's incoming-CSR bounds and counters), cleared here
// instead of by four memset nodes
struct ZeroSet { int32_t* p[4]; int n; };

__global__ void k_compact(PruneArgs a, const int32_t* __restrict__ pos, const int32_t* n_reg_in,
                          LeoEdges out, uint32_t* status, ZeroSet zero) {
  pdl_wait();
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < zero.n; x += gridDim.x * blockDim.x) {
    zero.p[0][x] = 0; zero.p[1][x] = 0; zero.p[2][x] = 0; zero.p[3][x] = 0;
  }
  const int n = *a.n_in;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    if (!a.keep[e]) continue;
    const int o = pos[e];
    if (o >= out.capacity) { atomicOr(status, (uint32_t)LEO_ST_EDGE_OVERFLOW); continue; }
    out.prod[o] = a.prod[e];
    out.cons[o] = a.cons[e];
    out.meta[o] = a.meta[e];
    a.paths.first[o] = a.pfirst[e];
    a.paths.npaths[o] = a.npaths[e];
    a.paths.dist[o] = a.dist[e];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *out.count = pos[n];
    if (out.n_regular) *out.n_regular = n_reg_in ? pos[*n_reg_in] : 0;
  }
}

}  // namespace leo
