// sync.cu — vendor synchronization edges (depgraph.py:296-501).
//
//   amd    s_waitcnt:  exact chain enumeration (_scan_backward :312-348 with the
//          _WaitcntState visitor :365-399): one thread per (wait, counter)
//          walks every simple backward block path (b0 pre-visited, forks inherit
//          the remaining 4096-instruction budget); member operations appended at
//          pending index >= level become edges; best_m drives the diagnostic.
//          Instructions are scanned through a packed 32-bit word per instruction
//          (waitcnt flag, counter values, membership bits), eight per batch of
//          independent loads.
//   nvidia barrier / intel SWSB setter search (_trace_setter :431-443): closed
//          form — nearest setter before the wait in its own block, otherwise a
//          node-weighted Dijkstra over setter-free predecessor blocks (b0
//          excluded): a setter block p yields its last setter iff the cheapest
//          path reaches it within the budget.  Shortest paths are simple, so
//          this equals the union over the reference's per-chain simple paths.
//          Per-block "last setter of id" summaries make every Dijkstra node O(1).
//
// Raw (producer, wait) keys are appended to a buffer; they are then grouped by
// producer, sorted + deduplicated per producer and appended after the
// raw/guard edges in (producer, consumer) order (_materialize_sync :485-492).
#include "prims.cuh"
#include "stage.cuh"

namespace leo {

constexpr int kSyncBudget = 4096;   // SYNC_SCAN_BUDGET depgraph.py:43

// packed amd scan word
constexpr uint32_t kWcNone = 0x3FF;
constexpr uint32_t kWcIsWait = 1u << 20, kWcVm = 1u << 21, kWcLgkm = 1u << 22, kWcBig = 1u << 23;

struct SyncArgs {
  int32_t dbg;
  uint64_t* keys;            // raw (producer << 32 | consumer)
  int64_t key_cap;
  int32_t* key_count;
  int32_t* slow_list;        // (instr << 6 | sub-item) items re-run on global scratch
  int32_t* slow_count;
  int64_t slow_cap;
  LeoDiags diags;
  uint32_t* status;
  const uint32_t* wcword;    // [N] amd packed scan words
  const uint8_t* setword;    // [N] nvidia set mask (w|r) / intel set token (255 none)
  const int32_t* lastset;    // [B * ids] last setter of id in block, -1 none
  int32_t n_ids;             // 8 (nvidia, ids 1..6) or 32 (intel)
  const int32_t* wait_list;  // compact waiting instructions
  const int32_t* wait_count;
  int32_t* wc_list;          // waitcnt items for the warp tier
  int32_t* wc_count;
  int32_t defer_search;      // nvidia/intel: block searches all go to k_sync_setter_cta
  // slow tier scratch geometry: a concatenated batch (LeoKernel.seg_block) is
  // searched member by member, so a worker's block-indexed scratch spans the
  // largest member (bcap blocks), addressed relative to the item's member
  const int32_t* seg_block;  // [n_seg + 1] or null
  int32_t n_seg;
  int32_t bcap;
};

// first block of the batch member holding block b (0 without segments)
LEO_DEV int seg_base_of(const SyncArgs& a, int b) {
  if (!a.seg_block || a.n_seg <= 1) return 0;
  int lo = 0, hi = a.n_seg - 1;                 // largest s with seg_block[s] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.seg_block[mid] <= b) lo = mid; else hi = mid - 1;
  }
  return a.seg_block[lo];
}

__global__ void k_sync_pack(KView k, uint32_t* __restrict__ wcword, uint8_t* __restrict__ setword,
                            uint32_t* __restrict__ bev) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k.N; i += gridDim.x * blockDim.x) {
    const uint8_t sk = k.sync_kind[i];
    const uint32_t a = k.sync_a[i], b = k.sync_b[i];
    if (k.dialect == LEO_AMD) {
      uint32_t w = 0;
      if (sk == LEO_SYNC_WAITCNT) {
        w |= kWcIsWait;
        uint32_t vm = a == LEO_NONE_U32 ? kWcNone : a, lg = b == LEO_NONE_U32 ? kWcNone : b;
        if ((a != LEO_NONE_U32 && a >= kWcNone) || (b != LEO_NONE_U32 && b >= kWcNone)) w |= kWcBig;
        w |= (min(vm, kWcNone)) | (min(lg, kWcNone) << 10);
      } else {
        w |= kWcNone | (kWcNone << 10);
        if (kVmcnt & BIT(k.opclass[i])) w |= kWcVm;
        if (kLgkmcnt & BIT(k.opclass[i])) w |= kWcLgkm;
      }
      wcword[i] = w;
      // per-block event flags: bit c = the block holds an instruction the
      // counter-c visitor reacts to (a wait with a value for c, or a member)
      uint32_t ev = 0;
      if (w & kWcIsWait) {
        if ((w & kWcBig) || (w & 0x3FF) != kWcNone) ev |= 1;
        if ((w & kWcBig) || ((w >> 10) & 0x3FF) != kWcNone) ev |= 2;
      } else {
        if (w & kWcVm) ev |= 1;
        if (w & kWcLgkm) ev |= 2;
      }
      if (ev) atomicOr(&bev[k.block_of[i]], ev);
    } else if (k.dialect == LEO_NVIDIA) {
      setword[i] = sk == LEO_SYNC_BARRIER ? (uint8_t)((a | (a >> 8)) & 0x7E) : 0;
    } else {
      setword[i] = (sk == LEO_SYNC_SWSB && a < 32) ? (uint8_t)a : 0xFF;
    }
  }
}

// lastset rows, and setmask[b] = the ids some instruction of block b sets
__global__ void k_block_setters(KView k, const uint8_t* __restrict__ setword, int n_ids,
                                int32_t* __restrict__ lastset, uint32_t* __restrict__ setmask) {
  pdl_wait();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < k.B; b += gridDim.x * blockDim.x) {
    int32_t* row = lastset + (size_t)b * n_ids;
    for (int t = 0; t < n_ids; t++) row[t] = -1;
    uint32_t m = 0;
    for (int x = k.blk_first[b]; x <= k.blk_last[b]; x++) {
      const uint8_t s = setword[x];
      if (k.dialect == LEO_NVIDIA) {
        for (int id = 1; id <= 6; id++) if ((s >> id) & 1) row[id] = x;
        m |= s & 0x7E;
      } else if (s != 0xFF) {
        row[s] = x;
        m |= 1u << s;
      }
    }
    setmask[b] = m;
  }
}

LEO_DEV void sync_emit(const SyncArgs& a, int producer, int wait) {
  int s = atomicAdd(a.key_count, 1);
  if (s < a.key_cap) a.keys[s] = ((uint64_t)(uint32_t)producer << 32) | (uint32_t)wait;
  else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
}

struct Frame { int blk, q, m, a, budget; };

// Chain-walk state of one (wait, counter).  Edges found are buffered (and
// deduplicated) in `seen` and emitted in batches, one global atomic per batch
// (the destructor flushes, so every return path emits).
constexpr int kWcSeen = 32;
struct WcState {
  int counter, level, wait;
  uint32_t member_bit;
  int32_t seen[kWcSeen];
  int nseen = 0;
  uint64_t filt = 0;
  const SyncArgs* sa = nullptr;
  uint64_t* cbuf = nullptr;   // optional CTA buffer in shared memory (one global reservation per CTA)
  int* ccnt = nullptr;
  int ccap = 0;
  LEO_DEV void flush() {
    if (nseen == 0 || !sa) return;
    if (cbuf) {
      const int pos = atomicAdd(ccnt, nseen);
      if (pos + nseen <= ccap) {
        for (int t = 0; t < nseen; t++) cbuf[pos + t] = ((uint64_t)(uint32_t)seen[t] << 32) | (uint32_t)wait;
        nseen = 0;
        return;
      }
    }
    const int base = atomicAdd(sa->key_count, nseen);
    for (int t = 0; t < nseen; t++) {
      if (base + t < sa->key_cap) sa->keys[base + t] = ((uint64_t)(uint32_t)seen[t] << 32) | (uint32_t)wait;
      else atomicOr(sa->status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
    }
    nseen = 0;
  }
  LEO_DEV ~WcState() { flush(); }
};

// waitcnt visitor (depgraph.py:368-384) on a packed word; returns 0 to stop,
// 1 to continue, -1 when the word needs the exact (unpacked) path.
LEO_DEV int wc_visit(uint32_t w, int x, WcState& s, int& m, int& a, const SyncArgs& sa) {
  if (w & kWcIsWait) {
    if (w & kWcBig) return -1;
    uint32_t v = s.counter == 0 ? (w & 0x3FF) : ((w >> 10) & 0x3FF);
    if (v != kWcNone) {
      a = (a < 0) ? (int)v : min(a, (int)v);
      if (a == 0) return 0;
    }
  } else if (w & s.member_bit) {
    if (a != 0) {
      if (m >= s.level) {   // pending[level:] -> edge (buffered, deduplicated per batch)
        // register presence filter first: most members are new to the batch
        const uint64_t fb = 1ull << (((uint32_t)x * 2654435761u) >> 26);
        bool dup = false;
        if (s.filt & fb)
          for (int t = 0; t < s.nseen; t++) if (s.seen[t] == x) { dup = true; break; }
        if (!dup) {
          if (s.nseen == kWcSeen) { s.flush(); s.filt = 0; }
          s.seen[s.nseen++] = x;
          s.filt |= fb;
        }
      }
      m++;
      if (a > 0) { a--; if (a == 0) return 0; }
    }
  }
  return 1;
}

// Scan instructions hi..lo backward (budget per chain).  Returns 0 stopped,
// 1 ran off the block, -1 needs the exact path.
LEO_DEV int wc_scan(const SyncArgs& sa, int hi, int lo, int& budget, WcState& s, int& m, int& a) {
  for (int x = hi; x >= lo; x -= 8) {
    uint32_t w[8];
#pragma unroll
    for (int t = 0; t < 8; t++) w[t] = (x - t >= lo) ? sa.wcword[x - t] : 0u;
#pragma unroll
    for (int t = 0; t < 8; t++) {
      if (x - t < lo) return 1;
      if (budget == 0) return 0;
      budget--;
      int r = wc_visit(w[t], x - t, s, m, a, sa);
      if (r <= 0) return r;
    }
  }
  return 1;
}

LEO_DEV bool on_path(const Frame* fr, int top, int blk) {
  for (int t = 0; t < top; t++) if (fr[t].blk == blk) return true;
  return false;
}

// Enumerate all chains of one (wait, counter).  Returns false on frame
// overflow (re-run with a bigger frame stack) or an unpackable counter value.
constexpr int kT1ChainSteps = 48;   // block scans before a waitcnt item moves to the warp tier

LEO_DEV bool trace_waitcnt_one(const KView& k, int wait, int counter, int level, const SyncArgs& sa,
                               Frame* fr, int fcap, int& best_m, int max_steps = kT1ChainSteps) {
  int steps = 0;
  WcState s;
  s.counter = counter; s.level = level; s.wait = wait;
  s.member_bit = counter == 0 ? kWcVm : kWcLgkm;
  s.nseen = 0; s.sa = &sa;
  const int b0 = k.block_of[wait];
  int m = 0, a = -1, budget = kSyncBudget;
  int r = wc_scan(sa, wait - 1, k.blk_first[b0], budget, s, m, a);
  if (r < 0) return false;
  best_m = 0;
  if (r == 0) { best_m = m; return true; }
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
    if (++steps > max_steps) return false;
    m = f.m; a = f.a; budget = f.budget;
    r = wc_scan(sa, k.blk_last[p], k.blk_first[p], budget, s, m, a);
    if (r < 0) return false;
    if (r == 0) { best_m = max(best_m, m); continue; }
    if (top == fcap) return false;
    fr[top++] = Frame{p, k.pred_ptr[p], m, a, budget};
    bool any = false;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1] && !any; q++)
      if (!on_path(fr, top, k.pred[q])) any = true;
    if (!any) { best_m = max(best_m, m); top--; }
  }
  return true;
}

// ---- tier W: one warp per long waitcnt item ---------------------------------
// Chains are records in shared memory: (block, m, allowance, budget, parent).
// A record is a chain that scanned its whole block without stopping and still
// has unvisited predecessors; its path (the chain's visited set) is the
// parent walk.  Each round every lane expands one record: for each
// predecessor not on the record's path it scans that block with the record's
// state and either ends the chain (stop / no unvisited predecessors: a
// terminal, folded into best_m) or appends a child record.  Same chain set as
// _scan_backward, enumerated breadth-first across lanes.
constexpr int kWcCap = 768;
constexpr int kWcSmemInts = 5 * kWcCap + 8;

LEO_DEV bool rec_on_path(const int32_t* blk, const int32_t* par, int r, int b) {
  for (int x = r; x >= 0; x = par[x]) if (blk[x] == b) return true;
  return false;
}

__global__ void k_sync_wc_warp(KView k, SyncArgs a, const int32_t* __restrict__ list, const int32_t* count,
                               int64_t list_cap, int32_t* slow_list, int32_t* slow_count) {
  pdl_wait();
  extern __shared__ int32_t smw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  int32_t* blk = smw + (size_t)wid * kWcSmemInts;
  int32_t* rm = blk + kWcCap;
  int32_t* ra = rm + kWcCap;
  int32_t* rb = ra + kWcCap;
  int32_t* par = rb + kWcCap;
  int32_t* c = par + kWcCap;     // 0 tail, 1 best_m, 2 ovf
  const int n = (int)min((int64_t)*count, list_cap);
  for (int t = blockIdx.x * wpc + wid; t < n; t += gridDim.x * wpc) {
    const int it = list[t];
    const int wait = it >> 6, counter = it & 63;
    const uint32_t lv = counter == 0 ? k.sync_a[wait] : k.sync_b[wait];
    const int level = (int)lv;
    WcState s;
    s.counter = counter; s.level = level; s.wait = wait;
    s.member_bit = counter == 0 ? kWcVm : kWcLgkm;
    s.nseen = 0; s.sa = &a;
    const int b0 = k.block_of[wait];
    if (lane == 0) {
      c[0] = 0; c[1] = 0; c[2] = 0;
      int m = 0, av = -1, budget = kSyncBudget;
      int r = wc_scan(a, wait - 1, k.blk_first[b0], budget, s, m, av);
      if (r < 0) c[2] = 1;
      else if (r == 0) c[1] = m;
      else {
        bool any = false;
        for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) if (k.pred[q] != b0) any = true;
        if (!any) c[1] = m;
        else { blk[0] = b0; rm[0] = m; ra[0] = av; rb[0] = budget; par[0] = -1; c[0] = 1; }
      }
    }
    __syncwarp();
    int head = 0;
    while (true) {
      // every lane reads the loop control before any lane can modify it
      const int tail = c[0];
      const bool stop = head >= tail || c[2];
      __syncwarp();
      if (stop) break;
      for (int r = head + lane; r < tail; r += 32) {
        const int b = blk[r];
        for (int q = k.pred_ptr[b]; q < k.pred_ptr[b + 1]; q++) {
          const int p = k.pred[q];
          if (rec_on_path(blk, par, r, p)) continue;
          int m = rm[r], av = ra[r], budget = rb[r];
          const int res = wc_scan(a, k.blk_last[p], k.blk_first[p], budget, s, m, av);
          if (res < 0) { c[2] = 1; continue; }
          if (res == 0) { atomicMax(&c[1], m); continue; }
          // child chain: terminal unless it has a predecessor off its path (p included)
          bool any = false;
          for (int q2 = k.pred_ptr[p]; q2 < k.pred_ptr[p + 1] && !any; q2++) {
            const int pp = k.pred[q2];
            if (pp != p && !rec_on_path(blk, par, r, pp)) any = true;
          }
          if (!any) { atomicMax(&c[1], m); continue; }
          const int slot = atomicAdd(&c[0], 1);
          if (slot >= kWcCap) { c[2] = 1; continue; }
          blk[slot] = p; rm[slot] = m; ra[slot] = av; rb[slot] = budget; par[slot] = r;
        }
      }
      __syncwarp();
      head = tail;
      if (c[0] > kWcCap) c[2] = 1;
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) {
      if (c[2]) {
        const int s2 = atomicAdd(slow_count, 1);
        if (s2 < a.slow_cap) slow_list[s2] = it;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      } else if (c[1] < level) {
        diag_push(a.diags, a.status, LEO_DIAG_WAITCNT, wait, counter, level, c[1], counter);
      }
    }
    __syncwarp();
  }
}

// ---- waitcnt items that outgrow the warp tier: CTA per item ------------------
// The same exact chain-tree enumeration as k_sync_wc_warp (one record per
// chain: block, state m / a / budget, parent), but breadth-first over the
// whole CTA with the record arena in global memory (kWcCtaCap records per
// CTA), so a tree of 10^5 chains runs level by level on 1024 threads instead
// of depth-first on one (C4's AMD members: a single such item was ~5 ms on the
// exact walker).  A full arena still ends in the exact walker.
__host__ __device__ inline int wc_cta_cap(int B) {      // records per CTA arena
  return (int)min((int64_t)1 << 20, max((int64_t)1 << 16, (int64_t)64 * B));
}

__global__ void __launch_bounds__(1024) k_sync_wc_cta(KView k, SyncArgs a, const int32_t* __restrict__ list,
                                                      const int32_t* count, int64_t list_cap, int32_t* arena,
                                                      int32_t* slow_list, int32_t* slow_count) {
  pdl_wait();
  __shared__ int c[4];   // 0 tail, 1 best_m, 2 ovf
  const int kWcCtaCap = wc_cta_cap(k.B);
  int32_t* blk = arena + (size_t)blockIdx.x * 5 * kWcCtaCap;
  int32_t* rm = blk + kWcCtaCap;
  int32_t* ra = rm + kWcCtaCap;
  int32_t* rb = ra + kWcCtaCap;
  int32_t* par = rb + kWcCtaCap;
  const int n = (int)min((int64_t)*count, list_cap);
  for (int t = blockIdx.x; t < n; t += gridDim.x) {
    const int it = list[t];
    const int wait = it >> 6, counter = it & 63;
    const uint32_t lv = counter == 0 ? k.sync_a[wait] : k.sync_b[wait];
    const int level = (int)lv;
    WcState s;
    s.counter = counter; s.level = level; s.wait = wait;
    s.member_bit = counter == 0 ? kWcVm : kWcLgkm;
    s.nseen = 0; s.sa = &a;
    const int b0 = k.block_of[wait];
    if (threadIdx.x == 0) {
      c[0] = 0; c[1] = 0; c[2] = 0;
      int m = 0, av = -1, budget = kSyncBudget;
      const int r = wc_scan(a, wait - 1, k.blk_first[b0], budget, s, m, av);
      if (r < 0) c[2] = 1;
      else if (r == 0) c[1] = m;
      else {
        bool any = false;
        for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) if (k.pred[q] != b0) any = true;
        if (!any) c[1] = m;
        else { blk[0] = b0; rm[0] = m; ra[0] = av; rb[0] = budget; par[0] = -1; c[0] = 1; }
      }
    }
    __syncthreads();
    int head = 0;
    while (true) {
      const int tail = c[0];
      const bool stop = head >= tail || c[2];
      __syncthreads();                 // every thread read the loop control
      if (stop) break;
      for (int r = head + (int)threadIdx.x; r < tail; r += blockDim.x) {
        const int b = blk[r];
        for (int q = k.pred_ptr[b]; q < k.pred_ptr[b + 1]; q++) {
          const int p = k.pred[q];
          if (rec_on_path(blk, par, r, p)) continue;
          int m = rm[r], av = ra[r], budget = rb[r];
          const int res = wc_scan(a, k.blk_last[p], k.blk_first[p], budget, s, m, av);
          if (res < 0) { c[2] = 1; continue; }
          if (res == 0) { atomicMax(&c[1], m); continue; }
          bool any = false;
          for (int q2 = k.pred_ptr[p]; q2 < k.pred_ptr[p + 1] && !any; q2++) {
            const int pp = k.pred[q2];
            if (pp != p && !rec_on_path(blk, par, r, pp)) any = true;
          }
          if (!any) { atomicMax(&c[1], m); continue; }
          const int slot = atomicAdd(&c[0], 1);
          if (slot >= kWcCtaCap) { c[2] = 1; continue; }
          blk[slot] = p; rm[slot] = m; ra[slot] = av; rb[slot] = budget; par[slot] = r;
        }
      }
      __syncthreads();
      head = tail;
      if (threadIdx.x == 0 && c[0] > kWcCtaCap) c[2] = 1;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (c[2]) {
        const int s2 = atomicAdd(slow_count, 1);
        if (s2 < a.slow_cap) slow_list[s2] = it;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      } else if (c[1] < level) {
        diag_push(a.diags, a.status, LEO_DIAG_WAITCNT, wait, counter, level, c[1], counter);
      }
    }
    __syncthreads();
  }
}

// ---- exact (unpacked) waitcnt walker for the slow path ----------------------
LEO_DEV int wc_visit_exact(const KView& k, int x, WcState& s, int& m, int& a, const SyncArgs& sa) {
  if (k.sync_kind[x] == LEO_SYNC_WAITCNT) {
    uint32_t v = s.counter == 0 ? k.sync_a[x] : k.sync_b[x];
    if (v != LEO_NONE_U32) {
      long long nv = (a < 0) ? (long long)v : min((long long)a, (long long)v);
      a = (int)min(nv, (long long)0x7FFFFFFF);
      if (a == 0) return 0;
    }
  } else if ((s.counter == 0 ? kVmcnt : kLgkmcnt) & BIT(k.opclass[x])) {
    if (a != 0) {
      if (m >= s.level) sync_emit(sa, x, s.wait);
      m++;
      if (a > 0) { a--; if (a == 0) return 0; }
    }
  }
  return 1;
}
// Exact walker (global scratch).  `onp` (optional, zeroed, one int per
// block) marks the blocks of the current chain (O(1) on-path tests, left
// zeroed on return); `wcword` (optional) lets packable instructions take the
// one-load packed visitor, only big counter values reading the unpacked
// fields.
LEO_DEV bool trace_waitcnt_exact(const KView& k, int wait, int counter, int level, const SyncArgs& sa,
                                 Frame* fr, int fcap, int& best_m, int32_t* onp = nullptr,
                                 const uint32_t* wcword = nullptr) {
  WcState s;
  s.counter = counter; s.level = level; s.wait = wait; s.nseen = 0; s.sa = &sa;
  s.member_bit = counter == 0 ? kWcVm : kWcLgkm;
  auto visit = [&](int x, int& m, int& a) -> int {
    if (wcword) {
      const uint32_t w = wcword[x];
      if (!(w & kWcBig)) return wc_visit(w, x, s, m, a, sa);
    }
    return wc_visit_exact(k, x, s, m, a, sa);
  };
  auto onpath = [&](int top, int blk) { return onp ? onp[blk] != 0 : on_path(fr, top, blk); };
  const int b0 = k.block_of[wait];
  int m = 0, a = -1, budget = kSyncBudget;
  bool stopped = false;
  for (int x = wait - 1; x >= k.blk_first[b0]; x--) {
    if (budget == 0) { stopped = true; break; }
    budget--;
    if (!visit(x, m, a)) { stopped = true; break; }
  }
  best_m = 0;
  if (stopped) { best_m = m; return true; }
  bool any0 = false;
  for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) if (k.pred[q] != b0) any0 = true;
  if (!any0) { best_m = m; return true; }
  int top = 0;
  fr[top++] = Frame{b0, k.pred_ptr[b0], m, a, budget};
  if (onp) onp[b0] = 1;
  while (top > 0) {
    Frame& f = fr[top - 1];
    int p = -1;
    while (f.q < k.pred_ptr[f.blk + 1]) {
      int c = k.pred[f.q++];
      if (!onpath(top, c)) { p = c; break; }
    }
    if (p < 0) { if (onp) onp[f.blk] = 0; top--; continue; }
    m = f.m; a = f.a; budget = f.budget; stopped = false;
    for (int x = k.blk_last[p]; x >= k.blk_first[p]; x--) {
      if (budget == 0) { stopped = true; break; }
      budget--;
      if (!visit(x, m, a)) { stopped = true; break; }
    }
    if (stopped) { best_m = max(best_m, m); continue; }
    if (top == fcap) { if (onp) for (int t = 0; t < top; t++) onp[fr[t].blk] = 0; return false; }
    fr[top++] = Frame{p, k.pred_ptr[p], m, a, budget};
    if (onp) onp[p] = 1;
    bool any = false;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1] && !any; q++)
      if (!onpath(top, k.pred[q])) any = true;
    if (!any) { best_m = max(best_m, m); if (onp) onp[p] = 0; top--; }
  }
  return true;
}

LEO_DEV bool set_hit(int dialect, uint8_t s, int id) {
  return dialect == LEO_NVIDIA ? ((s >> id) & 1) : (s == (uint8_t)id);
}

// Dijkstra state: a small list (fast path) or block-indexed stamp arrays +
// binary heap (slow path).
struct DijSmall {
  int32_t* node; int32_t* dist; uint8_t* done; int cap, n;
  LEO_DEV bool relax(int blk, int d) {
    for (int t = 0; t < n; t++)
      if (node[t] == blk) { if (!done[t] && d < dist[t]) dist[t] = d; return true; }
    if (n == cap) return false;
    node[n] = blk; dist[n] = d; done[n] = 0; n++;
    return true;
  }
  LEO_DEV bool pop(int& blk, int& d) {
    int best = -1;
    for (int t = 0; t < n; t++)
      if (!done[t] && (best < 0 || dist[t] < dist[best])) best = t;
    if (best < 0) return false;
    done[best] = 1; blk = node[best]; d = dist[best];
    return true;
  }
};
struct DijHeap {
  int32_t* stamp; int32_t* dist; uint64_t* heap; int stamp_val, n, cap;
  LEO_DEV bool relax(int blk, int d) {
    if (stamp[blk] == -stamp_val) return true;              // finalised
    if (stamp[blk] == stamp_val && dist[blk] <= d) return true;
    stamp[blk] = stamp_val; dist[blk] = d;
    if (n == cap) return false;
    int i = n++;
    uint64_t key = ((uint64_t)(uint32_t)d << 32) | (uint32_t)blk;
    while (i > 0) { int p = (i - 1) >> 1; if (heap[p] <= key) break; heap[i] = heap[p]; i = p; }
    heap[i] = key;
    return true;
  }
  LEO_DEV bool pop(int& blk, int& d) {
    while (n > 0) {
      uint64_t top = heap[0];
      uint64_t last = heap[--n];
      int i = 0;
      while (true) {
        int c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && heap[c + 1] < heap[c]) c++;
        if (heap[c] >= last) break;
        heap[i] = heap[c]; i = c;
      }
      if (n > 0) heap[i] = last;
      blk = (int)(uint32_t)top; d = (int)(top >> 32);
      if (stamp[blk] == stamp_val && dist[blk] == d) { stamp[blk] = -stamp_val; return true; }
    }
    return false;
  }
};

// The wait's own block: 1 = setter found (emitted), 0 = none and no budget
// left for other blocks, -1 = the block search is needed.
LEO_DEV int setter_in_block(const KView& k, int wait, int id, const SyncArgs& sa) {
  const int b0 = k.block_of[wait];
  const int first0 = k.blk_first[b0];
  const int lo = wait - min(wait - first0, kSyncBudget);
  for (int x = wait - 1; x >= lo; x -= 8) {
    uint8_t w[8];
#pragma unroll
    for (int t = 0; t < 8; t++) w[t] = (x - t >= lo) ? sa.setword[x - t] : 0;
#pragma unroll
    for (int t = 0; t < 8; t++)
      if (x - t >= lo && set_hit(k.dialect, w[t], id)) { sync_emit(sa, x - t, wait); return 1; }
  }
  return wait - first0 >= kSyncBudget ? 0 : -1;
}

// Setter search for one (wait, id).  Returns -1 on overflow, else found (0/1).
template <class Dij>
LEO_DEV int setter_search(const KView& k, int wait, int id, const SyncArgs& sa, Dij& dj) {
  const int b0 = k.block_of[wait];
  const int first0 = k.blk_first[b0];
  const int lo = wait - min(wait - first0, kSyncBudget);
  for (int x = wait - 1; x >= lo; x -= 8) {                 // nearest setter in b0
    uint8_t w[8];
#pragma unroll
    for (int t = 0; t < 8; t++) w[t] = (x - t >= lo) ? sa.setword[x - t] : 0;
#pragma unroll
    for (int t = 0; t < 8; t++)
      if (x - t >= lo && set_hit(k.dialect, w[t], id)) { sync_emit(sa, x - t, wait); return 1; }
  }
  const int cost0 = wait - first0;
  if (cost0 >= kSyncBudget) return 0;
  int found = 0;
  for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) {
    const int p = k.pred[q];
    if (p != b0 && !dj.relax(p, cost0)) return -1;
  }
  int p, d;
  while (dj.pop(p, d)) {
    if (d >= kSyncBudget) break;                             // entering with no budget left
    const int s = sa.lastset[(size_t)p * sa.n_ids + id];
    if (s >= 0) {
      if (d + (k.blk_last[p] - s + 1) <= kSyncBudget) { sync_emit(sa, s, wait); found = 1; }
      continue;
    }
    const int nd = d + (k.blk_last[p] - k.blk_first[p] + 1);
    if (nd >= kSyncBudget) continue;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1]; q++) {
      const int pp = k.pred[q];
      if (pp != b0 && !dj.relax(pp, nd)) return -1;
    }
  }
  return found;
}

// Dijkstra state in shared memory (one CTA per overflowed setter item): an
// open-addressing table block -> (dist, state) and a binary heap with lazy
// deletion.  A search never leaves the 4096-instruction budget, so it
// settles at most 4096 blocks: 8192 table slots and a 16384-entry heap
// always suffice (a full table / heap still reports overflow).
constexpr int kDHSlots = 8192, kDHHeap = 16384;
constexpr size_t kDHBytes = (size_t)kDHSlots * 9 + (size_t)kDHHeap * 8 + 64;

struct DijHash {
  int32_t* key; int32_t* dist; uint8_t* state; uint64_t* heap; int n;
  LEO_DEV int slot(int blk) {              // existing or new slot, -1 when full
    uint32_t h = ((uint32_t)blk * 2654435761u) >> 19;     // 13 bits
    for (int p = 0; p < kDHSlots; p++) {
      const int sl = (int)((h + p) & (kDHSlots - 1));
      if (key[sl] == blk) return sl;
      if (key[sl] == -1) { key[sl] = blk; state[sl] = 0; return sl; }
    }
    return -1;
  }
  LEO_DEV bool relax(int blk, int d) {
    const int sl = slot(blk);
    if (sl < 0) return false;
    if (state[sl] == 2) return true;                       // finalised
    if (state[sl] == 1 && dist[sl] <= d) return true;
    state[sl] = 1; dist[sl] = d;
    if (n == kDHHeap) return false;
    int i = n++;
    const uint64_t kk = ((uint64_t)(uint32_t)d << 32) | (uint32_t)blk;
    while (i > 0) { const int pp = (i - 1) >> 1; if (heap[pp] <= kk) break; heap[i] = heap[pp]; i = pp; }
    heap[i] = kk;
    return true;
  }
  LEO_DEV bool pop(int& blk, int& d) {
    while (n > 0) {
      const uint64_t top = heap[0], last = heap[--n];
      int i = 0;
      while (true) {
        int c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && heap[c + 1] < heap[c]) c++;
        if (heap[c] >= last) break;
        heap[i] = heap[c]; i = c;
      }
      if (n > 0) heap[i] = last;
      blk = (int)(uint32_t)top; d = (int)(top >> 32);
      const int sl = slot(blk);
      if (sl >= 0 && state[sl] == 1 && dist[sl] == d) { state[sl] = 2; return true; }
    }
    return false;
  }
};

constexpr int kFrames = 24, kDij = 64;

__host__ __device__ inline size_t sync_slow_bytes_per_worker(int B) {
  // frames (B+2) + stamp/dist (B+2 each) + heap (4B+8 u64)
  return ((size_t)(B + 2) * (sizeof(Frame) + 8) + (size_t)(4 * B + 16) * 8 + 255) & ~(size_t)255;
}

// compact list of waiting instructions (so no lane idles on non-waits)
__global__ void k_wait_list(KView k, Range own, int32_t* __restrict__ list, int32_t* count) {
  pdl_wait();
  for (int i0 = blockIdx.x * blockDim.x; i0 < k.N; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    bool w = false;
    if (i < k.N && own.has(i)) {
      const uint8_t sk = k.sync_kind[i];
      if (k.dialect == LEO_AMD) w = sk == LEO_SYNC_WAITCNT;
      else if (k.dialect == LEO_NVIDIA) w = sk == LEO_SYNC_BARRIER && ((k.sync_a[i] >> 16) & 0x7E);
      else w = sk == LEO_SYNC_SWSB && k.sync_b[i] != 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, w);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (w) list[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1))] = i;
  }
}

// One thread per waiting instruction; sub-items: amd counters 0/1, nvidia
// barriers 1..6, intel tokens 0..31.  Overflowing items go to the slow list.
template <bool SLOW>
__global__ void k_sync(KView k, SyncArgs a, char* scratch, int nworkers) {
  pdl_wait();
  const int dialect = k.dialect;
  int n_items, stride, start;
  if (SLOW) {
    n_items = (int)min((int64_t)*a.slow_count, a.slow_cap);
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = nworkers;
    if (start >= nworkers) return;
  } else {
    n_items = *a.wait_count;
    start = blockIdx.x * blockDim.x + threadIdx.x;
    stride = gridDim.x * blockDim.x;
  }
  Frame lfr[SLOW ? 1 : kFrames];
  int32_t lnode[SLOW ? 1 : kDij], ldist[SLOW ? 1 : kDij];
  uint8_t ldone[SLOW ? 1 : kDij];
  Frame* fr = lfr;
  int fcap = kFrames;
  int32_t *stamp = nullptr, *gdist = nullptr;
  uint64_t* heap = nullptr;
  const int bcap = SLOW ? a.bcap : k.B;
  if (SLOW) {
    char* base = scratch + (size_t)start * sync_slow_bytes_per_worker(bcap);
    fr = (Frame*)base;
    stamp = (int32_t*)(base + (size_t)(bcap + 2) * sizeof(Frame));
    gdist = stamp + (bcap + 2);
    heap = (uint64_t*)(((uintptr_t)(gdist + (bcap + 2)) + 7) & ~(uintptr_t)7);
    fcap = bcap + 2;
    // a worker with items clears its own stamps (no memset of every worker's
    // scratch ahead of a tier that usually has little to do); the walkers
    // leave the on-path flags cleared after each item
    if (start < n_items)
      for (int x = 0; x < bcap + 2; x++) stamp[x] = 0;
  }
  for (int t = start; t < n_items; t += stride) {
    int i, only = -1;
    if (SLOW) { int it = a.slow_list[t]; i = it >> 6; only = it & 63; }
    else i = a.wait_list[t];
    // block-indexed scratch relative to the item's batch member
    const int sbase = SLOW ? seg_base_of(a, k.block_of[i]) : 0;
    int32_t* stamp_m = SLOW ? stamp - sbase : nullptr;
    int32_t* gdist_m = SLOW ? gdist - sbase : nullptr;
    if (dialect == LEO_AMD) {
      if (k.sync_kind[i] != LEO_SYNC_WAITCNT) continue;
      for (int counter = 0; counter < 2; counter++) {   // vmcnt before lgkmcnt (:410-415)
        if (only >= 0 && only != counter) continue;
        uint32_t lv = counter == 0 ? k.sync_a[i] : k.sync_b[i];
        if (lv == LEO_NONE_U32) continue;
        int best_m = 0;
        bool ok = SLOW ? trace_waitcnt_exact(k, i, counter, (int)min(lv, 0x7FFFFFFFu), a, fr, fcap, best_m,
                                             stamp_m, a.wcword)
                       : (!(a.dbg & LEO_DBG_SYNC_SLOW) && lv < kWcNone &&
                          trace_waitcnt_one(k, i, counter, (int)lv, a, fr, fcap, best_m));
        if (!ok) {
          // fast tier: long chain trees go to the warp tier (or the exact
          // walker for unpackable counter values / when forced); slow tier:
          // frame overflow cannot recur there (frames = B + 2)
          const bool to_warp = !SLOW && lv < kWcNone && !(a.dbg & LEO_DBG_SYNC_SLOW);
          int32_t* lst = to_warp ? a.wc_list : a.slow_list;
          int32_t* cnt = to_warp ? a.wc_count : a.slow_count;
          int s = atomicAdd(cnt, 1);
          if (s < a.slow_cap) lst[s] = (i << 6) | counter;
          else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
          continue;
        }
        if ((long long)best_m < (long long)lv)
          diag_push(a.diags, a.status, LEO_DIAG_WAITCNT, i, counter, (int)min(lv, 0x7FFFFFFFu), best_m, counter);
      }
    } else {
      uint32_t mask;
      if (dialect == LEO_NVIDIA) {
        if (k.sync_kind[i] != LEO_SYNC_BARRIER) continue;
        mask = (k.sync_a[i] >> 16) & 0x7E;
      } else {
        if (k.sync_kind[i] != LEO_SYNC_SWSB) continue;
        mask = k.sync_b[i];
      }
      while (mask) {
        int id = __ffs(mask) - 1;
        mask &= mask - 1;
        if (only >= 0 && only != id) continue;
        int f;
        if (SLOW) {
          DijHeap dj{stamp_m, gdist_m, heap, t + 1, 0, 4 * bcap + 8};
          f = setter_search(k, i, id, a, dj);
        } else if (a.dbg & LEO_DBG_SYNC_SLOW) {
          f = -1;
        } else if (a.defer_search) {
          // nearest setter inside the wait's own block; block searches go to
          // the warp-per-item tier (CFG image in shared memory)
          f = setter_in_block(k, i, id, a);
        } else {
          DijSmall dj{lnode, ldist, ldone, kDij, 0};
          f = setter_search(k, i, id, a, dj);
        }
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

// Block scan with the per-block event flag: a block without events for the
// counter only spends budget (same stop rule as wc_scan: a chain stops when it
// would visit an instruction with no budget left).
// Per-block event lists (shared memory): for counter c, the instructions of
// block b the visitor reacts to, as offsets from the block's first
// instruction, ascending: rel[c][ptr[c][b] .. ptr[c][b+1]).
struct EvList {
  const int32_t* ptr[2];
  const uint16_t* rel[2];
  const int32_t* bf;
  const uint32_t* ww;
};

LEO_DEV int wc_scan_blk(const SyncArgs& sa, const uint32_t* bev, int blk, int hi, int lo, int& budget,
                        WcState& s, int& m, int& a, const EvList* ev = nullptr) {
  if (ev) {
    // visit only the events in [lo, hi], youngest first; the instructions in
    // between only spend budget (a chain stops before visiting an
    // instruction with no budget left, as in wc_scan)
    const int c = s.counter, base = ev->bf[blk], B0 = budget;
    const int e0 = ev->ptr[c][blk];
    for (int e = ev->ptr[c][blk + 1] - 1; e >= e0; e--) {
      const int x = base + ev->rel[c][e];
      if (x > hi) continue;
      if (x < lo) break;
      const int used = hi - x + 1;
      if (B0 < used) { budget = 0; return 0; }
      budget = B0 - used;
      const int r = wc_visit(ev->ww[x], x, s, m, a, sa);
      if (r <= 0) return r;
    }
    const int len = hi - lo + 1;
    if (len <= 0) { budget = B0; return 1; }
    if (B0 >= len) { budget = B0 - len; return 1; }
    budget = 0;
    return 0;
  }
  if (!((bev[blk] >> s.counter) & 1)) {
    const int len = hi - lo + 1;
    if (len <= 0) return 1;
    if (budget >= len) { budget -= len; return 1; }
    budget = 0;
    return 0;
  }
  return wc_scan(sa, hi, lo, budget, s, m, a);
}

// trace_waitcnt_one with O(1) on-path tests: the blocks of the current chain
// are bits of a thread-private bitmap in shared memory (column `pb`, stride
// T words), set on push and cleared on pop.
LEO_DEV bool trace_waitcnt_bits(const KView& k, const uint32_t* bev, uint32_t* pb, int T, int wait, int counter,
                                int level, const SyncArgs& sa, Frame* fr, int fcap, int& best_m, int max_steps,
                                uint64_t* cbuf, int* ccnt, int ccap, const EvList* ev) {
  auto bit = [&](int b) -> bool { return (pb[(b >> 5) * T] >> (b & 31)) & 1u; };
  auto setb = [&](int b) { pb[(b >> 5) * T] |= 1u << (b & 31); };
  auto clrb = [&](int b) { pb[(b >> 5) * T] &= ~(1u << (b & 31)); };
  int steps = 0;
  WcState s;
  s.counter = counter; s.level = level; s.wait = wait;
  s.member_bit = counter == 0 ? kWcVm : kWcLgkm;
  s.nseen = 0; s.sa = &sa; s.cbuf = cbuf; s.ccnt = ccnt; s.ccap = ccap;
  const int b0 = k.block_of[wait];
  int m = 0, a = -1, budget = kSyncBudget;
  int r = wc_scan_blk(sa, bev, b0, wait - 1, k.blk_first[b0], budget, s, m, a, ev);
  if (r < 0) return false;
  best_m = 0;
  if (r == 0) { best_m = m; return true; }
  {
    bool any = false;
    for (int q = k.pred_ptr[b0]; q < k.pred_ptr[b0 + 1]; q++) if (k.pred[q] != b0) any = true;
    if (!any) { best_m = m; return true; }
  }
  int top = 0;
  fr[top++] = Frame{b0, k.pred_ptr[b0], m, a, budget};
  setb(b0);
  auto bail = [&]() { for (int t = 0; t < top; t++) clrb(fr[t].blk); return false; };
  while (top > 0) {
    Frame& f = fr[top - 1];
    int p = -1;
    const int qe = k.pred_ptr[f.blk + 1];
    while (f.q < qe) {
      const int c = k.pred[f.q++];
      if (!bit(c)) { p = c; break; }
    }
    if (p < 0) { clrb(f.blk); top--; continue; }
    if (++steps > max_steps) return bail();
    m = f.m; a = f.a; budget = f.budget;
    r = wc_scan_blk(sa, bev, p, k.blk_last[p], k.blk_first[p], budget, s, m, a, ev);
    if (r < 0) return bail();
    if (r == 0) { best_m = max(best_m, m); continue; }
    if (top == fcap) return bail();
    fr[top++] = Frame{p, k.pred_ptr[p], m, a, budget};
    setb(p);
    bool any = false;
    for (int q = k.pred_ptr[p]; q < k.pred_ptr[p + 1] && !any; q++)
      if (!bit(k.pred[q])) any = true;
    if (!any) { best_m = max(best_m, m); clrb(p); top--; }
  }
  return true;
}

// Shared-memory-resident waitcnt tier (amd): every CTA stages the packed scan
// words and the block table / predecessor CSR with TMA bulk copies, then runs
// the exact chain enumeration of trace_waitcnt_one at shared-memory latency.
// Items are spread one per warp first (item t -> warp t % nwarps, lane
// t / nwarps), so lanes of a warp rarely serialise behind each other.  Items
// whose chain tree outgrows the frame stack or the step bound go to the warp
// tier (global memory); unpackable counter values to the exact walker.
constexpr int kWcSmemSteps = 4096;

constexpr int kWcCtaKeys = 1024;
__host__ __device__ inline size_t sync_smem_bytes(int N, int B, int threads) {
  return 16 + 8 * kWcCtaKeys + 2 * carve_bytes(B + 1, 4) + 2 * carve_bytes(N, 2) + carve_bytes(N, 4) + carve_bytes(B, 4) * 3 + carve_bytes(B + 1, 4) + carve_bytes(2 * (size_t)B + 4, 4)
         + carve_bytes((size_t)((B + 31) >> 5) * threads, 4);
}

__global__ void k_sync_wc_smem(KView k, SyncArgs a, const uint32_t* __restrict__ bev_g, int max_steps) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int N = k.N, B = k.B;
  SmemCarve cv{sm_raw};
  uint64_t* bar = cv.take<uint64_t>(2);
  uint64_t* kbuf = cv.take<uint64_t>(kWcCtaKeys);
  __shared__ int kcnt, kbase;
  if (threadIdx.x == 0) kcnt = 0;
  uint32_t* ww = cv.take<uint32_t>(N);
  int32_t* bf = cv.take<int32_t>(B);
  int32_t* bl = cv.take<int32_t>(B);
  int32_t* pp = cv.take<int32_t>(B + 1);
  int32_t* pr = cv.take<int32_t>(2 * (size_t)B + 4);
  uint32_t* bev4 = cv.take<uint32_t>(B);
  const int T = blockDim.x, W = (B + 31) >> 5;
  uint32_t* pbits = cv.take<uint32_t>((size_t)W * T);
  int32_t* evp0 = cv.take<int32_t>(B + 1);
  int32_t* evp1 = cv.take<int32_t>(B + 1);
  uint16_t* evr0 = cv.take<uint16_t>(N);
  uint16_t* evr1 = cv.take<uint16_t>(N);
  __shared__ int swarp[33];
  __shared__ int ev_ok;
  if (threadIdx.x == 0) ev_ok = 1;
  for (int x = threadIdx.x; x < W * T; x += T) pbits[x] = 0u;
  PhaseMarks pm(a.dbg);
  StageBar sb;
  sb.init(bar, true);                          // one fetch per cluster (launched with a cluster dim)
  sb.begin();
  sb.copy(ww, a.wcword, (size_t)N * 4);
  sb.copy(bf, k.blk_first, (size_t)B * 4);
  sb.copy(bl, k.blk_last, (size_t)B * 4);
  sb.copy(pp, k.pred_ptr, (size_t)(B + 1) * 4);
  sb.copy(pr, k.pred, (size_t)k.pred_ptr[B] * 4);
  sb.copy(bev4, bev_g, (size_t)B * 4);
  sb.commit_and_wait();
  pm.mark(1, 1);
  const uint32_t* bev = bev4;
  // per-block event lists for both counters (count, scan, fill; in smem)
  auto evbits = [](uint32_t w) -> uint32_t {
    if (w & kWcIsWait)
      return (w & kWcBig) ? 3u : (((w & 0x3FF) != kWcNone) ? 1u : 0u) | ((((w >> 10) & 0x3FF) != kWcNone) ? 2u : 0u);
    return ((w & kWcVm) ? 1u : 0u) | ((w & kWcLgkm) ? 2u : 0u);
  };
  {
    // counts: block per thread round-robin (neighbouring lanes read
    // neighbouring instructions: few bank conflicts)
    for (int b = threadIdx.x; b < B; b += T) {
      if (bl[b] - bf[b] >= 65535) ev_ok = 0;
      int c0 = 0, c1 = 0;
      for (int x = bf[b]; x <= bl[b]; x++) { const uint32_t f = evbits(ww[x]); c0 += f & 1; c1 += f >> 1; }
      evp0[b] = c0; evp1[b] = c1;
    }
    __syncthreads();
    pm.mark(1, 4);
    // exclusive scan of the counts (thread-contiguous chunks)
    const int per = (B + T - 1) / T, lo = min(B, (int)threadIdx.x * per), hi = min(B, lo + per);
    int s0 = 0, s1 = 0;
    for (int b = lo; b < hi; b++) { s0 += evp0[b]; s1 += evp1[b]; }
    int t0, t1;
    int r0 = block_excl_scan(s0, swarp, &t0);
    int r1 = block_excl_scan(s1, swarp, &t1);
    for (int b = lo; b < hi; b++) {
      const int c0 = evp0[b], c1 = evp1[b];
      evp0[b] = r0; evp1[b] = r1;
      r0 += c0; r1 += c1;
    }
    if (threadIdx.x == 0) { evp0[B] = t0; evp1[B] = t1; }
    __syncthreads();
    pm.mark(1, 5);
    for (int b = threadIdx.x; b < B; b += T) {
      int q0 = evp0[b], q1 = evp1[b];
      for (int x = bf[b]; x <= bl[b]; x++) {
        const uint32_t f = evbits(ww[x]);
        if (f & 1) evr0[q0++] = (uint16_t)(x - bf[b]);
        if (f & 2) evr1[q1++] = (uint16_t)(x - bf[b]);
      }
    }
    __syncthreads();
  }
  pm.mark(1, 2);
  EvList evl{{evp0, evp1}, {evr0, evr1}, bf, ww};
  const EvList* ev = ev_ok ? &evl : nullptr;
  KView ks = k;
  ks.blk_first = bf; ks.blk_last = bl; ks.pred_ptr = pp; ks.pred = pr;
  SyncArgs as = a;
  as.wcword = ww;
  const int n_items = *a.wait_count;
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  Frame fr[kFrames];
  for (int t = lane * nwarps + gw; t < n_items; t += 32 * nwarps) {
    const int i = a.wait_list[t];
    if (k.sync_kind[i] != LEO_SYNC_WAITCNT) continue;
    for (int counter = 0; counter < 2; counter++) {   // vmcnt before lgkmcnt (:410-415)
      const uint32_t lv = counter == 0 ? k.sync_a[i] : k.sync_b[i];
      if (lv == LEO_NONE_U32) continue;
      int best_m = 0;
      const long long c0 = clock64();
      const bool ok = !(a.dbg & LEO_DBG_SYNC_SLOW) && lv < kWcNone &&
                      trace_waitcnt_bits(ks, bev, pbits + threadIdx.x, T, i, counter, (int)lv, as, fr, kFrames,
                                         best_m, max_steps, kbuf, &kcnt, kWcCtaKeys, ev);
      if ((a.dbg & LEO_DBG_PHASES) && t < 4096) g_item_cycles[t * 2 + counter] = clock64() - c0;
      if (!ok) {
        const bool to_warp = lv < kWcNone && !(a.dbg & LEO_DBG_SYNC_SLOW);
        int32_t* lst = to_warp ? a.wc_list : a.slow_list;
        int32_t* cnt = to_warp ? a.wc_count : a.slow_count;
        const int s2 = atomicAdd(cnt, 1);
        if (s2 < a.slow_cap) lst[s2] = (i << 6) | counter;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
        continue;
      }
      if ((long long)best_m < (long long)lv)
        diag_push(a.diags, a.status, LEO_DIAG_WAITCNT, i, counter, (int)lv, best_m, counter);
    }
  }
  __syncthreads();
  const int nk = min(kcnt, kWcCtaKeys);
  if (threadIdx.x == 0) kbase = nk > 0 ? atomicAdd(a.key_count, nk) : 0;
  __syncthreads();
  for (int x = threadIdx.x; x < nk; x += blockDim.x) {
    if (kbase + x < a.key_cap) a.keys[kbase + x] = kbuf[x];
    else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
  }
  pm.mark(1, 3);
}

// Setter searches that overflowed the thread tier's 64-node Dijkstra (nvidia
// barriers / intel SWSB tokens): one CTA per item, the search state in shared
// memory (DijHash); items still overflowing go to the global-scratch worker.
__global__ void k_sync_setter_smem(KView k, SyncArgs a, int32_t* slow_out, int32_t* slow_out_count) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  SmemCarve cv{sm_raw};
  uint64_t* heap = cv.take<uint64_t>(kDHHeap);
  int32_t* key = cv.take<int32_t>(kDHSlots);
  int32_t* dist = cv.take<int32_t>(kDHSlots);
  uint8_t* state = cv.take<uint8_t>(kDHSlots);
  const int n_items = (int)min((int64_t)*a.slow_count, a.slow_cap);
  for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
    for (int x = threadIdx.x; x < kDHSlots; x += blockDim.x) key[x] = -1;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int it = a.slow_list[t], i = it >> 6, id = it & 63;
      DijHash dj{key, dist, state, heap, 0};
      const int f = (a.dbg & LEO_DBG_SYNC_SLOW) ? -1 : setter_search(k, i, id, a, dj);
      if (f < 0) {
        const int s2 = atomicAdd(slow_out_count, 1);
        if (s2 < a.slow_cap) slow_out[s2] = it;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      } else if (!f) {
        diag_push(a.diags, a.status, LEO_DIAG_NO_SETTER, i, id, 0, 0, id);
      }
    }
    __syncthreads();
  }
}

// ---- setter searches: warp per item, CFG image in shared memory -------------
// The block search of _trace_setter (depgraph.py:431-443) reduces to shortest
// paths: setter block p yields its last setter s iff dist(p) + (last(p) - s +
// 1) <= budget, dist over setter-free, b0-free predecessor paths weighted by
// block length.  Any exact shortest-path method gives the same set, so a warp
// relaxes a frontier in parallel (label-correcting Bellman-Ford) instead of
// one thread running Dijkstra: each round every lane expands one frontier
// block, and a block whose distance drops joins the next frontier once.
// Distances live in a per-warp open-addressing table in shared memory; the
// CFG image (block bounds, setter-id masks, predecessor CSR) is staged once
// per CTA with TMA bulk copies.  A full table or frontier sends the item on
// to the global-scratch Dijkstra tier.
constexpr int kSWSlots = 1024, kSWFront = 512, kSWWarps = 4;

__host__ __device__ inline size_t setter_warp_tables_smem() {
  return (size_t)kSWWarps * (carve_bytes(kSWSlots, 4) * 3 + carve_bytes(2 * kSWFront, 4) + 16);
}
__host__ __device__ inline size_t setter_cta_smem(int B) {
  return 16 + carve_bytes(B, 4) * 3 + carve_bytes((size_t)B + 1, 4) + carve_bytes(2 * (size_t)B + 4, 4)
         + setter_warp_tables_smem();
}

// STAGE = false (the CFG image does not fit): the same searches read the
// block tables from global memory (L2-resident), only the per-warp tables
// live in shared memory.
template <bool STAGE>
__global__ void __launch_bounds__(kSWWarps * 32) k_sync_setter_cta(KView k, SyncArgs a, const uint32_t* __restrict__ setmask_g,
                                                                 int32_t* slow_out, int32_t* slow_out_count) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int B = k.B, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SmemCarve cv{sm_raw};
  uint64_t* bar = cv.take<uint64_t>(2);
  const int32_t* bf = k.blk_first;
  const int32_t* bl = k.blk_last;
  const uint32_t* smask = setmask_g;
  const int32_t* pptr = k.pred_ptr;
  const int32_t* pred = k.pred;
  int32_t *sbf = nullptr, *sbl = nullptr, *spptr = nullptr, *spred = nullptr;
  uint32_t* ssmask = nullptr;
  if (STAGE) {
    sbf = cv.take<int32_t>(B); sbl = cv.take<int32_t>(B); ssmask = cv.take<uint32_t>(B);
    spptr = cv.take<int32_t>(B + 1); spred = cv.take<int32_t>(2 * (size_t)B + 4);
    bf = sbf; bl = sbl; smask = ssmask; pptr = spptr; pred = spred;
  }
  unsigned char* wbase = cv.p;
  cv.p = wbase + (size_t)wid * (carve_bytes(kSWSlots, 4) * 3 + carve_bytes(2 * kSWFront, 4) + 16);
  int32_t* key = cv.take<int32_t>(kSWSlots);
  int32_t* dist = cv.take<int32_t>(kSWSlots);
  int32_t* fst = cv.take<int32_t>(kSWSlots);
  int32_t* front = cv.take<int32_t>(2 * kSWFront);
  int32_t* wctl = cv.take<int32_t>(4);        // [0] next frontier size, [1] overflow
  const int n_items = (int)min((int64_t)*a.slow_count, a.slow_cap);
  if ((int)blockIdx.x * kSWWarps >= n_items) return;
  if (STAGE) {
    StageBar sb;
    sb.init(bar);
    sb.begin();
    const int P = k.pred_ptr[B];
    sb.copy(sbf, k.blk_first, (size_t)B * 4);
    sb.copy(sbl, k.blk_last, (size_t)B * 4);
    sb.copy(ssmask, setmask_g, (size_t)B * 4);
    sb.copy(spptr, k.pred_ptr, (size_t)(B + 1) * 4);
    sb.copy(spred, k.pred, (size_t)P * 4);
    sb.commit_and_wait();
  }

  auto find = [&](int p) -> int {
    uint32_t h = ((uint32_t)p * 2654435761u) >> 22;             // 10 bits
    for (int t = 0; t < kSWSlots; t++) {
      const int sl = (int)((h + t) & (kSWSlots - 1));
      const int kk = key[sl];
      if (kk == p) return sl;
      if (kk == -1) return -1;
    }
    return -1;
  };
  for (int it = blockIdx.x * kSWWarps + wid; it < n_items; it += gridDim.x * kSWWarps) {
    const int item = a.slow_list[it], i = item >> 6, id = item & 63;
    const int b0 = k.block_of[i];
    const int cost0 = i - bf[b0];
    for (int x = lane; x < kSWSlots; x += 32) { key[x] = -1; dist[x] = 0x7FFFFFFF; fst[x] = 0; }
    if (lane == 0) { wctl[0] = 0; wctl[1] = 0; }
    __syncwarp();
    int round = 1;
    int32_t* cur = front;
    int32_t* nxt = front + kSWFront;
    // relax pp with distance d; a drop queues pp for round `round + 1`
    auto relax = [&](int pp, int d) {
      uint32_t h = ((uint32_t)pp * 2654435761u) >> 22;
      int sl = -1;
      for (int t = 0; t < kSWSlots; t++) {
        const int c = (int)((h + t) & (kSWSlots - 1));
        const int prev = atomicCAS(&key[c], -1, pp);
        if (prev == -1 || prev == pp) { sl = c; break; }
      }
      if (sl < 0) { wctl[1] = 1; return; }
      if (atomicMin(&dist[sl], d) > d && atomicExch(&fst[sl], round + 1) != round + 1) {
        const int f = atomicAdd(&wctl[0], 1);
        if (f < kSWFront) nxt[f] = pp; else wctl[1] = 1;
      }
    };
    // round 0: the wait block's predecessors (b0 itself is never re-entered)
    for (int q = pptr[b0] + lane; q < pptr[b0 + 1]; q += 32) {
      const int pp = pred[q];
      if (pp != b0) relax(pp, cost0);
    }
    __syncwarp();
    int nf = min(wctl[0], kSWFront);
    bool ovf = wctl[1] != 0;
    __syncwarp();
    while (nf > 0 && !ovf) {
      { int32_t* t = cur; cur = nxt; nxt = t; }
      round++;
      if (lane == 0) wctl[0] = 0;
      __syncwarp();
      for (int x = lane; x < nf; x += 32) {
        const int p = cur[x];
        if ((smask[p] >> id) & 1) continue;                   // setter blocks end the path
        const int sl = find(p);
        const int nd = dist[sl] + (bl[p] - bf[p] + 1);
        if (nd >= kSyncBudget) continue;
        for (int q = pptr[p]; q < pptr[p + 1]; q++) {
          const int pp = pred[q];
          if (pp != b0) relax(pp, nd);
        }
      }
      __syncwarp();
      nf = min(wctl[0], kSWFront);
      ovf = wctl[1] != 0;
      __syncwarp();
    }
    if (ovf) {
      if (lane == 0) {
        const int s2 = atomicAdd(slow_out_count, 1);
        if (s2 < a.slow_cap) slow_out[s2] = item;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      }
      __syncwarp();
      continue;
    }
    // settled: every reached setter block within the budget yields its last setter
    bool found = false;
    for (int x = lane; x < kSWSlots; x += 32) {
      const int p = key[x];
      if (p < 0 || !((smask[p] >> id) & 1)) continue;
      const int s = a.lastset[(size_t)p * a.n_ids + id];
      if (dist[x] + (bl[p] - s + 1) <= kSyncBudget) { sync_emit(a, s, i); found = true; }
    }
    if (!__any_sync(0xffffffffu, found) && lane == 0) diag_push(a.diags, a.status, LEO_DIAG_NO_SETTER, i, id, 0, 0, id);
    __syncwarp();
  }
}

template __global__ void k_sync_setter_cta<true>(KView, SyncArgs, const uint32_t*, int32_t*, int32_t*);
template __global__ void k_sync_setter_cta<false>(KView, SyncArgs, const uint32_t*, int32_t*, int32_t*);
template __global__ void k_sync<false>(KView, SyncArgs, char*, int);
template __global__ void k_sync<true>(KView, SyncArgs, char*, int);

// ---- group raw keys by producer, dedup, append after the raw/guard edges ----
__global__ void k_key_hist(const uint64_t* __restrict__ keys, const int32_t* n_dev, int64_t cap,
                           int32_t* __restrict__ cnt) {
  pdl_wait();
  int64_t n = min((int64_t)*n_dev, cap);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[(int)(keys[x] >> 32)], 1);
}
__global__ void k_key_scatter(const uint64_t* __restrict__ keys, const int32_t* n_dev, int64_t cap,
                              const int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                              uint64_t* __restrict__ out) {
  pdl_wait();
  int64_t n = min((int64_t)*n_dev, cap);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
    int p = (int)(keys[x] >> 32);
    out[off[p] + atomicAdd(&cursor[p], 1)] = keys[x];
  }
}
__global__ void k_sync_emit(int N, int kind, const uint64_t* __restrict__ sorted,
                            const int32_t* __restrict__ off, const int32_t* __restrict__ uniq,
                            const int32_t* __restrict__ uoff, const int32_t* n_regular,
                            const int32_t* n_sync, LeoEdges out, uint32_t* status) {
  pdl_wait();
  const int base = *n_regular;
  if (blockIdx.x == 0 && threadIdx.x == 0) {     // edge totals (was k_edge_totals)
    const int t = base + *n_sync;
    if (t > out.capacity) atomicOr(status, (uint32_t)LEO_ST_EDGE_OVERFLOW);
    *out.n_regular = min(base, out.capacity);
    *out.count = min(t, out.capacity);
  }
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
// (edge totals are clamped to the capacity so downstream kernels never read
// past the buffers; an overflow is signalled in the status word and the host
// re-runs)

}  // namespace leo
