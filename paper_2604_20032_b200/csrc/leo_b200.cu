// leo_b200.cu — extern "C" entry points of libleo_b200.so (include/leo_b200.h).
//
// Each entry point enqueues its kernels on the caller's stream; scratch comes
// from the stream-ordered allocator (cudaMallocAsync) and is released on the
// same stream.  No host synchronisation happens inside the pipeline: every
// data-dependent size lives in device memory and the kernels read it there.
#include <algorithm>
#include <functional>
#include <vector>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "prims.cuh"
#include "graph.cu"
#include "sync.cu"
#include "prune.cu"
#include "blame.cu"
#include "report.cu"
#include "api_ops.cu"


using namespace leo;

namespace leo {
int scan_coop_grid() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& g = cache[dev & 63];
  if (!g) {
    int per = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, scan_coop, kCsThreads, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = std::max(1, per) * std::max(1, sms);
  }
  return g;
}
}  // namespace leo

namespace {

// ---- optional device-time trace (LeoTrace) ---------------------------------
enum KernelId {
  KID_BIN = 0, KID_BIN_FINALIZE, KID_UNIT_COUNTS, KID_SCAN, KID_BLOCK_WALK, KID_REACH_FAST,
  KID_REACH_SLOW, KID_LINK_COUNT, KID_LINK_FILL, KID_SEGSORT, KID_LINK_EMIT, KID_SYNC,
  KID_SYNC_SLOW, KID_KEY_HIST, KID_KEY_SCATTER, KID_SYNC_EMIT, KID_EDGE_TOTALS, KID_PRUNE,
  KID_PRUNE_SLOW, KID_COMPACT, KID_SEG_BOUNDS, KID_SYNC_HIST, KID_SYNC_FILL, KID_BLAME_COUNT,
  KID_SELFBLAME_SLOW, KID_BLAME_FILL, KID_BLAME_TOTAL, KID_LINES, KID_SLICE, KID_REACH_WARP, KID_RUN_HEADS, KID_BIN_HIST, KID_BIN_PLAN, KID_BIN_SCATTER, KID_SYNC_PACK, KID_SYNC_WARP, KID_SELFBLAME_WARP, KID_SELF_ADDR, KID_COUNT_
};
const char* const kKernelNames[] = {
  "bin_samples", "bin_finalize", "unit_counts", "scan", "block_walk", "reach_fast",
  "reach_slow", "link_count", "link_fill", "segsort_unique", "link_emit", "sync_trace",
  "sync_trace_slow", "key_hist", "key_scatter", "sync_emit", "edge_totals", "prune_edges",
  "prune_slow", "compact", "seg_bounds", "sync_hist", "sync_fill", "blame_count",
  "selfblame_slow", "blame_fill", "blame_total", "lines", "slice", "reach_warp", "run_heads", "bin_hist", "bin_plan", "bin_scatter", "sync_pack", "sync_warp", "selfblame_warp", "self_addr",
};

struct TraceScope {
  LeoTrace* t; cudaStream_t st; int slot = -1;
  TraceScope(LeoTrace* tr, int id, cudaStream_t s) : t(tr), st(s) {
    if (!t || (t->only_kernel >= 0 && t->only_kernel != id)) return;
    int x = t->count++;
    if (x >= t->capacity) return;
    slot = x;
    t->kernel_id[x] = id;
    record((cudaEvent_t)t->ev_begin[x]);
  }
  // inside a stream capture the record becomes an event-record node (a
  // timeline of graph replays)
  void record(cudaEvent_t ev) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
    else cudaEventRecord(ev, st);
  }
  ~TraceScope() { if (slot >= 0) record((cudaEvent_t)t->ev_end[slot]); }
};
// LEO_DEBUG_SYNC=1: synchronise after every kernel and report the first
// failing (or hanging: last printed) kernel on stderr (debugging aid)
bool debug_sync_env() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("LEO_DEBUG_SYNC"); v = (e && e[0] == '1') ? 1 : 0; }
  return v == 1;
}
inline void debug_sync_after(int id, cudaStream_t st) {
  if (!debug_sync_env()) return;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "[leo debug] kernel %d failed: %s\n", id, cudaGetErrorString(e));
}
#define TRACED(id, ...) do { if (debug_sync_env()) { fprintf(stderr, "[leo debug] launch %d\n", (int)(id)); fflush(stderr); } \
  { TraceScope _ts(tr, id, st); __VA_ARGS__; } debug_sync_after(id, st); } while (0)

// LEO_NO_FORK=1: run every stage on the caller's stream (debugging aid)
// critical-path probe (profiling only): LEO_DBG_DELAY_<BRANCH>=<us> puts a
// spin of that length at the head of the branch; if the step grows by the
// same amount, the branch has no slack
__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
void dbg_delay(const char* env, cudaStream_t st) {
  const char* v = getenv(env);
  if (!v) return;
  const double us = atof(v);
  if (us > 0) k_spin<<<1, 1, 0, st>>>((long long)(us * 1965.0));
}
bool no_fork_env() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("LEO_NO_FORK"); v = (e && e[0] == '1') ? 1 : 0; }
  return v == 1;
}

// SM count of the calling thread's current device (cached per device: one
// process may drive several GPUs)
int num_sms() {
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = cache[dev & 63];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Caller-owned workspace (LeoCaps.workspace): every arena of one entry-point
// call is bump-allocated from it (no reuse inside a call, so concurrent
// branches never alias); the bytes wanted are reported back so the caller can
// size it.  Without a big enough workspace the stream-ordered allocator is used.
struct WsCursor { char* base = nullptr; size_t cap = 0, off = 0, needed = 0; };
thread_local WsCursor* t_ws = nullptr;
struct WsScope {
  WsCursor c;
  WsCursor* prev;
  const LeoCaps* caps;
  explicit WsScope(const LeoCaps* cp) : prev(t_ws), caps(cp) {
    if (cp && cp->workspace && cp->workspace_bytes > 0) {
      c.base = (char*)cp->workspace;
      c.cap = (size_t)cp->workspace_bytes;
    }
    t_ws = &c;
  }
  ~WsScope() {
    if (caps && caps->workspace_needed) *caps->workspace_needed = (int64_t)c.needed;
    t_ws = prev;
  }
};

// Stream-ordered bump arena: one allocation per stage.
struct Arena {
  cudaStream_t st;
  char* base = nullptr;
  size_t cap = 0, off = 0;
  struct Req { void** dst; size_t bytes; };
  Req reqs[96];
  int nreq = 0;
  template <typename T> void want(T** dst, int64_t n) {
    reqs[nreq++] = Req{(void**)dst, (size_t)std::max<int64_t>(n, 1) * sizeof(T)};
  }
  bool from_ws = false;
  cudaError_t commit() {
    size_t total = 0;
    for (int i = 0; i < nreq; i++) total += (reqs[i].bytes + 255) & ~(size_t)255;
    if (t_ws) t_ws->needed += total;
    if (t_ws && t_ws->base && t_ws->off + total <= t_ws->cap) {
      base = t_ws->base + t_ws->off;
      t_ws->off += total;
      from_ws = true;
    } else {
      cudaError_t e = cudaMallocAsync((void**)&base, total, st);
      if (e != cudaSuccess) return e;
    }
    cap = total;
    for (int i = 0; i < nreq; i++) {
      *reqs[i].dst = base + off;
      off += (reqs[i].bytes + 255) & ~(size_t)255;
    }
    return cudaSuccess;
  }
  void release() { if (base && !from_ws) cudaFreeAsync(base, st); base = nullptr; }
};

inline int64_t pick(int64_t hint, int64_t dflt) { return hint > 0 ? hint : dflt; }

// Side streams + events for fork/join concurrency inside one pipeline call
// (independent stages run as parallel branches; under stream capture they
// become parallel branches of the CUDA graph).  One pool per (host thread,
// device, caller stream): calls on different streams or devices never share
// side streams (no false serialisation between them).
struct SidePool {
  cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t e[8] = {};
  bool ok = false;
  void init() {
    if (ok) return;
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    for (auto& x : e) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
    ok = true;
  }
};
SidePool& side_pool(cudaStream_t caller) {
  struct Key { int dev; cudaStream_t st; SidePool* p; };
  static thread_local std::vector<Key> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& k : pools)
    if (k.dev == dev && k.st == caller) return *k.p;
  pools.push_back(Key{dev, caller, new SidePool()});
  pools.back().p->init();
  return *pools.back().p;
}
// `to` waits for all work enqueued so far on `from`
inline void link_streams(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  cudaEventRecord(ev, from);
  cudaStreamWaitEvent(to, ev, 0);
}

// kernels that take more than 48 KiB of dynamic shared memory (a per-device
// function attribute: set once per device)
void set_smem_attributes() {
  static uint64_t done_mask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done_mask & bit) return;
  cudaFuncSetAttribute(k_reach_fast<int32_t, 128, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT1Threads * 128 * 4);
  cudaFuncSetAttribute(k_reach_fast<uint16_t, 128, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT1Threads * 128 * 2);
  cudaFuncSetAttribute(k_reach_fast<uint16_t, 64, 48>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT1Threads * 64 * 2);
  cudaFuncSetAttribute(k_reach_fast<int32_t, 64, 48>, cudaFuncAttributeMaxDynamicSharedMemorySize, kT1Threads * 64 * 4);
  cudaFuncSetAttribute(k_bin_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kBinRMax * 8 * 4);
  for (auto f : {k_bin_hash<8192, 8>, k_bin_hash<8192, 4>, k_bin_hash<16384, 4>,
                 k_bin_hash<16384, 2>, k_bin_hash<26624, 4>, k_bin_hash<26624, 2>,
                 k_bin_hash<26624, 8>, k_bin_hash<16384, 2, 4>, k_bin_hash<16384, 2, 3>,
                 k_bin_hash<16384, 2, 3, 5>})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 26624 * 8);
  cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kBinMaxBuckets * 12 + kBinSub * 4);
  cudaFuncSetAttribute(k_block_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(k_sync_wc_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kWcSmemInts * 4);
  cudaFuncSetAttribute(k_reach_unit, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemResidentMax);
  cudaFuncSetAttribute(k_sync_wc_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemResidentMax);
  cudaFuncSetAttribute(k_sync_setter_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDHBytes);
  cudaFuncSetAttribute(k_sync_setter_cta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemResidentMax);
  cudaFuncSetAttribute(k_sync_setter_cta<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(16 + setter_warp_tables_smem()));
  cudaFuncSetAttribute(k_prune_edges_smem<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemResidentMax);
  cudaFuncSetAttribute(k_prune_edges_smem<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemResidentMax);
  done_mask |= bit;
}

int check_kernel(const LeoKernel* k) {
  set_smem_attributes();
  if (!k || k->n_instr < 0 || k->n_blocks < 0 || k->n_units < 0) return -1;
  if (k->n_instr >= (1 << 30) || k->n_units > (1 << 24)) return -2;
  if ((int64_t)k->n_blocks * k->n_units > ((int64_t)1 << 30)) return -4;   // dense last-def table
  return 0;
}

// ---------------------------------------------------------------------------
// build_graph
int build_graph_impl(const LeoKernel* kk, const LeoCaps* caps, LeoEdges* out, LeoDiags* diags,
                     uint32_t* status, cudaStream_t st, Range own = Range{0, 0},
                     const std::function<int()>& after_walk = {}, LeoReachIn* rall = nullptr) {
  LeoTrace* tr = caps ? caps->trace : nullptr;
  KView k = make_kview(kk);
  const int N = k.N, B = k.B, U = k.U;
  const int64_t NU = kk->n_use_units, ND = kk->n_def_units;
  // rall (leo_reaching_definitions): every (block, unit) pair is a query
  const int64_t NQ = NU + (rall ? (int64_t)B * U : 0);
  const int64_t cap_qres = pick(caps ? caps->query_results : 0, 4 * NQ + 1024);
  const int64_t cap_cand = pick(caps ? caps->candidates : 0, 6 * NU + 1024);
  const int64_t cap_sync = pick(caps ? caps->sync_keys : 0, 2 * (int64_t)N + 1024);
  const int64_t cap_slow = pick(caps ? caps->slow_items : 0, N / 4 + 1024);
  const int SM = num_sms();
  constexpr int kWcCtaGrid = 8;   // CTAs of the CTA waitcnt tier (items that outgrow the warp tier are few)

  // per-warp unit tables in shared memory when they fit
  auto walk_bytes = [&](int w, bool tab) { return (size_t)w * ((tab ? 4 * (size_t)U : 0) + kWalkStage) * 4; };
  int wpc = 8;
  while (wpc > 1 && walk_bytes(wpc, true) > 96 * 1024) wpc >>= 1;
  const bool smem_tab = walk_bytes(wpc, true) <= 96 * 1024;
  if (!smem_tab) wpc = 8;
  const int walk_ctas = std::min<int>((B + wpc - 1) / wpc, SM * 8);
  const int walk_warps = std::max(1, walk_ctas) * wpc;

  const int RW = 128;        // slow reach workers
  // slow sync workers: block-indexed scratch spans the largest batch member;
  // as many workers as ~192 MB of scratch allows (16..2048)
  const int sync_bcap = (kk->n_segments > 1 && kk->seg_block) ? std::max(1, (int)kk->max_seg_blocks) : B;
  const int SW = (int)std::max<int64_t>(16, std::min<int64_t>(2048, ((int64_t)192 << 20) /
                                        (int64_t)sync_slow_bytes_per_worker(sync_bcap)) & ~(int64_t)15);
  Arena ar{st};
  int32_t *ucnt, *dcnt, *use_ptr, *def_ptr, *ev_res, *q_block, *q_unit, *q_list, *q_off, *q_len, *qres;
  int32_t *ctr, *slow_list, *slow2, *slow3, *cand_cnt, *cand_off, *uniq, *eoff, *ldtab, *scan_tmp, *gtab = nullptr;
  int4* brec;
  int32_t *pcnt, *poff, *pcur, *puniq, *puoff, *reach_scr, *scan_tmp2, *wlist, *wclist, *qtab, *rhead, *slow3s;
  uint64_t *cand, *skeys, *ssorted;
  uint32_t *wcword, *bev;
  uint8_t* setword;
  int32_t* lastset;
  char* sync_scr;
  ar.want(&ucnt, N); ar.want(&dcnt, N); ar.want(&use_ptr, N + 1); ar.want(&def_ptr, N + 1);
  ar.want(&ev_res, NU); ar.want(&q_block, NQ); ar.want(&q_unit, NQ); ar.want(&q_list, NQ);
  ar.want(&q_off, NQ); ar.want(&q_len, NQ); ar.want(&qres, cap_qres); ar.want(&ctr, 16);
  ar.want(&slow_list, NQ + 1024); ar.want(&slow2, cap_slow); ar.want(&slow3, NQ + 1024); ar.want(&cand_cnt, N); ar.want(&cand_off, N + 1);
  const int Bp = (B + 3) & ~3;   // 16-byte aligned unit columns
  ar.want(&uniq, N); ar.want(&eoff, N + 1); ar.want(&ldtab, (int64_t)Bp * U); ar.want(&qtab, (int64_t)Bp * U);
  ar.want(&brec, B); ar.want(&rhead, B);
  ar.want(&cand, cap_cand); ar.want(&skeys, cap_sync); ar.want(&ssorted, cap_sync);
  ar.want(&pcnt, N); ar.want(&poff, N + 1); ar.want(&pcur, N); ar.want(&puniq, N); ar.want(&puoff, N + 1);
  ar.want(&scan_tmp, scan_scratch_ints(std::max<int64_t>(std::max<int64_t>(N, cap_cand), 1)) + 64);
  ar.want(&reach_scr, (int64_t)RW * 3 * (B + 1));
  ar.want(&scan_tmp2, scan_scratch_ints(std::max<int64_t>(N, 1)) + 64);
  ar.want(&wlist, N); ar.want(&wclist, cap_slow); ar.want(&slow3s, cap_slow);
  // the CTA waitcnt tier's record arenas (amd): kWcCtaGrid x 5 x kWcCtaCap ints
  int32_t* wc_arena = nullptr;
  const bool use_wc_cta = k.dialect == LEO_AMD && !getenv("LEO_WC_NO_CTA") &&
                          (getenv("LEO_WC_CTA") || N >= (1 << 17) || kk->n_segments > 1);
  if (use_wc_cta) ar.want(&wc_arena, (int64_t)kWcCtaGrid * 5 * wc_cta_cap(B));
  ar.want(&sync_scr, (int64_t)SW * sync_slow_bytes_per_worker(sync_bcap));
  const int n_ids = k.dialect == LEO_INTEL ? 32 : 8;
  ar.want(&wcword, N); ar.want(&bev, B); ar.want(&setword, N); ar.want(&lastset, (int64_t)B * n_ids);
  if (!smem_tab) ar.want(&gtab, (int64_t)walk_warps * 2 * U);
  int32_t *rcnt = nullptr, *rscan = nullptr;
  if (rall) { ar.want(&rcnt, (int64_t)B * U); ar.want(&rscan, scan_scratch_ints(std::max<int64_t>((int64_t)B * U, 1)) + 64); }
  LEO_CUDA_CHECK(ar.commit());
  // counters: 0 q_count, 1 qres_count, 2 reach slow, 3 sync keys, 4 sync slow, 5 n_regular, 6 n_sync
  cudaMemsetAsync(ctr, 0, 16 * sizeof(int32_t), st);
  const int T = 256;
  // fork: vendor sync tracing runs on a side stream, concurrently with the
  // register dataflow chain below
  SidePool& sp = side_pool(st);
  // traced runs stay on one stream so per-kernel event times are not
  // inflated by queueing behind concurrent branches
  const bool fork = (tr == nullptr || (tr->mode & 1)) && !no_fork_env();
  cudaStream_t s_sync = fork ? sp.s[0] : st;
  dbg_delay("LEO_DBG_DELAY_REACH", st);
  const int kind = k.dialect == LEO_AMD ? LEO_EK_MEM_WAITCNT : k.dialect == LEO_NVIDIA ? LEO_EK_MEM_BARRIER : LEO_EK_MEM_SWSB;
  // the sync branch yields the SMs to the dataflow chain only when it runs a
  // shared-memory tier (then it is the shorter branch; the thread-private
  // Dijkstra path of big NVIDIA / Intel kernels is the long one)
  const int sdbg0 = caps ? caps->debug_flags : 0;
  const bool sync_smem_tier = !(sdbg0 & LEO_DBG_NO_SMEM) && B > 0 &&
      (k.dialect == LEO_AMD ? sync_smem_bytes(N, B, 128) <= (size_t)kSmemResidentMax
                            : setter_cta_smem(B) <= (size_t)kSmemResidentMax);
  // The sync branch forks off the dataflow chain.  With a shared-memory sync
  // tier (the shorter branch) it forks only once the chain's first kernels
  // are queued (after the unit-count scans), so its CTAs do not take the SMs the
  // chain's head needs; LEO_SYNC_FORK_AT=0/1/2 (start / after the unit
  // scans / after the block walk) overrides.
  const char* fa_env = getenv("LEO_SYNC_FORK_AT");
  const int fork_at = fa_env ? atoi(fa_env) : (sync_smem_tier ? 1 : 0);
  auto enqueue_sync = [&]() {
    if (fork) link_streams(st, s_sync, sp.e[0]);
    dbg_delay("LEO_DBG_DELAY_SYNC", s_sync);
    LowPriority low_prio(sync_smem_tier || getenv("LEO_FORCE_PRIO"));
    cudaStream_t st = s_sync;   // shadows the caller's stream for the TRACED scopes
    cudaMemsetAsync(pcnt, 0, (size_t)std::max(N, 1) * 4, st);
    cudaMemsetAsync(pcur, 0, (size_t)std::max(N, 1) * 4, st);
    cudaMemsetAsync(bev, 0, (size_t)std::max(B, 1) * 4, st);
    TRACED(KID_SYNC_PACK, leo_launch(k_sync_pack, grid_for(N, T), T, 0, st, k, wcword, setword, bev));
    if (k.dialect != LEO_AMD && B > 0)
      TRACED(KID_SYNC_PACK, leo_launch(k_block_setters, grid_for(B, T), T, 0, st, k, setword, n_ids, lastset, bev));
    TRACED(KID_SYNC_PACK, leo_launch(k_wait_list, grid_for(N, T), T, 0, st, k, own, wlist, &ctr[8]));
    SyncArgs sa{caps ? caps->debug_flags : 0, skeys, cap_sync, &ctr[3], slow2, &ctr[4], cap_slow, *diags, status,
                wcword, setword, lastset, n_ids, wlist, &ctr[8], wclist, &ctr[10], 0,
                kk->n_segments > 1 ? kk->seg_block : nullptr, kk->n_segments, sync_bcap};
    const int sdbg = caps ? caps->debug_flags : 0;
    const bool setter_staged = setter_cta_smem(B) <= (size_t)kSmemResidentMax && !getenv("LEO_SETTER_GLOBAL");
    const bool setter_cta = k.dialect != LEO_AMD && B > 0 && !(sdbg & (LEO_DBG_NO_SMEM | LEO_DBG_SYNC_SLOW));
    // staged: every block search goes to the warp tier; from L2 the warp tier
    // only takes what overflows the thread-private Dijkstra (measured on C5)
    sa.defer_search = setter_cta && (setter_staged || getenv("LEO_SETTER_DEFER")) ? 1 : 0;
    // as many threads per CTA as the image allows: more warps hide the
    // shared-memory latency of the event-list build and spread the items
    int wc_threads = 512;
    while (wc_threads > 128 && sync_smem_bytes(N, B, wc_threads) > (size_t)kSmemResidentMax) wc_threads >>= 1;
    const size_t wc_smem = sync_smem_bytes(N, B, wc_threads);
    const int dbg_flags = caps ? caps->debug_flags : 0;
    if (k.dialect == LEO_AMD && B > 0 && wc_smem <= (size_t)kSmemResidentMax && !(dbg_flags & LEO_DBG_NO_SMEM))
      {
      const char* ws = getenv("LEO_WC_STEPS");
      const int wc_steps = ws ? atoi(ws) : kWcSmemSteps;
      // half the SMs: the run time is the longest item's, and the other half
      // stays free for the reach tier running beside it
      const char* wcc = getenv("LEO_WC_CTAS");
      // CTAs in clusters of LEO_WC_CLUSTER (default 2): the image is staged once
      // per cluster by TMA multicast
      const char* wcl = getenv("LEO_WC_CLUSTER");
      const int csz = std::max(1, std::min(8, wcl ? atoi(wcl) : 2));
      const int wc_ctas = std::max(csz, ((wcc ? atoi(wcc) : std::max(1, SM / 2)) / csz) * csz);
      TRACED(KID_SYNC, leo_launch_cluster(k_sync_wc_smem, wc_ctas, csz, wc_threads, wc_smem, st, k, sa, bev, wc_steps));
    }
    else
      TRACED(KID_SYNC, leo_launch(k_sync<false>, grid_for(N, 64), 64, 0, st, k, sa, nullptr, 0));
    if (k.dialect == LEO_AMD)
      TRACED(KID_SYNC_WARP, leo_launch(k_sync_wc_warp, num_sms() * 2, 128, 4 * kWcSmemInts * 4, st, 
          k, sa, wclist, &ctr[10], cap_slow, slow2, &ctr[4]));
    if (k.dialect != LEO_AMD) {
      // setter searches: CTA per item in shared memory first; the rest (and
      // forced-slow items) on the global-scratch workers
      // warp per item; the CFG image staged in shared memory when it fits,
      // else read from L2 (big NVIDIA / Intel kernels)
      if (setter_cta && setter_staged)
        TRACED(KID_SYNC_SLOW, leo_launch(k_sync_setter_cta<true>, SM, kSWWarps * 32, setter_cta_smem(B), st, k, sa, bev,
                                         slow3s, &ctr[11]));
      else if (setter_cta)
        TRACED(KID_SYNC_SLOW, leo_launch(k_sync_setter_cta<false>, SM * 4, kSWWarps * 32, 16 + setter_warp_tables_smem(), st,
                                         k, sa, bev, slow3s, &ctr[11]));
      else
        TRACED(KID_SYNC_SLOW, leo_launch(k_sync_setter_smem, SM, 32, kDHBytes, st, k, sa, slow3s, &ctr[11]));
      SyncArgs sb = sa;
      sb.slow_list = slow3s; sb.slow_count = &ctr[11];
      TRACED(KID_SYNC_SLOW, leo_launch(k_sync<true>, (SW + 63) / 64, 64, 0, st, k, sb, sync_scr, SW));
    } else {
      // items that outgrew the warp tier: CTA per item over a global record arena first
      SyncArgs sb = sa;
      // on big kernels / batches only: on C2 the extra launch on the (near-critical) sync branch cost 8 us
      if (use_wc_cta) {
        TRACED(KID_SYNC_SLOW, leo_launch(k_sync_wc_cta, kWcCtaGrid, 1024, 0, st, k, sa, slow2, &ctr[4], cap_slow,
                                         wc_arena, slow3s, &ctr[11]));
        sb.slow_list = slow3s; sb.slow_count = &ctr[11];
      }
      TRACED(KID_SYNC_SLOW, leo_launch(k_sync<true>, (SW + 63) / 64, 64, 0, st, k, sb, sync_scr, SW));
    }
    TRACED(KID_KEY_HIST, leo_launch(k_key_hist, grid_for(cap_sync, T), T, 0, st, skeys, &ctr[3], cap_sync, pcnt));
    TRACED(KID_SCAN, scan_exclusive(pcnt, poff, nullptr, N, scan_tmp2, nullptr, st));
    TRACED(KID_KEY_SCATTER, leo_launch(k_key_scatter, grid_for(cap_sync, T), T, 0, st, skeys, &ctr[3], cap_sync, poff, pcur, ssorted));
    TRACED(KID_SEGSORT, leo_launch(segsort_unique_u64, grid_for(N, 128), 128, 0, st, ssorted, poff, pcnt, nullptr, N, puniq, cap_sync));
    TRACED(KID_SCAN, scan_exclusive(puniq, puoff, nullptr, N, scan_tmp2, &ctr[6], st));
  };
  const bool with_sync = rall == nullptr;     // reaching_definitions alone: no sync branch
  if (fork_at <= 0 && with_sync) enqueue_sync();
  // (a fused one-CTA count + scan is latency-bound on the operand loads: the
  // grid-wide count and two single-pass scans are faster)
  TRACED(KID_UNIT_COUNTS, leo_launch(k_unit_counts, std::max(grid_for(N, T), grid_for(B, T)), T, 0, st, k, ucnt, dcnt,
                                     B > 0 ? brec : nullptr, rhead));
  if (N <= kScanSingleMax) {        // both unit prefix sums in one launch (one CTA each)
    TRACED(KID_SCAN, leo_launch(scan_single_cta_pair, 2, 1024, 0, st, ucnt, use_ptr, dcnt, def_ptr, N));
  } else {
    TRACED(KID_SCAN, scan_exclusive(ucnt, use_ptr, nullptr, N, scan_tmp, nullptr, st));
    TRACED(KID_SCAN, scan_exclusive(dcnt, def_ptr, nullptr, N, scan_tmp, nullptr, st));
  }
  if (fork_at == 1 && with_sync) enqueue_sync();

  // tier 0 (shared-memory reach) reads the query columns, not the list
  const int n_seg0 = (kk->n_segments > 1 && kk->seg_block) ? kk->n_segments : 1;
  const int bcap0 = n_seg0 > 1 ? kk->max_seg_blocks : B;
  int ru_threads0 = 128;
  while (ru_threads0 > 32 && reach_unit_smem(bcap0, ru_threads0) > (size_t)kSmemResidentMax) ru_threads0 >>= 1;
  const int wdbg = caps ? caps->debug_flags : 0;
  const bool tier0 = B > 0 && U > 0 && reach_unit_smem(bcap0, ru_threads0) <= (size_t)kSmemResidentMax &&
                     !(wdbg & LEO_DBG_NO_SMEM) && !getenv("LEO_REACH_NO_T0");
  // (every use resolves, also under stalled-PC sharding: the indirect-
  // addressing test walks the base graph's RAW edges of non-owned consumers)
  WalkArgs wa{use_ptr, def_ptr, ev_res, q_block, q_unit, tier0 ? nullptr : q_list, &ctr[0], ldtab, qtab, Bp, gtab};
  const size_t smem = walk_bytes(wpc, smem_tab);
  if (B > 0 && U > 0) {     // the walk writes the unit columns sparsely
    cudaMemsetAsync(ldtab, 0xFF, (size_t)Bp * U * 4, st);
    cudaMemsetAsync(qtab, 0xFF, (size_t)Bp * U * 4, st);
  }
  if (B > 0) TRACED(KID_BLOCK_WALK, leo_launch(k_block_walk, std::max(1, walk_ctas), wpc * 32, smem, st, k, wa, wpc));
  // a caller's side branch (leo_analyze: stage-0 binning) forks here, after
  // the dataflow chain's head has been queued
  if (after_walk) {
    if (int e = after_walk()) return e;
  }
  if (rall && B > 0 && U > 0)
    leo_launch(k_reach_claim_all, grid_for((int64_t)B * U, 256), 256, 0, st, k, Bp, NU, qtab, q_block, q_unit,
               tier0 ? nullptr : q_list, &ctr[0]);
  if (fork_at >= 2 && with_sync) enqueue_sync();

  ReachArgs ra{caps ? caps->debug_flags : 0, ldtab, brec, U, Bp, q_block, q_unit, q_off, q_len, qres, cap_qres, &ctr[1],
               slow_list, &ctr[2], NQ + 1024, status};
  const int dbg = caps ? caps->debug_flags : 0;
  if (dbg & LEO_DBG_PHASES) {
    static const int zero = 0;
    cudaMemcpyToSymbolAsync(g_reach_item_ctr, &zero, sizeof(int), 0, cudaMemcpyHostToDevice, st);
  }
  // segments: members of a concatenated batch are staged one at a time
  const int n_seg = (kk->n_segments > 1 && kk->seg_block) ? kk->n_segments : 1;
  const int bcap = n_seg > 1 ? kk->max_seg_blocks : B;
  int ru_threads = getenv("LEO_RU_THREADS") ? std::max(32, atoi(getenv("LEO_RU_THREADS"))) : 128;
  while (ru_threads > 32 && reach_unit_smem(bcap, ru_threads) > (size_t)kSmemResidentMax) ru_threads >>= 1;
  const size_t ru_smem = reach_unit_smem(bcap, ru_threads);
  // CTAs per unit: one when the units alone cover the SMs (every extra CTA
  // re-stages the CFG and takes shared memory the sync branch also wants),
  // else enough to reach ~1.5 CTAs per SM (measured: C2 1 part 283 us vs 2
  // parts 289 us; C3 5 parts 381 us vs 7 parts 387 us).  LEO_RU_PARTS overrides.
  const char* rp_env = getenv("LEO_RU_PARTS");
  const int ru_parts = n_seg > 1 ? 1 : rp_env ? std::max(1, atoi(rp_env))
                       : U >= SM ? 1 : std::max(1, std::min(8, (3 * SM + 2 * U - 1) / (2 * std::max(U, 1))));
  const char* ps_env = getenv("LEO_RU_PERSEG");
  const int per_seg = n_seg > 1 ? (ps_env ? std::max(1, std::min(U, atoi(ps_env)))
                                          : std::max(1, std::min(U, (4 * SM + n_seg - 1) / n_seg)))
                                : std::min(U, SM * 8) * ru_parts;
  if (tier0) {
    // tier 0: the CFG and one unit's columns resident in shared memory, CTA per unit
    TRACED(KID_REACH_FAST, leo_launch(k_reach_unit, n_seg * per_seg, ru_threads, ru_smem, st, k, ra, qtab, rhead, ru_parts,
                                                 n_seg > 1 ? kk->seg_block : nullptr, per_seg, bcap));
  } else {
    // tier 1 is persistent: enough CTAs to fill the chip, queries fetched dynamically
    // geometry A/B knob LEO_T1 (profiling only): 0 i32/128, 1 u16/128, 2 u16/64, 3 i32/64
    const int t1 = getenv("LEO_T1") ? atoi(getenv("LEO_T1")) : 2;
    const bool narrow = B < 0xFFFF && t1 != 0 && t1 != 3;
    auto f = k_reach_fast<int32_t, 128, 96>;
    int slots = 128, kb = 4;
    if (narrow && t1 == 2) { f = k_reach_fast<uint16_t, 64, 48>; slots = 64; kb = 2; }
    else if (narrow) { f = k_reach_fast<uint16_t, 128, 96>; kb = 2; }
    else if (t1 == 3) { f = k_reach_fast<int32_t, 64, 48>; slots = 64; }
    const size_t t1_smem = (size_t)kT1Threads * slots * kb;
    const int per_sm = std::max(1, std::min(16, (int)((220 * 1024) / (t1_smem + 1024))));
    TRACED(KID_REACH_FAST, leo_launch(f, std::max(1, std::min<int>(grid_for(NU, kT1Threads), SM * per_sm)), kT1Threads,
                                          t1_smem, st, k, ra, q_list, &ctr[0], &ctr[9]));
  }
  {
    const int wpc_r = 4;
    const size_t sm_r = (size_t)wpc_r * kWarpSmemInts * 4;
    TRACED(KID_REACH_WARP, leo_launch(k_reach_warp, std::max(1, std::min<int>(SM * 4, (int)((NQ + 1024 + wpc_r - 1) / wpc_r))),
                                          wpc_r * 32, sm_r, st, k, ra, slow_list, &ctr[2], NQ + 1024, slow3, &ctr[7]));
  }
  TRACED(KID_REACH_SLOW, leo_launch(k_reach_slow, (RW + 63) / 64, 64, 0, st, k, ra, slow3, &ctr[7], reach_scr, RW));
  if (rall) {                     // export the reach-in set of every (block, unit) as a CSR
    const int64_t P = (int64_t)B * U;
    if (P > 0) {
      leo_launch(k_reach_export_count, grid_for(P, 256), 256, 0, st, k, Bp, qtab, q_len, rcnt);
      scan_exclusive(rcnt, rall->set_off, nullptr, P, rscan, nullptr, st);
      leo_launch(k_reach_export_fill, grid_for(P, 256), 256, 0, st, k, Bp, qtab, q_off, q_len, qres, *rall, status);
    } else {
      cudaMemsetAsync(rall->set_off, 0, sizeof(int32_t), st);
      cudaMemsetAsync(rall->count, 0, sizeof(int32_t), st);
    }
    ar.release();
    LEO_CUDA_CHECK(cudaGetLastError());
    return 0;
  }

  LinkArgs la{use_ptr, ev_res, q_off, q_len, qres, cand_cnt, cand_off, cand, cap_cand, *diags, status, own};
  TRACED(KID_LINK_COUNT, leo_launch(k_link<0>, grid_for(N, T), T, 0, st, k, la));
  TRACED(KID_SCAN, scan_exclusive(cand_cnt, cand_off, nullptr, N, scan_tmp, nullptr, st));
  TRACED(KID_LINK_FILL, leo_launch(k_link<1>, grid_for(N, T), T, 0, st, k, la));
  TRACED(KID_SEGSORT, leo_launch(segsort_unique_u64, grid_for(N, 128), 128, 0, st, cand, cand_off, cand_cnt, nullptr, N, uniq, cap_cand));
  TRACED(KID_SCAN, scan_exclusive(uniq, eoff, nullptr, N, scan_tmp, &ctr[5], st));
  TRACED(KID_LINK_EMIT, leo_launch(k_link_emit, grid_for(N, T), T, 0, st, k, cand_off, cand, uniq, eoff, *out, status));

  if (fork) link_streams(s_sync, st, sp.e[1]);   // join
  // (also writes the edge totals)
  TRACED(KID_SYNC_EMIT, leo_launch(k_sync_emit, grid_for(N, T), T, 0, st, N, kind, ssorted, poff, puniq, puoff, &ctr[5],
                                   &ctr[6], *out, status));
  if (caps && (caps->debug_flags & LEO_DBG_PHASES)) k_copy_counts<<<1, 32, 0, st>>>(ctr, 16);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// run_pruning
int prune_impl(const LeoKernel* kk, const LeoProfile* pp, const LeoConfig* cfg, const LeoEdges* in,
               LeoEdges* out, LeoPaths* paths, LeoDiags* diags, const LeoCaps* caps, uint32_t* status,
               cudaStream_t st, ZeroSet zero = ZeroSet{{nullptr, nullptr, nullptr, nullptr}, 0},
               const LeoPaths* in_paths = nullptr, const double* wpre_pre = nullptr) {
  LeoTrace* tr = caps ? caps->trace : nullptr;
  KView k = make_kview(kk);
  PView p = make_pview(pp);
  const int64_t cap_in = in->capacity;
  const int64_t cap_slow = std::max<int64_t>(caps ? caps->slow_items : 0, cap_in / 8 + 1024);
  const int PW = 32;
  const size_t pslow = prune_slow_bytes(cfg->max_depth, cfg->max_paths);
  Arena ar{st};
  int32_t *keep, *npaths, *pfirst, *pos, *slow_list, *ctr, *scan_tmp, *n_reg_in;
  double* dist;
  char* slow_scr;
  ar.want(&keep, cap_in); ar.want(&npaths, cap_in); ar.want(&pfirst, cap_in); ar.want(&dist, cap_in);
  ar.want(&pos, cap_in + 1); ar.want(&slow_list, cap_slow); ar.want(&ctr, 4);
  ar.want(&scan_tmp, scan_scratch_ints(cap_in) + 64); ar.want(&slow_scr, (int64_t)PW * pslow);
  (void)n_reg_in;
  // nvidia issue weights vary: straight runs are resolved through per-block prefix sums
  const bool weighted = kk->dialect == LEO_NVIDIA && (cfg->stage_mask & 4) && !getenv("LEO_PRUNE_NO_WPRE");
  double* wpre = nullptr;
  if (weighted && !wpre_pre) ar.want(&wpre, std::max(kk->n_instr, 1));
  LEO_CUDA_CHECK(ar.commit());
  if (weighted && wpre_pre) wpre = (double*)wpre_pre;      // computed on a side branch (leo_analyze)
  else if (weighted && kk->n_blocks > 0)
    leo_launch(k_weight_prefix, grid_for(kk->n_blocks, 128), 128, 0, st, k, wpre);
  cudaMemsetAsync(ctr, 0, 4 * sizeof(int32_t), st);
  LeoPaths inp{};
  if (in_paths && in_paths->first) {
    inp = *in_paths;
    leo_launch(k_copy_pool, grid_for(in_paths->capacity, 256), 256, 0, st, *in_paths, *paths, status);
  } else {
    cudaMemsetAsync(paths->count, 0, sizeof(int32_t), st);
  }
  PruneArgs a{caps ? caps->debug_flags : 0, *cfg, in->prod, in->cons, in->meta, in->count, (int32_t)cap_in, keep, npaths, pfirst, dist,
              *paths, wpre, inp, slow_list, &ctr[0], cap_slow, *diags, status};
  {
    const int dbg = caps ? caps->debug_flags : 0;
    const char* pt_env = getenv("LEO_PRUNE_THREADS");
    const char* pc_env = getenv("LEO_PRUNE_CTAS");
    // 256 threads per CTA when the image and the per-thread DFS state fit
    // (one edge per thread per round at C2 size: prune 45 -> 37 us)
    const int pthreads = pt_env ? atoi(pt_env)
                         : prune_smem_bytes(k.N, k.B, 256, true) <= (size_t)kSmemResidentMax ? 256 : 128;
    const size_t staged = prune_smem_bytes(k.N, k.B, pthreads, true), unstaged = prune_smem_bytes(k.N, k.B, 128, false);
    // staged CFG image when it fits; otherwise the many-CTA global-memory
    // kernel (thread per edge, no per-round CTA barriers) balances better
    (void)unstaged;
    if (!(dbg & LEO_DBG_NO_SMEM) && staged <= (size_t)kSmemResidentMax)
      TRACED(KID_PRUNE, leo_launch(k_prune_edges_smem<true>, pc_env ? atoi(pc_env) : num_sms(), pthreads, staged, st, k, p, a));
    else
      TRACED(KID_PRUNE, leo_launch(k_prune_edges, grid_for(cap_in, 128, num_sms() * 16), 128, 0, st, k, p, a));
  }
  TRACED(KID_PRUNE_SLOW, leo_launch(k_prune_slow, 1, PW, 0, st, k, p, a, slow_scr, PW));
  TRACED(KID_SCAN, scan_exclusive(keep, pos, in->count, cap_in, scan_tmp, nullptr, st));
  TRACED(KID_COMPACT, leo_launch(k_compact, grid_for(std::max<int64_t>(cap_in, zero.n), 256), 256, 0, st, a, pos,
                                 in->n_regular, *out, status, zero));
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// incoming CSR of an edge list (regular part consumer-sorted, sync part not)
struct IncomingBufs {
  int32_t *rbeg, *rend, *scnt, *soff, *scur, *tmp, *uniq;
  uint64_t* sidx;
};
void want_incoming(Arena& ar, IncomingBufs& b, int N, int64_t cap) {
  ar.want(&b.rbeg, N); ar.want(&b.rend, N); ar.want(&b.scnt, N); ar.want(&b.soff, N + 1);
  ar.want(&b.scur, N); ar.want(&b.sidx, cap); ar.want(&b.tmp, scan_scratch_ints(std::max(N, 1)) + 64);
  ar.want(&b.uniq, N);
}
Incoming build_incoming(IncomingBufs& b, int N, const LeoEdges* e, bool with_sync, LeoTrace* tr, cudaStream_t st,
                        bool prezeroed = false) {
  if (!prezeroed) {                // (else the producing kernel cleared rbeg / rend / scnt / scur)
    const size_t nb = (size_t)std::max(N, 1) * 4;
    cudaMemsetAsync(b.rbeg, 0, nb, st);
    cudaMemsetAsync(b.rend, 0, nb, st);
    cudaMemsetAsync(b.scnt, 0, nb, st);
    cudaMemsetAsync(b.scur, 0, nb, st);
  }
  TRACED(KID_SEG_BOUNDS, leo_launch(k_seg_bounds, grid_for(e->capacity, 256), 256, 0, st, e->cons, e->n_regular, b.rbeg, b.rend));
  if (with_sync) {
    TRACED(KID_SYNC_HIST, leo_launch(k_sync_hist, grid_for(e->capacity, 256), 256, 0, st, e->cons, e->n_regular, e->count, b.scnt));
    TRACED(KID_SCAN, scan_exclusive(b.scnt, b.soff, nullptr, N, b.tmp, nullptr, st));
    TRACED(KID_SYNC_FILL, leo_launch(k_sync_fill, grid_for(e->capacity, 256), 256, 0, st, e->cons, e->n_regular, e->count, b.soff, b.scur, b.sidx));
    TRACED(KID_SEGSORT, leo_launch(segsort_unique_u64, grid_for(N, 128), 128, 0, st, b.sidx, b.soff, b.scnt, nullptr, N, b.uniq, e->capacity));
  } else {
    cudaMemsetAsync(b.soff, 0, (size_t)(N + 1) * 4, st);
  }
  return Incoming{b.rbeg, b.rend, b.soff, b.sidx};
}

int slice_impl(const LeoKernel* kk, const LeoProfile* pp, const LeoEdges* pruned, const Incoming& inc,
               uint32_t* bitmap, int32_t* level, LeoTrace* tr, cudaStream_t st) {
  const int N = kk->n_instr;
  Arena ar{st};
  int32_t *fa, *fb, *counts;
  ar.want(&fa, N); ar.want(&fb, N); ar.want(&counts, 4);
  LEO_CUDA_CHECK(ar.commit());
  SliceArgs a{pp->lat, pruned->prod, inc, level, fa, fb, counts, bitmap};
  int dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_slice, 256, 0);
  int grid = std::max(1, std::min(per_sm, 4)) * num_sms();
  int n = N;
  void* args[] = {&n, &a};
  cudaError_t le;
  TRACED(KID_SLICE, le = cudaLaunchCooperativeKernel((void*)k_slice, grid, 256, args, 0, st));
  LEO_CUDA_CHECK(le);
  ar.release();
  return 0;
}

// _address_traces_to_load for all instructions (k_mp_round x7 + k_mp_final)
// over the base graph's RAW incoming edges; the CSR is kept for blame.
struct AddrBufs {
  IncomingBufs bb;
  uint2 *la, *lb;
  int32_t* ep;
  uint8_t* ok;
  int32_t* flags;       // [3] k_mp_coop round flags
};
void want_addr(Arena& ar, AddrBufs& b, int N, int64_t edge_cap) {
  want_incoming(ar, b.bb, N, 1);
  ar.want(&b.la, N); ar.want(&b.lb, N); ar.want(&b.ok, N); ar.want(&b.ep, std::max<int64_t>(edge_cap, 1));
  ar.want(&b.flags, 4);
}
// The labels pack a 24-bit instruction id (kMpT): kernels of >= 2^24
// instructions take the exact per-candidate BFS tiers instead (mp_ok = null).
inline bool mp_labels_fit(int n_instr) { return n_instr < (int)kMpT; }
Incoming addr_impl(const KView& k, const LeoEdges* base, AddrBufs& b, LeoTrace* tr, cudaStream_t st) {
  Incoming binc = build_incoming(b.bb, k.N, base, false, tr, st);   // RAW edges only
  if (!mp_labels_fit(k.N)) return binc;
  const int g = grid_for(k.N, 128);
  TRACED(KID_SELF_ADDR, leo_launch(k_mp_edges, grid_for(base->capacity, 256, num_sms() * 8), 256, 0, st, k,
                                   base->n_regular, (int64_t)base->capacity, base->prod, base->meta, b.ep));
  if (getenv("LEO_MP_COOP")) {
    // one cooperative kernel, in-place rounds until nothing changes.  Opt-in:
    // its grid holds every SM for the whole search and starves the pruning
    // branch it runs beside (C5 +245 us, measured A/B)
    static int coop_grid[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!coop_grid[dev & 63]) {
      int per = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_mp_coop, 256, 0);
      coop_grid[dev & 63] = std::max(1, per) * num_sms();
    }
    const int grid = std::max(1, std::min(coop_grid[dev & 63], grid_for(k.N, 256, 1 << 30)));
    KView kv = k;
    int32_t* flags = b.flags;
    void* args[] = {&kv, (void*)&binc.rbeg, (void*)&binc.rend, &b.ep, &b.la, &flags, &b.ok};
    TRACED(KID_SELF_ADDR, cudaLaunchCooperativeKernel((void*)k_mp_coop, grid, 256, args, 0, st));
    return binc;
  }
  TRACED(KID_SELF_ADDR, leo_launch(k_mp_round, g, 128, 0, st, k, binc.rbeg, binc.rend, b.ep, b.la, b.la, 1));
  for (int r = 1; r < 7; r++) {
    const uint2* in = (r & 1) ? b.la : b.lb;
    uint2* out = (r & 1) ? b.lb : b.la;
    TRACED(KID_SELF_ADDR, leo_launch(k_mp_round, g, 128, 0, st, k, binc.rbeg, binc.rend, b.ep, in, out, 0));
  }
  // round r writes lb when r is odd, la when even: round 6 (the last) wrote la
  TRACED(KID_SELF_ADDR, leo_launch(k_mp_final, g, 128, 0, st, k, binc.rbeg, binc.rend, b.ep, b.la, b.ok));
  return binc;
}

// Caller edge lists whose LeoEdges.n_regular is NULL are in arbitrary order
// (the reference's DependencyGraph holds any edge tuple): the incoming CSR then
// takes every edge through the stable counting sort (list order per consumer).
LeoEdges any_order(const LeoEdges& e, int32_t* zero_scalar) {
  LeoEdges v = e;
  if (!v.n_regular) v.n_regular = zero_scalar;
  return v;
}

// consumer-sorted (stable) copy of an arbitrary-order edge list: the base
// graph's RAW CSR of the indirect-addressing test needs consumer runs
struct CanonBufs {
  IncomingBufs ib;
  int32_t *prod, *cons, *count, *nreg;
  uint32_t* meta;
};
void want_canon(Arena& ar, CanonBufs& b, int N, int64_t cap) {
  want_incoming(ar, b.ib, N, cap);
  ar.want(&b.prod, cap); ar.want(&b.cons, cap); ar.want(&b.meta, cap); ar.want(&b.count, 1); ar.want(&b.nreg, 1);
}
LeoEdges canon_by_consumer(CanonBufs& b, int N, const LeoEdges& in, int32_t* zero_scalar, cudaStream_t st) {
  const LeoEdges v = any_order(in, zero_scalar);
  Incoming t = build_incoming(b.ib, N, &v, true, nullptr, st);
  LeoEdges out{in.capacity, b.prod, b.cons, b.meta, b.count, b.nreg};
  leo_launch(k_gather_edges, grid_for(in.capacity, 256), 256, 0, st, in.count, t.sidx, in.prod, in.cons, in.meta, out);
  return out;
}

int blame_impl(const LeoKernel* kk, const LeoProfile* pp, const LeoEdges* pruned, const LeoPaths* paths,
               const LeoEdges* base, const Incoming& inc, const int32_t* line_id, int32_t n_lines,
               LeoBlame* out, double* line_blame, double* line_stall, const LeoCaps* caps,
               uint32_t* status, cudaStream_t st, Range own = Range{0, 0},
               const Incoming* binc_pre = nullptr, const uint8_t* mp_ok_pre = nullptr) {
  LeoTrace* tr = caps ? caps->trace : nullptr;
  KView k = make_kview(kk);
  const int N = k.N;
  PView p = make_pview(pp);
  const int64_t cap_slow = pick(caps ? caps->slow_items : 0, N / 4 + 1024);
  const int BW = 64;
  Arena ar{st};
  AddrBufs ab;
  int32_t *ecount, *self_sub, *eoff, *slow_list, *slow2, *ctr, *scan_tmp, *slow_scr;
  double *jtotal, *jnsum;
  const int dbg = caps ? caps->debug_flags : 0;
  const bool own_addr = binc_pre == nullptr;
  if (own_addr) want_addr(ar, ab, N, base->capacity);
  ar.want(&ecount, N); ar.want(&self_sub, N); ar.want(&eoff, N + 1); ar.want(&slow_list, cap_slow);
  ar.want(&slow2, cap_slow);
  ar.want(&ctr, 4); ar.want(&scan_tmp, scan_scratch_ints(std::max(N, 1)) + 64);
  ar.want(&slow_scr, (int64_t)BW * 2 * (N + 1)); ar.want(&jtotal, N); ar.want(&jnsum, N);
  // staged edge entries (pass 0): at most one per pruned edge
  const bool two_pass = getenv("LEO_BLAME_2PASS") != nullptr;   // A/B: recompute in pass 1
  const int64_t stg_cap = two_pass ? 1 : std::max<int64_t>(pruned->capacity, 1);
  int32_t *stg_off, *stg_edge, *stg_cause, *elist;
  double *stg_blame, *stg_fac;
  ar.want(&elist, N);
  ar.want(&stg_off, N); ar.want(&stg_edge, stg_cap); ar.want(&stg_cause, stg_cap);
  ar.want(&stg_blame, stg_cap); ar.want(&stg_fac, 4 * stg_cap);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(ctr, 0, 16, st);
  // the slow self-blame worker's stamps matter only when it runs (no
  // precomputed addressing verdict: LEO_DBG_SELF_SLOW)
  if (dbg & LEO_DBG_SELF_SLOW) cudaMemsetAsync(slow_scr, 0, (size_t)BW * 2 * (N + 1) * sizeof(int32_t), st);
  // the indirect-addressing test comes precomputed from a side branch
  // (leo_analyze) or is computed here; LEO_DBG_SELF_SLOW keeps the per-
  // candidate BFS tiers instead (cross-checked against the same goldens)
  Incoming binc = own_addr ? addr_impl(k, base, ab, tr, st) : *binc_pre;
  const uint8_t* mp_ok = (dbg & LEO_DBG_SELF_SLOW) || !mp_labels_fit(N) ? nullptr : (own_addr ? ab.ok : mp_ok_pre);
  BlameArgs a{dbg, mp_ok, own, p, pruned->prod, pruned->meta, paths->dist, inc, binc.rbeg, binc.rend,
              base ? base->prod : nullptr, base ? base->meta : nullptr,
              ecount, self_sub, jtotal, jnsum, eoff, *out, slow_list, &ctr[0], cap_slow, status, nullptr, nullptr, 0,
              stg_off, &ctr[2], two_pass ? 0 : stg_cap, stg_edge, stg_cause, stg_blame, stg_fac};
  const bool lines_on = line_id && line_blame && line_stall && n_lines > 0;
  if (lines_on && !(caps && (caps->options & LEO_OPT_ACCUMULATE_LINES))) {
    a.zero_lb = line_blame; a.zero_ls = line_stall; a.n_lines = n_lines;
  }
  // split pass 0 on big kernels only (C5 -35 us, C3 -4; on C2 the extra launch on the chain costs +11 us)
  if (two_pass || getenv("LEO_BLAME_UNSPLIT") || (N < (1 << 15) && !getenv("LEO_BLAME_SPLIT"))) {
    TRACED(KID_BLAME_COUNT, leo_launch(k_blame<0>, grid_for(N, 128), 128, 0, st, k, a));
  } else {
    // light pass (self verdicts, list the instructions with edges), then Eq. 1 on the list
    TRACED(KID_BLAME_COUNT, leo_launch(k_blame_light, grid_for(N, 256), 256, 0, st, k, a, elist, &ctr[3]));
    TRACED(KID_BLAME_COUNT, leo_launch(k_blame_edges, grid_for(std::max<int64_t>(pruned->capacity, 1), 128), 128, 0, st,
                                       k, a, elist, &ctr[3]));
  }
  if (!mp_ok) {
    TRACED(KID_SELFBLAME_WARP, leo_launch(k_selfblame_warp, num_sms(), 128, 4 * kSBWarpInts * 4, st, k, a, slow2, &ctr[1]));
    TRACED(KID_SELFBLAME_SLOW, leo_launch(k_selfblame_slow, 1, BW, 0, st, k, a, slow2, &ctr[1], slow_scr, BW));
  }
  TRACED(KID_SCAN, scan_exclusive(ecount, eoff, nullptr, N, scan_tmp, nullptr, st));
  if (two_pass) {
    TRACED(KID_BLAME_FILL, leo_launch(k_blame<1>, grid_for(N, 128), 128, 0, st, k, a));
    // (k_blame<1> also wrote the entry count)
    if (lines_on) {
      TRACED(KID_LINES, leo_launch(k_lines, grid_for(std::max<int64_t>(out->capacity, N), 256), 256, 0, st, k, p, own, pruned->prod, *out,
                                                                                 line_id, line_blame, line_stall));
    }
  } else {
    // staged entries into stalled order + the line rollup, one pass
    TRACED(KID_BLAME_FILL, leo_launch(k_blame_compact, grid_for(N, 256), 256, 0, st, k, a,
                                      lines_on ? line_id : nullptr, lines_on ? line_blame : nullptr,
                                      lines_on ? line_stall : nullptr));
  }
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

}  // namespace


extern "C" {

int leo_abi_version(void) { return LEO_ABI_VERSION; }

// `status`: the caller's status word (LEO_ST_BAD_INPUT: a sample pc outside [0, n_instr))
static int bin_impl(const LeoSamples* s, int32_t n_instr, int32_t* lat, int32_t* cls_cnt, uint32_t* status,
                    LeoTrace* tr, cudaStream_t st) {
  set_smem_attributes();
  cudaMemsetAsync(cls_cnt, 0, (size_t)std::max(n_instr, 1) * 32, st);
  const int64_t S = s->n_samples;
  const bool packed = s->packed != nullptr;
  // bytes per packed word: 4 (pc << 8 | category) or 3 (pc << 4 | category)
  const int pw = s->packed_bytes == 3 ? 3 : 4;
  // 3-byte words: category bits (4 default, 5 for up to 32 category ids)
  const int cb = s->packed_cat_bits == 0 ? 4 : s->packed_cat_bits;
  if (packed && s->packed_bytes != 0 && s->packed_bytes != 3 && s->packed_bytes != 4) return -3;
  if (packed && pw == 3 && cb != 4 && cb != 5) return -3;
  if (packed && (int64_t)n_instr > (pw == 3 ? (1 << (24 - cb)) : (1 << 24))) return -3;   // pc must fit the word
  if (packed && pw == 3 && ((uintptr_t)s->packed & 3)) return -3;                  // read as u32 triples
  if (S > 0 && packed && s->packed_host)
    LEO_CUDA_CHECK(cudaMemcpyAsync((void*)s->packed, s->packed_host, (size_t)S * pw, cudaMemcpyHostToDevice, st));
  if (S > 0 && !packed && s->pc_host)
    LEO_CUDA_CHECK(cudaMemcpyAsync((void*)s->pc, s->pc_host, (size_t)S * 4, cudaMemcpyHostToDevice, st));
  if (S > 0 && !packed && s->cat_host)
    LEO_CUDA_CHECK(cudaMemcpyAsync((void*)s->cat, s->cat_host, (size_t)S, cudaMemcpyHostToDevice, st));
  // big streams: one pass, per-CTA shared-memory hash (LEO_BIN_BUCKETED=1: the bucketed passes)
  if (S >= (4ll << 20) && (int64_t)n_instr * 8 < 0xFFFFFFFFll && !getenv("LEO_BIN_BUCKETED")) {
    // table geometry (A/B knobs LEO_BIN_SLOTS / LEO_BIN_PROBE; profiling only)
    const int slots = getenv("LEO_BIN_SLOTS") ? atoi(getenv("LEO_BIN_SLOTS")) : 16384;
    const int probe = getenv("LEO_BIN_PROBE") ? atoi(getenv("LEO_BIN_PROBE")) : 2;
    auto f = k_bin_hash<26624, 4>;
    int threads = 1024, per_sm = 1;
    if (slots == 8192) { f = probe == 8 ? k_bin_hash<8192, 8> : k_bin_hash<8192, 4>; threads = 512; per_sm = 3; }
    else if (slots == 16384) f = probe == 2 ? k_bin_hash<16384, 2> : k_bin_hash<16384, 4>;
    else f = probe == 2 ? k_bin_hash<26624, 2> : probe == 8 ? k_bin_hash<26624, 8> : k_bin_hash<26624, 4>;
    if (packed && pw == 3) {
      static int ng = -1;
      if (ng < 0) {                                      // profiling knob: set once, before any capture
        ng = getenv("LEO_BIN_NOGROUP") ? 1 : 0;
        if (ng) cudaMemcpyToSymbol(g_bin_nogroup, &ng, sizeof(int));
      }
    }
    if (packed) {                                        // default geometry
      f = pw == 4 ? k_bin_hash<16384, 2, 4> : cb == 5 ? k_bin_hash<16384, 2, 3, 5> : k_bin_hash<16384, 2, 3>;
      threads = 1024; per_sm = 1;
    }
    const int G = getenv("LEO_BIN_CTAS") ? std::max(1, atoi(getenv("LEO_BIN_CTAS"))) : num_sms() * per_sm;
    TRACED(KID_BIN, leo_launch(f, G, threads, (size_t)(packed ? 16384 : slots) * 8, st, S, s->pc, s->cat,
                               s->cat_to_cs, n_instr, cls_cnt, status, s->packed));
    TRACED(KID_BIN_FINALIZE, leo_launch(k_bin_finalize, grid_for(n_instr, 256), 256, 0, st, n_instr, cls_cnt, lat));
    LEO_CUDA_CHECK(cudaGetLastError());
    return 0;
  }
  const int R = (n_instr + kBinR - 1) / kBinR <= kBinMaxBuckets ? kBinR : kBinRMax;
  const int nb = std::max(1, (n_instr + R - 1) / R);
  const bool bucketed = nb <= kBinMaxBuckets && S > 0 && !packed;
  // chunks: enough CTAs to stream the samples, bounded so the [G x nb] matrix stays small
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 4, (S + 8191) / 8192));
  Arena ar{st};
  int32_t *M, *btot, *boff, *soff;
  uint16_t* keys;
  ar.want(&M, bucketed ? (int64_t)G * nb : 1);
  ar.want(&btot, nb + 1); ar.want(&boff, nb + 1); ar.want(&soff, nb + 1);
  ar.want(&keys, bucketed ? S + 8 : 1);
  LEO_CUDA_CHECK(ar.commit());
  if (bucketed) {
    const int smem = R * 8 * 4;
    const int slice = (int)std::min<int64_t>(65536, std::max<int64_t>(4096, S / (num_sms() * 3)));
    TRACED(KID_BIN_HIST, leo_launch(k_bin_hist, G, 512, nb * 4, st, S, s->pc, n_instr, nb, R, M, status));
    TRACED(KID_BIN_PLAN, leo_launch(k_bin_colscan, std::min(nb, num_sms() * 4), 256, 0, st, nb, G, M, btot));
    TRACED(KID_BIN_PLAN, leo_launch(k_bin_plan, 1, 1024, 0, st, nb, slice, btot, boff, soff));
    TRACED(KID_BIN_SCATTER, leo_launch(k_bin_scatter, G, 512, (size_t)nb * 12 + (size_t)kBinSub * 4, st, S, s->pc, s->cat,
                                       s->cat_to_cs, n_instr, nb, R, M, boff, keys));
    TRACED(KID_BIN, leo_launch(k_bin_count, num_sms() * 3, 512, smem, st, n_instr, nb, R, slice, boff, soff, keys, cls_cnt));
  } else if (S > 0) {
    TRACED(KID_BIN, leo_launch(!packed ? k_bin_samples<0> : pw == 4 ? k_bin_samples<4> : cb == 5 ? k_bin_samples<3, 5> : k_bin_samples<3>, grid_for(S / 4 + 1, 256, num_sms() * 8),
                               256, 0, st, S, s->pc, s->cat, s->cat_to_cs, n_instr, cls_cnt, status, s->packed));
  }
  TRACED(KID_BIN_FINALIZE, leo_launch(k_bin_finalize, grid_for(n_instr, 256), 256, 0, st, n_instr, cls_cnt, lat));
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_bin_samples(const LeoSamples* s, int32_t n_instr, int32_t* lat, int32_t* cls_cnt, uint32_t* status,
                    void* stream) {
  if (!s || n_instr < 0 || !status) return -1;
  return bin_impl(s, n_instr, lat, cls_cnt, status, nullptr, (cudaStream_t)stream);
}

int leo_events_create(int32_t n, void** events) {
  for (int i = 0; i < n; i++) {
    cudaEvent_t e;
    LEO_CUDA_CHECK(cudaEventCreate(&e));
    events[i] = (void*)e;
  }
  return 0;
}
int leo_events_elapsed(int32_t n, void* const* begin, void* const* end, float* ms) {
  for (int i = 0; i < n; i++) LEO_CUDA_CHECK(cudaEventElapsedTime(&ms[i], (cudaEvent_t)begin[i], (cudaEvent_t)end[i]));
  return 0;
}
int leo_events_destroy(int32_t n, void** events) {
  for (int i = 0; i < n; i++) cudaEventDestroy((cudaEvent_t)events[i]);
  return 0;
}

int leo_debug_tiers(int32_t* out) {
  LEO_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_tier_counts, 16 * sizeof(int)));
  return 0;
}

int leo_debug_items(int64_t* out, int32_t n) {
  if (n < 0 || n > 16384) return -1;
  LEO_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_item_cycles, (size_t)n * sizeof(long long)));
  return 0;
}

int leo_debug_phases(int32_t slot, int64_t* out, int32_t n_ctas) {
  if (slot < 0 || slot >= 4 || n_ctas < 0 || n_ctas > 1024) return -1;
  LEO_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_phase_ts, (size_t)n_ctas * 8 * sizeof(long long),
                                      (size_t)slot * 1024 * 8 * sizeof(long long)));
  return 0;
}

const char* leo_kernel_name(int id) { return (id >= 0 && id < KID_COUNT_) ? kKernelNames[id] : nullptr; }

int leo_build_graph(const LeoKernel* k, const LeoCaps* caps, LeoEdges* out, LeoDiags* diags,
                    uint32_t* status, void* stream) {
  WsScope ws_scope(caps);
  if (int e = check_kernel(k)) return e;
  return build_graph_impl(k, caps, out, diags, status, (cudaStream_t)stream);
}

int leo_prune(const LeoKernel* k, const LeoProfile* p, const LeoConfig* cfg, const LeoEdges* in,
              const LeoPaths* in_paths, LeoEdges* out, LeoPaths* paths, LeoDiags* diags, uint32_t* status,
              void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!cfg || cfg->max_paths < 0 || cfg->max_depth < 0 || !in || !out || !paths || !diags || !status) return -3;
  return prune_impl(k, p, cfg, in, out, paths, diags, nullptr, status, (cudaStream_t)stream,
                    ZeroSet{{nullptr, nullptr, nullptr, nullptr}, 0}, in_paths);
}

int leo_slice(const LeoKernel* k, const LeoProfile* p, const LeoEdges* pruned, uint32_t* bitmap,
              int32_t* level, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!pruned || !bitmap || !level) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar{st};
  IncomingBufs ib;
  int32_t* zero;
  ar.want(&zero, 4);
  want_incoming(ar, ib, k->n_instr, pruned->capacity);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(zero, 0, 16, st);
  const LeoEdges pv = any_order(*pruned, zero);
  Incoming inc = build_incoming(ib, k->n_instr, &pv, true, nullptr, st);
  int r = slice_impl(k, p, &pv, inc, bitmap, level, nullptr, st);
  ar.release();
  return r;
}

int leo_blame(const LeoKernel* k, const LeoProfile* p, const LeoEdges* pruned, const LeoPaths* paths,
              const LeoEdges* base, const int32_t* line_id, int32_t n_lines, LeoBlame* out,
              double* line_blame, double* line_stall, uint32_t* status, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!pruned || !out || !status) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = k->n_instr;
  Arena ar{st};
  IncomingBufs ib;
  int32_t *zero, *zn = nullptr;
  double* dist;
  uint8_t* no_mp = nullptr;
  CanonBufs cb;
  ar.want(&zero, 4);
  want_incoming(ar, ib, N, pruned->capacity);
  ar.want(&dist, pruned->capacity);
  if (base && !base->n_regular) want_canon(ar, cb, N, base->capacity);
  if (!base) { ar.want(&no_mp, N); ar.want(&zn, N + 1); }
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(zero, 0, 16, st);
  const LeoEdges pv = any_order(*pruned, zero);
  Incoming inc = build_incoming(ib, N, &pv, true, nullptr, st);
  // _edge_distance of the given edges and their valid_paths (analysis.py:371-376)
  LeoPaths dp = paths ? *paths : LeoPaths{};
  leo_launch(k_edge_dist, grid_for(pruned->capacity, 256), 256, 0, st, pruned->count, pruned->capacity, pruned->prod,
             pruned->cons, dp, dist);
  dp.dist = dist;
  int r;
  if (base) {
    LeoEdges bv = *base;
    if (!base->n_regular) bv = canon_by_consumer(cb, N, *base, zero, st);
    r = blame_impl(k, p, &pv, &dp, &bv, inc, line_id, n_lines, out, line_blame, line_stall, nullptr, status, st);
  } else {
    // no base graph: self-blame never upgrades to indirect addressing (analysis.py:422-426)
    cudaMemsetAsync(no_mp, 0, (size_t)std::max(N, 1), st);
    cudaMemsetAsync(zn, 0, (size_t)(N + 1) * 4, st);
    const Incoming none{zn, zn, zn, nullptr};
    r = blame_impl(k, p, &pv, &dp, nullptr, inc, line_id, n_lines, out, line_blame, line_stall, nullptr, status, st,
                   Range{0, 0}, &none, no_mp);
  }
  ar.release();
  return r;
}

int leo_self_blame(const LeoKernel* k, const LeoProfile* p, const LeoEdges* base, int32_t n,
                   const int32_t* index, uint8_t* sub, double* cycles, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (n < 0 || (n > 0 && (!index || !sub || !cycles))) return -3;
  if (base && !mp_labels_fit(k->n_instr)) return -5;      // (the label search needs N < 2^24)
  cudaStream_t st = (cudaStream_t)stream;
  const int N = k->n_instr;
  Arena ar{st};
  int32_t* zero;
  AddrBufs ab;
  CanonBufs cb;
  ar.want(&zero, 4);
  if (base) want_addr(ar, ab, N, base->capacity);
  if (base && !base->n_regular) want_canon(ar, cb, N, base->capacity);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(zero, 0, 16, st);
  const KView kv = make_kview(k);
  const uint8_t* mp_ok = nullptr;
  if (base) {
    LeoEdges bv = *base;
    if (!base->n_regular) bv = canon_by_consumer(cb, N, *base, zero, st);
    addr_impl(kv, &bv, ab, nullptr, st);
    mp_ok = ab.ok;
  }
  if (n > 0) leo_launch(k_self_entries, grid_for(n, 128), 128, 0, st, kv, make_pview(p), mp_ok, n, index, sub, cycles);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_coverage(const LeoKernel* k, const LeoEdges* edges, int32_t* out, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!edges || !out) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = k->n_instr;
  Arena ar{st};
  int32_t *mask, *cnt;
  ar.want(&mask, N); ar.want(&cnt, N);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(out, 0, 2 * sizeof(int32_t), st);
  cudaMemsetAsync(mask, 0, (size_t)std::max(N, 1) * 4, st);
  cudaMemsetAsync(cnt, 0, (size_t)std::max(N, 1) * 4, st);
  leo_launch(k_cov_edges, grid_for(edges->capacity, 256), 256, 0, st, edges->cons, edges->meta, edges->count,
             edges->capacity, mask, cnt);
  leo_launch(k_cov_nodes, grid_for(N, 256, num_sms() * 4), 256, 0, st, N, mask, cnt, out);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_rank_hotspots(const LeoKernel* k, const LeoProfile* p, int32_t top_n, int32_t include_unsampled,
                      int32_t* hot, int32_t* n_hot, void* stream) {
  if (int e = check_kernel(k)) return e;
  if (top_n < 0 || top_n > 4096 || !n_hot || (top_n > 0 && !hot)) return -3;
  leo_launch(k_report_rank, 1, 1024, 0, (cudaStream_t)stream, k->n_instr, p->lat, top_n, include_unsampled, hot, n_hot);
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_trace_chain(const LeoKernel* k, int32_t n_entries, const int32_t* stalled, const int32_t* cause,
                    const double* blame, int32_t start, int32_t max_depth, int32_t* chain_node,
                    int32_t* chain_entry, int32_t* chain_len, int32_t* chain_self, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  const int N = k->n_instr;
  if (n_entries < 0 || start < 0 || start >= N || max_depth < 1 || !chain_node || !chain_entry || !chain_len ||
      !chain_self)
    return -3;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar{st};
  int32_t *cnt, *off, *cur, *uniq, *tmp, *sst, *sedge, *sprod, *one, *ent, *self, *dummy, *ncount;
  uint64_t* perm;
  double* sbl;
  const int64_t M = std::max(n_entries, 1);
  ar.want(&cnt, N); ar.want(&off, N + 1); ar.want(&cur, N); ar.want(&uniq, N);
  ar.want(&tmp, scan_scratch_ints(std::max(N, 1)) + 64); ar.want(&perm, M);
  ar.want(&sst, M); ar.want(&sedge, M); ar.want(&sprod, M); ar.want(&sbl, M);
  ar.want(&one, 4); ar.want(&ent, max_depth); ar.want(&self, 1); ar.want(&dummy, 4); ar.want(&ncount, 1);
  LEO_CUDA_CHECK(ar.commit());
  // entries grouped by stalled instruction, list order kept inside a group
  cudaMemsetAsync(cnt, 0, (size_t)std::max(N, 1) * 4, st);
  cudaMemsetAsync(cur, 0, (size_t)std::max(N, 1) * 4, st);
  leo_launch(k_chain_prep, 1, 32, 0, st, start, n_entries, one, ncount, dummy);
  leo_launch(k_sync_hist, grid_for(M, 256), 256, 0, st, stalled, dummy, ncount, cnt);
  scan_exclusive(cnt, off, nullptr, N, tmp, nullptr, st);
  leo_launch(k_sync_fill, grid_for(M, 256), 256, 0, st, stalled, dummy, ncount, off, cur, perm);
  leo_launch(segsort_unique_u64, grid_for(N, 128), 128, 0, st, perm, off, cnt, nullptr, N, uniq, M);
  leo_launch(k_chain_gather, grid_for(M, 256), 256, 0, st, n_entries, perm, stalled, cause, blame, sst, sedge, sprod, sbl);
  ReportArgs ra{one, one + 1, sst, sedge, sbl, ncount, (int32_t)M, sprod, 0, max_depth, dummy + 1, dummy + 2,
                chain_len, chain_node, ent, self, (uint32_t*)(dummy + 3)};
  leo_launch(k_report_hot, 1, 32, 0, st, ra);
  leo_launch(k_chain_unperm, 1, 32, 0, st, perm, chain_len, ent, self, chain_entry, chain_self);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_liveness_filter(const LeoKernel* k, const LeoEdges* links, uint8_t* keep, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!links || !keep) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const KView kv = make_kview(k);
  const int W = std::max(1, (k->n_units + 31) / 32);
  Arena ar{st};
  uint32_t *gen, *kill, *lin, *lout;
  const int64_t BW = (int64_t)std::max(k->n_blocks, 1) * W;
  ar.want(&gen, BW); ar.want(&kill, BW); ar.want(&lin, BW); ar.want(&lout, BW);
  LEO_CUDA_CHECK(ar.commit());
  if (k->n_blocks > 0) {
    leo_launch(k_live_genkill, grid_for(k->n_blocks, 128), 128, 0, st, kv, W, gen, kill);
    leo_launch(k_live_solve, (W + 31) / 32, 32, 0, st, kv, W, gen, kill, lin, lout);
  }
  leo_launch(k_live_filter, grid_for(links->capacity, 256), 256, 0, st, kv, W, lout, links->count, links->capacity,
             links->prod, links->cons, links->meta, keep);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_line_rollup(const LeoKernel* k, const LeoProfile* p, int32_t n_entries, const int32_t* stalled,
                    const int32_t* cause, const double* blame, const int32_t* line_id, int32_t n_lines,
                    double* line_blame, double* line_stall, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (n_entries < 0 || !line_id || n_lines <= 0 || !line_blame || !line_stall) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar{st};
  int32_t *edge, *cnt;
  ar.want(&edge, std::max(n_entries, 1)); ar.want(&cnt, 1);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(line_blame, 0, (size_t)n_lines * 8, st);
  cudaMemsetAsync(line_stall, 0, (size_t)n_lines * 8, st);
  leo_launch(k_entry_edges, grid_for(std::max(n_entries, 1), 256), 256, 0, st, n_entries, cause, edge, cnt);
  LeoBlame bv{std::max(n_entries, 1), (int32_t*)stalled, edge, nullptr, (double*)blame, nullptr, cnt};
  leo_launch(k_lines, grid_for(std::max<int64_t>(n_entries, k->n_instr), 256), 256, 0, st, make_kview(k), make_pview(p),
             Range{0, 0}, cause, bv, line_id, line_blame, line_stall);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_line_compact(const double* line_blame, const double* line_stall, int32_t n_lines, int32_t capacity,
                     int32_t* line_ids, double* blame_out, double* stall_out, int32_t* count, void* stream) {
  if (n_lines < 0 || capacity < 0 || !line_blame || !line_stall || !line_ids || !blame_out || !stall_out || !count)
    return -3;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar{st};
  int32_t *flag, *off, *scr;
  ar.want(&flag, std::max(n_lines, 1)); ar.want(&off, (int64_t)n_lines + 1);
  ar.want(&scr, scan_scratch_ints(std::max(n_lines, 1)) + 64);
  LEO_CUDA_CHECK(ar.commit());
  leo_launch(k_line_flag, grid_for(std::max(n_lines, 1), 256), 256, 0, st, n_lines, line_blame, line_stall, flag);
  scan_exclusive(flag, off, nullptr, n_lines, scr, nullptr, st);
  leo_launch(k_line_scatter, grid_for(std::max(n_lines, 1), 256), 256, 0, st, n_lines, line_blame, line_stall,
             off, capacity, line_ids, blame_out, stall_out, count);
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_reaching_definitions(const LeoKernel* k, const LeoCaps* caps, LeoReachIn* out, uint32_t* status,
                             void* stream) {
  WsScope ws_scope(caps);
  if (int e = check_kernel(k)) return e;
  if (!out || !out->set_off || !out->count || !status) return -3;
  return build_graph_impl(k, caps, nullptr, nullptr, status, (cudaStream_t)stream, Range{0, 0}, {}, out);
}

int leo_report(const LeoKernel* k, const LeoProfile* p, const LeoEdges* base, const LeoEdges* pruned,
               const LeoBlame* blame, LeoReport* r, uint32_t* status, void* stream) {
  WsScope ws_scope(nullptr);
  if (int e = check_kernel(k)) return e;
  if (!r || r->top_n < 0 || r->top_n > 4096 || r->chain_depth < 0 || r->max_causes < 0) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  const int N = k->n_instr;
  Arena ar{st};
  int32_t *mask, *cnt;
  ar.want(&mask, N); ar.want(&cnt, N);
  LEO_CUDA_CHECK(ar.commit());
  cudaMemsetAsync(r->coverage, 0, 4 * sizeof(int32_t), st);
  const int T = 256;
  // before: base graph minus sync edges (the raw/guard prefix, report.py:135-137)
  cudaMemsetAsync(mask, 0, (size_t)std::max(N, 1) * 4, st);
  cudaMemsetAsync(cnt, 0, (size_t)std::max(N, 1) * 4, st);
  leo_launch(k_cov_edges, grid_for(base->capacity, T), T, 0, st, base->cons, base->meta, base->n_regular, base->capacity, mask, cnt);
  leo_launch(k_cov_nodes, grid_for(N, T, num_sms() * 4), T, 0, st, N, mask, cnt, r->coverage);
  // after: every pruned edge
  cudaMemsetAsync(mask, 0, (size_t)std::max(N, 1) * 4, st);
  cudaMemsetAsync(cnt, 0, (size_t)std::max(N, 1) * 4, st);
  leo_launch(k_cov_edges, grid_for(pruned->capacity, T), T, 0, st, pruned->cons, pruned->meta, pruned->count, pruned->capacity, mask, cnt);
  leo_launch(k_cov_nodes, grid_for(N, T, num_sms() * 4), T, 0, st, N, mask, cnt, r->coverage + 2);
  leo_launch(k_report_rank, 1, 1024, 0, st, N, p->lat, r->top_n, r->include_unsampled, r->hot, r->n_hot);
  if (r->top_n > 0) {
    ReportArgs a{r->n_hot, r->hot, blame->stalled, blame->edge, blame->blame, blame->count, blame->capacity,
                 pruned->prod, r->max_causes, r->chain_depth, r->n_causes, r->causes, r->chain_len,
                 r->chain_node, r->chain_entry, r->chain_self, status};
    leo_launch(k_report_hot, r->top_n, 32, 0, st, a);
  }
  ar.release();
  LEO_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leo_analyze(const LeoKernel* k, const LeoProfile* p, const LeoSamples* samples, const LeoConfig* cfg,
                const LeoCaps* caps, LeoEdges* base, LeoEdges* pruned, LeoPaths* paths, LeoDiags* diags,
                LeoBlame* blame, uint32_t* slice_bitmap, int32_t* slice_level, const int32_t* line_id,
                int32_t n_lines, double* line_blame, double* line_stall, uint32_t* status, void* stream) {
  WsScope ws_scope(caps);
  if (int e = check_kernel(k)) return e;
  if (!cfg) return -3;
  cudaStream_t st = (cudaStream_t)stream;
  SidePool& sp = side_pool(st);
  // Launch priorities only where measured to help: kernels whose vendor sync
  // tracing runs a shared-memory tier (the dataflow chain is then the critical
  // branch).  Big NVIDIA / Intel kernels run everything at the default.
  const int adbg = caps ? caps->debug_flags : 0;
  const bool prio = getenv("LEO_FORCE_PRIO") ? true : !(adbg & LEO_DBG_NO_SMEM) && k->n_blocks > 0 &&
      (k->dialect == LEO_AMD ? sync_smem_bytes(k->n_instr, k->n_blocks, 128) <= (size_t)kSmemResidentMax
                             : setter_cta_smem(k->n_blocks) <= (size_t)kSmemResidentMax);
  HighPriority high_prio(prio);
  LeoTrace* tr = caps ? caps->trace : nullptr;
  // stage-0 binning only feeds pruning and blame: run it beside build_graph
  const bool fork = (tr == nullptr || (tr->mode & 1)) && !no_fork_env();
  // nvidia pruning's per-block issue-weight prefix (kernel data only): built
  // on the binning branch when there is one
  double* wpre_pre = nullptr;
  Arena ar_w{st};
  struct Release { Arena& a; ~Release() { a.release(); } } release_w{ar_w};   // after the last use is queued
  if (samples && k->dialect == LEO_NVIDIA && (cfg->stage_mask & 4) && !getenv("LEO_PRUNE_NO_WPRE")) {
    ar_w.want(&wpre_pre, std::max(k->n_instr, 1));
    LEO_CUDA_CHECK(ar_w.commit());
  }
  auto enqueue_bin = [&]() -> int {
    if (!samples) return 0;
    cudaStream_t s_bin = fork ? sp.s[1] : st;
    if (fork) link_streams(st, s_bin, sp.e[2]);
    dbg_delay("LEO_DBG_DELAY_BIN", s_bin);
    // small streams bin at the least priority; a big stream (C5) is itself a
    // long branch and keeps the default
    const int bin_lo = getenv("LEO_BIN_LOWPRIO") ? atoi(getenv("LEO_BIN_LOWPRIO")) : -1;
    LowPriority low_prio(bin_lo >= 0 ? bin_lo == 1 : samples->n_samples <= (16ll << 20));
    const int rb = bin_impl(samples, k->n_instr, (int32_t*)p->lat, (int32_t*)p->cls_cnt, status, tr, s_bin);
    // the nvidia issue-weight prefix pruning needs, off the dataflow chain
    if (!rb && wpre_pre && k->n_blocks > 0)
      leo_launch(k_weight_prefix, grid_for(k->n_blocks, 128), 128, 0, s_bin, make_kview(k), wpre_pre);
    return rb;
  };
  // Up to 16 M samples the binning branch forks after the block walk: it has
  // the whole build as slack, and started with the build it takes SMs from
  // the dataflow chain's head.  Bigger streams (C5: 100 M, ~1 ms of binning)
  // need the whole build to hide in.
  // (a stream still in host memory forks at once: its transfer needs the
  // whole build to hide in)
  // (the one-pass hashed binning of big streams is short enough to fork late too;
  // LEO_BIN_EARLY=1 forks it at the start)
  const bool late_bin = samples && !samples->pc_host && !samples->packed_host && !getenv("LEO_BIN_EARLY") &&
                        (samples->n_samples <= (16ll << 20) || !getenv("LEO_BIN_BUCKETED"));
  if (!late_bin) {
    if (int e = enqueue_bin()) return e;
  }
  const Range own{cfg->consumer_lo, cfg->consumer_hi};
  int r = build_graph_impl(k, caps, base, diags, status, st, own,
                           late_bin ? std::function<int()>(enqueue_bin) : std::function<int()>());
  if (r) return r;
  // LEO_DBG_STOP=s (profiling only): end the pipeline after stage s
  // (1 build, 2 prune, 3 incoming CSR, 4 slice) to time prefixes in a graph
  const char* stop_env = getenv("LEO_DBG_STOP");
  const int stop = stop_env ? atoi(stop_env) : 0;
  if (stop == 1 || stop == 6) {                 // 6: build + pruning, no addressing branch
    if (samples && fork) link_streams(sp.s[1], st, sp.e[3]);
    if (stop == 6) r = prune_impl(k, p, cfg, base, pruned, paths, diags, caps, status, st);
    return r;
  }
  // side branch: base-graph RAW CSR + the indirect-addressing test for all
  // instructions, overlapping pruning; joined before blame
  Arena ar_addr{st};
  AddrBufs ab;
  want_addr(ar_addr, ab, k->n_instr, base->capacity);
  LEO_CUDA_CHECK(ar_addr.commit());
  cudaStream_t s_addr = fork ? sp.s[3] : st;
  if (fork) link_streams(st, s_addr, sp.e[6]);
  Incoming binc;
  {
    LowPriority low_prio;
    binc = addr_impl(make_kview(k), base, ab, tr, s_addr);
  }
  if (stop == 5) {                              // build + the addressing branch
    if (fork) link_streams(s_addr, st, sp.e[7]);
    if (samples && fork) link_streams(sp.s[1], st, sp.e[3]);
    ar_addr.release();
    return 0;
  }
  if (samples && fork) link_streams(sp.s[1], st, sp.e[3]);
  // the pruned graph's incoming-CSR buffers exist before pruning so its
  // compaction kernel can clear them
  Arena ar{st};
  IncomingBufs ib;
  want_incoming(ar, ib, k->n_instr, pruned->capacity);
  LEO_CUDA_CHECK(ar.commit());
  r = prune_impl(k, p, cfg, base, pruned, paths, diags, caps, status, st,
                 ZeroSet{{ib.rbeg, ib.rend, ib.scnt, ib.scur}, k->n_instr}, nullptr, wpre_pre);
  if (r) { ar.release(); return r; }
  if (stop == 2) {
    if (fork) link_streams(s_addr, st, sp.e[7]);
    ar.release();
    ar_addr.release();
    return 0;
  }
  Incoming inc = build_incoming(ib, k->n_instr, pruned, true, tr, st, true);
  if (stop == 3) {
    if (fork) link_streams(s_addr, st, sp.e[7]);
    ar.release();
    ar_addr.release();
    return 0;
  }
  // the slice and blame attribution both read the pruned incoming CSR: run
  // them as parallel branches
  const bool do_slice = slice_level && slice_bitmap;
  if (do_slice) {
    if (fork) link_streams(st, sp.s[2], sp.e[4]);
    r = slice_impl(k, p, pruned, inc, slice_bitmap, slice_level, tr, fork ? sp.s[2] : st);
    if (r) { ar.release(); return r; }
  }
  if (fork) link_streams(s_addr, st, sp.e[7]);
  if (stop == 4) {
    if (do_slice && fork) link_streams(sp.s[2], st, sp.e[5]);
    ar.release();
    ar_addr.release();
    return 0;
  }
  r = blame_impl(k, p, pruned, paths, base, inc, line_id, n_lines, blame, line_blame, line_stall, caps, status, st, own,
                 &binc, ab.ok);
  if (do_slice && fork) link_streams(sp.s[2], st, sp.e[5]);
  ar.release();
  ar_addr.release();
  return r;
}

}  // extern "C"
