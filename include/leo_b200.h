/*
 * leo_b200.h — C ABI of the B200-native LEO analysis hot path.
 *
 * Drop-in boundary for the `stalltrace` analyzer (reference: arXiv 2604.20032
 * reproduction, /root/reference/pkg/src/stalltrace).  The reference has no FFI;
 * its contract is the Python API re-exported in `stalltrace/__init__.py:9-64`.
 * Each entry point below replaces one of those Python functions; the host mirror
 * in `paper_2604_20032_b200/api.py` keeps the reference names and types and
 * marshals them into the structure-of-arrays (SoA) layout declared here.
 *
 *   leo_bin_samples   <- new stage 0 (reference reads pre-binned counts,
 *                        profile.py:186-239; breakdown_at profile.py:307-313)
 *   leo_build_graph   <- depgraph.build_graph            depgraph.py:507-528
 *                        (reaching_definitions :135-177, per_use_link :188-223,
 *                         liveness_filter :274-293, trace_waitcnt :402-416,
 *                         trace_barriers :446-463, trace_swsb :466-482)
 *   leo_prune         <- analysis.run_pruning            analysis.py:302-314
 *                        (prune_opcode :143, prune_barrier :165,
 *                         prune_latency :256, prune_execution :289)
 *   leo_blame         <- analysis.attribute_blame        analysis.py:431-484
 *                        (self_blame :414-428) + per-source-line rollup
 *   leo_slice         <- multi-source backward slice over DependencyGraph.incoming
 *                        (depgraph.py:102-108; semantics frozen in DESIGN.md)
 *   leo_analyze       <- fused build -> prune -> slice -> blame -> lines
 *                        (report.py:132-142 call sequence)
 *   leo_reaching_definitions <- depgraph.reaching_definitions  depgraph.py:135-177
 *   leo_liveness_filter      <- depgraph.liveness_filter       depgraph.py:274-293
 *   leo_self_blame           <- analysis.self_blame            analysis.py:414-428
 *   leo_coverage             <- analysis.single_dep_coverage   analysis.py:547-561
 *   leo_trace_chain          <- analysis.trace_chain           analysis.py:499-538
 *   leo_rank_hotspots        <- report.rank_hotspots           report.py:96-109
 *   leo_line_rollup          <- per-source-line rollup of any blame list
 *   leo_line_compact         <- the touched lines of a rollup as a sparse list (read-back)
 *   leo_report               <- report.build_report assembly   report.py:132-199
 *
 * Conventions
 *  - Every pointer inside a struct is a DEVICE pointer owned by the caller.
 *  - Calls are stream-ordered and asynchronous; `stream` is a cudaStream_t
 *    passed as void*.  Scratch memory is taken from the stream-ordered
 *    allocator (or LeoCaps.workspace) and released on the same stream.  No
 *    global analysis state: per-device caches (SM count, the >48 KiB shared-
 *    memory function attributes) are set once per device, fork/join side
 *    streams are kept per (host thread, device, caller stream), and the only
 *    device globals are profiling counters written under LEO_DBG_PHASES.
 *  - Variable-size outputs use "capacity + device counter": the kernel writes
 *    the true count to the device counter even when it exceeds capacity; the
 *    host reads the counter after synchronising, and re-runs with larger
 *    buffers when count > capacity (status LEO_ERR_CAPACITY in the status word).
 *  - Return value: 0 = launched; < 0 = argument error detected on the host
 *    (mapped to InputError by the Python layer, errors.py:12-39).
 *  - Non-fatal findings are typed diagnostic records (LeoDiag) which the host
 *    renders with the reference's exact format strings.
 */
#ifndef LEO_B200_H
#define LEO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LEO_ABI_VERSION 4

/* ---- enumerations (indices follow the reference enum definition order) --- */
/* Dialect  isa.py:19-22 */
enum { LEO_NVIDIA = 0, LEO_AMD = 1, LEO_INTEL = 2 };
/* RegClass isa.py:32-39 */
enum { LEO_RC_VECTOR = 0, LEO_RC_SCALAR = 1, LEO_RC_PREDICATE = 2, LEO_RC_BARRIER = 3,
       LEO_RC_UNIFORM = 4, LEO_RC_SBID = 5, LEO_RC_SPECIAL = 6, LEO_N_RC = 7 };
/* OpcodeClass isa.py:42-58 */
enum { LEO_OC_GLOBAL_LOAD = 0, LEO_OC_GLOBAL_STORE, LEO_OC_LOCAL_LOAD, LEO_OC_LOCAL_STORE,
       LEO_OC_SCALAR_LOAD, LEO_OC_CONSTANT_LOAD, LEO_OC_ATOMIC, LEO_OC_FP_ARITH,
       LEO_OC_INT_ARITH, LEO_OC_CONVERSION, LEO_OC_CONTROL_FLOW, LEO_OC_SYNC_WAIT,
       LEO_OC_BARRIER_ALL, LEO_OC_SEND, LEO_OC_NOP, LEO_OC_OTHER, LEO_N_OC };
/* CommonStall profile.py:29-43 (order = dominant-class tie-break) */
enum { LEO_CS_MEMORY_DEP = 0, LEO_CS_EXECUTION_DEP, LEO_CS_SYNCHRONIZATION,
       LEO_CS_INSTRUCTION_FETCH, LEO_CS_PIPELINE_BUSY, LEO_CS_NOT_SELECTED,
       LEO_CS_IDLE, LEO_CS_OTHER, LEO_N_CS };
/* EdgeKind depgraph.py:46-51 */
enum { LEO_EK_RAW = 0, LEO_EK_GUARD = 1, LEO_EK_MEM_WAITCNT = 2, LEO_EK_MEM_BARRIER = 3,
       LEO_EK_MEM_SWSB = 4 };
/* DepClass depgraph.py:57-60 */
enum { LEO_DC_MEMORY = 0, LEO_DC_EXECUTION = 1, LEO_DC_SYNCHRONIZATION = 2 };
/* SelfBlame analysis.py:320-326 */
enum { LEO_SB_MEMORY_LATENCY = 0, LEO_SB_COMPUTE_SATURATION, LEO_SB_SYNCHRONIZATION_OVERHEAD,
       LEO_SB_PIPELINE_CONTENTION, LEO_SB_INSTRUCTION_FETCH, LEO_SB_INDIRECT_ADDRESSING };
/* per-instruction sync variant (isa.py:153-206) */
enum { LEO_SYNC_NONE = 0, LEO_SYNC_WAITCNT = 1, LEO_SYNC_BARRIER = 2, LEO_SYNC_SWSB = 3 };
#define LEO_NONE_U32 0xFFFFFFFFu

/* ---- operand record: one RegisterRef (isa.py:92-117) with its role ------- */
/* bits 0-15 index, 16-23 span, 24-26 RegClass, 27-28 role                  */
enum { LEO_ROLE_SRC = 0, LEO_ROLE_GUARD = 1, LEO_ROLE_DST = 2 };
#define LEO_OPND(role, cls, index, span) \
  ((uint32_t)(index) | ((uint32_t)(span) << 16) | ((uint32_t)(cls) << 24) | ((uint32_t)(role) << 27))

/* ---- edge meta word --------------------------------------------------------
 * bits 0-26 register ref (index|span<<16|class<<24; zero for sync edges),
 * 27-29 EdgeKind, 30-31 DepClass                                            */
#define LEO_META(kind, dc, ref27) ((uint32_t)(ref27) | ((uint32_t)(kind) << 27) | ((uint32_t)(dc) << 30))

/* ---- one kernel: instruction stream + CFG (disasm.py:477-499) ------------ */
typedef struct LeoKernel {
  int32_t n_instr;            /* N */
  int32_t n_blocks;           /* B */
  int32_t n_units;            /* U: dense register-unit ids (depgraph.py:41) */
  int32_t dialect;            /* LEO_NVIDIA / LEO_AMD / LEO_INTEL */
  int32_t n_opnd;             /* operand records */
  int32_t n_use_units;        /* sum of spans over src + guard operands (host-computed) */
  int32_t n_def_units;        /* sum of spans over dest operands (host-computed) */
  int32_t unit_base[8];       /* RegClass -> first unit id */
  const uint8_t*  opclass;    /* [N] OpcodeClass */
  const int32_t*  block_of;   /* [N] */
  const int32_t*  opnd_ptr;   /* [N+1] CSR; per instruction: srcs, guard, dests */
  const uint32_t* opnd;       /* [n_opnd] LEO_OPND records */
  const uint8_t*  sync_kind;  /* [N] LEO_SYNC_* */
  const uint32_t* sync_a;     /* [N] waitcnt: vmcnt | barrier: w|r<<8|wait<<16 | swsb: set token */
  const uint32_t* sync_b;     /* [N] waitcnt: lgkmcnt | barrier: stall cycles | swsb: wait mask */
  const int32_t*  blk_first;  /* [B] */
  const int32_t*  blk_last;   /* [B] */
  const int32_t*  succ_ptr;   /* [B+1] successor order [target, fallthrough] disasm.py:572 */
  const int32_t*  succ;
  const int32_t*  pred_ptr;   /* [B+1] predecessors sorted disasm.py:596 */
  const int32_t*  pred;
  /* optional: the kernel is a concatenation of independent kernels (a batch,
   * no CFG edge between members); seg_block[n_segments+1] are the members'
   * first blocks (device), max_seg_blocks the largest member.  0 / NULL: one
   * segment.  Shared-memory tiers then stage one member at a time. */
  int32_t n_segments;
  int32_t max_seg_blocks;
  const int32_t*  seg_block;
} LeoKernel;

/* ---- per-instruction profile (profile.py:114-170, 284-329) --------------- */
typedef struct LeoProfile {
  int64_t period;             /* sampling_period_cycles */
  const int32_t* lat;         /* [N] latency_samples */
  const int32_t* cls_cnt;     /* [N*8] latency samples per CommonStall */
  const int64_t* exec_cnt;    /* [N] exec_count, -1 = None */
  const int32_t* total;       /* [N] total_samples, -1 = None (effective total = lat) */
  const double*  eff;         /* [N] efficiency */
  const uint8_t* sampled;     /* [N] a profile record attached (profile.py:296) */
} LeoProfile;

/* ---- raw PC-sample stream (new stage 0) ---------------------------------- */
typedef struct LeoSamples {
  int64_t n_samples;          /* S */
  const int32_t* pc;          /* [S] instruction index */
  const uint8_t* cat;         /* [S] vendor stall category id */
  const uint8_t* cat_to_cs;   /* [256] vendor category id -> CommonStall (map_stall) */
  /* optional host sources (pinned memory): when set, pc / cat are device
   * buffers the library fills with an asynchronous copy on the binning branch,
   * so the transfer of the sample stream overlaps graph construction */
  const int32_t* pc_host;
  const uint8_t* cat_host;
  /* ABI v3, optional packed stream (kernels below 2^24 instructions): one u32
   * word per sample, pc << 8 | category (4 bytes instead of 5).  When set,
   * pc / cat are ignored; packed_host (pinned) is copied into packed on the
   * binning branch as pc_host / cat_host are. */
  const uint32_t* packed;
  const uint32_t* packed_host;
  /* ABI v4: bytes per packed word.  0 or 4: the u32 words above.  3: one
   * little-endian 24-bit word per sample, pc << 4 | category (kernels of at
   * most 2^20 instructions, category ids below 16; 3 bytes per sample over
   * PCIe instead of 4); packed / packed_host then hold 3 * n_samples bytes,
   * `packed` 4-byte aligned. */
  int32_t packed_bytes;
  /* ABI v4, 3-byte words only: category bits, 0 / 4 (pc << 4 | category) or 5
   * (pc << 5 | category: up to 32 category ids, Intel's 17; kernels of at
   * most 2^19 instructions) */
  int32_t packed_cat_bits;
} LeoSamples;

/* ---- analysis configuration (analysis.py:115-124) ------------------------ */
typedef struct LeoConfig {
  uint32_t stage_mask;        /* bit s-1 set when stage s is enabled */
  int32_t  prune_exec;
  int32_t  max_paths;         /* DEFAULT_MAX_PATHS 64 */
  int32_t  max_depth;         /* DEFAULT_MAX_DEPTH 512 */
  double   threshold[16];     /* LatencyTable.get per OpcodeClass (fallback = max) */
  int32_t  consumer_lo;       /* stalled-PC sharding: this call owns consumers          */
  int32_t  consumer_hi;       /*   [lo, hi); hi <= 0 means all (single-GPU / replica)   */
} LeoConfig;

/* ---- edge list (DepEdge depgraph.py:77-91) --------------------------------
 * Library-made lists are canonical: raw/guard edges sorted by consumer first
 * (n_regular of them), then sync edges.  A caller's list may be in ANY order
 * (the reference's DependencyGraph holds any edge tuple: chained stages,
 * hand-built graphs): pass n_regular = NULL; the library then keeps list order
 * per consumer wherever the reference's `incoming` order matters.           */
typedef struct LeoEdges {
  int32_t   capacity;
  int32_t*  prod;             /* [cap] */
  int32_t*  cons;             /* [cap] */
  uint32_t* meta;             /* [cap] LEO_META */
  int32_t*  count;            /* device scalar: total edges */
  int32_t*  n_regular;        /* device scalar: raw/guard edges (they precede sync edges),
                                 or NULL: arbitrary order (inputs); not written (outputs) */
} LeoEdges;

/* ---- valid_paths of pruned edges (PathRecord depgraph.py:71-74) ---------- */
typedef struct LeoPaths {
  int32_t  capacity;          /* path-record capacity */
  int32_t* first;             /* [edge cap] first record of edge, -1 = none */
  int32_t* npaths;            /* [edge cap] */
  double*  dist;              /* [edge cap] _edge_distance analysis.py:371-376 */
  int32_t* len;               /* [cap] length_instructions */
  double*  accum;             /* [cap] accumulated_issue_cycles */
  int32_t* count;             /* device scalar */
} LeoPaths;

/* ---- diagnostics ----------------------------------------------------------- */
enum {
  LEO_DIAG_UNRESOLVED = 1,    /* depgraph.py:219-222  a0 = operand record            */
  LEO_DIAG_WAITCNT = 2,       /* depgraph.py:395-399  a0 = counter(0 vm,1 lgkm), a1 = level, a2 = best_m */
  LEO_DIAG_NO_SETTER = 3,     /* depgraph.py:461-462 / 480-481  a0 = barrier or token */
  LEO_DIAG_PATH_CAPPED = 4    /* analysis.py:277-284  instr = producer, a0 = consumer, a1 = 1 kept-with-partial / 0 conservative */
};
typedef struct LeoDiag { int32_t code, instr, a0, a1, a2, seq; } LeoDiag;
typedef struct LeoDiags {
  int32_t  capacity;
  LeoDiag* rec;               /* [cap] unordered; host sorts by (code group, instr, seq) */
  int32_t* count;             /* device scalar */
} LeoDiags;

/* ---- blame entries (BlameEntry analysis.py:360-368) ---------------------- */
typedef struct LeoBlame {
  int32_t  capacity;
  int32_t* stalled;           /* [cap] */
  int32_t* edge;              /* [cap] index into pruned edges, -1 = self-blame */
  uint8_t* sub;               /* [cap] SelfBlame for self entries, 255 otherwise */
  double*  blame;             /* [cap] blame_cycles */
  double*  factors;           /* [cap*4] dist, eff, isu, match */
  int32_t* count;             /* device scalar */
  /* optional (NULL: not written): the entry's cause instruction (-1 for
   * self) and its edge's meta word (kind, dep class, register ref), so a
   * service reads back self-contained entries without the pruned graph */
  int32_t*  cause;            /* [cap] */
  uint32_t* meta;             /* [cap] */
} LeoBlame;

/* ---- optional device-time trace ------------------------------------------
 * When LeoCaps.trace is non-NULL the library records the caller's CUDA events
 * (cudaEvent_t passed as void*) on the launching stream around every kernel
 * (or only around kernel id `only_kernel` when >= 0): slot x brackets kernel
 * kernel_id[x]; `count` advances past `capacity` when slots run out.       */
typedef struct LeoTrace {
  int32_t capacity;
  int32_t count;
  int32_t only_kernel;        /* -1: all kernels */
  int32_t mode;               /* 0: stages serialised on the caller's stream (per-kernel
                                 times not inflated by concurrent branches);
                                 1: keep the fork/join branches (timeline) */
  void**  ev_begin;           /* [capacity] cudaEvent_t */
  void**  ev_end;             /* [capacity] cudaEvent_t */
  int32_t* kernel_id;         /* [capacity] host array */
} LeoTrace;

/* ---- capacity hints for internal scratch (0 = default heuristic) --------- */
typedef struct LeoCaps {
  int64_t query_results;      /* reaching-definition results pool        (default 4 x use units) */
  int64_t candidates;         /* per-use link candidates                  (default 6 x use units) */
  int64_t sync_keys;          /* raw sync edges before dedup              (default 2 x N + 1024) */
  int64_t slow_items;         /* work items re-run on the global-scratch path (default N/4 + 1024) */
  LeoTrace* trace;            /* optional, host struct (NULL = no tracing) */
  int32_t debug_flags;        /* testing: route every item to a larger tier (LEO_DBG_*) */
  int32_t options;            /* LEO_OPT_* */
  void*    workspace;         /* optional caller-owned device scratch (bump-allocated per call) */
  int64_t  workspace_bytes;
  int64_t* workspace_needed;  /* optional HOST out: bytes this call wanted; when it exceeds
                                 workspace_bytes the library used the stream-ordered allocator */
} LeoCaps;
/* LEO_OPT_ACCUMULATE_LINES: add into line_blame / line_stall instead of
 * zeroing them first (many kernels of one batch share one per-line vector) */
enum { LEO_OPT_ACCUMULATE_LINES = 1 };
/* LEO_DBG_NO_SMEM: skip the shared-memory-resident tiers (global-memory tiers only) */
enum { LEO_DBG_REACH_T2 = 1, LEO_DBG_REACH_T3 = 2, LEO_DBG_SYNC_SLOW = 4, LEO_DBG_PRUNE_SLOW = 8,
       LEO_DBG_SELF_SLOW = 16, LEO_DBG_NO_SMEM = 32, LEO_DBG_PHASES = 64 };
/* LEO_DBG_PHASES: the shared-memory tiers record per-CTA clock64 phase
 * marks, read back with leo_debug_phases (profiling aid) */

/* ---- status word (device) ------------------------------------------------ */
enum { LEO_ST_EDGE_OVERFLOW = 1, LEO_ST_PATH_OVERFLOW = 2, LEO_ST_DIAG_OVERFLOW = 4,
       LEO_ST_BLAME_OVERFLOW = 8, LEO_ST_SCRATCH_OVERFLOW = 16, LEO_ST_BAD_INPUT = 32 };

/* ---- entry points ---------------------------------------------------------- */
int leo_abi_version(void);
/* name of traced kernel id (LeoTrace.kernel_id), NULL past the last id */
const char* leo_kernel_name(int id);
/* per-CTA phase marks of kernel slot `slot` (0 reach, 1 waitcnt, 2 prune):
 * out[cta * 8 + phase] = clock64 delta from the CTA's start (LEO_DBG_PHASES) */
int leo_debug_phases(int32_t slot, int64_t* out, int32_t n_ctas);
/* build_graph work counters of the last LEO_DBG_PHASES call: [0] queries,
 * [2] reach tier-2 items, [7] tier-3 items, [3] sync keys, [4] exact-walker
 * items, [8] waits, [10] waitcnt warp-tier items */
int leo_debug_tiers(int32_t* out);
/* per-item clock64 cycles of the shared-memory waitcnt tier (LEO_DBG_PHASES) */
int leo_debug_items(int64_t* out, int32_t n);

/* stage 0: raw (pc, category) stream -> lat[N], cls_cnt[N*8] (zeroed here).
 * A sample whose pc is outside [0, n_instr) is dropped and sets
 * LEO_ST_BAD_INPUT in *status (device word, caller-zeroed). */
int leo_bin_samples(const LeoSamples* s, int32_t n_instr, int32_t* lat, int32_t* cls_cnt,
                    uint32_t* status, void* stream);

/* build_graph: raw/guard edges sorted (consumer, producer, kind, class, index, span)
 * followed by the dialect's sync edges sorted (producer, consumer). */
int leo_build_graph(const LeoKernel* k, const LeoCaps* caps, LeoEdges* out, LeoDiags* diags,
                    uint32_t* status, void* stream);

/* run_pruning: stages 1->2->3->4 honouring cfg; `out` keeps input order.
 * Any single stage (prune_opcode / prune_barrier / prune_latency /
 * prune_execution, analysis.py:143-299) is the same call with one bit of
 * cfg->stage_mask.  `in_paths` (may be NULL): the input edges' valid_paths
 * (first / npaths per input edge, len / accum pool, count); a kept edge keeps
 * them unless stage 3 finds valid paths for it (analysis.py:276); the input
 * records are copied to the front of `paths`. */
int leo_prune(const LeoKernel* k, const LeoProfile* p, const LeoConfig* cfg,
              const LeoEdges* in, const LeoPaths* in_paths, LeoEdges* out, LeoPaths* paths,
              LeoDiags* diags, uint32_t* status, void* stream);

/* backward slice from every instruction with S_j > 0 over `pruned` incoming
 * adjacency: bitmap[(N+31)/32], level[N] (-1 outside the slice). */
int leo_slice(const LeoKernel* k, const LeoProfile* p, const LeoEdges* pruned,
              uint32_t* bitmap, int32_t* level, void* stream);

/* attribute_blame(pruned, base_graph=base) + per-line rollup.
 * `paths` (may be NULL: no valid paths): the pruned edges' valid_paths, from
 * which _edge_distance (analysis.py:371-376) is computed here.  `base` may be
 * NULL (attribute_blame(graph) without base_graph: no indirect-addressing
 * upgrade).  line_id[N] (may be NULL), line_blame[n_lines], line_stall[n_lines]
 * zeroed here. */
int leo_blame(const LeoKernel* k, const LeoProfile* p, const LeoEdges* pruned,
              const LeoPaths* paths, const LeoEdges* base, const int32_t* line_id,
              int32_t n_lines, LeoBlame* out, double* line_blame, double* line_stall,
              uint32_t* status, void* stream);

/* self_blame(index, attached, base_graph) (analysis.py:414-428) for n given
 * instructions: SelfBlame subcategory and S_j (any instruction, stalled or
 * not).  base may be NULL (no indirect-addressing upgrade). */
int leo_self_blame(const LeoKernel* k, const LeoProfile* p, const LeoEdges* base, int32_t n,
                   const int32_t* index, uint8_t* sub, double* cycles, void* stream);

/* single_dep_coverage(graph) (analysis.py:547-561): out[0] = nodes with
 * incoming edges, out[1] = qualifying nodes (device int32[2]). */
int leo_coverage(const LeoKernel* k, const LeoEdges* edges, int32_t* out, void* stream);

/* rank_hotspots(attached, top_n, include_unsampled) (report.py:96-109):
 * hot[<= top_n] instruction indices, *n_hot (device); top_n <= 4096. */
int leo_rank_hotspots(const LeoKernel* k, const LeoProfile* p, int32_t top_n,
                      int32_t include_unsampled, int32_t* hot, int32_t* n_hot, void* stream);

/* trace_chain(graph, blame, start, max_depth) (analysis.py:499-538) over an
 * arbitrary list of n blame entries (stalled, cause or -1 for self,
 * blame_cycles), any order: chain_node[<= max_depth] instructions,
 * chain_entry[] the entry that reached each hop (-1 for the start),
 * *chain_len, *chain_self = the self entry ending the chain or -1.
 * Cause offsets are taken to increase with the instruction index
 * (disasm.py:391-392).  All pointers are device pointers. */
int leo_trace_chain(const LeoKernel* k, int32_t n_entries, const int32_t* stalled,
                    const int32_t* cause, const double* blame, int32_t start, int32_t max_depth,
                    int32_t* chain_node, int32_t* chain_entry, int32_t* chain_len,
                    int32_t* chain_self, void* stream);

/* liveness_filter(cfg, links) (depgraph.py:274-293; liveness :235-271):
 * keep[e] = 1 when link e survives.  links: raw/guard edges (meta carries the
 * linking register ref), any order. */
int leo_liveness_filter(const LeoKernel* k, const LeoEdges* links, uint8_t* keep, void* stream);

/* per-source-line rollup (frozen semantics) of an arbitrary list
 * of n blame entries (stalled, cause or -1, blame_cycles; device pointers):
 * line_blame[line_id[cause, else stalled]] += blame_cycles and
 * line_stall[line_id[j]] += S_j; both vectors are zeroed here. */
int leo_line_rollup(const LeoKernel* k, const LeoProfile* p, int32_t n_entries, const int32_t* stalled,
                    const int32_t* cause, const double* blame, const int32_t* line_id, int32_t n_lines,
                    double* line_blame, double* line_stall, void* stream);

/* The lines a result touches, as a sparse list for read-back: every line x
 * with line_blame[x] != 0 or line_stall[x] != 0, ascending, into line_ids /
 * blame_out / stall_out (capacity entries; *count = the number of such lines,
 * which may exceed capacity: re-run bigger).  A service reads back these
 * instead of the dense per-line vectors (4.3 M lines at C5's line table). */
int leo_line_compact(const double* line_blame, const double* line_stall, int32_t n_lines, int32_t capacity,
                     int32_t* line_ids, double* blame_out, double* stall_out, int32_t* count, void* stream);

/* reaching_definitions(cfg) (depgraph.py:135-177): the reach-in set of every
 * (block b, unit u) pair, as the CSR defs[set_off[b*U+u] .. set_off[b*U+u+1])
 * (set order unspecified; a def may be listed more than once).  Two-phase: *count is the total even when it
 * exceeds `capacity` (then LEO_ST_SCRATCH_OVERFLOW is set in *status). */
typedef struct LeoReachIn {
  int64_t  capacity;          /* defs capacity */
  int32_t* set_off;           /* [B*U + 1] */
  int32_t* defs;              /* [capacity] */
  int32_t* count;             /* device scalar */
} LeoReachIn;
int leo_reaching_definitions(const LeoKernel* k, const LeoCaps* caps, LeoReachIn* out,
                             uint32_t* status, void* stream);

/* profiling helpers for LeoTrace: create / time / destroy CUDA events */
int leo_events_create(int32_t n, void** events);
int leo_events_elapsed(int32_t n, void* const* begin, void* const* end, float* ms);
int leo_events_destroy(int32_t n, void** events);

/* fused pipeline (report.py:132-142 order): optional stage-0 binning of `samples`
 * into `p->lat` / `p->cls_cnt` (which must then be writable), build_graph,
 * run_pruning, slice, attribute_blame(pruned, base) and the per-line rollup,
 * all stream-ordered with no host synchronisation. */
/* ---- report assembly on device outputs (report.py:96-199, analysis.py:499-561)
 * single_dep_coverage before (base graph minus sync edges) and after (pruned),
 * rank_hotspots, per-hotspot cause order and trace_chain.  Blame entries must
 * be the ones leo_analyze / leo_blame produced (grouped by stalled instruction
 * in increasing order).  Variable-size results use the given capacities; a
 * hotspot with more than max_causes entries sets LEO_ST_SCRATCH_OVERFLOW and
 * reports its true count in n_causes. */
typedef struct LeoReport {
  int32_t  top_n;             /* hotspots wanted (<= 4096 on the device path) */
  int32_t  include_unsampled; /* zero-stall instructions after the sampled ones */
  int32_t  chain_depth;       /* trace_chain max_depth (hops incl. the start) */
  int32_t  max_causes;        /* capacity of each hotspot's cause list */
  int32_t* coverage;          /* [4] nodes/qualified before, nodes/qualified after */
  int32_t* n_hot;             /* [1] */
  int32_t* hot;               /* [top_n] instruction indices, ranked */
  int32_t* n_causes;          /* [top_n] */
  int32_t* causes;            /* [top_n * max_causes] blame entry indices, report order */
  int32_t* chain_len;         /* [top_n] hops incl. the start */
  int32_t* chain_node;        /* [top_n * chain_depth] instruction of each hop */
  int32_t* chain_entry;       /* [top_n * chain_depth] entry that reached the hop (-1: start) */
  int32_t* chain_self;        /* [top_n] self-blame entry ending the chain, -1 none */
} LeoReport;

/* replaces report.build_report's assembly (report.py:132-199) after the
 * analysis: all outputs stay on the device, stream-ordered. */
int leo_report(const LeoKernel* k, const LeoProfile* p, const LeoEdges* base, const LeoEdges* pruned,
               const LeoBlame* blame, LeoReport* out, uint32_t* status, void* stream);

int leo_analyze(const LeoKernel* k, const LeoProfile* p, const LeoSamples* samples,
                const LeoConfig* cfg, const LeoCaps* caps, LeoEdges* base, LeoEdges* pruned,
                LeoPaths* paths, LeoDiags* diags, LeoBlame* blame, uint32_t* slice_bitmap,
                int32_t* slice_level, const int32_t* line_id, int32_t n_lines,
                double* line_blame, double* line_stall, uint32_t* status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LEO_B200_H */
