/*
 * leo_oracle.c — CPU restatement of the LEO analysis hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path (and the `--impl reference` CPU baseline of bench.py).  The product
 * (paper_2604_20032_b200/) never links, loads or calls it.
 *
 * It restates, function by function, the reference `stalltrace` package
 * (/root/reference/pkg/src/stalltrace, pure Python) over the SoA layout of
 * include/leo_b200.h.  Pinned against the reference itself: tests/golden/
 * holds vectors produced by running the reference (tests/golden/make_golden.py)
 * and tests/test_oracle_golden.py checks this file against every one of them.
 *
 * Single-threaded per kernel (the reference is single-threaded);
 * the Python wrapper runs independent kernels on separate host threads.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <math.h>

#include "../include/leo_b200.h"

/* ------------------------------------------------------------------------ */
/* small growable vectors                                                    */
typedef struct { int32_t* v; int64_t n, cap; } vi32;
typedef struct { uint64_t* v; int64_t n, cap; } vu64;
typedef struct { double* v; int64_t n, cap; } vf64;

static void vi32_push(vi32* a, int32_t x) {
  if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 64; a->v = (int32_t*)realloc(a->v, a->cap * sizeof(int32_t)); }
  a->v[a->n++] = x;
}
static void vu64_push(vu64* a, uint64_t x) {
  if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 64; a->v = (uint64_t*)realloc(a->v, a->cap * sizeof(uint64_t)); }
  a->v[a->n++] = x;
}
static void vf64_push(vf64* a, double x) {
  if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 64; a->v = (double*)realloc(a->v, a->cap * sizeof(double)); }
  a->v[a->n++] = x;
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static double now_s(void) {
  struct timespec ts; clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

/* ------------------------------------------------------------------------ */
/* enum helpers (isa.py:61-85, depgraph.py:63-68)                            */
#define BIT(c) (1u << (c))
static const uint32_t MEMORY_PRODUCER = BIT(LEO_OC_GLOBAL_LOAD) | BIT(LEO_OC_LOCAL_LOAD) |
    BIT(LEO_OC_SCALAR_LOAD) | BIT(LEO_OC_CONSTANT_LOAD) | BIT(LEO_OC_ATOMIC) | BIT(LEO_OC_SEND);
static const uint32_t MEMORY_CLASSES_ = (BIT(LEO_OC_GLOBAL_LOAD) | BIT(LEO_OC_LOCAL_LOAD) |
    BIT(LEO_OC_SCALAR_LOAD) | BIT(LEO_OC_CONSTANT_LOAD) | BIT(LEO_OC_ATOMIC) | BIT(LEO_OC_SEND)) |
    BIT(LEO_OC_GLOBAL_STORE) | BIT(LEO_OC_LOCAL_STORE);
static const uint32_t COMPUTE = BIT(LEO_OC_FP_ARITH) | BIT(LEO_OC_INT_ARITH) | BIT(LEO_OC_CONVERSION);
static const uint32_t VMCNT_CL = BIT(LEO_OC_GLOBAL_LOAD) | BIT(LEO_OC_GLOBAL_STORE) | BIT(LEO_OC_ATOMIC);
static const uint32_t LGKMCNT_CL = BIT(LEO_OC_LOCAL_LOAD) | BIT(LEO_OC_LOCAL_STORE) |
    BIT(LEO_OC_SCALAR_LOAD) | BIT(LEO_OC_CONSTANT_LOAD);
/* RegClass rank in `.value` string order (depgraph.py:514-516 sort key) */
static const int RC_RANK[8] = {6, 2, 1, 0, 5, 3, 4, 7};

static int dep_class_of(const LeoKernel* k, int producer, int kind) {
  if (kind >= LEO_EK_MEM_WAITCNT) return LEO_DC_MEMORY;
  uint32_t oc = k->opclass[producer];
  if (MEMORY_PRODUCER & BIT(oc)) return LEO_DC_MEMORY;
  if (oc == LEO_OC_BARRIER_ALL) return LEO_DC_SYNCHRONIZATION;
  return LEO_DC_EXECUTION;
}

#define OP_INDEX(r) ((int)((r) & 0xFFFF))
#define OP_SPAN(r) ((int)(((r) >> 16) & 0xFF))
#define OP_CLASS(r) ((int)(((r) >> 24) & 7))
#define OP_ROLE(r) ((int)(((r) >> 27) & 3))
#define OP_REF27(r) ((r) & 0x07FFFFFFu)

/* ------------------------------------------------------------------------ */
/* output                                                                    */
typedef struct OracleOut {
  /* base graph */
  int32_t n_edges, n_regular;
  int32_t *prod, *cons; uint32_t* meta;
  /* pruned graph */
  int32_t np_edges;
  int32_t *p_prod, *p_cons, *p_src; uint32_t* p_meta;
  int32_t *p_npaths, *p_first; double* p_dist;
  int32_t n_paths; int32_t* path_len; double* path_acc;
  /* diagnostics (build then prune, reference order) */
  int32_t n_diags; LeoDiag* diags;
  /* blame */
  int32_t n_entries;
  int32_t *e_stalled, *e_edge; uint8_t* e_sub; double *e_blame, *e_factors;
  /* slice */
  int32_t* level;            /* [N] */
  int32_t slice_size;
  /* lines */
  double *line_blame, *line_stall;
  /* per-stage seconds: graph, sync, s12, s3, s4, blame, slice, lines, binning */
  double t[10];
} OracleOut;

/* ------------------------------------------------------------------------ */
/* register dataflow                                                         */
typedef struct {
  const LeoKernel* k;
  int N, B, U;
  /* per-unit sorted def instruction list (CSR) */
  int32_t *udef_ptr, *udef;
  /* search scratch */
  int32_t* stamp; int32_t cur_stamp;
  int32_t* stack;
} Dataflow;

static void df_init(Dataflow* d, const LeoKernel* k) {
  d->k = k; d->N = k->n_instr; d->B = k->n_blocks; d->U = k->n_units;
  d->udef_ptr = (int32_t*)calloc(d->U + 1, sizeof(int32_t));
  for (int i = 0; i < d->N; i++)
    for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
      uint32_t r = k->opnd[q];
      if (OP_ROLE(r) != LEO_ROLE_DST) continue;
      int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
      for (int s = 0; s < OP_SPAN(r); s++) d->udef_ptr[u0 + s + 1]++;
    }
  for (int u = 0; u < d->U; u++) d->udef_ptr[u + 1] += d->udef_ptr[u];
  int32_t* fill = (int32_t*)malloc((d->U + 1) * sizeof(int32_t));
  memcpy(fill, d->udef_ptr, (d->U + 1) * sizeof(int32_t));
  d->udef = (int32_t*)malloc((d->udef_ptr[d->U] + 1) * sizeof(int32_t));
  for (int i = 0; i < d->N; i++)
    for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
      uint32_t r = k->opnd[q];
      if (OP_ROLE(r) != LEO_ROLE_DST) continue;
      int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
      for (int s = 0; s < OP_SPAN(r); s++) {
        int u = u0 + s;
        /* one instruction may list a unit twice: keep one entry */
        if (fill[u] > d->udef_ptr[u] && d->udef[fill[u] - 1] == i) continue;
        d->udef[fill[u]++] = i;
      }
    }
  /* compact duplicates (entries left unused at the tail of each segment) */
  int w = 0;
  int32_t* np = (int32_t*)malloc((d->U + 1) * sizeof(int32_t));
  for (int u = 0; u < d->U; u++) {
    np[u] = w;
    for (int x = d->udef_ptr[u]; x < fill[u]; x++) d->udef[w++] = d->udef[x];
  }
  np[d->U] = w;
  free(d->udef_ptr); free(fill);
  d->udef_ptr = np;
  d->stamp = (int32_t*)calloc(d->B > 0 ? d->B : 1, sizeof(int32_t));
  d->cur_stamp = 0;
  d->stack = (int32_t*)malloc((size_t)(d->B + 1) * sizeof(int32_t) * 2 + 64);
}
static void df_free(Dataflow* d) {
  free(d->udef_ptr); free(d->udef); free(d->stamp); free(d->stack);
}

/* last definition of unit u inside block p, or -1 (block_defs depgraph.py:143-149) */
static int lastdef_in_block(const Dataflow* d, int p, int u) {
  int lo = d->udef_ptr[u], hi = d->udef_ptr[u + 1] - 1;
  int last = d->k->blk_last[p], first = d->k->blk_first[p];
  int ans = -1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    if (d->udef[mid] <= last) { ans = d->udef[mid]; lo = mid + 1; } else hi = mid - 1;
  }
  return (ans >= first) ? ans : -1;
}

/* reach_in(b)[u] of reaching_definitions (depgraph.py:135-177): the least
 * fixed point of  in(b,u) = U_{p in preds(b)} (lastdef(p,u) if p defines u
 * else in(p,u))  is the set of last-defs of every defining block that reaches
 * b backward through blocks transparent to u.  Result appended (unsorted). */
static void reach_query(Dataflow* d, int b, int u, vi32* out) {
  const LeoKernel* k = d->k;
  int st = ++d->cur_stamp;
  int sp = 0;
  for (int q = k->pred_ptr[b]; q < k->pred_ptr[b + 1]; q++) {
    int p = k->pred[q];
    if (d->stamp[p] != st) { d->stamp[p] = st; d->stack[sp++] = p; }
  }
  while (sp > 0) {
    int p = d->stack[--sp];
    int ld = lastdef_in_block(d, p, u);
    if (ld >= 0) { vi32_push(out, ld); continue; }
    for (int q = k->pred_ptr[p]; q < k->pred_ptr[p + 1]; q++) {
      int pp = k->pred[q];
      if (d->stamp[pp] != st) { d->stamp[pp] = st; d->stack[sp++] = pp; }
    }
  }
}

/* liveness (depgraph.py:235-271) as per-block unit bitsets */
typedef struct { int W; uint64_t *gen, *kill, *in, *out; } Live;

static void unit_set(uint64_t* row, int u) { row[u >> 6] |= 1ull << (u & 63); }
static int unit_get(const uint64_t* row, int u) { return (row[u >> 6] >> (u & 63)) & 1; }

static void liveness(const LeoKernel* k, Live* L) {
  int B = k->n_blocks, W = (k->n_units + 63) / 64;
  if (W == 0) W = 1;
  L->W = W;
  L->gen = (uint64_t*)calloc((size_t)B * W, 8);
  L->kill = (uint64_t*)calloc((size_t)B * W, 8);
  L->in = (uint64_t*)calloc((size_t)B * W, 8);
  L->out = (uint64_t*)calloc((size_t)B * W, 8);
  for (int b = 0; b < B; b++) {
    uint64_t *g = L->gen + (size_t)b * W, *kl = L->kill + (size_t)b * W;
    for (int i = k->blk_first[b]; i <= k->blk_last[b]; i++) {
      for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
        uint32_t r = k->opnd[q];
        if (OP_ROLE(r) == LEO_ROLE_DST) continue;
        int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
        for (int s = 0; s < OP_SPAN(r); s++)
          if (!unit_get(kl, u0 + s)) unit_set(g, u0 + s);
      }
      for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
        uint32_t r = k->opnd[q];
        if (OP_ROLE(r) != LEO_ROLE_DST) continue;
        int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
        for (int s = 0; s < OP_SPAN(r); s++) unit_set(kl, u0 + s);
      }
    }
  }
  /* FIFO worklist, initial order B-1..0 (depgraph.py:254) */
  int32_t* wl = (int32_t*)malloc((size_t)(B + 1) * sizeof(int32_t));
  uint8_t* inwl = (uint8_t*)malloc(B > 0 ? B : 1);
  int head = 0, tail = 0, cnt = 0;
  for (int b = B - 1; b >= 0; b--) { wl[tail] = b; tail = (tail + 1) % (B + 1); inwl[b] = 1; cnt++; }
  uint64_t* tmp = (uint64_t*)malloc((size_t)W * 8);
  while (cnt > 0) {
    int b = wl[head]; head = (head + 1) % (B + 1); cnt--; inwl[b] = 0;
    uint64_t* o = L->out + (size_t)b * W;
    memset(o, 0, (size_t)W * 8);
    for (int q = k->succ_ptr[b]; q < k->succ_ptr[b + 1]; q++) {
      uint64_t* si = L->in + (size_t)k->succ[q] * W;
      for (int w = 0; w < W; w++) o[w] |= si[w];
    }
    int changed = 0;
    uint64_t *g = L->gen + (size_t)b * W, *kl = L->kill + (size_t)b * W, *in = L->in + (size_t)b * W;
    for (int w = 0; w < W; w++) {
      tmp[w] = g[w] | (o[w] & ~kl[w]);
      if (tmp[w] != in[w]) changed = 1;
    }
    if (changed) {
      memcpy(in, tmp, (size_t)W * 8);
      for (int q = k->pred_ptr[b]; q < k->pred_ptr[b + 1]; q++) {
        int p = k->pred[q];
        if (!inwl[p]) { inwl[p] = 1; wl[tail] = p; tail = (tail + 1) % (B + 1); cnt++; }
      }
    }
  }
  free(wl); free(inwl); free(tmp);
}

/* per-consumer candidate key: producer | kind rank (guard < raw) | class rank | index | span */
static uint64_t link_key(int producer, int kind, uint32_t r) {
  uint64_t ref = ((uint64_t)RC_RANK[OP_CLASS(r)] << 24) | ((uint64_t)OP_INDEX(r) << 8) | (uint64_t)OP_SPAN(r);
  return ((uint64_t)producer << 28) | ((uint64_t)(kind == LEO_EK_RAW ? 1 : 0) << 27) | ref;
}

/* diag buffer */
typedef struct { LeoDiag* v; int n, cap; } vdiag;
static void diag_push(vdiag* a, int code, int instr, int a0, int a1, int a2, int seq) {
  if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 32; a->v = (LeoDiag*)realloc(a->v, a->cap * sizeof(LeoDiag)); }
  LeoDiag d = {code, instr, a0, a1, a2, seq};
  a->v[a->n++] = d;
}

/* build the raw/guard edges: reaching_definitions + per_use_link +
 * liveness_filter + sort (depgraph.py:510-524) */
static void build_regular(const LeoKernel* k, vi32* prod, vi32* cons, vi32* meta, vdiag* diags) {
  Dataflow d; df_init(&d, k);
  int N = k->n_instr, U = k->n_units;
  /* running map: in-block last def per unit (stamped by block) and cached
   * reach-in query per (block, unit) */
  int32_t* tb = (int32_t*)malloc((U + 1) * sizeof(int32_t));
  int32_t* td = (int32_t*)malloc((U + 1) * sizeof(int32_t));
  int32_t* qb = (int32_t*)malloc((U + 1) * sizeof(int32_t));
  int32_t* qoff = (int32_t*)malloc((U + 1) * sizeof(int32_t));
  int32_t* qlen = (int32_t*)malloc((U + 1) * sizeof(int32_t));
  for (int u = 0; u <= U; u++) { tb[u] = -1; qb[u] = -1; }
  vi32 pool = {0}; vu64 cand = {0};
  Live L; liveness(k, &L);
  for (int b = 0; b < k->n_blocks; b++) {
    pool.n = 0;
    for (int i = k->blk_first[b]; i <= k->blk_last[b]; i++) {
      cand.n = 0;
      for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
        uint32_t r = k->opnd[q];
        int role = OP_ROLE(r);
        if (role == LEO_ROLE_DST) continue;
        int kind = role == LEO_ROLE_GUARD ? LEO_EK_GUARD : LEO_EK_RAW;
        int found = 0;
        int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
        for (int s = 0; s < OP_SPAN(r); s++) {
          int u = u0 + s;
          if (tb[u] == b) { vu64_push(&cand, link_key(td[u], kind, r)); found = 1; continue; }
          if (qb[u] != b) {
            qb[u] = b; qoff[u] = (int32_t)pool.n;
            reach_query(&d, b, u, &pool);
            qlen[u] = (int32_t)(pool.n - qoff[u]);
          }
          for (int x = 0; x < qlen[u]; x++) { vu64_push(&cand, link_key(pool.v[qoff[u] + x], kind, r)); found = 1; }
        }
        if (!found) diag_push(diags, LEO_DIAG_UNRESOLVED, i, (int32_t)r, 0, 0, q - k->opnd_ptr[i]);
      }
      for (int q = k->opnd_ptr[i]; q < k->opnd_ptr[i + 1]; q++) {
        uint32_t r = k->opnd[q];
        if (OP_ROLE(r) != LEO_ROLE_DST) continue;
        int u0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
        for (int s = 0; s < OP_SPAN(r); s++) { tb[u0 + s] = b; td[u0 + s] = i; }
      }
      /* links are keyed (d, i, ref, kind) and sorted per consumer */
      qsort(cand.v, cand.n, sizeof(uint64_t), cmp_u64);
      for (int64_t x = 0; x < cand.n; x++) {
        if (x > 0 && cand.v[x] == cand.v[x - 1]) continue;
        uint64_t key = cand.v[x];
        int producer = (int)(key >> 28);
        int kind = ((key >> 27) & 1) ? LEO_EK_RAW : LEO_EK_GUARD;
        int rank = (int)((key >> 24) & 7);
        int cls = 0;
        for (int c = 0; c < 8; c++) if (RC_RANK[c] == rank) cls = c;
        uint32_t ref27 = (uint32_t)((key >> 8) & 0xFFFF) | ((uint32_t)(key & 0xFF) << 16) | ((uint32_t)cls << 24);
        /* liveness_filter (depgraph.py:274-293): cross-block links need the
         * linking units live out of the producer's block */
        int pb = k->block_of[producer], cb = k->block_of[i];
        if (pb != cb) {
          int use0 = k->unit_base[cls] + (int)(ref27 & 0xFFFF), span = (int)((ref27 >> 16) & 0xFF);
          uint64_t* lo = L.out + (size_t)pb * L.W;
          int any_written = 0, live = 0;
          for (int s = 0; s < span; s++) {
            int u = use0 + s, w = 0;
            for (int q = k->opnd_ptr[producer]; q < k->opnd_ptr[producer + 1]; q++) {
              uint32_t r = k->opnd[q];
              if (OP_ROLE(r) != LEO_ROLE_DST) continue;
              int a0 = k->unit_base[OP_CLASS(r)] + OP_INDEX(r);
              if (u >= a0 && u < a0 + OP_SPAN(r)) w = 1;
            }
            if (w) { any_written = 1; if (unit_get(lo, u)) live = 1; }
          }
          if (!any_written)
            for (int s = 0; s < span; s++) if (unit_get(lo, use0 + s)) live = 1;
          if (!live) continue;
        }
        vi32_push(prod, producer); vi32_push(cons, i);
        vi32_push(meta, (int32_t)LEO_META(kind, dep_class_of(k, producer, kind), ref27));
      }
    }
  }
  free(tb); free(td); free(qb); free(qoff); free(qlen); free(pool.v); free(cand.v);
  free(L.gen); free(L.kill); free(L.in); free(L.out);
  df_free(&d);
}

/* ------------------------------------------------------------------------ */
/* synchronization tracing: _scan_backward chains (depgraph.py:312-348)      */
#define SYNC_SCAN_BUDGET 4096

typedef struct {
  const LeoKernel* k;
  int32_t* onpath;        /* per block: 1 while the block is on the chain path */
  int32_t* mark;          /* per instruction: stamp of the wait that linked it */
  int32_t* pend;          /* pending members (waitcnt), youngest first */
  vu64* edges;            /* (producer << 32 | consumer) */
  /* chain DFS frames */
  int32_t *f_block, *f_q, *f_m, *f_a, *f_budget;
} SyncCtx;

/* waitcnt visitor (depgraph.py:368-384).  Returns 0 to stop the chain. */
static int visit_waitcnt(SyncCtx* c, int x, int counter, uint32_t members, int level, int wait,
                         int* m, int* a) {
  const LeoKernel* k = c->k;
  if (k->sync_kind[x] == LEO_SYNC_WAITCNT) {
    uint32_t v = counter == 0 ? k->sync_a[x] : k->sync_b[x];
    if (v != LEO_NONE_U32) {
      *a = (*a < 0) ? (int)v : (*a < (int)v ? *a : (int)v);
      if (*a == 0) return 0;
    }
  } else if (members & BIT(k->opclass[x])) {
    if (*a < 0 || *a > 0) {
      c->pend[*m] = x;
      if (*m >= level && c->mark[x] != wait + 1) {
        c->mark[x] = wait + 1;
        vu64_push(c->edges, ((uint64_t)x << 32) | (uint32_t)wait);
      }
      (*m)++;
      if (*a > 0) { (*a)--; if (*a == 0) return 0; }
    }
  }
  return 1;
}

/* setter visitor (depgraph.py:435-440): match -> edge + stop */
static int visit_setter(SyncCtx* c, int x, int kind, int id, int wait, int* found) {
  const LeoKernel* k = c->k;
  int hit = 0;
  if (kind == LEO_EK_MEM_BARRIER)
    hit = k->sync_kind[x] == LEO_SYNC_BARRIER && (((k->sync_a[x] | (k->sync_a[x] >> 8)) >> id) & 1);
  else
    hit = k->sync_kind[x] == LEO_SYNC_SWSB && k->sync_a[x] == (uint32_t)id;
  if (hit) {
    if (c->mark[x] != wait + 1) {
      c->mark[x] = wait + 1;
      vu64_push(c->edges, ((uint64_t)x << 32) | (uint32_t)wait);
    }
    *found = 1;
    return 0;
  }
  return 1;
}

/* Enumerate every chain (= simple backward block path from the wait, b0
 * pre-visited, forks inherit the remaining budget) exactly as _scan_backward
 * does; the result (edge union, best_m / found) is chain-order independent.
 * mode 0: waitcnt(counter, level, members)  mode 1: setter(kind, id) */
static void trace_chains(SyncCtx* c, int wait, int mode, int counter_or_kind, int level_or_id,
                         uint32_t members, int* best_m, int* found) {
  const LeoKernel* k = c->k;
  int b0 = k->block_of[wait];
  int top = 0;
  c->onpath[b0] = 1;
  /* scan the root chain */
  int m = 0, a = -1, budget = SYNC_SCAN_BUDGET, stopped = 0;
  for (int x = wait - 1; x >= k->blk_first[b0]; x--) {
    if (budget == 0) { stopped = 1; break; }
    budget--;
    int go = mode == 0 ? visit_waitcnt(c, x, counter_or_kind, members, level_or_id, wait, &m, &a)
                       : visit_setter(c, x, counter_or_kind, level_or_id, wait, found);
    if (!go) { stopped = 1; break; }
  }
  if (stopped) { if (m > *best_m) *best_m = m; c->onpath[b0] = 0; return; }
  /* frame: block whose predecessors are being expanded */
  c->f_block[0] = b0; c->f_q[0] = k->pred_ptr[b0]; c->f_m[0] = m; c->f_a[0] = a; c->f_budget[0] = budget;
  top = 1;
  /* a chain with no unvisited preds is terminal */
  {
    int any = 0;
    for (int q = k->pred_ptr[b0]; q < k->pred_ptr[b0 + 1]; q++) if (!c->onpath[k->pred[q]]) any = 1;
    if (!any) { if (m > *best_m) *best_m = m; c->onpath[b0] = 0; return; }
  }
  while (top > 0) {
    int f = top - 1;
    int blk = c->f_block[f];
    /* next unvisited predecessor */
    int p = -1;
    while (c->f_q[f] < k->pred_ptr[blk + 1]) {
      int cand = k->pred[c->f_q[f]++];
      if (!c->onpath[cand]) { p = cand; break; }
    }
    if (p < 0) { c->onpath[blk] = 0; top--; continue; }
    /* child chain: copy of the state */
    m = c->f_m[f]; a = c->f_a[f]; budget = c->f_budget[f]; stopped = 0;
    for (int x = k->blk_last[p]; x >= k->blk_first[p]; x--) {
      if (budget == 0) { stopped = 1; break; }
      budget--;
      int go = mode == 0 ? visit_waitcnt(c, x, counter_or_kind, members, level_or_id, wait, &m, &a)
                         : visit_setter(c, x, counter_or_kind, level_or_id, wait, found);
      if (!go) { stopped = 1; break; }
    }
    if (stopped) { if (m > *best_m) *best_m = m; continue; }
    c->onpath[p] = 1;
    int any = 0;
    for (int q = k->pred_ptr[p]; q < k->pred_ptr[p + 1]; q++) if (!c->onpath[k->pred[q]]) any = 1;
    if (!any) { if (m > *best_m) *best_m = m; c->onpath[p] = 0; continue; }
    c->f_block[top] = p; c->f_q[top] = k->pred_ptr[p]; c->f_m[top] = m; c->f_a[top] = a;
    c->f_budget[top] = budget; top++;
  }
}

static void build_sync(const LeoKernel* k, vi32* prod, vi32* cons, vi32* meta, vdiag* diags) {
  int N = k->n_instr, B = k->n_blocks;
  SyncCtx c; memset(&c, 0, sizeof c);
  vu64 edges = {0};
  c.k = k; c.edges = &edges;
  c.onpath = (int32_t*)calloc(B + 1, sizeof(int32_t));
  c.mark = (int32_t*)calloc(N + 1, sizeof(int32_t));
  c.pend = (int32_t*)malloc((SYNC_SCAN_BUDGET + 8) * sizeof(int32_t));
  int fcap = B + 2;
  c.f_block = (int32_t*)malloc(fcap * sizeof(int32_t)); c.f_q = (int32_t*)malloc(fcap * sizeof(int32_t));
  c.f_m = (int32_t*)malloc(fcap * sizeof(int32_t)); c.f_a = (int32_t*)malloc(fcap * sizeof(int32_t));
  c.f_budget = (int32_t*)malloc(fcap * sizeof(int32_t));
  int kind = k->dialect == LEO_AMD ? LEO_EK_MEM_WAITCNT : k->dialect == LEO_NVIDIA ? LEO_EK_MEM_BARRIER : LEO_EK_MEM_SWSB;
  for (int i = 0; i < N; i++) {
    if (k->dialect == LEO_AMD) {
      if (k->sync_kind[i] != LEO_SYNC_WAITCNT) continue;
      for (int counter = 0; counter < 2; counter++) {  /* vmcnt before lgkmcnt (depgraph.py:410-415) */
        uint32_t lv = counter == 0 ? k->sync_a[i] : k->sync_b[i];
        if (lv == LEO_NONE_U32) continue;
        int best_m = 0, found = 0;
        trace_chains(&c, i, 0, counter, (int)lv, counter == 0 ? VMCNT_CL : LGKMCNT_CL, &best_m, &found);
        if (best_m < (int)lv) diag_push(diags, LEO_DIAG_WAITCNT, i, counter, (int)lv, best_m, counter);
      }
    } else if (k->dialect == LEO_NVIDIA) {
      if (k->sync_kind[i] != LEO_SYNC_BARRIER) continue;
      uint32_t wait = (k->sync_a[i] >> 16) & 0xFF;
      for (int b = 1; b <= 6; b++) {
        if (!((wait >> b) & 1)) continue;
        int best_m = 0, found = 0;
        trace_chains(&c, i, 1, LEO_EK_MEM_BARRIER, b, 0, &best_m, &found);
        if (!found) diag_push(diags, LEO_DIAG_NO_SETTER, i, b, 0, 0, b);
      }
    } else {
      if (k->sync_kind[i] != LEO_SYNC_SWSB) continue;
      uint32_t wait = k->sync_b[i];
      for (int t = 0; t < 32; t++) {
        if (!((wait >> t) & 1)) continue;
        int best_m = 0, found = 0;
        trace_chains(&c, i, 1, LEO_EK_MEM_SWSB, t, 0, &best_m, &found);
        if (!found) diag_push(diags, LEO_DIAG_NO_SETTER, i, t, 0, 0, t);
      }
    }
  }
  /* _materialize_sync: sorted (producer, consumer) (depgraph.py:485-492) */
  qsort(edges.v, edges.n, sizeof(uint64_t), cmp_u64);
  for (int64_t x = 0; x < edges.n; x++) {
    if (x > 0 && edges.v[x] == edges.v[x - 1]) continue;
    int p = (int)(edges.v[x] >> 32), cns = (int)(edges.v[x] & 0xFFFFFFFFu);
    vi32_push(prod, p); vi32_push(cons, cns);
    vi32_push(meta, (int32_t)LEO_META(kind, LEO_DC_MEMORY, 0));
  }
  free(edges.v); free(c.onpath); free(c.mark); free(c.pend);
  free(c.f_block); free(c.f_q); free(c.f_m); free(c.f_a); free(c.f_budget);
}

/* ------------------------------------------------------------------------ */
/* pruning (analysis.py:143-314)                                             */
static double issue_weight(const LeoKernel* k, int i) {  /* _issue_weights :188-199 */
  if (k->dialect == LEO_NVIDIA && k->sync_kind[i] == LEO_SYNC_BARRIER && k->sync_b[i] != LEO_NONE_U32)
    return (double)k->sync_b[i];
  return 1.0;
}
static int only_class(const LeoProfile* p, int j, int cls) {  /* _only_class :134-140 */
  if (p->lat[j] == 0) return 0;
  for (int c = 0; c < 8; c++) if (c != cls && p->cls_cnt[(size_t)j * 8 + c] > 0) return 0;
  return 1;
}

typedef struct { int32_t node, len, back; double acc; } DfsEnt;
typedef struct { int32_t nb, cb, parent; } BackNode;
typedef struct { int32_t len; double acc; } PathRec;
static int cmp_path(const void* a, const void* b) {
  const PathRec *x = (const PathRec*)a, *y = (const PathRec*)b;
  if (x->len != y->len) return x->len < y->len ? -1 : 1;
  return x->acc < y->acc ? -1 : x->acc > y->acc;
}

/* _enumerate_paths (analysis.py:210-253), LIFO order reproduced exactly */
static int enumerate_paths(const LeoKernel* k, const double* w, int producer, int consumer,
                           double threshold, int max_paths, int max_depth,
                           PathRec* valid, int* nvalid, DfsEnt* stack, BackNode* arena) {
  int budget = 65536, truncated = 0, sp = 0, na = 0;
  *nvalid = 0;
  if (w[producer] > threshold) return 0;
  stack[sp].node = producer; stack[sp].len = 1; stack[sp].acc = w[producer]; stack[sp].back = -1; sp++;
  while (sp > 0) {
    DfsEnt e = stack[--sp];
    if (budget <= 0 || *nvalid >= max_paths) { truncated = 1; break; }
    budget--;
    int nb = k->block_of[e.node];
    int succ_n, s0 = -1, s1 = -1;
    if (e.node < k->blk_last[nb]) { succ_n = 1; s0 = e.node + 1; }
    else {
      succ_n = k->succ_ptr[nb + 1] - k->succ_ptr[nb];
      if (succ_n > 0) s0 = k->blk_first[k->succ[k->succ_ptr[nb]]];
      if (succ_n > 1) s1 = k->blk_first[k->succ[k->succ_ptr[nb] + 1]];
    }
    for (int t = 0; t < succ_n; t++) {
      int nxt = t == 0 ? s0 : s1;
      if (nxt == consumer) {
        valid[*nvalid].len = e.len; valid[*nvalid].acc = e.acc; (*nvalid)++;
        if (*nvalid >= max_paths) truncated = 1;
        continue;
      }
      int cb = k->block_of[nxt];
      int nback = e.back;
      if (nb != cb && k->blk_first[cb] <= k->blk_first[nb]) {
        int hit = 0;
        for (int x = e.back; x >= 0; x = arena[x].parent)
          if (arena[x].nb == nb && arena[x].cb == cb) { hit = 1; break; }
        if (hit) continue;
        arena[na].nb = nb; arena[na].cb = cb; arena[na].parent = e.back; nback = na++;
      }
      int nlen = e.len + 1;
      double nacc = e.acc + w[nxt];
      if (nacc > threshold) continue;
      if (nlen >= max_depth) { truncated = 1; continue; }
      stack[sp].node = nxt; stack[sp].len = nlen; stack[sp].acc = nacc; stack[sp].back = nback; sp++;
    }
  }
  qsort(valid, *nvalid, sizeof(PathRec), cmp_path);
  return truncated;
}

/* ------------------------------------------------------------------------ */
/* blame (analysis.py:371-484)                                               */
/* builtins.sum over floats as CPython >= 3.12 evaluates it (Neumaier
 * compensated summation; the int start value 0 makes the first addend exact).
 * Used where the reference calls sum() on floats (analysis.py:464, 472). */
typedef struct { double s, c; int n; } PySum;
static void pysum_add(PySum* a, double x) {
  if (a->n++ == 0) { a->s = 0.0 + x; a->c = 0.0; return; }
  volatile double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) { volatile double d = a->s - t; a->c += d + x; }
  else { volatile double d = x - t; a->c += d + a->s; }
  a->s = t;
}
static double pysum_value(const PySum* a) {
  if (a->c != 0.0 && isfinite(a->c)) return a->s + a->c;
  return a->s;
}

static double issue_count(const LeoProfile* p, int i) {  /* profile.py:321-329 */
  if (p->exec_cnt[i] >= 0) return (double)p->exec_cnt[i];
  if (p->sampled[i]) return (double)(p->total[i] >= 0 ? p->total[i] : p->lat[i]);
  return 1.0;
}
static const int MATCH_CLASS[3] = {LEO_CS_MEMORY_DEP, LEO_CS_EXECUTION_DEP, LEO_CS_SYNCHRONIZATION};
static const int SELF_BY_CLASS[8] = {LEO_SB_MEMORY_LATENCY, LEO_SB_COMPUTE_SATURATION,
    LEO_SB_SYNCHRONIZATION_OVERHEAD, LEO_SB_INSTRUCTION_FETCH, LEO_SB_PIPELINE_CONTENTION,
    LEO_SB_PIPELINE_CONTENTION, LEO_SB_PIPELINE_CONTENTION, LEO_SB_PIPELINE_CONTENTION};

/* consumer CSR in edge-list order (DependencyGraph.incoming depgraph.py:102-108) */
static void incoming_csr(int N, int E, const int32_t* cons, int32_t** ptr_out, int32_t** idx_out) {
  int32_t* ptr = (int32_t*)calloc(N + 1, sizeof(int32_t));
  int32_t* idx = (int32_t*)malloc((E + 1) * sizeof(int32_t));
  for (int e = 0; e < E; e++) ptr[cons[e] + 1]++;
  for (int i = 0; i < N; i++) ptr[i + 1] += ptr[i];
  int32_t* f = (int32_t*)malloc((N + 1) * sizeof(int32_t));
  memcpy(f, ptr, (N + 1) * sizeof(int32_t));
  for (int e = 0; e < E; e++) idx[f[cons[e]]++] = e;
  free(f);
  *ptr_out = ptr; *idx_out = idx;
}

/* _address_traces_to_load (analysis.py:390-411) over the unpruned graph */
static int traces_to_load(const LeoKernel* k, const int32_t* bptr, const int32_t* bidx,
                          const int32_t* bprod, const uint32_t* bmeta, int index,
                          int32_t* seen, int stamp, int32_t* fr, int32_t* nx) {
  int nf = 1; fr[0] = index; seen[index] = stamp;
  for (int depth = 0; depth < 8; depth++) {
    int nn = 0;
    for (int a = 0; a < nf; a++) {
      int node = fr[a];
      for (int q = bptr[node]; q < bptr[node + 1]; q++) {
        int e = bidx[q];
        if (((bmeta[e] >> 27) & 7) != LEO_EK_RAW) continue;
        int p = bprod[e];
        if (seen[p] == stamp) continue;
        if (MEMORY_PRODUCER & BIT(k->opclass[p])) return 1;
        seen[p] = stamp; nx[nn++] = p;
      }
    }
    if (nn == 0) return 0;
    memcpy(fr, nx, nn * sizeof(int32_t)); nf = nn;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* entry points                                                              */
enum { OR_GRAPH = 1, OR_PRUNE = 2, OR_BLAME = 4, OR_SLICE = 8, OR_LINES = 16 };

int oracle_bin_samples(int64_t S, const int32_t* pc, const uint8_t* cat, const uint8_t* lut,
                       int32_t n_instr, int32_t* lat, int32_t* cls_cnt) {
  memset(lat, 0, (size_t)n_instr * 4);
  memset(cls_cnt, 0, (size_t)n_instr * 32);
  for (int64_t s = 0; s < S; s++) {
    int32_t j = pc[s];
    if (j < 0 || j >= n_instr) return -1;
    lat[j]++;
    cls_cnt[(size_t)j * 8 + lut[cat[s]]]++;
  }
  return 0;
}

/* Run the hot path on one kernel.  `base_in` (optional, prod/cons/meta of a
 * prebuilt base graph with n_base edges) replaces graph construction. */
int oracle_run(const LeoKernel* k, const LeoProfile* p, const LeoConfig* cfg, int flags,
               const int32_t* line_id, int32_t n_lines, OracleOut* out) {
  memset(out, 0, sizeof *out);
  int N = k->n_instr;
  vdiag diags = {0};
  vi32 prod = {0}, cons = {0}, meta = {0};
  double t0 = now_s();
  build_regular(k, &prod, &cons, &meta, &diags);
  int n_regular = (int)prod.n;
  double t1 = now_s();
  build_sync(k, &prod, &cons, &meta, &diags);
  double t2 = now_s();
  out->t[0] = t1 - t0; out->t[1] = t2 - t1;
  int E = (int)prod.n;
  out->n_edges = E; out->n_regular = n_regular;
  out->prod = prod.v; out->cons = cons.v; out->meta = (uint32_t*)meta.v;
  if (!(flags & OR_PRUNE)) { out->n_diags = diags.n; out->diags = diags.v; return 0; }

  /* ---- pruning ---- */
  double* w = (double*)malloc((N + 1) * sizeof(double));
  for (int i = 0; i < N; i++) w[i] = issue_weight(k, i);
  uint8_t* keep = (uint8_t*)malloc(E + 1);
  int32_t* npaths = (int32_t*)calloc(E + 1, sizeof(int32_t));
  int32_t* first = (int32_t*)malloc((E + 1) * sizeof(int32_t));
  vi32 plen = {0}; vf64 pacc = {0};
  PathRec* valid = (PathRec*)malloc((cfg->max_paths + 2) * sizeof(PathRec));
  DfsEnt* stack = (DfsEnt*)malloc((size_t)(2 * 65536 + 16) * sizeof(DfsEnt));
  BackNode* arena = (BackNode*)malloc((size_t)(2 * 65536 + 16) * sizeof(BackNode));
  double ts = now_s(), t_s3 = 0;
  for (int e = 0; e < E; e++) {
    int kind = (out->meta[e] >> 27) & 7;
    int pr = out->prod[e], cn = out->cons[e];
    first[e] = -1;
    keep[e] = 1;
    if (kind >= LEO_EK_MEM_WAITCNT) continue;             /* sync edges exempt */
    uint32_t poc = k->opclass[pr];
    if (cfg->stage_mask & 1) {                              /* prune_opcode :143-162 */
      if (only_class(p, cn, LEO_CS_MEMORY_DEP) && (COMPUTE & BIT(poc))) { keep[e] = 0; continue; }
      if (only_class(p, cn, LEO_CS_EXECUTION_DEP) && poc == LEO_OC_GLOBAL_LOAD) { keep[e] = 0; continue; }
    }
    if ((cfg->stage_mask & 2) && k->dialect == LEO_NVIDIA) {   /* prune_barrier :165-185 */
      uint32_t sets = 0, waits = 0;
      if (k->sync_kind[pr] == LEO_SYNC_BARRIER) sets = (k->sync_a[pr] | (k->sync_a[pr] >> 8)) & 0xFF;
      if (sets) {
        if (k->sync_kind[cn] == LEO_SYNC_BARRIER) waits = (k->sync_a[cn] >> 16) & 0xFF;
        if (!(sets & waits)) { keep[e] = 0; continue; }
      }
    }
    if (cfg->stage_mask & 4) {                              /* prune_latency :256-286 */
      double t3 = now_s();
      int nv = 0;
      int trunc = enumerate_paths(k, w, pr, cn, cfg->threshold[poc], cfg->max_paths, cfg->max_depth,
                                  valid, &nv, stack, arena);
      t_s3 += now_s() - t3;
      if (nv > 0) {
        first[e] = (int32_t)plen.n; npaths[e] = nv;
        for (int x = 0; x < nv; x++) { vi32_push(&plen, valid[x].len); vf64_push(&pacc, valid[x].acc); }
        if (trunc) diag_push(&diags, LEO_DIAG_PATH_CAPPED, pr, cn, 1, 0, e);
      } else if (trunc) {
        diag_push(&diags, LEO_DIAG_PATH_CAPPED, pr, cn, 0, 0, e);
      } else { keep[e] = 0; continue; }
    }
    if ((cfg->stage_mask & 8) && cfg->prune_exec && p->exec_cnt[pr] == 0) { keep[e] = 0; continue; }  /* :289-299 */
  }
  double te = now_s();
  out->t[2] = (te - ts) - t_s3; out->t[3] = t_s3;
  int EP = 0;
  for (int e = 0; e < E; e++) EP += keep[e];
  out->np_edges = EP;
  out->p_prod = (int32_t*)malloc((EP + 1) * 4); out->p_cons = (int32_t*)malloc((EP + 1) * 4);
  out->p_src = (int32_t*)malloc((EP + 1) * 4); out->p_meta = (uint32_t*)malloc((EP + 1) * 4);
  out->p_npaths = (int32_t*)malloc((EP + 1) * 4); out->p_first = (int32_t*)malloc((EP + 1) * 4);
  out->p_dist = (double*)malloc((EP + 1) * 8);
  int x = 0;
  for (int e = 0; e < E; e++) {
    if (!keep[e]) continue;
    out->p_prod[x] = out->prod[e]; out->p_cons[x] = out->cons[e]; out->p_meta[x] = out->meta[e];
    out->p_src[x] = e; out->p_npaths[x] = npaths[e]; out->p_first[x] = first[e];
    if (npaths[e] > 0) {                                   /* _edge_distance :371-376 */
      int64_t s = 0;
      for (int q = 0; q < npaths[e]; q++) s += plen.v[first[e] + q];
      out->p_dist[x] = (double)s / (double)npaths[e];
    } else {
      int d = out->cons[e] - out->prod[e]; if (d < 0) d = -d; if (d < 1) d = 1;
      out->p_dist[x] = (double)d;
    }
    x++;
  }
  out->n_paths = (int32_t)plen.n; out->path_len = plen.v; out->path_acc = pacc.v;
  out->n_diags = diags.n; out->diags = diags.v;
  free(w); free(keep); free(npaths); free(first); free(valid); free(stack); free(arena);
  if (!(flags & (OR_BLAME | OR_SLICE | OR_LINES))) return 0;

  /* ---- blame ---- */
  double tb0 = now_s();
  int32_t *pptr, *pidx, *bptr, *bidx;
  incoming_csr(N, EP, out->p_cons, &pptr, &pidx);
  incoming_csr(N, E, out->cons, &bptr, &bidx);
  vi32 es = {0}, ee = {0}; vf64 eb = {0}, ef = {0}; vi32 esub = {0};
  int32_t* seen = (int32_t*)calloc(N + 1, sizeof(int32_t));
  int32_t* fr = (int32_t*)malloc((N + 1) * sizeof(int32_t));
  int32_t* nx = (int32_t*)malloc((N + 1) * sizeof(int32_t));
  int stamp = 0;
  double* dists = NULL; double *effs = NULL, *isus = NULL, *matches = NULL;
  int maxdeg = 1;
  for (int j = 0; j < N; j++) if (pptr[j + 1] - pptr[j] > maxdeg) maxdeg = pptr[j + 1] - pptr[j];
  dists = (double*)malloc(maxdeg * 8); effs = (double*)malloc(maxdeg * 8);
  isus = (double*)malloc(maxdeg * 8); matches = (double*)malloc(maxdeg * 8);
  for (int j = 0; j < N; j++) {
    double s_j = (double)((int64_t)p->lat[j] * p->period);
    if (s_j == 0) continue;
    int deg = pptr[j + 1] - pptr[j];
    int self = deg == 0;
    double total = 0, n_sum = 0, d_min = 0, e_min = 0;
    if (!self) {
      for (int q = 0; q < deg; q++) {
        int e = pidx[pptr[j] + q];
        int pr = out->p_prod[e];
        dists[q] = out->p_dist[e];
        effs[q] = p->eff[pr];
        isus[q] = issue_count(p, pr);
        int dc = (out->p_meta[e] >> 30) & 3;
        matches[q] = (double)p->cls_cnt[(size_t)j * 8 + MATCH_CLASS[dc]] / (double)p->lat[j];
      }
      d_min = dists[0]; e_min = effs[0];
      for (int q = 1; q < deg; q++) { if (dists[q] < d_min) d_min = dists[q]; if (effs[q] < e_min) e_min = effs[q]; }
      PySum ns = {0, 0, 0};
      for (int q = 0; q < deg; q++) pysum_add(&ns, isus[q]);
      n_sum = pysum_value(&ns);
      if (n_sum == 0) self = 1;
      else {
        PySum ts = {0, 0, 0};
        for (int q = 0; q < deg; q++) {
          volatile double f0 = d_min / dists[q], f1 = e_min / effs[q], f2 = isus[q] / n_sum, f3 = matches[q];
          volatile double pr0 = f0 * f1; volatile double pr1 = pr0 * f2; volatile double pr2 = pr1 * f3;
          pysum_add(&ts, pr2);
        }
        total = pysum_value(&ts);
        if (total == 0.0) self = 1;
      }
    }
    if (self) {                                             /* self_blame :414-428 */
      int dom = 0, best = -1;
      for (int c = 0; c < 8; c++) if (p->cls_cnt[(size_t)j * 8 + c] > best) { best = p->cls_cnt[(size_t)j * 8 + c]; dom = c; }
      int sub = SELF_BY_CLASS[dom];
      if (sub == LEO_SB_MEMORY_LATENCY && (MEMORY_CLASSES_ & BIT(k->opclass[j]))) {
        stamp++;
        if (traces_to_load(k, bptr, bidx, out->prod, out->meta, j, seen, stamp, fr, nx))
          sub = LEO_SB_INDIRECT_ADDRESSING;
      }
      vi32_push(&es, j); vi32_push(&ee, -1); vi32_push(&esub, sub); vf64_push(&eb, s_j);
      for (int c = 0; c < 4; c++) vf64_push(&ef, 0.0);
      continue;
    }
    for (int q = 0; q < deg; q++) {
      int e = pidx[pptr[j] + q];
      volatile double f0 = d_min / dists[q], f1 = e_min / effs[q], f2 = isus[q] / n_sum, f3 = matches[q];
      volatile double pr0 = f0 * f1; volatile double pr1 = pr0 * f2; volatile double prod_ = pr1 * f3;
      volatile double num = s_j * prod_;
      double bl = num / total;
      vi32_push(&es, j); vi32_push(&ee, e); vi32_push(&esub, 255); vf64_push(&eb, bl);
      vf64_push(&ef, f0); vf64_push(&ef, f1); vf64_push(&ef, f2); vf64_push(&ef, f3);
    }
  }
  out->n_entries = (int32_t)es.n;
  out->e_stalled = es.v; out->e_edge = ee.v; out->e_blame = eb.v; out->e_factors = ef.v;
  out->e_sub = (uint8_t*)malloc(es.n + 1);
  for (int64_t q = 0; q < es.n; q++) out->e_sub[q] = (uint8_t)esub.v[q];
  free(esub.v); free(dists); free(effs); free(isus); free(matches);
  double tb1 = now_s();
  out->t[5] = tb1 - tb0;

  /* ---- slice: multi-source BFS over pruned incoming ---- */
  out->level = (int32_t*)malloc((N + 1) * sizeof(int32_t));
  int nf = 0, size = 0;
  for (int j = 0; j < N; j++) {
    out->level[j] = -1;
    if ((int64_t)p->lat[j] * p->period != 0) { out->level[j] = 0; fr[nf++] = j; size++; }
  }
  for (int lv = 1; nf > 0; lv++) {
    int nn = 0;
    for (int a = 0; a < nf; a++) {
      int v = fr[a];
      for (int q = pptr[v]; q < pptr[v + 1]; q++) {
        int pr = out->p_prod[pidx[q]];
        if (out->level[pr] < 0) { out->level[pr] = lv; nx[nn++] = pr; size++; }
      }
    }
    memcpy(fr, nx, nn * sizeof(int32_t)); nf = nn;
  }
  out->slice_size = size;
  double tb2 = now_s();
  out->t[6] = tb2 - tb1;

  /* ---- per-source-line rollup ---- */
  out->line_blame = (double*)calloc(n_lines + 1, 8);
  out->line_stall = (double*)calloc(n_lines + 1, 8);
  if (line_id) {
    for (int64_t q = 0; q < es.n; q++) {
      int e = out->e_edge[q];
      int at = e < 0 ? out->e_stalled[q] : out->p_prod[e];
      out->line_blame[line_id[at]] += out->e_blame[q];
    }
    for (int j = 0; j < N; j++) {
      double s_j = (double)((int64_t)p->lat[j] * p->period);
      if (s_j != 0) out->line_stall[line_id[j]] += s_j;
    }
  }
  out->t[7] = now_s() - tb2;
  free(pptr); free(pidx); free(bptr); free(bidx); free(seen); free(fr); free(nx);
  return 0;
}

void oracle_free(OracleOut* o) {
  free(o->prod); free(o->cons); free(o->meta);
  free(o->p_prod); free(o->p_cons); free(o->p_src); free(o->p_meta);
  free(o->p_npaths); free(o->p_first); free(o->p_dist); free(o->path_len); free(o->path_acc);
  free(o->diags); free(o->e_stalled); free(o->e_edge); free(o->e_sub); free(o->e_blame);
  free(o->e_factors); free(o->level); free(o->line_blame); free(o->line_stall);
  memset(o, 0, sizeof *o);
}

int oracle_sizeof_out(void) { return (int)sizeof(OracleOut); }
