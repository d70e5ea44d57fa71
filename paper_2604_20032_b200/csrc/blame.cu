// blame.cu — stage-0 binning, backward slice, blame attribution, line rollup.
//
//   k_bin_hash        big raw (pc, category) streams (>= 4 M samples, packed
//                     u32 words or pc / cat arrays) -> cls_cnt[N, 8] in one
//                     pass: a per-CTA open-addressing hash of (pc*8 + class)
//                     keys in shared memory (two probe slots read up front;
//                     cold keys straight to L2); k_bin_samples (small streams,
//                     warp-aggregated atomics) and the bucketed passes
//                     k_bin_hist/plan/scatter/count; k_bin_finalize sums lat[N]
//                     (map_stall profile.py:106-111, breakdown_at :307-313).
//   incoming CSR      DependencyGraph.incoming (depgraph.py:102-108): raw/guard
//                     edges are consumer-sorted (segment bounds by adjacent-
//                     difference), sync edges producer-sorted (stable counting
//                     sort by consumer); incoming(j) = regular(j) ++ sync(j).
//   k_mp_*            _address_traces_to_load (analysis.py:390-411) for every
//                     instruction: Jacobi rounds over the base RAW graph.
//   k_blame_light /   pass 0 of attribute_blame (analysis.py:431-484): self
//   k_blame_edges /   verdicts (self_blame :414-428) for instructions without
//   k_blame<0>        pruned in-edges, Eq. 1 for the rest in the reference's
//                     exact floating-point order (no FMA contraction, CPython
//                     3.12 sum()); entries staged once.
//   k_blame_compact   entries into stalled order + the per-line FP64 rollup
//                     (k_blame<1> + k_lines in the two-pass A/B mode).
//   k_slice           multi-source backward BFS over pruned incoming edges from
//                     every S_j > 0, level-synchronous in one
//                     cooperative kernel.
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>

#include "prims.cuh"

namespace cg = cooperative_groups;

namespace leo {


// ---- stage 0 ---------------------------------------------------------------
// PACK: 0 = pc / category arrays; 4 = one u32 word per sample, pc << 8 |
// category (4 B per sample instead of 5; kernels below 2^24 instructions);
// 3 = one little-endian 24-bit word per sample, pc << CB | category (3 B per
// sample; kernels of at most 2^(24 - CB) instructions, categories below 2^CB)
LEO_DEV void unpack4(const uint4 w, int4& p, uint32_t& c) {
  p = make_int4((int)(w.x >> 8), (int)(w.y >> 8), (int)(w.z >> 8), (int)(w.w >> 8));
  c = (w.x & 0xFFu) | ((w.y & 0xFFu) << 8) | ((w.z & 0xFFu) << 16) | ((w.w & 0xFFu) << 24);
}
// four 24-bit words from their 12 bytes (three u32 little-endian); CB
// category bits (4, or 5 for Intel's 17 category ids)
template <int CB>
LEO_DEV void unpack4_24(const uint32_t x, const uint32_t y, const uint32_t z, int4& p, uint32_t& c) {
  constexpr uint32_t m = (1u << CB) - 1u;
  const uint32_t w0 = x & 0xFFFFFFu, w1 = (x >> 24) | ((y & 0xFFFFu) << 8);
  const uint32_t w2 = (y >> 16) | ((z & 0xFFu) << 16), w3 = z >> 8;
  p = make_int4((int)(w0 >> CB), (int)(w1 >> CB), (int)(w2 >> CB), (int)(w3 >> CB));
  c = (w0 & m) | ((w1 & m) << 8) | ((w2 & m) << 16) | ((w3 & m) << 24);
}
// one sample of a packed stream (tails)
template <int PACK, int CB>
LEO_DEV void unpack1(const uint32_t* packed, int64_t s, int& j, uint32_t& c) {
  if (PACK == 4) { const uint32_t w = packed[s]; j = (int)(w >> 8); c = w & 0xFFu; return; }
  const uint8_t* b = reinterpret_cast<const uint8_t*>(packed) + 3 * s;
  const uint32_t w = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16);
  j = (int)(w >> CB); c = w & ((1u << CB) - 1u);
}
// the v-th vector of four samples
template <int PACK, int CB>
LEO_DEV void load4(const uint32_t* packed, int64_t v, bool valid, int4& p, uint32_t& c) {
  if (!valid) { p = make_int4(0, 0, 0, 0); c = 0u; return; }
  if (PACK == 4) { unpack4(reinterpret_cast<const uint4*>(packed)[v], p, c); return; }
  const uint32_t* w = packed + 3 * v;
  unpack4_24<CB>(w[0], w[1], w[2], p, c);
}

template <int PACK, int CB = 4>
__global__ void k_bin_samples(int64_t S, const int32_t* __restrict__ pc, const uint8_t* __restrict__ cat,
                              const uint8_t* __restrict__ lut, int N, int32_t* __restrict__ cls_cnt,
                              uint32_t* status, const uint32_t* __restrict__ packed) {
  pdl_wait();
  __shared__ uint8_t slut[256];
  for (int x = threadIdx.x; x < 256; x += blockDim.x) slut[x] = lut[x];
  __syncthreads();
  const int64_t nvec = S / 4;
  const int4* pc4 = reinterpret_cast<const int4*>(pc);
  const uint32_t* cat4 = reinterpret_cast<const uint32_t*>(cat);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v - threadIdx.x < nvec; v += stride) {
    const bool valid = v < nvec;
    int4 p;
    uint32_t c;
    if (PACK) load4<PACK, CB>(packed, v, valid, p, c);
    else { p = valid ? pc4[v] : make_int4(0, 0, 0, 0); c = valid ? cat4[v] : 0u; }
    int pcs[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
    for (int t = 0; t < 4; t++) {
      int j = pcs[t];
      bool ok = valid && j >= 0 && j < N;
      if (valid && !ok) atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT);
      int key = ok ? j * 8 + slut[(c >> (8 * t)) & 0xFF] : -1;
      unsigned grp = __match_any_sync(0xffffffffu, key);
      if (ok && (__ffs(grp) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&cls_cnt[key], __popc(grp));
    }
  }
  // tail
  for (int64_t s = nvec * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += stride) {
    int j;
    uint32_t cb;
    if (PACK) unpack1<PACK, CB>(packed, s, j, cb);
    else { j = pc[s]; cb = cat[s]; }
    if (j < 0 || j >= N) { atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT); continue; }
    atomicAdd(&cls_cnt[j * 8 + slut[cb]], 1);
  }
}

// ---- stage 0, one pass: every CTA streams a contiguous chunk of the samples
// (16-byte pc / 4-byte category loads) and counts (pc * 8 + class) keys in a
// private open-addressing hash in shared memory.  Zipf-hot keys occupy the table early and are counted
// on chip; a key that finds no slot within kBinProbe probes (the cold tail) is
// added to cls_cnt in L2 directly.  The table is flushed with one global atomic
// per occupied slot.  One read of the 5 bytes per sample (vs the bucketed
// passes' hist + scatter + count: ~3 reads and a key write).
constexpr uint32_t kBinEmpty = 0xFFFFFFFFu;
// A/B knob (LEO_BIN_NOGROUP=1, set by the host): the per-vector 3-byte loads
__device__ int g_bin_nogroup;
LEO_DEV bool getenv_bin_nogroup() { return g_bin_nogroup != 0; }

template <int SLOTS, int PROBE, int PACK = 0, int CB = 4>
__global__ void __launch_bounds__(1024) k_bin_hash(int64_t S, const int32_t* __restrict__ pc,
                                                   const uint8_t* __restrict__ cat,
                                                   const uint8_t* __restrict__ lut, int N,
                                                   int32_t* __restrict__ cls_cnt, uint32_t* status,
                                                   const uint32_t* __restrict__ packed = nullptr) {
  pdl_wait();
  extern __shared__ uint32_t hsh[];
  uint32_t* keys = hsh;
  uint32_t* cnts = hsh + SLOTS;
  __shared__ uint8_t slut[256];
  for (int x = threadIdx.x; x < 256; x += blockDim.x) slut[x] = lut[x];
  for (int x = threadIdx.x; x < SLOTS; x += blockDim.x) { keys[x] = kBinEmpty; cnts[x] = 0u; }
  __syncthreads();
  // this CTA's chunk, in whole 4-sample vectors
  const int64_t nvec = S / 4;
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
  const int4* pc4 = reinterpret_cast<const int4*>(pc);
  const uint32_t* cat4 = reinterpret_cast<const uint32_t*>(cat);
  bool bad = false;
  // (no warp aggregation: __match_any_sync cost more than the shared-memory
  // atomics it saves; a hot key's lanes serialise only on their shared counter)
  // Slow path: probe past the home slot, claim an empty slot, or count a cold
  // key in L2.  Fully unrolled, and every vector of four samples ends with a
  // __syncwarp(): a warp left diverged by the probe loop otherwise issues the
  // next vector's loads once per lane group (measured 8x the load requests).
  auto slow = [&](uint32_t key, uint32_t h) {
#pragma unroll
    for (int probe = 0; probe < PROBE; probe++) {
      uint32_t k0 = keys[h];
      if (k0 == kBinEmpty) k0 = atomicCAS(&keys[h], kBinEmpty, key);
      if (k0 == kBinEmpty || k0 == key) { atomicAdd(&cnts[h], 1u); return; }
      h = h + 1 == (uint32_t)SLOTS ? 0u : h + 1;
    }
    atomicAdd(&cls_cnt[key], 1);                         // cold key: straight to L2
  };
  auto vec = [&](const int4 p, const uint32_t c, const bool valid) {
    const int js[4] = {p.x, p.y, p.z, p.w};
    uint32_t key[4], h[4], k0[4], k1[4];
#pragma unroll
    for (int t = 0; t < 4; t++) {                        // both probe slots read up front
      const bool ok = valid && (uint32_t)js[t] < (uint32_t)N;
      bad |= valid && !ok;
      key[t] = ok ? (uint32_t)js[t] * 8u + slut[(c >> (8 * t)) & 0xFF] : kBinEmpty;
      h[t] = __umulhi(key[t] * 2654435761u, (uint32_t)SLOTS);
      k0[t] = keys[h[t]];
      k1[t] = PROBE == 2 ? keys[h[t] + 1 == (uint32_t)SLOTS ? 0u : h[t] + 1] : 0u;
    }
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (key[t] == kBinEmpty) continue;
      if (k0[t] == key[t]) {                             // the hot-key hit
        atomicAdd(&cnts[h[t]], 1u);
      } else if (PROBE == 2 && k1[t] == key[t]) {        // displaced by one slot
        atomicAdd(&cnts[h[t] + 1 == (uint32_t)SLOTS ? 0u : h[t] + 1], 1u);
      } else if (PROBE == 2 && k0[t] != kBinEmpty && k1[t] != kBinEmpty) {
        atomicAdd(&cls_cnt[key[t]], 1);                  // both slots taken: cold key to L2
      } else {
        slow(key[t], h[t]);                              // claim an empty slot (or re-probe)
      }
    }
    __syncwarp();
  };
  // two 16-byte pc loads (and their category words) in flight per thread; the
  // loop is warp-uniform (lanes past the chunk end run as no-ops) so that the
  // __syncwarp() in vec() always sees the full warp
  const int64_t bd = blockDim.x;
  const int lane = threadIdx.x & 31;
  // 3-byte words from a 16-byte-aligned stream: a thread takes 16 samples
  // (48 bytes) as three 16-byte loads instead of twelve 4-byte ones; the
  // chunk's < 4 head and tail vectors outside whole groups go to warp 0
  const bool groups = PACK == 3 && !(reinterpret_cast<uintptr_t>(packed) & 15) && !getenv_bin_nogroup();
  if (PACK == 3 && groups) {
    const int64_t g0 = (v0 + 3) / 4, g1 = v1 / 4;
    const uint4* q = reinterpret_cast<const uint4*>(packed);
    for (int64_t g = g0 + threadIdx.x; g - lane < g1; g += bd) {
      const bool in = g < g1;
      const uint4 zero = make_uint4(0, 0, 0, 0);
      const uint4 a = in ? q[3 * g] : zero, b = in ? q[3 * g + 1] : zero, c = in ? q[3 * g + 2] : zero;
      int4 p;
      uint32_t cc;
      unpack4_24<CB>(a.x, a.y, a.z, p, cc); vec(p, cc, in);
      unpack4_24<CB>(a.w, b.x, b.y, p, cc); vec(p, cc, in);
      unpack4_24<CB>(b.z, b.w, c.x, p, cc); vec(p, cc, in);
      unpack4_24<CB>(c.y, c.z, c.w, p, cc); vec(p, cc, in);
    }
    if (threadIdx.x < 32) {
      const int64_t hmax = min(v1, 4 * g0), tmin = max(hmax, 4 * g1);
      const int64_t v = lane < 4 ? v0 + lane : tmin + (lane - 4);
      const bool in = lane < 4 ? v < hmax : (lane < 8 && v < v1);
      int4 p;
      uint32_t cc;
      load4<PACK, CB>(packed, v, in, p, cc);
      vec(p, cc, in);
    }
  }
  for (int64_t v = v0 + threadIdx.x; !groups && v - lane < v1; v += 2 * bd) {
    const bool in0 = v < v1, in1 = v + bd < v1;
    int4 p0, p1;
    uint32_t c0, c1;
    if (PACK) {
      load4<PACK, CB>(packed, v, in0, p0, c0);
      load4<PACK, CB>(packed, v + bd, in1, p1, c1);
    } else {
      p0 = in0 ? pc4[v] : make_int4(0, 0, 0, 0);
      p1 = in1 ? pc4[v + bd] : make_int4(0, 0, 0, 0);
      c0 = in0 ? cat4[v] : 0u;
      c1 = in1 ? cat4[v + bd] : 0u;
    }
    vec(p0, c0, in0);
    vec(p1, c1, in1);
  }
  // tail samples (S mod 4): the last CTA
  if (blockIdx.x == gridDim.x - 1) {
    const int64_t s = nvec * 4 + threadIdx.x;
    if (s < S) {
      int j;
      uint32_t cb;
      if (PACK) unpack1<PACK, CB>(packed, s, j, cb);
      else { j = pc[s]; cb = cat[s]; }
      const bool ok = (uint32_t)j < (uint32_t)N;
      bad |= !ok;
      if (ok) atomicAdd(&cls_cnt[(uint32_t)j * 8u + slut[cb]], 1);
    }
  }
  if (bad) atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT);
  __syncthreads();
  for (int x = threadIdx.x; x < SLOTS; x += blockDim.x)
    if (keys[x] != kBinEmpty) atomicAdd(&cls_cnt[keys[x]], (int)cnts[x]);
}

// ---- stage 0, bucketed: samples are partitioned by pc / R into NB buckets
// (R instructions x 8 classes of u32 counters fit in shared memory), packed to
// u16 keys ((pc mod R) * 8 + class), then each (bucket, slice) is counted in
// shared memory with warp-aggregated atomics and merged into cls_cnt.  Hot
// buckets (Zipf-heavy PCs) are split over many CTAs, so no counter sees more
// than one global atomic per CTA.
constexpr int kBinR = 2048;          // default instructions per bucket (64 KiB of counters)
constexpr int kBinRMax = 4096;       // 128 KiB of counters: up to 16.7M instructions
constexpr int kBinMaxBuckets = 4096;

// chunk c of the sample stream = [c*per, min(S, (c+1)*per)), per a multiple of 4
LEO_DEV int64_t bin_chunk_per(int64_t S, int G) { return (((S + G - 1) / G) + 3) & ~(int64_t)3; }

// pass 1: chunk-local bucket histogram -> M[c * nb + b]
__global__ void __launch_bounds__(512) k_bin_hist(int64_t S, const int32_t* __restrict__ pc, int N, int nb, int R,
                                                  int32_t* __restrict__ M, uint32_t* status) {
  pdl_wait();
  extern __shared__ int32_t h[];                 // nb
  for (int x = threadIdx.x; x < nb; x += blockDim.x) h[x] = 0;
  __syncthreads();
  const int64_t per = bin_chunk_per(S, gridDim.x);
  const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(S, s0 + per);
  if (s0 < s1) {
    const int64_t v0 = s0 / 4, v1 = s1 / 4;     // s0 is a multiple of 4
    const int4* pc4 = reinterpret_cast<const int4*>(pc);
    // four 16-byte loads in flight per thread
    const int64_t step = (int64_t)blockDim.x;
    int64_t v = v0 + threadIdx.x;
    for (; v + 3 * step < v1; v += 4 * step) {
      int4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = pc4[v + u * step];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int ps[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const int j = ps[t];
          if (j < 0 || j >= N) { atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT); continue; }
          atomicAdd(&h[j / R], 1);
        }
      }
    }
    for (; v < v1; v += step) {
      const int4 p = pc4[v];
      const int ps[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int j = ps[t];
        if (j < 0 || j >= N) { atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT); continue; }
        atomicAdd(&h[j / R], 1);
      }
    }
    for (int64_t x = v1 * 4 + threadIdx.x; x < s1; x += blockDim.x) {
      const int j = pc[x];
      if (j < 0 || j >= N) { atomicOr(status, (uint32_t)LEO_ST_BAD_INPUT); continue; }
      atomicAdd(&h[j / R], 1);
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < nb; x += blockDim.x) M[(size_t)blockIdx.x * nb + x] = h[x];
}

// pass 2a: CTA per bucket: exclusive scan of the bucket's chunk counts in
// place (M[c][b] becomes the chunk's offset inside the bucket) + bucket total
__global__ void k_bin_colscan(int nb, int G, int32_t* __restrict__ M, int32_t* __restrict__ tot) {
  pdl_wait();
  __shared__ int sw[33];
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    int carry = 0;
    for (int base = 0; base < G; base += blockDim.x) {
      const int c = base + threadIdx.x;
      const int v = c < G ? M[(size_t)c * nb + b] : 0;
      int t;
      const int ex = block_excl_scan(v, sw, &t);
      if (c < G) M[(size_t)c * nb + b] = carry + ex;
      carry += t;
    }
    if (threadIdx.x == 0) tot[b] = carry;
  }
}

// pass 2b (single CTA): bucket offsets + slice offsets
__global__ void k_bin_plan(int nb, int slice, const int32_t* __restrict__ bucket_cnt, int32_t* __restrict__ bucket_off,
                           int32_t* __restrict__ slice_off) {
  pdl_wait();
  __shared__ int sw[33];
  int carry = 0, scarry = 0;
  for (int base = 0; base < nb; base += blockDim.x) {
    int i = base + threadIdx.x;
    int c = i < nb ? bucket_cnt[i] : 0;
    int ns = (c + slice - 1) / slice;
    int tot, stot;
    int ex = block_excl_scan(c, sw, &tot);
    int sex = block_excl_scan(ns, sw, &stot);
    if (i < nb) { bucket_off[i] = carry + ex; slice_off[i] = scarry + sex; }
    carry += tot; scarry += stot;
  }
  if (threadIdx.x == 0) { bucket_off[nb] = carry; slice_off[nb] = scarry; }
}

// pass 3: scatter u16 keys ((pc mod R) * 8 + class) into bucket ranges.
// A sample-by-sample scatter writes one 2-byte key per 32-byte sector (16x
// write amplification at 100 M samples).  Instead each CTA sorts sub-chunks
// of kBinSub samples by bucket in shared memory (histogram, scan, local
// scatter) and copies every bucket's run out contiguously, so consecutive
// threads write consecutive keys.
constexpr int kBinSub = 8192;

__global__ void __launch_bounds__(512) k_bin_scatter(int64_t S, const int32_t* __restrict__ pc, const uint8_t* __restrict__ cat,
                                                     const uint8_t* __restrict__ lut, int N, int nb, int R,
                                                     const int32_t* __restrict__ M, const int32_t* __restrict__ bucket_off,
                                                     uint16_t* __restrict__ keys) {
  pdl_wait();
  extern __shared__ int32_t dyn[];
  int32_t* cur = dyn;                            // nb: global cursor per bucket (this chunk)
  int32_t* lcnt = dyn + nb;                      // nb: sub-chunk histogram, then local offsets
  int32_t* lpos = lcnt + nb;                     // nb: local fill cursors
  uint16_t* lkey = reinterpret_cast<uint16_t*>(lpos + nb);      // kBinSub keys
  uint16_t* lbkt = lkey + kBinSub;                              // kBinSub buckets
  __shared__ uint8_t slut[256];
  __shared__ int sw[33];
  for (int x = threadIdx.x; x < nb; x += blockDim.x) cur[x] = bucket_off[x] + M[(size_t)blockIdx.x * nb + x];
  for (int x = threadIdx.x; x < 256; x += blockDim.x) slut[x] = lut[x];
  const int64_t per = bin_chunk_per(S, gridDim.x);
  const int64_t s0 = (int64_t)blockIdx.x * per, s1 = min(S, s0 + per);
  for (int64_t c0 = s0; c0 < s1; c0 += kBinSub) {
    const int n = (int)min((int64_t)kBinSub, s1 - c0);
    for (int x = threadIdx.x; x < nb; x += blockDim.x) lcnt[x] = 0;
    __syncthreads();
    // histogram of the sub-chunk (c0 is a multiple of 4: int4 loads)
    const int nv = n / 4;
    const int4* pc4 = reinterpret_cast<const int4*>(pc + c0);
    const uint32_t* cat4 = reinterpret_cast<const uint32_t*>(cat + c0);
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const int4 p = pc4[v];
      const int ps[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (ps[t] >= 0 && ps[t] < N) atomicAdd(&lcnt[ps[t] / R], 1);
    }
    for (int x = nv * 4 + threadIdx.x; x < n; x += blockDim.x) {
      const int j = pc[c0 + x];
      if (j >= 0 && j < N) atomicAdd(&lcnt[j / R], 1);
    }
    __syncthreads();
    // local offsets (exclusive scan over buckets, thread-contiguous chunks)
    {
      const int pb = (nb + blockDim.x - 1) / blockDim.x, lo = min(nb, (int)threadIdx.x * pb), hi = min(nb, lo + pb);
      int sum = 0;
      for (int x = lo; x < hi; x++) sum += lcnt[x];
      int tot;
      int run = block_excl_scan(sum, sw, &tot);
      for (int x = lo; x < hi; x++) { const int v = lcnt[x]; lcnt[x] = run; lpos[x] = run; run += v; }
    }
    __syncthreads();
    // local scatter into shared memory
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const int4 p = pc4[v];
      const uint32_t c = cat4[v];
      const int ps[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int j = ps[t];
        if (j < 0 || j >= N) continue;
        const int b = j / R;
        const int q = atomicAdd(&lpos[b], 1);
        lkey[q] = (uint16_t)(((j - b * R) << 3) | slut[(c >> (8 * t)) & 0xFF]);
        lbkt[q] = (uint16_t)b;
      }
    }
    for (int x = nv * 4 + threadIdx.x; x < n; x += blockDim.x) {
      const int j = pc[c0 + x];
      if (j < 0 || j >= N) continue;
      const int b = j / R;
      const int q = atomicAdd(&lpos[b], 1);
      lkey[q] = (uint16_t)(((j - b * R) << 3) | slut[cat[c0 + x]]);
      lbkt[q] = (uint16_t)b;
    }
    __syncthreads();
    // runs out: element q of bucket b lands at cur[b] + (q - lcnt[b])
    const int nk = lpos[nb - 1] > 0 ? lpos[nb - 1] : 0;   // valid keys = end of the last bucket
    for (int q = threadIdx.x; q < nk; q += blockDim.x) {
      const int b = lbkt[q];
      keys[cur[b] + (q - lcnt[b])] = lkey[q];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nb; x += blockDim.x) cur[x] += lpos[x] - lcnt[x];
    __syncthreads();
  }
}

// pass 4: count each (bucket, slice) in shared memory, merge into cls_cnt
__global__ void __launch_bounds__(512) k_bin_count(int N, int nb, int R, int slice, const int32_t* __restrict__ bucket_off,
                                                   const int32_t* __restrict__ slice_off,
                                                   const uint16_t* __restrict__ keys,
                                                   int32_t* __restrict__ cls_cnt) {
  pdl_wait();
  extern __shared__ int32_t cnt[];              // R * 8
  const int total_slices = slice_off[nb];
  for (int sl = blockIdx.x; sl < total_slices; sl += gridDim.x) {
    int lo = 0, hi = nb - 1;                      // bucket: largest b with slice_off[b] <= sl
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (slice_off[mid] <= sl) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int k = sl - slice_off[b];
    const int64_t e0 = (int64_t)bucket_off[b] + (int64_t)k * slice;
    const int64_t e1 = min((int64_t)bucket_off[b + 1], e0 + slice);
    for (int x = threadIdx.x; x < R * 8; x += blockDim.x) cnt[x] = 0;
    __syncthreads();
    // aligned body: 8 keys per uint4
    const int64_t a0 = min(e1, (e0 + 7) & ~(int64_t)7), a1 = max(a0, e1 & ~(int64_t)7);
    for (int64_t e = e0 + threadIdx.x; e < a0; e += blockDim.x) atomicAdd(&cnt[keys[e]], 1);
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    for (int64_t v = a0 / 8 + threadIdx.x; v < a1 / 8; v += blockDim.x) {
      const uint4 q = k4[v];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int t = 0; t < 4; t++) {
        atomicAdd(&cnt[w[t] & 0xFFFF], 1);
        atomicAdd(&cnt[w[t] >> 16], 1);
      }
    }
    for (int64_t e = a1 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&cnt[keys[e]], 1);
    __syncthreads();
    const int64_t base = (int64_t)b * R * 8;
    const int lim = (int)min((int64_t)R * 8, ((int64_t)N - (int64_t)b * R) * 8);
    for (int x = threadIdx.x; x < lim; x += blockDim.x)
      if (cnt[x]) atomicAdd(&cls_cnt[base + x], cnt[x]);
    __syncthreads();
  }
}

__global__ void k_bin_finalize(int N, const int32_t* __restrict__ cls_cnt, int32_t* __restrict__ lat) {
  pdl_wait();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
    const int4* row = reinterpret_cast<const int4*>(cls_cnt + (size_t)j * 8);
    int4 a = row[0], b = row[1];
    lat[j] = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
}

// ---- incoming CSR ------------------------------------------------------------
// regular (raw/guard) edges [0, n_reg) are sorted by consumer
__global__ void k_seg_bounds(const int32_t* __restrict__ cons, const int32_t* n_reg_dev,
                             int32_t* __restrict__ rbeg, int32_t* __restrict__ rend) {
  pdl_wait();
  const int n = *n_reg_dev;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    int c = cons[e];
    if (e == 0 || cons[e - 1] != c) rbeg[c] = e;
    if (e == n - 1 || cons[e + 1] != c) rend[c] = e + 1;
  }
}
// sync edges [n_reg, n) : histogram by consumer
__global__ void k_sync_hist(const int32_t* __restrict__ cons, const int32_t* n_reg_dev, const int32_t* n_dev,
                            int32_t* __restrict__ cnt) {
  pdl_wait();
  const int r = *n_reg_dev, n = *n_dev;
  for (int e = r + blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    atomicAdd(&cnt[cons[e]], 1);
}
__global__ void k_sync_fill(const int32_t* __restrict__ cons, const int32_t* n_reg_dev, const int32_t* n_dev,
                            const int32_t* __restrict__ off, int32_t* __restrict__ cursor,
                            uint64_t* __restrict__ out) {
  pdl_wait();
  const int r = *n_reg_dev, n = *n_dev;
  for (int e = r + blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    int c = cons[e];
    out[off[c] + atomicAdd(&cursor[c], 1)] = (uint64_t)(uint32_t)e;
  }
}

struct Incoming {
  const int32_t* rbeg;      // [N] regular edge range (rbeg == rend when none)
  const int32_t* rend;
  const int32_t* soff;      // [N+1] sync edge list offsets
  const uint64_t* sidx;     // sync edge indices (sorted per consumer = edge-list order)
  LEO_DEV int deg(int j) const { return (rend[j] - rbeg[j]) + (soff[j + 1] - soff[j]); }
  LEO_DEV int edge(int j, int x) const {
    int r = rend[j] - rbeg[j];
    return x < r ? rbeg[j] + x : (int)sidx[soff[j] + (x - r)];
  }
};

// ---- self blame ----------------------------------------------------------------
__constant__ static const int kMatchClass[3] = {LEO_CS_MEMORY_DEP, LEO_CS_EXECUTION_DEP, LEO_CS_SYNCHRONIZATION};
__constant__ static const int kSelfByClass[8] = {LEO_SB_MEMORY_LATENCY, LEO_SB_COMPUTE_SATURATION,
    LEO_SB_SYNCHRONIZATION_OVERHEAD, LEO_SB_INSTRUCTION_FETCH, LEO_SB_PIPELINE_CONTENTION,
    LEO_SB_PIPELINE_CONTENTION, LEO_SB_PIPELINE_CONTENTION, LEO_SB_PIPELINE_CONTENTION};

// _address_traces_to_load on the base graph's RAW edges (regular part only:
// sync edges are never RAW).  Returns 1/0, or -1 when `seen` overflowed.
LEO_DEV int traces_to_load(const KView& k, const int32_t* brbeg, const int32_t* brend,
                           const int32_t* bprod, const uint32_t* bmeta, int index,
                           int32_t* seen, int cap, int32_t* stamp, int stamp_val) {
  // seen[0..n) holds visited nodes in BFS order; frontier = seen[lo..hi)
  int n = 1, lo = 0, hi = 1;
  seen[0] = index;
  if (stamp) stamp[index] = stamp_val;
  // 64-bit presence filter in a register: most discoveries are new and skip
  // the linear scan of `seen` (local memory) entirely
  uint64_t filt = 1ull << (((uint32_t)index * 2654435761u) >> 26);
  for (int depth = 0; depth < 8; depth++) {
    for (int a = lo; a < hi; a++) {
      const int node = seen[a];
      for (int e = brbeg[node]; e < brend[node]; e++) {
        if (((bmeta[e] >> 27) & 7) != LEO_EK_RAW) continue;
        const int p = bprod[e];
        bool dup = false;
        const uint64_t fb = 1ull << (((uint32_t)p * 2654435761u) >> 26);
        if (stamp) dup = stamp[p] == stamp_val;
        else if (filt & fb) for (int x = 0; x < n; x++) if (seen[x] == p) { dup = true; break; }
        if (dup) continue;
        if (kMemoryProducer & BIT(k.opclass[p])) return 1;
        if (n == cap) return -1;
        seen[n++] = p;
        filt |= fb;
        if (stamp) stamp[p] = stamp_val;
      }
    }
    if (n == hi) return 0;
    lo = hi; hi = n;
  }
  return 0;
}

// ---- _address_traces_to_load for every instruction at once -------------------
// The reference BFS (analysis.py:390-411) answers: is some MEMORY_PRODUCER q
// other than j within 8 RAW hops of j, through intermediates that are not
// memory producers?  That is a shortest-path question, so it is computed for
// all nodes by 7 rounds of Jacobi relaxation over the base graph's RAW
// incoming edges, keeping per node the two nearest producer targets with
// distinct ids (the second one answers "nearest target != j" for a load j),
// then one evaluation round.  Runs on a side branch beside pruning.
constexpr uint8_t kMpInf = 99;
// Labels pack (distance << 24 | target) in one 32-bit word per candidate
// (target -1 -> 0xFFFFFF); a node's two candidates are one 8-byte load.
// The RAW in-edges are first rewritten as one word per base edge (producer
// id, flagged when it is a memory producer; -1 for other kinds), so a round
// issues its edge loads and then its label loads independently.
constexpr uint32_t kMpT = 0xFFFFFFu, kMpPF = 0x40000000u;
LEO_DEV uint32_t mp_pack(int d, int t) { return ((uint32_t)d << 24) | ((uint32_t)t & kMpT); }
LEO_DEV int mp_d(uint32_t w) { return (int)(w >> 24); }
LEO_DEV int mp_t(uint32_t w) { const uint32_t t = w & kMpT; return t == kMpT ? -1 : (int)t; }

LEO_DEV void mp_insert(int d, int t, int& D1, int& T1, int& D2, int& T2) {
  if (t == T1) { if (d < D1) D1 = d; return; }
  if (d < D1) { D2 = D1; T2 = T1; D1 = d; T1 = t; return; }
  if (t == T2) { if (d < D2) D2 = d; return; }
  if (d < D2) { D2 = d; T2 = t; }
}

__global__ void k_mp_edges(KView k, const int32_t* __restrict__ n_regular, int64_t cap,
                           const int32_t* __restrict__ bprod, const uint32_t* __restrict__ bmeta,
                           int32_t* __restrict__ ep) {
  pdl_wait();
  const int64_t n = min((int64_t)*n_regular, cap);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int w = -1;
    if (((bmeta[e] >> 27) & 7) == LEO_EK_RAW) {
      const int p = bprod[e];
      w = (kMemoryProducer & BIT(k.opclass[p])) ? (int)(p | kMpPF) : p;
    }
    ep[e] = w;
  }
}

constexpr int kMpUnroll = 4;

__global__ void k_mp_round(KView k, const int32_t* __restrict__ rbeg, const int32_t* __restrict__ rend,
                           const int32_t* __restrict__ ep, const uint2* __restrict__ in,
                           uint2* __restrict__ out, int first) {
  pdl_wait();
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < k.N; v += gridDim.x * blockDim.x) {
    int D1 = kMpInf, T1 = -1, D2 = kMpInf, T2 = -1;
    if (!(kMemoryProducer & BIT(k.opclass[v]))) {            // producers never relay
      const int e1 = rend[v];
      for (int e = rbeg[v]; e < e1; e += kMpUnroll) {
        int q[kMpUnroll];
        uint2 L[kMpUnroll];
#pragma unroll
        for (int x = 0; x < kMpUnroll; x++) q[x] = e + x < e1 ? ep[e + x] : -1;
#pragma unroll
        for (int x = 0; x < kMpUnroll; x++)
          L[x] = (!first && q[x] >= 0 && !(q[x] & kMpPF)) ? in[q[x]] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
#pragma unroll
        for (int x = 0; x < kMpUnroll; x++) {
          if (q[x] < 0) continue;
          if (q[x] & kMpPF) { mp_insert(1, (int)(q[x] & ~kMpPF), D1, T1, D2, T2); continue; }
          if (first) continue;
          if (mp_d(L[x].x) < 8) mp_insert(mp_d(L[x].x) + 1, mp_t(L[x].x), D1, T1, D2, T2);
          if (mp_d(L[x].y) < 8) mp_insert(mp_d(L[x].y) + 1, mp_t(L[x].y), D1, T1, D2, T2);
        }
      }
    }
    out[v] = make_uint2(mp_pack(D1, T1), mp_pack(D2, T2));
  }
}

__global__ void k_mp_final(KView k, const int32_t* __restrict__ rbeg, const int32_t* __restrict__ rend,
                           const int32_t* __restrict__ ep, const uint2* __restrict__ lab,
                           uint8_t* __restrict__ ok) {
  pdl_wait();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k.N; j += gridDim.x * blockDim.x) {
    bool hit = false;
    const int e1 = rend[j];
    for (int e = rbeg[j]; e < e1 && !hit; e += kMpUnroll) {
      int q[kMpUnroll];
      uint2 L[kMpUnroll];
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++) q[x] = e + x < e1 ? ep[e + x] : -1;
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++)
        L[x] = (q[x] >= 0 && !(q[x] & kMpPF)) ? lab[q[x]] : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++) {
        if (hit || q[x] < 0) continue;
        if (q[x] & kMpPF) { hit = (int)(q[x] & ~kMpPF) != j; continue; }
        const int d = mp_t(L[x].x) != j ? mp_d(L[x].x) : mp_d(L[x].y);   // nearest target other than j
        hit = d + 1 <= 8;
      }
    }
    ok[j] = hit ? 1 : 0;
  }
}

// All rounds in one cooperative kernel, relaxing IN PLACE (Gauss-Seidel):
// a label is always the top-2 of real paths of <= 8 hops, so it only
// decreases and its fixpoint is the Jacobi result; rounds stop at the first
// one that changes nothing (<= 7 relaxations, the Jacobi bound), then the
// evaluation round.  flags[3]: "changed" per round, reset two rounds ahead.
LEO_DEV uint2 mp_relax(const KView& k, const int32_t* __restrict__ rbeg, const int32_t* __restrict__ rend,
                       const int32_t* __restrict__ ep, const uint2* lab, int v, bool first) {
  int D1 = kMpInf, T1 = -1, D2 = kMpInf, T2 = -1;
  if (!(kMemoryProducer & BIT(k.opclass[v]))) {
    const int e1 = rend[v];
    for (int e = rbeg[v]; e < e1; e += kMpUnroll) {
      int q[kMpUnroll];
      uint2 L[kMpUnroll];
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++) q[x] = e + x < e1 ? ep[e + x] : -1;
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++)
        L[x] = (!first && q[x] >= 0 && !(q[x] & kMpPF)) ? __ldcg(&lab[q[x]])   // L2: other SMs' writes
                                                         : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
#pragma unroll
      for (int x = 0; x < kMpUnroll; x++) {
        if (q[x] < 0) continue;
        if (q[x] & kMpPF) { mp_insert(1, (int)(q[x] & ~kMpPF), D1, T1, D2, T2); continue; }
        if (first) continue;
        if (mp_d(L[x].x) < 8) mp_insert(mp_d(L[x].x) + 1, mp_t(L[x].x), D1, T1, D2, T2);
        if (mp_d(L[x].y) < 8) mp_insert(mp_d(L[x].y) + 1, mp_t(L[x].y), D1, T1, D2, T2);
      }
    }
  }
  return make_uint2(mp_pack(D1, T1), mp_pack(D2, T2));
}

__global__ void k_mp_coop(KView k, const int32_t* __restrict__ rbeg, const int32_t* __restrict__ rend,
                          const int32_t* __restrict__ ep, uint2* lab, int32_t* flags, uint8_t* __restrict__ ok) {
  cg::grid_group grid = cg::this_grid();
  const int stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int r = 0; r < 7; r++) {
    if (t0 == 0) flags[(r + 1) % 3] = 0;
    bool changed = false;
    for (int v = t0; v < k.N; v += stride) {
      const uint2 nl = mp_relax(k, rbeg, rend, ep, lab, v, r == 0);
      if (r == 0) { __stcg(&lab[v], nl); continue; }
      const uint2 ol = __ldcg(&lab[v]);
      if (nl.x != ol.x || nl.y != ol.y) { __stcg(&lab[v], nl); changed = true; }
    }
    if (changed) flags[r % 3] = 1;
    grid.sync();
    if (r > 0 && *(volatile int32_t*)&flags[r % 3] == 0) break;
  }
  for (int j = t0; j < k.N; j += stride) {
    bool hit = false;
    const int e1 = rend[j];
    for (int e = rbeg[j]; e < e1 && !hit; e++) {
      const int q = ep[e];
      if (q < 0) continue;
      if (q & kMpPF) { hit = (int)(q & ~kMpPF) != j; continue; }
      const uint2 L = __ldcg(&lab[q]);
      const int d = mp_t(L.x) != j ? mp_d(L.x) : mp_d(L.y);   // nearest target other than j
      hit = d + 1 <= 8;
    }
    ok[j] = hit ? 1 : 0;
  }
}

struct BlameArgs {
  int32_t dbg;
  const uint8_t* mp_ok;       // per-instruction _address_traces_to_load (null: search here)
  Range own;
  PView p;
  const int32_t* pprod;
  const uint32_t* pmeta;
  const double* pdist;
  Incoming inc;
  const int32_t* brbeg;     // base graph regular incoming
  const int32_t* brend;
  const int32_t* bprod;
  const uint32_t* bmeta;
  int32_t* ecount;          // [N] entries per instruction (pass 0)
  int32_t* self_sub;        // [N] subcategory for self entries (-1 when edges)
  double* jtotal;           // [N] cached normaliser
  double* jnsum;            // [N]
  const int32_t* eoff;      // [N+1] (pass 1)
  LeoBlame out;
  int32_t* slow_list;
  int32_t* slow_count;
  int64_t slow_cap;
  uint32_t* status;
  double* zero_lb;          // pass 0 also zeroes the line vectors (null: accumulate / no lines)
  double* zero_ls;
  int32_t n_lines;
  // edge entries staged by pass 0 (any order; k_blame_compact moves them into
  // stalled-instruction order): j's entries at stg_off[j] .. + ecount[j]
  int32_t* stg_off;         // [N]
  int32_t* stg_count;       // reservation counter
  int64_t stg_cap;
  int32_t* stg_edge;
  int32_t* stg_cause;
  double* stg_blame;        // product until the normaliser is known, then blame_cycles
  double* stg_fac;          // [4 x]
};

// warp-aggregated reservation of n staging slots (divergent callers)
LEO_DEV int stage_reserve(const BlameArgs& a, int n) {
  cg::coalesced_group g = cg::coalesced_threads();
  const int incl = cg::inclusive_scan(g, n);
  int base = 0;
  if (g.thread_rank() == g.size() - 1) base = atomicAdd(a.stg_count, incl);
  base = g.shfl(base, g.size() - 1);
  const int o = base + incl - n;
  if ((int64_t)o + n > a.stg_cap) { atomicOr(a.status, (uint32_t)LEO_ST_BLAME_OVERFLOW); return -1; }
  return o;
}

LEO_DEV double issue_count(const PView& p, int i) {   // profile.py:321-329
  if (p.exec_cnt[i] >= 0) return (double)p.exec_cnt[i];
  if (p.sampled[i]) return (double)(p.total[i] >= 0 ? p.total[i] : p.lat[i]);
  return 1.0;
}

LEO_DEV int dominant_self(const PView& p, int j) {     // _dominant_class :379-387
  int dom = 0, best = -1;
  for (int c = 0; c < 8; c++) {
    int v = p.cls_cnt[(size_t)j * 8 + c];
    if (v > best) { best = v; dom = c; }
  }
  return kSelfByClass[dom];
}

constexpr int kSeenCap = 24;

// issue_count with its loads issued together (no dependent branch on exec_cnt)
LEO_DEV double issue_count_ld(const PView& p, int i) {
  const int64_t ec = p.exec_cnt[i];
  const uint8_t sm = p.sampled[i];
  const int32_t tt = p.total[i], lt = p.lat[i];
  if (ec >= 0) return (double)ec;
  if (sm) return (double)(tt >= 0 ? tt : lt);
  return 1.0;
}

// The per-edge operands of one stalled instruction, loaded kBU edges at a
// time (independent loads), consumed in edge order so every floating-point
// sum keeps the reference's order.
constexpr int kBU = 4;
struct EdgeBatch {
  int e[kBU], pr[kBU], cls[kBU];
  double d[kBU], ef[kBU], ic[kBU];
  LEO_DEV void load(const BlameArgs& a, int j, int r0, int nr, int s0, int deg, int x0, bool with_cls) {
#pragma unroll
    for (int u = 0; u < kBU; u++) {
      const int x = x0 + u;
      e[u] = x < deg ? (x < nr ? r0 + x : (int)a.inc.sidx[s0 + (x - nr)]) : -1;
    }
#pragma unroll
    for (int u = 0; u < kBU; u++) {
      pr[u] = 0; d[u] = 1.0; cls[u] = 0;
      if (e[u] >= 0) {
        pr[u] = a.pprod[e[u]];
        d[u] = a.pdist[e[u]];
        if (with_cls) cls[u] = kMatchClass[(a.pmeta[e[u]] >> 30) & 3];
      }
    }
#pragma unroll
    for (int u = 0; u < kBU; u++) {
      ef[u] = 1.0; ic[u] = 0.0;
      if (e[u] >= 0) {
        ef[u] = a.p.eff[pr[u]];
        ic[u] = issue_count_ld(a.p, pr[u]);
        if (with_cls) cls[u] = a.p.cls_cnt[(size_t)j * 8 + cls[u]];
      }
    }
  }
};

// self verdict of stalled instruction j (dominant class, indirect addressing)
LEO_DEV void blame_self(const KView& k, const BlameArgs& a, int j) {
  int sub = dominant_self(a.p, j);
  if (sub == LEO_SB_MEMORY_LATENCY && (kMemoryClasses & BIT(k.opclass[j])) && a.mp_ok) {
    if (a.mp_ok[j]) sub = LEO_SB_INDIRECT_ADDRESSING;
  } else if (sub == LEO_SB_MEMORY_LATENCY && (kMemoryClasses & BIT(k.opclass[j]))) {
    // _address_traces_to_load: small searches inline (<= kSeenCap nodes),
    // larger ones in k_selfblame_warp (warp per candidate)
    int32_t seen[kSeenCap];
    const int r = (a.dbg & LEO_DBG_SELF_SLOW) ? -1
                  : traces_to_load(k, a.brbeg, a.brend, a.bprod, a.bmeta, j, seen, kSeenCap, nullptr, 0);
    if (r < 0) {
      int s2 = atomicAdd(a.slow_count, 1);
      if (s2 < a.slow_cap) a.slow_list[s2] = j;
      else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
    } else if (r) {
      sub = LEO_SB_INDIRECT_ADDRESSING;
    }
  }
  a.self_sub[j] = sub;
  a.ecount[j] = 1;
}

// Stalled instructions with more than kBlameWarpDeg incoming edges (a
// waitcnt consumer can have hundreds of sync producers) are done by the whole
// warp: lanes load and evaluate edges in parallel, and every lane replays the
// ordered sums / first-minimum scans through shuffles, so the floating-point
// order is the reference's.
constexpr int kBlameWarpDeg = 12;

// one instruction, thread path; returns true when the warp path must take it
template <int PASS>
LEO_DEV bool blame_one(const KView& k, const BlameArgs& a, int j) {
  {
    const int lat = a.p.lat[j];
    const double s_j = (double)((int64_t)lat * a.p.period);
    if (PASS == 0) { a.ecount[j] = 0; a.self_sub[j] = -1; }
    if (s_j == 0 || !a.own.has(j)) return false;
    const int r0 = a.inc.rbeg[j], nr = a.inc.rend[j] - r0, s0 = a.inc.soff[j];
    const int deg = nr + (a.inc.soff[j + 1] - s0);
    if (deg > kBlameWarpDeg && (PASS == 0 || a.self_sub[j] < 0)) return true;
    if (PASS == 1 && a.self_sub[j] >= 0) {
      const int o = a.eoff[j];
      if (o + 1 > a.out.capacity) { atomicOr(a.status, (uint32_t)LEO_ST_BLAME_OVERFLOW); return false; }
      a.out.stalled[o] = j;
      a.out.edge[o] = -1;
      if (a.out.cause) { a.out.cause[o] = -1; a.out.meta[o] = 0u; }
      a.out.sub[o] = (uint8_t)a.self_sub[j];
      a.out.blame[o] = s_j;
      for (int c = 0; c < 4; c++) a.out.factors[(size_t)o * 4 + c] = 0.0;
      return false;
    }
    bool self = deg == 0;
    double total = 0.0, n_sum = 0.0, d_min = 0, e_min = 0;
    if (!self) {
      PySum ns;
      for (int x0 = 0; x0 < deg; x0 += kBU) {
        EdgeBatch eb;
        eb.load(a, j, r0, nr, s0, deg, x0, false);
#pragma unroll
        for (int u = 0; u < kBU; u++) {
          if (eb.e[u] < 0) continue;
          if (x0 + u == 0 || eb.d[u] < d_min) d_min = eb.d[u];
          if (x0 + u == 0 || eb.ef[u] < e_min) e_min = eb.ef[u];
          if (PASS == 0) ns.add(eb.ic[u]);
        }
      }
      if (PASS == 0) n_sum = ns.value();
      else { total = a.jtotal[j]; n_sum = a.jnsum[j]; }
      if (PASS == 0 && n_sum == 0) self = true;
      else {
        const bool stg = PASS == 0 && a.stg_cap > 0;
        const int o = PASS == 1 ? a.eoff[j] : stg ? stage_reserve(a, deg) : 0;
        if (PASS == 0 && o < 0) return false;
        if (PASS == 1 && o + a.ecount[j] > a.out.capacity) { atomicOr(a.status, (uint32_t)LEO_ST_BLAME_OVERFLOW); return false; }
        PySum ts;
        for (int x0 = 0; x0 < deg; x0 += kBU) {
          EdgeBatch eb;
          eb.load(a, j, r0, nr, s0, deg, x0, true);
#pragma unroll
          for (int u = 0; u < kBU; u++) {
            if (eb.e[u] < 0) continue;
            const double f0 = __ddiv_rn(d_min, eb.d[u]);
            const double f1 = __ddiv_rn(e_min, eb.ef[u]);
            const double f2 = __ddiv_rn(eb.ic[u], n_sum);
            const double f3 = __ddiv_rn((double)eb.cls[u], (double)lat);
            const double prod = __dmul_rn(__dmul_rn(__dmul_rn(f0, f1), f2), f3);
            if (PASS == 0) {
              ts.add(prod);
              const int x = o + x0 + u;
              if (stg) {
              a.stg_edge[x] = eb.e[u];
              a.stg_cause[x] = eb.pr[u];
              a.stg_blame[x] = prod;
              double* f = a.stg_fac + (size_t)x * 4;
              f[0] = f0; f[1] = f1; f[2] = f2; f[3] = f3;
              }
            } else {
              const int x = o + x0 + u;
              a.out.stalled[x] = j;
              a.out.edge[x] = eb.e[u];
              if (a.out.cause) { a.out.cause[x] = eb.pr[u]; a.out.meta[x] = a.pmeta[eb.e[u]]; }
              a.out.sub[x] = 255;
              a.out.blame[x] = __ddiv_rn(__dmul_rn(s_j, prod), total);
              double* f = a.out.factors + (size_t)x * 4;
              f[0] = f0; f[1] = f1; f[2] = f2; f[3] = f3;
            }
          }
        }
        if (PASS == 0) {
          total = ts.value();
          if (total == 0.0) self = true;
          else if (stg) {
            a.stg_off[j] = o;
            for (int x = o; x < o + deg; x++) a.stg_blame[x] = __ddiv_rn(__dmul_rn(s_j, a.stg_blame[x]), total);
          }
        }
      }
    }
    if (PASS == 1) return false;
    if (self) {
      blame_self(k, a, j);
    } else {
      a.ecount[j] = deg;
      a.jtotal[j] = total;
      a.jnsum[j] = n_sum;
    }
  }
  return false;
}

template <int PASS>
LEO_DEV void blame_warp(const KView& k, const BlameArgs& a, int j, int lane) {
  const int lat = a.p.lat[j];
  const double s_j = (double)((int64_t)lat * a.p.period);
  const int r0 = a.inc.rbeg[j], nr = a.inc.rend[j] - r0, s0 = a.inc.soff[j];
  const int deg = nr + (a.inc.soff[j + 1] - s0);
  const int o = PASS == 1 ? a.eoff[j] : 0;
  if (PASS == 1 && o + a.ecount[j] > a.out.capacity) {
    if (lane == 0) atomicOr(a.status, (uint32_t)LEO_ST_BLAME_OVERFLOW);
    return;
  }
  // first minima (x == 0 || v < min) and the issue-count sum, in edge order
  double d_min = 0, e_min = 0;
  PySum ns;
  for (int x0 = 0; x0 < deg; x0 += 32) {
    const int x = x0 + lane;
    double d = 0, ef = 0, ic = 0;
    if (x < deg) {
      const int e = x < nr ? r0 + x : (int)a.inc.sidx[s0 + (x - nr)];
      const int pr = a.pprod[e];
      d = a.pdist[e];
      ef = a.p.eff[pr];
      if (PASS == 0) ic = issue_count_ld(a.p, pr);
    }
    const int m = min(32, deg - x0);
    for (int t = 0; t < m; t++) {
      const double dv = __shfl_sync(0xffffffffu, d, t), ev = __shfl_sync(0xffffffffu, ef, t);
      if (x0 + t == 0 || dv < d_min) d_min = dv;
      if (x0 + t == 0 || ev < e_min) e_min = ev;
      if (PASS == 0) ns.add(__shfl_sync(0xffffffffu, ic, t));
    }
  }
  double n_sum, total = 0.0;
  if (PASS == 0) {
    n_sum = ns.value();
    if (n_sum == 0) {
      if (lane == 0) blame_self(k, a, j);
      return;
    }
  } else {
    n_sum = a.jnsum[j];
    total = a.jtotal[j];
  }
  PySum ts;
  int so = 0;                                  // pass 0: staging slots of j's entries
  const bool stg = PASS == 0 && a.stg_cap > 0;
  if (stg) {
    if (lane == 0) so = stage_reserve(a, deg);
    so = __shfl_sync(0xffffffffu, so, 0);
    if (so < 0) return;
  }
  for (int x0 = 0; x0 < deg; x0 += 32) {
    const int x = x0 + lane;
    double prod = 0;
    if (x < deg) {
      const int e = x < nr ? r0 + x : (int)a.inc.sidx[s0 + (x - nr)];
      const int pr = a.pprod[e];
      const double f0 = __ddiv_rn(d_min, a.pdist[e]);
      const double f1 = __ddiv_rn(e_min, a.p.eff[pr]);
      const double f2 = __ddiv_rn(issue_count_ld(a.p, pr), n_sum);
      const double f3 = __ddiv_rn((double)a.p.cls_cnt[(size_t)j * 8 + kMatchClass[(a.pmeta[e] >> 30) & 3]], (double)lat);
      prod = __dmul_rn(__dmul_rn(__dmul_rn(f0, f1), f2), f3);
      if (stg) {
        const int w = so + x;
        a.stg_edge[w] = e;
        a.stg_cause[w] = pr;
        a.stg_blame[w] = prod;
        double* f = a.stg_fac + (size_t)w * 4;
        f[0] = f0; f[1] = f1; f[2] = f2; f[3] = f3;
      }
      if (PASS == 1) {
        const int w = o + x;
        a.out.stalled[w] = j;
        a.out.edge[w] = e;
        if (a.out.cause) { a.out.cause[w] = pr; a.out.meta[w] = a.pmeta[e]; }
        a.out.sub[w] = 255;
        a.out.blame[w] = __ddiv_rn(__dmul_rn(s_j, prod), total);
        double* f = a.out.factors + (size_t)w * 4;
        f[0] = f0; f[1] = f1; f[2] = f2; f[3] = f3;
      }
    }
    if (PASS == 0) {
      const int m = min(32, deg - x0);
      for (int t = 0; t < m; t++) ts.add(__shfl_sync(0xffffffffu, prod, t));
    }
  }
  if (PASS == 0) {
    total = ts.value();                        // every lane holds the same ordered sum
    if (total == 0.0) {
      if (lane == 0) blame_self(k, a, j);
    } else {
      __syncwarp();
      if (stg)
        for (int x = so + lane; x < so + deg; x += 32) a.stg_blame[x] = __ddiv_rn(__dmul_rn(s_j, a.stg_blame[x]), total);
      if (lane == 0) {
        if (stg) a.stg_off[j] = so;
        a.ecount[j] = deg;
        a.jtotal[j] = total;
        a.jnsum[j] = n_sum;
      }
    }
  }
}

// pass 0: decide self vs edges, entry count, cached sums; pass 1: write entries
template <int PASS>
__global__ void k_blame(KView k, BlameArgs a) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  if (PASS == 1 && blockIdx.x == 0 && threadIdx.x == 0) *a.out.count = a.eoff[k.N];
  if (PASS == 0) {
    // the line vectors k_blame_compact / k_lines add into
    if (a.zero_lb)
      for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.n_lines; x += gridDim.x * blockDim.x) {
        a.zero_lb[x] = 0.0;
        a.zero_ls[x] = 0.0;
      }
  }
  // whole warps iterate together (the warp path needs every lane)
  for (int j0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); j0 < k.N; j0 += gridDim.x * blockDim.x) {
    const int j = j0 + lane;
    const bool heavy = j < k.N && blame_one<PASS>(k, a, j);
    unsigned hv = __ballot_sync(0xffffffffu, heavy);
    while (hv) {
      const int src = __ffs(hv) - 1;
      hv &= hv - 1;
      blame_warp<PASS>(k, a, j0 + src, lane);
      __syncwarp();
    }
  }
}
template __global__ void k_blame<0>(KView, BlameArgs);
template __global__ void k_blame<1>(KView, BlameArgs);

// Pass 0 split by work: most stalled instructions have no pruned in-edge (C5:
// 90 %) and take the self verdict, a few loads; the rest are listed for
// k_blame_edges.  Keeps the light majority out of the register-heavy,
// divergent Eq. 1 code (k_blame<0>: 94 registers, 6.8 threads / instruction).
__global__ void k_blame_light(KView k, BlameArgs a, int32_t* __restrict__ list, int32_t* list_count) {
  pdl_wait();
  if (a.zero_lb)
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.n_lines; x += gridDim.x * blockDim.x) {
      a.zero_lb[x] = 0.0;
      a.zero_ls[x] = 0.0;
    }
  const int lane = threadIdx.x & 31;
  for (int j0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); j0 < k.N; j0 += gridDim.x * blockDim.x) {
    const int j = j0 + lane;
    bool edges = false;
    if (j < k.N) {
      a.ecount[j] = 0;
      a.self_sub[j] = -1;
      if (a.p.lat[j] != 0 && a.own.has(j)) {
        if (a.inc.deg(j) == 0) blame_self(k, a, j);
        else edges = true;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, edges);
    if (m) {
      int base = 0;
      if (lane == 0) base = atomicAdd(list_count, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (edges) list[base + __popc(m & ((1u << lane) - 1))] = j;
    }
  }
}

__global__ void k_blame_edges(KView k, BlameArgs a, const int32_t* __restrict__ list, const int32_t* list_count) {
  pdl_wait();
  const int lane = threadIdx.x & 31, n = *list_count;
  for (int t0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); t0 < n; t0 += gridDim.x * blockDim.x) {
    const int t = t0 + lane;
    const int j = t < n ? list[t] : -1;
    const bool heavy = j >= 0 && blame_one<0>(k, a, j);
    unsigned hv = __ballot_sync(0xffffffffu, heavy);
    while (hv) {
      const int src = __ffs(hv) - 1;
      hv &= hv - 1;
      blame_warp<0>(k, a, __shfl_sync(0xffffffffu, j, src), lane);
      __syncwarp();
    }
  }
}

// Pass 1 without recomputation: every stalled instruction's entries move from
// the staging area (pass 0, reservation order) to eoff[j] (stalled order), and
// the per-line rollup (k_lines) is done on the way: line_blame[line(cause)] +=
// blame_cycles, line_stall[line(j)] += S_j.  Instructions with many entries
// are copied by the whole warp.
LEO_DEV void compact_one(const KView& k, const BlameArgs& a, int j, int c, int lane, int step,
                         const int32_t* __restrict__ line_id, double* line_blame) {
  const int o = a.eoff[j], so = a.stg_off[j];
  for (int x = lane; x < c; x += step) {
    const int w = o + x, r = so + x;
    const int e = a.stg_edge[r], pr = a.stg_cause[r];
    const double bl = a.stg_blame[r];
    a.out.stalled[w] = j;
    a.out.edge[w] = e;
    if (a.out.cause) { a.out.cause[w] = pr; a.out.meta[w] = a.pmeta[e]; }
    a.out.sub[w] = 255;
    a.out.blame[w] = bl;
    const double2* f = reinterpret_cast<const double2*>(a.stg_fac + (size_t)r * 4);
    double2* g = reinterpret_cast<double2*>(a.out.factors + (size_t)w * 4);
    g[0] = f[0];
    g[1] = f[1];
    if (line_blame) atomicAdd(&line_blame[line_id[pr]], bl);
  }
}

__global__ void k_blame_compact(KView k, BlameArgs a, const int32_t* __restrict__ line_id,
                                double* line_blame, double* line_stall) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int total = a.eoff[k.N];
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.out.count = total;
  if (total > a.out.capacity) {                 // the host re-runs with a bigger list
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.status, (uint32_t)LEO_ST_BLAME_OVERFLOW);
    return;
  }
  for (int j0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); j0 < k.N; j0 += gridDim.x * blockDim.x) {
    const int j = j0 + lane;
    int c = 0;
    bool heavy = false;
    if (j < k.N) {
      c = a.ecount[j];
      if (c > 0) {
        const double s_j = (double)((int64_t)a.p.lat[j] * a.p.period);
        if (a.self_sub[j] >= 0) {
          const int o = a.eoff[j];
          a.out.stalled[o] = j;
          a.out.edge[o] = -1;
          if (a.out.cause) { a.out.cause[o] = -1; a.out.meta[o] = 0u; }
          a.out.sub[o] = (uint8_t)a.self_sub[j];
          a.out.blame[o] = s_j;
          double2* g = reinterpret_cast<double2*>(a.out.factors + (size_t)o * 4);
          g[0] = make_double2(0.0, 0.0);
          g[1] = make_double2(0.0, 0.0);
          if (line_blame) atomicAdd(&line_blame[line_id[j]], s_j);
        } else if (c > kBlameWarpDeg) {
          heavy = true;
        } else {
          compact_one(k, a, j, c, 0, 1, line_id, line_blame);
        }
      }
      if (line_stall && a.p.lat[j] && a.own.has(j))
        atomicAdd(&line_stall[line_id[j]], (double)((int64_t)a.p.lat[j] * a.p.period));
    }
    unsigned hv = __ballot_sync(0xffffffffu, heavy);
    while (hv) {
      const int src = __ffs(hv) - 1;
      hv &= hv - 1;
      compact_one(k, a, j0 + src, __shfl_sync(0xffffffffu, c, src), lane, 32, line_id, line_blame);
      __syncwarp();
    }
  }
}

// _address_traces_to_load (analysis.py:390-411), warp per candidate: the BFS
// frontier is expanded by all lanes at once (one level per round, <= 8
// rounds), visited set = open-addressing hash in shared memory.  The answer
// is whether some MEMORY_PRODUCER other than the stalled instruction is
// discovered within 8 RAW hops through non-producer intermediates, which is
// what the reference's sequential BFS returns.  Hash / frontier overflow
// re-runs the candidate on the global-stamp worker.
constexpr int kSBHash = 512, kSBFront = 256;
constexpr int kSBWarpInts = kSBHash + 2 * kSBFront + 8;

__global__ void k_selfblame_warp(KView k, BlameArgs a, int32_t* slow2, int32_t* slow2_count) {
  pdl_wait();
  extern __shared__ int32_t sbm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  int32_t* hash = sbm + (size_t)wid * kSBWarpInts;
  int32_t* fa = hash + kSBHash;
  int32_t* fb = fa + kSBFront;
  int32_t* c = fb + kSBFront;     // 0 ncur, 1 nnext, 2 found, 3 ovf, 4 nhash
  const int n = (int)min((int64_t)*a.slow_count, a.slow_cap);
  for (int t = blockIdx.x * wpc + wid; t < n; t += gridDim.x * wpc) {
    const int j = a.slow_list[t];
    for (int x = lane; x < kSBHash; x += 32) hash[x] = -1;
    __syncwarp();
    if (lane == 0) {
      c[0] = 1; c[1] = 0; c[2] = 0; c[3] = (a.dbg & LEO_DBG_SELF_SLOW) ? 1 : 0; c[4] = 1;
      fa[0] = j;
      hash[(((uint32_t)j * 2654435761u) >> 23) & (kSBHash - 1)] = j;
    }
    __syncwarp();
    int32_t *cur = fa, *nxt = fb;
    for (int depth = 0; depth < 8; depth++) {
      // every lane reads the loop control before any lane can modify it
      const int ncur = c[0];
      const bool stop = ncur == 0 || c[2] || c[3];
      __syncwarp();
      if (stop) break;
      for (int x = lane; x < ncur; x += 32) {
        const int node = cur[x];
        for (int e = a.brbeg[node]; e < a.brend[node]; e++) {
          if (((a.bmeta[e] >> 27) & 7) != LEO_EK_RAW) continue;
          const int p = a.bprod[e];
          uint32_t h = (((uint32_t)p * 2654435761u) >> 23) & (kSBHash - 1);
          bool fresh = false;
          for (int probe = 0; probe < kSBHash; probe++) {
            const int32_t prev = atomicCAS(&hash[h], -1, p);
            if (prev == -1) { fresh = true; atomicAdd(&c[4], 1); break; }
            if (prev == p) break;
            h = (h + 1) & (kSBHash - 1);
          }
          if (!fresh) continue;
          if (kMemoryProducer & BIT(k.opclass[p])) { c[2] = 1; continue; }
          const int pos = atomicAdd(&c[1], 1);
          if (pos < kSBFront) nxt[pos] = p; else c[3] = 1;
        }
      }
      __syncwarp();
      if (c[4] > kSBHash / 2) c[3] = 1;
      if (lane == 0) { c[0] = c[1]; c[1] = 0; }
      __syncwarp();
      int32_t* tmp = cur; cur = nxt; nxt = tmp;
    }
    __syncwarp();
    if (lane == 0) {
      if (c[2]) a.self_sub[j] = LEO_SB_INDIRECT_ADDRESSING;
      else if (c[3]) {
        const int s2 = atomicAdd(slow2_count, 1);
        if (s2 < a.slow_cap) slow2[s2] = j;
        else atomicOr(a.status, (uint32_t)LEO_ST_SCRATCH_OVERFLOW);
      }
    }
    __syncwarp();
  }
}

__global__ void k_selfblame_slow(KView k, BlameArgs a, const int32_t* list, const int32_t* count,
                                 int32_t* scratch, int nworkers) {
  pdl_wait();
  const int ns = (int)min((int64_t)*count, a.slow_cap);
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nworkers) return;
  int32_t* stamp = scratch + (size_t)w * 2 * (k.N + 1);
  int32_t* seen = stamp + (k.N + 1);
  for (int t = w; t < ns; t += nworkers) {
    int j = list[t];
    int r = traces_to_load(k, a.brbeg, a.brend, a.bprod, a.bmeta, j, seen, k.N + 1, stamp, j + 1);
    if (r > 0) a.self_sub[j] = LEO_SB_INDIRECT_ADDRESSING;
  }
}


// ---- per-source-line rollup -----------------------------------------------------
__global__ void k_lines(KView k, PView p, Range own, const int32_t* __restrict__ pprod, LeoBlame b,
                        const int32_t* __restrict__ line_id, double* __restrict__ line_blame,
                        double* __restrict__ line_stall) {
  pdl_wait();
  // an overflowed entry list has unwritten holes: the host re-runs bigger
  const int n = *b.count <= b.capacity ? *b.count : 0;
  const int stride = gridDim.x * blockDim.x;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride) {
    int e = b.edge[x];
    int at = e < 0 ? b.stalled[x] : pprod[e];
    atomicAdd(&line_blame[line_id[at]], b.blame[x]);
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k.N; j += stride) {
    int lat = p.lat[j];
    if (lat && own.has(j)) atomicAdd(&line_stall[line_id[j]], (double)((int64_t)lat * p.period));
  }
}

// ---- backward slice ----------------------------------------------------------------
struct SliceArgs {
  const int32_t* lat;
  const int32_t* pprod;
  Incoming inc;
  int32_t* level;
  int32_t* fa;        // frontier buffers [N]
  int32_t* fb;
  int32_t* counts;    // [2] frontier sizes (ping-pong) + [2] scratch
  uint32_t* bitmap;
};

// Appends of newly levelled nodes to the next frontier: one atomic per
// coalesced group of lanes (a per-node atomic on the one frontier counter
// serialised ~1 M sources at C5).
LEO_DEV void slice_push(int32_t* nxt, int32_t* count, int p) {
  cg::coalesced_group g = cg::coalesced_threads();
  int base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(count, (int)g.size());
  base = g.shfl(base, 0);
  nxt[base + g.thread_rank()] = p;
}

// level lv for every unlevelled producer of node v's incoming (pruned) edges
LEO_DEV void slice_expand(const SliceArgs& a, int v, int lv, int32_t* nxt, int32_t* count) {
  const int r0 = a.inc.rbeg[v], nr = a.inc.rend[v] - r0, s0 = a.inc.soff[v];
  const int deg = nr + (a.inc.soff[v + 1] - s0);
  for (int x = 0; x < deg; x++) {
    const int e = x < nr ? r0 + x : (int)a.inc.sidx[s0 + (x - nr)];
    const int p = a.pprod[e];
    if (a.level[p] < 0 && atomicCAS(&a.level[p], -1, lv) == -1) slice_push(nxt, count, p);
  }
}

// Level-synchronous BFS in one cooperative kernel, thread per frontier node
// (pruned in-degrees are small: 0.19 per instruction at C5).  Level 0 is every
// instruction with S_j > 0; level 1 expands them straight from lat[] (no
// level-0 frontier list: at C5 that is ~1 M nodes).
__global__ void k_slice(int N, SliceArgs a) {
  pdl_wait();
  cg::grid_group grid = cg::this_grid();
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  if (tid == 0) { a.counts[0] = 0; a.counts[1] = 0; }
  for (int j = tid; j < N; j += nt) a.level[j] = a.lat[j] != 0 ? 0 : -1;
  grid.sync();
  for (int j = tid; j < N; j += nt)
    if (a.lat[j] != 0) slice_expand(a, j, 1, a.fa, &a.counts[0]);
  grid.sync();
  int32_t *cur = a.fa, *nxt = a.fb;
  int ci = 0;
  for (int lv = 2;; lv++) {
    const int n = a.counts[ci];
    if (n == 0) break;
    for (int f = tid; f < n; f += nt) slice_expand(a, cur[f], lv, nxt, &a.counts[ci ^ 1]);
    grid.sync();
    if (tid == 0) a.counts[ci] = 0;
    int32_t* t = cur; cur = nxt; nxt = t;
    ci ^= 1;
    grid.sync();
  }
  // bitmap words
  for (int w = tid; w < (N + 31) / 32; w += nt) {
    uint32_t word = 0;
    for (int b = 0; b < 32; b++) {
      int j = w * 32 + b;
      if (j < N && a.level[j] >= 0) word |= 1u << b;
    }
    a.bitmap[w] = word;
  }
}

}  // namespace leo
