// occx_score.cu -- occupancy dump (Kd), fused score + per-segment top-k
// (K2), top-k merge (K3), suggestion sweep (K4), scorer feature table and
// the on-device candidate generator.  sm_100a.
//
// K2 is the hot path: a persistent grid streams 16-byte
// candidate records from HBM (one pass, streaming loads, 4 records in
// flight per thread), evaluates the occupancy core (occx_common.cuh) and
// the membership / cost-rank bits per candidate, packs a u64 key and keeps
// a CTA-local top-k per segment in shared memory.  Candidates whose key
// does not beat the segment's current k-th key are rejected with one
// shared-memory compare; survivors are inserted warp-cooperatively under
// a per-segment shared-memory lock.  K3 merges the per-CTA tables.
#include <cstdio>
#include <cstdlib>
#include "occx_common.cuh"
#include "occx_k2.cuh"

using namespace occx;

namespace {

#ifdef OCCX_K2_TIMING
__device__ unsigned long long g_k2_cnt[8 * 1024];
__device__ unsigned long long g_k2_hist[16 * 1024];
#define K2_COUNT(i) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_k2_cnt[blockIdx.x * 8 + (i)], 1ull); } while (0)
#define K2_ADD(i, v) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_k2_cnt[blockIdx.x * 8 + (i)], (unsigned long long)(v)); } while (0)
__device__ __forceinline__ long long k2_clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }
#else
#define K2_COUNT(i) do { } while (0)
#endif

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}


// ---------------------------------------------------------------------------
// Kd: full OccupancyResult per candidate
// ---------------------------------------------------------------------------
struct DumpParams {
  ArchParams archs;
  const uint4* cand;
  uint64_t n;
  occx_occ_t* out;
};

template <int MODE>
__global__ void __launch_bounds__(256) occ_dump_kernel(const __grid_constant__ DumpParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  SmemArch sa = build_arch_tables<MODE>(p.archs, smem);
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) {
    uint4 r = ld_stream(p.cand + i);
    uint32_t T = r.z & 0xffffu, R = r.w & 0xffffu, a = (r.w >> 16) & 0xffu, S = r.y;
    occx_occ_t o;
    if (a >= (uint32_t)p.archs.n) {
      o = occx_occ_t{};
      o.status = OCCX_ERR_VALUE;
      o.limiter = OCCX_LIMIT_ILLEGAL;
    } else {
      OccOut e = eval_full<MODE>(sa, a, T, R, S);
      o.wpb = (uint8_t)e.wpb;
      o.limit_warps = (uint8_t)e.lw;
      o.active_blocks = (uint8_t)e.blocks;
      o.active_warps = (uint8_t)e.aw;
      o.limiter = (uint8_t)e.limiter;
      o.status = (uint8_t)e.status;
      o.reserved0 = o.reserved1 = 0;
      o.limit_regs = e.lr;
      o.limit_smem = e.ls;
      o.reg_warp_limit = e.rwl;
      o.reserved2 = 0;
      // occupancy.py:192: active_warps / max_warps_per_mp, correctly rounded
      o.occupancy = __ddiv_rn((double)e.aw, (double)sa.d[a].wmp);
    }
    p.out[i] = o;
  }
}

// ---------------------------------------------------------------------------
// K2: fused score + CTA-local per-segment top-k (occx_k2.cuh for the core)
// ---------------------------------------------------------------------------
struct ScoreParams {
  ArchParams archs;
  const uint4* cand;
  uint64_t n;
  uint64_t index_base;
  const occx_vent_t* vtab;
  uint32_t n_var, n_seg, k, vt_smem;
  uint64_t chunk;           // candidates per CTA, multiple of the tile (static feeds)
  uint64_t* partials;       // [gridDim.x][n_seg][k]
  uint32_t* sched;          // TMA feed: taken[gridDim.x], CTAs done; zero on entry and exit
  uint32_t steal;           // TMA feed: idle CTAs take tiles of the busiest chunk
  unsigned long long* gthr; // TMA feed: grid-wide per-segment bound [n_seg]; zero on entry/exit
};

// Descending bitonic sort of one u64 per lane across the warp (lane 0 = largest).
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t x, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, x, stride);
      const bool keep_max = ((lane & stride) == 0) == ((lane & size) == 0);
      x = keep_max ? (x > o ? x : o) : (x < o ? x : o);
    }
  }
  return x;
}

// Many lanes beat a top-k list at once (a better thread count starts, a
// fresh list, a whole warp list flushed into the CTA table): instead of up to
// 32 dependent insertions, sort the batch and merge -- lane i < k takes
// max(list[i], batch[k-1-i]), a bitonic sequence holding exactly the top k of
// both (Batcher), then one bitonic merge.  Same result as inserting the keys
// one at a time (keys are unique).  Lanes >= k come back 0.
constexpr int kBatchMerge = 6;

// Merge two descending top-k lists held in lanes 0..k-1 (lanes >= k of x may
// hold anything): the top k of both, descending, lanes >= k zero.
__device__ __noinline__ uint64_t list_merge_sorted(uint64_t list, uint64_t x, int lane, uint32_t k) {
  const uint64_t xr = __shfl_sync(0xffffffffu, x, ((int)k - 1 - lane) & 31);
  uint64_t y = lane < (int)k ? (list > xr ? list : xr) : 0ull;
  if ((k & (k - 1)) == 0) {
    for (uint32_t stride = k >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, y, stride);
      y = (lane & stride) == 0 ? (y > o ? y : o) : (y < o ? y : o);
    }
  } else {
    y = warp_sort_desc(y, lane);
  }
  return y;
}

__device__ __forceinline__ uint64_t list_merge_batch(uint64_t list, uint64_t x, int lane, uint32_t k) {
  return list_merge_sorted(list, warp_sort_desc(x, lane), lane, k);
}

// s_thr[seg] is a lower bound of the segment's final k-th best key: the
// CTA table's k-th best, or any warp's k-th best once its list is full (k
// real keys of the segment).  Only ever raised; keys below it cannot enter
// the result, so filters may drop them.
__device__ __forceinline__ void thr_raise(volatile uint64_t* s_thr, uint32_t seg, uint64_t v) {
  atomicMax(reinterpret_cast<unsigned long long*>(const_cast<uint64_t*>(s_thr + seg)),
            (unsigned long long)v);
}

// A warp whose full list's k-th key rose: raise the CTA bound; with a
// grid-wide bound (TMA feed) also raise that, and pull a higher grid value
// back into the CTA bound (the CTA's filters then use it).
__device__ __forceinline__ void share_bound(volatile uint64_t* s_thr, unsigned long long* g_thr,
                                            uint32_t seg, uint64_t v) {
  thr_raise(s_thr, seg, v);
  if (g_thr) {
    const unsigned long long old = atomicMax(g_thr + seg, (unsigned long long)v);
    if (old > v) thr_raise(s_thr, seg, old);
  }
}

__device__ __forceinline__ void cta_insert(unsigned pend, uint64_t key, uint32_t seg,
                                           int lane, uint32_t k, volatile uint64_t* s_thr,
                                           volatile uint64_t* s_list, int* s_lock) {
  while (pend) {
    K2_COUNT(4);
    const int src = __ffs(pend) - 1;
    const uint32_t sseg = __shfl_sync(0xffffffffu, seg, src);
    const unsigned same = pend & __ballot_sync(0xffffffffu, seg == sseg);
    if (lane == 0) {
      while (atomicCAS(&s_lock[sseg], 0, 1) != 0) __nanosleep(32);
      __threadfence_block();
    }
    __syncwarp();
    uint64_t mine = (lane < (int)k) ? s_list[sseg * k + lane] : 0ull;
    unsigned todo = same;
    if (__popc(todo) >= kBatchMerge) {
      mine = list_merge_batch(mine, (todo >> lane) & 1u ? key : 0ull, lane, k);
      todo = 0;
    }
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint64_t kk = __shfl_sync(0xffffffffu, key, l);
      if (kk > warp_list_min(mine, (int)k)) warp_list_insert(mine, kk, (int)k, lane);
    }
    if (lane < (int)k) s_list[sseg * k + lane] = mine;
    const uint64_t thr = warp_list_min(mine, (int)k);
    __syncwarp();
    if (lane == 0) {
      thr_raise(s_thr, sseg, thr);
      __threadfence_block();
      atomicExch(&s_lock[sseg], 0);
    }
    __syncwarp();
    pend &= ~same;
  }
}

// Per-warp top-k list held in registers (lane j < k: j-th best key of the
// warp's current segment).  Candidates are offered against the warp's own
// exact threshold, so the common case costs one 64-bit compare and a ballot
// and improvement bursts need no lock.  When the warp moves to another
// segment its list becomes the warp's "previous" list (still in registers);
// both are staged in shared memory at the end of the chunk and merged by one
// warp.  Only a third segment in one chunk merges the previous list into the
// CTA's shared table under its lock -- at a segment boundary all warps of
// the CTA change segment within one tile, and taking the lock there was a
// 16-warp convoy that made boundary CTAs up to 2x slower.
constexpr uint32_t kNoSeg = 0xffffffffu;

struct WarpList {
  uint64_t v;
  uint64_t thr;
  uint32_t seg;
  uint32_t pseg;        // segment of the previous list (kNoSeg: none)
  uint64_t pv;          // previous list, lane j < k
};

__device__ __forceinline__ void wl_flush(WarpList& w, int lane, uint32_t k, volatile uint64_t* s_thr,
                                         volatile uint64_t* s_list, int* s_lock) {
  if (w.seg != kNoSeg) {
    if (w.pseg != kNoSeg) {
      // ">=": s_thr may be this very list's k-th key (a shared bound), which must survive
      const unsigned pend = __ballot_sync(0xffffffffu, lane < (int)k && w.pv != 0 &&
                                                           w.pv >= s_thr[w.pseg]);
      if (pend) cta_insert(pend, w.pv, w.pseg, lane, k, s_thr, s_list, s_lock);
    }
    w.pv = w.v;
    w.pseg = w.seg;
  }
  w.v = 0;
  w.thr = 0;
  w.seg = kNoSeg;
}

__device__ __forceinline__ void wl_offer(uint64_t key, uint32_t seg, WarpList& w, int lane,
                                         uint32_t k, volatile uint64_t* s_thr,
                                         volatile uint64_t* s_list, int* s_lock,
                                         unsigned long long* g_thr = nullptr) {
  const bool mine = seg == w.seg;
  unsigned pend = __ballot_sync(0xffffffffu, !mine || key > w.thr);   // key 0 carries w.seg
  if (pend == 0) return;
  K2_COUNT(0);
  const unsigned other = pend & __ballot_sync(0xffffffffu, !mine);
  if (other) {
    const uint32_t s0 = __shfl_sync(0xffffffffu, seg, __ffs(other) - 1);
    const unsigned same0 = other & __ballot_sync(0xffffffffu, seg == s0);
    if (same0 == other && other == pend) {
      // the warp has moved on to segment s0: publish the old list, adopt s0
      K2_COUNT(2);
      wl_flush(w, lane, k, s_thr, s_list, s_lock);
      w.seg = s0;
    } else {
      // mixed segments in one batch (segment boundary / unordered input)
      K2_COUNT(3);
      const bool in_other = (other >> lane) & 1u;
      const unsigned o2 = __ballot_sync(0xffffffffu, in_other && key >= s_thr[seg]);
      if (o2) cta_insert(o2, key, seg, lane, k, s_thr, s_list, s_lock);
      pend &= ~other;
    }
  }
  if (__popc(pend) >= kBatchMerge) {
    K2_COUNT(1);
    w.v = list_merge_batch(w.v, (pend >> lane) & 1u ? key : 0ull, lane, k);
    w.thr = warp_list_min(w.v, (int)k);
    if (lane == 0 && w.thr > s_thr[w.seg]) share_bound(s_thr, g_thr, w.seg, w.thr);
    return;
  }
  const uint64_t before = w.thr;
  while (pend) {
    const int l = __ffs(pend) - 1;
    pend &= pend - 1;
    const uint64_t kk = __shfl_sync(0xffffffffu, key, l);
    if (kk > w.thr) {
      warp_list_insert(w.v, kk, (int)k, lane);
      w.thr = warp_list_min(w.v, (int)k);
    }
  }
  if (lane == 0 && w.thr != before && w.thr > s_thr[w.seg])
    share_bound(s_thr, g_thr, w.seg, w.thr);
}

// Shared-memory carve-up common to both feeds (after an optional TMA ring).
struct K2Shared {
  K2Ctx c;
  volatile uint64_t* thr;
  volatile uint64_t* list;
  int* lock;
};

// Stage slots (k keys + segment id each) after the CTA's shared tables:
// current lists in slots [0, n_warps), previous lists in [n_warps, 2 n_warps).
constexpr uint32_t kStageSlots = 48;

__host__ __device__ inline size_t k2_tail_bytes(const ArchParams& a, uint32_t n_var,
                                                uint32_t n_seg, uint32_t k, bool vt_smem) {
  size_t b = k2_arch_bytes(a);
  if (vt_smem) b += (size_t)n_var * a.n * sizeof(occx_vent_t);
  return b + (size_t)n_seg * 8 + (size_t)n_seg * k * 8 + (size_t)n_seg * 4 + 16 +
         (size_t)kStageSlots * (OCCX_MAX_K + 1) * 8;
}

template <int MODE, bool VT_SMEM>
__device__ inline K2Shared k2_setup(const ScoreParams& p, unsigned char* base) {
  K2Shared s;
  K2Arch* rows = reinterpret_cast<K2Arch*>(base);
  uint32_t* tab = reinterpret_cast<uint32_t*>(base + sizeof(K2Arch) * p.archs.n);
  k2_build<MODE>(p.archs, rows, tab);
  unsigned char* q = base + k2_arch_bytes(p.archs);
  const occx_vent_t* vt = p.vtab;
  if (VT_SMEM) {
    occx_vent_t* v = reinterpret_cast<occx_vent_t*>(q);
    const uint32_t rows_n = p.n_var * (uint32_t)p.archs.n;
    const uint4* src = reinterpret_cast<const uint4*>(p.vtab);
    uint4* dst = reinterpret_cast<uint4*>(v);
    for (uint32_t i = threadIdx.x; i < rows_n * 2; i += blockDim.x) dst[i] = src[i];
    vt = v;
    q += (size_t)rows_n * sizeof(occx_vent_t);
  }
  s.c = K2Ctx{rows, tab, vt, (uint32_t)p.archs.n, p.n_var};
  s.thr = reinterpret_cast<volatile uint64_t*>(q);
  s.list = s.thr + p.n_seg;
  s.lock = reinterpret_cast<int*>(const_cast<uint64_t*>(s.list + (size_t)p.n_seg * p.k));
  for (uint32_t i = threadIdx.x; i < p.n_seg; i += blockDim.x) {
    s.thr[i] = 0;
    s.lock[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i < p.n_seg * p.k; i += blockDim.x) s.list[i] = 0;
  return s;
}

// End of chunk: every warp stages its list; after a barrier warp 0 merges
// the staged lists into the shared table alone (no lock traffic), then
// the table is written out.  `stage` holds n_warps x (k keys + segment).
__device__ inline void k2_stage(const WarpList& wl, int lane, uint32_t k, uint64_t* stage,
                                uint32_t slot, uint32_t n_warps) {
  uint64_t* row = stage + (size_t)slot * (OCCX_MAX_K + 1);
  if (lane < (int)k) row[lane] = wl.v;
  if (lane == 0) row[OCCX_MAX_K] = wl.seg;
  row += (size_t)n_warps * (OCCX_MAX_K + 1);
  if (lane < (int)k) row[lane] = wl.pv;
  if (lane == 0) row[OCCX_MAX_K] = wl.pseg;
}

__device__ inline void k2_merge_staged(const uint64_t* stage, uint32_t n_slots, uint32_t k,
                                       volatile uint64_t* s_thr, volatile uint64_t* s_list,
                                       int* s_lock) {
  const int lane = threadIdx.x & 31;
  for (uint32_t w = 0; w < n_slots; ++w) {
    const uint64_t* row = stage + (size_t)w * (OCCX_MAX_K + 1);
    const uint32_t seg = (uint32_t)row[OCCX_MAX_K];
    if (seg == kNoSeg) continue;
    const uint64_t key = lane < (int)k ? row[lane] : 0ull;
    if (!__any_sync(0xffffffffu, key != 0 && key >= s_thr[seg])) continue;
    // one warp merges after the CTA barrier: no lock; staged lists are sorted
    uint64_t mine = lane < (int)k ? s_list[seg * k + lane] : 0ull;
    mine = list_merge_sorted(mine, key, lane, k);
    if (lane < (int)k) s_list[seg * k + lane] = mine;
    const uint64_t thr = warp_list_min(mine, (int)k);
    __syncwarp();                      // every lane's s_thr[seg] read above is done
    if (lane == 0) s_thr[seg] = thr;
    __syncwarp();
  }
}

__device__ inline void k2_flush(const ScoreParams& p, const K2Shared& s) {
  uint64_t* out = p.partials + (size_t)blockIdx.x * p.n_seg * p.k;
  for (uint32_t i = threadIdx.x; i < p.n_seg * p.k; i += blockDim.x) out[i] = s.list[i];
}

// Four records of one thread (the warp's 128-record slice: j*32 + lane).
// Common case: one VOTE.ALL (cache valid for all four) and one VOTE.ANY
// (nothing beats the warp list) for four candidates.
template <int MODE, bool VT_SMEM>
__device__ __forceinline__ void k2_process4(const K2Shared& s, K2Cache& cc, WarpList& wl,
                                            const uint4 (&r)[4], const uint64_t inv, int lane,
                                            uint32_t k, bool exact = false,
                                            unsigned long long* g_thr = nullptr,
                                            uint32_t g_hi = 0) {
  uint64_t key[4];
  uint32_t seg[4];
  const bool hit = k2_hit(cc, r[0]) & k2_hit(cc, r[1]) & k2_hit(cc, r[2]) & k2_hit(cc, r[3]);
  if (__all_sync(0xffffffffu, hit)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      key[j] = k2_key<MODE>(s.c, cc, r[j], inv - 32u * j);
      seg[j] = cc.seg;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!__all_sync(0xffffffffu, k2_hit(cc, r[j]))) { K2_COUNT(5); k2_fill<VT_SMEM>(s.c, r[j], cc); }
      key[j] = k2_key<MODE>(s.c, cc, r[j], inv - 32u * j);
      seg[j] = cc.seg;
    }
  }
  // branch-free filter (bitwise on bools: no short-circuit branches); a
  // legal key has bit 63 set, so its high word alone says "non-zero"
  // High words only: every key already in the warp list comes from an earlier
  // (lower-index) batch of this warp's forward walk, so a key whose high
  // word equals the list threshold's has a smaller inverse index and is
  // below it.  Once the walk has stepped back (a stolen tile: `exact`) the
  // full keys are compared.  g_hi: the high word of the CTA / grid bound of
  // the warp's segment (some warp's full list holds k keys at or above it,
  // so a key not above it cannot make the top k; ">=" on high words since
  // its index bits are foreign).  wl_offer compares the full keys.
  bool any = false;
  if (exact) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t h = (uint32_t)(key[j] >> 32);
      any = any | ((h != 0u) & ((seg[j] != wl.seg) | ((key[j] > wl.thr) & (h >= g_hi))));
    }
  } else {
    const uint32_t thr_hi = (uint32_t)(wl.thr >> 32);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t h = (uint32_t)(key[j] >> 32);
      any = any | ((h != 0u) & ((seg[j] != wl.seg) | ((h > thr_hi) & (h >= g_hi))));
    }
  }
  if (__any_sync(0xffffffffu, any)) {
#ifdef OCCX_K2_TIMING
    const long long c0 = k2_clk();
#endif
#pragma unroll
    for (int j = 0; j < 4; ++j)
      wl_offer(key[j], key[j] ? seg[j] : wl.seg, wl, lane, k, s.thr, s.list, s.lock, g_thr);
#ifdef OCCX_K2_TIMING
    K2_ADD(6, k2_clk() - c0);
#endif
  }
}

// ---- LDG feed ---------------------------------------------------------------
constexpr int kLdgThreads = 512;
constexpr int kLdgUnroll = 4;

template <int MODE, bool VT_SMEM>
__global__ void __launch_bounds__(kLdgThreads, 2) score_topk_ldg_kernel(const __grid_constant__ ScoreParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const K2Shared s = k2_setup<MODE, VT_SMEM>(p, smem);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t begin = (uint64_t)blockIdx.x * p.chunk;
  const uint64_t end = begin + p.chunk < p.n ? begin + p.chunk : p.n;
  constexpr int kTile = kLdgThreads * kLdgUnroll;
  static_assert(kLdgUnroll == 4, "k2_process4");
  WarpList wl{0, 0, kNoSeg, kNoSeg, 0};
  K2Cache cc;
  cc.x = cc.z = cc.w = 0xffffffffu;
  k2_fill<VT_SMEM>(s.c, make_uint4(0xffffffffu, 0, 0, 0xffffffffu), cc);
  const uint32_t slice = (threadIdx.x >> 5) * 128u + lane;     // warp-contiguous 128 records
  for (uint64_t base = begin; base < end; base += kTile) {
    uint4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i = base + slice + 32u * u;
      r[u] = (i < end) ? ld_stream(p.cand + i) : make_uint4(0, 0, 0, 0xffffffffu);
    }
    k2_process4<MODE, VT_SMEM>(s, cc, wl, r, kIdxMask - p.index_base - base - slice, lane, p.k);
  }
  uint64_t* stage = reinterpret_cast<uint64_t*>(const_cast<int*>(s.lock + p.n_seg)) + 1;
  stage = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(stage) + 7) & ~uintptr_t(7));
  k2_stage(wl, lane, p.k, stage, threadIdx.x >> 5, kLdgThreads / 32);
  __syncthreads();
  if (threadIdx.x < 32) k2_merge_staged(stage, 2 * kLdgThreads / 32, p.k, s.thr, s.list, s.lock);
  __syncthreads();
  k2_flush(p, s);
}

// ---- implicit-grid feed (no records) ---------------------------------------
// Candidates are decoded from their global index (enumerate_space order,
// tuning.py:75-77) instead of being read: only the (R, S) digits change
// between neighbouring candidates, so each thread caches its current
// (TC, BC, UIF, PL, CFLAGS) block and derives R/S with one invariant-divisor
// multiply (Granlund-Montgomery) and two table loads.  The synthesized
// record is bit-identical to what gen_space_kernel writes, so keys match the
// record path exactly.
struct FastDiv {
  uint32_t m, s1, s2;
};

__device__ __forceinline__ FastDiv fastdiv_make(uint32_t d) {
  if (d <= 1) return FastDiv{1u, 0u, 0u};
  const uint32_t l = 32 - __clz(d - 1);                               // ceil(log2 d)
  const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;     // < 2^32
  return FastDiv{(uint32_t)m, 1u, l - 1};
}
__device__ __forceinline__ uint32_t fastdiv(uint32_t x, const FastDiv& f) {
  const uint32_t t = __umulhi(x, f.m);
  return (t + ((x - t) >> f.s1)) >> f.s2;
}

struct IgCache {
  uint64_t blk_lo;       // global index of the current block's first candidate
  uint32_t blk_n;        // candidates per block = |REGS| * |SMEM|
  uint32_t n_s, r_off, s_off;
  FastDiv ds;
  uint32_t x, z, w_hi;   // record words: variant, T | BC << 16, arch << 16 | PL << 24
  uint32_t seg;          // segment descriptor index
  uint32_t d_cf, d_pl, d_uif, d_bc, d_tc;   // block digits (enumerate_space order)
};

struct SpaceParams {
  ScoreParams sp;        // archs, vtab, n_var, n_seg, k, chunk, partials (cand unused)
  const occx_segdesc_t* desc;
  const uint32_t* pool;
  uint32_t n_desc, n_pool, pool_smem, pad;
  uint64_t begin;        // global index of the first candidate scored
  uint64_t key_off;      // added to the global index in keys (weak-scaling copies)
  uint32_t sep_words;    // per-warp separable-table capacity (0: general path only)
  uint32_t prune;        // skip blocks whose best possible key cannot enter the warp list
};

// Record words of the block the digits point at.
__device__ __forceinline__ void ig_derive(const SpaceParams& q, const uint32_t* pool, IgCache& c) {
  const occx_segdesc_t* d = q.desc + c.seg;
  const uint32_t T = pool[__ldg(&d->dim_off[0]) + c.d_tc];
  const uint32_t B = pool[__ldg(&d->dim_off[1]) + c.d_bc];
  c.x = __ldg(&d->var_base) + c.d_uif * __ldg(&d->dim_len[4]) + c.d_cf;
  c.z = min(T, 0xffffu) | (min(B, 0xffffu) << 16);
  c.w_hi = ((__ldg(&d->arch) & 0xffu) << 16) | ((c.d_pl & 0xffu) << 24);
}

// Full decode of g (binary search + divisions): warp start / segment change.
__device__ __noinline__ void ig_fill(const SpaceParams& q, const uint32_t* pool, uint64_t g,
                                     IgCache& c) {
  uint32_t lo = 0, hi = q.n_desc;                      // last segment with start <= g
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&q.desc[mid].start) <= g) lo = mid; else hi = mid;
  }
  const occx_segdesc_t* d = q.desc + lo;
  const uint64_t start = __ldg(&d->start);
  uint32_t len[7];
#pragma unroll
  for (int i = 0; i < 7; ++i) len[i] = __ldg(&d->dim_len[i]);
  const uint64_t blk = (uint64_t)len[5] * len[6];
  uint64_t o = (g - start) / blk;
  c.blk_lo = start + o * blk;
  c.blk_n = (uint32_t)blk;
  c.d_cf = (uint32_t)(o % len[4]);
  o /= len[4];
  c.d_pl = (uint32_t)(o % len[3]);
  o /= len[3];
  c.d_uif = (uint32_t)(o % len[2]);
  o /= len[2];
  c.d_bc = (uint32_t)(o % len[1]);
  c.d_tc = (uint32_t)(o / len[1]);
  c.seg = lo;
  c.n_s = len[6];
  c.r_off = __ldg(&d->dim_off[5]);
  c.s_off = __ldg(&d->dim_off[6]);
  c.ds = fastdiv_make(len[6]);
  ig_derive(q, pool, c);
}

// Step to the next block of the same segment (digit carry); false at the
// segment's end.
__device__ __forceinline__ bool ig_advance(const SpaceParams& q, const uint32_t* pool,
                                           IgCache& c) {
  const occx_segdesc_t* d = q.desc + c.seg;
  if (++c.d_cf == __ldg(&d->dim_len[4])) {
    c.d_cf = 0;
    if (++c.d_pl == __ldg(&d->dim_len[3])) {
      c.d_pl = 0;
      if (++c.d_uif == __ldg(&d->dim_len[2])) {
        c.d_uif = 0;
        if (++c.d_bc == __ldg(&d->dim_len[1])) {
          c.d_bc = 0;
          if (++c.d_tc == __ldg(&d->dim_len[0])) return false;
        }
      }
    }
  }
  c.blk_lo += c.blk_n;
  ig_derive(q, pool, c);
  return true;
}

// Make the cache cover g (g >= the cache's block start: warps walk forward).
__device__ __forceinline__ void ig_seek(const SpaceParams& q, const uint32_t* pool, uint64_t g,
                                        IgCache& c) {
  const uint64_t off = g - c.blk_lo;
  if (off < c.blk_n) return;
  if (c.blk_n != 0 && off < 2ull * c.blk_n && ig_advance(q, pool, c)) return;
  ig_fill(q, pool, g, c);
}

__device__ __forceinline__ uint4 ig_record(const IgCache& c, const uint32_t* pool, uint64_t g) {
  const uint32_t rs = (uint32_t)(g - c.blk_lo);
  const uint32_t ri = fastdiv(rs, c.ds);
  const uint32_t si = rs - ri * c.n_s;
  const uint32_t R = pool[c.r_off + ri], S = pool[c.s_off + si];
  return make_uint4(c.x, S, c.z, min(R, 0xffffu) | c.w_hi);
}

constexpr int kIgThreads = 768;                 // 24 warps per SM: 0.83 ms vs 0.94 (16) and 0.92 (32) on config 5
constexpr int kIgWarps = kIgThreads / 32;
static_assert(2 * kIgWarps <= (int)kStageSlots, "stage slots");
constexpr int kIgTab = 1024;                    // per-warp separable-table words (|REGS| + |SMEM|)

// ---- separable block tables (implicit grid) --------------------------------
// Inside one block of the space (fixed TC, BC, UIF, PL, CFLAGS, i.e. fixed
// (T, variant, arch)) a candidate differs from its neighbours only in (R, S),
// and the occupancy core is separable in them (occupancy.py:176-187):
//   blocks = min(limit_by_warps(T), limit_by_registers(T, R), limit_by_smem(S))
//   active_warps = min(blocks * wpb, Wmp)               (occupancy.py:186)
// and because x -> min(x * wpb, Wmp) is monotone,
//   active_warps = min(AR(R), AS(S)),  AR = min(min(lw, lr(R)) * wpb, Wmp),
//                                      AS = min(ls(S) * wpb, Wmp).
// When a warp enters a block it evaluates limit_by_registers over the block's
// REGS values and limit_by_smem over its SMEM values once (exact integer
// restatements below) into two per-warp tables holding the key's high word
// with the active-warps field filled in; every candidate is then scored by
// min(TR[ri], TS[si]) -- the same key bits k2_key produces from the record.
// A zero active-warps field (no block fits, or an illegal launch) makes the
// key 0, exactly as in k2_key.

// limit_by_registers(T, R) (occupancy.py:127-145), clamped to 255 (>= lw).
template <int MODE>
__device__ __forceinline__ uint32_t sep_lr(const occx_arch_t& a, uint32_t wpb, uint32_t R) {
  const uint32_t ws = (uint32_t)a.warp_size, gran = (uint32_t)a.register_alloc_granularity;
  const uint32_t rfs = (uint32_t)a.register_file_size, rmax = (uint32_t)a.max_regs_per_thread;
  const uint32_t bmp = (uint32_t)a.max_blocks_per_mp;
  if (R > rmax) return 0u;
  if (R == 0) return bmp;
  uint32_t v;
  if (MODE == OCCX_MODE_CORRECTED) {
    const uint32_t alloc = (R * ws + gran - 1) / gran * gran;            // _round_up
    v = min(bmp, (rfs / alloc) / wpb);                                   // :144-145
  } else {
    v = ((gran / (R * ws)) + wpb - 1) / wpb * ((rfs + gran - 1) / gran); // :139-143
  }
  return min(v, 255u);
}

// limit_by_smem(S) (occupancy.py:148-160), clamped to 255.
template <int MODE>
__device__ __forceinline__ uint32_t sep_ls(const occx_arch_t& a, uint32_t S) {
  const uint32_t smax = (uint32_t)a.shared_mem_per_block, bmp = (uint32_t)a.max_blocks_per_mp;
  if (S > smax) return 0u;
  if (S == 0) return bmp;
  const uint32_t v = (MODE == OCCX_MODE_CORRECTED) ? min(bmp, smax / S) : (smax + S - 1) / S;
  return min(v, 255u);
}

struct SepBlock {            // warp-uniform description of the tabled block
  uint64_t lo;               // global index of the block's first candidate
  uint32_t n, ns, seg;       // block size, |SMEM|, segment
  uint32_t ts;               // shared address of TS (TR starts at the warp's table)
  FastDiv ds;                // divide by |SMEM|
  uint32_t hi;               // the block's key bits (high word) outside the warps field
  // what the tables were built for: (T, arch, REGS pool, SMEM pool, ok)
  uint32_t kt, ka, kr, ks;
  uint32_t rmq;              // bytes between the TS range-max levels (0: not built)
  uint32_t rmq_k;            // top level: 4 (16-wide windows) or 5 (32-wide, TS padded by 31)
  uint32_t rmq_ready;        // the levels for the current tables are built
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Range-max levels over the padded TS (level k holds max(TS[i .. i + 2^k)),
// k = 1 .. rmq_k, sb.rmq bytes apart; the padded length is the stride - 1).
__device__ __forceinline__ void rmq_build(SepBlock& sb, int lane) {
  const uint32_t len = sb.rmq / 4u - 1u;
#pragma unroll 1
  for (uint32_t k = 1; k <= sb.rmq_k; ++k) {
    const uint32_t src = sb.ts + (k - 1) * sb.rmq, dst = sb.ts + k * sb.rmq, half = 1u << (k - 1);
    for (uint32_t i = (uint32_t)lane; i + 2 * half <= len; i += 32)
      sts_u32(dst + 4u * i, max(lds_u32(src + 4u * i), lds_u32(src + 4u * (i + half))));
    __syncwarp();
  }
  sb.rmq_ready = 1;
}


// Fill TR[0, nR] and TS[0, nS + 7) (tr = the warp's table, shared address)
// for the block ic points at; TR[nR] = 0 and TS[nS + t] = TS[t mod nS] pad
// the +j lookups.  False (tables untouched) when they do not fit.
// Upper bound of the active-warps field over a block: inside a block T and
// the arch are fixed, so the warps field of candidate (R, S) is
// min(awR(R), awS(S)) and its maximum is min(max awR, max awS) -- the same
// separable form the tables use.  Cached per warp on (T, arch, pool offsets):
// consecutive blocks of a segment differ in BC / UIF / PL / CFLAGS only.
struct BlockBound {
  uint32_t z, w, r_off, s_off;   // cache key: T | BC << 16 (T part), arch, pools
  uint32_t aw;                   // min(max awR, max awS)
};

template <int MODE>
__device__ __forceinline__ uint32_t block_aw_max(const SpaceParams& q, const uint32_t* pool,
                                                 const IgCache& ic, const K2Cache& kc,
                                                 BlockBound& bb, int lane) {
  const uint32_t a = min((ic.w_hi >> 16) & 0xffu, (uint32_t)q.sp.archs.n - 1);
  if (bb.z == (ic.z & 0xffffu) && bb.w == a && bb.r_off == ic.r_off && bb.s_off == ic.s_off)
    return bb.aw;
  const occx_arch_t& arch = q.sp.archs.a[a];
  const uint32_t ns = ic.n_s, nr = ic.blk_n / ic.n_s;
  const uint32_t lw = min(kc.lw, 255u), wpb = max(kc.wpb, 1u), wmp = kc.wmp;
  uint32_t mr = 0, ms = 0;
  for (uint32_t i = (uint32_t)lane; i < nr; i += 32) {
    const uint32_t R = min(pool[ic.r_off + i], 0xffffu);
    mr = max(mr, min(min(lw, sep_lr<MODE>(arch, wpb, R)) * wpb, wmp));
  }
  for (uint32_t i = (uint32_t)lane; i < ns; i += 32)
    ms = max(ms, min(sep_ls<MODE>(arch, pool[ic.s_off + i]) * wpb, wmp));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, o));
    ms = max(ms, __shfl_xor_sync(0xffffffffu, ms, o));
  }
  bb.z = ic.z & 0xffffu;
  bb.w = a;
  bb.r_off = ic.r_off;
  bb.s_off = ic.s_off;
  bb.aw = min(mr, ms);
  return bb.aw;
}

// The tables hold only the active-warps field (aw << 22; 0 when the launch
// is illegal): they depend on (T, arch, REGS values, SMEM values) and not on
// BC / UIF / PL / CFLAGS, so consecutive blocks of a segment (the last
// five dimensions before REGS, SMEM vary fastest) reuse them and only the
// block's key bits (sb.hi: legal | rule | static | rank) change.  A key's
// high word is sb.hi | min(TR[r], TS[s]) | index bits, exactly k2_key's.
template <int MODE, bool VT_SMEM>
__device__ __forceinline__ bool sep_build(const SpaceParams& q, const K2Shared& s,
                                          const uint32_t* pool, const IgCache& ic,
                                          uint32_t tr, SepBlock& sb, int lane) {
  const uint32_t ns = ic.n_s, nr = ic.blk_n / ic.n_s;
  if (nr + ns + 16 > q.sep_words) return false;
  K2Cache kc;
  const uint4 r0 = make_uint4(ic.x, 0u, ic.z, ic.w_hi);       // R, S irrelevant here
  k2_fill<VT_SMEM>(s.c, r0, kc);
  const uint32_t a = min((ic.w_hi >> 16) & 0xffu, (uint32_t)q.sp.archs.n - 1);
  const bool ok = kc.ok && kc.wpb != 0;
  const uint32_t T = ic.z & 0xffffu;
  const uint32_t kt = T | (ok ? 0x80000000u : 0u);
  if (sb.kt != kt || sb.ka != a || sb.kr != (ic.r_off | (nr << 20)) || sb.ks != ic.s_off ||
      sb.ns != ns) {
    const occx_arch_t& arch = q.sp.archs.a[a];
    const uint32_t lw = min(kc.lw, 255u), wpb = kc.wpb, wmp = kc.wmp;
    __syncwarp();                                             // previous block's readers
    for (uint32_t i = (uint32_t)lane; i < nr; i += 32) {
      const uint32_t R = min(pool[ic.r_off + i], 0xffffu);   // record clamp (ig_record)
      const uint32_t aw = min(min(lw, sep_lr<MODE>(arch, max(wpb, 1u), R)) * wpb, wmp);
      sts_u32(tr + 4u * i, ok ? (aw << 22) : 0u);
    }
    if (lane == 0) sts_u32(tr + 4u * nr, 0u);
    // 32-candidate runs (levels up to 32-wide) when the padded tables fit
    const bool wide = ns >= 32 && nr + 1 + 6 * (ns + 32) <= q.sep_words;
    const uint32_t pad = wide ? 31u : 15u;
    for (uint32_t i = (uint32_t)lane; i < ns + pad; i += 32) {
      const uint32_t S = pool[ic.s_off + i % ns];
      const uint32_t aw = min(sep_ls<MODE>(arch, S) * wpb, wmp);
      sts_u32(tr + 4u * (nr + 1 + i), ok ? (aw << 22) : 0u);
    }
    __syncwarp();
    // Range maxima over the padded TS for the quad filter: level k (k = 1..4)
    // holds max(TS[i .. i + 2^k)), levels ns + 16 words apart.
    const uint32_t stride = 4u * (ns + pad + 1);
    const uint32_t top = wide ? 5u : 4u;
    sb.rmq = 0;
    sb.rmq_k = 0;
    sb.rmq_ready = 0;              // levels are built on the first quad (rmq_build)
    if (ns >= 16 && nr + 1 + (top + 1) * (ns + pad + 1) <= q.sep_words) {
      sb.rmq = stride;
      sb.rmq_k = top;
    }
    sb.kt = kt;
    sb.ka = a;
    sb.kr = ic.r_off | (nr << 20);
    sb.ks = ic.s_off;
  }
  sb.lo = ic.blk_lo;
  sb.n = ic.blk_n;
  sb.ns = ns;
  sb.seg = kc.seg;
  sb.ts = tr + 4u * (nr + 1);
  sb.ds = ic.ds;
  sb.hi = kc.key_hi;
  return true;
}

template <int MODE, bool VT_SMEM>
__global__ void __launch_bounds__(kIgThreads, 1) score_space_kernel(const __grid_constant__ SpaceParams q) {
  extern __shared__ __align__(128) unsigned char smem[];
  const ScoreParams& p = q.sp;
  const K2Shared s = k2_setup<MODE, VT_SMEM>(p, smem);
  uint64_t* stage = reinterpret_cast<uint64_t*>(const_cast<int*>(s.lock + p.n_seg)) + 1;
  stage = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(stage) + 7) & ~uintptr_t(7));
  uint32_t* sep_tab = reinterpret_cast<uint32_t*>(stage + kStageSlots * (OCCX_MAX_K + 1));
  const uint32_t* pool = q.pool;
  if (q.pool_smem) {
    uint32_t* sp = sep_tab + kIgWarps * q.sep_words;
    for (uint32_t i = threadIdx.x; i < q.n_pool; i += blockDim.x) sp[i] = __ldg(q.pool + i);
    pool = sp;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t tr = (uint32_t)__cvta_generic_to_shared(sep_tab) +
                      4u * (threadIdx.x >> 5) * q.sep_words;
  const uint64_t begin = q.begin + (uint64_t)blockIdx.x * p.chunk;
  const uint64_t stop = q.begin + p.n;
  const uint64_t end = begin + p.chunk < stop ? begin + p.chunk : stop;
  WarpList wl{0, 0, kNoSeg, kNoSeg, 0};
  K2Cache cc;
  cc.x = cc.z = cc.w = 0xffffffffu;
  k2_fill<VT_SMEM>(s.c, make_uint4(0xffffffffu, 0, 0, 0xffffffffu), cc);
  IgCache ic;
  ic.blk_lo = 0;
  ic.blk_n = 0;
  SepBlock sb;
  sb.lo = 0;
  sb.n = 0;
  sb.ns = 0;
  sb.kt = sb.ka = sb.kr = sb.ks = 0xffffffffu;          // no tables yet
  sb.rmq = 0;
  sb.rmq_k = 0;
  sb.rmq_ready = 0;
  BlockBound bbnd;
  bbnd.z = 0xffffffffu;
  bbnd.w = bbnd.r_off = bbnd.s_off = bbnd.aw = 0;
  // each warp walks its own contiguous range in 128-candidate slices, so a
  // lane's block advances by +1 (digit carry) instead of being re-decoded
  const uint64_t wsz = p.chunk / kIgWarps;               // multiple of 128
  const uint64_t wb = begin + (threadIdx.x >> 5) * wsz;
  const uint64_t we = wb + wsz < end ? wb + wsz : end;
  // fast-path state: slices left in the tabled block, the lane's offset o
  // in the block and its (REGS, SMEM) digits, their step per slice
  uint32_t left = 0, o = 0, ri = 0, si = 0, dq = 0, dr = 0;
  // Score the slice at `sb_base` from the block tables: lane l takes
  // candidates sb_base + 4l + j, all inside the tabled block.
  auto fast_slice = [&](uint64_t sb_base) {
    uint32_t v[4];
    if (sb.ns >= 4) {              // at most one REGS step among the lane's four
      const uint32_t t0 = lds_u32(tr + 4u * ri), t1 = lds_u32(tr + 4u * ri + 4u);
      const uint32_t sa = sb.ts + 4u * si;
      const int jb = (int)(sb.ns - si);       // first j in the next REGS row
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = min(j < jb ? t0 : t1, lds_u32(sa + 4u * j));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t rj = fastdiv(o + j, sb.ds), sj = o + j - rj * sb.ns;
        v[j] = min(lds_u32(tr + 4u * rj), lds_u32(sb.ts + 4u * sj));
      }
    }
    // Filter on the high word only: the warp list holds keys of earlier
    // slices of this warp's forward walk (smaller indices), so a key with
    // the list threshold's high word is always below it.  The lane's best
    // high word is at most max(v) | inv_hi (the rare borrow case only makes
    // this conservative); wl_offer compares exactly.
    const uint64_t inv0 = kIdxMask - q.key_off - (sb_base + 4u * (uint32_t)lane);
    const uint32_t m = max(max(v[0], v[1]), max(v[2], v[3]));
    const uint32_t mh = m | sb.hi | (uint32_t)(inv0 >> 32);
    const bool any = (m & 0x1fc00000u) && mh >= (uint32_t)(s.thr[sb.seg] >> 32) &&
                     (sb.seg != wl.seg || mh > (uint32_t)(wl.thr >> 32));
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t inv = inv0 - (uint64_t)j;
        const uint64_t key = (v[j] & 0x1fc00000u)
            ? (((uint64_t)(v[j] | sb.hi | (uint32_t)(inv >> 32)) << 32) | (uint32_t)inv) : 0ull;
        wl_offer(key, key ? sb.seg : wl.seg, wl, lane, p.k, s.thr, s.list, s.lock, p.gthr);
      }
    }
    o += 128;
    si += dr;
    ri += dq;
    if (si >= sb.ns) {
      si -= sb.ns;
      ++ri;
    }
  };
  // Two slices at `pb` as one: lane l takes candidates pb + 8l + j (j < 8),
  // (ri, si) by one division; at most one REGS step when |SMEM| >= 8.
  auto fast_pair = [&](uint64_t pb) {
    const uint32_t o8 = (uint32_t)(pb - sb.lo) + 8u * (uint32_t)lane;
    uint32_t v[8];
    if (sb.ns >= 8) {
      const uint32_t r0 = fastdiv(o8, sb.ds), s0 = o8 - r0 * sb.ns;
      const uint32_t t0 = lds_u32(tr + 4u * r0), t1 = lds_u32(tr + 4u * r0 + 4u);
      const uint32_t sa = sb.ts + 4u * s0;
      const int jb = (int)(sb.ns - s0);       // first j in the next REGS row
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = min(j < jb ? t0 : t1, lds_u32(sa + 4u * j));
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t rj = fastdiv(o8 + j, sb.ds), sj = o8 + j - rj * sb.ns;
        v[j] = min(lds_u32(tr + 4u * rj), lds_u32(sb.ts + 4u * sj));
      }
    }
    const uint64_t inv0 = kIdxMask - q.key_off - (pb + 8u * (uint32_t)lane);
    const uint32_t m = max(max(max(v[0], v[1]), max(v[2], v[3])),
                           max(max(v[4], v[5]), max(v[6], v[7])));
    const uint32_t mh = m | sb.hi | (uint32_t)(inv0 >> 32);
    const bool any = (m & 0x1fc00000u) && mh >= (uint32_t)(s.thr[sb.seg] >> 32) &&
                     (sb.seg != wl.seg || mh > (uint32_t)(wl.thr >> 32));
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint64_t inv = inv0 - (uint64_t)j;
        const uint64_t key = (v[j] & 0x1fc00000u)
            ? (((uint64_t)(v[j] | sb.hi | (uint32_t)(inv >> 32)) << 32) | (uint32_t)inv) : 0ull;
        wl_offer(key, key ? sb.seg : wl.seg, wl, lane, p.k, s.thr, s.list, s.lock, p.gthr);
      }
    }
  };
  // Eight slices at `pb` as one filter: lane l's run is pb + 32l + j
  // (j < 32), its bound from the 32-wide range maxima (|SMEM| >= 32: at most
  // one REGS step in a run).  Only when some lane may offer are the eight
  // slices scored as two quads (finer filters; the top-k does not depend on
  // the order keys are offered in).
  auto fast_oct = [&](uint64_t pb) {
    const uint32_t o8 = (uint32_t)(pb - sb.lo) + 32u * (uint32_t)lane;
    const uint32_t r0 = fastdiv(o8, sb.ds), s0 = o8 - r0 * sb.ns;
    const uint32_t t0 = lds_u32(tr + 4u * r0), t1 = lds_u32(tr + 4u * r0 + 4u);
    const uint32_t len1 = min(sb.ns - s0, 32u);          // >= 1
    const uint32_t len2 = max(32u - len1, 1u);           // (1 when unused)
    const uint32_t k1 = 31u - __clz(len1), k2 = 31u - __clz(len2);
    const uint32_t l1 = sb.ts + k1 * sb.rmq, l2 = sb.ts + k2 * sb.rmq;
    const uint32_t a2 = s0 + len1;
    const uint32_t m1 = max(lds_u32(l1 + 4u * s0), lds_u32(l1 + 4u * (a2 - (1u << k1))));
    const uint32_t m2 = max(lds_u32(l2 + 4u * a2), lds_u32(l2 + 4u * (a2 + len2 - (1u << k2))));
    const uint32_t m = max(min(t0, m1), len1 < 32u ? min(t1, m2) : 0u);
    const uint64_t inv0 = kIdxMask - q.key_off - (pb + 32u * (uint32_t)lane);
    const uint32_t mh = m | sb.hi | (uint32_t)(inv0 >> 32);
    const bool any = (m & 0x1fc00000u) && mh >= (uint32_t)(s.thr[sb.seg] >> 32) &&
                     (sb.seg != wl.seg || mh > (uint32_t)(wl.thr >> 32));
    return __any_sync(0xffffffffu, any);
  };
  auto fast_quad = [&](uint64_t pb) {
    const uint32_t o8 = (uint32_t)(pb - sb.lo) + 16u * (uint32_t)lane;
    if (sb.rmq) {
      // Filter first from range maxima: the lane's best warps field is
      // max(min(t0, max TS[s0, s0 + len1)), min(t1, max TS[s0 + len1, s0 + 16)))
      // (min distributes over max) -- four LDS instead of sixteen; the
      // per-candidate fields are only formed when some lane may offer.
      const uint32_t r0 = fastdiv(o8, sb.ds), s0 = o8 - r0 * sb.ns;
      const uint32_t t0 = lds_u32(tr + 4u * r0), t1 = lds_u32(tr + 4u * r0 + 4u);
      const uint32_t len1 = min(sb.ns - s0, 16u);          // >= 1
      const uint32_t len2 = max(16u - len1, 1u);           // (1 when unused)
      const uint32_t k1 = 31u - __clz(len1), k2 = 31u - __clz(len2);
      const uint32_t l1 = sb.ts + k1 * sb.rmq, l2 = sb.ts + k2 * sb.rmq;
      const uint32_t a2 = s0 + len1;
      const uint32_t m1 = max(lds_u32(l1 + 4u * s0), lds_u32(l1 + 4u * (a2 - (1u << k1))));
      const uint32_t m2 = max(lds_u32(l2 + 4u * a2), lds_u32(l2 + 4u * (a2 + len2 - (1u << k2))));
      const uint32_t m = max(min(t0, m1), len1 < 16u ? min(t1, m2) : 0u);
      const uint64_t inv0 = kIdxMask - q.key_off - (pb + 16u * (uint32_t)lane);
      const uint32_t mh = m | sb.hi | (uint32_t)(inv0 >> 32);
      const bool any = (m & 0x1fc00000u) && mh >= (uint32_t)(s.thr[sb.seg] >> 32) &&
                       (sb.seg != wl.seg || mh > (uint32_t)(wl.thr >> 32));
      if (__any_sync(0xffffffffu, any)) {
        const uint32_t sa = sb.ts + 4u * s0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t vj = min((uint32_t)j < len1 ? t0 : t1, lds_u32(sa + 4u * j));
          const uint64_t inv = inv0 - (uint64_t)j;
          const uint64_t key = (vj & 0x1fc00000u)
              ? (((uint64_t)(vj | sb.hi | (uint32_t)(inv >> 32)) << 32) | (uint32_t)inv) : 0ull;
          wl_offer(key, key ? sb.seg : wl.seg, wl, lane, p.k, s.thr, s.list, s.lock, p.gthr);
        }
      }
      return;
    }
    uint32_t v[16];
    if (sb.ns >= 16) {
      const uint32_t r0 = fastdiv(o8, sb.ds), s0 = o8 - r0 * sb.ns;
      const uint32_t t0 = lds_u32(tr + 4u * r0), t1 = lds_u32(tr + 4u * r0 + 4u);
      const uint32_t sa = sb.ts + 4u * s0;
      const int jb = (int)(sb.ns - s0);       // first j in the next REGS row
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = min(j < jb ? t0 : t1, lds_u32(sa + 4u * j));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t rj = fastdiv(o8 + j, sb.ds), sj = o8 + j - rj * sb.ns;
        v[j] = min(lds_u32(tr + 4u * rj), lds_u32(sb.ts + 4u * sj));
      }
    }
    const uint64_t inv0 = kIdxMask - q.key_off - (pb + 16u * (uint32_t)lane);
    uint32_t m = v[0];
#pragma unroll
    for (int j = 1; j < 16; ++j) m = max(m, v[j]);
    const uint32_t mh = m | sb.hi | (uint32_t)(inv0 >> 32);
    const bool any = (m & 0x1fc00000u) && mh >= (uint32_t)(s.thr[sb.seg] >> 32) &&
                     (sb.seg != wl.seg || mh > (uint32_t)(wl.thr >> 32));
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint64_t inv = inv0 - (uint64_t)j;
        const uint64_t key = (v[j] & 0x1fc00000u)
            ? (((uint64_t)(v[j] | sb.hi | (uint32_t)(inv >> 32)) << 32) | (uint32_t)inv) : 0ull;
        wl_offer(key, key ? sb.seg : wl.seg, wl, lane, p.k, s.thr, s.list, s.lock, p.gthr);
      }
    }
  };
  for (uint64_t base = wb; base < we; base += 128) {
    if (base + 128 <= we) {
      ig_seek(q, pool, base, ic);                          // same g on every lane
      if (q.prune && base + 128 - ic.blk_lo <= (uint64_t)ic.blk_n) {
        // Block bound: every key of the block is at most (hi | aw_max) in its
        // high word plus the index bits of the block's first slice (the walk
        // goes forward, indices only grow).  When that cannot beat the warp
        // list of the same segment -- the test fast_quad applies per lane --
        // none of the block's whole slices can, and they are skipped.
        K2Cache kb;
        k2_fill<VT_SMEM>(s.c, make_uint4(ic.x, 0u, ic.z, ic.w_hi), kb);
        const uint32_t aw = (kb.ok && kb.wpb != 0) ? block_aw_max<MODE>(q, pool, ic, kb, bbnd, lane)
                                                   : 0u;
        const uint32_t bound = aw ? (kb.key_hi | (aw << 22)) : 0u;
        const uint32_t inv_hi = (uint32_t)((kIdxMask - q.key_off - base) >> 32);
        // (own list: an equal high word loses on the index bits; the CTA-wide
        // bound s.thr comes from other warps' indices, so it needs "<")
        if (!(bound & 0x1fc00000u) ||
            (kb.seg == wl.seg && (bound | inv_hi) <= (uint32_t)(wl.thr >> 32)) ||
            (bound | inv_hi) < (uint32_t)(s.thr[kb.seg] >> 32)) {
          const uint64_t lb = (ic.blk_lo + ic.blk_n - base) >> 7, lr = (we - base) >> 7;
          base += ((lb < lr ? lb : lr) - 1) * 128;         // + the for-increment
          continue;
        }
      }
      if (base + 128 - ic.blk_lo <= (uint64_t)ic.blk_n &&
          sep_build<MODE, VT_SMEM>(q, s, pool, ic, tr, sb, lane)) {
        const uint64_t lb = (sb.lo + sb.n - base) >> 7, lr = (we - base) >> 7;
        left = (uint32_t)(lb < lr ? lb : lr);
        // tight loop over the block's whole slices, two per trip
        if (left >= 4 && sb.rmq && !sb.rmq_ready) rmq_build(sb, lane);
        if (sb.rmq_k == 5)
          for (; left >= 8; left -= 8, base += 1024)
            if (fast_oct(base)) {
              fast_quad(base);
              fast_quad(base + 512);
            }
        for (; left >= 4; left -= 4, base += 512) fast_quad(base);
        for (; left >= 2; left -= 2, base += 256) fast_pair(base);
        if (left) {                                        // an odd last slice
          o = (uint32_t)(base - sb.lo) + 4u * (uint32_t)lane;
          ri = fastdiv(o, sb.ds);
          si = o - ri * sb.ns;
          dq = 128u / sb.ns;
          dr = 128u - dq * sb.ns;
          fast_slice(base);
          left = 0;
          base += 128;
        }
        base -= 128;                                       // the for-increment
        continue;
      }
    }
    // general path: per-lane decode (block / segment boundaries, big tables)
    const uint64_t g0 = base + lane;
    uint4 r[4];
    bool hit = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t g = g0 + 32u * j;
      hit &= (g >= we) || (g - ic.blk_lo < (uint64_t)ic.blk_n);
    }
    if (!__all_sync(0xffffffffu, hit)) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t g = g0 + 32u * j;
        if (g < we) ig_seek(q, pool, g, ic);
        r[j] = g < we ? ig_record(ic, pool, g) : make_uint4(0, 0, 0, 0xffffffffu);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t g = g0 + 32u * j;
        r[j] = g < we ? ig_record(ic, pool, g) : make_uint4(0, 0, 0, 0xffffffffu);
      }
    }
    k2_process4<MODE, VT_SMEM>(s, cc, wl, r, kIdxMask - q.key_off - g0, lane, p.k, false, p.gthr,
                               wl.seg != kNoSeg ? (uint32_t)(s.thr[wl.seg] >> 32) : 0u);
  }
  k2_stage(wl, lane, p.k, stage, threadIdx.x >> 5, kIgWarps);
  __syncthreads();
  if (threadIdx.x < 32) k2_merge_staged(stage, 2 * kIgWarps, p.k, s.thr, s.list, s.lock);
  __syncthreads();
  k2_flush(p, s);
  if (threadIdx.x == 0) {           // the last CTA returns the grid bounds to zero
    __threadfence();
    if (atomicAdd(p.sched + gridDim.x, 1u) == gridDim.x - 1) {
      for (uint32_t v = 0; v < p.n_seg; ++v) p.gthr[v] = 0;
      p.sched[gridDim.x] = 0;
    }
  }
}

// ---- TMA feed ---------------------------------------------------------------
constexpr int kTmaConsumerWarps = 16;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;
// Ring geometry by SL = contiguous 128-record slices per consumer warp per
// tile: SL = 1: 4 stages of 2,048 records (32 KB); SL = 2: 3 stages of 4,096
// (64 KB) -- each warp then sees 256 consecutive records per tile, halving
// its (T, variant, arch) cache refills; used for large calls (config 5:
// 3.11 -> 3.01 ms) where the deeper tiles' fill / drain cost is amortised.
template <int SL> struct TmaRing {
  static constexpr int kTile = 2048 * SL;
  static constexpr int kStages = SL == 1 ? 4 : 3;
  static constexpr size_t kBytes = (size_t)kStages * kTile * 16;
};
constexpr int kTmaTile = TmaRing<1>::kTile;     // chunk granularity (multiple of both tiles)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

#ifdef OCCX_K2_TIMING
// experiment-only (scripts/k2_profile.py): per CTA {entry, after setup,
// consumers done, end, smid, tiles, 0, 0} (globaltimer ns)
__device__ uint64_t g_k2_timing[8 * 1024];
__device__ __forceinline__ uint64_t k2_gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
}  // namespace
extern "C" int occx_debug_k2_timing(uint64_t* out, int n) {
  return cudaMemcpyFromSymbol(out, g_k2_timing, (size_t)n * 8 * 8) == cudaSuccess ? 0 : 6;
}
extern "C" int occx_debug_k2_counts(uint64_t* out, int n, int reset) {
  if (cudaMemcpyFromSymbol(out, g_k2_cnt, (size_t)n * 8 * 8) != cudaSuccess) return 6;
  if (reset) {
    static unsigned long long zero[16 * 1024];
    if (cudaMemcpyToSymbol(g_k2_cnt, zero, 8 * 1024 * 8) != cudaSuccess) return 6;
    if (cudaMemcpyToSymbol(g_k2_hist, zero, sizeof(zero)) != cudaSuccess) return 6;
  }
  return 0;
}
extern "C" int occx_debug_k2_hist(uint64_t* out, int n) {
  return cudaMemcpyFromSymbol(out, g_k2_hist, (size_t)n * 16 * 8) == cudaSuccess ? 0 : 6;
}
namespace {
#endif
// Tile schedule: CTA c owns the contiguous chunk [c*per, (c+1)*per) of
// 16-byte-record tiles and walks it front to back, claiming kOwnBatch tiles
// per atomicAdd on its counter taken[c] (the next batch's atomic is issued
// when the current one starts, so its latency hides behind the ring).  A
// CTA whose chunk is exhausted steals kStealBatch tiles at a time from the
// front of the chunk with the most tiles left (warp 0 scans the counters),
// so CTAs on slower SMs no longer set the kernel's end (a static split
// left the slowest SMs ~20 % behind the median).  Owner and thieves claim
// through the same counter, so every tile is taken exactly once.  Fully
// dynamic single-counter schedules were measured 1.45-2.8x slower (contended
// atomics on the producer's critical path).  The tile index reaches the
// consumers in the stage's tile_of slot; kTileEnd ends the CTA's work.  The
// last CTA to finish returns the counters to zero for the next launch.
constexpr uint32_t kTileEnd = 0xffffffffu;
constexpr uint32_t kTileStolen = 0x80000000u;   // tile_of flag: the walk may step back
constexpr uint32_t kOwnBatch = 4, kStealBatch = 2;

template <int MODE, bool VT_SMEM, int SL>
__global__ void __launch_bounds__(kTmaThreads, 1) score_topk_tma_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int kTmaSlices = SL;
  constexpr int kTmaTile = TmaRing<SL>::kTile;
  constexpr int kTmaStages = TmaRing<SL>::kStages;
  constexpr size_t kTmaRingBytes = TmaRing<SL>::kBytes;
  extern __shared__ __align__(128) unsigned char smem[];
  uint4* ring = reinterpret_cast<uint4*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTmaRingBytes);
  uint64_t* empty = full + kTmaStages;
  volatile uint32_t* tile_of = reinterpret_cast<volatile uint32_t*>(empty + kTmaStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_tiles = (uint32_t)((p.n + kTmaTile - 1) / kTmaTile);
  uint64_t policy = 0;
  // producer state (warp 0, warp-uniform; lane 0 issues)
  uint32_t issued = 0, next = 0;
  bool ended = false;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t per = (n_tiles + G - 1) / G;
  auto chunk_len = [&](uint32_t v) -> uint32_t {
    const uint64_t lo = (uint64_t)v * per;
    return lo < n_tiles ? (uint32_t)min((uint64_t)per, n_tiles - lo) : 0u;
  };
  const uint32_t own_len = chunk_len(c);
  uint32_t cur = 0, cur_hi = 0, pre = 0;       // current claimed range; prefetched claim
  bool own_done = own_len == 0, steal_done = p.steal == 0;
  if (warp == 0 && lane == 0 && !own_done) pre = atomicAdd(p.sched + c, kOwnBatch);
  // next tile of this CTA (warp 0, all lanes), n_tiles at the end
  auto grab = [&]() -> uint32_t {
    if (cur < cur_hi) return cur++;
    if (!own_done) {
      const uint32_t t0 = __shfl_sync(0xffffffffu, pre, 0);
      if (t0 < own_len) {
        cur = c * per + t0;
        cur_hi = c * per + min(t0 + kOwnBatch, own_len);
        if (lane == 0) pre = atomicAdd(p.sched + c, kOwnBatch);
        return cur++;
      }
      own_done = true;
    }
    while (!steal_done) {
      // the chunk with the most unclaimed tiles (ties: lowest index)
      uint64_t best = 0;
      for (uint32_t v = (uint32_t)lane; v < G; v += 32) {
        const uint32_t tk = *(volatile uint32_t*)(p.sched + v), len = chunk_len(v);
        if (tk < len) best = max(best, ((uint64_t)(len - tk) << 32) | (0xffffffffu - v));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (best == 0) break;
      const uint32_t v = 0xffffffffu - (uint32_t)best;
      uint32_t t0 = 0;
      if (lane == 0) t0 = atomicAdd(p.sched + v, kStealBatch);
      t0 = __shfl_sync(0xffffffffu, t0, 0);
      const uint32_t len = chunk_len(v);
      if (t0 < len) {
        cur = v * per + t0;
        cur_hi = v * per + min(t0 + kStealBatch, len);
        return kTileStolen | cur++;
      }
    }
    steal_done = true;
    return n_tiles;
  };
#ifdef OCCX_K2_TIMING
  if (threadIdx.x == 0) g_k2_timing[blockIdx.x * 8 + 0] = k2_gt();
#endif
  // issue tile `tile` into stage st (or the end marker)
  auto issue = [&](uint32_t st, uint32_t tagged) {   // warp 0; lane 0 issues
    const uint32_t tile = tagged & ~kTileStolen;
    if (tile >= n_tiles) {
      if (lane == 0) {
        tile_of[st] = kTileEnd;
        mbar_arrive(&full[st]);
      }
      ended = true;
      return;
    }
    if (lane == 0) {
      tile_of[st] = tagged;
      const uint64_t tb = (uint64_t)tile * kTmaTile;
      const uint32_t cnt = (uint32_t)min((uint64_t)kTmaTile, p.n - tb);
      mbar_expect_tx(&full[st], cnt * 16u);
      tma_load_1d(ring + (size_t)st * kTmaTile, p.cand + tb, cnt * 16u, &full[st], policy);
    }
  };
  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < kTmaStages; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], kTmaConsumerWarps);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    }
    __syncwarp();
    // the first ring round needs no free slot: start it before the table setup
    next = grab();
    while (issued < (uint32_t)kTmaStages && !ended) {
      issue(issued++, next);
      if (!ended) next = grab();
    }
  }
  const K2Shared s = k2_setup<MODE, VT_SMEM>(p, smem + kTmaRingBytes + 2 * kTmaStages * 8 + 16);
  uint64_t* stage = reinterpret_cast<uint64_t*>(const_cast<int*>(s.lock + p.n_seg)) + 1;
  stage = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(stage) + 7) & ~uintptr_t(7));
  __syncthreads();
#ifdef OCCX_K2_TIMING
  if (threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    g_k2_timing[blockIdx.x * 8 + 1] = k2_gt();
    g_k2_timing[blockIdx.x * 8 + 4] = sm;
  }
#endif
  if (warp == 0) {
    for (uint32_t t = issued; !ended; ++t) {
      const uint32_t st = t % kTmaStages;
      mbar_wait(&empty[st], ((t / kTmaStages) & 1u) ^ 1u);
      // the consumers' generic-proxy reads of this slot (ordered before
      // their empty arrivals) precede the async-proxy TMA write into it
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(st, next);
      if (!ended) next = grab();
      issued = t + 1;
    }
#ifdef OCCX_K2_TIMING
    if (lane == 0) g_k2_timing[blockIdx.x * 8 + 5] = issued - 1;
#endif
  } else {
    WarpList wl{0, 0, kNoSeg, kNoSeg, 0};
    K2Cache cc;
    cc.x = cc.z = cc.w = 0xffffffffu;
    k2_fill<VT_SMEM>(s.c, make_uint4(0xffffffffu, 0, 0, 0xffffffffu), cc);
    bool stepped_back = false;         // a stolen tile came: exact list filter from then on
    // grid-wide bound of the warp's segment, read one tile ahead (L2 latency)

    for (uint32_t t = 0;; ++t) {
      const uint32_t st = t % kTmaStages;
#ifdef OCCX_K2_TIMING
      const long long w0 = k2_clk();
#endif
      mbar_wait(&full[st], (t / kTmaStages) & 1u);
#ifdef OCCX_K2_TIMING
      K2_ADD(7, k2_clk() - w0);
#endif
      const uint32_t tagged = tile_of[st];
      if (tagged == kTileEnd) break;
      const uint32_t tile = tagged & ~kTileStolen;
      stepped_back |= (tagged & kTileStolen) != 0;
      // the CTA bound of the warp's segment (it absorbs the grid-wide bound
      // whenever a warp of this CTA raises it: share_bound)
      const uint32_t cta_hi = wl.seg != kNoSeg ? (uint32_t)(s.thr[wl.seg] >> 32) : 0u;
      const uint64_t tb = (uint64_t)tile * kTmaTile;
      const uint32_t cnt = (uint32_t)min((uint64_t)kTmaTile, p.n - tb);
      const uint4* ring_tile = ring + (size_t)st * kTmaTile;
      // warp w takes kTmaSlices contiguous 128-record slices of the tile, so
      // its (T, variant, arch) cache sees kTmaSlices x 128 consecutive records
      const uint32_t slice = (uint32_t)(warp - 1) * (128u * kTmaSlices) + lane;
      uint4 r[kTmaSlices][4];
      if (cnt == (uint32_t)kTmaTile) {                // every tile but the last
#pragma unroll
        for (int h = 0; h < kTmaSlices; ++h)
#pragma unroll
          for (int j = 0; j < 4; ++j) r[h][j] = ring_tile[slice + 128u * h + 32u * j];
      } else {
#pragma unroll
        for (int h = 0; h < kTmaSlices; ++h)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t idx = slice + 128u * h + 32u * j;
            r[h][j] = idx < cnt ? ring_tile[idx] : make_uint4(0, 0, 0, 0xffffffffu);
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);      // records are in registers
#ifdef OCCX_K2_TIMING
      const long long p0 = k2_clk();
#endif
#ifdef OCCX_K2_STREAM_ONLY
      // experiment build: stream the records, fold them into one word, no scoring
      uint32_t fold = 0;
#pragma unroll
      for (int h = 0; h < kTmaSlices; ++h)
#pragma unroll
        for (int j = 0; j < 4; ++j) fold ^= r[h][j].x ^ r[h][j].y ^ r[h][j].z ^ r[h][j].w;
      if (fold == 0x9e3779b9u && lane == 0) wl.seg = fold;
#else
#pragma unroll
      for (int h = 0; h < kTmaSlices; ++h)
        k2_process4<MODE, VT_SMEM>(s, cc, wl, r[h], kIdxMask - p.index_base - tb - slice - 128u * h,
                                   lane, p.k, stepped_back, p.gthr, cta_hi);
#endif
#ifdef OCCX_K2_TIMING
      if (lane == 0)
        atomicAdd(&g_k2_hist[blockIdx.x * 16 + (tile * 16u) / n_tiles], (unsigned long long)(k2_clk() - p0));
#endif
    }
    k2_stage(wl, lane, p.k, stage, warp - 1, kTmaConsumerWarps);
  }
  __syncthreads();
#ifdef OCCX_K2_TIMING
  if (threadIdx.x == 0) g_k2_timing[blockIdx.x * 8 + 2] = k2_gt();
#endif
  if (warp == 1) k2_merge_staged(stage, 2 * kTmaConsumerWarps, p.k, s.thr, s.list, s.lock);
  __syncthreads();
  k2_flush(p, s);
  if (threadIdx.x == 0) {
    // every producer of the grid has finished taking tiles once all CTAs
    // have counted themselves here: the last one resets the scheduler
    if (atomicAdd(p.sched + gridDim.x, 1u) == gridDim.x - 1) {
      for (uint32_t v = 0; v <= gridDim.x; ++v) p.sched[v] = 0;
      for (uint32_t v = 0; v < p.n_seg; ++v) p.gthr[v] = 0;
    }
  }
#ifdef OCCX_K2_TIMING
  __syncthreads();
  if (threadIdx.x == 0) g_k2_timing[blockIdx.x * 8 + 3] = k2_gt();
#endif
}

// ---------------------------------------------------------------------------
// K3: merge n_lists tables [n_lists][n_seg][k] -> [n_seg][k]; one CTA/segment
// ---------------------------------------------------------------------------
constexpr int kMergeThreads = 1024;

__global__ void __launch_bounds__(kMergeThreads)
topk_merge_kernel(const uint64_t* __restrict__ lists, uint32_t n_lists, uint32_t n_seg, uint32_t k,
                  uint64_t* __restrict__ out) {
  __shared__ uint64_t s_w[kMergeThreads / 32][OCCX_MAX_K];
  // launched as a programmatic dependent of the scorer: the CTAs are
  // scheduled while the scorer's last CTAs drain; wait for its writes here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t seg = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kMergeThreads / 32;
  uint64_t mine = 0;
  const uint64_t total = (uint64_t)n_lists * k;
  const uint64_t step = (uint64_t)kWarps * 32;
  auto load = [&](uint64_t i) -> uint64_t {
    if (i >= total) return 0ull;
    const uint64_t l = i / k, j = i - l * k;
    return lists[(l * n_seg + seg) * k + j];
  };
  uint64_t next = load((uint64_t)warp * 32 + lane);         // one batch ahead
  for (uint64_t b = (uint64_t)warp * 32; b < total; b += step) {
    const uint64_t key = next;
    next = load(b + step + lane);
    unsigned pend = __ballot_sync(0xffffffffu, key > warp_list_min(mine, (int)k));
    if (__popc(pend) >= kBatchMerge) {
      mine = list_merge_batch(mine, (pend >> lane) & 1u ? key : 0ull, lane, k);
      pend = 0;
    }
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
      if (kk > warp_list_min(mine, (int)k)) warp_list_insert(mine, kk, (int)k, lane);
    }
  }
  if (lane < (int)k) s_w[warp][lane] = mine;
  __syncthreads();
  // the warps' lists are sorted: a tree of pairwise sorted merges
  for (int stride = 1; stride < kWarps; stride <<= 1) {
    if (warp % (2 * stride) == 0) {
      const uint64_t a = (lane < (int)k) ? s_w[warp][lane] : 0ull;
      const uint64_t b = (lane < (int)k) ? s_w[warp + stride][lane] : 0ull;
      const uint64_t m = list_merge_sorted(a, b, lane, k);
      if (lane < (int)k) s_w[warp][lane] = m;
    }
    __syncthreads();
  }
  if (warp == 0 && lane < (int)k) out[(size_t)seg * k + lane] = s_w[0][lane];
}

// ---------------------------------------------------------------------------
// K4: suggest() sweep, one thread per request
// ---------------------------------------------------------------------------
struct SuggParams {
  ArchParams archs;
  const occx_sugg_in_t* in;
  uint32_t n;
  int mode;
  occx_sugg_t* out;
};

__device__ uint32_t lim_regs_verbatim(const occx_arch_t& a, uint32_t wpb, uint32_t R) {
  if (R > (uint32_t)a.max_regs_per_thread) return 0;
  if (R == 0) return a.max_blocks_per_mp;
  const uint32_t avail = (uint32_t)a.register_alloc_granularity / (R * (uint32_t)a.warp_size);
  const uint32_t c = ((uint32_t)a.register_file_size + a.register_alloc_granularity - 1) /
                     (uint32_t)a.register_alloc_granularity;
  return ((avail + wpb - 1) / wpb) * c;
}

__device__ uint32_t reg_warp_limit(const occx_arch_t& a, uint32_t R) {
  if (R == 0) return a.max_warps_per_mp;
  if (R > (uint32_t)a.max_regs_per_thread) return 0;
  const uint32_t g = a.register_alloc_granularity;
  const uint32_t per_warp = ((R * (uint32_t)a.warp_size + g - 1) / g) * g;
  return (uint32_t)a.register_file_size / per_warp;
}

__device__ uint32_t lim_smem(const occx_arch_t& a, uint32_t S, int mode) {
  const uint32_t smax = a.shared_mem_per_block, bmp = a.max_blocks_per_mp;
  if (S > smax) return 0;
  if (S == 0) return bmp;
  if (mode == OCCX_MODE_VERBATIM) return (smax + S - 1) / S;
  const uint32_t q = smax / S;
  return q < bmp ? q : bmp;
}

__global__ void suggest_kernel(const __grid_constant__ SuggParams p) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const occx_sugg_in_t q = p.in[i];
  occx_sugg_t o{};
  if (q.arch >= (uint32_t)p.archs.n) {
    o.status = OCCX_ERR_VALUE;
    p.out[i] = o;
    return;
  }
  const occx_arch_t a = p.archs.a[q.arch];
  // occupancy.py:239-248: unlaunchable footprints raise
  if (q.regs > (uint32_t)a.max_regs_per_thread || q.smem > (uint32_t)a.shared_mem_per_block) {
    o.status = OCCX_ERR_ILLEGAL_LAUNCH;
    p.out[i] = o;
    return;
  }
  const uint32_t ws = a.warp_size, wmp = a.max_warps_per_mp, bmp = a.max_blocks_per_mp;
  uint32_t best_t = 0;
  int64_t best_w = -1;
  // thread_candidates (occupancy.py:198-211) in ascending order
  for (uint32_t wpb = 1; wpb * ws <= (uint32_t)a.max_threads_per_block; ++wpb) {
    const uint32_t blocks = min(bmp, wmp / wpb);
    if (!(blocks >= 1 && wpb * blocks == wmp)) continue;
    const uint32_t T = wpb * ws;
    if (best_t == 0) best_t = T;
    // _active_warps_at (occupancy.py:214-229)
    uint32_t bound = min(blocks * wpb, wmp);
    if (p.mode == OCCX_MODE_VERBATIM) bound = min(bound, lim_regs_verbatim(a, wpb, q.regs) * wpb);
    else bound = min(bound, reg_warp_limit(a, q.regs));
    bound = min(bound, lim_smem(a, q.smem, p.mode) * wpb);
    if ((int64_t)bound > best_w) {
      best_t = T;
      best_w = bound;
    }
  }
  if (best_t == 0) {               // candidates[0] on an empty tuple
    o.status = OCCX_ERR_INDEX;
    p.out[i] = o;
    return;
  }
  const uint32_t bw = (uint32_t)best_w;
  const uint32_t wpb = (best_t + ws - 1) / ws;
  o.status = OCCX_OK;
  o.best_threads = best_t;
  o.best_warps = bw;
  o.best_occupancy = __ddiv_rn((double)bw, (double)wmp);
  o.best_blocks = bw ? (bw + wpb - 1) / wpb : 0;
  o.smem_budget = o.best_blocks ? (uint32_t)a.shared_mem_per_block / o.best_blocks : 0;
  if (bw) {
    const int64_t sustainable = (int64_t)((uint32_t)a.register_file_size / (bw * ws));
    const int64_t h = sustainable - (int64_t)q.regs;
    o.register_headroom = h > 0 ? (uint32_t)h : 0;
  }
  p.out[i] = o;
}

// ---------------------------------------------------------------------------
// Scorer feature table: rule side, membership words, dense cost rank
// ---------------------------------------------------------------------------
__global__ void build_vtab_kernel(const occx_mixsum_t* __restrict__ sum,
                                  const occx_feat_t* __restrict__ feat, uint32_t n_var,
                                  uint32_t n_arch, const uint32_t* __restrict__ var_kernel,
                                  const uint64_t* __restrict__ segmask,
                                  occx_vent_t* __restrict__ vtab) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_var * n_arch) return;
  const uint32_t v = t / n_arch, a = t - v * n_arch;
  const uint32_t kern = var_kernel[v];
  const uint32_t seg = kern * n_arch + a;
  // tuning.py:120: strictly above 4.0 keeps the upper half
  const bool upper = sum[v].intensity > 4.0;
  const uint64_t st = segmask[(size_t)seg * 3 + 0];
  const uint64_t ru = segmask[(size_t)seg * 3 + (upper ? 2 : 1)];
  occx_vent_t e{};
  for (int b = 0; b < 64; ++b) {
    const uint32_t two = (uint32_t)((st >> b) & 1ull) | ((uint32_t)((ru >> b) & 1ull) << 1);
    e.member[b >> 4] |= two << ((b & 15) * 2);
  }
  e.seg = seg;
  const occx_feat_t& f = feat[t];
  uint32_t rank_bits = 0;
  if (f.status == OCCX_OK) {
    // dense rank: distinct cost values strictly below mine among the
    // variants of the same kernel (variants of a kernel are contiguous)
    const double c = f.cost;
    uint32_t lo = v, hi = v;
    while (lo > 0 && var_kernel[lo - 1] == kern) --lo;
    while (hi + 1 < n_var && var_kernel[hi + 1] == kern) ++hi;
    uint32_t rank = 0;
    for (uint32_t u = lo; u <= hi; ++u) {
      const double cu = feat[(size_t)u * n_arch + a].cost;
      if (!(cu < c)) continue;
      bool first = true;                      // count each distinct value once
      for (uint32_t w = lo; w < u; ++w)
        if (feat[(size_t)w * n_arch + a].cost == cu) { first = false; break; }
      rank += first ? 1u : 0u;
    }
    rank_bits = (rank < (1u << 20)) ? ((1u << 20) - 1u - rank) : 0u;
  }
  e.rank_bits = rank_bits;
  e.key_hi = 0x80000000u | (rank_bits << 2);   // key bits 63 and 53-34, pre-shifted
  vtab[t] = e;
}

// ---------------------------------------------------------------------------
// Candidate generator: enumerate_space (tuning.py:75-77) decoded on device
// ---------------------------------------------------------------------------
__global__ void gen_space_kernel(const occx_segdesc_t* __restrict__ desc, uint32_t n_desc,
                                 const uint32_t* __restrict__ pool, uint64_t begin, uint64_t n,
                                 uint4* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t g = begin + i;
    uint32_t lo = 0, hi = n_desc;      // last desc with start <= g
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (desc[mid].start <= g) lo = mid; else hi = mid;
    }
    const occx_segdesc_t& d = desc[lo];
    uint64_t local = g - d.start;
    uint32_t idx[7];
#pragma unroll
    for (int dim = 6; dim >= 0; --dim) {
      const uint64_t len = d.dim_len[dim];
      const uint64_t q = local / len;
      idx[dim] = (uint32_t)(local - q * len);
      local = q;
    }
    const uint32_t T = pool[d.dim_off[0] + idx[0]];
    const uint32_t B = pool[d.dim_off[1] + idx[1]];
    const uint32_t R = pool[d.dim_off[5] + idx[5]];
    const uint32_t S = pool[d.dim_off[6] + idx[6]];
    uint4 r;
    r.x = d.var_base + idx[2] * d.dim_len[4] + idx[4];
    r.y = S;
    r.z = min(T, 0xffffu) | (min(B, 0xffffu) << 16);
    r.w = min(R, 0xffffu) | ((d.arch & 0xffu) << 16) | ((idx[3] & 0xffu) << 24);
    out[i] = r;
  }
}

bool pack_archs(const occx_arch_t* h, int n, ArchParams& p) {
  if (n < 1 || n > kMaxArchs || h == nullptr) return false;
  p = ArchParams{};
  for (int i = 0; i < n; ++i) p.a[i] = h[i];
  p.n = n;
  return true;
}

template <typename K>
int set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
        cudaSuccess)
      return OCCX_ERR_CUDA;
  return OCCX_OK;
}

}  // namespace

// ===========================================================================
// C ABI launchers
// ===========================================================================
extern "C" int occx_check_archs(const occx_arch_t* h, int n, int* bad) {
  if (bad) *bad = -1;
  if (h == nullptr || n < 1 || n > kMaxArchs) return OCCX_ERR_CAPACITY;
  for (int i = 0; i < n; ++i) {
    const occx_arch_t& a = h[i];
    bool ok = a.warp_size > 0 && (a.warp_size & (a.warp_size - 1)) == 0 &&
              a.max_threads_per_block > 0 && a.max_threads_per_block % a.warp_size == 0 &&
              a.max_threads_per_block / a.warp_size <= kMaxWpb &&
              a.max_threads_per_block <= 2048 &&         // membership masks: bit T/32 - 1 < 64
              a.max_blocks_per_mp > 0 &&
              a.max_blocks_per_mp <= 255 && a.max_warps_per_mp > 0 && a.max_warps_per_mp <= 127 &&
              a.register_file_size > 0 && a.register_file_size < (1 << 20) &&
              a.register_alloc_granularity > 0 && a.register_alloc_granularity < (1 << 20) &&
              a.max_regs_per_thread > 0 && a.max_regs_per_thread <= 1023 &&
              a.shared_mem_per_block > 0 && a.shared_mem_per_block < (1 << 24);
    if (!ok) {
      if (bad) *bad = i;
      return OCCX_ERR_CAPACITY;
    }
  }
  return OCCX_OK;
}

extern "C" int occx_occupancy_batch(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                                    const occx_cand_t* d_cand, uint64_t n, int mode,
                                    occx_occ_t* d_out, void* stream) {
  if (!ctx || (mode != 0 && mode != 1)) return OCCX_ERR_VALUE;
  int bad;
  int st = occx_check_archs(h_archs, n_arch, &bad);
  if (st) return st;
  if (n == 0) return OCCX_OK;
  DumpParams p{};
  pack_archs(h_archs, n_arch, p.archs);
  p.cand = reinterpret_cast<const uint4*>(d_cand);
  p.n = n;
  p.out = d_out;
  const size_t smem = arch_smem_bytes(p.archs);
  const uint64_t want = (n + 255) / 256;
  const int grid = (int)(want < (uint64_t)ctx->sm_count * 8 ? want : (uint64_t)ctx->sm_count * 8);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (mode == OCCX_MODE_CORRECTED) {
    if (set_smem(occ_dump_kernel<0>, smem)) return OCCX_ERR_CUDA;
    occ_dump_kernel<0><<<grid, 256, smem, s>>>(p);
  } else {
    if (set_smem(occ_dump_kernel<1>, smem)) return OCCX_ERR_CUDA;
    occ_dump_kernel<1><<<grid, 256, smem, s>>>(p);
  }
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}

enum { kFeedTma = 0, kFeedLdg = 1 };

static int score_feed(const occx_ctx* ctx) {
  // fixed per context (occx_ctx_create_ex options): the workspace size follows it
  return (ctx->options & OCCX_CTX_K2_FEED_LDG) ? kFeedLdg : kFeedTma;
}

static int score_grid(const occx_ctx* ctx) {
  // persistent: TMA feed one 544-thread CTA per SM; LDG feed two 512-thread CTAs
  return score_feed(ctx) == kFeedTma ? ctx->sm_count : ctx->sm_count * 2;
}

// Workspace: [score_grid][n_seg][k] per-CTA tables, then a 256-byte
// scheduler block (TMA feed tile counter); zero before the first call,
// every call leaves it zero.
// taken[grid] + done, then the grid-wide per-segment bounds gthr[n_seg]; 256-B units
static uint64_t sched_words_bytes(const occx_ctx* ctx) {
  return ((uint64_t)(score_grid(ctx) + 1) * 4 + 255) / 256 * 256;
}
static uint64_t sched_bytes(const occx_ctx* ctx, uint32_t n_seg) {
  return sched_words_bytes(ctx) + ((uint64_t)n_seg * 8 + 255) / 256 * 256;
}

extern "C" int occx_score_workspace_bytes(const occx_ctx* ctx, uint32_t n_seg, uint32_t k,
                                          uint64_t* bytes) {
  if (!ctx || !bytes || k == 0 || k > OCCX_MAX_K || n_seg == 0) return OCCX_ERR_VALUE;
  *bytes = (uint64_t)score_grid(ctx) * n_seg * k * 8 + sched_bytes(ctx, n_seg);
  return OCCX_OK;
}

extern "C" int occx_score_lists(const occx_ctx* ctx) { return ctx ? score_grid(ctx) : 0; }

extern "C" int occx_score_workspace_init(const occx_ctx* ctx, void* d_ws, uint32_t n_seg,
                                         uint32_t k, void* stream) {
  if (!ctx || !d_ws || k == 0 || k > OCCX_MAX_K || n_seg == 0) return OCCX_ERR_VALUE;
  const uint64_t tables = (uint64_t)score_grid(ctx) * n_seg * k * 8;
  OCCX_CUDA_TRY(cudaMemsetAsync(static_cast<char*>(d_ws) + tables, 0, sched_bytes(ctx, n_seg),
                                reinterpret_cast<cudaStream_t>(stream)));
  return OCCX_OK;
}

extern "C" int occx_topk_merge(const occx_ctx* ctx, const uint64_t* d_lists, uint32_t n_lists,
                               uint32_t n_seg, uint32_t k, uint64_t* d_out, void* stream) {
  if (!ctx || k == 0 || k > OCCX_MAX_K || n_lists == 0) return OCCX_ERR_VALUE;
  if (n_seg == 0) return OCCX_OK;
  // programmatic dependent launch: K3's launch overlaps the tail of the
  // kernel before it on the stream (K2); griddepcontrol.wait in K3 orders
  // the reads (a no-op when the previous work is not a kernel)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_seg);
  cfg.blockDim = dim3(kMergeThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OCCX_CUDA_TRY(cudaLaunchKernelEx(&cfg, topk_merge_kernel, d_lists, n_lists, n_seg, k, d_out));
  return OCCX_OK;
}

extern "C" int occx_score_topk(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                               const occx_cand_t* d_cand, uint64_t n, uint64_t index_base,
                               int mode, const occx_vent_t* d_vtab, uint32_t n_var,
                               uint32_t n_seg, uint32_t k, void* d_ws, uint64_t ws_bytes,
                               uint64_t* d_topk, void* stream) {
  if (!ctx || (mode != 0 && mode != 1) || k == 0 || k > OCCX_MAX_K || n_seg == 0)
    return OCCX_ERR_VALUE;
  int bad;
  int st = occx_check_archs(h_archs, n_arch, &bad);
  if (st) return st;
  if (index_base + n > kIdxMask + 1 || index_base + n < index_base) return OCCX_ERR_CAPACITY;
  uint64_t need = 0;
  occx_score_workspace_bytes(ctx, n_seg, k, &need);
  if (d_ws == nullptr || ws_bytes < need) return OCCX_ERR_VALUE;
  ScoreParams p{};
  pack_archs(h_archs, n_arch, p.archs);
  p.cand = reinterpret_cast<const uint4*>(d_cand);
  p.n = n;
  p.index_base = index_base;
  p.vtab = d_vtab;
  p.n_var = n_var;
  p.n_seg = n_seg;
  p.k = k;
  p.partials = static_cast<uint64_t*>(d_ws);
  const int grid = score_grid(ctx);
  const int feed = score_feed(ctx);
  p.sched = reinterpret_cast<uint32_t*>(static_cast<char*>(d_ws) + need - sched_bytes(ctx, n_seg));
  p.gthr = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(p.sched) +
                                                 sched_words_bytes(ctx));
  p.steal = (ctx->options & OCCX_CTX_K2_NO_STEAL) ? 0u : 1u;
  p.vt_smem = ((uint64_t)n_var * n_arch <= (uint64_t)kVtSmemMax) ? 1u : 0u;
  size_t smem = k2_tail_bytes(p.archs, n_var, n_seg, k, p.vt_smem != 0);
  // two slices per warp (64 KB stages, 192 KB in flight per SM) whenever the
  // ring fits: per-SM bandwidth is bytes-in-flight bound (config 2: 0.123 ->
  // 0.107 ms, config 4: 0.309 -> 0.298 ms vs one slice).  OCCX_CTX_K2_ONE_SLICE
  // (context option) forces one.
  const bool one_slice = (ctx->options & OCCX_CTX_K2_ONE_SLICE) != 0;
  int sl = (feed == kFeedTma && !one_slice &&
            smem + TmaRing<2>::kBytes + 2 * TmaRing<2>::kStages * 8 + 16 <= (size_t)ctx->max_smem_optin)
               ? 2 : 1;
  if (feed == kFeedTma)
    smem += (sl == 2 ? TmaRing<2>::kBytes + 2 * TmaRing<2>::kStages * 8
                     : TmaRing<1>::kBytes + 2 * TmaRing<1>::kStages * 8) + 16;   // + tile_of
  const uint64_t tile = feed == kFeedTma ? (uint64_t)kTmaTile * sl : (uint64_t)kLdgThreads * kLdgUnroll;
  const uint64_t tiles = (n + tile - 1) / tile;
  p.chunk = ((tiles + grid - 1) / grid) * tile;
  if (p.chunk == 0) p.chunk = tile;
  if (smem > (size_t)ctx->max_smem_optin) {
    if (!p.vt_smem) return OCCX_ERR_CAPACITY;
    p.vt_smem = 0;
    smem -= (size_t)n_var * n_arch * sizeof(occx_vent_t);
    if (smem > (size_t)ctx->max_smem_optin) return OCCX_ERR_CAPACITY;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define OCCX_LAUNCH_K2(KERNEL, THREADS)                                              \
  do {                                                                               \
    if (set_smem(KERNEL, smem)) return OCCX_ERR_CUDA;                                \
    KERNEL<<<grid, THREADS, smem, s>>>(p);                                           \
  } while (0)
  const bool vts = p.vt_smem != 0;
  if (feed == kFeedTma && sl == 2) {
    if (mode == OCCX_MODE_CORRECTED) {
      if (vts) OCCX_LAUNCH_K2((score_topk_tma_kernel<0, true, 2>), kTmaThreads);
      else OCCX_LAUNCH_K2((score_topk_tma_kernel<0, false, 2>), kTmaThreads);
    } else {
      if (vts) OCCX_LAUNCH_K2((score_topk_tma_kernel<1, true, 2>), kTmaThreads);
      else OCCX_LAUNCH_K2((score_topk_tma_kernel<1, false, 2>), kTmaThreads);
    }
  } else if (feed == kFeedTma) {
    if (mode == OCCX_MODE_CORRECTED) {
      if (vts) OCCX_LAUNCH_K2((score_topk_tma_kernel<0, true, 1>), kTmaThreads);
      else OCCX_LAUNCH_K2((score_topk_tma_kernel<0, false, 1>), kTmaThreads);
    } else {
      if (vts) OCCX_LAUNCH_K2((score_topk_tma_kernel<1, true, 1>), kTmaThreads);
      else OCCX_LAUNCH_K2((score_topk_tma_kernel<1, false, 1>), kTmaThreads);
    }
  } else {
    if (mode == OCCX_MODE_CORRECTED) {
      if (vts) OCCX_LAUNCH_K2((score_topk_ldg_kernel<0, true>), kLdgThreads);
      else OCCX_LAUNCH_K2((score_topk_ldg_kernel<0, false>), kLdgThreads);
    } else {
      if (vts) OCCX_LAUNCH_K2((score_topk_ldg_kernel<1, true>), kLdgThreads);
      else OCCX_LAUNCH_K2((score_topk_ldg_kernel<1, false>), kLdgThreads);
    }
  }
#undef OCCX_LAUNCH_K2
  OCCX_CUDA_TRY(cudaGetLastError());
  if (d_topk == nullptr) return OCCX_OK;     // partials only: [grid][n_seg][k] in d_ws
  return occx_topk_merge(ctx, p.partials, (uint32_t)grid, n_seg, k, d_topk, stream);
}

extern "C" int occx_suggest_batch(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                                  const occx_sugg_in_t* d_in, uint32_t n, int mode,
                                  occx_sugg_t* d_out, void* stream) {
  if (!ctx || (mode != 0 && mode != 1)) return OCCX_ERR_VALUE;
  int bad;
  int st = occx_check_archs(h_archs, n_arch, &bad);
  if (st) return st;
  if (n == 0) return OCCX_OK;
  SuggParams p{};
  pack_archs(h_archs, n_arch, p.archs);
  p.in = d_in;
  p.n = n;
  p.mode = mode;
  p.out = d_out;
  suggest_kernel<<<(n + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}

extern "C" int occx_build_vtab(const occx_ctx* ctx, const occx_mixsum_t* d_sum,
                               const occx_feat_t* d_feat, uint32_t n_var, uint32_t n_arch,
                               const uint32_t* d_var_kernel, const uint64_t* d_segmask,
                               occx_vent_t* d_vtab, void* stream) {
  if (!ctx || n_arch == 0 || n_arch > (uint32_t)kMaxArchs) return OCCX_ERR_VALUE;
  const uint64_t total = (uint64_t)n_var * n_arch;
  if (total == 0) return OCCX_OK;
  build_vtab_kernel<<<(unsigned)((total + 127) / 128), 128, 0,
                      reinterpret_cast<cudaStream_t>(stream)>>>(d_sum, d_feat, n_var, n_arch,
                                                                d_var_kernel, d_segmask, d_vtab);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}

// ---------------------------------------------------------------------------
// score_space() in one call: H2D description -> K1 -> feature table -> K2i ->
// K3 -> D2H.  d_buf: blob | K1 sums | K1 features | feature table | K2
// workspace | top-k table, each 256-byte aligned.
// ---------------------------------------------------------------------------
static uint64_t align256(uint64_t b) { return (b + 255) / 256 * 256; }

struct SpaceBuf {
  uint64_t sum, feat, vtab, ws, ws_bytes, topk, total;
};

static int space_buf_layout(const occx_ctx* ctx, uint64_t blob_bytes, uint32_t n_var,
                            uint32_t n_arch, uint32_t n_seg, uint32_t k, SpaceBuf* b) {
  if (!ctx || k == 0 || k > OCCX_MAX_K || n_seg == 0 || n_arch == 0) return OCCX_ERR_VALUE;
  uint64_t ws = 0;
  occx_score_workspace_bytes(ctx, n_seg, k, &ws);
  const uint64_t cells = (uint64_t)n_var * n_arch;
  b->sum = align256(blob_bytes);
  b->feat = b->sum + align256((uint64_t)n_var * sizeof(occx_mixsum_t));
  b->vtab = b->feat + align256(cells * sizeof(occx_feat_t));
  b->ws = b->vtab + align256(cells * sizeof(occx_vent_t));
  b->ws_bytes = ws;
  b->topk = b->ws + align256(ws);
  b->total = b->topk + align256((uint64_t)n_seg * k * 8);
  return OCCX_OK;
}

extern "C" int occx_space_buf_bytes(const occx_ctx* ctx, uint64_t blob_bytes, uint32_t n_var,
                                    uint32_t n_arch, uint32_t n_seg, uint32_t k,
                                    uint64_t* bytes, uint64_t* topk_off) {
  SpaceBuf b;
  const int st = space_buf_layout(ctx, blob_bytes, n_var, n_arch, n_seg, k, &b);
  if (st) return st;
  if (bytes) *bytes = b.total;
  if (topk_off) *topk_off = b.topk;
  return OCCX_OK;
}

extern "C" int occx_score_space_host(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                                     const void* h_blob, uint64_t blob_bytes,
                                     const uint64_t* blob_off, uint32_t n_seg, uint32_t n_pool,
                                     uint32_t n_var, const double* h_cpi, double scale,
                                     int sum_mode, uint64_t begin, uint64_t n,
                                     uint64_t key_offset, int mode, uint32_t flags, uint32_t k,
                                     void* d_buf, uint64_t buf_bytes, uint64_t* h_topk,
                                     void* stream) {
  if (!ctx || !h_archs || !h_blob || !blob_off || !h_cpi || !d_buf || n_arch < 1 ||
      n_arch > kMaxArchs || n_var == 0)
    return OCCX_ERR_VALUE;
  for (int i = 0; i < 5; ++i)
    if (blob_off[i] > blob_bytes || (blob_off[i] & 15u)) return OCCX_ERR_VALUE;
  if ((uint64_t)n_seg % (uint64_t)n_arch) return OCCX_ERR_VALUE;
  SpaceBuf b;
  int st = space_buf_layout(ctx, blob_bytes, n_var, (uint32_t)n_arch, n_seg, k, &b);
  if (st) return st;
  if (buf_bytes < b.total) return OCCX_ERR_VALUE;
  int bad;
  st = occx_check_archs(h_archs, n_arch, &bad);
  if (st) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char* base = static_cast<char*>(d_buf);
  OCCX_CUDA_TRY(cudaMemcpyAsync(base, h_blob, blob_bytes, cudaMemcpyHostToDevice, s));
  // the workspace's scheduler block (done counter, grid-wide segment bounds)
  // starts zeroed; the scorer leaves it zero
  OCCX_CUDA_TRY(cudaMemsetAsync(base + b.ws + (b.ws_bytes - sched_bytes(ctx, n_seg)), 0,
                                sched_bytes(ctx, n_seg), s));
  int32_t cols[kMaxArchs];
  for (int i = 0; i < n_arch; ++i) cols[i] = h_archs[i].cost_key;
  auto at = [&](int i) { return base + blob_off[i]; };
  occx_mixsum_t* d_sum = reinterpret_cast<occx_mixsum_t*>(base + b.sum);
  occx_feat_t* d_feat = reinterpret_cast<occx_feat_t*>(base + b.feat);
  occx_vent_t* d_vtab = reinterpret_cast<occx_vent_t*>(base + b.vtab);
  st = occx_feature_score(ctx, reinterpret_cast<const occx_mix_t*>(at(4)), n_var, cols,
                          (uint32_t)n_arch, h_cpi, scale, sum_mode, d_sum, d_feat, stream);
  if (st) return st;
  st = occx_build_vtab(ctx, d_sum, d_feat, n_var, (uint32_t)n_arch,
                       reinterpret_cast<const uint32_t*>(at(3)),
                       reinterpret_cast<const uint64_t*>(at(2)), d_vtab, stream);
  if (st) return st;
  uint64_t* d_topk = reinterpret_cast<uint64_t*>(base + b.topk);
  st = occx_score_space(ctx, h_archs, n_arch, reinterpret_cast<const occx_segdesc_t*>(at(0)),
                        n_seg, reinterpret_cast<const uint32_t*>(at(1)), n_pool, begin, n,
                        key_offset, mode, flags, d_vtab, n_var, n_seg, k, base + b.ws,
                        b.ws_bytes, d_topk, stream);
  if (st) return st;
  if (h_topk == nullptr) return OCCX_OK;
  OCCX_CUDA_TRY(cudaMemcpyAsync(h_topk, d_topk, (size_t)n_seg * k * 8, cudaMemcpyDeviceToHost, s));
  OCCX_CUDA_TRY(cudaStreamSynchronize(s));
  return OCCX_OK;
}

extern "C" int occx_gen_space(const occx_ctx* ctx, const occx_segdesc_t* d_desc, uint32_t n_desc,
                              const uint32_t* d_pool, uint64_t begin, uint64_t n,
                              occx_cand_t* d_out, void* stream) {
  if (!ctx || n_desc == 0) return OCCX_ERR_VALUE;
  if (n == 0) return OCCX_OK;
  const uint64_t want = (n + 255) / 256;
  const unsigned grid = (unsigned)(want < (uint64_t)ctx->sm_count * 16 ? want : ctx->sm_count * 16);
  gen_space_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      d_desc, n_desc, d_pool, begin, n, reinterpret_cast<uint4*>(d_out));
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}

extern "C" int occx_score_space(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                                const occx_segdesc_t* d_desc, uint32_t n_desc,
                                const uint32_t* d_pool, uint32_t n_pool, uint64_t begin,
                                uint64_t n, uint64_t key_offset, int mode, uint32_t flags,
                                const occx_vent_t* d_vtab, uint32_t n_var,
                                uint32_t n_seg, uint32_t k, void* d_ws, uint64_t ws_bytes,
                                uint64_t* d_topk, void* stream) {
  if (!ctx || (mode != 0 && mode != 1) || k == 0 || k > OCCX_MAX_K || n_seg == 0 ||
      n_desc == 0 || d_desc == nullptr || d_pool == nullptr ||
      (flags & ~(uint32_t)OCCX_SCORE_EVERY_KEY) != 0)
    return OCCX_ERR_VALUE;
  int bad;
  int st = occx_check_archs(h_archs, n_arch, &bad);
  if (st) return st;
  if (begin + n > kIdxMask + 1 || begin + n < begin) return OCCX_ERR_CAPACITY;
  if (key_offset > kIdxMask + 1 - (begin + n)) return OCCX_ERR_CAPACITY;
  uint64_t need = 0;
  occx_score_workspace_bytes(ctx, n_seg, k, &need);
  if (d_ws == nullptr || ws_bytes < need) return OCCX_ERR_VALUE;
  SpaceParams q{};
  q.key_off = key_offset;
  pack_archs(h_archs, n_arch, q.sp.archs);
  q.sp.n = n;
  q.sp.index_base = begin;
  q.sp.vtab = d_vtab;
  q.sp.n_var = n_var;
  q.sp.n_seg = n_seg;
  q.sp.k = k;
  q.sp.partials = static_cast<uint64_t*>(d_ws);
  // scheduler block: the done counter (after grid tables' worth of words) and
  // the grid-wide per-segment bounds, as for the record scorer
  q.sp.sched = reinterpret_cast<uint32_t*>(static_cast<char*>(d_ws) + need -
                                           sched_bytes(ctx, n_seg));
  q.sp.gthr = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(q.sp.sched) +
                                                    sched_words_bytes(ctx));
  q.desc = d_desc;
  q.pool = d_pool;
  q.n_desc = n_desc;
  q.n_pool = n_pool;
  q.begin = begin;
  const int grid = ctx->sm_count;                         // one kIgThreads CTA per SM
  const uint64_t tile = (uint64_t)kIgWarps * 128;          // each warp walks chunk / kIgWarps
  const uint64_t tiles = (n + tile - 1) / tile;
  q.sp.chunk = ((tiles + grid - 1) / grid) * tile;
  if (q.sp.chunk == 0) q.sp.chunk = tile;
  q.sp.vt_smem = ((uint64_t)n_var * n_arch <= (uint64_t)kVtSmemMax) ? 1u : 0u;
  size_t smem = k2_tail_bytes(q.sp.archs, n_var, n_seg, k, q.sp.vt_smem != 0);
  q.pool_smem = (n_pool <= 8192u) ? 1u : 0u;
  if (q.pool_smem) smem += (size_t)n_pool * 4;
  if (smem > (size_t)ctx->max_smem_optin) return OCCX_ERR_CAPACITY;
  // per-warp separable tables when they fit (else the general path only)
  q.sep_words = smem + (size_t)kIgWarps * kIgTab * 4 <= (size_t)ctx->max_smem_optin ? kIgTab : 0;
  q.prune = (flags & OCCX_SCORE_EVERY_KEY) ? 0u : 1u;    // exact block-bound pruning
  smem += (size_t)kIgWarps * q.sep_words * 4;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
#define OCCX_LAUNCH_IG(KERNEL)                                                       \
  do {                                                                               \
    if (set_smem(KERNEL, smem)) return OCCX_ERR_CUDA;                                \
    KERNEL<<<grid, kIgThreads, smem, s>>>(q);                                        \
  } while (0)
  const bool vts = q.sp.vt_smem != 0;
  if (mode == OCCX_MODE_CORRECTED) {
    if (vts) OCCX_LAUNCH_IG((score_space_kernel<0, true>));
    else OCCX_LAUNCH_IG((score_space_kernel<0, false>));
  } else {
    if (vts) OCCX_LAUNCH_IG((score_space_kernel<1, true>));
    else OCCX_LAUNCH_IG((score_space_kernel<1, false>));
  }
#undef OCCX_LAUNCH_IG
  OCCX_CUDA_TRY(cudaGetLastError());
  if (d_topk == nullptr) return OCCX_OK;
  return occx_topk_merge(ctx, q.sp.partials, (uint32_t)grid, n_seg, k, d_topk, stream);
}
