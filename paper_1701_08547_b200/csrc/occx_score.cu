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
#include "occx_common.cuh"

using namespace occx;

namespace {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

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
  extern __shared__ __align__(16) unsigned char smem[];
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
// K2: fused score + CTA-local per-segment top-k
// ---------------------------------------------------------------------------
struct ScoreParams {
  ArchParams archs;
  const uint4* cand;
  uint64_t n;
  uint64_t index_base;
  const occx_vent_t* vtab;
  uint32_t n_var, n_seg, k, pad;
  uint64_t chunk;           // candidates per CTA, multiple of the tile
  uint64_t* partials;       // [gridDim.x][n_seg][k]
};

constexpr int kScoreThreads = 512;
constexpr int kScoreUnroll = 4;

template <int MODE>
__device__ __forceinline__ void score_one(const SmemArch& sa, const ScoreParams& p, uint4 r,
                                          uint64_t gidx, uint64_t& key, uint32_t& seg) {
  const uint32_t variant = r.x, S = r.y, T = r.z & 0xffffu, R = r.w & 0xffffu,
                 a = (r.w >> 16) & 0xffu;
  key = 0;
  seg = 0;
  if (a >= (uint32_t)p.archs.n || variant >= p.n_var) return;
  const uint32_t aw = eval_active_warps<MODE>(sa, a, T, R, S);
  if (aw == 0) return;                      // illegal launch or zero blocks
  const occx_vent_t* e = p.vtab + ((size_t)variant * p.archs.n + a);
  const uint2 sr = __ldg(reinterpret_cast<const uint2*>(&e->seg));
  const uint32_t b = T >> 5;
  uint32_t bits = 0;
  if ((T & 31u) == 0 && b < 64) bits = (__ldg(&e->member[b >> 4]) >> ((b & 15u) * 2)) & 3u;
  const uint64_t inv = kIdxMask - gidx;
  const uint32_t hi = 0x80000000u | (bits << 29) | (aw << 22) | (sr.y << 2) |
                      (uint32_t)(inv >> 32);
  key = ((uint64_t)hi << 32) | (uint32_t)inv;
  seg = sr.x;
}

__device__ __forceinline__ void cta_insert(unsigned pend, uint64_t key, uint32_t seg,
                                           int lane, uint32_t k, volatile uint64_t* s_thr,
                                           volatile uint64_t* s_list, int* s_lock) {
  while (pend) {
    const int src = __ffs(pend) - 1;
    const uint32_t sseg = __shfl_sync(0xffffffffu, seg, src);
    const unsigned same = pend & __ballot_sync(0xffffffffu, seg == sseg);
    if (lane == 0) {
      while (atomicCAS(&s_lock[sseg], 0, 1) != 0) {
      }
      __threadfence_block();
    }
    __syncwarp();
    uint64_t mine = (lane < (int)k) ? s_list[sseg * k + lane] : 0ull;
    unsigned todo = same;
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
      s_thr[sseg] = thr;
      __threadfence_block();
      atomicExch(&s_lock[sseg], 0);
    }
    __syncwarp();
    pend &= ~same;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kScoreThreads) score_topk_kernel(const __grid_constant__ ScoreParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  SmemArch sa = build_arch_tables<MODE>(p.archs, smem);
  const size_t arch_bytes = align16(arch_smem_bytes(p.archs));
  volatile uint64_t* s_thr = reinterpret_cast<volatile uint64_t*>(smem + arch_bytes);
  volatile uint64_t* s_list = s_thr + p.n_seg;
  int* s_lock = reinterpret_cast<int*>(const_cast<uint64_t*>(s_list + (size_t)p.n_seg * p.k));
  for (uint32_t i = threadIdx.x; i < p.n_seg; i += blockDim.x) {
    s_thr[i] = 0;
    s_lock[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i < p.n_seg * p.k; i += blockDim.x) s_list[i] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const uint64_t begin = (uint64_t)blockIdx.x * p.chunk;
  const uint64_t end = begin + p.chunk < p.n ? begin + p.chunk : p.n;
  constexpr int kTile = kScoreThreads * kScoreUnroll;
  for (uint64_t base = begin; base < end; base += kTile) {
    uint4 r[kScoreUnroll];
#pragma unroll
    for (int u = 0; u < kScoreUnroll; ++u) {
      const uint64_t i = base + (uint64_t)u * kScoreThreads + threadIdx.x;
      r[u] = (i < end) ? ld_stream(p.cand + i) : make_uint4(0, 0, 0, 0xffffffffu);
    }
#pragma unroll
    for (int u = 0; u < kScoreUnroll; ++u) {
      const uint64_t i = base + (uint64_t)u * kScoreThreads + threadIdx.x;
      uint64_t key;
      uint32_t seg;
      score_one<MODE>(sa, p, r[u], p.index_base + i, key, seg);   // OOB: arch 0xff -> key 0
      const bool want = key > s_thr[seg];
      const unsigned pend = __ballot_sync(0xffffffffu, want);
      if (pend) cta_insert(pend, key, seg, lane, p.k, s_thr, s_list, s_lock);
    }
  }
  __syncthreads();
  uint64_t* out = p.partials + (size_t)blockIdx.x * p.n_seg * p.k;
  for (uint32_t i = threadIdx.x; i < p.n_seg * p.k; i += blockDim.x) out[i] = s_list[i];
}

// ---------------------------------------------------------------------------
// K3: merge n_lists tables [n_lists][n_seg][k] -> [n_seg][k]; one CTA/segment
// ---------------------------------------------------------------------------
constexpr int kMergeThreads = 256;

__global__ void __launch_bounds__(kMergeThreads)
topk_merge_kernel(const uint64_t* __restrict__ lists, uint32_t n_lists, uint32_t n_seg, uint32_t k,
                  uint64_t* __restrict__ out) {
  __shared__ uint64_t s_w[kMergeThreads / 32][OCCX_MAX_K];
  const uint32_t seg = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kMergeThreads / 32;
  uint64_t mine = 0;
  const uint64_t total = (uint64_t)n_lists * k;
  for (uint64_t b = (uint64_t)warp * 32; b < total; b += (uint64_t)kWarps * 32) {
    const uint64_t i = b + lane;
    uint64_t key = 0;
    if (i < total) {
      const uint64_t l = i / k, j = i - l * k;
      key = lists[(l * n_seg + seg) * k + j];
    }
    unsigned pend = __ballot_sync(0xffffffffu, key > warp_list_min(mine, (int)k));
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1;
      const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
      if (kk > warp_list_min(mine, (int)k)) warp_list_insert(mine, kk, (int)k, lane);
    }
  }
  if (lane < (int)k) s_w[warp][lane] = mine;
  __syncthreads();
  if (warp == 0) {
    uint64_t acc = (lane < (int)k) ? s_w[0][lane] : 0ull;
    for (int w = 1; w < kWarps; ++w) {
      const uint64_t key = (lane < (int)k) ? s_w[w][lane] : 0ull;
      unsigned pend = __ballot_sync(0xffffffffu, key > warp_list_min(acc, (int)k));
      while (pend) {
        const int src = __ffs(pend) - 1;
        pend &= pend - 1;
        const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
        if (kk > warp_list_min(acc, (int)k)) warp_list_insert(acc, kk, (int)k, lane);
      }
    }
    if (lane < (int)k) out[(size_t)seg * k + lane] = acc;
  }
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
              a.max_threads_per_block / a.warp_size <= kMaxWpb && a.max_blocks_per_mp > 0 &&
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

static size_t score_smem_bytes(const ArchParams& a, uint32_t n_seg, uint32_t k) {
  return align16(arch_smem_bytes(a)) + (size_t)n_seg * 8 + (size_t)n_seg * k * 8 +
         (size_t)n_seg * 4;
}

static int score_grid(const occx_ctx* ctx) {
  // persistent: 2 CTAs of 512 threads per SM (64 warps / SM)
  return ctx->sm_count * 2;
}

extern "C" int occx_score_workspace_bytes(const occx_ctx* ctx, uint32_t n_seg, uint32_t k,
                                          uint64_t* bytes) {
  if (!ctx || !bytes || k == 0 || k > OCCX_MAX_K || n_seg == 0) return OCCX_ERR_VALUE;
  *bytes = (uint64_t)score_grid(ctx) * n_seg * k * 8;
  return OCCX_OK;
}

extern "C" int occx_topk_merge(const occx_ctx* ctx, const uint64_t* d_lists, uint32_t n_lists,
                               uint32_t n_seg, uint32_t k, uint64_t* d_out, void* stream) {
  if (!ctx || k == 0 || k > OCCX_MAX_K || n_lists == 0) return OCCX_ERR_VALUE;
  if (n_seg == 0) return OCCX_OK;
  topk_merge_kernel<<<n_seg, kMergeThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      d_lists, n_lists, n_seg, k, d_out);
  OCCX_CUDA_TRY(cudaGetLastError());
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
  constexpr uint64_t tile = (uint64_t)kScoreThreads * kScoreUnroll;
  const uint64_t tiles = (n + tile - 1) / tile;
  p.chunk = ((tiles + grid - 1) / grid) * tile;
  if (p.chunk == 0) p.chunk = tile;
  const size_t smem = score_smem_bytes(p.archs, n_seg, k);
  if (smem > (size_t)ctx->max_smem_optin) return OCCX_ERR_CAPACITY;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (mode == OCCX_MODE_CORRECTED) {
    if (set_smem(score_topk_kernel<0>, smem)) return OCCX_ERR_CUDA;
    score_topk_kernel<0><<<grid, kScoreThreads, smem, s>>>(p);
  } else {
    if (set_smem(score_topk_kernel<1>, smem)) return OCCX_ERR_CUDA;
    score_topk_kernel<1><<<grid, kScoreThreads, smem, s>>>(p);
  }
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
