// occx_common.cuh -- device-side occupancy core shared by the Kd dump, the
// K2 fused scorer and the K4 suggestion sweep.
//
// Restates occmix/occupancy.py:85-195 with integer arithmetic that is exact
// for every input the packed record can carry:
//   wpb  = ceil(T / ws)                                  occupancy.py:93-94
//   lw   = min(Bmp, Wmp // wpb)                          :104-108
//   rwl  = R==0 ? Wmp : R>Rmax ? 0 : rfs // roundup(R*ws, gran)   :111-124
//   lr   = CORRECTED min(Bmp, rwl // wpb)                :144-145
//          VERBATIM ceil((gran // (R*ws)) / wpb) * ceil(rfs/gran) :139-143
//   ls   = CORRECTED min(Bmp, Smax // S), VERBATIM ceil(Smax / S)  :148-160
//   blocks = min(lw, lr, ls); limiter tie-break warps > regs > smem  :176-184
//   active_warps = min(blocks*wpb, Wmp)                  :186
//
// Per-arch lookup tables live in shared memory and are built by every CTA
// in its prologue from the occx_arch_t rows passed in the parameter block:
//   lw_tab[wpb]      wpb in [0, Tmax/ws]   (u32)
//   r_tab[R]         R in [0, Rmax]: CORRECTED rwl(R) << 6, VERBATIM
//                    gran // (R*ws)        (u32)
// Division by wpb (<= 64) uses q = umulhi(n << 6, M6[wpb]) with
// M6[d] = ceil(2^26 / d): exact for n < 2^20 (error n*e/(d*2^26) < 1/d with
// e < d <= 64).  Smax // S uses a float reciprocal plus one integer
// correction step, valid because the clamp to Bmp (<= 255) is taken first.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/occx.h"

namespace occx {

constexpr int kMaxArchs = OCCX_MAX_ARCHS;
constexpr int kMaxWpb = 64;
constexpr uint64_t kIdxMask = (1ull << 34) - 1;

struct ArchParams {           // host-packed copy of occx_arch_t, kernel param
  occx_arch_t a[kMaxArchs];
  int n;
};

// Per-arch derived constants kept in shared memory (32 B, one LDS.128 x2).
struct DArch {
  uint32_t tmax, ws_shift, ws_m1, bmp;
  uint32_t wmp, rmax, smax, verb_c;    // verb_c = ceil(rfs / gran)
  uint32_t lw_off, r_off, rfs, gran;   // offsets into the u32 table area
  uint32_t ws, pad0, pad1, pad2;
};

struct SmemArch {
  DArch* d;          // [n]
  uint32_t* m6;      // [kMaxWpb + 1]
  uint32_t* tab;     // lw / r tables
};

// Bytes of the shared-memory area needed for the arch tables.
__host__ __device__ inline uint32_t arch_tab_words(const occx_arch_t& a) {
  return (uint32_t)(a.max_threads_per_block / a.warp_size + 1) +
         (uint32_t)(a.max_regs_per_thread + 1);
}
__host__ __device__ inline size_t arch_smem_bytes(const ArchParams& p) {
  size_t words = kMaxWpb + 1;
  for (int i = 0; i < p.n; ++i) words += arch_tab_words(p.a[i]);
  return sizeof(DArch) * p.n + words * 4;
}

__device__ __forceinline__ uint32_t ilog2u(uint32_t x) { return 31 - __clz(x); }

// Build the tables cooperatively; caller syncs afterwards.  `base` must be
// 16-byte aligned.
template <int MODE>
__device__ inline SmemArch build_arch_tables(const ArchParams& p, unsigned char* base) {
  SmemArch s;
  s.d = reinterpret_cast<DArch*>(base);
  s.m6 = reinterpret_cast<uint32_t*>(base + sizeof(DArch) * p.n);
  s.tab = s.m6 + (kMaxWpb + 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  // offsets: every thread computes the prefix sums (n <= 32, cheap)
  uint32_t off = 0;
  for (int i = 0; i < p.n; ++i) {
    const occx_arch_t& a = p.a[i];
    uint32_t nlw = (uint32_t)(a.max_threads_per_block / a.warp_size + 1);
    uint32_t nr = (uint32_t)(a.max_regs_per_thread + 1);
    if (tid == 0) {
      DArch d;
      d.tmax = a.max_threads_per_block;
      d.ws = a.warp_size;
      d.ws_shift = ilog2u((uint32_t)a.warp_size);
      d.ws_m1 = a.warp_size - 1;
      d.bmp = a.max_blocks_per_mp;
      d.wmp = a.max_warps_per_mp;
      d.rmax = a.max_regs_per_thread;
      d.smax = a.shared_mem_per_block;
      d.rfs = a.register_file_size;
      d.gran = a.register_alloc_granularity;
      d.verb_c = (uint32_t)((a.register_file_size + a.register_alloc_granularity - 1) /
                            a.register_alloc_granularity);
      d.lw_off = off;
      d.r_off = off + nlw;
      d.pad0 = d.pad1 = d.pad2 = 0;
      s.d[i] = d;
    }
    const uint32_t ws = a.warp_size, bmp = a.max_blocks_per_mp, wmp = a.max_warps_per_mp;
    for (uint32_t w = tid; w < nlw; w += nt) {
      uint32_t v = 0;
      if (w > 0) { uint32_t q = wmp / w; v = q < bmp ? q : bmp; }
      s.tab[off + w] = v;
    }
    const uint32_t gran = a.register_alloc_granularity, rfs = a.register_file_size;
    for (uint32_t r = tid; r < nr; r += nt) {
      uint32_t v;
      if (MODE == OCCX_MODE_CORRECTED) {
        uint32_t rwl;
        if (r == 0) rwl = wmp;
        else {
          uint32_t per_warp = ((r * ws + gran - 1) / gran) * gran;  // _round_up
          rwl = rfs / per_warp;
        }
        v = rwl << 6;
      } else {
        v = (r == 0) ? 0u : gran / (r * ws);   // regs_available (VERBATIM)
      }
      s.tab[off + nlw + r] = v;
    }
    off += nlw + nr;
  }
  for (int d = tid; d <= kMaxWpb; d += nt)
    s.m6[d] = d == 0 ? 0u : (uint32_t)(((1u << 26) + (uint32_t)d - 1) / (uint32_t)d);
  return s;
}

// Exact floor(n / d) for n < 2^20, 1 <= d <= 64.
__device__ __forceinline__ uint32_t div_small(uint32_t n_shl6, uint32_t m6) {
  return __umulhi(n_shl6, m6);
}

// floor(smax / s) clamped to bmp, for 0 < s <= smax < 2^24 and bmp <= 255.
__device__ __forceinline__ uint32_t smem_blocks_corrected(uint32_t smax, uint32_t s,
                                                          uint32_t bmp) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint2float_rn(s)));
  uint32_t q = __float2uint_rz(__fmul_rz(__uint2float_rn(smax), r));
  int32_t rem = (int32_t)(smax - q * s);
  q += (rem >= (int32_t)s) ? 1u : 0u;
  q -= (rem < 0) ? 1u : 0u;
  return (s * bmp <= smax) ? bmp : q;   // s*bmp < 2^32 (s < 2^24, bmp < 2^8)
}

struct OccOut {
  uint32_t wpb, lw, lr, ls, blocks, aw, limiter, status, rwl;
};

// The full evaluation (Kd).  `a` must be < n_arch (checked by the caller).
template <int MODE>
__device__ __forceinline__ OccOut eval_full(const SmemArch& s, uint32_t a, uint32_t T,
                                            uint32_t R, uint32_t S) {
  const DArch d = s.d[a];
  OccOut o;
  o.status = (T - 1u < d.tmax) ? OCCX_OK : OCCX_ERR_ILLEGAL_LAUNCH;
  uint32_t wpb = (T + d.ws_m1) >> d.ws_shift;
  o.wpb = wpb;
  if (o.status != OCCX_OK) {
    o.lw = o.lr = o.ls = o.blocks = o.aw = 0;
    o.limiter = OCCX_LIMIT_ILLEGAL;
    o.rwl = 0;
    return o;
  }
  uint32_t m6 = s.m6[wpb];
  o.lw = s.tab[d.lw_off + wpb];
  // registers
  if (R > d.rmax) { o.lr = 0; o.rwl = 0; }
  else if (R == 0) { o.lr = d.bmp; o.rwl = d.wmp; }
  else {
    uint32_t rv = s.tab[d.r_off + R];
    if (MODE == OCCX_MODE_CORRECTED) {
      o.rwl = rv >> 6;
      uint32_t q = div_small(rv, m6);
      o.lr = q < d.bmp ? q : d.bmp;
    } else {
      // ceil(regs_available / wpb) * ceil(rfs / gran), unclamped
      uint32_t q = div_small((rv + wpb - 1) << 6, m6);
      o.lr = q * d.verb_c;
      uint32_t per_warp = ((R * d.ws + d.gran - 1) / d.gran) * d.gran;
      o.rwl = d.rfs / per_warp;
    }
  }
  // shared memory (no thread dependence)
  if (S > d.smax) o.ls = 0;
  else if (S == 0) o.ls = d.bmp;
  else if (MODE == OCCX_MODE_CORRECTED) o.ls = smem_blocks_corrected(d.smax, S, d.bmp);
  else o.ls = (d.smax + S - 1) / S;
  uint32_t b = o.lw < o.lr ? o.lw : o.lr;
  b = b < o.ls ? b : o.ls;
  o.blocks = b;
  o.limiter = b == 0 ? OCCX_LIMIT_ILLEGAL
            : b == o.lw ? OCCX_LIMIT_WARPS
            : b == o.lr ? OCCX_LIMIT_REGISTERS : OCCX_LIMIT_SMEM;
  uint32_t aw = b * wpb;
  o.aw = aw < d.wmp ? aw : d.wmp;
  return o;
}

// Lean evaluation for the fused scorer: returns active_warps, 0 when the
// candidate is illegal (status != OK or blocks == 0).  Same arithmetic as
// eval_full (shared helpers), fewer outputs.
template <int MODE>
__device__ __forceinline__ uint32_t eval_active_warps(const SmemArch& s, uint32_t a,
                                                      uint32_t T, uint32_t R, uint32_t S) {
  const DArch d = s.d[a];
  if (T - 1u >= d.tmax) return 0;
  uint32_t wpb = (T + d.ws_m1) >> d.ws_shift;
  uint32_t lw = s.tab[d.lw_off + wpb];
  uint32_t lr;
  if (R > d.rmax) return 0;
  if (R == 0) lr = d.bmp;
  else {
    uint32_t rv = s.tab[d.r_off + R];
    uint32_t m6 = s.m6[wpb];
    if (MODE == OCCX_MODE_CORRECTED) {
      uint32_t q = div_small(rv, m6);
      lr = q < d.bmp ? q : d.bmp;
    } else {
      lr = div_small((rv + wpb - 1) << 6, m6) * d.verb_c;
    }
  }
  uint32_t ls;
  if (S > d.smax) return 0;
  if (MODE == OCCX_MODE_CORRECTED) ls = smem_blocks_corrected(d.smax, S, d.bmp);  // S==0 -> bmp
  else ls = (S == 0) ? d.bmp : (d.smax + S - 1) / S;
  uint32_t b = lw < lr ? lw : lr;
  b = b < ls ? b : ls;
  uint32_t aw = b * wpb;
  return aw < d.wmp ? aw : d.wmp;
}

// ---------------------------------------------------------------------------
// Warp-resident sorted top-k list: lane j < k holds the j-th largest key.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_list_insert(uint64_t& mine, uint64_t key, int k,
                                                 int lane) {
  unsigned gt = __ballot_sync(0xffffffffu, lane < k && mine > key);
  int pos = __popc(gt);
  uint64_t up = __shfl_up_sync(0xffffffffu, mine, 1);
  if (pos < k) {
    if (lane > pos && lane < k) mine = up;
    if (lane == pos) mine = key;
  }
}

__device__ __forceinline__ uint64_t warp_list_min(uint64_t mine, int k) {
  return __shfl_sync(0xffffffffu, mine, k - 1);
}

#define OCCX_CUDA_TRY(expr)                                        \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) return OCCX_ERR_CUDA;                   \
  } while (0)

}  // namespace occx

struct occx_ctx {
  int device;
  int sm_count;
  int max_smem_optin;
  int cc_major, cc_minor;
  uint32_t options;      // OCCX_CTX_* bits, fixed at create (include/occx.h)
};
