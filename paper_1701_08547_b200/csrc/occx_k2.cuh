// occx_k2.cuh -- K2, the fused score + per-segment top-k hot path.
//
// Two feeds share one branch-free per-candidate core (k2_key):
//   * TMA  (default): warp-specialised persistent CTA, one per SM.  Warp 0
//     lane 0 streams 16 KB tiles of candidate records HBM -> shared memory
//     with cp.async.bulk into an 8-stage mbarrier ring; 16 consumer warps
//     read records with conflict-free LDS.128, score them and release the
//     stage.  HBM traffic is decoupled from the integer work.
//   * LDG  (fallback / A-B): each thread streams records with 128-bit
//     non-allocating loads, 4 in flight.
//
// Per-candidate work (CORRECTED, see occx_common.cuh for the maths):
//   T,R,arch unpack      LOP, LOP, PRMT
//   arch row             2 x LDS.128 (broadcast: records are segment-major)
//   warps                Tc = min(T, Tmax); wpb = (Tc+ws-1)>>ws_shift;
//                        LDS.64 {lw, M6[wpb]}   (wpb = 0 row is {0,0})
//   registers            LDS r_tab[min(R, Rmax+1)]: rwl<<6, 0xFFFFFFC0 at
//                        R=0 (-> Bmp), 0 at Rmax+1 (-> 0 blocks);
//                        lr = min(umulhi(r, M6), Bmp)
//   shared memory        float reciprocal + one integer correction
//   blocks, warps        VIMNMX3, IMAD, VIMNMX
//   membership / rank    vtab row (smem copy): {seg, key_hi_base} + one
//                        interleaved member word
//   key                  LOP3 x2, 64-bit running inverse index
//   top-k                LDS.64 threshold compare + ballot; rare inserts
#pragma once
#include "occx_common.cuh"

namespace occx {

constexpr int kTStride = 2 * (kMaxWpb + 1);     // words of one arch's {lw, M6} table
constexpr int kVtSmemMax = 1024;                // vtab rows copied to smem (32 KB)

struct K2Arch {
  uint4 p0;   // {tmax, ws_m1, ws_shift, bmp}
  uint4 p1;   // {wmp, rmax + 1, smax, t_off}   r_tab at t_off + kTStride
};

// words of one arch's tables, kept even so every {lw, M6} pair is 8-byte aligned
__host__ __device__ inline uint32_t k2_arch_words(const occx_arch_t& a) {
  return (kTStride + (uint32_t)a.max_regs_per_thread + 2 + 1) & ~1u;
}
__host__ __device__ inline size_t k2_tab_words(const ArchParams& p) {
  size_t w = 0;
  for (int i = 0; i < p.n; ++i) w += k2_arch_words(p.a[i]);
  return w;
}
__host__ __device__ inline size_t k2_arch_bytes(const ArchParams& p) {
  return (sizeof(K2Arch) * p.n + k2_tab_words(p) * 4 + 15) & ~size_t(15);
}

// Build the arch rows and tables; caller syncs.
template <int MODE>
__device__ inline void k2_build(const ArchParams& p, K2Arch* rows, uint32_t* tab) {
  const int tid = threadIdx.x, nt = blockDim.x;
  uint32_t off = 0;
  for (int i = 0; i < p.n; ++i) {
    const occx_arch_t& a = p.a[i];
    const uint32_t ws = a.warp_size, bmp = a.max_blocks_per_mp, wmp = a.max_warps_per_mp;
    const uint32_t rmax = a.max_regs_per_thread, gran = a.register_alloc_granularity;
    const uint32_t rfs = a.register_file_size;
    if (tid == 0) {
      K2Arch r;
      r.p0 = make_uint4(a.max_threads_per_block, ws - 1, ilog2u(ws), bmp);
      r.p1 = make_uint4(wmp, rmax + 1, a.shared_mem_per_block, off);
      rows[i] = r;
    }
    const uint32_t nwpb = (uint32_t)(a.max_threads_per_block / a.warp_size);
    for (uint32_t w = tid; w <= kMaxWpb; w += nt) {
      uint32_t lw = 0, m6 = 0;
      if (w >= 1 && w <= nwpb) {
        const uint32_t q = wmp / w;
        lw = q < bmp ? q : bmp;
        m6 = (uint32_t)(((1u << 26) + w - 1) / w);
      }
      tab[off + 2 * w] = lw;
      tab[off + 2 * w + 1] = m6;
    }
    for (uint32_t r = tid; r <= rmax + 1; r += nt) {
      uint32_t v;
      if (MODE == OCCX_MODE_CORRECTED) {
        if (r == 0) v = 0xFFFFFFC0u;                 // unspecified -> Bmp after the clamp
        else if (r > rmax) v = 0;                    // over the limit -> 0 blocks
        else v = (rfs / (((r * ws + gran - 1) / gran) * gran)) << 6;
      } else {
        if (r == 0) v = 0;
        else if (r > rmax) v = (rfs + gran - 1) / gran;   // sentinel slot holds verb_c
        else v = gran / (r * ws);
      }
      tab[off + kTStride + r] = v;
    }
    off += k2_arch_words(a);
  }
}

struct K2Ctx {
  const K2Arch* rows;
  const uint32_t* tab;
  const occx_vent_t* vt;
  uint32_t n_arch, n_var;
};

// Per-thread cache of everything that depends only on (T, variant, arch).
// Segment-major records repeat that triple for long runs (R and S vary
// fastest), so the warp refills the cache only when some lane's triple
// changed (one VOTE.ALL per candidate decides, warp-uniformly).
struct K2Cache {
  uint32_t x, z, w;          // raw record words the cache was filled from (masked compare)
  uint32_t wpb, lw, m6, r_off, rmax_p1, bmp, wmp, smax;
  float smax_f;
  uint32_t key_hi, seg, ok;  // key bits 63/62/61/53-34, segment, record+threads legal
};

template <bool VT_SMEM>
__device__ __forceinline__ void k2_fill(const K2Ctx& c, const uint4 r, K2Cache& k) {
  const uint32_t T = r.z & 0xffffu;
  const uint32_t a = __byte_perm(r.w, 0, 0x4442);
  const uint32_t ac = min(a, c.n_arch - 1);
  const uint4 p0 = c.rows[ac].p0, p1 = c.rows[ac].p1;
  const uint32_t Tc = min(T, p0.x);
  const uint32_t wpb = (Tc + p0.y) >> p0.z;
  const uint2 tw = *reinterpret_cast<const uint2*>(c.tab + p1.w + 2 * wpb);
  const uint32_t v = r.x;
  const uint32_t vcl = min(v, c.n_var - 1);
  const occx_vent_t* e = c.vt + (vcl * c.n_arch + ac);
  const uint32_t tb = (T >> 5) - 1u;   // mask bit of T = 32 (b + 1): T in [32, 2048]
  uint2 sh;            // {seg, key_hi}
  uint32_t word;
  if (VT_SMEM) {       // explicit address spaces: LDS for the smem copy, LDG.NC otherwise
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(e);
    asm("ld.shared.v2.u32 {%0, %1}, [%2+16];" : "=r"(sh.x), "=r"(sh.y) : "r"(a0));
    asm("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(a0 + ((tb >> 2) & 12u)));
  } else {
    sh = __ldg(reinterpret_cast<const uint2*>(&e->seg));
    word = __ldg(&e->member[(tb >> 4) & 3u]);
  }
  uint32_t bits = (word >> ((tb & 15u) << 1)) & 3u;
  bits = ((T & 31u) | (tb >> 6)) ? 0u : bits;                       // T % 32 == 0, 32 <= T <= 2048
  k.x = r.x;
  k.z = r.z;
  k.w = r.w;
  k.wpb = wpb;
  k.lw = tw.x;
  k.m6 = tw.y;
  k.r_off = p1.w + kTStride;
  k.rmax_p1 = p1.y;
  k.bmp = p0.w;
  k.wmp = p1.x;
  k.smax = p1.z;
  k.smax_f = __uint2float_rn(p1.z);
  k.key_hi = sh.y | (bits << 29);
  k.seg = sh.x;
  k.ok = (a < c.n_arch) & (v < c.n_var) & (T <= p0.x);
}

__device__ __forceinline__ bool k2_hit(const K2Cache& k, const uint4 r) {
  return ((r.x ^ k.x) | ((r.z ^ k.z) & 0xffffu) | ((r.w ^ k.w) & 0xff0000u)) == 0;
}

// The (R, S)-dependent remainder.  Returns the key (0 = not a legal
// candidate); seg is the cached segment.
template <int MODE>
__device__ __forceinline__ uint64_t k2_key(const K2Ctx& c, const K2Cache& k, const uint4 r,
                                           const uint64_t inv) {
  const uint32_t R = r.w & 0xffffu, S = r.y;
  const uint32_t rv = c.tab[k.r_off + min(R, k.rmax_p1)];
  uint32_t b;
  if (MODE == OCCX_MODE_CORRECTED) {
    // min(lw, lr, ls) with lr = min(Bmp, rwl // wpb) and ls = min(Bmp, Smax // S).
    // Only min(m, Smax // S) is needed (m <= Bmp <= 255): the float quotient is
    // within 1 of the truth whenever it is below 2^8 and one integer
    // correction makes it exact; larger quotients stay >= m.
    const uint32_t m = min(min(k.lw, __umulhi(rv, k.m6)), k.bmp);
    float rc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(__uint2float_rn(S)));
    uint32_t q = __float2uint_rz(__fmul_rz(k.smax_f, rc));
    const int32_t rem = (int32_t)(k.smax - q * S);
    q += (rem >= (int32_t)S) ? 1u : 0u;
    q -= (rem < 0) ? 1u : 0u;
    const uint32_t ls = (S - 1u >= k.smax) ? (S == 0 ? 0xffffffffu : 0u) : q;
    b = min(m, ls);
  } else {
    const uint32_t vc = c.tab[k.r_off + k.rmax_p1];
    const uint32_t q = __umulhi((rv + k.wpb - 1) << 6, k.m6) * vc;
    const uint32_t lr = R == 0 ? k.bmp : (R >= k.rmax_p1 ? 0u : q);
    const uint32_t ls = S == 0 ? k.bmp : (S > k.smax ? 0u : (k.smax + S - 1) / S);
    b = min(min(k.lw, lr), ls);
  }
  const uint32_t aw = min(b * k.wpb, k.wmp);
  const bool ok = k.ok & (aw != 0);
  const uint32_t hi = k.key_hi | (aw << 22) | (uint32_t)(inv >> 32);
  return ok ? (((uint64_t)hi << 32) | (uint32_t)inv) : 0ull;
}

}  // namespace occx
