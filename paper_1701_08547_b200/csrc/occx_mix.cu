// occx_mix.cu -- K0 instruction-mix reducer (restates occmix/mix.py:245-261).
//
// Input: a CSR array of 4-byte instruction records (include/occx.h
// OCCX_INSTR) with n_kernels + 1 offsets.  Per record:
//   cls = LUT[sig]                 classify(), mix.py:176-187 (host-built LUT)
//   counts[cls] += 1               mix.py:256-257
//   if guard and cls not CTRL:     mix.py:258-259 (Unclassified included:
//       counts[PredIns] += 1        CATEGORY_OF.get(UNCLASSIFIED) is None)
//   reg_operands += regops         mix.py:260
//
// Work split (cost-balanced, segmented): warp w of the persistent grid
// owns the kernels k whose key off[k] + kKernelWeight * k lies in the w-th
// of W equal slices of the key range -- found by a 16-ary lower_bound per
// half-warp -- and streams
// that run of kernels as ONE contiguous record range in 256-record chunks,
// two LDG.128 per lane, the next chunk in flight while the current one is
// counted.  Chunks fully inside one kernel (the common case) are counted
// without masks; a chunk holding kernel boundaries is counted piece by piece
// with position masks.  Every warp gets ~1/W of the records-plus-kernels
// cost (at most one kernel more), so unequal kernel lengths do not leave a
// tail, and no kernel pads its last chunk.
//
// Counting: the class table holds, per (signature, guard), one byte
// 4c | 128g (c = class, g = the guard adds a PredIns); 0x7c is "not in this
// kernel".  A record's sixteen-nibble increment (class nibble, plus the
// PredIns nibble and a "guard counted" marker in the spare nibble 15) is
// read from a 64-entry u64 table at byte 2 * entry for 6 of a lane's 8
// records and computed as (1 << 4c) + g * (nibble 11 + nibble 15) for the
// other 2: the split balances the shared-memory and ALU pipes (sweep over
// 0/2/4/6/8 table records: 0.148/0.143/0.139/0.137/0.143 ms on config 3).
// Each piece of <= 8 records per lane is folded into byte counters (even /
// odd classes), reduced over the warp with 16-bit-lane REDUX.SUM before
// they can overflow.
// Dict insertion order (it decides the summation order of the FLOPS terms
// in mix.py:278) is recovered as first_key[c] = min over occurrences of
// 2*i (class of instruction i) or 2*i+1 (guard PredIns of instruction i).
// The streaming count does not track it: when a kernel is finished, its
// counters name the classes present, and its records are re-read from the
// start (L2 hits) in 32-position rows until each of them is located -- one
// MATCH.ANY per row (first_keys()).
#include "occx_common.cuh"

using namespace occx;

namespace {

#ifndef OCCX_K0_THREADS
#define OCCX_K0_THREADS 1024   // one CTA per SM; 64 registers per thread
#define OCCX_K0_DEEP 4         // ring chunks per warp (class tables <= 64 KB)
#define OCCX_K0_SHALLOW 2      // ring chunks per warp (larger class tables)
#endif
constexpr int kMixThreads = OCCX_K0_THREADS;
constexpr int kDeep = OCCX_K0_DEEP, kShallow = OCCX_K0_SHALLOW;
constexpr int kWarps = kMixThreads / 32;
constexpr uint32_t kChunk = 256;                      // records per warp-chunk (8 per lane)
constexpr int kFlushPieces = 255 / 8;                 // byte counters cannot overflow
constexpr uint32_t kPred = 11;                        // OpClass.PREDICATE device id
constexpr uint32_t kAbsent = 0xffffffffu;
constexpr uint32_t kNullLv = 0x7cu;                   // class 15, shift 124: counts nothing
constexpr uint32_t kMaxKernelRecords = 1u << 29;      // positions (2 * pos) and lane sums fit u32
#ifndef OCCX_K0_LDS
#define OCCX_K0_LDS 6
#endif
constexpr int kLdsRecords = OCCX_K0_LDS;              // of a lane's 8 records, via the table

struct MixParams {
  const uint32_t* instr;
  const uint64_t* off;
  uint32_t n_kernels;
  const uint8_t* sig_class;
  uint32_t n_sig;
  occx_mix_t* out;
};

// Sum 16 byte counters held as even classes (w[0] classes 0,2,4,6; w[1]
// 8,10,12,14) and odd classes (w[2] 1,3,5,7; w[3] 9,11,13,15) over the
// warp; lane c < 16 adds class c's total to `total`.  16-bit lanes: 32 x
// 255 < 2^16.  The eight warp sums (uniform) go through the warp's 8-word
// scratch so each lane picks its own 16-bit half with one LDS.U16.
__device__ __forceinline__ void reduce_counters_eo(const uint32_t (&w)[4], int lane,
                                                   uint32_t& total, uint32_t* xch) {
  uint32_t r[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    r[2 * q] = __reduce_add_sync(0xffffffffu, w[q] & 0x00ff00ffu);            // bytes 0, 2
    r[2 * q + 1] = __reduce_add_sync(0xffffffffu, (w[q] >> 8) & 0x00ff00ffu);  // bytes 1, 3
  }
  if (lane == 0) {
    reinterpret_cast<uint4*>(xch)[0] = make_uint4(r[0], r[1], r[2], r[3]);
    reinterpret_cast<uint4*>(xch)[1] = make_uint4(r[4], r[5], r[6], r[7]);
  }
  __syncwarp();
  // class c: word q = 2*(c & 1) + (c >> 3), byte b = (c >> 1) & 3 -> u16
  // index 4q + 2(b & 1) + (b >> 1)
  const uint32_t c = (uint32_t)lane & 15u, b = (c >> 1) & 3u;
  const uint32_t idx = 4u * (2u * (c & 1u) + (c >> 3)) + 2u * (b & 1u) + (b >> 1);
  const uint32_t v = reinterpret_cast<const uint16_t*>(xch)[idx];
  __syncwarp();
  total += v;
}

// Work split: a kernel costs about as much fixed work (boundary pieces,
// counter reduction, first-position rescan, output) as kKernelWeight
// records, so warps are balanced on off[k] + kKernelWeight * k (monotone in
// k) rather than on records alone: record-balanced runs varied by 14-33
// kernels per warp on config 3.
#ifndef OCCX_K0_KW
#define OCCX_K0_KW 1024
#endif
constexpr uint64_t kKernelWeight = OCCX_K0_KW;

// lower_bound: smallest k in [0, n] with off[k] + kKernelWeight * k >=
// bound (k = n satisfies it).  Each half-warp searches its own bound, 16
// probes per round.
__device__ __forceinline__ uint32_t seg_search(const uint64_t* off, uint32_t n, uint64_t bound,
                                               uint64_t off_n, uint64_t& off_lo, int lane) {
  const int half = lane >> 4, sub = lane & 15;
  uint32_t lo = 0, hi = n;
  uint64_t hv = off_n;                                     // off[hi]
  while (__any_sync(0xffffffffu, hi > lo)) {
    const uint32_t span = hi - lo;
    const uint32_t probe = lo + (uint32_t)(((uint64_t)span * (uint32_t)(sub + 1)) >> 4);
    const uint64_t v = __ldg(off + probe);
    const unsigned b = __ballot_sync(0xffffffffu, v + kKernelWeight * probe >= bound);
    const int f = __ffs((b >> (16 * half)) & 0xffffu) - 1;   // >= 0: probe 15 is hi
    const uint32_t pf = __shfl_sync(0xffffffffu, probe, 16 * half + f);
    const uint64_t vf = __shfl_sync(0xffffffffu, v, 16 * half + f);
    const uint32_t pp = __shfl_sync(0xffffffffu, probe, 16 * half + (f > 0 ? f - 1 : 0));
    if (hi > lo) {
      lo = f > 0 ? pp + 1 : lo;
      hi = pf;
      hv = vf;
    }
  }
  off_lo = hv;                                             // lo == hi: off[lo], no extra load
  return lo;
}

// Per-warp state of the kernel being reduced.
struct MixAcc {
  uint32_t be0, be1, bo0, bo1;     // byte counters: even / odd classes
  uint32_t regs, total;
  int pieces;
};

// Class records (the 15-entry identity class table, what the tokenizer
// emits): the increment table is indexed directly by the record's low byte
// (sig << 1 | guard), 256 entries + a zero (null) entry per lane, so a
// record's increment address is ONE byte permute (low byte << 8 | lane * 8)
// instead of mask + class-table LDS.U8 + shift.
constexpr uint32_t kIdentEntries = 257;
constexpr uint32_t kIdentNull = 256u << 8;
__device__ __forceinline__ uint32_t ident_offset(uint32_t r, uint32_t lane8) {
  return __byte_perm(r, lane8, 0x5504u);      // bytes: lane8.b0, r.b0, 0, 0
}

// A record's sixteen-nibble increment: lv is the lookup value -- a
// class-table byte (byte offset / 64 into the increment table, kNullLv = not
// in this kernel), or with kIdent the increment's byte offset itself
// (kIdentNull + lane * 8 = not in this kernel).
template <bool kIdent>
__device__ __forceinline__ void increment(uint32_t l, int e, const unsigned char* incb,
                                          uint32_t& dx, uint32_t& dy) {
  if (kIdent) {
    const uint2 d = *reinterpret_cast<const uint2*>(incb + l);
    dx = d.x;
    dy = d.y;
  } else if (e < kLdsRecords) {    // shared increment table: entry at byte 2 * l
    const uint2 d = *reinterpret_cast<const uint2*>(incb + (l << 6));   // entry l/4, this lane's copy
    dx = d.x;
    dy = d.y;
  } else {                         // arithmetic: balances the shared-memory and ALU pipes
    // class nibble increment 1 << 4c as a 64-bit shift (shift >= 64, the
    // null entry, gives 0); a counted guard adds PredIns (nibble 11) and the
    // marker (nibble 15): bit 7 of the entry times 0x10001000 >> 7
    asm("{\n\t.reg .b64 t;\n\tshl.b64 t, 1, %2;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "=r"(dx), "=r"(dy) : "r"(l & 0x7fu));
    dy += (l & 0x80u) * 0x200020u;
  }
}

// Fold a piece's per-lane nibble sums (<= 8 records: no nibble overflows)
// into the byte counters.
__device__ __forceinline__ void add_piece(MixAcc& a, uint32_t v0, uint32_t v1, uint32_t* xch,
                                          int lane) {
  a.be0 += v0 & 0x0f0f0f0fu;
  a.bo0 += (v0 >> 4) & 0x0f0f0f0fu;
  a.be1 += v1 & 0x0f0f0f0fu;
  a.bo1 += (v1 >> 4) & 0x0f0f0f0fu;
  if (++a.pieces == kFlushPieces) {
    a.pieces = 0;
    const uint32_t w[4] = {a.be0, a.be1, a.bo0, a.bo1};
    reduce_counters_eo(w, lane, a.total, xch);
    a.be0 = a.be1 = a.bo0 = a.bo1 = 0;
  }
}

// Count one piece.  Counting only: the first positions are found once per
// kernel by first_keys().
template <bool kIdent>
__device__ __forceinline__ void count_piece(MixAcc& a, const uint32_t (&lv)[8],
                                            const unsigned char* incb, uint32_t* xch, int lane) {
  uint32_t v0 = 0, v1 = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    uint32_t dx, dy;
    increment<kIdent>(lv[e], e, incb, dx, dy);
    v0 += dx;
    v1 += dy;
  }
  add_piece(a, v0, v1, xch, lane);
}

// Dict insertion order (mix.py:256-259): first_key[c] = 2 * (position of the
// first class-c record), and for PredIns the smaller of that and 2 * (first
// counted guard) + 1.  The kernel's records are re-read from its start (L2
// hits: the warp streamed them moments ago) in blocks of 128 positions,
// lane l holding positions 4l..4l+3, until every class the counters saw is
// located.  A lane's class mask (bit c, bit 15 = a counted guard) ORed
// over the lower lanes (a 5-step shuffle scan) leaves, in the lane's own
// mask, exactly the classes whose first occurrence in the block it holds.
// `need` bits: classes 0-14 (bit 11 = class-11 records, i.e. nibble 11
// minus the guards) and 15 = a counted guard.
template <bool kIdent>
__device__ __forceinline__ void first_keys(const uint32_t* kin, uint32_t n, uint32_t need,
                                           const unsigned char* lut, uint32_t lut_mask,
                                           const uint16_t* fbits, uint32_t* slot, int lane) {
  for (uint32_t s = 4u * (uint32_t)lane; need; s += 128u) {
    uint32_t bits[4], pres = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t pos = s + (uint32_t)j;
      if (kIdent) {               // class records: the mask from the record's low byte
        bits[j] = pos < n ? (uint32_t)fbits[__ldg(kin + pos) & 0xffu] : 0u;
      } else {
        const uint32_t lv = pos < n ? (uint32_t)lut[__ldg(kin + pos) & lut_mask] : kNullLv;
        // bit c (class 15 = not counted, e.g. the null entry), bit 15 = a counted guard
        bits[j] = ((1u << (lv >> 2 & 15u)) & 0x7fffu) | ((lv & 128u) << 8);
      }
      pres |= bits[j];
    }
    uint32_t incl = pres;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl |= y;
    }
    uint32_t excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0;
    uint32_t mine = pres & ~excl & need;
    if (mine) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t hit = bits[j] & mine;
        const uint32_t pos = s + (uint32_t)j;
        if (hit & 0x7fffu) slot[__ffs(hit & 0x7fffu) - 1] = 2u * pos;
        if (hit & 0x8000u) slot[15] = 2u * pos + 1u;
        mine &= ~hit;
      }
    }
    need &= ~__shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
}

template <bool kIdent>
__device__ __forceinline__ void finish_kernel(MixAcc& a, uint32_t* my_first, occx_mix_t* o,
                                              const uint32_t* kin, uint32_t n_instr,
                                              const unsigned char* lut, uint32_t lut_mask,
                                              const uint16_t* fbits, int lane) {
  {
    const uint32_t w[4] = {a.be0, a.be1, a.bo0, a.bo1};
    reduce_counters_eo(w, lane, a.total, my_first + 24);
  }
  // lane c < 16 holds nibble c's total: class c's count (PredIns includes the
  // counted guards), nibble 15 = counted guards
  const uint32_t guards = __shfl_sync(0xffffffffu, a.total, 15);
  const uint32_t own = lane == (int)kPred ? a.total - guards : a.total;
  const uint32_t need = __ballot_sync(0xffffffffu, lane < 16 && own != 0u) & 0xffffu;
  first_keys<kIdent>(kin, n_instr, need, lut, lut_mask, fbits, my_first, lane);
  uint32_t first = (lane < 16 && ((need >> lane) & 1u)) ? my_first[lane] : kAbsent;
  const uint32_t gfirst = __shfl_sync(0xffffffffu, first, 15);
  if (lane == (int)kPred && gfirst < first) first = gfirst;
  __syncwarp();
  // 64-bit total from two 16-bit-half warp sums (a lane's u32 cannot wrap:
  // kernels are < 2^29 records, <= 255 operands each, 1/32 of them per lane)
  const uint64_t reg_total =
      (uint64_t)__reduce_add_sync(0xffffffffu, a.regs & 0xffffu) +
      ((uint64_t)__reduce_add_sync(0xffffffffu, a.regs >> 16) << 16);
  if (lane < 16) {
    o->counts[lane] = lane < 15 ? a.total : 0u;
    o->first_key[lane] = lane < 15 ? first : kAbsent;
  }
  if (lane == 0) {
    o->reg_operands = reg_total;
    o->n_instr = n_instr;
    o->reserved = n_instr >= kMaxKernelRecords ? (uint32_t)OCCX_ERR_CAPACITY : 0u;
  }
  a = MixAcc{};
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared-memory layout: increments ([64][32] u64, or [257][32] when the
// call may use class records) | [warps][32] first positions (slots 0-15)
// and reduction scratch (24-31) | per-warp ring of kDepth chunks (kChunk
// records each) | class table.
constexpr int kFirstStride = 32;                      // per warp: 16 first slots, 8-word scratch at 24
__host__ __device__ constexpr size_t mix_inc_bytes(bool may_ident) {
  return may_ident ? kIdentEntries * 32u * 8u + 256u * 2u : 64u * 32u * 8u;   // + class masks
}
__host__ __device__ constexpr size_t mix_ring_offset(bool may_ident) {
  return mix_inc_bytes(may_ident) + kWarps * kFirstStride * 4;
}

// The streaming loop over the warp's record range (see the file comment).
struct MixRun {
  const uint4* gsrc;          // vector 64c + 32u of the warp's chunk grid, this lane
  uint4* my_ring;
  uint32_t ring_s, re, kb, ks, ke;
  uint64_t cs0;
};

template <bool kIdent, int kDepth>
__device__ __forceinline__ void mix_stream(const MixParams& p, const MixRun& w, const unsigned char* incb,
                                           uint32_t* my_first, const unsigned char* lut,
                                           uint32_t lut_mask, const uint16_t* fbits, int lane) {
  const uint32_t l4 = 4u * (uint32_t)lane, lane8 = 8u * (uint32_t)lane;
  const uint32_t null_lv = kIdent ? kIdentNull + lane8 : kNullLv;
  // kernel ends in a 32-wide register window: lane j holds off[kw + 1 + j]
  uint32_t k = w.ks, kw = w.ks, kb = w.kb;
  uint32_t ends = (uint32_t)(__ldg(p.off + min(kw + 1 + (uint32_t)lane, p.n_kernels)) - w.cs0);
  uint32_t kend = __shfl_sync(0xffffffffu, ends, 0);

  MixAcc a{};
  uint32_t cs = 0, slot = 0;
  while (true) {
    const uint32_t ce = cs + kChunk;
    cp_async_wait<kDepth - 1>();
    uint32_t r[8], lv[8];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint4 v = w.my_ring[64 * slot + 32 * u];
      r[4 * u + 0] = v.x; r[4 * u + 1] = v.y; r[4 * u + 2] = v.z; r[4 * u + 3] = v.w;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) lv[e] = kIdent ? ident_offset(r[e], lane8) : (uint32_t)lut[r[e] & lut_mask];
    {
      // refill this slot with chunk c + kDepth (the records are in registers)
      const uint32_t nb = cs + kDepth * kChunk;
      const uint4* src = w.gsrc + (size_t)(nb / 4);
#pragma unroll
      for (int u = 0; u < 2; ++u)
        cp_async16(w.ring_s + 16u * (64u * slot + 32u * u), src + 32 * u,
                   nb + 128u * u + l4 < w.re ? 16u : 0u);
      cp_async_commit();
      slot = slot + 1 == kDepth ? 0 : slot + 1;
    }
    if (kb <= cs && ce < kend) {
      // fast path: the whole chunk lies inside kernel k, which continues
#pragma unroll
      for (int e = 0; e < 8; ++e) a.regs += r[e] >> 17;
      count_piece<kIdent>(a, lv, incb, my_first + 24, lane);
    } else if (kb <= cs && ce <= w.re && kend < ce && k + 1 - kw < 32u &&
               __shfl_sync(0xffffffffu, ends, (int)(k + 1 - kw)) > ce) {
      // the common boundary chunk: kernel k (begun earlier) ends at sp inside
      // it and kernel k + 1 runs past its end -- one pass sums the chunk and
      // the piece before sp; k + 1's piece is the difference (per nibble:
      // <= 8 records each, so no borrows)
      const uint32_t sp = kend - cs;
      uint32_t a0 = 0, a1 = 0, p0 = 0, p1 = 0, ra = 0, rp = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t pic = 128u * (uint32_t)(e >> 2) + l4 + (uint32_t)(e & 3);
        uint32_t dx, dy;
        increment<kIdent>(lv[e], e, incb, dx, dy);
        const uint32_t rg = r[e] >> 17;
        a0 += dx;
        a1 += dy;
        ra += rg;
        if (pic < sp) {
          p0 += dx;
          p1 += dy;
          rp += rg;
        }
      }
      add_piece(a, p0, p1, my_first + 24, lane);
      a.regs += rp;
      finish_kernel<kIdent>(a, my_first, p.out + k, p.instr + (w.cs0 + kb), kend - kb, lut,
                            lut_mask, fbits, lane);
      ++k;
      kb = kend;
      kend = __shfl_sync(0xffffffffu, ends, (int)(k - kw));
      add_piece(a, a0 - p0, a1 - p1, my_first + 24, lane);
      a.regs += ra - rp;
    } else {
      while (true) {
        const uint32_t lo = cs > kb ? cs : kb, hi = ce < kend ? ce : kend;
        if (lo < hi) {
          const uint32_t plo = lo - cs, phi = hi - cs;
          uint32_t mv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t pic = 128u * (uint32_t)(e >> 2) + l4 + (uint32_t)(e & 3);
            const bool in = pic - plo < phi - plo;           // plo <= pic < phi
            mv[e] = in ? lv[e] : null_lv;
            a.regs += in ? (r[e] >> 17) : 0u;
          }
          count_piece<kIdent>(a, mv, incb, my_first + 24, lane);
        }
        if (kend > ce) break;                                // kernel continues in the next chunk
        finish_kernel<kIdent>(a, my_first, p.out + k, p.instr + (w.cs0 + kb), kend - kb, lut,
                              lut_mask, fbits, lane);
        if (++k == w.ke) {
          cp_async_wait<0>();
          return;
        }
        kb = kend;
        if (k - kw == 32) {                                  // next window of kernel ends
          kw = k;
          ends = (uint32_t)(__ldg(p.off + min(kw + 1 + (uint32_t)lane, p.n_kernels)) - w.cs0);
        }
        kend = __shfl_sync(0xffffffffu, ends, (int)(k - kw));
      }
    }
    cs = ce;
  }
}

template <int kDepth, bool kMayIdent>
__global__ void __launch_bounds__(kMixThreads, 1) mix_reduce_kernel(const __grid_constant__ MixParams p,
                                                                     uint32_t lut_mask) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* inc = reinterpret_cast<uint64_t*>(smem);
  uint32_t* firsts = reinterpret_cast<uint32_t*>(smem + mix_inc_bytes(kMayIdent));
  uint4* ring = reinterpret_cast<uint4*>(smem + mix_ring_offset(kMayIdent));
  unsigned char* lut = reinterpret_cast<unsigned char*>(ring + (size_t)kWarps * kDepth * (kChunk / 4));
  const int lane = threadIdx.x & 31;
  const uint32_t warps_total = gridDim.x * kWarps;
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);

  // this warp's kernel run [ks, ke): half-warp 0 searches bound(gw), half 1 bound(gw + 1)
  const uint64_t base = __ldg(p.off), n_rec = __ldg(p.off + p.n_kernels) - base;
  if (n_rec >> 32) {              // positions are u32: flag every kernel, count nothing
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < p.n_kernels;
         k += gridDim.x * blockDim.x) {
      p.out[k].n_instr = 0;
      p.out[k].reserved = (uint32_t)OCCX_ERR_CAPACITY;
    }
    return;
  }
  uint32_t ks, ke;
  uint64_t rs, rend;
  {
    const uint32_t w = gw + (uint32_t)(lane >> 4);
    const uint64_t total = n_rec + kKernelWeight * p.n_kernels;          // < 2^42
    const uint64_t bound = base + (total * (uint64_t)w) / warps_total;
    uint64_t ov;
    uint32_t r = seg_search(p.off, p.n_kernels, bound, base + n_rec, ov, lane);
    if (w >= warps_total) {                                // trailing empty kernels: last warp
      r = p.n_kernels;
      ov = base + n_rec;
    }
    ks = __shfl_sync(0xffffffffu, r, 0);
    ke = __shfl_sync(0xffffffffu, r, 16);
    rs = __shfl_sync(0xffffffffu, ov, 0);                  // off[ks]
    rend = __shfl_sync(0xffffffffu, ov, 16);               // off[ke]
  }

  // Positions are kept relative to the warp's first chunk start cs0 (u32:
  // a call holds < 2^32 records).  The chunk grid is aligned to 16-byte
  // addresses; lane holds records c + 128u + 4*lane + j (u = 0, 1; j = 0..3)
  // of chunk c, copied by the lane itself into its slots of the warp's
  // ring (cp.async, zero-fill past the end), so only the lane's own
  // wait_group orders them -- no barriers.
  MixRun w;
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(p.instr) >> 2) & 3u;
  w.cs0 = ((rs + mis) & ~3ull) - mis;                      // may be "-mis" (wraps; used as an offset)
  w.re = (uint32_t)(rend - w.cs0);
  w.gsrc = reinterpret_cast<const uint4*>(p.instr + w.cs0) + lane;   // vector 64c + 32u
  w.my_ring = ring + (size_t)(threadIdx.x >> 5) * kDepth * (kChunk / 4) + lane;
  w.ring_s = (uint32_t)__cvta_generic_to_shared(w.my_ring);
  w.kb = (uint32_t)(rs - w.cs0);
  w.ks = ks;
  w.ke = ke;
  // the ring fill goes out before the tables are built (its DRAM latency
  // covers them)
  const uint32_t l4 = 4u * (uint32_t)lane;
#pragma unroll
  for (int d = 0; d < kDepth; ++d) {
    if (ks >= ke) break;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t i = (uint32_t)d * kChunk + 128u * u + l4;
      cp_async16(w.ring_s + 16u * (64u * d + 32u * u), w.gsrc + 64 * d + 32 * u, i < w.re ? 16u : 0u);
    }
    cp_async_commit();
  }

  // class table indexed by the record's low 17 bits (sig << 1 | guard) and
  // the mask lut_mask (power of two - 1 >= 2*n_sig + 1): entry = 4 * class
  // | 128 when the guard adds a PredIns (mix.py:258-259: not for CTRL
  // classes 11-13).  Signatures >= n_sig count as Unclassified (out-of-range
  // ids are a caller error; the mask keeps them inside the table).
  const uint32_t words = (lut_mask + 1) / 8;                // 4 signatures per word pair
  const bool lut_vec = (reinterpret_cast<uintptr_t>(p.sig_class) & 3u) == 0;
  bool ident = kMayIdent;   // the table is the identity over its n_sig == 15 entries
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
    uint32_t w4 = 0;
    if (4 * i < p.n_sig) {
      if (lut_vec && 4 * i + 4 <= p.n_sig) {             // whole word inside the table
        w4 = __ldg(reinterpret_cast<const uint32_t*>(p.sig_class) + i);
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (4 * i + b < p.n_sig) w4 |= (uint32_t)__ldg(p.sig_class + 4 * i + b) << (8 * b);
      }
    }
    uint32_t o[2];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t sig = 4 * i + (uint32_t)b;
      const uint32_t c = sig < p.n_sig ? ((w4 >> (8 * b)) & 15u) : 14u;
      if (sig < p.n_sig && ((w4 >> (8 * b)) & 0xffu) != sig) ident = false;
      const uint32_t g = (c < 11 || c == 14) ? 16u : 0u;
      const uint32_t pair = (c << 2) | (((c << 2) | (g << 3)) << 8);   // byte: 4c | guard<<7
      if (b & 1) o[b >> 1] |= pair << 16; else o[b >> 1] = pair;
    }
    *reinterpret_cast<uint2*>(lut + 8 * i) = make_uint2(o[0], o[1]);
  }
  ident = kMayIdent && __syncthreads_and(ident) != 0;

  // increment table, replicated per lane ([entry][lane]): lane l reads banks
  // 2l, 2l+1 only, so an LDS.64 of 32 lanes is two conflict-free wavefronts
  // whatever the classes.  Indexed by class-table byte / 4 (= c + 32 *
  // guard; entries 15..31 and 47..63 are zero, 31 = the null entry), or for
  // class records by the record's low byte (sig' = byte >> 1 & 31: the
  // class-table lookup of the same record under lut_mask = 63, 256 = null).
  const uint32_t n_inc = (ident ? kIdentEntries : 64u) * 32u;
  for (uint32_t i = threadIdx.x; i < n_inc; i += blockDim.x) {
    const uint32_t e = i >> 5;
    uint32_t c, g;
    if (ident) {
      const uint32_t s = e >> 1 & 31u;
      c = e >= 256u ? 15u : (s < 15u ? s : 14u);
      g = e & 1u;
    } else {
      c = e & 31u;
      g = e >> 5;
    }
    uint64_t v = 0;
    if (c < 15) {
      v = 1ull << (4 * c);
      if (g && !(c >= 11 && c <= 13)) v += (1ull << (4 * kPred)) + (1ull << 60);  // PredIns + marker
    }
    inc[i] = v;
  }
  // class records: first_keys()' class mask per low byte (bit c, bit 15 =
  // a counted guard), after the increments
  uint16_t* fbits = reinterpret_cast<uint16_t*>(inc + kIdentEntries * 32u);
  if (ident)
    for (uint32_t i = threadIdx.x; i < 256u; i += blockDim.x) {
      const uint32_t s = i >> 1 & 31u, c = s < 15u ? s : 14u;
      fbits[i] = (uint16_t)((1u << c) | ((i & 1u) && !(c >= 11 && c <= 13) ? 0x8000u : 0u));
    }
  for (uint32_t i = threadIdx.x; i < kWarps * kFirstStride; i += blockDim.x) firsts[i] = kAbsent;
  __syncthreads();
  if (ks >= ke) return;
  uint32_t* my_first = firsts + (threadIdx.x >> 5) * kFirstStride;

  if (kMayIdent && ident)
    mix_stream<true, kDepth>(p, w, reinterpret_cast<const unsigned char*>(inc), my_first, lut,
                             lut_mask, fbits, lane);
  else
    mix_stream<false, kDepth>(p, w, reinterpret_cast<const unsigned char*>(inc) + 8 * lane,
                              my_first, lut, lut_mask, fbits, lane);
}

}  // namespace

extern "C" int occx_mix_reduce(const occx_ctx* ctx, const uint32_t* d_instr,
                               const uint64_t* d_kernel_off, uint32_t n_kernels,
                               const uint8_t* d_sig_class, uint32_t n_sig, occx_mix_t* d_out,
                               void* stream) {
  if (!ctx || n_sig == 0 || n_sig > 65535) return OCCX_ERR_VALUE;
  if ((reinterpret_cast<uintptr_t>(d_instr) & 3u) != 0) return OCCX_ERR_VALUE;
  if (n_kernels == 0) return OCCX_OK;
  MixParams p{};
  p.instr = d_instr;
  p.off = d_kernel_off;
  p.n_kernels = n_kernels;
  p.sig_class = d_sig_class;
  p.n_sig = n_sig;
  p.out = d_out;
  uint32_t lut_bytes = 64;                                 // power of two >= 2 * (n_sig + 1)
  while (lut_bytes < 2 * (n_sig + 1)) lut_bytes <<= 1;
  const bool deep = lut_bytes <= 64 * 1024;
  const bool may_ident = n_sig == 15;                      // a 15-entry table may be the identity
  const size_t ring = (size_t)kWarps * (deep ? kDeep : kShallow) * kChunk * 4;
  const size_t smem = mix_ring_offset(may_ident) + ring + lut_bytes;
  const void* fn = may_ident ? (const void*)mix_reduce_kernel<kDeep, true>
                   : deep    ? (const void*)mix_reduce_kernel<kDeep, false>
                             : (const void*)mix_reduce_kernel<kShallow, false>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return OCCX_ERR_CUDA;
  // persistent: one 32-warp CTA per SM (one copy of the class table per SM)
  const uint32_t grid = (uint32_t)ctx->sm_count;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (may_ident)
    mix_reduce_kernel<kDeep, true><<<grid, kMixThreads, smem, st>>>(p, lut_bytes - 1);
  else if (deep)
    mix_reduce_kernel<kDeep, false><<<grid, kMixThreads, smem, st>>>(p, lut_bytes - 1);
  else
    mix_reduce_kernel<kShallow, false><<<grid, kMixThreads, smem, st>>>(p, lut_bytes - 1);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}
