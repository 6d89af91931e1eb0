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
// Work split (record-balanced, segmented): warp w of the persistent grid
// owns the kernels whose first record lies in [off0 + w*N/W, off0 +
// (w+1)*N/W) -- found by a 16-ary lower_bound per half-warp -- and streams
// that run of kernels as ONE contiguous record range in 256-record chunks,
// two LDG.128 per lane, the next chunk in flight while the current one is
// counted.  Chunks fully inside one kernel (the common case) are counted
// without masks; a chunk holding kernel boundaries is counted piece by piece
// with position masks.  Every warp gets ~N/W records (at most one kernel
// more), so unequal kernel lengths do not leave a tail, and no kernel pads
// its last chunk.
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
// 2*i (class of instruction i) or 2*i+1 (guard PredIns of instruction i);
// a warp OR-reduction per piece finds classes not seen before in the
// kernel and only then are their first positions located (one shared
// atomicMin per (row, class) leader found with MATCH.ANY).
#include "occx_common.cuh"

using namespace occx;

namespace {

constexpr int kMixThreads = 1024;
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

// lower_bound: smallest k in [0, n] with off[k] >= bound (off[n] >= bound
// holds).  Each half-warp searches its own bound, 16 probes per round.
__device__ __forceinline__ uint32_t seg_search(const uint64_t* off, uint32_t n, uint64_t bound,
                                               int lane) {
  const int half = lane >> 4, sub = lane & 15;
  uint32_t lo = 0, hi = n;
  while (__any_sync(0xffffffffu, hi > lo)) {
    const uint32_t span = hi - lo;
    const uint32_t probe = lo + (uint32_t)(((uint64_t)span * (uint32_t)(sub + 1)) >> 4);
    const unsigned b = __ballot_sync(0xffffffffu, __ldg(off + probe) >= bound);
    const int f = __ffs((b >> (16 * half)) & 0xffffu) - 1;   // >= 0: probe 15 is hi
    const uint32_t pf = __shfl_sync(0xffffffffu, probe, 16 * half + f);
    const uint32_t pp = __shfl_sync(0xffffffffu, probe, 16 * half + (f > 0 ? f - 1 : 0));
    if (hi > lo) {
      lo = f > 0 ? pp + 1 : lo;
      hi = pf;
    }
  }
  return lo;
}

// One bit (the nibble's low bit) per non-zero 4-bit counter.
__device__ __forceinline__ uint32_t nibble_presence(uint32_t v) {
  const uint32_t t = v | (v >> 1);
  return (t | (t >> 2)) & 0x11111111u;
}

// Per-warp state of the kernel being reduced.
struct MixAcc {
  uint32_t be0, be1, bo0, bo1;     // byte counters: even / odd classes
  uint32_t seen_lo, seen_hi;       // nibble presence so far in this kernel
  uint32_t regs, total;
  int pieces;
};

// Count one piece: lv[e] are the class-table values (byte offsets into the
// increment table, kNullLv = not in this kernel); keybase + pic(e) is the
// record's position in its kernel.
__device__ __forceinline__ void count_piece(MixAcc& a, const uint32_t (&lv)[8],
                                            const unsigned char* incb, uint32_t* my_first,
                                            uint32_t keybase, int lane) {
  uint32_t h0 = 0, h1 = 0, v0 = 0, v1 = 0;        // h: records of the first row block (u = 0)
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    // class nibble increment 1 << 4c as a 64-bit shift (shift >= 64, the
    // null entry, gives 0); a counted guard adds PredIns (nibble 11) and the
    // marker (nibble 15): bit 7 of the entry times 0x10001000 >> 7
    const uint32_t l = lv[e];
    uint32_t dx, dy;
    if (e < kLdsRecords) {         // shared increment table: entry at byte 2 * l
      const uint2 d = *reinterpret_cast<const uint2*>(incb + (l << 6));   // entry l/4, this lane's copy
      dx = d.x;
      dy = d.y;
    } else {                       // arithmetic: balances the shared-memory and ALU pipes
      asm("{\n\t.reg .b64 t;\n\tshl.b64 t, 1, %2;\n\tmov.b64 {%0, %1}, t;\n\t}"
          : "=r"(dx), "=r"(dy) : "r"(l & 0x7fu));
      dy += (l & 0x80u) * 0x200020u;
    }
    if (e < 4) {
      h0 += dx;
      h1 += dy;
    } else {
      v0 += dx;
      v1 += dy;
    }
  }
  v0 += h0;
  v1 += h1;
  // classes (nibbles) present in this lane's piece -> warp presence
  const uint32_t pres_lo = __reduce_or_sync(0xffffffffu, nibble_presence(v0));
  const uint32_t pres_hi = __reduce_or_sync(0xffffffffu, nibble_presence(v1));
  const uint32_t new_lo = pres_lo & ~a.seen_lo, new_hi = pres_hi & ~a.seen_hi;
  if (new_lo | new_hi) {                                   // a class new to this kernel
    a.seen_lo |= pres_lo;
    a.seen_hi |= pres_hi;
    // Record e of every lane forms a row ordered by lane, so the first
    // occurrence of a class in the row is its lowest lane: one leader per
    // (row, class) does the shared atomicMin (no same-address serialisation).
    // Rows 0-3 (u = 0) hold positions below rows 4-7; the second block is
    // only searched when a new class is absent from the first.
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const uint32_t first_lo = __reduce_or_sync(0xffffffffu, nibble_presence(h0));
    const uint32_t first_hi = __reduce_or_sync(0xffffffffu, nibble_presence(h1));
    // rows of block 0 only when a new class occurs there, of block 1 only
    // when one is absent from block 0 (a piece may start or end mid-chunk);
    // the guard rows only while no counted guard has been seen (nibble 15)
    const int row0 = ((new_lo & first_lo) | (new_hi & first_hi)) ? 0 : 4;
    const int rows = ((new_lo & ~first_lo) | (new_hi & ~first_hi)) ? 8 : 4;
    const bool guard_new = (new_hi & 0x10000000u) != 0u;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e >= rows) break;
      if (e < row0) continue;
      const uint32_t c = lv[e] >> 2 & 15u;
      const uint32_t pos = keybase + 128u * (uint32_t)(e >> 2) + 4u * (uint32_t)lane + (uint32_t)(e & 3);
      const uint32_t same = __match_any_sync(0xffffffffu, c);
      if ((same & lt) == 0) atomicMin(my_first + c, 2u * pos);   // slot 15 (padding) is never read
      // guard PredIns (non-CTRL class): key 2*pos + 1, tracked in slot 16
      if (guard_new) {
        const uint32_t gb = __ballot_sync(0xffffffffu, lv[e] & 128u);
        if ((lv[e] & 128u) && (gb & lt) == 0) atomicMin(my_first + 16, 2u * pos + 1);
      }
    }
  }
  a.be0 += v0 & 0x0f0f0f0fu;
  a.bo0 += (v0 >> 4) & 0x0f0f0f0fu;
  a.be1 += v1 & 0x0f0f0f0fu;
  a.bo1 += (v1 >> 4) & 0x0f0f0f0fu;
  if (++a.pieces == kFlushPieces) {
    a.pieces = 0;
    const uint32_t w[4] = {a.be0, a.be1, a.bo0, a.bo1};
    reduce_counters_eo(w, lane, a.total, my_first + 24);
    a.be0 = a.be1 = a.bo0 = a.bo1 = 0;
  }
}

__device__ __forceinline__ void finish_kernel(MixAcc& a, uint32_t* my_first, occx_mix_t* o,
                                              uint32_t n_instr, int lane) {
  {
    const uint32_t w[4] = {a.be0, a.be1, a.bo0, a.bo1};
    reduce_counters_eo(w, lane, a.total, my_first + 24);
  }
  uint32_t first = lane < 17 ? my_first[lane] : kAbsent;
  const uint32_t gfirst = __shfl_sync(0xffffffffu, first, 16);
  if (lane == (int)kPred && gfirst < first) first = gfirst;
  if (lane < 17) my_first[lane] = kAbsent;               // reset for the warp's next kernel
  __syncwarp();
  // 64-bit total from two 16-bit-half warp sums (a lane's u32 cannot wrap:
  // kernels are < 2^29 records, <= 255 operands each, 1/32 of them per lane)
  const uint64_t reg_total =
      (uint64_t)__reduce_add_sync(0xffffffffu, a.regs & 0xffffu) +
      ((uint64_t)__reduce_add_sync(0xffffffffu, a.regs >> 16) << 16);
  if (lane < 16) {
    o->counts[lane] = lane < 15 ? a.total : 0u;
    o->first_key[lane] = (lane < 15 && a.total) ? first : kAbsent;
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

// Shared-memory layout: [64] u64 increments | [warps][32] first positions
// (slots 0-16) and reduction scratch (24-31) | per-warp ring of kDepth chunks (kChunk records each) | class table.
constexpr int kFirstStride = 32;                      // per warp: 17 first slots, 8-word scratch at 24
__host__ __device__ constexpr size_t mix_ring_offset() { return 64 * 32 * 8 + kWarps * kFirstStride * 4; }

template <int kDepth>
__global__ void __launch_bounds__(kMixThreads, 1) mix_reduce_kernel(const __grid_constant__ MixParams p,
                                                                     uint32_t lut_mask) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* inc = reinterpret_cast<uint64_t*>(smem);
  uint32_t* firsts = reinterpret_cast<uint32_t*>(inc + 64 * 32);
  uint4* ring = reinterpret_cast<uint4*>(smem + mix_ring_offset());
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
  {
    const uint32_t w = gw + (uint32_t)(lane >> 4);
    const uint64_t bound = base + (n_rec * (uint64_t)w) / warps_total;   // n_rec < 2^32
    uint32_t r = seg_search(p.off, p.n_kernels, bound, lane);
    if (w >= warps_total) r = p.n_kernels;                 // trailing empty kernels: last warp
    ks = __shfl_sync(0xffffffffu, r, 0);
    ke = __shfl_sync(0xffffffffu, r, 16);
  }

  // increment table indexed by class-table byte / 4 (= c + 32 * guard):
  // entries 15..31 and 47..63 are zero (31 = the null entry).  Replicated
  // per lane ([entry][lane], 16 KB): lane l reads banks 2l, 2l+1 only, so an
  // LDS.64 of 32 lanes is two conflict-free wavefronts whatever the classes.
  for (uint32_t i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
    const uint32_t e = i >> 5, c = e & 31u, g = e >> 5;
    uint64_t v = 0;
    if (c < 15) {
      v = 1ull << (4 * c);
      if (g && !(c >= 11 && c <= 13)) v += (1ull << (4 * kPred)) + (1ull << 60);  // PredIns + marker
    }
    inc[i] = v;
  }
  for (uint32_t i = threadIdx.x; i < kWarps * kFirstStride; i += blockDim.x) firsts[i] = kAbsent;
  // class table indexed by the record's low 17 bits (sig << 1 | guard) and
  // the mask lut_mask (power of two - 1 >= 2*n_sig + 1): entry = 8 * (class
  // | 16 when the guard adds a PredIns), i.e. the byte offset of the
  // increment.  Signatures >= n_sig count as Unclassified (out-of-range ids
  // are a caller error; the mask keeps them inside the table).
  const uint32_t words = (lut_mask + 1) / 8;                // 4 signatures per word pair
  const bool lut_vec = (reinterpret_cast<uintptr_t>(p.sig_class) & 3u) == 0;
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
      const uint32_t g = (c < 11 || c == 14) ? 16u : 0u;
      const uint32_t pair = (c << 2) | (((c << 2) | (g << 3)) << 8);   // byte: 4c | guard<<7
      if (b & 1) o[b >> 1] |= pair << 16; else o[b >> 1] = pair;
    }
    *reinterpret_cast<uint2*>(lut + 8 * i) = make_uint2(o[0], o[1]);
  }
  __syncthreads();
  if (ks >= ke) return;
  const unsigned char* incb = reinterpret_cast<const unsigned char*>(inc) + 8 * lane;
  uint32_t* my_first = firsts + (threadIdx.x >> 5) * kFirstStride;

  // Positions are kept relative to the warp's first chunk start cs0 (u32:
  // a call holds < 2^32 records).  The chunk grid is aligned to 16-byte
  // addresses; lane holds records c + 128u + 4*lane + j (u = 0, 1; j = 0..3)
  // of chunk c, copied by the lane itself into its slots of the warp's
  // ring (cp.async, zero-fill past the end), so only the lane's own
  // wait_group orders them -- no barriers.
  const uint64_t rs = __ldg(p.off + ks);
  const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(p.instr) >> 2) & 3u;
  const uint64_t cs0 = ((rs + mis) & ~3ull) - mis;         // may be "-mis" (wraps; used as an offset)
  const uint32_t re = (uint32_t)(__ldg(p.off + ke) - cs0);
  const uint4* gsrc = reinterpret_cast<const uint4*>(p.instr + cs0) + lane;   // vector 64c + 32u
  uint4* my_ring = ring + (size_t)(threadIdx.x >> 5) * kDepth * (kChunk / 4) + lane;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(my_ring);
  const uint32_t l4 = 4u * (uint32_t)lane;
#pragma unroll
  for (int d = 0; d < kDepth; ++d) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t i = (uint32_t)d * kChunk + 128u * u + l4;
      cp_async16(ring_s + 16u * (64u * d + 32u * u), gsrc + 64 * d + 32 * u, i < re ? 16u : 0u);
    }
    cp_async_commit();
  }
  // kernel ends in a 32-wide register window: lane j holds off[kw + 1 + j]
  uint32_t k = ks, kw = ks;
  uint32_t ends = (uint32_t)(__ldg(p.off + min(kw + 1 + (uint32_t)lane, p.n_kernels)) - cs0);
  uint32_t kb = (uint32_t)(rs - cs0), kend = __shfl_sync(0xffffffffu, ends, 0);

  MixAcc a{};
  uint32_t cs = 0, slot = 0;
  while (true) {
    const uint32_t ce = cs + kChunk;
    cp_async_wait<kDepth - 1>();
    uint32_t r[8], lv[8];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint4 v = my_ring[64 * slot + 32 * u];
      r[4 * u + 0] = v.x; r[4 * u + 1] = v.y; r[4 * u + 2] = v.z; r[4 * u + 3] = v.w;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) lv[e] = lut[r[e] & lut_mask];
    {
      // refill this slot with chunk c + kDepth (the records are in registers)
      const uint32_t nb = cs + kDepth * kChunk;
      const uint4* src = gsrc + (size_t)(nb / 4);
#pragma unroll
      for (int u = 0; u < 2; ++u)
        cp_async16(ring_s + 16u * (64u * slot + 32u * u), src + 32 * u,
                   nb + 128u * u + l4 < re ? 16u : 0u);
      cp_async_commit();
      slot = slot + 1 == kDepth ? 0 : slot + 1;
    }
    if (kb <= cs && ce < kend) {
      // fast path: the whole chunk lies inside kernel k, which continues
#pragma unroll
      for (int e = 0; e < 8; ++e) a.regs += r[e] >> 17;
      count_piece(a, lv, incb, my_first, cs - kb, lane);
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
            mv[e] = in ? lv[e] : kNullLv;
            a.regs += in ? (r[e] >> 17) : 0u;
          }
          count_piece(a, mv, incb, my_first, cs - kb, lane);
        }
        if (kend > ce) break;                                // kernel continues in the next chunk
        finish_kernel(a, my_first, p.out + k, kend - kb, lane);
        if (++k == ke) {
          cp_async_wait<0>();
          return;
        }
        kb = kend;
        if (k - kw == 32) {                                  // next window of kernel ends
          kw = k;
          ends = (uint32_t)(__ldg(p.off + min(kw + 1 + (uint32_t)lane, p.n_kernels)) - cs0);
        }
        kend = __shfl_sync(0xffffffffu, ends, (int)(k - kw));
      }
    }
    cs = ce;
  }
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
  const size_t ring = (size_t)kWarps * (deep ? 4 : 2) * kChunk * 4;
  const size_t smem = mix_ring_offset() + ring + lut_bytes;
  const void* fn = deep ? (const void*)mix_reduce_kernel<4> : (const void*)mix_reduce_kernel<2>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return OCCX_ERR_CUDA;
  // persistent: one 32-warp CTA per SM (one copy of the class table per SM)
  const uint32_t grid = (uint32_t)ctx->sm_count;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (deep)
    mix_reduce_kernel<4><<<grid, kMixThreads, smem, st>>>(p, lut_bytes - 1);
  else
    mix_reduce_kernel<2><<<grid, kMixThreads, smem, st>>>(p, lut_bytes - 1);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}
