// occx_mix.cu -- K0 instruction-mix reducer (restates occmix/mix.py:245-261).
//
// One warp per kernel segment of a CSR array of 4-byte instruction records
// (include/occx.h OCCX_INSTR).  Per record:
//   cls = LUT[sig]                 classify(), mix.py:176-187 (host-built LUT)
//   counts[cls] += 1               mix.py:256-257
//   if guard and cls not CTRL:     mix.py:258-259 (Unclassified included:
//       counts[PredIns] += 1        CATEGORY_OF.get(UNCLASSIFIED) is None)
//   reg_operands += regops         mix.py:260
//
// Counting: a 32-entry table indexed by (class | guard << 4) holds the u64
// increment of each case over sixteen 4-bit counters (class nibble, plus
// the PredIns nibble and a "guard counted" marker in the spare nibble 15
// when the guard adds a PredIns), so a record costs one LDS.U8, one LDS.64
// and a 64-bit add.  Each chunk of 8 records per lane is folded into two
// u64 byte-counter words (even / odd classes), reduced over the warp with
// 16-bit-lane REDUX.SUM before they can overflow.
// Dict insertion order (it decides the summation order of the FLOPS terms
// in mix.py:278) is recovered as first_key[c] = min over occurrences of
// 2*i (class of instruction i) or 2*i+1 (guard PredIns of instruction i);
// a warp OR-reduction per chunk finds classes not seen before and only
// then are their first positions located (ballots, warp-uniform).
#include "occx_common.cuh"

using namespace occx;

namespace {

constexpr int kMixThreads = 256;
constexpr int kMixPer = 8;                            // records per lane per chunk
constexpr int kFlushChunks = 255 / kMixPer;           // byte counters cannot overflow
constexpr uint32_t kPred = 11;                        // OpClass.PREDICATE device id
constexpr uint32_t kAbsent = 0xffffffffu;
constexpr uint32_t kNullClass = 15;                   // padding record: counts nothing

struct MixParams {
  const uint32_t* instr;
  const uint64_t* off;
  uint32_t n_kernels;
  const uint8_t* sig_class;
  uint32_t n_sig;
  occx_mix_t* out;
};

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Sum 16 byte counters held as even classes (w[0] classes 0,2,4,6; w[1]
// 8,10,12,14) and odd classes (w[2] 1,3,5,7; w[3] 9,11,13,15); lane c < 16
// receives class c's total.  16-bit lanes: 32 x 255 < 2^16.
__device__ __forceinline__ void reduce_counters_eo(const uint32_t (&w)[4], int lane,
                                                   uint32_t& total) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t lo = __reduce_add_sync(0xffffffffu, w[q] & 0x00ff00ffu);   // bytes 0, 2
    const uint32_t hi = __reduce_add_sync(0xffffffffu, (w[q] >> 8) & 0x00ff00ffu);  // bytes 1, 3
    const int base = (q & 1) * 8 + (q >> 1);             // class of byte 0 in this word
    if (lane == base) total += lo & 0xffffu;
    if (lane == base + 2) total += hi & 0xffffu;
    if (lane == base + 4) total += lo >> 16;
    if (lane == base + 6) total += hi >> 16;
  }
}

__global__ void __launch_bounds__(kMixThreads) mix_reduce_kernel(const __grid_constant__ MixParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  // [32] u64 nibble increments, [warps][17] first positions, [n_sig + 1] class LUT
  uint64_t* inc = reinterpret_cast<uint64_t*>(smem);
  uint32_t* firsts = reinterpret_cast<uint32_t*>(inc + 32);
  unsigned char* lut = reinterpret_cast<unsigned char*>(firsts + (kMixThreads / 32) * 17 + 2);
  for (uint32_t i = threadIdx.x; i < 32; i += blockDim.x) {
    const uint32_t c = i & 15u, g = i >> 4;
    uint64_t v = 0;
    if (c < 15) {
      v = 1ull << (4 * c);
      if (g && !(c >= 11 && c <= 13)) v += (1ull << (4 * kPred)) + (1ull << 60);  // PredIns + marker
    }
    inc[i] = v;
  }
  for (uint32_t i = threadIdx.x; i < (kMixThreads / 32) * 17; i += blockDim.x) firsts[i] = kAbsent;
  // class table indexed by the record's low 17 bits (sig << 1 | guard):
  // entry = class | 16 when the guard adds a PredIns (class not CTRL);
  // signature n_sig is the padding record (class 15, counts nothing)
  for (uint32_t i = threadIdx.x; i <= p.n_sig; i += blockDim.x) {
    const uint32_t c = i < p.n_sig ? (p.sig_class[i] & 15u) : kNullClass;
    lut[2 * i] = (uint8_t)c;
    lut[2 * i + 1] = (uint8_t)(c | ((c < 11 || c == 14) ? 16u : 0u));
  }
  __syncthreads();
  const uint32_t inc_base = (uint32_t)__cvta_generic_to_shared(inc);
  const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(lut);
  uint32_t* my_first = firsts + (threadIdx.x >> 5) * 17;
  const uint32_t null_rec = p.n_sig << 1;                   // sig = n_sig -> class 15

  const int lane = threadIdx.x & 31;
  const uint32_t warps_total = gridDim.x * (kMixThreads / 32);
  uint32_t kern = blockIdx.x * (kMixThreads / 32) + (threadIdx.x >> 5);
  // software pipeline across kernels: the next kernel's offsets and first
  // chunk are loaded while the current kernel is being reduced
  uint64_t beg = 0, end = 0;
  if (kern < p.n_kernels) {
    beg = __ldg(p.off + kern);
    end = __ldg(p.off + kern + 1);
  }
  uint32_t rec[kMixPer];
  {
    const uint32_t len = (uint32_t)min(end - beg, (uint64_t)0x7fffffff);
#pragma unroll
    for (int u = 0; u < kMixPer; ++u) {
      const uint32_t i = (uint32_t)u * 32 + lane;
      rec[u] = (i < len) ? __ldcs(p.instr + beg + i) : null_rec;
    }
  }
  while (kern < p.n_kernels) {
    const uint32_t nkern = kern + warps_total;
    uint64_t nbeg = 0, nend = 0;
    if (nkern < p.n_kernels) {
      nbeg = __ldg(p.off + nkern);
      nend = __ldg(p.off + nkern + 1);
    }
    const uint32_t nlen = (uint32_t)min(nend - nbeg, (uint64_t)0x7fffffff);
    const uint32_t len = (uint32_t)min(end - beg, (uint64_t)0x7fffffff);
    const uint32_t* src = p.instr + beg;
    // byte counters: even classes (0,2,..,14) and odd classes (1,3,..,15)
    uint32_t be0 = 0, be1 = 0, bo0 = 0, bo1 = 0;
    uint32_t seen_lo = 0, seen_hi = 0;                      // nibble presence so far
    uint32_t regs = 0, total = 0;
    int since_flush = 0;
    uint32_t nxt[kMixPer];
    for (uint32_t rb = 0; rb < len; rb += 32 * kMixPer) {
      const uint32_t nb = rb + 32 * kMixPer;
      if (nb + 32 * kMixPer <= len) {                      // next chunk, fully inside
#pragma unroll
        for (int u = 0; u < kMixPer; ++u) nxt[u] = __ldcs(src + nb + (uint32_t)u * 32 + lane);
      } else if (nb < len) {                               // next chunk, partial
#pragma unroll
        for (int u = 0; u < kMixPer; ++u) {
          const uint32_t i = nb + (uint32_t)u * 32 + lane;
          nxt[u] = (i < len) ? __ldcs(src + i) : null_rec;
        }
      } else {                                             // first chunk of the next kernel
#pragma unroll
        for (int u = 0; u < kMixPer; ++u) {
          const uint32_t i = (uint32_t)u * 32 + lane;
          nxt[u] = (i < nlen) ? __ldcs(p.instr + nbeg + i) : null_rec;
        }
      }
      uint32_t v0 = 0, v1 = 0;                             // 4-bit counters, classes 0-7 / 8-15
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) {
        const uint32_t r = rec[u];
        const uint32_t idx = lds_u8(lut_base + (r & 0x1ffffu));  // class | counted-guard << 4
        uint32_t d0, d1;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(d0), "=r"(d1) : "r"(inc_base + idx * 8u));
        v0 += d0;
        v1 += d1;
        regs += r >> 17;                                    // register operands (bits 17-24)
      }
      // classes (nibbles) present in this lane's chunk -> warp presence
      uint32_t t0 = v0 | (v0 >> 1), t1 = v1 | (v1 >> 1);
      t0 = (t0 | (t0 >> 2)) & 0x11111111u;
      t1 = (t1 | (t1 >> 2)) & 0x11111111u;
      const uint32_t pres_lo = __reduce_or_sync(0xffffffffu, t0);
      const uint32_t pres_hi = __reduce_or_sync(0xffffffffu, t1);
      if ((pres_lo & ~seen_lo) | (pres_hi & ~seen_hi)) {   // a class new to this kernel
        seen_lo |= pres_lo;
        seen_hi |= pres_hi;
#pragma unroll
        for (int u = 0; u < kMixPer; ++u) {                // rare: re-read the classes
          const uint32_t idx = lds_u8(lut_base + (rec[u] & 0x1ffffu));
          const uint32_t c = idx & 15u;
          const uint32_t pos = rb + (uint32_t)u * 32 + lane;
          if (c != kNullClass) {
            atomicMin(my_first + c, 2u * pos);
            // guard PredIns (non-CTRL class): key 2*pos + 1, tracked in slot 16
            if (idx & 16u) atomicMin(my_first + 16, 2u * pos + 1);
          }
        }
      }
      be0 += v0 & 0x0f0f0f0fu;
      bo0 += (v0 >> 4) & 0x0f0f0f0fu;
      be1 += v1 & 0x0f0f0f0fu;
      bo1 += (v1 >> 4) & 0x0f0f0f0fu;
      if (++since_flush == kFlushChunks) {
        since_flush = 0;
        const uint32_t w[4] = {be0, be1, bo0, bo1};
        reduce_counters_eo(w, lane, total);
        be0 = be1 = bo0 = bo1 = 0;
      }
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) rec[u] = nxt[u];
    }
    if (len == 0) {                                        // empty kernel: load the next chunk now
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) {
        const uint32_t i = (uint32_t)u * 32 + lane;
        rec[u] = (i < nlen) ? __ldcs(p.instr + nbeg + i) : null_rec;
      }
    }
    {
      const uint32_t w[4] = {be0, be1, bo0, bo1};
      reduce_counters_eo(w, lane, total);
    }
    __syncwarp();
    uint32_t first = lane < 17 ? my_first[lane] : kAbsent;
    const uint32_t gfirst = __shfl_sync(0xffffffffu, first, 16);
    if (lane == (int)kPred && gfirst < first) first = gfirst;
    if (lane < 17) my_first[lane] = kAbsent;               // reset for the warp's next kernel
    __syncwarp();
    const uint32_t reg_total = __reduce_add_sync(0xffffffffu, regs);
    occx_mix_t* o = p.out + kern;
    if (lane < 16) {
      o->counts[lane] = lane < 15 ? total : 0u;
      o->first_key[lane] = (lane < 15 && total) ? first : kAbsent;
    }
    if (lane == 0) {
      o->reg_operands = reg_total;
      o->n_instr = (uint32_t)(end - beg);
      o->reserved = 0;
    }
    kern = nkern;
    beg = nbeg;
    end = nend;
  }
}

}  // namespace

extern "C" int occx_mix_reduce(const occx_ctx* ctx, const uint32_t* d_instr,
                               const uint64_t* d_kernel_off, uint32_t n_kernels,
                               const uint8_t* d_sig_class, uint32_t n_sig, occx_mix_t* d_out,
                               void* stream) {
  if (!ctx || n_sig == 0 || n_sig > 65535) return OCCX_ERR_VALUE;
  if (n_kernels == 0) return OCCX_OK;
  MixParams p{};
  p.instr = d_instr;
  p.off = d_kernel_off;
  p.n_kernels = n_kernels;
  p.sig_class = d_sig_class;
  p.n_sig = n_sig;
  p.out = d_out;
  const size_t smem = 32 * 8 + ((kMixThreads / 32) * 17 + 2) * 4 + ((2 * (n_sig + 1) + 15) & ~15u);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(mix_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return OCCX_ERR_CUDA;
  // persistent: exactly one wave (LUT staged once per CTA, no tail wave)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mix_reduce_kernel, kMixThreads,
                                                    smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const uint32_t want = (n_kernels + kMixThreads / 32 - 1) / (kMixThreads / 32);
  const uint32_t cap = (uint32_t)ctx->sm_count * (uint32_t)per_sm;
  const uint32_t grid = want < cap ? want : cap;
  mix_reduce_kernel<<<grid, kMixThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}
