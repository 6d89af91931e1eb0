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
// Counting: each lane keeps sixteen 8-bit counters packed in four u32
// registers.  A second 32-entry table indexed by (class | guard << 4) holds
// the 16-byte increment vector of each case (the class byte, plus the
// PredIns byte when the guard counts), so a record costs one LDS.U8, one
// LDS.128 and four IADDs.  Counters are reduced with 16-bit-lane REDUX.SUM
// (bytes 0/2 and 1/3 separately) before they can overflow.
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
constexpr int kFlushChunks = 255 / (2 * kMixPer);     // byte counters cannot overflow
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
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

// Sum the 16 packed byte counters over the warp; lane c < 16 receives
// class c's total.  Bytes 0/2 and 1/3 are reduced in separate 16-bit lanes
// (32 x 255 < 2^16), 8 REDUX.SUM for 16 counters.
__device__ __forceinline__ void reduce_counters(const uint32_t (&w)[4], int lane,
                                                uint32_t& total) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t even = __reduce_add_sync(0xffffffffu, w[q] & 0x00ff00ffu);
    const uint32_t odd = __reduce_add_sync(0xffffffffu, (w[q] >> 8) & 0x00ff00ffu);
    const int c = 4 * q;
    if (lane == c) total += even & 0xffffu;
    if (lane == c + 1) total += odd & 0xffffu;
    if (lane == c + 2) total += even >> 16;
    if (lane == c + 3) total += odd >> 16;
  }
}

__global__ void __launch_bounds__(kMixThreads) mix_reduce_kernel(const __grid_constant__ MixParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint4* inc = reinterpret_cast<uint4*>(smem);              // [32] increment vectors
  unsigned char* lut = smem + 32 * sizeof(uint4);           // [n_sig + 1] class ids
  for (uint32_t i = threadIdx.x; i < 32; i += blockDim.x) {
    const uint32_t c = i & 15u, g = i >> 4;
    uint32_t v[4] = {0, 0, 0, 0};
    if (c < 15) {
      v[c >> 2] += 1u << ((c & 3) * 8);
      if (g && !(c >= 11 && c <= 13)) {
        v[kPred >> 2] += 1u << ((kPred & 3) * 8);
        v[3] += 1u << 24;               // byte 15: "guard added a PredIns" marker
      }
    }
    inc[i] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  for (uint32_t i = threadIdx.x; i <= p.n_sig; i += blockDim.x)
    lut[i] = i < p.n_sig ? (uint8_t)(p.sig_class[i] & 15u) : (uint8_t)kNullClass;
  __syncthreads();
  const uint32_t inc_base = (uint32_t)__cvta_generic_to_shared(inc);
  const uint32_t lut_base = (uint32_t)__cvta_generic_to_shared(lut);
  const uint32_t null_rec = p.n_sig;                        // sig = n_sig -> class 15

  const int lane = threadIdx.x & 31;
  const uint32_t warps_total = gridDim.x * (kMixThreads / 32);
  for (uint32_t kern = blockIdx.x * (kMixThreads / 32) + (threadIdx.x >> 5); kern < p.n_kernels;
       kern += warps_total) {
    const uint64_t beg = __ldg(p.off + kern), end = __ldg(p.off + kern + 1);
    uint32_t w[4] = {0, 0, 0, 0};     // 16 byte counters
    uint32_t total = 0;               // lane c < 16 holds counts[c]
    uint32_t first = kAbsent;         // lane c holds first_key[c]; lane 16 guard-PredIns
    uint32_t regs = 0;
    uint32_t warp_seen = 0;
    int since_flush = 0;
    const uint32_t len = (uint32_t)min(end - beg, (uint64_t)0x7fffffff);
    const uint32_t* src = p.instr + beg;
    uint32_t rec[kMixPer];
#pragma unroll
    for (int u = 0; u < kMixPer; ++u) {
      const uint32_t i = (uint32_t)u * 32 + lane;
      rec[u] = (i < len) ? __ldcs(src + i) : null_rec;
    }
    for (uint32_t rb = 0; rb < len; rb += 32 * kMixPer) {
      // prefetch the next chunk while this one is processed
      uint32_t nxt[kMixPer];
      const uint32_t nb = rb + 32 * kMixPer;
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) {
        const uint32_t i = nb + (uint32_t)u * 32 + lane;
        nxt[u] = (i < len) ? __ldcs(src + i) : null_rec;
      }
      uint32_t bits[kMixPer], seen = 0;
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) {
        const uint32_t r = rec[u];
        const uint32_t c = lds_u8(lut_base + (r & 0xffffu));
        const uint32_t idx = c | ((r >> 20) & 16u);          // guard bit 24 -> bit 4
        const uint4 d = lds_v4(inc_base + idx * 16u);
        w[0] += d.x;
        w[1] += d.y;
        w[2] += d.z;
        w[3] += d.w;
        regs += __byte_perm(r, 0, 0x4442);                  // register operands (byte 2)
        // class bit (bit 15 = padding, masked below) + guard-PredIns at bit 16
        bits[u] = (1u << c) | ((d.w >> 24) << 16);
        seen |= bits[u];
      }
      const uint32_t chunk_seen = __reduce_or_sync(0xffffffffu, seen) & 0x17fffu;
      uint32_t fresh = chunk_seen & ~warp_seen;
      if (fresh) {
        warp_seen |= chunk_seen;
        // first position of each new class: the lane's earliest slot, then
        // one REDUX.MIN over the warp (positions are distinct)
        const uint32_t rel0 = rb + (uint32_t)lane;
        while (fresh) {
          const uint32_t bt = __ffs(fresh) - 1;
          fresh &= fresh - 1;
          uint32_t mine = kAbsent;
#pragma unroll
          for (int u = kMixPer - 1; u >= 0; --u)
            if ((bits[u] >> bt) & 1u) mine = rel0 + (uint32_t)u * 32;
          const uint32_t pos = __reduce_min_sync(0xffffffffu, mine);
          if (lane == (int)bt) first = 2u * pos + (bt == 16 ? 1u : 0u);
        }
      }
      if (++since_flush == kFlushChunks) {
        since_flush = 0;
        reduce_counters(w, lane, total);
        w[0] = w[1] = w[2] = w[3] = 0;
      }
#pragma unroll
      for (int u = 0; u < kMixPer; ++u) rec[u] = nxt[u];
    }
    reduce_counters(w, lane, total);
    const uint32_t gfirst = __shfl_sync(0xffffffffu, first, 16);
    if (lane == (int)kPred && gfirst < first) first = gfirst;
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
  const size_t smem = 32 * 16 + ((n_sig + 1 + 15) & ~15u);
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
