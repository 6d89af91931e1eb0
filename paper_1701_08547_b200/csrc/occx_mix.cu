// occx_mix.cu -- K0 instruction-mix reducer (restates occmix/mix.py:245-261).
//
// One warp per kernel segment of a CSR array of 4-byte instruction records
// (include/occx.h OCCX_INSTR).  Per record:
//   cls = LUT[sig]                 classify(), mix.py:176-187 (host-built LUT)
//   counts[cls] += 1               mix.py:256-257
//   if guard and cls not CTRL:     mix.py:258-259 (Unclassified included:
//       counts[PredIns] += 1        CATEGORY_OF.get(UNCLASSIFIED) is None)
//   reg_operands += regops         mix.py:260
// Counting uses sixteen 8-bit lane-private counters packed in four u32
// registers (flushed with __reduce_add_sync before they can overflow), so
// the per-record work is shifts and adds -- no shared-memory atomics.
// Dict insertion order (it decides the summation order of the FLOPS terms
// in mix.py:278) is recovered as first_key[c] = min over occurrences of
// 2*i (class of instruction i) or 2*i+1 (guard PredIns of instruction i):
// a warp OR-reduction per chunk detects classes not seen before and only
// then computes their first position.
#include "occx_common.cuh"

using namespace occx;

namespace {

constexpr int kMixThreads = 256;
constexpr int kMixUnroll = 4;                         // records per lane per chunk
constexpr int kFlushChunks = 255 / (2 * kMixUnroll);  // byte counters cannot overflow
constexpr uint32_t kPred = 11;                        // OpClass.PREDICATE device id
constexpr uint32_t kAbsent = 0xffffffffu;

__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));   // s >= 32 -> 0
  return r;
}

struct MixParams {
  const uint32_t* instr;
  const uint64_t* off;
  uint32_t n_kernels;
  const uint8_t* sig_class;
  uint32_t n_sig;
  uint32_t lut_in_smem;
  occx_mix_t* out;
};

__global__ void __launch_bounds__(kMixThreads) mix_reduce_kernel(const __grid_constant__ MixParams p) {
  extern __shared__ __align__(16) unsigned char s_lut[];
  // LUT entry: bits 0-3 class id, bit 4 = "a guard adds PredIns" (class not CTRL)
  const uint8_t* lut = p.sig_class;
  if (p.lut_in_smem) {
    for (uint32_t i = threadIdx.x; i < p.n_sig; i += blockDim.x) {
      const uint32_t c = p.sig_class[i] & 15u;
      s_lut[i] = (uint8_t)(c | ((c >= 11 && c <= 13) ? 0u : 16u));
    }
    __syncthreads();
    lut = s_lut;
  }
  const int lane = threadIdx.x & 31;
  const uint32_t warps_total = gridDim.x * (kMixThreads / 32);
  for (uint32_t kern = blockIdx.x * (kMixThreads / 32) + (threadIdx.x >> 5); kern < p.n_kernels;
       kern += warps_total) {
    const uint64_t beg = p.off[kern], end = p.off[kern + 1];
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;   // 16 byte counters
    uint32_t total = 0;                         // lane c < 16 holds counts[c]
    uint32_t first = kAbsent;                   // lane c holds first_key[c]; lane 16 guard-pred
    uint32_t regs = 0;
    uint32_t warp_seen = 0;
    int since_flush = 0;
    for (uint64_t base = beg; base < end; base += 32 * kMixUnroll) {
      uint32_t rec[kMixUnroll];
#pragma unroll
      for (int u = 0; u < kMixUnroll; ++u) {
        const uint64_t i = base + (uint64_t)u * 32 + lane;
        rec[u] = (i < end) ? __ldcs(p.instr + i) : 0xffffffffu;
      }
      uint32_t seen = 0;
      uint32_t cls[kMixUnroll], gp[kMixUnroll];
#pragma unroll
      for (int u = 0; u < kMixUnroll; ++u) {
        const uint32_t r = rec[u];
        const bool valid = r != 0xffffffffu;
        uint32_t sig = r & 0xffffu;
        uint32_t e;
        if (p.lut_in_smem) e = lut[sig < p.n_sig ? sig : 0];
        else {
          const uint32_t c = __ldg(lut + (sig < p.n_sig ? sig : 0)) & 15u;
          e = c | ((c >= 11 && c <= 13) ? 0u : 16u);
        }
        const uint32_t c = valid ? (e & 15u) : 15u;          // 15 = nothing
        const uint32_t g = valid ? ((r >> 24) & (e >> 4) & 1u) : 0u;
        const uint32_t sh = valid ? c * 8u : 128u;
        w0 += shl_clamp(1u, sh);
        w1 += shl_clamp(1u, sh - 32u);
        w2 += shl_clamp(1u, sh - 64u) + (g << 24);          // PredIns byte 11
        w3 += shl_clamp(1u, sh - 96u);
        regs += valid ? ((r >> 16) & 0xffu) : 0u;
        seen |= (valid ? (1u << c) : 0u) | (g << 16);
        cls[u] = c;
        gp[u] = g;
      }
      const uint32_t chunk_seen = __reduce_or_sync(0xffffffffu, seen);
      uint32_t fresh = chunk_seen & ~warp_seen;
      if (fresh) {
        warp_seen |= chunk_seen;
        while (fresh) {
          const uint32_t b = __ffs(fresh) - 1;
          fresh &= fresh - 1;
          uint32_t best = kAbsent;
#pragma unroll
          for (int u = 0; u < kMixUnroll; ++u) {
            const uint32_t pos = (uint32_t)(base - beg) + (uint32_t)u * 32 + lane;
            const bool hit = (b == 16) ? (gp[u] != 0) : (cls[u] == b);
            const uint32_t key = 2u * pos + (b == 16 ? 1u : 0u);
            if (hit && key < best) best = key;
          }
          best = __reduce_min_sync(0xffffffffu, best);
          if (lane == (int)b) first = best;
        }
      }
      if (++since_flush == kFlushChunks) {
        since_flush = 0;
#pragma unroll
        for (int c = 0; c < 15; ++c) {
          const uint32_t word = c < 4 ? w0 : c < 8 ? w1 : c < 12 ? w2 : w3;
          const uint32_t v = __reduce_add_sync(0xffffffffu, (word >> ((c & 3) * 8)) & 0xffu);
          if (lane == c) total += v;
        }
        w0 = w1 = w2 = w3 = 0;
      }
    }
#pragma unroll
    for (int c = 0; c < 15; ++c) {
      const uint32_t word = c < 4 ? w0 : c < 8 ? w1 : c < 12 ? w2 : w3;
      const uint32_t v = __reduce_add_sync(0xffffffffu, (word >> ((c & 3) * 8)) & 0xffu);
      if (lane == c) total += v;
    }
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
  if (!ctx || n_sig == 0 || n_sig > 65536) return OCCX_ERR_VALUE;
  if (n_kernels == 0) return OCCX_OK;
  MixParams p{};
  p.instr = d_instr;
  p.off = d_kernel_off;
  p.n_kernels = n_kernels;
  p.sig_class = d_sig_class;
  p.n_sig = n_sig;
  p.lut_in_smem = n_sig <= 48 * 1024 ? 1u : 0u;
  p.out = d_out;
  const size_t smem = p.lut_in_smem ? n_sig : 0;
  const uint32_t warps = n_kernels;
  const uint32_t want = (warps + kMixThreads / 32 - 1) / (kMixThreads / 32);
  const uint32_t cap = (uint32_t)ctx->sm_count * 8;
  const uint32_t grid = want < cap ? want : cap;
  mix_reduce_kernel<<<grid, kMixThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}
