// occx_feat.cu -- K1 feature scoring (restates occmix/mix.py:268-352).
//
// Compiled with -fmad=false and written with explicit __dadd_rn/__dmul_rn/
// __ddiv_rn: every double operation is the single IEEE operation CPython
// performs, in the same order, so results are bit-identical to the
// reference on the same interpreter.  CPython's builtin float sum() is
// restated exactly (Python/bltinmodule.c, builtin_sum_impl):
//   * items arrive after the int start value 0, so the first item x0 turns
//     the running result into the float 0 + x0;
//   * CPython >= 3.12 then does Neumaier-compensated summation and adds the
//     compensation at the end only when it is non-zero and finite;
//   * CPython <= 3.11 adds left to right.
// The interpreter version is the caller's `sum_mode` (the Python host picks
// it from sys.version_info).
#include <cmath>
#include "occx_common.cuh"

using namespace occx;

namespace {

constexpr uint32_t kAbsent = 0xffffffffu;
constexpr int kFp32 = 0, kLdSt = 9, kCtrl = 12, kRegsRow = 14, kUnclassified = 14;

struct FeatParams {
  double cpi[4][16];
  int32_t cols[kMaxArchs];
  uint32_t n_col, n_mix;
  double scale;
  int sum_mode;
  const occx_mix_t* mix;
  occx_mixsum_t* sum;
  occx_feat_t* feat;
};

__device__ double py_float_sum(const double* x, int n, int mode) {
  double f = __dadd_rn(0.0, x[0]);
  if (mode == OCCX_SUM_NAIVE) {
    for (int i = 1; i < n; ++i) f = __dadd_rn(f, x[i]);
    return f;
  }
  double c = 0.0;
  for (int i = 1; i < n; ++i) {
    const double xi = x[i];
    const double t = __dadd_rn(f, xi);
    if (fabs(f) >= fabs(xi)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), xi));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(xi, t), f));
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f = __dadd_rn(f, c);
  return f;
}

__global__ void feature_kernel(const __grid_constant__ FeatParams p) {
  const uint32_t per_mix = p.n_col > 0 ? p.n_col : 1;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (uint64_t)p.n_mix * per_mix) return;
  const uint32_t m = (uint32_t)(t / per_mix), j = (uint32_t)(t - (uint64_t)m * per_mix);
  const occx_mix_t& mx = p.mix[m];
  uint64_t flops = 0, mem = 0, ctrl = 0, all = 0;
  for (int c = 0; c < 8; ++c) flops += mx.counts[c];
  for (int c = 8; c < 11; ++c) mem += mx.counts[c];
  for (int c = 11; c < 14; ++c) ctrl += mx.counts[c];
  for (int c = 0; c < 15; ++c) all += mx.counts[c];
  if (j == 0) {
    occx_mixsum_t s;
    s.flops = flops;
    s.mem = mem;
    s.ctrl = ctrl;
    s.unclassified = mx.counts[kUnclassified];
    s.total = all;
    // mix.py:333-337
    if (mem == 0) s.intensity = flops > 0 ? INFINITY : 0.0;
    else s.intensity = __ddiv_rn((double)flops, (double)mem);
    p.sum[m] = s;
  }
  if (p.n_col == 0) return;
  occx_feat_t f;
  for (int i = 0; i < 16; ++i) f.per_class[i] = NAN;
  f.pc_status = 0;
  const int key = p.cols[j];
  if (key < 0 || key > 3) {                       // sm_key raises, mix.py:99-106
    f.status = f.pc_status = OCCX_ERR_UNSUPPORTED_ARCH;
    f.cost = NAN;
    for (int i = 0; i < 4; ++i) f.coef[i] = f.cycles[i] = f.shares[i] = NAN;
    p.feat[t] = f;
    return;
  }
  const double* cp = p.cpi[key];
  // Two lookup sets, as in the reference: cost / coefficients / cycles /
  // shares need the FLOPS classes present (or FP32) plus LdSt, Ctrl, Regs
  // (mix.py:268-306); per_class_cycles needs every class with n != 0 and
  // Regs when reg_operands != 0 (mix.py:309-318).  A partial table can fail
  // one and not the other.
  bool missing = false, pc_missing = false;
  // _flops_coefficient, mix.py:268-281
  double coef_f;
  if (flops == 0) {
    coef_f = cp[kFp32];
    missing |= isnan(coef_f);
  } else {
    // FLOPS classes present in the dict, in insertion order
    int order[8], n = 0;
    for (int c = 0; c < 8; ++c)
      if (mx.first_key[c] != kAbsent) order[n++] = c;
    for (int a = 1; a < n; ++a) {               // insertion sort by first_key
      const int v = order[a];
      int b = a - 1;
      while (b >= 0 && mx.first_key[order[b]] > mx.first_key[v]) { order[b + 1] = order[b]; --b; }
      order[b + 1] = v;
    }
    double terms[8];
    for (int i = 0; i < n; ++i) {
      const double c = cp[order[i]];
      missing |= isnan(c);
      terms[i] = __dmul_rn((double)mx.counts[order[i]], c);
    }
    const double weighted = py_float_sum(terms, n, p.sum_mode);
    coef_f = __ddiv_rn(weighted, (double)flops);
  }
  // category_coefficients / category_cycles, mix.py:284-306
  f.coef[0] = coef_f;
  f.coef[1] = cp[kLdSt];
  f.coef[2] = cp[kCtrl];
  f.coef[3] = cp[kRegsRow];
  missing |= isnan(f.coef[1]) || isnan(f.coef[2]) || isnan(f.coef[3]);
  f.cycles[0] = __dmul_rn(f.coef[0], (double)flops);
  f.cycles[1] = __dmul_rn(f.coef[1], (double)mem);
  f.cycles[2] = __dmul_rn(f.coef[2], (double)ctrl);
  f.cycles[3] = __dmul_rn(f.coef[3], (double)mx.reg_operands);
  // cost_estimate, mix.py:321-330: scale * sum(cycles.values())
  const double total = py_float_sum(f.cycles, 4, p.sum_mode);
  f.cost = __dmul_rn(p.scale, total);
  // pipeline_utilization, mix.py:340-352
  for (int i = 0; i < 4; ++i) f.shares[i] = (total == 0.0) ? 0.0 : __ddiv_rn(f.cycles[i], total);
  // per_class_cycles, mix.py:309-318 (n != 0 only; Unclassified excluded)
  for (int c = 0; c < 14; ++c)
    if (mx.first_key[c] != kAbsent && mx.counts[c] != 0) {
      pc_missing |= isnan(cp[c]);
      f.per_class[c] = __dmul_rn((double)mx.counts[c], cp[c]);
    }
  if (mx.reg_operands != 0) {
    pc_missing |= isnan(cp[kRegsRow]);
    f.per_class[kRegsRow] = __dmul_rn((double)mx.reg_operands, cp[kRegsRow]);
  }
  if (missing) {                // cost_estimate raises: no cost enters any rank
    f.cost = NAN;
    for (int i = 0; i < 4; ++i) f.cycles[i] = f.shares[i] = NAN;
  }
  f.status = missing ? OCCX_ERR_KEY : OCCX_OK;
  f.pc_status = pc_missing ? OCCX_ERR_KEY : OCCX_OK;
  p.feat[t] = f;
}

}  // namespace

extern "C" int occx_feature_score(const occx_ctx* ctx, const occx_mix_t* d_mix, uint32_t n_mix,
                                  const int32_t* h_cols, uint32_t n_col, const double* h_cpi,
                                  double scale, int sum_mode, occx_mixsum_t* d_sum,
                                  occx_feat_t* d_feat, void* stream) {
  if (!ctx || n_col > (uint32_t)kMaxArchs || (sum_mode != 0 && sum_mode != 1)) return OCCX_ERR_VALUE;
  if (n_col > 0 && (h_cols == nullptr || h_cpi == nullptr || d_feat == nullptr)) return OCCX_ERR_VALUE;
  if (n_mix == 0) return OCCX_OK;
  FeatParams p{};
  if (h_cpi)
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 16; ++c) p.cpi[r][c] = h_cpi[r * 16 + c];
  for (uint32_t j = 0; j < n_col; ++j) p.cols[j] = h_cols[j];
  p.n_col = n_col;
  p.n_mix = n_mix;
  p.scale = scale;
  p.sum_mode = sum_mode;
  p.mix = d_mix;
  p.sum = d_sum;
  p.feat = d_feat;
  const uint64_t threads = (uint64_t)n_mix * (n_col ? n_col : 1);
  feature_kernel<<<(unsigned)((threads + 127) / 128), 128, 0,
                   reinterpret_cast<cudaStream_t>(stream)>>>(p);
  OCCX_CUDA_TRY(cudaGetLastError());
  return OCCX_OK;
}
