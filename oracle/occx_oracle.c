/*
 * occx_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the occmix
 * reference algorithm for the scored hot path, used by tests/ (parity),
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing in paper_1701_08547_b200/ links or calls this file.
 *
 * Written independently of the CUDA path: plain 64-bit integer arithmetic
 * with real divisions, a dense T-bitset per segment for membership (the
 * product uses 64-bit T/32 masks), nested-loop enumeration of Cartesian
 * spaces (the product decodes mixed-radix indices), and a sorted-array
 * top-k (the product uses warp lists).
 *
 * Each function cites the reference lines it follows
 * (/root/reference/pkg/src/occmix/...).  Parity of this file against the
 * reference itself is pinned by tests/test_oracle_golden.py using
 * fixtures generated from the reference (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t ws, tmax, bmp, wmp, rfs, gran, rmax, smax;
} ora_arch;

typedef struct {
  int64_t wpb, lw, lr, ls, blocks, aw, limiter, status, rwl;
  double occ;
} ora_occ;

enum { ST_OK = 0, ST_ILLEGAL = 2 };
enum { LIM_WARPS = 0, LIM_REGS = 1, LIM_SMEM = 2, LIM_ILLEGAL = 3 };

/* occupancy.py:85-87 _ceil_div (non-negative operands) */
static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t min2(int64_t a, int64_t b) { return a < b ? a : b; }

/* occupancy.py:111-124 register_warp_limit */
static int64_t reg_warp_limit(const ora_arch* A, int64_t R) {
  if (R == 0) return A->wmp;
  if (R > A->rmax) return 0;
  int64_t per_warp = ceil_div(R * A->ws, A->gran) * A->gran;
  return A->rfs / per_warp;
}

/* occupancy.py:127-145 limit_by_registers (thread check done by caller) */
static int64_t lim_regs(const ora_arch* A, int64_t wpb, int64_t R, int mode) {
  if (R > A->rmax) return 0;
  if (R == 0) return A->bmp;
  if (mode == 1) {
    int64_t avail = A->gran / (R * A->ws);
    return ceil_div(avail, wpb) * ceil_div(A->rfs, A->gran);
  }
  return min2(A->bmp, reg_warp_limit(A, R) / wpb);
}

/* occupancy.py:148-160 limit_by_smem */
static int64_t lim_smem(const ora_arch* A, int64_t S, int mode) {
  if (S > A->smax) return 0;
  if (S == 0) return A->bmp;
  if (mode == 1) return ceil_div(A->smax, S);
  return min2(A->bmp, A->smax / S);
}

/* occupancy.py:38-52 (LaunchInput checks) + :163-195 occupancy() */
int ora_occupancy(const ora_arch* A, int64_t T, int64_t R, int64_t S, int mode, ora_occ* o) {
  memset(o, 0, sizeof(*o));
  o->limiter = LIM_ILLEGAL;
  if (T < 1 || R < 0 || S < 0 || T > A->tmax) { /* LaunchInput / _check_threads raise */
    o->status = ST_ILLEGAL;
    return ST_ILLEGAL;
  }
  o->wpb = ceil_div(T, A->ws);
  o->lw = min2(A->bmp, A->wmp / o->wpb);
  o->lr = lim_regs(A, o->wpb, R, mode);
  o->ls = lim_smem(A, S, mode);
  o->rwl = reg_warp_limit(A, R);
  int64_t b = min2(o->lw, min2(o->lr, o->ls));
  o->blocks = b;
  if (b == 0) o->limiter = LIM_ILLEGAL;
  else if (b == o->lw) o->limiter = LIM_WARPS;
  else if (b == o->lr) o->limiter = LIM_REGS;
  else o->limiter = LIM_SMEM;
  o->aw = min2(b * o->wpb, A->wmp);
  o->occ = (double)o->aw / (double)A->wmp;
  o->status = ST_OK;
  return ST_OK;
}

void ora_occupancy_many(const ora_arch* archs, const int64_t* arch_idx, const int64_t* T,
                        const int64_t* R, const int64_t* S, int64_t n, int mode, ora_occ* out) {
  for (int64_t i = 0; i < n; ++i) ora_occupancy(&archs[arch_idx[i]], T[i], R[i], S[i], mode, &out[i]);
}

/* ------------------------------------------------------------------------
 * Scoring composition: key per candidate and
 * per-segment top-k.  Membership: static_prune / rule_prune kept sets
 * (tuning.py:94-127) as dense bitsets over T in [0, 65536).
 * --------------------------------------------------------------------- */
#define TBITS_WORDS (65536 / 64)
typedef struct {
  uint64_t st[TBITS_WORDS], lo[TBITS_WORDS], hi[TBITS_WORDS];
} ora_segsets;

typedef struct {
  int64_t seg;    /* kernel * n_arch + arch */
  int64_t rank;   /* dense cost rank, -1 = arch has no cost column */
  int64_t upper;  /* intensity > 4.0 */
} ora_vent;

static int tbit(const uint64_t* w, int64_t t) {
  if (t < 0 || t >= 65536) return 0;
  return (int)((w[t >> 6] >> (t & 63)) & 1u);
}

static uint64_t ora_key(const ora_arch* archs, int64_t n_arch, const ora_vent* vt, int64_t n_var,
                        const ora_segsets* sets, int64_t variant, int64_t a, int64_t T, int64_t R,
                        int64_t S, int mode, uint64_t gidx, int64_t* seg_out) {
  *seg_out = -1;
  if (a < 0 || a >= n_arch || variant < 0 || variant >= n_var) return 0;
  ora_occ o;
  if (ora_occupancy(&archs[a], T, R, S, mode, &o) != ST_OK) return 0;
  if (o.blocks == 0) return 0;
  const ora_vent* v = &vt[variant * n_arch + a];
  const ora_segsets* s = &sets[v->seg];
  uint64_t st = (uint64_t)tbit(s->st, T);
  uint64_t ru = (uint64_t)tbit(v->upper ? s->hi : s->lo, T);
  uint64_t rank_bits = v->rank >= 0 ? (uint64_t)((1 << 20) - 1 - v->rank) : 0;
  *seg_out = v->seg;
  return (1ull << 63) | (ru << 62) | (st << 61) | ((uint64_t)o.aw << 54) | (rank_bits << 34) |
         (((1ull << 34) - 1) - gidx);
}

/* sorted descending top-k per segment, keys unique (global index bits) */
static void topk_push(uint64_t* list, int64_t k, uint64_t key) {
  if (key <= list[k - 1]) return;
  int64_t i = k - 1;
  while (i > 0 && list[i - 1] < key) { list[i] = list[i - 1]; --i; }
  list[i] = key;
}

/* records: occx_cand_t layout (u32 variant, u32 smem, u16 threads, u16 blocks,
 * u16 regs, u8 arch, u8 aux) */
void ora_score_records(const ora_arch* archs, int64_t n_arch, const uint8_t* rec, int64_t n,
                       uint64_t index_base, int mode, const ora_vent* vt, int64_t n_var,
                       const ora_segsets* sets, int64_t n_seg, int64_t k, uint64_t* out) {
  memset(out, 0, sizeof(uint64_t) * n_seg * k);
  for (int64_t i = 0; i < n; ++i) {
    const uint8_t* r = rec + 16 * i;
    uint32_t variant, smem;
    uint16_t threads, regs;
    memcpy(&variant, r, 4);
    memcpy(&smem, r + 4, 4);
    memcpy(&threads, r + 8, 2);
    memcpy(&regs, r + 12, 2);
    int64_t seg;
    uint64_t key = ora_key(archs, n_arch, vt, n_var, sets, variant, r[14], threads, regs, smem,
                           mode, index_base + (uint64_t)i, &seg);
    if (key) topk_push(out + seg * k, k, key);
  }
}

/* One Cartesian segment (tuning.py:30-77 enumerate_space order), dims
 * TC, BC, UIF, PL, CFLAGS, REGS, SMEM; variant = var_base + i_uif*n_cf + i_cf. */
typedef struct {
  int64_t arch, var_base;
  const int64_t* tc; int64_t n_tc;
  int64_t n_bc, n_uif, n_pl, n_cf;
  const int64_t* regs; int64_t n_regs;
  const int64_t* smem; int64_t n_smem;
} ora_space;

/* Score a concatenation of spaces by nested loops (no records stored);
 * candidates [lo, hi) of the concatenation only. */
void ora_score_spaces(const ora_arch* archs, int64_t n_arch, const ora_space* sp, int64_t n_sp,
                      uint64_t lo, uint64_t hi, int mode, const ora_vent* vt, int64_t n_var,
                      const ora_segsets* sets, int64_t n_seg, int64_t k, uint64_t* out) {
  memset(out, 0, sizeof(uint64_t) * n_seg * k);
  uint64_t g = 0;
  for (int64_t s = 0; s < n_sp; ++s) {
    const ora_space* p = &sp[s];
    uint64_t size = (uint64_t)p->n_tc * p->n_bc * p->n_uif * p->n_pl * p->n_cf * p->n_regs * p->n_smem;
    if (g + size <= lo || g >= hi) { g += size; continue; }
    for (int64_t it = 0; it < p->n_tc; ++it)
      for (int64_t ib = 0; ib < p->n_bc; ++ib)
        for (int64_t iu = 0; iu < p->n_uif; ++iu)
          for (int64_t ip = 0; ip < p->n_pl; ++ip)
            for (int64_t ic = 0; ic < p->n_cf; ++ic) {
              const int64_t variant = p->var_base + iu * p->n_cf + ic;
              for (int64_t ir = 0; ir < p->n_regs; ++ir)
                for (int64_t is = 0; is < p->n_smem; ++is, ++g) {
                  if (g < lo || g >= hi) continue;
                  int64_t seg;
                  uint64_t key = ora_key(archs, n_arch, vt, n_var, sets, variant, p->arch,
                                         p->tc[it], p->regs[ir], p->smem[is], mode, g, &seg);
                  if (key) topk_push(out + seg * k, k, key);
                }
            }
  }
}

/* Merge tables [n_lists][n_seg][k] -> [n_seg][k] */
void ora_topk_merge(const uint64_t* lists, int64_t n_lists, int64_t n_seg, int64_t k, uint64_t* out) {
  memset(out, 0, sizeof(uint64_t) * n_seg * k);
  for (int64_t l = 0; l < n_lists; ++l)
    for (int64_t s = 0; s < n_seg; ++s)
      for (int64_t j = 0; j < k; ++j) {
        uint64_t key = lists[(l * n_seg + s) * k + j];
        if (key) topk_push(out + s * k, k, key);
      }
}

/* ------------------------------------------------------------------------
 * aggregate() mix.py:245-261 over 4-byte instruction records
 * (guard:1 | sig:16 | regops:8, include/occx.h OCCX_INSTR).  class ids: 0..13 OpClass rows in enum
 * order, 14 = Unclassified; CTRL rows are 11..13 (Pred, Ctrl, Move).
 * order_out[k][j] = class of the j-th dict insertion (-1 = none).
 * --------------------------------------------------------------------- */
void ora_aggregate(const uint32_t* rec, const uint64_t* off, int64_t n_kernels,
                   const uint8_t* sig_class, int64_t n_sig, int64_t* counts_out,
                   int64_t* order_out, int64_t* regops_out) {
  for (int64_t kk = 0; kk < n_kernels; ++kk) {
    int64_t* counts = counts_out + kk * 15;
    int64_t* order = order_out + kk * 15;
    int64_t n_order = 0;
    memset(counts, 0, 15 * sizeof(int64_t));
    for (int j = 0; j < 15; ++j) order[j] = -1;
    int present[15] = {0};
    int64_t regs = 0;
    for (uint64_t i = off[kk]; i < off[kk + 1]; ++i) {
      uint32_t r = rec[i];
      uint32_t sig = (r >> 1) & 0xffffu;
      int cls = sig < (uint64_t)n_sig ? sig_class[sig] : 14;
      if (!present[cls]) { present[cls] = 1; order[n_order++] = cls; }
      counts[cls] += 1;
      int guard = r & 1;
      int is_ctrl = cls >= 11 && cls <= 13;
      if (guard && !is_ctrl) {
        if (!present[11]) { present[11] = 1; order[n_order++] = 11; }
        counts[11] += 1;
      }
      regs += (r >> 17) & 0xffu;
    }
    regops_out[kk] = regs;
  }
}
