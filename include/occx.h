/*
 * occx.h -- C ABI of the B200 (sm_100a) backend for the occmix hot path
 * (arXiv 1701.08547 static autotuner: batched search-space scoring).
 *
 * The reference (occmix 0.1.0, pure Python) has no FFI; its boundary is the
 * Python package API (pkg/src/occmix/__init__.py:7-42).  Each entry point
 * below names the reference function whose per-candidate / per-kernel math
 * it replaces.  INTEGRATION.md shows the ctypes binding a maintainer would
 * add to occmix; paper_1701_08547_b200/_lib.py is that binding.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes.  Every d_* pointer is device
 *    memory owned by the caller; the library never frees caller memory.
 *  - Stream-ordered: `stream` is a cudaStream_t passed as void* (NULL = the
 *    legacy default stream).  Calls return after enqueueing; results are
 *    valid once the stream is synchronised.
 *  - Return value is an occx_status; codes map 1:1 onto the reference's
 *    exception classes (pkg/src/occmix/errors.py:4-48).
 *  - A context caches device properties (SM count, smem limit) and the
 *    options it was created with; it is immutable after create and safe to
 *    share across threads and streams.  The library reads no environment
 *    variables.
 */
#ifndef OCCX_H
#define OCCX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCCX_ABI_VERSION 2
#define OCCX_MAX_K 32          /* top-k list length limit                     */
#define OCCX_MAX_ARCHS 32      /* archs per launch (u8 index, param block)    */
#define OCCX_N_CLASSES 15      /* 14 countable OpClass rows + Unclassified    */

typedef enum occx_status {
  OCCX_OK = 0,
  OCCX_ERR_VALUE = 1,              /* ValueError                               */
  OCCX_ERR_ILLEGAL_LAUNCH = 2,     /* IllegalLaunchError   errors.py:43       */
  OCCX_ERR_UNSUPPORTED_ARCH = 3,   /* UnsupportedArchitectureError errors.py:39 */
  OCCX_ERR_NO_CANDIDATES = 4,      /* NoCandidatesError    errors.py:47       */
  OCCX_ERR_ARCH_SPEC = 5,          /* ArchSpecError        errors.py:22       */
  OCCX_ERR_CUDA = 6,
  OCCX_ERR_NCCL = 7,
  OCCX_ERR_CAPACITY = 8,           /* input exceeds a documented table limit  */
  OCCX_ERR_KEY = 9,                /* KeyError (missing throughput entry)      */
  OCCX_ERR_INDEX = 10,             /* IndexError (empty thread-candidate list) */
  OCCX_ERR_PARSE = 11,             /* ParseError           errors.py:8-15     */
  OCCX_ERR_EMPTY = 12,             /* EmptyInputError      errors.py:18       */
  OCCX_ERR_ATTRIBUTE = 13          /* AttributeError: reference parser quirk, sass.py:278-279 */
} occx_status;

typedef enum occx_mode { OCCX_MODE_CORRECTED = 0, OCCX_MODE_VERBATIM = 1 } occx_mode;

/* Context options (occx_ctx_create_ex).  They pick among implementations
 * with identical results: K2 fed by 128-bit LDG instead of the TMA ring
 * (two 512-thread CTAs per SM; the workspace doubles), or the TMA ring with
 * one slice per warp per stage.  Default 0: TMA, two slices.             */
#define OCCX_CTX_K2_FEED_LDG 0x1u
#define OCCX_CTX_K2_ONE_SLICE 0x2u
#define OCCX_CTX_K2_NO_STEAL 0x4u  /* record scorer: static chunks, no tile stealing */

/* occx_score_space flags.  EVERY_KEY: evaluate every candidate's key (no
 * block-bound pruning); the top-k is the same either way.               */
#define OCCX_SCORE_EVERY_KEY 0x1u
typedef enum occx_sum_mode {
  OCCX_SUM_NEUMAIER = 0,   /* CPython >= 3.12 float sum()                     */
  OCCX_SUM_NAIVE = 1       /* CPython <= 3.11 float sum()                     */
} occx_sum_mode;
typedef enum occx_limiter {
  OCCX_LIMIT_WARPS = 0, OCCX_LIMIT_REGISTERS = 1, OCCX_LIMIT_SMEM = 2,
  OCCX_LIMIT_ILLEGAL = 3
} occx_limiter;

/* ArchSpec formula fields (arch.py:29-48) + throughput column.  40 B.
 * cost_key: 0..3 = sm20/sm35/sm52/sm60 column (mix.py:74-106), -1 = none. */
typedef struct occx_arch_t {
  int32_t warp_size, max_threads_per_block, max_blocks_per_mp, max_warps_per_mp;
  int32_t register_file_size, register_alloc_granularity, max_regs_per_thread;
  int32_t shared_mem_per_block, cost_key, reserved;
} occx_arch_t;

/* Canonical 16-byte candidate record; little endian.
 * variant indexes the per-variant feature table; arch indexes occx_arch_t[];
 * blocks / aux (L1-preference index) identify the candidate but feed no
 * formula.  The candidate's global index is its position + index_base.   */
typedef struct occx_cand_t {
  uint32_t variant;
  uint32_t smem;       /* shared bytes per block  (LaunchInput.shared_per_block) */
  uint16_t threads;    /* threads per block       (LaunchInput.threads_per_block) */
  uint16_t blocks;
  uint16_t regs;       /* registers per thread    (LaunchInput.regs_per_thread)  */
  uint8_t arch;
  uint8_t aux;
} occx_cand_t;

/* Full OccupancyResult (occupancy.py:55-65) for one candidate.  32 B.
 * status: OCCX_OK, OCCX_ERR_ILLEGAL_LAUNCH (threads outside [1, max] --
 * the reference raises), OCCX_ERR_VALUE (arch index out of range).       */
typedef struct occx_occ_t {
  uint8_t wpb, limit_warps, active_blocks, active_warps;
  uint8_t limiter, status, reserved0, reserved1;
  uint32_t limit_regs, limit_smem, reg_warp_limit, reserved2;
  double occupancy;
} occx_occ_t;

/* Instruction record for the mix reducer: bit 0 predicate guard, bits 1-16
 * signature id, bits 17-24 register-operand count (sass.py:105-107), bits
 * 25-31 zero.  The low 17 bits (sig << 1 | guard) index the reducer's
 * class table directly.                                                   */
#define OCCX_INSTR(sig, regops, guard) \
  ((uint32_t)(guard) | ((uint32_t)(sig) << 1) | ((uint32_t)(regops) << 17))

/* InstructionMix (mix.py:194-208) in device form.  144 B.
 * counts[c] for device class c (14 OpClass rows in enum order, then
 * Unclassified at 14).  first_key[c] orders dict insertion: 2*i for the
 * class of instruction i, 2*i+1 for the guard PredIns it adds; 0xFFFFFFFF
 * = class absent.  Host-built mixes put the insertion rank there.         */
typedef struct occx_mix_t {
  uint32_t counts[16];
  uint32_t first_key[16];
  uint64_t reg_operands;
  uint32_t n_instr;
  uint32_t reserved;      /* K0 status: OCCX_ERR_CAPACITY when the call holds
                             >= 2^32 records or the kernel >= 2^29 (nothing
                             else of the row is meaningful then), else 0   */
} occx_mix_t;

/* Per-mix sums: flops/mem/ctrl (mix.py:213-223) and intensity (:333-337). */
typedef struct occx_mixsum_t {
  double intensity;
  uint64_t flops, mem, ctrl, unclassified, total;
} occx_mixsum_t;

/* Per (mix, column) Eq. 6 features.  Index order FLOPS, MEM, CTRL, REG.
 * per_class[r] by CPI row (14 classes, Regs at 14); NaN when the reference
 * omits the row (mix.py:309-318).  status: OK / UNSUPPORTED_ARCH / KEY for
 * the lookups cost, coef, cycles and shares make (mix.py:268-306; cost and
 * cycles/shares are NaN on KEY); pc_status: the same for the lookups
 * per_class_cycles makes (mix.py:309-318).  A partial throughput table can
 * fail one set and not the other, exactly as the reference raises.       */
typedef struct occx_feat_t {
  double cost;            /* cost_estimate(mix, cc, scale)  mix.py:321-330 */
  double coef[4];         /* category_coefficients          mix.py:284-293 */
  double cycles[4];       /* category_cycles                mix.py:296-306 */
  double shares[4];       /* pipeline_utilization           mix.py:340-352 */
  double per_class[16];   /* per_class_cycles               mix.py:309-318 */
  int32_t status, pc_status;
} occx_feat_t;

/* One (variant, arch) row of the scorer's feature table.  32 B.
 * member: 128-bit interleaved membership, for b = t/32 - 1 (t % 32 == 0,
 * 32 <= t <= 2048): bit 2b = t survives static_prune, bit 2b+1 = t survives
 * rule_prune (tuning.py:94-127) for this segment, the rule half already
 * chosen by the variant's intensity.  rank_bits = 2^20-1 - dense cost rank
 * among the kernel's variants on this arch, 0 when the arch has no cost
 * column (mix.py:99-106 raises).                                         */
typedef struct occx_vent_t {
  uint32_t member[4];
  uint32_t seg;
  uint32_t key_hi;        /* 0x80000000 | rank_bits << 2: key bits 63, 53-34 */
  uint32_t rank_bits;
  uint32_t reserved;
} occx_vent_t;

/* Cartesian segment of a TuningSpace (tuning.py:30-77) for the on-device
 * candidate generator.  Dimension order TC, BC, UIF, PL, CFLAGS, REGS,
 * SMEM (last fastest).  dim_off/dim_len index a uint32 value pool; UIF,
 * PL and CFLAGS contribute only their index (variant = var_base +
 * i_uif * len_cflags + i_cflags; aux = i_pl).                              */
typedef struct occx_segdesc_t {
  uint64_t start;          /* global index of the segment's first candidate */
  uint64_t size;
  uint32_t arch, var_base;
  uint32_t dim_off[7], dim_len[7];
} occx_segdesc_t;

/* suggest() (occupancy.py:232-279) request / result. */
typedef struct occx_sugg_in_t { uint32_t arch, regs, smem, reserved; } occx_sugg_in_t;
typedef struct occx_sugg_t {
  int32_t status;
  uint32_t best_threads, best_blocks, best_warps, smem_budget, register_headroom;
  double best_occupancy;
} occx_sugg_t;

typedef struct occx_ctx occx_ctx;

/* ---- library / context ------------------------------------------------ */
int occx_abi_version(void);
const char* occx_status_string(int status);
int occx_ctx_create(int device, occx_ctx** out);          /* options 0 */
int occx_ctx_create_ex(int device, uint32_t options, occx_ctx** out);
uint32_t occx_ctx_options(const occx_ctx* ctx);
int occx_ctx_destroy(occx_ctx* ctx);
int occx_ctx_sm_count(const occx_ctx* ctx);
/* Host-side check that h_archs fit the device tables; *bad = first failing
 * index or -1.  Replaces nothing (ArchSpec invariants stay host-side).
 * Small configuration tables (h_archs <= OCCX_MAX_ARCHS entries, the CPI
 * table, the cost columns) are HOST pointers: they travel in the kernel
 * parameter block (constant bank), not through HBM.                      */
int occx_check_archs(const occx_arch_t* h_archs, int n_arch, int* bad);

/* ---- Kd: full occupancy dump ------------------------------------------
 * Replaces occupancy() occupancy.py:163-195 (with limit_by_warps :104-108,
 * register_warp_limit :111-124, limit_by_registers :127-145,
 * limit_by_smem :148-160) over n candidates.  d_occ_f64 may be NULL.   */
int occx_occupancy_batch(const occx_ctx* ctx, const occx_arch_t* h_archs,
                         int n_arch, const occx_cand_t* d_cand, uint64_t n,
                         int mode, occx_occ_t* d_out, void* stream);

/* ---- K4: suggestion sweep ---------------------------------------------
 * Replaces suggest() occupancy.py:232-279 (+ _active_warps_at :214-229). */
int occx_suggest_batch(const occx_ctx* ctx, const occx_arch_t* h_archs,
                       int n_arch, const occx_sugg_in_t* d_in, uint32_t n,
                       int mode, occx_sugg_t* d_out, void* stream);

/* ---- K0: instruction-mix reducer --------------------------------------
 * Replaces aggregate() mix.py:245-261 (classify :176-187 is the d_sig_class
 * LUT lookup).  d_kernel_off has n_kernels+1 entries (CSR).  With the
 * 15-entry identity table (class records, occx_sass_classify) the kernel
 * indexes its increment table by the record's low byte; any other table,
 * 15 entries included, takes the generic lookup -- same results.      */
int occx_mix_reduce(const occx_ctx* ctx, const uint32_t* d_instr,
                    const uint64_t* d_kernel_off, uint32_t n_kernels,
                    const uint8_t* d_sig_class, uint32_t n_sig,
                    occx_mix_t* d_out, void* stream);

/* ---- K1: feature scoring ----------------------------------------------
 * Replaces intensity() mix.py:333-337 per mix and cost_estimate :321-330,
 * category_coefficients/cycles :284-306, per_class_cycles :309-318,
 * pipeline_utilization :340-352 per (mix, column).  h_cols[j] = cost key
 * (-1 unsupported), n_col <= OCCX_MAX_ARCHS; h_cpi = double[4][16] CPI
 * table by CPI row (NaN = missing entry -> OCCX_ERR_KEY).
 * d_feat is [n_mix][n_col]; d_feat may be NULL when n_col == 0.        */
int occx_feature_score(const occx_ctx* ctx, const occx_mix_t* d_mix,
                       uint32_t n_mix, const int32_t* h_cols, uint32_t n_col,
                       const double* h_cpi, double scale, int sum_mode,
                       occx_mixsum_t* d_sum, occx_feat_t* d_feat, void* stream);

/* ---- scorer feature table ---------------------------------------------
 * Builds occx_vent_t[n_var][n_arch] from K1 output: rule side from
 * intensity > 4.0 (tuning.py:22, :120), masks from d_segmask
 * [n_kernel*n_arch][3] = {static, rule-lower, rule-upper}, dense cost rank
 * among the variants of the same kernel.  d_feat is [n_var][n_arch].   */
int occx_build_vtab(const occx_ctx* ctx, const occx_mixsum_t* d_sum,
                    const occx_feat_t* d_feat, uint32_t n_var, uint32_t n_arch,
                    const uint32_t* d_var_kernel, const uint64_t* d_segmask,
                    occx_vent_t* d_vtab, void* stream);

/* ---- K2 + K3: fused score + per-segment top-k -------------------------
 * For every candidate: occupancy (as Kd), static/rule membership, u64 key
 *   bit 63 legal | 62 rule_keep | 61 static_keep | 60-54 active_warps |
 *   53-34 rank_bits | 33-0 (2^34-1 - global index)
 * and the k largest keys per segment (descending; 0-padded) into
 * d_topk[n_seg][k].  Workspace size from occx_score_workspace_bytes.
 * `variant`/`arch` out of range -> candidate excluded.  d_topk == NULL
 * stops after K2: the per-CTA tables stay in d_ws as
 * [occx_score_lists(ctx)][n_seg][k] for occx_topk_merge.  The workspace
 * ends in a scheduler block (the record scorer's per-CTA tile counters
 * and grid-wide per-segment bounds, a multiple of 256 bytes): it must be
 * zero before the first call, and every call leaves it zero.             */
int occx_score_workspace_bytes(const occx_ctx* ctx, uint32_t n_seg, uint32_t k,
                               uint64_t* bytes);
int occx_score_lists(const occx_ctx* ctx);
/* cudaStreamSynchronize(stream) (the scalar API's one-launch path waits on
 * results the kernel wrote into pinned host memory).                     */
int occx_stream_sync(void* stream);
/* Zero the scheduler block of a workspace sized for (n_seg, k) (once,
 * before the first occx_score_topk call on it; cudaMemsetAsync).        */
int occx_score_workspace_init(const occx_ctx* ctx, void* d_ws, uint32_t n_seg, uint32_t k,
                              void* stream);
int occx_score_topk(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                    const occx_cand_t* d_cand, uint64_t n, uint64_t index_base,
                    int mode, const occx_vent_t* d_vtab, uint32_t n_var,
                    uint32_t n_seg, uint32_t k, void* d_ws, uint64_t ws_bytes,
                    uint64_t* d_topk, void* stream);

/* K3 alone: merge n_lists top-k tables [n_lists][n_seg][k] into one
 * (multi-GPU: after the all-gather of per-rank tables).  Launched as a
 * programmatic dependent of the kernel before it on the stream (it waits
 * for that kernel's writes before reading d_lists).                    */
int occx_topk_merge(const occx_ctx* ctx, const uint64_t* d_lists,
                    uint32_t n_lists, uint32_t n_seg, uint32_t k,
                    uint64_t* d_out, void* stream);

/* ---- K2i: implicit-grid score + top-k -----------------------------------
 * Same result as generating candidates [begin, begin+n) with
 * occx_gen_space and scoring them with occx_score_topk (index_base = begin),
 * without materialising records: each candidate is decoded from its global
 * index inside the scorer (enumerate_space order, tuning.py:75-77).
 * Segment blocks (|REGS| x |SMEM|) must be < 2^32 candidates.
 * key_offset is added to every candidate's global index in its key (0 for
 * the plain space; r * total when rank r of a weak-scaling run scores its
 * own copy of the space, so keys stay unique across ranks).  flags: 0 or
 * OCCX_SCORE_EVERY_KEY (same top-k; no block skipping).                  */
int occx_score_space(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                     const occx_segdesc_t* d_desc, uint32_t n_desc,
                     const uint32_t* d_pool, uint32_t n_pool, uint64_t begin,
                     uint64_t n, uint64_t key_offset, int mode, uint32_t flags,
                     const occx_vent_t* d_vtab, uint32_t n_var,
                     uint32_t n_seg, uint32_t k, void* d_ws, uint64_t ws_bytes,
                     uint64_t* d_topk, void* stream);

/* ---- score_space() in one call ----------------------------------------
 * The whole public score_space() step on `stream`: copy the packed space
 * description h_blob (blob_off[5] byte offsets of: occx_segdesc_t[n_seg] |
 * u32 value pool[n_pool] | u64 membership masks[n_seg][3] (static,
 * rule-lower, rule-upper; bit t/32-1) | u32 var_kernel[n_var] |
 * occx_mix_t[n_var]) to d_buf, run K1 (h_cpi[4][16], scale, sum_mode) + the
 * feature table + K2i over candidates [begin, begin+n) (keys carry index +
 * key_offset) + K3, and copy the [n_seg][k] top-k keys to h_topk, returning
 * when they are there.  h_topk == NULL: no copy and no wait; the table is
 * left at d_buf + occx_space_buf_bytes' *topk_off.  Replaces the
 * per-candidate occupancy / static_prune / rule_prune / cost_estimate loop
 * the reference's users write (occupancy.py:163-195, tuning.py:94-127,
 * mix.py:321-337).                                                       */
int occx_space_buf_bytes(const occx_ctx* ctx, uint64_t blob_bytes, uint32_t n_var,
                         uint32_t n_arch, uint32_t n_seg, uint32_t k, uint64_t* bytes,
                         uint64_t* topk_off);
int occx_score_space_host(const occx_ctx* ctx, const occx_arch_t* h_archs, int n_arch,
                          const void* h_blob, uint64_t blob_bytes, const uint64_t* blob_off,
                          uint32_t n_seg, uint32_t n_pool, uint32_t n_var,
                          const double* h_cpi, double scale, int sum_mode,
                          uint64_t begin, uint64_t n, uint64_t key_offset, int mode,
                          uint32_t flags, uint32_t k, void* d_buf, uint64_t buf_bytes,
                          uint64_t* h_topk, void* stream);

/* ---- candidate generator ----------------------------------------------
 * enumerate_space() tuning.py:75-77 decoded on device: writes candidates
 * [begin, begin+n) of the concatenated segments.                       */
int occx_gen_space(const occx_ctx* ctx, const occx_segdesc_t* d_desc,
                   uint32_t n_desc, const uint32_t* d_pool, uint64_t begin,
                   uint64_t n, occx_cand_t* d_out, void* stream);

/* ---- host: disassembly tokenizer -----------------
 * Replaces parse_disassembly() sass.py:300-339 (+ parse_instruction_line
 * :236-288, register_operand_count :105-107) for the K0 path: UTF-8 text
 * (str encoded with 'surrogatepass') -> per-function names, CSR offsets and
 * 4-byte OCCX_INSTR records over an interned signature table (opcode and
 * modifiers joined by 0x1F, dots dropped).  Same functions, instructions and
 * errors as the reference; on OCCX_ERR_PARSE / _ATTRIBUTE, *err_line is the
 * 1-based line and occx_sass_error_text() the message (for the ';' error:
 * the offending opcode token).  The result is owned by the library until
 * occx_sass_free (also call it after errors).                           */
typedef struct occx_sass occx_sass;
int occx_sass_parse(const char* utf8, uint64_t n_bytes, occx_sass** out, int64_t* err_line);
/* Same, with the minimum bytes per worker-thread chunk (0 = 1 MB default);
 * small values split the text at many line boundaries (results identical). */
int occx_sass_parse_ex(const char* utf8, uint64_t n_bytes, uint64_t chunk_bytes_min,
                       occx_sass** out, int64_t* err_line);
uint32_t occx_sass_n_kernels(const occx_sass* r);
uint64_t occx_sass_n_instr(const occx_sass* r);
const uint32_t* occx_sass_records(const occx_sass* r);
const uint64_t* occx_sass_offsets(const occx_sass* r);
const char* occx_sass_kernel_name(const occx_sass* r, uint32_t k);
uint32_t occx_sass_n_sigs(const occx_sass* r);
const char* occx_sass_signature(const occx_sass* r, uint32_t i);
const char* occx_sass_error_text(const occx_sass* r);
/* All kernel names / all signatures in one buffer, joined by 0x1E (a line
 * break, so neither contains it); *n_bytes = its length.  One call instead
 * of one per name / signature.                                           */
const char* occx_sass_names_blob(const occx_sass* r, uint64_t* n_bytes);
const char* occx_sass_signatures_blob(const occx_sass* r, uint64_t* n_bytes);
/* Rewrite the records in place with class ids instead of signature ids
 * (sig_class[n_sig]: classify() per interned signature, mix.py:176-187;
 * values <= 14): "class records" for occx_mix_reduce with the identity
 * class table (n_sig = 15).                                              */
int occx_sass_classify(occx_sass* r, const uint8_t* sig_class, uint32_t n_sig);
void occx_sass_free(occx_sass* r);

#ifdef __cplusplus
}
#endif
#endif /* OCCX_H */
