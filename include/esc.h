/*
 * esc.h — C ABI of the B200-native exact-selectivity-computation (ESC) hot path.
 *
 * The reference (`escdb`, /root/reference/pkg/src/escdb) is pure Python + numpy and has no
 * FFI layer; its drop-in boundary is a set of Python function signatures.  Each entry point
 * below replaces the numpy body of one of them (file:line in the reference):
 *
 *   esc_scan_count   executor.count_star            executor.py:218-224  (+ _eval_mask :180-199,
 *                    _eval_atom :149-177, _eval_fncall :128-146, _text_lut/_apply_lut :73-94)
 *                    reached through optimizer.compute_exact_selectivity optimizer.py:152-168
 *                    and executor.execute_count executor.py:232-250
 *   esc_compact      executor.eval_predicate        executor.py:202-215  (row ids, ascending)
 *                    optimizer.materialize_pushdown  optimizer.py:180-194 (eval + Column.take
 *                    storage.py:176-184 of every needed column, fused into one pass)
 *   esc_gather       storage.Column.take             storage.py:176-184
 *
 * All pointers in esc_column_t / output arrays are DEVICE pointers (or host-mapped pinned
 * memory for `result`).  No entry point allocates or frees caller memory; scratch lives in a
 * caller-provided workspace (esc_workspace_bytes / esc_workspace_init).  Every entry point is
 * asynchronous on `stream` (a cudaStream_t passed as void*) and returns ESC_OK or an error
 * code; esc_last_error() returns a thread-local message for the last failure.
 *
 * Semantics (bit-exact with the reference):
 *   - every atom is false when any operand is NULL; AND/OR/NOT are two-valued above that;
 *   - comparisons happen in the numpy (NEP 50) promotion domain chosen by the host compiler
 *     (int64 exact / float32 / float64), carried in esc_instr_t.domain;
 *   - UDF programs evaluate CPython float semantics (no FMA contraction, floored %, //);
 *   - row order of every compaction output is ascending logical row order.
 */
#ifndef ESC_H_
#define ESC_H_

#ifdef __CUDACC_RTC__  /* compiled by NVRTC for the JIT tier: no system headers */
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* 2: esc_csv_parse takes d_null_seen; esc_set_hit_lists; the ESC_UDF_RINT opcode */
#define ESC_ABI_VERSION 2

#define ESC_MAX_COLS 32     /* column slots one program may reference            */
#define ESC_MAX_INSTRS 96   /* boolean program length                              */
#define ESC_MAX_UDFS 8      /* UDF atoms per program                               */
#define ESC_MAX_UDF_OPS 128 /* total UDF arithmetic ops per program                */
#define ESC_MAX_UDF_ARGS 8  /* arguments per UDF                                   */
#define ESC_MAX_STACK 16    /* nesting depth of the boolean program                */
#define ESC_MAX_PROJ 32     /* projected columns one compaction may emit           */

/* status codes */
enum {
  ESC_OK = 0,
  ESC_ERR_INVALID = 1,   /* malformed program / arguments                     */
  ESC_ERR_CUDA = 2,      /* CUDA runtime error (message has the CUDA string)    */
  ESC_ERR_WORKSPACE = 3, /* workspace too small / misaligned                    */
  ESC_ERR_UNSUPPORTED = 4
};

/* physical storage types of a column (native widths, little endian) */
enum {
  ESC_I8 = 0, ESC_I16 = 1, ESC_I32 = 2, ESC_I64 = 3,
  ESC_F32 = 4, ESC_F64 = 5, ESC_U8 = 6, ESC_U16 = 7, ESC_U32 = 8
};

/* boolean-program opcodes */
enum {
  ESC_OP_CMP = 1,     /* col_a <cmp> k0                 (Equality / Comparison)       */
  ESC_OP_RANGE = 2,   /* k0 <= col_a <= k1 (inclusive)  (Range)                       */
  ESC_OP_LUT = 3,     /* bit lut[aux + code(col_a)]      (TEXT range/ordering)         */
  ESC_OP_COLCMP = 4,  /* col_a <cmp> col_b              (ColumnCompare)               */
  ESC_OP_NOTNULL = 5, /* ~null(col_a)                   (FoldedAtom(True))            */
  ESC_OP_FALSE = 6,   /* all false                      (FoldedAtom(False))           */
  ESC_OP_UDF = 7,     /* udf[aux](args) <cmp> k0.f      (FnCall)                      */
  ESC_OP_PUSH = 8,    /* open a nested group combined into the outer result by `combine` */
  ESC_OP_POP = 9,     /* close the group: acc = saved <combine> acc                     */
  ESC_OP_NOT = 10     /* acc = ~acc (two-valued NOT)                                   */
};

/* how an atom / group result merges into the running accumulator */
enum { ESC_COMB_SET = 0, ESC_COMB_AND = 1, ESC_COMB_OR = 2 };

/* comparison operators */
enum { ESC_CMP_EQ = 0, ESC_CMP_NE = 1, ESC_CMP_LT = 2, ESC_CMP_LE = 3, ESC_CMP_GT = 4, ESC_CMP_GE = 5 };

/* comparison domains (numpy NEP 50 promotion of column dtype with the constant) */
enum { ESC_DOM_I64 = 0, ESC_DOM_F32 = 1, ESC_DOM_F64 = 2 };

/* UDF opcodes (postfix, float64 stack; CPython float semantics) */
enum {
  ESC_UDF_ARG = 1,      /* push float64(arg[a]) (DECIMAL: / divisor[a])  */
  ESC_UDF_CONST = 2,    /* push k                                        */
  ESC_UDF_ADD = 3, ESC_UDF_SUB = 4, ESC_UDF_MUL = 5,
  ESC_UDF_DIV = 6,      /* ZeroDivisionError on /0                      */
  ESC_UDF_MOD = 7,      /* CPython float_rem (floored), error on %0     */
  ESC_UDF_FLOORDIV = 8, /* CPython float_floor_div, error on //0        */
  ESC_UDF_NEG = 9, ESC_UDF_ABS = 10,
  ESC_UDF_SQUARE = 11,  /* x ** 2 (OverflowError when finite x overflows) */
  /* comparisons: pop b, a; push 1.0 if (a op b) else 0.0 (IEEE: NaN compares false, != true) */
  ESC_UDF_LT = 12, ESC_UDF_LE = 13, ESC_UDF_GT = 14, ESC_UDF_GE = 15, ESC_UDF_EQ = 16, ESC_UDF_NE = 17,
  /* control flow of traced branches (if / else, conditional expressions, min / max): offsets in
   * `arg`, relative to the next op, always forward */
  ESC_UDF_JMPF = 18,    /* pop c; skip `arg` ops when c == 0.0 */
  ESC_UDF_JMP = 19,     /* skip `arg` ops */
  /* math.floor / math.ceil / int(): integral result (ValueError on NaN, OverflowError on inf) */
  ESC_UDF_FLOOR = 20, ESC_UDF_CEIL = 21, ESC_UDF_TRUNC = 22,
  ESC_UDF_SQRT = 23,    /* math.sqrt (ValueError "math domain error" below zero) */
  ESC_UDF_RINT = 24     /* round(x): nearest integer, ties to even (errors as ESC_UDF_FLOOR) */
};

/* UDF failure codes (low 3 bits of esc_result_t.udf_fail[]) */
enum { ESC_FAIL_DIV = 1, ESC_FAIL_MOD = 2, ESC_FAIL_FLOORDIV = 3, ESC_FAIL_POW = 4, ESC_FAIL_NAN_INT = 5,
       ESC_FAIL_INF_INT = 6, ESC_FAIL_DOMAIN = 7 };

typedef union {
  int64_t i;
  double f;
} esc_const_t;

typedef struct {
  uint8_t op;      /* ESC_OP_*                                      */
  uint8_t combine; /* ESC_COMB_*                                    */
  uint8_t cmp;     /* ESC_CMP_*                                     */
  uint8_t domain;  /* ESC_DOM_*                                     */
  uint8_t col_a;   /* column slot                                   */
  uint8_t col_b;   /* second column slot (COLCMP)                   */
  uint8_t neg;     /* invert the atom result before combining       */
  uint8_t pad0;
  uint32_t aux;    /* LUT word offset (LUT) / UDF index (UDF)      */
  uint32_t aux2;   /* LUT size in codes (LUT)                       */
  esc_const_t k0;
  esc_const_t k1;
} esc_instr_t; /* 32 bytes */

typedef struct {
  uint8_t op;  /* ESC_UDF_* */
  uint8_t arg; /* argument index for ESC_UDF_ARG */
  uint8_t pad[6];
  double k;    /* constant for ESC_UDF_CONST */
} esc_udf_op_t; /* 16 bytes */

typedef struct {
  uint16_t first_op; /* index into udf_ops                               */
  uint8_t n_ops;
  uint8_t n_args;
  uint8_t dense;     /* 1: evaluate on every row to detect failures      */
  uint8_t pad[3];
  uint8_t arg_col[ESC_MAX_UDF_ARGS];  /* column slot per argument          */
  double arg_div[ESC_MAX_UDF_ARGS];   /* DECIMAL descale divisor, 0 = none */
} esc_udf_t;

/* A compiled predicate (host memory; passed to the kernel by value). */
typedef struct {
  uint32_t abi_version;
  uint16_t n_instrs;
  uint16_t n_udfs;
  uint16_t n_udf_ops;
  uint16_t max_depth;
  uint32_t lut_words;            /* 32-bit words at `lut` (device memory)  */
  const uint32_t* lut;           /* device pointer to concatenated LUT bitmaps, may be NULL */
  esc_instr_t instrs[ESC_MAX_INSTRS];
  esc_udf_t udfs[ESC_MAX_UDFS];
  esc_udf_op_t udf_ops[ESC_MAX_UDF_OPS];
} esc_program_t;

/* One column slot: device buffers at native width. */
typedef struct {
  const void* data;     /* device pointer, `nrows` values of `dtype`                  */
  const uint8_t* nulls; /* device pointer to a bool mask (1 = NULL), or NULL if none  */
  int32_t dtype;        /* ESC_I8 ...                                                 */
  int32_t flags;        /* ESC_COL_* hints                                            */
  const uint32_t* null_bits; /* optional: the same NULLs packed 1 bit per row (bit r%32 of word
                                r/32; esc_pack_nulls); count / selection scans then stream N/8
                                bytes of NULL state instead of N.  NULL = use the byte mask */
} esc_column_t;

/* esc_column_t.flags: stage this column through shared memory even when the program does not
 * reference it (a projection-only column of a dense compaction: reading it whole by TMA beats
 * sector-granular gathers once most sectors hold a hit). */
#define ESC_COL_STAGE 1

/* Result block written by the last CTA of a launch (device or host-mapped pinned memory). */
typedef struct {
  uint64_t count;                  /* exact qualifying rows                               */
  uint64_t udf_fail[ESC_MAX_UDFS]; /* (first failing logical row << 3 | code), ~0 = none  */
} esc_result_t;

/* Output of a compaction: one destination per projected slot. */
/* esc_outputs_t.flags */
#define ESC_OUT_SKIP_OVER_CAPACITY 1 /* materialisation: do nothing when the selection's device
                                        count (esc_selection_t.d_count) exceeds `capacity`, so a
                                        caller can launch it before reading the count back */

typedef struct {
  int32_t n_proj;
  int32_t flags;                       /* ESC_OUT_*                                   */
  int32_t slot[ESC_MAX_PROJ];          /* column slot of each projected column        */
  void* out_values[ESC_MAX_PROJ];      /* device buffers, `capacity` values each      */
  uint8_t* out_nulls[ESC_MAX_PROJ];    /* device bool buffers or NULL                 */
  int64_t* out_row_ids;                /* optional: physical row id of every hit      */
  int64_t capacity;                    /* rows beyond capacity are counted, not written */
} esc_outputs_t;

/* ---- workspace ------------------------------------------------------------------------ */

/* Bytes of workspace a launch over `nrows` rows needs (tile status words + counters). */
size_t esc_workspace_bytes(int64_t nrows);

/* One-time initialisation of a workspace (async memset on `stream`). Launches leave the
 * workspace clean again, so this is only needed after allocation or after a failed launch. */
int esc_workspace_init(void* d_ws, size_t ws_bytes, void* stream);

/* ---- hot path --------------------------------------------------------------------------- */

/* Exact count of rows satisfying `prog` over logical rows [0, nrows).
 * replaces executor.count_star (executor.py:218-224).
 * d_row_ids: optional device int64 array; logical row i reads physical row d_row_ids[i]
 * (RowSelection chaining, executor.py:211-215).  Writes `result` on completion. */
int esc_scan_count(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                   int64_t nrows, const int64_t* d_row_ids, esc_result_t* result,
                   void* d_ws, size_t ws_bytes, void* stream);

/* Predicate + exact count + order-preserving compaction of the projected columns (and/or the
 * physical row ids of the hits).  replaces executor.eval_predicate (executor.py:202-215) and
 * optimizer.materialize_pushdown (optimizer.py:180-194).  Runs esc_scan_select into the
 * workspace, then esc_materialize_selection.  Rows beyond outs->capacity are counted, not
 * written. */
int esc_compact(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                int64_t nrows, const int64_t* d_row_ids, const esc_outputs_t* outs,
                esc_result_t* result, void* d_ws, size_t ws_bytes, void* stream);

/* The same result in ONE pass over the predicate columns: tiles are ranked with a
 * decoupled look-back over per-tile status words (a writer warp per smem stage) and copied
 * out coalesced.  Bit-identical to esc_compact; on B200 the cross-CTA look-back latency makes it
 * slower than the selection path for persistent grids, so it is not the default. */
int esc_compact_onepass(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                        int64_t nrows, const int64_t* d_row_ids, const esc_outputs_t* outs,
                        esc_result_t* result, void* d_ws, size_t ws_bytes, void* stream);

/* A selection recorded by esc_scan_select (device buffers owned by the caller).
 *  - bitmap: bit i of word i/32 = logical row i qualifies (row-linear);
 *  - seg_counts: hits per warp segment of seg_rows rows (set by the scan), OR-ed with
 *    ESC_SEG_CAPTURED when the segment was sparse enough (<= seg_rows/32 hits) for the scan to
 *    CAPTURE the hits' projected values into cap_values (cap_per_seg slots per segment, stored
 *    slot-major: hit j of segment s is entry j * cap_stride + s, so the compaction's reads of the
 *    few slots sparse segments use are contiguous), and the materialisation copies them instead
 *    of gathering rows from HBM again. */
#define ESC_SEG_CAPTURED 0x80000000u
typedef struct {
  uint32_t* bitmap;
  uint32_t* seg_counts;
  int32_t seg_rows;     /* out: rows per segment                                  */
  int32_t cap_per_seg;  /* out: capture slots per segment (seg_rows / 32)         */
  int32_t n_cap;        /* in: captured projections (0 = none)                     */
  int32_t cap_stride;   /* out: entries between a segment's consecutive slots      */
  int32_t cap_slot[ESC_MAX_PROJ];   /* in: column slot (of the scan's cols) per capture */
  void* cap_values[ESC_MAX_PROJ];   /* in: esc_selection_sizes().cap_entries values each */
  uint8_t* cap_nulls[ESC_MAX_PROJ]; /* in: null bytes per capture, or NULL                */
  uint64_t* d_count;                /* in: optional device word; the scan stores the exact count
                                       there when it completes (ESC_OUT_SKIP_OVER_CAPACITY) */
  const uint64_t* d_gate;           /* in: optional device word the materialisation's
                                       ESC_OUT_SKIP_OVER_CAPACITY test reads INSTEAD of d_count —
                                       written between the scan and the compaction by
                                       esc_count_gate (multi-GPU: the GLOBAL count decides) */
} esc_selection_t;

/* Upper bounds of the selection buffers for `nrows` rows: bitmap words, segments (seg_counts
 * entries) and capture entries (per captured column). */
int esc_selection_sizes(int64_t nrows, int64_t* bitmap_words, int64_t* max_segments, int64_t* cap_entries);

/* The count sub-query that also RECORDS its selection (bitmap + segment counts, and the
 * projected values of sparse segments' hits).  Costs N/8 bytes of bitmap writes on top of
 * esc_scan_count; materialisation then never re-evaluates the predicate (the reference re-scans:
 * optimizer.py:191). */
int esc_scan_select(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                    int64_t nrows, const int64_t* d_row_ids, esc_selection_t* sel,
                    esc_result_t* result, void* d_ws, size_t ws_bytes, void* stream);

/* Order-preserving compaction of the rows a selection marks: per-segment offsets by a scan of
 * the segment counts; captured segments are copied from the capture buffers, the others
 * gathered through the bitmap (one row per lane of a word: contiguous reads and writes).
 * cols[outs->slot[k]] is projection k (cols as given to esc_scan_select). */
int esc_materialize_selection(const esc_selection_t* sel, int64_t nrows, const esc_column_t* cols,
                              int32_t ncols, const int64_t* d_row_ids, const esc_outputs_t* outs,
                              void* d_ws, size_t ws_bytes, void* stream);

/* A queued ESC step — esc_scan_select + esc_materialize_selection with the same arguments —
 * prepared ONCE (program lowering, tile geometry, JIT kernel lookup, compaction plan) and then
 * re-issued by esc_step_plan_launch with no host work beyond the launches.  Every pointer is
 * captured: the plan is valid while those buffers (workspace, selection, outputs, result) are.
 * sel == NULL (mat_cols unused) prepares the one-pass variant instead — esc_compact_onepass with
 * the same arguments — whose outputs esc_step_plan_rebind may later point at new buffers of the
 * same shape (small tables hand their output buffers over as the temp, so each step has new
 * ones; the prepared launch stays). */
int esc_step_plan_create(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                         esc_selection_t* sel, const esc_column_t* mat_cols, int32_t mat_ncols,
                         const esc_outputs_t* outs, esc_result_t* result, void* d_ws, size_t ws_bytes,
                         void** out_plan);
#define ESC_PLAN_GRAPH 4 /* esc_step_plan_launch parts flag: issue a single part as a (cached) CUDA graph too */
int esc_step_plan_launch(void* plan, int32_t parts, void* stream); /* parts: 1 scan, 2 compaction, 3 both
                                                                      (| ESC_PLAN_GRAPH) */
int esc_step_plan_rebind(void* plan, const esc_outputs_t* outs); /* one-pass plans; same n_proj,
                                                                     slots, capacity, null outputs */
int esc_step_plan_destroy(void* plan);

/* ---- multi-GPU row partitioner (K3) ------------------------------------------
 * Rank r of G holds rows [floor(r*N/G), floor((r+1)*N/G)) of a table (the reference's np.linspace
 * row-range split, executor.py:485-489).  After an all_gather of the ranks' device counts (int64
 * each, rank order; NCCL on the same stream), ONE thread folds them on the device:
 *   out[0] = global count  (sum)                 -> the push-down decision (optimizer.py:171-177)
 *   out[1] = exclusive offset of rank `rank`     -> where this rank's compacted slice starts in the
 *                                                   global, order-preserving temp (executor.py:500-504)
 *   out[2] = gate: 0 when the global count <= capacity, else 2^62 (> any capacity) — pointed to
 *            by esc_selection_t.d_gate, it makes the queued compaction of a table that does not
 *            qualify GLOBALLY a no-op on every rank.
 * No host round trip between the scan, the exchange and the compaction. */
int esc_count_gate(const int64_t* counts, int32_t world, int32_t rank, int64_t capacity, int64_t* out,
                   void* stream);

/* Packed NULL bitmap of a bool mask: bit (r & 31) of out[r >> 5] = nulls[r] != 0; out holds
 * esc_null_bits_words(n) words (the last ones zero-padded to a 16-byte multiple). */
int64_t esc_null_bits_words(int64_t n);
int esc_pack_nulls(const uint8_t* nulls, int64_t n, uint32_t* out, void* stream);

/* out[i] = col[idx[i]] (values and, when present, nulls).  replaces Column.take
 * (storage.py:176-184). */
int esc_gather(const esc_column_t* col, const int64_t* d_idx, int64_t n, void* out_values,
               uint8_t* out_nulls, void* stream);

/* dst[i] <- src[i] (bytes[i] bytes) for n <= ESC_MAX_REGIONS device regions, in ONE launch: the
 * trim of capacity-sized compaction outputs to their exact row counts (temp-table registration,
 * storage.py:344-352, without one copy launch per column). */
#define ESC_MAX_REGIONS 72
int esc_copy_regions(int32_t n, void* const* dst, const void* const* src, const int64_t* bytes, void* stream);

/* ---- device sort and grouping (esc_sort.cuh; no library kernels) --------------------------
 * Used by the hash build's grouping (f1: np.unique + stable argsort, executor.py:275-303), the CSV
 * loader's TEXT dictionary by first appearance (f3: Dictionary.encode order, storage.py:127-153,
 * :247-275) and the histogram arm's value sort (f4: np.sort, catalog.py:178-223). */

/* Temp bytes for esc_sort_pairs / esc_runs over n keys of key_bytes (4 | 8), with values or not. */
size_t esc_sort_temp_bytes(int64_t n, int32_t key_bytes, int32_t with_values);

/* Stable LSD radix sort of unsigned keys (key_bytes 4 | 8) by bits [begin_bit, end_bit), with
 * optional 64-bit values carried along (vals_in NULL: keys only).  Equal keys keep their input
 * order.  keys_in / vals_in are not modified; outputs must not alias inputs. */
int esc_sort_pairs(const void* keys_in, const uint64_t* vals_in, void* keys_out, uint64_t* vals_out, int64_t n,
                   int32_t key_bytes, int32_t begin_bit, int32_t end_bit, void* temp, size_t temp_bytes,
                   void* stream);

/* Runs of a SORTED key array: unique_keys[r] (decoded to int64: 0 raw, 1 u32, 2 int32 stored
 * ^ 2^31, 3 int64 stored ^ 2^63), starts[0..runs] (starts[runs] = n), counts[r] (optional),
 * run_of[i] (optional) and stats = {runs, first key, last key, largest run}.  Read stats after a
 * stream sync. */
int esc_runs(const void* sorted_keys, int32_t key_bytes, int32_t decode, int64_t n, int64_t* unique_keys,
             int64_t* starts, int64_t* counts, int64_t* run_of, int64_t* stats, void* temp, size_t temp_bytes,
             void* stream);

/* Order-preserving unsigned sort keys of an integer column: 1-4 byte signed -> uint32 ^ 2^31,
 * unsigned -> uint32, int64 -> uint64 ^ 2^63 (decode 2 / 1 / 3 in esc_runs). */
int esc_order_keys(const void* values, int32_t dtype, int64_t n, void* out, void* stream);
/* Values of a column given as runs (esc_runs output) at sorted positions ranks[0..k). */
int esc_rank_values(const int64_t* unique_keys, const int64_t* starts, const int64_t* stats, const int64_t* ranks,
                    int32_t k, int64_t* out, void* stream);
/* Equi-depth histogram buckets over a column given as runs: bucket j = [lo_j, hi_j) with hi_j the
 * end of the last run whose value <= bounds[j+1] (the last bucket ends at n), and its distinct
 * values (reference catalog.py:178-223: searchsorted(right) + distinct counts). */
int esc_hist_buckets(const int64_t* unique_keys, const int64_t* starts, const int64_t* stats, int64_t n,
                     const int64_t* bounds, int32_t nb, int64_t* out_hi, int64_t* out_distinct, void* stream);
/* First-appearance dictionary codes of n TEXT cells from their 64-bit content hashes (nulls:
 * optional bool mask): out_codes[i] (0 for NULL), out_rep[i] = the first row holding the same
 * content (-1 for NULL), out_first[c] = the first row of code c, *out_n_codes (device word) —
 * the reference's Dictionary.encode order (storage.py:127-153).  Hash collisions are the
 * caller's to detect (esc_csv_verify_text compares every cell with its representative). */
size_t esc_dict_temp_bytes(int64_t n);
int esc_dict_encode(const int64_t* hashes, const uint8_t* nulls, int64_t n, int32_t* out_codes, int64_t* out_rep,
                    int64_t* out_first, int64_t* out_n_codes, void* temp, size_t temp_bytes, void* stream);

/* ---- hash joins over the device-resident temps ------------------------ */
#define ESC_MAX_STEPS 8  /* build steps of one probe pipeline */

/* slots[0..capacity) <- -1, then slot of unique key i <- i: first free slot of the linear probe
 * sequence from splitmix64(bits(key)) & (capacity - 1).  capacity: a power of two > n_unique
 * (the reference sizes it for load <= 0.7).  replaces HashTableIndex._insert_all
 * (executor.py:304-325). */
int esc_hash_insert(const int64_t* unique_keys, int64_t n_unique, int64_t* slots, int64_t capacity, void* stream);

/* The grouping half of a hash build (replaces np.unique + the stable argsort of
 * HashTableIndex.__init__, executor.py:275-303): the build rows' keys (rows[i], or i when rows is
 * NULL; NULL keys already excluded by the caller) are sorted stably, so out_group_rows holds the
 * rows grouped by ascending key, each group in ascending row order; out_unique_keys[0..u) the
 * keys, out_group_counts[0..u) their sizes, out_group_start[0..u] the exclusive offsets, and the
 * device words out_stats[0..3] = {u, min key, max key, largest group} (read after a stream sync;
 * many builds can share one).  out_group_counts and out_group_start hold n + 1 entries. */
int esc_hash_build_temp_bytes(int64_t n, size_t* bytes);
/* A star step's dense factor array over keys lo .. lo+span-1 (out_bytes >= span*bits/8, zeroed
 * here): bits = 1 sets bit (key - lo) of every group's key (primary-key dimensions), 8/16/32/64
 * store the group's size there (esc_join_step_t.factor / factor_bits). */
int esc_factor_array(const int64_t* unique_keys, const int64_t* counts, int64_t u, int64_t lo, int64_t span,
                     int32_t bits, void* out, size_t out_bytes, void* stream);
/* A star step's (key, factor) pair table for sparse key ranges: pairs = esc_pairs_bytes(capacity)
 * bytes (16-byte aligned): int64[2 * capacity] (key, factor) slots, then the slots' occupancy
 * bits (capacity / 8 bytes); capacity a power of two > u; factor 0 marks an empty slot;
 * splitmix64 + linear probing as esc_hash_insert.  Probed by esc_join_count in ESC_JOIN_PAIRS
 * mode, which stages the occupancy bits on chip: a key whose home slot is empty is absent. */
size_t esc_pairs_bytes(int64_t capacity);
int esc_pairs_build(const int64_t* unique_keys, const int64_t* counts, int64_t u, int64_t* pairs, int64_t capacity,
                    void* stream);
int esc_hash_build(const void* keys, int32_t key_dtype, const int64_t* rows, int64_t n, int64_t* out_group_rows,
                   int64_t* out_unique_keys, int64_t* out_group_counts, int64_t* out_group_start, int64_t* out_stats,
                   void* d_temp, size_t temp_bytes, void* stream);

/* out_groups[i] = g with unique_keys[g] == key(i), else -1 (absent, NULL key or !valid[i]).
 * key(i) = keys[rows ? rows[i] : i] at native integer width key_dtype; key_nulls (bool mask
 * indexed like keys), rows and valid (bool per i) are optional.  replaces
 * HashTableIndex.probe_groups (executor.py:327-346). */
int esc_hash_probe(const int64_t* slots, int64_t capacity, const int64_t* unique_keys, const void* keys,
                   int32_t key_dtype, const uint8_t* key_nulls, const int64_t* rows, const uint8_t* valid,
                   int64_t n, int64_t* out_groups, void* stream);

/* One probe stage's expansion: tuple i with groups[i] = g >= 0 owns outputs offsets[i] ..
 * offsets[i] + (group_start[g+1] - group_start[g]) - 1, which receive out_tuple = i (optional)
 * and out_row = group_rows[group_start[g] + j] in group order.  replaces _expand_matches and the
 * np.repeat of _probe_chunk (executor.py:373-386, :436-447). */
int esc_expand(const int64_t* groups, const int64_t* offsets, int64_t n, const int64_t* group_start,
               const int64_t* group_rows, int64_t* out_tuple, int64_t* out_row, void* stream);

enum { ESC_JOIN_DENSE = 0, ESC_JOIN_HASH = 1, ESC_JOIN_PAIRS = 2 };

/* One probe-keyed build step of a COUNT pipeline. */
typedef struct {
  const void* key_data;     /* the probe table's key column (device, native integer width)   */
  const uint8_t* key_nulls; /* its bool NULL mask or NULL                                     */
  int32_t key_dtype;
  int32_t mode;             /* ESC_JOIN_DENSE, ESC_JOIN_HASH or ESC_JOIN_PAIRS               */
  /* DENSE (star joins): factor(k) = factor[k - dense_min] for 0 <= k - dense_min < dense_len,
   * else 0; factor_bits = 1 (bitmap of 32-bit words), 8, 16, 32 or 64; 16-byte aligned       */
  int64_t dense_min;
  int64_t dense_len;
  const void* factor;
  int32_t factor_bits;
  int32_t pad;
  /* HASH: g = the key's group (esc_hash_probe's table); weight[s][g] = its factor at stage s.
   * PAIRS (star joins): slots = an esc_pairs_build table of capacity (key, factor) pairs: one
   * dependent load per probed key instead of three (slot, key, weight)                        */
  const int64_t* slots;
  int64_t capacity;
  const int64_t* unique_keys;
  const uint64_t* weight[ESC_MAX_STEPS + 1];
} esc_join_step_t;

typedef struct {
  int32_t n_steps;   /* probe-keyed steps below (the others are folded into their weights)   */
  int32_t n_stages;  /* build steps of the pipeline: stages 1..n_stages are counted           */
  int32_t star;      /* 1: every step is probe-keyed and stage-invariant (DENSE allowed)      */
  int32_t pad;
  int64_t nrows;     /* probe table rows                                                      */
  const uint32_t* bitmap;          /* rows passing the probe predicate (esc_scan_select), or NULL */
  int32_t stage_of[ESC_MAX_STEPS]; /* stage (1..n_stages) of each probe-keyed step, increasing  */
  esc_join_step_t steps[ESC_MAX_STEPS];
} esc_join_t;

/* The fused probe pipeline of a COUNT(*) plan: d_stage_counts[s] (device u64[n_stages + 1]) =
 * tuples after stage s (s = 0: probe rows passing the predicate) = sum over those rows of the
 * product of their steps' factors — probe_joins' stats.probe_out and result_rows
 * (executor.py:403-474) without expanding a tuple. */
int esc_join_count(const esc_join_t* j, uint64_t* d_stage_counts, void* stream);

/* ---- CSV ingestion into device columns --------------------------------- */
/* replaces storage.load_csv + append_rows' cell conversion (storage.py:245-275, :385-409).
 * 1. esc_csv_count: totals[0] = field separators, totals[1] = record ends (outside quotes),
 *    totals[2] = 1 when the text ends inside a quote;
 * 2. esc_csv_fields: field_end[i] = byte position of separator i, field_kind[i] = 1 ',' / 2 '\n'
 *    or lone '\r' / 3 "\r\n"; rec_end_field[r] = separator index ending record r;
 * 3. esc_csv_parse per column: values (INT64 / DECIMAL scaled by 10**scale / DATE epoch days /
 *    TEXT FNV-1a-64 of the unescaped content + its length), nulls (the \N token), and
 *    first_error = min over failing cells of ((row * ncols + col) << 4 | code); *d_null_seen
 *    (optional) is set to 1 when the column holds a NULL.
 * The workspace (esc_csv_workspace_bytes) carries the chunk summaries from step 1 to step 2. */
enum { ESC_CSV_INT64 = 0, ESC_CSV_DECIMAL = 1, ESC_CSV_DATE = 2, ESC_CSV_TEXT = 3 };
size_t esc_csv_workspace_bytes(int64_t nbytes);
int esc_csv_count(const uint8_t* d_bytes, int64_t nbytes, uint64_t* d_totals, void* d_ws, size_t ws_bytes,
                  void* stream);
int esc_csv_fields(const uint8_t* d_bytes, int64_t nbytes, int64_t* d_field_end, uint8_t* d_field_kind,
                   int64_t* d_rec_end_field, void* d_ws, size_t ws_bytes, void* stream);
int esc_csv_parse(const uint8_t* d_bytes, const int64_t* d_field_end, const uint8_t* d_field_kind, int64_t first_field,
                  int64_t nrows, int32_t ncols, int32_t col, int32_t kind, int32_t scale, int64_t* d_values,
                  int64_t* d_lengths, uint8_t* d_nulls, uint64_t* d_first_error, uint32_t* d_null_seen,
                  void* stream);
/* Record validation (the reference's csv.reader + per-record field count, storage.py:247-275):
 * d_out[0] = min over malformed data records of (record << 32 | fields held; an empty line holds
 * 0), ~0 when all hold ncols fields; d_out[1] = the first record-ending '\r' that is not the last
 * byte (a lone CR inside a line, which Python's csv rejects), ~0 if none.  d_rec_end lists the
 * data records' last fields (header skipped); first_field = the first data record's first field. */
int esc_csv_check(const uint8_t* d_bytes, int64_t nbytes, const int64_t* d_field_end, const uint8_t* d_field_kind,
                  int64_t nsep, const int64_t* d_rec_end, int64_t nrows, int64_t first_field, int32_t ncols,
                  uint64_t* d_out, void* stream);
/* TEXT dictionary check: d_bad |= 1 when a cell's content differs from its group representative's
 * (rep[row], -1 for NULL) — i.e. a 64-bit hash collision. */
int esc_csv_verify_text(const uint8_t* d_bytes, const int64_t* d_field_end, const uint8_t* d_field_kind,
                        int64_t first_field, int64_t nrows, int32_t ncols, int32_t col, const int64_t* d_rep,
                        uint32_t* d_bad, void* stream);

/* ---- misc ------------------------------------------------------------------------------- */

const char* esc_last_error(void);
/* Kernels this library has launched since it was loaded (all entry points, all threads). */
int64_t esc_launch_count(void);
int esc_abi_version(void);
/* Number of SMs of the current device (0 when no device). */
int esc_device_sm_count(void);
/* JIT tier (NVRTC-specialised predicate evaluators for large scans).
 * mode 0 = off (interpreter only), 1 = auto (scans of >= min_rows rows; default 2^22),
 * 2 = always; min_rows < 0 keeps the current threshold. */
int esc_set_jit(int mode, int64_t min_rows);
/* Compile the JIT tier's device sources (every kernel instantiation it emits, with a trivial
 * evaluator) through NVRTC; needs no device.  ESC_OK, or ESC_ERR_UNSUPPORTED with the log. */
int esc_jit_selftest(void);
/* out[0..4] = modules compiled, cache hits, compile failures, total compile microseconds,
 * NVRTC available (0/1). */
int esc_jit_stats(int64_t* out);
/* Streamed compaction of dense tiles in esc_materialize_selection: a tile of the selection is
 * streamed through shared memory (instead of gathered row by row) when it holds at least
 * tile_rows / div hits.  div <= 0 turns streaming off; default 32 (env ESC_STREAM_DIV).
 * Returns the previous setting. */
int esc_set_stream_div(int div);
/* Selections over at most max_rows rows are compacted by ONE launch (sel_mid_kernel: block sums
 * published and read flat, then each block's hits expanded and written) instead of the offsets
 * scan + streamed/gathered compaction chain, when the output capacity is at most a quarter of the
 * rows (denser results stream better through the chain); 0 turns it off, >= 2^40 forces it for
 * every size and density, < 0 leaves it.  Default 32M rows (env ESC_MID_MAX_ROWS).  Returns the
 * previous setting. */
int64_t esc_set_mid_max_rows(int64_t max_rows);
/* Warp hit lists in the gathered compaction: sparse hits are listed per warp and gathered 32 at a
 * time by the whole warp (every projected column's loads in flight together) instead of by the
 * lane that found them.  mode 0 = off, 1 = auto (output capacity <= 1 row in 500, on tables
 * whose 32-segment groups fill the GPU; default, env ESC_HIT_LISTS), 2 = always; other values
 * leave it.  Returns the previous setting. */
int esc_set_hit_lists(int mode);
/* Diagnostics: when d_stamps (device, >= 8 x grid uint64) is non-null, every later scan launch
 * writes per-CTA %globaltimer stamps (start, first tile, consumers done, producer done, CTA
 * finished; last CTA: finalisation begin / end) into it.
 * nullptr turns it off (the default). */
int esc_debug_trace(void* d_stamps);
/* sizeof() of the ABI structs, for binding checks: 0 program, 1 instr, 2 udf, 3 udf_op,
 * 4 column, 5 result, 6 outputs, 7 selection, 8 join step, 9 join; -1 for an unknown id. */
int esc_struct_size(int which);
/* Tile geometry the kernels use for a program over these columns (for roofline accounting). */
int esc_tile_rows(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols);

#ifdef __cplusplus
}
#endif
#endif /* ESC_H_ */
