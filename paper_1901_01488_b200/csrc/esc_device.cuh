// esc_device.cuh — device side of the ESC kernels (design notes: esc_kernels.cu).
//
// Compiled twice: ahead of time by nvcc (esc_kernels.cu, predicate = the opcode interpreter) and
// at run time by NVRTC for the JIT tier (predicate = generated straight-line code, jit.cpp), so
// it includes no system headers.
#pragma once

#include "esc.h"

namespace esc {


#ifndef ESC_CONSUMER_WARPS
#define ESC_CONSUMER_WARPS 8
#endif
constexpr int kConsumerWarps = ESC_CONSUMER_WARPS;
constexpr int kChunkRows = 128;  // one warp chunk: 32 lanes x 4 consecutive rows
constexpr int kMaxStages = 16;  // narrow tiles (one 4-byte column: 16 KB) need many in flight
constexpr int kMaxWriters = 8;  // K2 one-pass: one writer warp per ring slot, so <= 8 stages
constexpr uint32_t kSmemBudget = 200 * 1024;  // dynamic smem for the stage ring
constexpr int kStatusValueBits = 46;
constexpr unsigned long long kStatusValueMask = (1ull << kStatusValueBits) - 1;
constexpr unsigned long long kFlagAggregate = 1;
constexpr unsigned long long kFlagPrefix = 2;
constexpr uint32_t kNoNulls = 0xFFFFFFFFu;
constexpr uint32_t kPackedNulls = 0x80000000u;  // KInstr.noff flag: the staged NULLs are 1 bit per row

template <bool COMPACT>
struct Layout {
  static constexpr int kWriters = COMPACT ? kMaxWriters : 0;  // K2: one look-back / copy-out warp per ring slot
  static constexpr int kFirstConsumer = 1 + kWriters;
  static constexpr int kThreads = (kFirstConsumer + kConsumerWarps) * 32;
};

// ------------------------------------------------------------------------------------------
// workspace layout
// ------------------------------------------------------------------------------------------
struct WsHeader {
  unsigned long long count;   // running count (atomicAdd per CTA)
  unsigned long long ticket;  // tile ticket counter (compaction)
  unsigned long long done;    // CTAs finished (last-CTA detection)
  unsigned long long pad0;
  unsigned long long fail[ESC_MAX_UDFS];  // first failing row per UDF (packed), ~0 = none
  unsigned long long mid_ticket;  // sel_mid_kernel block tickets   (reset by its last block)
  unsigned long long mid_done;    // sel_mid_kernel blocks past their prefix read (reset likewise)
  unsigned long long pad1[2];
};
static_assert(sizeof(WsHeader) == 128, "header is one 128-byte line");

// lowered (kernel-internal) opcodes
enum KOp : uint8_t {
  K_RANGE_S8 = 0, K_RANGE_U8, K_RANGE_S16, K_RANGE_U16, K_RANGE_S32,  // int32 domain
  K_RANGE_S64, K_RANGE_U32,                                           // int64 domain
  K_RANGE_F32,                                                        // float32 column
  K_RANGE_F64,                                                        // any column -> float64
  K_LUT, K_COLCMP, K_NOTNULL, K_FALSE, K_UDF, K_PUSH, K_POP, K_NOT
};

struct KInstr {
  uint8_t op, combine, neg, col, col_b, cmp, domain, inv;  // inv: NE lowered to !EQ, applied before the NULL floor
  uint32_t soff;  // smem offset of col's values in a stage
  uint32_t noff;  // smem offset of col's null bytes in a stage, kNoNulls if the column has none
  union { long long i; double f; } lo, hi;
  uint32_t aux, aux2;  // LUT word offset / size, UDF index
  uint32_t soff_b, noff_b;  // second column (COLCMP)
};

struct KCol {
  const uint8_t* data;
  const uint8_t* nulls;
  int32_t dtype;
  int32_t width;
  int32_t staged;       // values staged in smem for full tiles
  int32_t nulls_staged; // NULLs staged in smem for full tiles: 1 = a byte per row, 2 = a bit per row
  const uint32_t* null_bits;  // packed NULL bitmap (count / selection scans stage it), or nullptr
  uint32_t smem_off;
  uint32_t smem_null_off;
};

struct KParams {
  KInstr ins[ESC_MAX_INSTRS];
  esc_udf_t udfs[ESC_MAX_UDFS];
  esc_udf_op_t udf_ops[ESC_MAX_UDF_OPS];
  const uint32_t* lut;
  KCol cols[ESC_MAX_COLS];
  int32_t n_ins;
  int32_t ncols;
  int32_t chunks;       // C
  int32_t tile_rows;    // T = kConsumerWarps * 128 * C
  int32_t stages;
  uint32_t stage_bytes;  // stage stride
  uint32_t tma_bytes;    // bytes the bulk copies deliver per stage (expect_tx)
  uint32_t epoch;
  int32_t all_staged;   // every column the program reads is staged (fast evaluator usable)
  int64_t nrows;
  int64_t n_tiles;
  int64_t n_full_tiles;  // tiles [0, n_full_tiles) are staged with TMA
  const int64_t* row_ids;
  WsHeader* hdr;
  unsigned long long* status;
  esc_result_t* result;
  esc_outputs_t outs;
  // K2 fast tiles: every projection is compacted per warp into a stage region, then copied out
  uint32_t proj_off[ESC_MAX_PROJ];   // stage offset of projection k's compacted values
  uint32_t proj_noff[ESC_MAX_PROJ];  // stage offset of its compacted null bytes
  uint8_t proj_mode[ESC_MAX_PROJ];   // values: 0 compact in place, 1 gather hits from HBM, 2 alias
  uint8_t proj_nmode[ESC_MAX_PROJ];  // nulls:  0 in place, 1 gather, 2 alias, 3 none (write zeros)
  int32_t all_fast;      // full tiles use the fast (writer copy-out) path
  int32_t sel_on;             // K1 records the selection into `sel`
  esc_selection_t sel;
  uint32_t rows_off;     // stage offset of the u16 row-index scratch (row-id outputs)
  unsigned long long* trace;  // diagnostics (esc_debug_trace): per-CTA %globaltimer stamps, or nullptr
  int32_t ticket_tiles;       // K1: consecutive tiles per ticket (>= ~128 KB of staged data per ticket)
  int32_t prefetch_l2;        // K1 over a table whose staged bytes fit in L2: every CTA first asks L2 to
                              // prefetch its static share of the full tiles (bulk prefetch), so DRAM
                              // has the whole scan queued from the start instead of ramping with the ring
  unsigned long long* scan_done;  // select: the last CTA sets it (release) once the count, bitmap and
                                  // captures are complete: sel_mid_kernel starts on it, not on the grid's
                                  // completion (griddepcontrol.wait returns ~3 us later), or nullptr
  int32_t bitmap_lean;        // select in a step plan whose compaction reads no bitmap for captured
                              // or empty segments: their bitmap words are not written (DenseRule.lean)
};

// Programmatic dependent launch: the compaction chain's kernels are launched with
// programmaticStreamSerialization, so each may be scheduled while its predecessor still runs; it
// waits (griddepcontrol.wait) before touching anything the predecessor writes, and lets its own
// dependents launch early.  Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk copy, release/acquire
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of [g, g + bytes) (16-byte aligned and sized), 64 KB per instruction
__device__ __forceinline__ void bulk_prefetch_l2(const uint8_t* g, unsigned long long bytes) {
  for (unsigned long long o = 0; o < bytes; o += 65536ull) {
    const uint32_t n = (uint32_t)((bytes - o) < 65536ull ? (bytes - o) : 65536ull);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + o), "r"(n) : "memory");
  }
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// a status word that publishes only its own value (no other data hangs on it) needs no release
// fence before it: look-back readers take the value and nothing else
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

// ------------------------------------------------------------------------------------------
// scalar loads (cold paths: tail tiles, selections, UDF arguments, scatter)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ long long ld_int(const uint8_t* p, int dtype) {
  switch (dtype) {
    case ESC_I8: return *reinterpret_cast<const int8_t*>(p);
    case ESC_I16: return *reinterpret_cast<const int16_t*>(p);
    case ESC_I32: return *reinterpret_cast<const int32_t*>(p);
    case ESC_U8: return *reinterpret_cast<const uint8_t*>(p);
    case ESC_U16: return *reinterpret_cast<const uint16_t*>(p);
    case ESC_U32: return *reinterpret_cast<const uint32_t*>(p);
    default: return *reinterpret_cast<const long long*>(p);
  }
}
// float64 value of any column type (numpy's astype(float64): RN for int64)
__device__ __forceinline__ double ld_f64(const uint8_t* p, int dtype) {
  switch (dtype) {
    case ESC_F32: return (double)*reinterpret_cast<const float*>(p);
    case ESC_F64: return *reinterpret_cast<const double*>(p);
    case ESC_I64: return __ll2double_rn(*reinterpret_cast<const long long*>(p));
    default: return (double)ld_int(p, dtype);
  }
}

// ------------------------------------------------------------------------------------------
// hot path: staged tile, smem-only opcode loops
// ------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void lds4(const uint8_t* p, T (&v)[4]) {
  if constexpr (sizeof(T) == 1) {
    union { uint32_t u; T t[4]; } x;
    x.u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = x.t[0]; v[1] = x.t[1]; v[2] = x.t[2]; v[3] = x.t[3];
  } else if constexpr (sizeof(T) == 2) {
    union { uint2 u; T t[4]; } x;
    x.u = *reinterpret_cast<const uint2*>(p);
    v[0] = x.t[0]; v[1] = x.t[1]; v[2] = x.t[2]; v[3] = x.t[3];
  } else if constexpr (sizeof(T) == 4) {
    union { uint4 u; T t[4]; } x;
    x.u = *reinterpret_cast<const uint4*>(p);
    v[0] = x.t[0]; v[1] = x.t[1]; v[2] = x.t[2]; v[3] = x.t[3];
  } else {
    union { uint4 u[2]; T t[4]; } x;
    x.u[0] = reinterpret_cast<const uint4*>(p)[0];
    x.u[1] = reinterpret_cast<const uint4*>(p)[1];
    v[0] = x.t[0]; v[1] = x.t[1]; v[2] = x.t[2]; v[3] = x.t[3];
  }
}

// int32 domain: (u32)v - (u32)lo <= span  <=>  lo <= v <= hi (wrapping arithmetic)
template <typename T, int C>
__device__ __forceinline__ uint32_t range_i32(const uint8_t* col, int local0, int32_t lo, uint32_t span) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    T v[4];
    lds4<T>(col + (size_t)(local0 + kChunkRows * c) * sizeof(T), v);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((uint32_t)(int32_t)v[j] - (uint32_t)lo <= span) r |= 1u << (4 * c + j);  // unsigned: no UB
  }
  return r;
}

template <typename T, int C>
__device__ __forceinline__ uint32_t range_i64(const uint8_t* col, int local0, long long lo, unsigned long long span) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    T v[4];
    lds4<T>(col + (size_t)(local0 + kChunkRows * c) * sizeof(T), v);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((unsigned long long)(long long)v[j] - (unsigned long long)lo <= span) r |= 1u << (4 * c + j);
  }
  return r;
}

template <int C>
__device__ __forceinline__ uint32_t range_f32(const uint8_t* col, int local0, float lo, float hi) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    float v[4];
    lds4<float>(col + (size_t)(local0 + kChunkRows * c) * 4, v);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (v[j] >= lo && v[j] <= hi) r |= 1u << (4 * c + j);
  }
  return r;
}

template <int C>
__device__ __forceinline__ uint32_t null_bits_staged(const uint8_t* nb, int local0) {
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const uint32_t x = *reinterpret_cast<const uint32_t*>(nb + local0 + kChunkRows * c);
    bits |= ((((x & 0x01010101u) * 0x01020408u) >> 24) & 0xFu) << (4 * c);  // bit 0 of each byte
  }
  return bits;
}
// the same 4*C NULL flags from a staged 1-bit-per-row bitmap (row-linear words)
template <int C>
__device__ __forceinline__ uint32_t null_bits_packed(const uint8_t* nb, int local0) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(nb);
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int r = local0 + kChunkRows * c;  // 4 consecutive rows inside one word (r % 4 == 0)
    bits |= ((w[r >> 5] >> (r & 31)) & 0xFu) << (4 * c);
  }
  return bits;
}
template <int C>
__device__ __forceinline__ uint32_t staged_nulls(const uint8_t* stage, uint32_t noff, int local0) {
  return (noff & kPackedNulls) ? null_bits_packed<C>(stage + (noff & ~kPackedNulls), local0)
                               : null_bits_staged<C>(stage + noff, local0);
}

__device__ __forceinline__ bool cmp_any(int cmp, double a, double b) {
  switch (cmp) {
    case ESC_CMP_EQ: return a == b;
    case ESC_CMP_NE: return a != b;
    case ESC_CMP_LT: return a < b;
    case ESC_CMP_LE: return a <= b;
    case ESC_CMP_GT: return a > b;
    default: return a >= b;
  }
}
__device__ __forceinline__ bool cmp_any(int cmp, long long a, long long b) {
  switch (cmp) {
    case ESC_CMP_EQ: return a == b;
    case ESC_CMP_NE: return a != b;
    case ESC_CMP_LT: return a < b;
    case ESC_CMP_LE: return a <= b;
    case ESC_CMP_GT: return a > b;
    default: return a >= b;
  }
}
__device__ __forceinline__ bool cmp_any(int cmp, float a, float b) {
  switch (cmp) {
    case ESC_CMP_EQ: return a == b;
    case ESC_CMP_NE: return a != b;
    case ESC_CMP_LT: return a < b;
    case ESC_CMP_LE: return a <= b;
    case ESC_CMP_GT: return a > b;
    default: return a >= b;
  }
}

// ------------------------------------------------------------------------------------------
// row addressing for one lane of one tile
// ------------------------------------------------------------------------------------------
struct RowRef {
  const uint8_t* stage;  // smem stage (nullptr: direct HBM reads)
  int64_t grow0;         // logical row of the lane's chunk-0 first row
  int32_t local0;        // row of chunk 0 within the tile
  int64_t nrows;
  const int64_t* ids;    // row-id selection (logical -> physical) or nullptr
};

__device__ __forceinline__ int64_t logical_row(const RowRef& rr, int bit) {
  return rr.grow0 + kChunkRows * (bit >> 2) + (bit & 3);
}
__device__ __forceinline__ int32_t local_row(const RowRef& rr, int bit) {
  return rr.local0 + kChunkRows * (bit >> 2) + (bit & 3);
}
__device__ __forceinline__ int64_t phys_row(const RowRef& rr, int64_t r) {
  return rr.ids ? __ldg(rr.ids + r) : r;
}

// pointer to a column value of the row at `bit`: smem when staged, else HBM
__device__ __forceinline__ const uint8_t* value_ptr(const KCol& col, const RowRef& rr, int bit) {
  if (rr.stage != nullptr && col.staged) return rr.stage + col.smem_off + (size_t)local_row(rr, bit) * col.width;
  return col.data + (size_t)phys_row(rr, logical_row(rr, bit)) * col.width;
}
__device__ __forceinline__ bool is_null(const KCol& col, const RowRef& rr, int bit) {
  if (col.nulls == nullptr) return false;
  if (rr.stage != nullptr && col.nulls_staged) {
    const int32_t l = local_row(rr, bit);
    if (col.nulls_staged == 2)
      return (reinterpret_cast<const uint32_t*>(rr.stage + col.smem_null_off)[l >> 5] >> (l & 31)) & 1u;
    return rr.stage[col.smem_null_off + l] != 0;
  }
  return __ldg(col.nulls + phys_row(rr, logical_row(rr, bit))) != 0;
}

// ---- UDF: CPython float semantics ----------------------------------------------------------
// CPython float_rem (Objects/floatobject.c)
__device__ __forceinline__ double py_mod(double vx, double wx) {
  double mod = fmod(vx, wx);
  if (mod != 0.0) {
    if ((wx < 0.0) != (mod < 0.0)) mod = __dadd_rn(mod, wx);
  } else {
    mod = copysign(0.0, wx);
  }
  return mod;
}

// CPython _float_div_mod -> floordiv
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(__dsub_rn(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0.0) != (mod < 0.0)) div = __dsub_rn(div, 1.0);
  }
  double fd;
  if (div != 0.0) {
    fd = floor(div);
    if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
  } else {
    fd = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return fd;
}

__device__ __noinline__ double udf_eval(const KParams& p, const esc_udf_t& u, const RowRef& rr, int bit,
                                        uint32_t* fail) {
  double stk[16];
  int sp = 0;
  double args[ESC_MAX_UDF_ARGS];
  for (int a = 0; a < u.n_args; ++a) {
    const KCol& col = p.cols[u.arg_col[a]];
    double x = ld_f64(value_ptr(col, rr, bit), col.dtype);
    if (u.arg_div[a] != 0.0) x = __ddiv_rn(x, u.arg_div[a]);
    args[a] = x;
  }
  for (int i = 0; i < u.n_ops; ++i) {
    const esc_udf_op_t& o = p.udf_ops[u.first_op + i];
    switch (o.op) {
      case ESC_UDF_ARG: stk[sp++] = args[o.arg]; break;
      case ESC_UDF_CONST: stk[sp++] = o.k; break;
      case ESC_UDF_NEG: stk[sp - 1] = -stk[sp - 1]; break;
      case ESC_UDF_ABS: stk[sp - 1] = fabs(stk[sp - 1]); break;
      case ESC_UDF_SQUARE: {
        const double x = stk[sp - 1];
        const double y = __dmul_rn(x, x);
        if (isinf(y) && isfinite(x)) { *fail = ESC_FAIL_POW; return 0.0; }
        stk[sp - 1] = y;
        break;
      }
      case ESC_UDF_JMPF:
        if (stk[--sp] == 0.0) i += o.arg;
        break;
      case ESC_UDF_JMP: i += o.arg; break;
      case ESC_UDF_FLOOR: case ESC_UDF_CEIL: case ESC_UDF_TRUNC: case ESC_UDF_RINT: {
        const double x = stk[sp - 1];
        if (isnan(x)) { *fail = ESC_FAIL_NAN_INT; return 0.0; }
        if (isinf(x)) { *fail = ESC_FAIL_INF_INT; return 0.0; }
        stk[sp - 1] = o.op == ESC_UDF_FLOOR ? floor(x) : o.op == ESC_UDF_CEIL ? ceil(x)
                    : o.op == ESC_UDF_TRUNC ? trunc(x) : rint(x);  // rint: ties to even, as round()
        break;
      }
      case ESC_UDF_SQRT: {
        const double x = stk[sp - 1];
        if (x < 0.0) { *fail = ESC_FAIL_DOMAIN; return 0.0; }
        stk[sp - 1] = __dsqrt_rn(x);
        break;
      }
      default: {
        const double b = stk[--sp];
        const double a = stk[sp - 1];
        double r;
        switch (o.op) {
          case ESC_UDF_ADD: r = __dadd_rn(a, b); break;
          case ESC_UDF_SUB: r = __dsub_rn(a, b); break;
          case ESC_UDF_MUL: r = __dmul_rn(a, b); break;
          case ESC_UDF_DIV:
            if (b == 0.0) { *fail = ESC_FAIL_DIV; return 0.0; }
            r = __ddiv_rn(a, b);
            break;
          case ESC_UDF_MOD:
            if (b == 0.0) { *fail = ESC_FAIL_MOD; return 0.0; }
            r = py_mod(a, b);
            break;
          case ESC_UDF_FLOORDIV:
            if (b == 0.0) { *fail = ESC_FAIL_FLOORDIV; return 0.0; }
            r = py_floordiv(a, b);
            break;
          case ESC_UDF_LT: r = a < b ? 1.0 : 0.0; break;
          case ESC_UDF_LE: r = a <= b ? 1.0 : 0.0; break;
          case ESC_UDF_GT: r = a > b ? 1.0 : 0.0; break;
          case ESC_UDF_GE: r = a >= b ? 1.0 : 0.0; break;
          case ESC_UDF_EQ: r = a == b ? 1.0 : 0.0; break;
          default: r = a != b ? 1.0 : 0.0; break;  // ESC_UDF_NE
        }
        stk[sp - 1] = r;
      }
    }
  }
  return stk[0];
}

// UDF atom on the rows of `todo` (all valid rows when the UDF can fail, else the rows whose
// value can still change the result); false where any argument is NULL (executor.py:146)
__device__ __noinline__ uint32_t atom_udf(const KParams& p, const KInstr& I, const RowRef& rr, uint32_t care,
                                          uint32_t valid) {
  const esc_udf_t& u = p.udfs[I.aux];
  uint32_t todo = u.dense ? valid : (care & valid);
  uint32_t r = 0;
  while (todo) {
    const int bit = __ffs(todo) - 1;
    todo &= todo - 1;
    uint32_t failed = 0;
    const double v = udf_eval(p, u, rr, bit, &failed);
    if (failed) {
      atomicMin(&p.hdr->fail[I.aux], (unsigned long long)(logical_row(rr, bit) << 3) | failed);
      continue;
    }
    bool anynull = false;
    for (int a = 0; a < u.n_args; ++a) anynull |= is_null(p.cols[u.arg_col[a]], rr, bit);
    if (!anynull && cmp_any(I.cmp, v, I.lo.f)) r |= 1u << bit;
  }
  return r;
}

// ---- generic per-row atom evaluation (cold: tail tiles, selections, LUT, column compare) ----
__device__ __noinline__ uint32_t atom_generic(const KParams& p, const KInstr& I, const RowRef& rr, uint32_t valid) {
  uint32_t r = 0;
  uint32_t todo = valid;
  while (todo) {
    const int bit = __ffs(todo) - 1;
    todo &= todo - 1;
    bool t = false;
    switch (I.op) {
      case K_NOTNULL:
        t = true;
        break;
      case K_RANGE_F32: {
        const float v = *reinterpret_cast<const float*>(value_ptr(p.cols[I.col], rr, bit));
        t = v >= (float)I.lo.f && v <= (float)I.hi.f;
        break;
      }
      case K_RANGE_F64: {
        const KCol& col = p.cols[I.col];
        const double v = ld_f64(value_ptr(col, rr, bit), col.dtype);
        t = v >= I.lo.f && v <= I.hi.f;
        break;
      }
      case K_LUT: {
        const KCol& col = p.cols[I.col];
        const long long code = ld_int(value_ptr(col, rr, bit), col.dtype);
        if (code >= 0 && code < (long long)I.aux2) t = (__ldg(p.lut + I.aux + (code >> 5)) >> (code & 31)) & 1u;
        break;
      }
      case K_COLCMP: {
        const KCol& a = p.cols[I.col];
        const KCol& b = p.cols[I.col_b];
        const uint8_t* pa = value_ptr(a, rr, bit);
        const uint8_t* pb = value_ptr(b, rr, bit);
        if (I.domain == ESC_DOM_I64) {
          t = cmp_any(I.cmp, ld_int(pa, a.dtype), ld_int(pb, b.dtype));
        } else if (I.domain == ESC_DOM_F32) {  // f32 x {f32, int8, int16, uint8, uint16}: exact in f32
          t = cmp_any(I.cmp, (float)ld_f64(pa, a.dtype), (float)ld_f64(pb, b.dtype));
        } else {
          t = cmp_any(I.cmp, ld_f64(pa, a.dtype), ld_f64(pb, b.dtype));
        }
        if (is_null(b, rr, bit)) t = false;
        break;
      }
      default: {  // integer ranges
        const KCol& col = p.cols[I.col];
        const long long v = ld_int(value_ptr(col, rr, bit), col.dtype);
        t = v >= I.lo.i && v <= I.hi.i;
        break;
      }
    }
    if (I.inv) t = !t;
    if (t && !is_null(p.cols[I.col], rr, bit)) r |= 1u << bit;
  }
  return r;
}

__device__ __forceinline__ uint32_t combine(int mode, uint32_t acc, uint32_t r) {
  return mode == ESC_COMB_AND ? (acc & r) : mode == ESC_COMB_OR ? (acc | r) : r;
}
__device__ __forceinline__ uint32_t care_for(int mode, uint32_t acc, uint32_t care) {
  return mode == ESC_COMB_AND ? (care & acc) : mode == ESC_COMB_OR ? (care & ~acc) : care;
}

// Evaluate the program on this lane's 4*C rows. FAST: the tile is staged and every program
// column is in smem, so range opcodes run the smem loops; otherwise every atom takes the
// generic per-row path.
template <int C, bool FAST>
__device__ __forceinline__ uint32_t eval_program(const KParams& p, const RowRef& rr, uint32_t valid) {
  uint32_t acc = 0, care = valid;
  uint32_t stk_acc[ESC_MAX_STACK], stk_care[ESC_MAX_STACK];
  int sp = 0;
  const int n = p.n_ins;
  for (int pc = 0; pc < n; ++pc) {
    const KInstr& I = p.ins[pc];
    const int op = I.op;
    uint32_t r;
    const uint8_t* col = rr.stage + I.soff;
    const int l0 = rr.local0;
    switch (op) {
      case K_PUSH:
        stk_acc[sp] = acc;
        stk_care[sp] = care;
        ++sp;
        care = care_for(I.combine, acc, care);
        acc = 0;
        continue;
      case K_POP:
        --sp;
        acc = combine(I.combine, stk_acc[sp], acc);
        care = stk_care[sp];
        continue;
      case K_NOT:
        acc = ~acc;
        continue;
      case K_FALSE:
        r = 0;
        break;
      case K_UDF:
        r = atom_udf(p, I, rr, care_for(I.combine, acc, care), valid);
        break;
      case K_RANGE_S8:
        r = FAST ? range_i32<int8_t, C>(col, l0, (int32_t)I.lo.i, (uint32_t)(I.hi.i - I.lo.i)) : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_U8:
        r = FAST ? range_i32<uint8_t, C>(col, l0, (int32_t)I.lo.i, (uint32_t)(I.hi.i - I.lo.i)) : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_S16:
        r = FAST ? range_i32<int16_t, C>(col, l0, (int32_t)I.lo.i, (uint32_t)(I.hi.i - I.lo.i)) : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_U16:
        r = FAST ? range_i32<uint16_t, C>(col, l0, (int32_t)I.lo.i, (uint32_t)(I.hi.i - I.lo.i)) : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_S32:
        r = FAST ? range_i32<int32_t, C>(col, l0, (int32_t)I.lo.i, (uint32_t)(I.hi.i - I.lo.i)) : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_S64:
        r = FAST ? range_i64<long long, C>(col, l0, I.lo.i, (unsigned long long)I.hi.i - (unsigned long long)I.lo.i)
                 : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_U32:
        r = FAST ? range_i64<uint32_t, C>(col, l0, I.lo.i, (unsigned long long)I.hi.i - (unsigned long long)I.lo.i)
                 : atom_generic(p, I, rr, valid);
        break;
      case K_RANGE_F32:
        r = FAST ? range_f32<C>(col, l0, (float)I.lo.f, (float)I.hi.f) : atom_generic(p, I, rr, valid);
        break;
      case K_NOTNULL:
        r = FAST ? (I.noff != kNoNulls ? ~staged_nulls<C>(rr.stage, I.noff, l0) : 0xFFFFFFFFu)
                 : atom_generic(p, I, rr, valid);
        break;
      default:  // K_RANGE_F64, K_LUT, K_COLCMP
        r = atom_generic(p, I, rr, valid);
        break;
    }
    if (FAST && op <= K_RANGE_F32) {
      if (I.inv) r = ~r;
      if (I.noff != kNoNulls) r &= ~staged_nulls<C>(rr.stage, I.noff, l0);
    }
    if (I.neg) r = ~r;
    acc = combine(I.combine, acc, r);
  }
  return acc & valid;
}

template <int C>
__device__ __noinline__ uint32_t eval_direct(const KParams& p, const RowRef& rr, uint32_t valid) {
  return eval_program<C, false>(p, rr, valid);
}

// Scan-time capture of a sparse warp segment's hits (esc_selection_t): the hit rows' values of
// every captured column are copied from the staged tile into the segment's capture slots, in row
// order.  `excl`/`wtp`: the lane's exclusive / the warp's total per-chunk hit counts (8-bit fields).
template <int C>
__device__ __noinline__ void capture_generic(const KParams& p, const RowRef& rr, uint32_t bits, uint32_t excl,
                                             uint32_t wtp, int64_t seg) {
  const size_t stride = (size_t)p.sel.cap_stride;  // slot-major: hit r of segment seg at r * stride + seg
  for (int k = 0; k < p.sel.n_cap; ++k) {
    const KCol& col = p.cols[p.sel.cap_slot[k]];
    uint8_t* dst = static_cast<uint8_t*>(p.sel.cap_values[k]) + (size_t)seg * col.width;
    uint8_t* dn = p.sel.cap_nulls[k] ? p.sel.cap_nulls[k] + (size_t)seg : nullptr;
    uint32_t cb = 0;
    for (int c = 0; c < C; ++c) {
      uint32_t r = cb + ((excl >> (8 * c)) & 0xFFu);
      cb += (wtp >> (8 * c)) & 0xFFu;
      uint32_t m = (bits >> (4 * c)) & 0xFu;
      while (m) {
        const int bit = 4 * c + __ffs(m) - 1;
        m &= m - 1;
        const uint8_t* src = value_ptr(col, rr, bit);
        const size_t e = (size_t)r * stride;
        switch (col.width) {
          case 1: dst[e] = *src; break;
          case 2: reinterpret_cast<uint16_t*>(dst)[e] = *reinterpret_cast<const uint16_t*>(src); break;
          case 4: reinterpret_cast<uint32_t*>(dst)[e] = *reinterpret_cast<const uint32_t*>(src); break;
          default:
            reinterpret_cast<unsigned long long*>(dst)[e] = *reinterpret_cast<const unsigned long long*>(src);
            break;
        }
        if (dn) dn[e] = is_null(col, rr, bit) ? 1 : 0;
        ++r;
      }
    }
  }
}

// Predicate evaluator of the ahead-of-time kernels: the opcode interpreter over a staged tile.
// The JIT tier substitutes a generated straight-line evaluator (and a capture with the captured
// columns' widths and smem offsets baked in) with the same signatures.
struct InterpPred {
  template <int C>
  static __device__ __forceinline__ uint32_t eval(const KParams& p, const RowRef& rr, uint32_t valid) {
    return eval_program<C, true>(p, rr, valid);
  }
  template <int C>
  static __device__ __forceinline__ void capture(const KParams& p, const RowRef& rr, uint32_t bits, uint32_t excl,
                                                 uint32_t wtp, int64_t seg) {
    capture_generic<C>(p, rr, bits, excl, wtp, seg);
  }
};

__device__ __forceinline__ uint32_t valid_bits(int64_t grow0, int64_t nrows, int C) {
  uint32_t v = 0;
  for (int c = 0; c < C; ++c)
    for (int j = 0; j < 4; ++j) v |= (uint32_t)(grow0 + kChunkRows * c + j < nrows) << (4 * c + j);
  return v;
}

// ------------------------------------------------------------------------------------------
// decoupled look-back (one warp)
// ------------------------------------------------------------------------------------------
// Relaxed loads suffice: the status word itself is the only datum read, and it carries its own
// epoch/flag/value; relaxed (unlike acquire) loads of the window pipeline.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ unsigned long long lookback_warp(unsigned long long* status, int64_t tile, unsigned long long agg,
                                            uint32_t epoch, int lane) {
  // the tile's aggregate (tile 0: its inclusive prefix) was published by the last consumer warp
  const unsigned long long tag = (unsigned long long)epoch << 48;
  if (tile == 0) return 0;
  constexpr int J = 8;  // 8 x 32 predecessors in flight per round trip
  unsigned long long excl = 0;
  int64_t q = tile - 1;
  while (true) {
    unsigned long long w[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t idx = q - 32 * j - lane;
      w[j] = idx >= 0 ? ld_relaxed(&status[idx]) : 0ull;
    }
    int consumed = 0;
    bool done = false;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (done || consumed != j) break;
      const int64_t idx = q - 32 * j - lane;
      const bool ok = idx < 0 || (w[j] >> 48) == epoch;
      const bool pre = idx < 0 || (ok && ((w[j] >> kStatusValueBits) & 3ull) == kFlagPrefix);
      const unsigned pm = __ballot_sync(0xFFFFFFFFu, pre);
      const unsigned okm = __ballot_sync(0xFFFFFFFFu, ok);
      const int first = pm ? __ffs(pm) - 1 : 31;
      const unsigned need = first == 31 ? 0xFFFFFFFFu : ((1u << (first + 1)) - 1u);
      if ((okm & need) != need) break;  // a needed predecessor has not published: re-read from here
      unsigned long long part = (lane <= first && idx >= 0) ? (w[j] & kStatusValueMask) : 0ull;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, d);
      excl += part;
      if (pm) done = true;
      ++consumed;
    }
    if (done) break;
    q -= 32 * consumed;
  }
  if (lane == 0) st_relaxed(&status[tile], tag | (kFlagPrefix << kStatusValueBits) | (excl + agg));
  return excl;
}

// ---- scatter of one warp's hits (the warp's rows of a tile, ascending row order) -------------
// Output order inside a warp segment is chunk-major, then lane, then row: a lane's hits of chunk c
// start at chunk_base(c) + lane_excl(c) (both from the packed per-chunk scan).

// one value column / null column, direct per-lane stores (non-staged columns, tail tiles)
template <int C>
__device__ __forceinline__ void scatter_direct(const KParams& p, const RowRef& rr, uint32_t bits, uint32_t excl,
                                               uint32_t wtp, unsigned long long base, int k) {
  const esc_outputs_t& o = p.outs;
  const KCol& col = p.cols[o.slot[k]];
  uint8_t* out = static_cast<uint8_t*>(o.out_values[k]);
  uint8_t* onull = o.out_nulls[k];
  uint32_t cb = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    unsigned long long pos = base + cb + ((excl >> (8 * c)) & 0xFFu);
    cb += (wtp >> (8 * c)) & 0xFFu;
    uint32_t m = (bits >> (4 * c)) & 0xFu;
    while (m) {
      const int bit = 4 * c + __ffs(m) - 1;
      m &= m - 1;
      if ((int64_t)pos < o.capacity) {
        const uint8_t* src = value_ptr(col, rr, bit);
        uint8_t* dst = out + (size_t)pos * col.width;
        switch (col.width) {
          case 1: *dst = *src; break;
          case 2: *reinterpret_cast<uint16_t*>(dst) = *reinterpret_cast<const uint16_t*>(src); break;
          case 4: *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src); break;
          default: *reinterpret_cast<unsigned long long*>(dst) = *reinterpret_cast<const unsigned long long*>(src); break;
        }
        if (onull != nullptr) onull[pos] = is_null(col, rr, bit) ? 1 : 0;
      }
      ++pos;
    }
  }
}

// hits of a column that is not staged: read just the hit rows from HBM into compacted slots
template <typename T, int C>
__device__ __forceinline__ void gather_compact(const uint8_t* data, int64_t grow0, uint8_t* seg, uint32_t bits,
                                               uint32_t excl, uint32_t wtp) {
  const T* src = reinterpret_cast<const T*>(data);
  T* cs = reinterpret_cast<T*>(seg);
  uint32_t cb = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uint32_t r = cb + ((excl >> (8 * c)) & 0xFFu);
    cb += (wtp >> (8 * c)) & 0xFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((bits >> (4 * c + j)) & 1u) cs[r++] = __ldg(src + grow0 + kChunkRows * c + j);
  }
}

// phases 1+2 only: the warp's hits end up contiguous at the start of its segment
template <typename T, int C>
__device__ __forceinline__ void compact_inplace(uint8_t* seg, int lane, uint32_t bits, uint32_t excl, uint32_t wtp) {
  T v[4 * C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    T t[4];
    lds4<T>(seg + (size_t)(kChunkRows * c + 4 * lane) * sizeof(T), t);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[4 * c + j] = t[j];
  }
  __syncwarp();
  T* cs = reinterpret_cast<T*>(seg);
  uint32_t cb = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uint32_t r = cb + ((excl >> (8 * c)) & 0xFFu);
    cb += (wtp >> (8 * c)) & 0xFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((bits >> (4 * c + j)) & 1u) cs[r++] = v[4 * c + j];
  }
}

template <int C>
__device__ __forceinline__ void scatter_tile(const KParams& p, const RowRef& rr, uint32_t bits, uint32_t incl,
                                             uint32_t packed, uint32_t wtp, unsigned long long base) {
  const esc_outputs_t& o = p.outs;
  const uint32_t excl = incl - packed;
  uint32_t wtot = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) wtot += (wtp >> (8 * c)) & 0xFFu;
  if (wtot == 0) return;
  for (int k = 0; k < o.n_proj; ++k) scatter_direct<C>(p, rr, bits, excl, wtp, base, k);
  if (o.out_row_ids != nullptr) {
    uint32_t cb = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      unsigned long long pos = base + cb + ((excl >> (8 * c)) & 0xFFu);
      cb += (wtp >> (8 * c)) & 0xFFu;
      uint32_t m = (bits >> (4 * c)) & 0xFu;
      while (m) {
        const int bit = 4 * c + __ffs(m) - 1;
        m &= m - 1;
        if ((int64_t)pos < o.capacity) o.out_row_ids[pos] = phys_row(rr, logical_row(rr, bit));
        ++pos;
      }
    }
  }
}

__device__ __forceinline__ void finish_cta(const KParams& p, unsigned long long cta_count) {
  if (cta_count) atomicAdd(&p.hdr->count, cta_count);
  __threadfence();
  const unsigned long long prev = atomicAdd(&p.hdr->done, 1ull);
  if (prev == gridDim.x - 1) {
    if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 5] = gtimer();
    __threadfence();
    // the header's words are read from L2 (ld.global.cg) all at once: one round trip, where
    // volatile reads went one by one
    WsHeader* h = p.hdr;
    const unsigned long long count = __ldcg(&h->count);
    unsigned long long fail[ESC_MAX_UDFS];
#pragma unroll
    for (int i = 0; i < ESC_MAX_UDFS; ++i) fail[i] = __ldcg(&h->fail[i]);
    p.result->count = count;
    if (p.sel_on && p.sel.d_count != nullptr) *p.sel.d_count = count;
#pragma unroll
    for (int i = 0; i < ESC_MAX_UDFS; ++i) {
      p.result->udf_fail[i] = fail[i];
      __stcg(&h->fail[i], ~0ull);
    }
    __stcg(&h->count, 0ull);
    __stcg(&h->ticket, 0ull);
    __stcg(&h->done, 0ull);
    if (p.scan_done != nullptr) st_release(p.scan_done, 1ull);  // after the count and the resets
    // no system-scope fence: the host reads the result only after the kernel has completed (a
    // stream/event wait), and kernel completion makes every write visible (the fence cost ~5 us)
    if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 6] = gtimer();
  }
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------
template <int C, bool COMPACT, class Pred>
__global__ void __launch_bounds__(Layout<COMPACT>::kThreads, 1) esc_scan_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = p.stages;
  uint8_t* ring = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* agg_bar = empty_bar + kMaxStages;
  uint64_t* pref_bar = agg_bar + kMaxStages;
  long long* tile_of = reinterpret_cast<long long*>(pref_bar + kMaxStages);
  unsigned long long* s_base = reinterpret_cast<unsigned long long*>(tile_of + kMaxStages);
  unsigned long long* s_red = s_base + kMaxStages;                                  // [kConsumerWarps]
  uint32_t* s_wtot = reinterpret_cast<uint32_t*>(s_red + kConsumerWarps);           // [kMaxStages][NW]
  uint32_t* s_woff = s_wtot + kMaxStages * kConsumerWarps;                          // [kMaxStages][NW]
  uint32_t* s_tsum = s_woff + kMaxStages * kConsumerWarps;                          // [kMaxStages]
  uint32_t* s_writers_done = s_tsum + kMaxStages;                                   // [1]
  unsigned long long* s_cta_count = reinterpret_cast<unsigned long long*>(s_writers_done + 2);  // [1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kW = Layout<COMPACT>::kWriters;

  pdl_trigger();  // every CTA is resident from the start: the compaction chain may queue behind
  if (threadIdx.x < kMaxStages) s_tsum[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    if (p.trace != nullptr) p.trace[blockIdx.x * 8] = gtimer();
    *s_writers_done = 0;
    *s_cta_count = 0;
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps + (COMPACT ? 1 : 0));
      mbar_init(&agg_bar[s], kConsumerWarps);
      mbar_init(&pref_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t policy = evict_first_policy();
      if (!COMPACT && p.prefetch_l2 && p.n_full_tiles > 0) {
        // this CTA's static share of the full tiles' staged bytes, every column (16-byte units)
        const int64_t rows = p.n_full_tiles * (int64_t)p.tile_rows;
        const int64_t r0 = rows * blockIdx.x / gridDim.x, r1 = rows * (blockIdx.x + 1) / gridDim.x;
        for (int i = 0; i < p.ncols; ++i) {
          const KCol& col = p.cols[i];
          if (col.staged) {
            const unsigned long long a = ((unsigned long long)r0 * col.width) & ~15ull;
            const unsigned long long b = ((unsigned long long)r1 * col.width) & ~15ull;
            if (b > a) bulk_prefetch_l2(col.data + a, b - a);
          }
          if (col.nulls_staged == 1) {
            const unsigned long long a = (unsigned long long)r0 & ~15ull, b = (unsigned long long)r1 & ~15ull;
            if (b > a) bulk_prefetch_l2(col.nulls + a, b - a);
          }
        }
      }
      // K2: static round-robin schedule: round r of every CTA covers tiles [r*G, (r+1)*G), so a
      // tile's look-back predecessors are evaluated concurrently in the same round (K2 is a
      // cooperative launch: every CTA is resident, no look-back waits on an unscheduled CTA).
      // K1: after its first tile a CTA takes tickets from the header's counter (one tile ahead,
      // so the atomic's latency hides behind the ring wait): a CTA that DRAM serves late at the
      // start (first tiles arrive 2-120 us apart across CTAs) takes fewer tiles instead of
      // finishing last (600M rows: the static schedule's last CTA ended 37 us after the median)
      // K1 tickets cover ticket_tiles consecutive tiles (small tiles would otherwise wait on the
      // atomic's round trip): batch b = tiles [b*kb, (b+1)*kb); CTA i starts with batch i
      const int64_t kb = COMPACT ? 1 : p.ticket_tiles;
      int64_t tile = COMPACT ? blockIdx.x : blockIdx.x * kb;
      int64_t batch_end = tile + kb;
      int64_t next = COMPACT ? 0 : ((int64_t)atomicAdd(&p.hdr->ticket, 1ull) + gridDim.x) * kb;
      int s = 0;
      uint32_t ph = 0;
      int sentinels = 0;
      for (;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
        mbar_wait(&empty_bar[s], ph ^ 1u);
        if (tile >= p.n_tiles) {
          // K2: one end marker per ring slot (each slot has its own writer warp); consumers stop
          // at the first
          tile_of[s] = -1;
          mbar_arrive(&full_bar[s]);
          if (++sentinels >= (kW > 0 ? S : 1)) break;
          continue;
        }
        tile_of[s] = tile;
        if (tile < p.n_full_tiles) {
          mbar_arrive_expect_tx(&full_bar[s], p.tma_bytes);
          uint8_t* dst = ring + (size_t)s * p.stage_bytes;
          const int64_t row0 = tile * p.tile_rows;
          for (int i = 0; i < p.ncols; ++i) {
            const KCol& col = p.cols[i];
            if (col.staged)
              bulk_g2s(dst + col.smem_off, col.data + (size_t)row0 * col.width, (uint32_t)p.tile_rows * col.width,
                       &full_bar[s], policy);
            if (col.nulls_staged == 2)
              bulk_g2s(dst + col.smem_null_off, reinterpret_cast<const uint8_t*>(col.null_bits) + row0 / 8,
                       (uint32_t)p.tile_rows / 8, &full_bar[s], policy);
            else if (col.nulls_staged)
              bulk_g2s(dst + col.smem_null_off, col.nulls + row0, (uint32_t)p.tile_rows, &full_bar[s], policy);
          }
        } else if (!COMPACT && p.tma_bytes != 0) {
          // the partial tail tile is staged too (a cold per-row read of it was a ~20 us tail on
          // the CTA that drew it): 16-byte multiples by TMA, the last < 16 bytes of each region
          // by this lane (ordered before the arrive, whose release covers them)
          uint8_t* dst = ring + (size_t)s * p.stage_bytes;
          const int64_t row0 = tile * p.tile_rows;
          const uint32_t rows = (uint32_t)(p.nrows - row0);
          uint32_t tx = 0;
          for (int i = 0; i < p.ncols; ++i) {
            const KCol& col = p.cols[i];
            if (col.staged) {
              const uint32_t b = rows * (uint32_t)col.width, a = b & ~15u;
              const uint8_t* src = col.data + (size_t)row0 * col.width;
              for (uint32_t j = a; j < b; ++j) dst[col.smem_off + j] = src[j];
              tx += a;
            }
            if (col.nulls_staged) {
              // packed: the bytes holding the tail's bits (the bitmap is padded past the last row)
              const uint32_t nb = col.nulls_staged == 2 ? (rows + 7) / 8 : rows, a = nb & ~15u;
              const uint8_t* nsrc = col.nulls_staged == 2 ? reinterpret_cast<const uint8_t*>(col.null_bits) + row0 / 8
                                                          : col.nulls + row0;
              for (uint32_t j = a; j < nb; ++j) dst[col.smem_null_off + j] = nsrc[j];
              tx += a;
            }
          }
          mbar_arrive_expect_tx(&full_bar[s], tx);
          for (int i = 0; i < p.ncols; ++i) {
            const KCol& col = p.cols[i];
            const uint32_t a = (rows * (uint32_t)col.width) & ~15u;
            const uint32_t an = (col.nulls_staged == 2 ? (rows + 7) / 8 : rows) & ~15u;
            const uint8_t* nsrc = col.nulls_staged == 2 ? reinterpret_cast<const uint8_t*>(col.null_bits) + row0 / 8
                                                        : col.nulls + row0;
            if (col.staged && a) bulk_g2s(dst + col.smem_off, col.data + (size_t)row0 * col.width, a, &full_bar[s], policy);
            if (col.nulls_staged && an) bulk_g2s(dst + col.smem_null_off, nsrc, an, &full_bar[s], policy);
          }
        } else {
          mbar_arrive(&full_bar[s]);
        }
        if (COMPACT) {
          tile += gridDim.x;
        } else {
          if (++tile >= batch_end) {
            tile = next;
            batch_end = tile + kb;
            if (tile < p.n_tiles) next = ((int64_t)atomicAdd(&p.hdr->ticket, 1ull) + gridDim.x) * kb;
          }
        }
      }
      if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 3] = gtimer();
    }
    return;
  }

  if (COMPACT && warp <= kW) {
    // ===================== writer warps (K2) =====================
    // writer w owns ring slot w and meets its phases in order; per tile: warp offsets, decoupled
    // look-back, then either the coalesced copy-out of the consumers' compacted rows (fast tiles)
    // or handing the global base to the consumers (tail / selection tiles).  One writer per slot
    // keeps up to S look-backs in flight per SM.
    const int w = warp - 1;
    unsigned long long my_count = 0;
    if (w < S) {
    for (int64_t k = w;; k += S) {
      const int s = w;
      const uint32_t ph = (uint32_t)((k / S) & 1);
      mbar_wait(&full_bar[s], ph);
      const int64_t tile = tile_of[s];
      if (tile < 0) break;
      mbar_wait(&agg_bar[s], ph);
      const uint32_t v = lane < kConsumerWarps ? s_wtot[s * kConsumerWarps + lane] : 0u;
      uint32_t sc = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, sc, d);
        if (lane >= d) sc += t;
      }
      const uint32_t woff = sc - v;
      const uint32_t total = __shfl_sync(0xFFFFFFFFu, sc, 31);
      const unsigned long long excl = lookback_warp(p.status, tile, total, p.epoch, lane);
      my_count += total;
      const bool fast = tile < p.n_full_tiles && p.all_fast;
      if (fast && total > 0) {
        const esc_outputs_t& o = p.outs;
        const uint8_t* stage = ring + (size_t)s * p.stage_bytes;
        for (int w2 = 0; w2 < kConsumerWarps; ++w2) {
          const uint32_t n = __shfl_sync(0xFFFFFFFFu, v, w2);
          if (n == 0) continue;
          const unsigned long long base = excl + __shfl_sync(0xFFFFFFFFu, woff, w2);
          const int seg_row = w2 * kChunkRows * C;
          const long long cap = o.capacity;
          for (int kk = 0; kk < o.n_proj; ++kk) {
            const KCol& col = p.cols[o.slot[kk]];
            const uint8_t* src = stage + p.proj_off[kk] + (size_t)seg_row * col.width;
            uint8_t* dst = static_cast<uint8_t*>(o.out_values[kk]);
            switch (col.width) {
              case 1:
                for (uint32_t e = lane; e < n; e += 32) if ((long long)(base + e) < cap) dst[base + e] = src[e];
                break;
              case 2:
                for (uint32_t e = lane; e < n; e += 32)
                  if ((long long)(base + e) < cap) reinterpret_cast<uint16_t*>(dst)[base + e] = reinterpret_cast<const uint16_t*>(src)[e];
                break;
              case 4:
                for (uint32_t e = lane; e < n; e += 32)
                  if ((long long)(base + e) < cap) reinterpret_cast<uint32_t*>(dst)[base + e] = reinterpret_cast<const uint32_t*>(src)[e];
                break;
              default:
                for (uint32_t e = lane; e < n; e += 32)
                  if ((long long)(base + e) < cap)
                    reinterpret_cast<unsigned long long*>(dst)[base + e] = reinterpret_cast<const unsigned long long*>(src)[e];
                break;
            }
            if (o.out_nulls[kk] != nullptr) {
              const uint8_t* nsrc = p.proj_nmode[kk] == 3 ? nullptr : stage + p.proj_noff[kk] + seg_row;
              for (uint32_t e = lane; e < n; e += 32)
                if ((long long)(base + e) < cap) o.out_nulls[kk][base + e] = nsrc ? nsrc[e] : 0;
            }
          }
          if (o.out_row_ids != nullptr) {
            const uint16_t* rs = reinterpret_cast<const uint16_t*>(stage + p.rows_off) + seg_row;
            for (uint32_t e = lane; e < n; e += 32)
              if ((long long)(base + e) < cap) o.out_row_ids[base + e] = tile * p.tile_rows + rs[e];
          }
        }
      }
      if (lane < kConsumerWarps) s_woff[s * kConsumerWarps + lane] = woff;
      __syncwarp();
      if (lane == 0) {
        s_base[s] = excl;
        mbar_arrive(&pref_bar[s]);
        mbar_arrive(&empty_bar[s]);
      }
    }
    }
    if (w < S && lane == 0) {
      atomicAdd(s_cta_count, my_count);
      __threadfence_block();
      if (atomicAdd(s_writers_done, 1u) == (uint32_t)(S - 1)) {
        if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 2] = gtimer();
        finish_cta(p, *reinterpret_cast<volatile unsigned long long*>(s_cta_count));
        if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 4] = gtimer();
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int cw = warp - Layout<COMPACT>::kFirstConsumer;
  const int local0 = cw * (kChunkRows * C) + 4 * lane;
  unsigned long long my_count = 0;
  int s = 0;
  uint32_t ph = 0;
  for (;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
    mbar_wait(&full_bar[s], ph);
    if (p.trace != nullptr && cw == 0 && lane == 0 && my_count == 0 && s == 0 && ph == 0)
      p.trace[blockIdx.x * 8 + 1] = gtimer();
    const int64_t tile = tile_of[s];
    if (tile < 0) break;
    RowRef rr;
    const bool full = tile < p.n_full_tiles;
    rr.stage = (full || (!COMPACT && p.tma_bytes != 0)) ? ring + (size_t)s * p.stage_bytes : nullptr;
    rr.local0 = local0;
    rr.grow0 = tile * p.tile_rows + local0;
    rr.nrows = p.nrows;
    rr.ids = p.row_ids;
    uint32_t bits;
    if (rr.stage != nullptr && p.all_staged) {
      bits = Pred::template eval<C>(p, rr, full ? ((4 * C == 32) ? 0xFFFFFFFFu : ((1u << (4 * C)) - 1u))
                                                : valid_bits(rr.grow0, p.nrows, C));
    } else {
      bits = eval_direct<C>(p, rr, valid_bits(rr.grow0, p.nrows, C));
    }
    if constexpr (!COMPACT) {
      const uint32_t pc = __popc(bits);
      my_count += pc;
      if (p.sel_on) {
        const int64_t seg = tile * kConsumerWarps + cw;
        const uint32_t wtot = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(bits));
        const bool capt = C <= 4 && p.sel.n_cap > 0 && wtot > 0 && wtot <= (uint32_t)(4 * C);  // 8-bit fields: C <= 4
        if (!(p.bitmap_lean && (capt || wtot == 0))) {
          // 8 lanes x 4 rows of a chunk = one 32-row bitmap word (row-linear order); a lean
          // step skips the words of captured and empty segments (their 75 MB on config 4 cost
          // ~50 us of the scan: writes interleaved with the read stream)
          const int64_t word0 = tile * (p.tile_rows / 32) + cw * (4 * C) + (lane >> 3);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            uint32_t v = ((bits >> (4 * c)) & 0xFu) << (4 * (lane & 7));
            v |= __shfl_xor_sync(0xFFFFFFFFu, v, 1);
            v |= __shfl_xor_sync(0xFFFFFFFFu, v, 2);
            v |= __shfl_xor_sync(0xFFFFFFFFu, v, 4);
            if ((lane & 7) == 0) p.sel.bitmap[word0 + 4 * c] = v;
          }
        }
        uint32_t flag = 0;
        if (capt) {
          // very sparse segment: capture the hits' projected values now, while they sit in smem
          // (warp-local ranks: per-chunk lane counts in 8-bit fields, one scan ranks every chunk)
          flag = ESC_SEG_CAPTURED;
          uint32_t packed = 0;
#pragma unroll
          for (int c = 0; c < C; ++c) packed |= (uint32_t)__popc((bits >> (4 * c)) & 0xFu) << (8 * c);
          uint32_t incl = packed;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
            if (lane >= d) incl += t;
          }
          const uint32_t wtp = __shfl_sync(0xFFFFFFFFu, incl, 31);
          const uint32_t excl = incl - packed;
          if (bits) Pred::template capture<C>(p, rr, bits, excl, wtp, seg);
        }
        if (lane == 0) p.sel.seg_counts[seg] = wtot | flag;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    } else {
      // per-chunk lane counts in 8-bit fields: one warp scan ranks every chunk
      uint32_t packed = 0;
#pragma unroll
      for (int c = 0; c < C; ++c) packed |= (uint32_t)__popc((bits >> (4 * c)) & 0xFu) << (8 * c);
      uint32_t incl = packed;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t wtp = __shfl_sync(0xFFFFFFFFu, incl, 31);
      const uint32_t excl = incl - packed;
      uint32_t wtot = 0;
#pragma unroll
      for (int c = 0; c < C; ++c) wtot += (wtp >> (8 * c)) & 0xFFu;
      const bool fast = rr.stage != nullptr && p.all_fast;
      if (fast && wtot > 0) {
        // compact this warp's hits inside its own smem segments; a writer warp copies them out
        const int seg_row = local0 - 4 * lane;
        const esc_outputs_t& o = p.outs;
        uint8_t* stage = const_cast<uint8_t*>(rr.stage);
        for (int kk = 0; kk < o.n_proj; ++kk) {
          const KCol& col = p.cols[o.slot[kk]];
          uint8_t* seg = stage + p.proj_off[kk] + (size_t)seg_row * col.width;
          if (p.proj_mode[kk] == 0) {
            switch (col.width) {
              case 1: compact_inplace<uint8_t, C>(seg, lane, bits, excl, wtp); break;
              case 2: compact_inplace<uint16_t, C>(seg, lane, bits, excl, wtp); break;
              case 4: compact_inplace<uint32_t, C>(seg, lane, bits, excl, wtp); break;
              default: compact_inplace<unsigned long long, C>(seg, lane, bits, excl, wtp); break;
            }
          } else if (p.proj_mode[kk] == 1) {
            switch (col.width) {
              case 1: gather_compact<uint8_t, C>(col.data, rr.grow0, seg, bits, excl, wtp); break;
              case 2: gather_compact<uint16_t, C>(col.data, rr.grow0, seg, bits, excl, wtp); break;
              case 4: gather_compact<uint32_t, C>(col.data, rr.grow0, seg, bits, excl, wtp); break;
              default: gather_compact<unsigned long long, C>(col.data, rr.grow0, seg, bits, excl, wtp); break;
            }
          }
          if (p.proj_nmode[kk] == 0)
            compact_inplace<uint8_t, C>(stage + p.proj_noff[kk] + seg_row, lane, bits, excl, wtp);
          else if (p.proj_nmode[kk] == 1)
            gather_compact<uint8_t, C>(col.nulls, rr.grow0, stage + p.proj_noff[kk] + seg_row, bits, excl, wtp);
        }
        if (o.out_row_ids != nullptr) {
          uint16_t* rs = reinterpret_cast<uint16_t*>(stage + p.rows_off) + seg_row;
          uint32_t cb = 0;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            uint32_t r = cb + ((excl >> (8 * c)) & 0xFFu);
            cb += (wtp >> (8 * c)) & 0xFFu;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if ((bits >> (4 * c + j)) & 1u) rs[r++] = (uint16_t)(local0 + kChunkRows * c + j);
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        s_wtot[s * kConsumerWarps + cw] = wtot;
        // the last warp to finish the tile publishes its aggregate right away, so successors'
        // look-backs never wait for this CTA's writer warp to reach the tile
        const uint32_t now = atomicAdd(&s_tsum[s], (1u << 20) + wtot) + (1u << 20) + wtot;
        if ((now >> 20) == kConsumerWarps) {
          s_tsum[s] = 0;
          const unsigned long long tag = (unsigned long long)p.epoch << 48;
          const unsigned long long flag = tile == 0 ? kFlagPrefix : kFlagAggregate;
          st_relaxed(&p.status[tile], tag | (flag << kStatusValueBits) | (now & 0xFFFFFu));
        }
        mbar_arrive(&agg_bar[s]);
      }
      if (!fast) {
        // tail / selection / non-staged projections: scatter directly once the base is known
        mbar_wait(&pref_bar[s], ph);
        const unsigned long long base = s_base[s] + s_woff[s * kConsumerWarps + cw];
        if (wtot > 0) scatter_tile<C>(p, rr, bits, incl, packed, wtp, base);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[s]);
    }
  }

  if constexpr (!COMPACT) {
    // ---- CTA reduction, global accumulation, last-CTA finalisation ----
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) my_count += __shfl_down_sync(0xFFFFFFFFu, my_count, d);
    if (lane == 0) s_red[cw] = my_count;
    consumer_bar();
    if (cw == 0 && lane == 0) {
      unsigned long long tot = 0;
      for (int w = 0; w < kConsumerWarps; ++w) tot += s_red[w];
      if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 2] = gtimer();
      finish_cta(p, tot);
      if (p.trace != nullptr) p.trace[blockIdx.x * 8 + 4] = gtimer();
    }
  }
}

// ------------------------------------------------------------------------------------------
// selection -> order-preserving compaction (no cross-CTA dependency: offsets come from a scan of
// the per-tile counts the scan kernel recorded)
// ------------------------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanSeg = 4 * kScanThreads;  // segments per scan block

// Streamed compaction of dense tiles (sel_stream_kernel): a "stream tile" is `segs_per_tile`
// consecutive warp segments of the selection.  Dense tiles (>= dense_min hits) are streamed whole
// through shared memory by TMA; every other segment is compacted by sel_compact_kernel.  Both
// kernels and the scan that lists the dense tiles apply the same rule to the same counts.
struct DenseRule {
  uint32_t dense_min;      // hits that make a stream tile dense (0xFFFFFFFF: streaming off)
  int32_t segs_per_tile;   // 2, 4 or 8
  int64_t n_tiles;         // stream tiles over the selection's rows (the last may be partial)
  uint32_t* dense_list;    // out: dense tile ids (unordered; output positions come from offsets)
  uint32_t* n_dense;       // out: number of dense tiles
  const unsigned long long* skip_count;  // ESC_OUT_SKIP_OVER_CAPACITY: the selection's count ...
  long long skip_capacity;               // ... and the capacity it must not exceed
  uint32_t lean;           // K1 wrote no bitmap words for captured / empty segments: a stream tile
                           // holding one is never dense (its segments go to sel_compact_kernel)
};

// a segment's share in its stream tile's density (dense_rule_ok): the hit count, or with a lean
// bitmap a marker for a captured or empty segment that keeps its tile out of the dense list
constexpr uint32_t kLeanMarker = 1u << 24;  // > any tile's hits (<= 8 segments x 1024 rows)
__device__ __forceinline__ uint32_t dense_share(const DenseRule& r, uint32_t raw) {
  const uint32_t cnt = raw & ~ESC_SEG_CAPTURED;
  return (r.lean && ((raw & ESC_SEG_CAPTURED) || cnt == 0)) ? kLeanMarker : cnt;
}
__device__ __forceinline__ bool dense_rule_ok(const DenseRule& r, uint32_t tile_share) {
  return tile_share >= r.dense_min && tile_share < kLeanMarker;
}

__device__ __forceinline__ bool skip_materialize(const DenseRule& r) {
  return r.skip_count != nullptr && (long long)*r.skip_count > r.skip_capacity;
}

// block-wide exclusive scan of one value per thread; returns the exclusive prefix, *total set
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* sh,
                                                             unsigned long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    unsigned long long x = lane < nw ? sh[lane] : 0ull, y = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, y, d);
      if (lane >= d) y += t;
    }
    if (lane < nw) sh[lane] = y - x;
    if (lane == 31) sh[32] = y;
  }
  __syncthreads();
  const unsigned long long r = sh[warp] + incl - v;
  *total = sh[32];
  __syncthreads();
  return r;
}

// partial sums of kScanSeg-segment blocks (block 0 also resets the dense-tile counter)
__global__ void __launch_bounds__(kScanThreads) tile_scan_partials(const uint32_t* __restrict__ counts, int64_t n,
                                                                   unsigned long long* __restrict__ partial,
                                                                   uint32_t* __restrict__ n_dense,
                                                                   const unsigned long long* skip_count,
                                                                   long long skip_capacity) {
  pdl_wait();
  pdl_trigger();
  const bool skip = skip_count != nullptr && (long long)*skip_count > skip_capacity;
  __shared__ unsigned long long sh[33];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_dense = 0;
  if (skip) return;
  const int64_t base = (int64_t)blockIdx.x * kScanSeg + 4 * threadIdx.x;
  unsigned long long v = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) v += (base + j < n) ? (counts[base + j] & ~ESC_SEG_CAPTURED) : 0u;
  unsigned long long total;
  block_excl_scan(v, sh, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

// exclusive offsets of every segment (carry from the earlier blocks' partial sums), and the list
// of dense stream tiles
__global__ void __launch_bounds__(kScanThreads) tile_scan_apply(const uint32_t* __restrict__ counts, int64_t n,
                                                                const unsigned long long* __restrict__ partial,
                                                                unsigned long long* __restrict__ offsets,
                                                                const DenseRule rule) {
  __shared__ unsigned long long sh[33];
  __shared__ unsigned long long carry;
  pdl_wait();
  pdl_trigger();
  if (skip_materialize(rule)) return;
  if (threadIdx.x < 32) {  // one warp sums the earlier blocks' partials (independent loads in flight)
    unsigned long long c = 0, c1 = 0, c2 = 0, c3 = 0;  // four independent loads in flight per lane
    unsigned b = threadIdx.x;
    for (; b + 96 < blockIdx.x; b += 128) {
      c += __ldcg(partial + b);
      c1 += __ldcg(partial + b + 32);
      c2 += __ldcg(partial + b + 64);
      c3 += __ldcg(partial + b + 96);
    }
    for (; b < blockIdx.x; b += 32) c += __ldcg(partial + b);
    c += c1 + c2 + c3;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, d);
    if (threadIdx.x == 0) carry = c;
  }
  const int64_t base = (int64_t)blockIdx.x * kScanSeg + 4 * threadIdx.x;
  uint32_t x[4];
  unsigned long long v = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    x[j] = (base + j < n) ? (counts[base + j] & ~ESC_SEG_CAPTURED) : 0u;
    v += x[j];
  }
  unsigned long long total;
  unsigned long long e = block_excl_scan(v, sh, &total);  // its barriers also publish `carry`
  e += carry;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (base + j < n) offsets[base + j] = e;
    e += x[j];
  }
  if (rule.dense_min == 0xFFFFFFFFu) return;
  // dense stream tiles among this thread's 4 segments (8-segment tiles: thread pairs)
  uint32_t sh4[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sh4[j] = (base + j < n) ? dense_share(rule, counts[base + j]) : 0u;
  const uint32_t vs = sh4[0] + sh4[1] + sh4[2] + sh4[3];
  const uint32_t pair = vs + __shfl_xor_sync(0xFFFFFFFFu, vs, 1);
  bool d0 = false, d1 = false;
  int64_t t0 = -1, t1 = -1;
  if (rule.segs_per_tile == 8) {
    if ((threadIdx.x & 1) == 0) { t0 = base / 8; d0 = dense_rule_ok(rule, pair); }
  } else if (rule.segs_per_tile == 4) {
    t0 = base / 4; d0 = dense_rule_ok(rule, vs);
  } else {
    t0 = base / 2; d0 = dense_rule_ok(rule, sh4[0] + sh4[1]);
    t1 = t0 + 1;   d1 = dense_rule_ok(rule, sh4[2] + sh4[3]);
  }
  d0 = d0 && t0 >= 0 && t0 < rule.n_tiles;
  d1 = d1 && t1 >= 0 && t1 < rule.n_tiles;
  // warp-aggregated append
  const int lane = threadIdx.x & 31;
  const uint32_t m0 = __ballot_sync(0xFFFFFFFFu, d0), m1 = __ballot_sync(0xFFFFFFFFu, d1);
  const uint32_t tot = __popc(m0) + __popc(m1);
  if (tot == 0) return;
  uint32_t slot0 = 0;
  if (lane == 0) slot0 = atomicAdd(rule.n_dense, tot);
  slot0 = __shfl_sync(0xFFFFFFFFu, slot0, 0);
  const uint32_t lt = (1u << lane) - 1u;
  if (d0) rule.dense_list[slot0 + __popc(m0 & lt)] = (uint32_t)t0;
  if (d1) rule.dense_list[slot0 + __popc(m0) + __popc(m1 & lt)] = (uint32_t)t1;
}

struct SelParams {
  const uint32_t* bitmap;
  const uint32_t* seg_counts;            // | ESC_SEG_CAPTURED
  const unsigned long long* seg_offsets;
  const int64_t* row_ids;  // logical -> physical rows (selection chaining) or nullptr
  int64_t nrows;
  int64_t n_segs;
  int32_t seg_rows;
  int32_t cap_per_seg;
  int32_t cap_stride;                    // slot-major captures: entry = slot * cap_stride + segment
  int32_t n_proj;
  int32_t need_bitmap_captured;  // captured segments still need the bitmap (row ids / uncaptured columns)
  int32_t sparse_in_a;           // phase A also writes sparse segments (grids that fill the GPU)
  int32_t a_split;               // warps per 32-segment group in phase A (power of two; 1 if sparse_in_a)
  KCol cols[ESC_MAX_PROJ];  // projected columns (data, nulls, width)
  int32_t cap_index[ESC_MAX_PROJ];      // capture holding projection k, -1 = gather it
  const void* cap_values[ESC_MAX_PROJ];
  const uint8_t* cap_nulls[ESC_MAX_PROJ];
  esc_outputs_t outs;
  DenseRule rule;  // segments of dense stream tiles belong to sel_stream_kernel
};

constexpr int kSelWarps = 8;

__device__ __forceinline__ unsigned long long ld_bits(const KCol& col, int64_t row) {
  switch (col.width) {
    case 1: return __ldg(col.data + row);
    case 2: return __ldg(reinterpret_cast<const uint16_t*>(col.data) + row);
    case 4: return __ldg(reinterpret_cast<const uint32_t*>(col.data) + row);
    default: return __ldg(reinterpret_cast<const unsigned long long*>(col.data) + row);
  }
}
__device__ __forceinline__ void st_bits(int width, void* out, unsigned long long pos, unsigned long long v) {
  switch (width) {
    case 1: static_cast<uint8_t*>(out)[pos] = (uint8_t)v; break;
    case 2: static_cast<uint16_t*>(out)[pos] = (uint16_t)v; break;
    case 4: static_cast<uint32_t*>(out)[pos] = (uint32_t)v; break;
    default: static_cast<unsigned long long*>(out)[pos] = v; break;
  }
}
__device__ __forceinline__ unsigned long long ld_w(int width, const void* src, uint32_t e) {
  switch (width) {
    case 1: return static_cast<const uint8_t*>(src)[e];
    case 2: return static_cast<const uint16_t*>(src)[e];
    case 4: return static_cast<const uint32_t*>(src)[e];
    default: return static_cast<const unsigned long long*>(src)[e];
  }
}

// 4 rows of one column: loads first (in flight together), then the stores (ld.global.cg, see
// ldcg_rows).  The dense segments' path: one row per lane of each word, column by column.
template <typename T>
__device__ __forceinline__ void gather4(const uint8_t* data, void* out, const bool (&hit)[4], const int64_t (&prow)[4],
                                        const unsigned long long (&pos)[4]) {
  const T* src = reinterpret_cast<const T*>(data);
  T v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = hit[j] ? __ldcg(src + prow[j]) : (T)0;
#pragma unroll
  for (int j = 0; j < 4; ++j) if (hit[j]) static_cast<T*>(out)[pos[j]] = v[j];
}

// H rows of one column loaded into v (hit rows only; the width switch is per column).  The loads
// bypass L1 (ld.global.cg): scattered rows would otherwise each pull a whole 128-byte line
// through L1 into L2/DRAM traffic (measured: 4 sectors per request at 1% selectivity, ~5x the
// 32-byte sectors the hits occupy)
template <int H>
__device__ __forceinline__ void ldcg_rows(int width, const uint8_t* data, const bool (&hit)[H], const int64_t (&prow)[H],
                                          unsigned long long (&v)[H]) {
  switch (width) {
    case 1:
#pragma unroll
      for (int j = 0; j < H; ++j) v[j] = hit[j] ? __ldcg(data + prow[j]) : 0u;
      break;
    case 2:
#pragma unroll
      for (int j = 0; j < H; ++j) v[j] = hit[j] ? __ldcg(reinterpret_cast<const uint16_t*>(data) + prow[j]) : 0u;
      break;
    case 4:
#pragma unroll
      for (int j = 0; j < H; ++j) v[j] = hit[j] ? __ldcg(reinterpret_cast<const uint32_t*>(data) + prow[j]) : 0u;
      break;
    default:
#pragma unroll
      for (int j = 0; j < H; ++j) v[j] = hit[j] ? __ldcg(reinterpret_cast<const unsigned long long*>(data) + prow[j]) : 0ull;
      break;
  }
}
template <int H>
__device__ __forceinline__ void st_rows(int width, void* out, const bool (&hit)[H], const unsigned long long (&pos)[H],
                                        const unsigned long long (&v)[H]) {
  switch (width) {
    case 1:
#pragma unroll
      for (int j = 0; j < H; ++j) if (hit[j]) static_cast<uint8_t*>(out)[pos[j]] = (uint8_t)v[j];
      break;
    case 2:
#pragma unroll
      for (int j = 0; j < H; ++j) if (hit[j]) static_cast<uint16_t*>(out)[pos[j]] = (uint16_t)v[j];
      break;
    case 4:
#pragma unroll
      for (int j = 0; j < H; ++j) if (hit[j]) static_cast<uint32_t*>(out)[pos[j]] = (uint32_t)v[j];
      break;
    default:
#pragma unroll
      for (int j = 0; j < H; ++j) if (hit[j]) static_cast<unsigned long long*>(out)[pos[j]] = v[j];
      break;
  }
}

// H rows of every projected column (captured ones skipped when `skip_captured`): the value loads
// of up to 4 columns are all in flight before any of their stores, so a row's columns cost one
// DRAM round trip, not one per column.  NULL bytes (no BASELINE shape has them) follow per column.
template <int H>
__device__ __forceinline__ void gather_rows(const SelParams& p, const bool (&hit)[H], const int64_t (&prow)[H],
                                            const unsigned long long (&pos)[H], bool skip_captured) {
#pragma unroll 1
  for (int k0 = 0; k0 < p.n_proj; k0 += 4) {
    unsigned long long v[4][H];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k0 + kk;
      if (k < p.n_proj && !(skip_captured && p.cap_index[k] >= 0)) ldcg_rows<H>(p.cols[k].width, p.cols[k].data, hit, prow, v[kk]);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int k = k0 + kk;
      if (k < p.n_proj && !(skip_captured && p.cap_index[k] >= 0)) st_rows<H>(p.cols[k].width, p.outs.out_values[k], hit, pos, v[kk]);
    }
  }
#pragma unroll 1
  for (int k = 0; k < p.n_proj; ++k) {
    if (p.outs.out_nulls[k] == nullptr || (skip_captured && p.cap_index[k] >= 0)) continue;
    const uint8_t* nulls = p.cols[k].nulls;
    uint8_t nb[H];
#pragma unroll
    for (int j = 0; j < H; ++j) nb[j] = (hit[j] && nulls) ? __ldcg(nulls + prow[j]) : (uint8_t)0;
#pragma unroll
    for (int j = 0; j < H; ++j) if (hit[j]) p.outs.out_nulls[k][pos[j]] = nb[j];
  }
}

// Two grid-stride phases over the selection (segments of dense stream tiles are skipped:
// sel_stream_kernel writes them):
//  A. one warp per 32 consecutive segments (seg_rows = 128*C rows = 4*C <= 32 bitmap words):
//     captured segments - the group's captured hits (<= 4*C per segment) spread over the lanes;
//     dense segments (> one hit per 32 rows) - the whole warp, one row per lane of each word;
//  B. sparse segments, one LANE per 128-row chunk (4 bitmap words): a 16-byte bitmap load, a
//     width-CPS segmented scan for the chunk's output base, then the chunk's hits four at a time
//     (each column's 4 loads in flight before its stores).  Spreading chunks, not segments, over
//     the warps keeps small selections from running on a handful of SMs.  When the segment
//     groups alone fill the GPU (sparse_in_a), phase A writes its own sparse segments the same
//     way, chunk by chunk, and phase B is skipped: no second pass over the segment counts.
// sel_compact_kernel<true> (sparse selections, sparse_in_a): phase A's sparse segments go
// through per-warp hit lists instead (candidate-segment rounds, the hits listed in shared
// memory and gathered 32+ at a time by the whole warp, every column's loads in flight).
// The hits of one 128-row chunk (4 bitmap words `w4` of segment `seg`, chunk `sub`), written
// from output position `pos` on, four at a time.
__device__ __forceinline__ void sparse_chunk(const SelParams& p, int64_t seg, int sub, uint4 w4,
                                             unsigned long long pos, bool scap) {
  const int W = p.seg_rows / 32;
  const long long cap = p.outs.capacity;
  unsigned long long lo = ((unsigned long long)w4.y << 32) | w4.x;
  unsigned long long hi = ((unsigned long long)w4.w << 32) | w4.z;
  const int64_t row_base = (seg * W + sub * 4) * 32;
  while (lo | hi) {
    bool hit[4];
    unsigned long long ps[4];
    int64_t prow[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int bit = -1;
      if (lo) { bit = __ffsll((long long)lo) - 1; lo &= lo - 1; }
      else if (hi) { bit = 64 + __ffsll((long long)hi) - 1; hi &= hi - 1; }
      hit[j] = bit >= 0 && (long long)pos < cap;
      ps[j] = pos;
      pos += bit >= 0 ? 1 : 0;
      const int64_t row = row_base + (bit < 0 ? 0 : bit);
      prow[j] = (hit[j] && p.row_ids) ? __ldg(p.row_ids + row) : row;
    }
    for (int k = 0; k < p.n_proj; ++k) {
      if (scap && p.cap_index[k] >= 0) continue;
      const KCol& col = p.cols[k];
      switch (col.width) {
        case 1: gather4<uint8_t>(col.data, p.outs.out_values[k], hit, prow, ps); break;
        case 2: gather4<uint16_t>(col.data, p.outs.out_values[k], hit, prow, ps); break;
        case 4: gather4<uint32_t>(col.data, p.outs.out_values[k], hit, prow, ps); break;
        default: gather4<unsigned long long>(col.data, p.outs.out_values[k], hit, prow, ps); break;
      }
      if (p.outs.out_nulls[k] != nullptr) {
        uint8_t nb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) nb[j] = (hit[j] && col.nulls) ? __ldg(col.nulls + prow[j]) : (uint8_t)0;
#pragma unroll
        for (int j = 0; j < 4; ++j) if (hit[j]) p.outs.out_nulls[k][ps[j]] = nb[j];
      }
    }
    if (p.outs.out_row_ids != nullptr) {
#pragma unroll
      for (int j = 0; j < 4; ++j) if (hit[j]) p.outs.out_row_ids[ps[j]] = prow[j];
    }
  }
}

__device__ __forceinline__ bool in_dense_tile(const SelParams& p, int64_t seg) {
  if (p.rule.dense_min == 0xFFFFFFFFu) return false;
  const int64_t t = seg >> (__ffs(p.rule.segs_per_tile) - 1);  // segs_per_tile: a power of two
  if (t >= p.rule.n_tiles) return false;
  uint32_t ts = 0;
  for (int j = 0; j < p.rule.segs_per_tile; ++j) {
    const int64_t q = t * p.rule.segs_per_tile + j;
    if (q < p.n_segs) ts += dense_share(p.rule, __ldg(p.seg_counts + q));
  }
  return dense_rule_ok(p.rule, ts);
}

// A warp's list of sparse hits (phase A): entries (row | kHitSkipCaptured, output position), both
// 32-bit (the host uses lists only for tables of < 2^31 rows: 1.25 KB per warp), in row order.  A round adds at most 32 / CPS segments x 4*CPS bits = 128 entries, and the list is
// flushed whenever it holds 32 or more, so 160 entries suffice.
constexpr int kHitList = 160;
constexpr uint32_t kHitSkipCaptured = 1u << 31;  // the entry's captured columns are written elsewhere

// gathers the list's first entries with the whole warp, two per lane per pass (every column's
// loads of both in flight before the stores): all of them when `all`, else the largest multiple
// of 32; the rest move to the front.  Returns the entries left.
__device__ __noinline__ int flush_hits(const SelParams& p, uint32_t* hl_row, uint32_t* hl_pos, int n, bool all) {
  const int lane = threadIdx.x & 31;
  const long long cap = p.outs.capacity;
  __syncwarp();
  const int nf = all ? n : (n & ~31);
  for (int e0 = 0; e0 < nf; e0 += 64) {
    bool hit[2];
    int64_t prow[2];
    unsigned long long pos[2];
    bool scap = false;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int e = e0 + 32 * j + lane;
      const uint32_t re = e < nf ? hl_row[e] : 0u;
      pos[j] = e < nf ? hl_pos[e] : 0u;
      hit[j] = e < nf && (long long)pos[j] < cap;
      scap = scap || (hit[j] && (re & kHitSkipCaptured));
      const int64_t row = re & ~kHitSkipCaptured;
      prow[j] = (hit[j] && p.row_ids) ? __ldg(p.row_ids + row) : row;
    }
    if (scap) {  // a captured segment's entry: write its uncaptured columns one entry at a time
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = e0 + 32 * j + lane;
        const bool sj = hit[j] && (hl_row[e] & kHitSkipCaptured);
        bool h1[1] = {hit[j]};
        int64_t r1[1] = {prow[j]};
        unsigned long long p1[1] = {pos[j]};
        gather_rows<1>(p, h1, r1, p1, sj);
        hit[j] = false;
        if (p.outs.out_row_ids != nullptr && h1[0]) p.outs.out_row_ids[p1[0]] = r1[0];
      }
    }
    gather_rows<2>(p, hit, prow, pos, false);
    if (p.outs.out_row_ids != nullptr) {
#pragma unroll
      for (int j = 0; j < 2; ++j) if (hit[j]) p.outs.out_row_ids[pos[j]] = prow[j];
    }
  }
  const int rem = n - nf;
  uint32_t r = 0, q = 0;
  if (lane < rem) { r = hl_row[nf + lane]; q = hl_pos[nf + lane]; }
  __syncwarp();
  if (lane < rem) { hl_row[lane] = r; hl_pos[lane] = q; }
  __syncwarp();
  return rem;
}

template <bool kList>
__global__ void __launch_bounds__(kSelWarps * 32, kList ? 3 : 4) sel_compact_kernel(const __grid_constant__ SelParams p) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int W = p.seg_rows / 32;  // words per segment (<= 32)
  const long long cap = p.outs.capacity;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t sparse_max = (uint32_t)W;
  if (skip_materialize(p.rule)) return;
  __shared__ uint8_t cand_lanes[kSelWarps][32];
  __shared__ uint32_t hit_rows[kSelWarps][kList ? kHitList : 1];
  __shared__ uint32_t hit_pos[kSelWarps][kList ? kHitList : 1];
  uint32_t* hl_row = hit_rows[threadIdx.x >> 5];
  uint32_t* hl_pos = hit_pos[threadIdx.x >> 5];
  int hl_n = 0;  // warp-uniform: entries in the warp's hit list
  // ---------------- A: captured and dense segments ----------------
  // a_split (R, a power of two) warps share a group: warp r of it takes captured entries
  // r*32 + lane (mod 32R) and every R-th dense segment, so small selections use the whole grid
  const int R = p.a_split;
  const int r_log = __ffs(R) - 1;
  const int64_t n_units = ((p.n_segs + 31) >> 5) << r_log;
  // a group's segment counts and offsets are loaded together, one group ahead (the offsets
  // unconditionally: 256 contiguous bytes cost less than a second dependent round trip)
  uint32_t raw_n = 0;
  unsigned long long off_n = 0;
  {
    const int64_t sg = ((gwarp >> r_log) * 32) + lane;
    if (gwarp < n_units && sg < p.n_segs) {
      raw_n = __ldcg(p.seg_counts + sg);
      off_n = __ldcg(p.seg_offsets + sg);
    }
  }
  for (int64_t u = gwarp; u < n_units; u += nwarps) {
    const int64_t seg0 = (u >> r_log) * 32;
    const int r = (int)(u & (R - 1));
    const int64_t myseg = seg0 + lane;
    const uint32_t raw = raw_n;
    const unsigned long long off_l = off_n;
    {
      const int64_t un = u + nwarps, sg = ((un >> r_log) * 32) + lane;
      raw_n = 0;
      off_n = 0;
      if (un < n_units && sg < p.n_segs) {
        raw_n = __ldcg(p.seg_counts + sg);
        off_n = __ldcg(p.seg_offsets + sg);
      }
    }
    uint32_t cnt = raw & ~ESC_SEG_CAPTURED;
    if (p.rule.dense_min != 0xFFFFFFFFu) {
      // my stream tile's density (segments_per_tile consecutive lanes; lanes past the end add 0)
      uint32_t ts = myseg < p.n_segs ? dense_share(p.rule, raw) : 0u;
      for (int d = 1; d < p.rule.segs_per_tile; d <<= 1) ts += __shfl_xor_sync(0xFFFFFFFFu, ts, d);
      if (dense_rule_ok(p.rule, ts) && (myseg >> (__ffs(p.rule.segs_per_tile) - 1)) < p.rule.n_tiles) cnt = 0;
    }
    const bool captured = (raw & ESC_SEG_CAPTURED) != 0;
    const bool bitmap_work = cnt > 0 && (!captured || p.need_bitmap_captured);
    const bool dense_work = bitmap_work && cnt > sparse_max;
    const unsigned long long myoff = off_l;
    // captured hits: the group's entries are spread over the lanes (lane e: entries e, e+32, ...
    // of the group's concatenated captured lists), four columns' loads in flight per entry
    {
      const uint32_t ccnt = captured ? cnt : 0u;
      uint32_t incl = ccnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
      // two entries per lane per pass (e, e + 32R): both entries' loads are in flight before
      // their stores, so a group of up to 64 captured hits costs one round trip
      for (uint32_t e0 = (uint32_t)r * 32; e0 < total; e0 += 64u * R) {
        bool ok[2];
        unsigned long long pos[2];
        size_t slot[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t e = e0 + (uint32_t)h * 32u * R + lane;
          // owning lane: the first whose inclusive count exceeds e (binary search over the lanes)
          int sl = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, sl + step - 1);
            if (v <= e) sl += step;
          }
          const uint32_t s_incl = __shfl_sync(0xFFFFFFFFu, incl, sl);
          const uint32_t s_cnt = __shfl_sync(0xFFFFFFFFu, ccnt, sl);
          const unsigned long long s_off = __shfl_sync(0xFFFFFFFFu, myoff, sl);
          const uint32_t idx = e - (s_incl - s_cnt);
          pos[h] = s_off + idx;
          ok[h] = e < total && (long long)pos[h] < cap;
          slot[h] = (size_t)idx * p.cap_stride + (size_t)(seg0 + sl);
        }
        if (!ok[0] && !ok[1]) continue;
        for (int k0 = 0; k0 < p.n_proj; k0 += 4) {
          unsigned long long v[2][4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = k0 + j;
            const int ci = k < p.n_proj ? p.cap_index[k] : -1;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              v[h][j] = (ci >= 0 && ok[h])
                            ? ld_w(p.cols[k].width, static_cast<const uint8_t*>(p.cap_values[ci]) + slot[h] * p.cols[k].width, 0)
                            : 0ull;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int k = k0 + j;
            if (k < p.n_proj && p.cap_index[k] >= 0) {
              const int ci = p.cap_index[k];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (!ok[h]) continue;
                st_bits(p.cols[k].width, p.outs.out_values[k], pos[h], v[h][j]);
                if (p.outs.out_nulls[k] != nullptr)
                  p.outs.out_nulls[k][pos[h]] = p.cap_nulls[ci] != nullptr ? p.cap_nulls[ci][slot[h]] : (uint8_t)0;
              }
            }
          }
        }
      }
    }
    const bool sparse_work = bitmap_work && cnt <= sparse_max;
    if constexpr (!kList) {
      if (p.sparse_in_a && __any_sync(0xFFFFFFFFu, sparse_work)) {
        // large selections: this warp's own sparse segments, C lanes per segment, one 128-row chunk
        // each (32 chunks in flight per round); small ones leave them to phase B's wider spread
        const unsigned long long soff_l = off_l;
        const int CPS = W / 4;
        const int cps_log = __ffs(CPS) - 1;
        // the next round's bitmap chunk is loaded one round ahead (its latency hides behind this
        // round's ranking and gathers)
        auto load_round = [&](int b) {
          const int sl = (b * 32 + lane) >> cps_log;
          const bool work = __shfl_sync(0xFFFFFFFFu, sparse_work ? 1 : 0, sl) != 0;
          return work ? __ldg(reinterpret_cast<const uint4*>(p.bitmap + (seg0 + sl) * W + ((b * 32 + lane) & (CPS - 1)) * 4))
                      : make_uint4(0u, 0u, 0u, 0u);
        };
        uint4 w4n = load_round(0);
        for (int b = 0; b < CPS; ++b) {
          const int c = b * 32 + lane;
          const int sl = c >> cps_log;  // lane owning the chunk's segment
          const int sub = c & (CPS - 1);
          const bool work = __shfl_sync(0xFFFFFFFFu, sparse_work ? 1 : 0, sl) != 0;
          const unsigned long long soff = __shfl_sync(0xFFFFFFFFu, soff_l, sl);
          const bool scap = __shfl_sync(0xFFFFFFFFu, captured ? 1 : 0, sl) != 0;
          const int64_t seg = seg0 + sl;
          const uint4 w4 = w4n;
          if (b + 1 < CPS) w4n = load_round(b + 1);
          const uint32_t pc = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
          uint32_t incl = pc;
          for (int d = 1; d < CPS; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d, CPS);
            if ((lane & (CPS - 1)) >= d) incl += t;
          }
          if (work && pc != 0) sparse_chunk(p, seg, sub, w4, soff + incl - pc, scap);
        }
      }
    }
    const uint32_t cand = (kList && p.sparse_in_a) ? __ballot_sync(0xFFFFFFFFu, sparse_work) : 0u;
    if (kList && cand != 0u) {
      // large selections: this warp's own sparse segments, CPS lanes per segment (one 128-row
      // chunk each).  Rounds run over the group's CANDIDATE segments only (32 / CPS per round):
      // at low selectivity most segments of a group are empty, and a round per 32 / CPS segments
      // regardless of hits cost a bitmap round trip per round with nothing to write.  The next
      // round's bitmap chunk is loaded one round ahead.
      const unsigned long long soff_l = off_l;
      const int CPS = W / 4;
      const int cps_log = __ffs(CPS) - 1;
      const int ncand = __popc(cand);
      const int sub = lane & (CPS - 1);
      // the candidates' group lanes in order, through a per-warp shared-memory list
      uint8_t* clist = cand_lanes[threadIdx.x >> 5];
      __syncwarp();  // the previous group's reads of the list are done
      if (sparse_work) clist[__popc(cand & lt)] = (uint8_t)lane;
      __syncwarp();
      auto cand_lane = [&](int q0) {  // group lane (segment) of this lane's candidate in round q0, or -1
        const int ci = q0 + (lane >> cps_log);
        return ci < ncand ? (int)clist[ci] : -1;
      };
      auto load_round = [&](int sl) {
        return sl >= 0 ? __ldg(reinterpret_cast<const uint4*>(p.bitmap + (seg0 + sl) * W + sub * 4))
                       : make_uint4(0u, 0u, 0u, 0u);
      };
      const int per_round = 32 >> cps_log;
      int sl_n = cand_lane(0);
      uint4 w4n = load_round(sl_n);
      for (int q0 = 0; q0 < ncand; q0 += per_round) {
        const int sl = sl_n;
        const uint4 w4 = w4n;
        if (q0 + per_round < ncand) {
          sl_n = cand_lane(q0 + per_round);
          w4n = load_round(sl_n);
        }
        const int src = sl >= 0 ? sl : 0;
        const unsigned long long soff = __shfl_sync(0xFFFFFFFFu, soff_l, src);
        const bool scap = __shfl_sync(0xFFFFFFFFu, captured ? 1 : 0, src) != 0;
        const uint32_t pc = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
        uint32_t incl = pc;
        for (int d = 1; d < CPS; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d, CPS);
          if (sub >= d) incl += t;
        }
        // the round's hits go to the warp's hit list (row order = output order), and every full
        // 32 entries are gathered by the whole warp at once
        const uint32_t mine = sl >= 0 ? pc : 0u;
        uint32_t wincl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wincl, d);
          if (lane >= d) wincl += t;
        }
        if (mine != 0u) {
          int at = hl_n + (int)(wincl - mine);
          uint32_t pos = (uint32_t)(soff + incl - pc);
          const uint32_t row_base = (uint32_t)(((seg0 + sl) * W + sub * 4) * 32) | (scap ? kHitSkipCaptured : 0u);
          unsigned long long lo = ((unsigned long long)w4.y << 32) | w4.x;
          unsigned long long hi = ((unsigned long long)w4.w << 32) | w4.z;
          while (lo) { hl_row[at] = row_base + __ffsll((long long)lo) - 1; hl_pos[at++] = pos++; lo &= lo - 1; }
          while (hi) { hl_row[at] = row_base + 64 + __ffsll((long long)hi) - 1; hl_pos[at++] = pos++; hi &= hi - 1; }
        }
        hl_n += (int)__shfl_sync(0xFFFFFFFFu, wincl, 31);
        if (hl_n >= 32) hl_n = flush_hits(p, hl_row, hl_pos, hl_n, false);
      }
    }
    uint32_t dense = __ballot_sync(0xFFFFFFFFu, dense_work);
    for (int di = 0; dense; ++di) {
      const int l = __ffs(dense) - 1;
      dense &= dense - 1;
      if ((di & (R - 1)) != r) continue;
      const int64_t seg = seg0 + l;
      const bool seg_captured = __shfl_sync(0xFFFFFFFFu, captured ? 1 : 0, l) != 0;
      const unsigned long long base = __shfl_sync(0xFFFFFFFFu, myoff, l);
      const uint32_t mine = lane < W ? p.bitmap[seg * W + lane] : 0u;
      const uint32_t pc = __popc(mine);
      uint32_t excl = pc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, excl, d);
        if (lane >= d) excl += t;
      }
      excl -= pc;
      // 4 words per batch: each column's loads are issued for all 4 rows before the stores
      for (int i0 = 0; i0 < W; i0 += 4) {
        bool hit[4];
        unsigned long long pos[4];
        int64_t prow[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j < W ? i0 + j : 0;
          const uint32_t word = i0 + j < W ? __shfl_sync(0xFFFFFFFFu, mine, i) : 0u;
          pos[j] = base + __shfl_sync(0xFFFFFFFFu, excl, i) + __popc(word & lt);
          hit[j] = ((word >> lane) & 1u) && (long long)pos[j] < cap;
          const int64_t row = (seg * W + i) * 32 + lane;
          prow[j] = (hit[j] && p.row_ids) ? __ldg(p.row_ids + row) : row;
        }
        for (int k = 0; k < p.n_proj; ++k) {
          if (seg_captured && p.cap_index[k] >= 0) continue;
          const KCol& col = p.cols[k];
          switch (col.width) {
            case 1: gather4<uint8_t>(col.data, p.outs.out_values[k], hit, prow, pos); break;
            case 2: gather4<uint16_t>(col.data, p.outs.out_values[k], hit, prow, pos); break;
            case 4: gather4<uint32_t>(col.data, p.outs.out_values[k], hit, prow, pos); break;
            default: gather4<unsigned long long>(col.data, p.outs.out_values[k], hit, prow, pos); break;
          }
          if (p.outs.out_nulls[k] != nullptr) {
            uint8_t nb[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) nb[j] = (hit[j] && col.nulls) ? __ldg(col.nulls + prow[j]) : (uint8_t)0;
#pragma unroll
            for (int j = 0; j < 4; ++j) if (hit[j]) p.outs.out_nulls[k][pos[j]] = nb[j];
          }
        }
        if (p.outs.out_row_ids != nullptr) {
#pragma unroll
          for (int j = 0; j < 4; ++j) if (hit[j]) p.outs.out_row_ids[pos[j]] = prow[j];
        }
      }
    }
  }
  if (kList && hl_n > 0) flush_hits(p, hl_row, hl_pos, hl_n, true);
  // ---------------- B: sparse segments, one lane per 128-row chunk ----------------
  if (p.sparse_in_a) return;
  const int CPS = W / 4;  // chunks per segment (1, 2, 4, 8): a power of two dividing 32
  const int cps_log = __ffs(CPS) - 1;  // shifts, not 64-bit divisions, in the loop below
  const int64_t n_chunks = p.n_segs * CPS;
  const int64_t stride = nwarps * 32;
  // the next iteration's segment count is loaded one iteration ahead: most chunks have no sparse
  // work (captured, dense or empty), and their iterations should not each wait on a load
  uint32_t raw_next = gwarp * 32 + lane < n_chunks ? __ldg(p.seg_counts + ((gwarp * 32 + lane) >> cps_log)) : 0u;
  for (int64_t c0 = gwarp * 32; c0 < n_chunks; c0 += stride) {
    const int64_t c = c0 + lane;
    const int64_t seg = c >> cps_log;
    const int sub = (int)(c & (CPS - 1));
    const uint32_t raw = raw_next;
    raw_next = c + stride < n_chunks ? __ldg(p.seg_counts + ((c + stride) >> cps_log)) : 0u;
    const uint32_t cnt = raw & ~ESC_SEG_CAPTURED;
    const bool scap = (raw & ESC_SEG_CAPTURED) != 0;
    const bool work = cnt > 0 && cnt <= sparse_max && (!scap || p.need_bitmap_captured) && !in_dense_tile(p, seg);
    uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
    if (work) w4 = __ldg(reinterpret_cast<const uint4*>(p.bitmap + seg * W + sub * 4));
    const uint32_t pc = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
    uint32_t incl = pc;
    for (int d = 1; d < CPS; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d, CPS);
      if ((lane & (CPS - 1)) >= d) incl += t;
    }
    if (!work || pc == 0) continue;
    sparse_chunk(p, seg, sub, w4, p.seg_offsets[seg] + incl - pc, scap);
  }
}

// ------------------------------------------------------------------------------------------
// ONE-kernel selection compaction for mid-size tables (sel_mid_kernel): replaces the offsets scan
// (tile_scan_partials + tile_scan_apply), the streamed and the gathered compaction, i.e. four
// dependent launches, each a few us of launch + ramp at a few million rows.
//
// Block b (an atomic ticket, so it only ever waits on blocks that are already running) owns
// segments [b*SPB, (b+1)*SPB):
//   1. loads its segments' counts and publishes their sum at once (agg[b] = sum + 1, release);
//   2. expands its hits into a shared-memory list (row, capture slot) in row order and issues the
//      loads of every projected value of its first batch of entries (captured values from the
//      scan's capture slots, the rest gathered from HBM) — none of that needs the output base;
//   3. only then reads its base, the sum of agg[0..b): by now every predecessor has published
//      (each does so after one load round trip), so it is a flat parallel read, not a look-back
//      chain, and its latency hides behind the gathers in flight; the last block to have read
//      clears agg[] and the counters (no host reset: prepared graphs re-issue it as is);
//   4. writes entry e of the block to output position base + e (coalesced stores).
// ------------------------------------------------------------------------------------------
constexpr int kMidThreads = 256;
constexpr int kMidMaxBlocks = 4096;  // block-sum words reserved in the workspace
constexpr int kMidList = 2048;       // hit-list entries per batch (>= one whole segment: seg_rows <= 1024)

struct MidParams {
  int32_t segs_per_block;
  int32_t pad;
  int64_t n_blocks;
  unsigned long long* agg;       // [n_blocks] published block sums + 1 (0 = not yet), cleared by the last block
  unsigned long long* ticket;    // block tickets (cleared by the last block)
  unsigned long long* done;      // blocks past their prefix read (cleared by the last block)
  unsigned long long* trace;     // diagnostics (esc_debug_trace): 8 %globaltimer stamps per block, or nullptr
  // early start: the scan of the same step sets this word when its last CTA has published the
  // count (release); the blocks poll it instead of waiting for the scan grid's completion
  // (griddepcontrol.wait), and the last block clears it
  unsigned long long* scan_done;  // nullptr: wait for the scan's completion (PDL)
};

// one thread's share of a batch round: entries e0 + j*256 (j < kMidJ), projections k0 .. k0+3
constexpr int kMidJ = 2;  // entries per thread and round (x 4 projections: 8 loads in flight, no spills)
struct MidRound {
  int64_t prow[kMidJ];
  uint32_t slot[kMidJ];
  bool ok[kMidJ];
  unsigned long long v[4][kMidJ];
  uint8_t nb[4][kMidJ];
};

__device__ __forceinline__ void mid_rows(const SelParams& p, const uint32_t* l_row, const uint32_t* l_slot,
                                         int64_t row0, int nb, int e0, MidRound& r) {
#pragma unroll
  for (int j = 0; j < kMidJ; ++j) {
    const int e = e0 + j * kMidThreads;
    r.ok[j] = e < nb;
    const int64_t row = row0 + (r.ok[j] ? l_row[e] : 0u);
    r.slot[j] = r.ok[j] ? l_slot[e] : 0xFFFFFFFFu;
    r.prow[j] = (r.ok[j] && p.row_ids) ? __ldg(p.row_ids + row) : row;
  }
}

__device__ __forceinline__ void mid_load(const SelParams& p, int k0, MidRound& r) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
    for (int j = 0; j < kMidJ; ++j) {
      r.v[kk][j] = 0;
      r.nb[kk][j] = 0;
    }
    const int k = k0 + kk;
    if (k >= p.n_proj) continue;
    const KCol& col = p.cols[k];
    const int ci = p.cap_index[k];
#pragma unroll
    for (int j = 0; j < kMidJ; ++j) {
      if (!r.ok[j]) continue;
      if (ci >= 0 && r.slot[j] != 0xFFFFFFFFu) {
        r.v[kk][j] = ld_w(col.width, p.cap_values[ci], r.slot[j]);
        if (p.cap_nulls[ci] != nullptr) r.nb[kk][j] = p.cap_nulls[ci][r.slot[j]];
      } else {
        switch (col.width) {
          case 1: r.v[kk][j] = __ldcg(col.data + r.prow[j]); break;
          case 2: r.v[kk][j] = __ldcg(reinterpret_cast<const uint16_t*>(col.data) + r.prow[j]); break;
          case 4: r.v[kk][j] = __ldcg(reinterpret_cast<const uint32_t*>(col.data) + r.prow[j]); break;
          default: r.v[kk][j] = __ldcg(reinterpret_cast<const unsigned long long*>(col.data) + r.prow[j]); break;
        }
        if (col.nulls != nullptr) r.nb[kk][j] = __ldg(col.nulls + r.prow[j]);
      }
    }
  }
}

__device__ __forceinline__ void mid_store(const SelParams& p, int k0, const MidRound& r, unsigned long long pos0,
                                          int e0, long long cap) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = k0 + kk;
    if (k >= p.n_proj) continue;
    const int width = p.cols[k].width;
#pragma unroll
    for (int j = 0; j < kMidJ; ++j) {
      const unsigned long long pos = pos0 + (unsigned long long)(e0 + j * kMidThreads);
      if (!r.ok[j] || (long long)pos >= cap) continue;
      st_bits(width, p.outs.out_values[k], pos, r.v[kk][j]);
      if (p.outs.out_nulls[k] != nullptr) p.outs.out_nulls[k][pos] = r.nb[kk][j];
    }
  }
  if (k0 == 0 && p.outs.out_row_ids != nullptr) {
#pragma unroll
    for (int j = 0; j < kMidJ; ++j) {
      const unsigned long long pos = pos0 + (unsigned long long)(e0 + j * kMidThreads);
      if (r.ok[j] && (long long)pos < cap) p.outs.out_row_ids[pos] = r.prow[j];
    }
  }
}

// block-wide sum of one value per thread (s_red: >= kMidThreads/32 words)
__device__ __forceinline__ unsigned long long mid_block_sum(unsigned long long v, unsigned long long* s_red) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long t = 0;
#pragma unroll
  for (int w = 0; w < kMidThreads / 32; ++w) t += s_red[w];
  return t;
}

__global__ void __launch_bounds__(kMidThreads, 4) sel_mid_kernel(const __grid_constant__ SelParams p,
                                                                 const __grid_constant__ MidParams m) {
  __shared__ uint32_t l_row[kMidList];
  __shared__ uint32_t l_slot[kMidList];
  __shared__ unsigned long long s_red[kMidThreads / 32];
  __shared__ unsigned long long s_scan[33];
  __shared__ long long s_block;
  __shared__ bool s_last;
  extern __shared__ uint32_t s_cnt[];  // [segs_per_block]: counts, then exclusive offsets in the block
  const unsigned long long t_start = m.trace != nullptr ? gtimer() : 0ull;
  const bool early = m.scan_done != nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (early) {
    // the ticket is taken while the flag is polled; thread 0's acquire + the barrier order every
    // thread's later loads after the scan's last writes.  (Bounded: a compaction issued without
    // its scan would otherwise never return; after 0.5 s it reads what an earlier, completed
    // scan left, which is then the whole truth.)
    if (threadIdx.x == 0) {
      s_block = (long long)atomicAdd(m.ticket, 1ull);
      const unsigned long long t_wait = gtimer();
      while (ld_acquire(m.scan_done) == 0ull && gtimer() - t_wait < 500000000ull) __nanosleep(64);
    }
    __syncthreads();
    pdl_trigger();
  } else {
    pdl_wait();
    pdl_trigger();
    if (skip_materialize(p.rule)) return;
    if (threadIdx.x == 0) s_block = (long long)atomicAdd(m.ticket, 1ull);
    __syncthreads();
  }
  if (early && skip_materialize(p.rule)) {  // (the count is final here) every block still settles
    if (threadIdx.x == 0 && atomicAdd(m.done, 1ull) == (unsigned long long)m.n_blocks - 1) {
      __stcg(m.ticket, 0ull);
      __stcg(m.done, 0ull);
      __stcg(m.scan_done, 0ull);
    }
    return;
  }
  const int64_t b = s_block;
  unsigned long long* tr = (m.trace != nullptr && threadIdx.x == 0) ? m.trace + 8 * 1024 + b * 8 : nullptr;
  if (tr) { tr[0] = t_start; tr[1] = gtimer(); }
  const int SPB = m.segs_per_block;
  const int64_t seg0 = b * SPB;
  const int nseg = (int)((seg0 + SPB <= p.n_segs) ? SPB : (p.n_segs > seg0 ? p.n_segs - seg0 : 0));
  const int W = p.seg_rows / 32;
  // the bitmap words of this warp's first four segments are loaded with the counts (the
  // expansion of the first batch then needs no further round trip) — unless captured segments
  // need no bitmap at all (every projection captured, no row ids): then only the (rare)
  // uncaptured segments read theirs
  const bool cap_only = !p.need_bitmap_captured;
  uint32_t wpre[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int si = warp + q * (kMidThreads / 32);
    wpre[q] = (!cap_only && si < nseg && lane < W) ? __ldcg(p.bitmap + (seg0 + si) * W + lane) : 0u;
  }
  // 1. this block's segment counts; their sum is published at once
  unsigned long long mine = 0;
  for (int i = threadIdx.x; i < nseg; i += kMidThreads) {
    const uint32_t c = __ldcg(p.seg_counts + seg0 + i);
    s_cnt[i] = c;
    mine += c & ~ESC_SEG_CAPTURED;
  }
  const unsigned long long block_sum = mid_block_sum(mine, s_red);
  if (threadIdx.x == 0) {
    st_relaxed(m.agg + b, block_sum + 1);  // (the value is the only datum: no release fence)
    if (tr) tr[2] = gtimer();
  }
  // exclusive offsets of the block's segments (in place; chunks of 256 with a running carry;
  // < 2^31: a block's hits <= its rows, bounded on the host)
  unsigned long long carry = 0;
  for (int c0 = 0; c0 < nseg; c0 += kMidThreads) {
    const int i = c0 + threadIdx.x;
    const unsigned long long v = i < nseg ? (s_cnt[i] & ~ESC_SEG_CAPTURED) : 0u;
    unsigned long long tot;
    const unsigned long long ex = block_excl_scan(v, s_scan, &tot);
    if (i < nseg) s_cnt[i] = (uint32_t)(carry + ex) | (s_cnt[i] & ESC_SEG_CAPTURED);
    carry += tot;
  }
  __syncthreads();
  const long long cap = p.outs.capacity;
  const int64_t row0 = seg0 * (int64_t)p.seg_rows;
  const uint32_t block_hits = (uint32_t)carry;
  if (tr) tr[3] = gtimer();
  auto off_of = [&](int i) -> uint32_t { return i < nseg ? (s_cnt[i] & ~ESC_SEG_CAPTURED) : block_hits; };
  unsigned long long base = 0;
  bool have_base = false;
  // 2-4. hit lists, batch by batch of whole segments (a segment's <= 1024 hits always fit)
  for (int sb = 0; sb < nseg || !have_base;) {
    int se = sb;
    uint32_t first = 0, upto = 0;
    if (sb < nseg) {
      first = off_of(sb);
      se = sb + 1;
      while (se < nseg && off_of(se + 1) - first <= (uint32_t)kMidList) ++se;
      upto = off_of(se);
      // expand: warp per segment, lane per bitmap word, hits in row order (the first batch's
      // first four segments per warp use the words loaded at the start)
      for (int si = sb + warp, q = 0; si < se; si += kMidThreads / 32, ++q) {
        const uint32_t o = off_of(si);
        if (off_of(si + 1) == o) continue;  // empty segment
        const bool captured = (s_cnt[si] & ESC_SEG_CAPTURED) != 0;
        const int64_t seg = seg0 + si;
        if (captured && cap_only) {  // the hits' values sit in the capture slots, in row order
          const uint32_t cnt = off_of(si + 1) - o;
          for (uint32_t jj = lane; jj < cnt; jj += 32) {
            l_row[o - first + jj] = 0u;  // (unused: no gather, no row id)
            l_slot[o - first + jj] = (uint32_t)((size_t)jj * p.cap_stride + seg);
          }
          continue;
        }
        const bool pre = !cap_only && sb == 0 && q < 4;
        const uint32_t word = pre ? (q == 0 ? wpre[0] : q == 1 ? wpre[1] : q == 2 ? wpre[2] : wpre[3])
                                  : (lane < W ? __ldcg(p.bitmap + seg * W + lane) : 0u);
        const uint32_t pc = __popc(word);
        if (tr && si == 0 && sb == 0) tr[7] = gtimer() + (pc & 0);  // (diagnostic: first word in hand)
        uint32_t incl = pc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
          if (lane >= d) incl += t;
        }
        const uint32_t cnt = off_of(si + 1) - o;
        if (cnt > 2u * (uint32_t)W) {
          // dense segment: lane per row, word by word (W steps instead of up to 32 bit steps)
          const uint32_t lt = (1u << lane) - 1u, excl = incl - pc;
          for (int w = 0; w < W; ++w) {
            const uint32_t ww = __shfl_sync(0xFFFFFFFFu, word, w);
            const uint32_t wb = __shfl_sync(0xFFFFFFFFu, excl, w);
            if ((ww >> lane) & 1u) {
              const uint32_t jj = wb + __popc(ww & lt);
              const uint32_t e = o - first + jj;
              l_row[e] = (uint32_t)si * (uint32_t)p.seg_rows + (uint32_t)w * 32u + (uint32_t)lane;
              l_slot[e] = captured ? (uint32_t)((size_t)jj * p.cap_stride + seg) : 0xFFFFFFFFu;
            }
          }
          continue;
        }
        uint32_t j = incl - pc;  // rank of this word's first hit in the segment
        uint32_t wbits = word;
        const uint32_t rbase = (uint32_t)si * (uint32_t)p.seg_rows + (uint32_t)lane * 32u;
        while (wbits) {
          const int bit = __ffs(wbits) - 1;
          wbits &= wbits - 1;
          const uint32_t e = o - first + j;
          l_row[e] = rbase + (uint32_t)bit;
          l_slot[e] = captured ? (uint32_t)((size_t)j * p.cap_stride + seg) : 0xFFFFFFFFu;
          ++j;
        }
      }
      __syncthreads();
    }
    if (tr && sb == 0) tr[4] = gtimer();
    const int nb = (int)(upto - first);
    // the first round's loads are issued BEFORE the base is read (they do not need it)
    for (int e0 = threadIdx.x, round = 0; round == 0 || e0 < nb; e0 += kMidJ * kMidThreads, ++round) {
      for (int k0 = 0; k0 < (p.n_proj > 0 ? p.n_proj : 1); k0 += 4) {
        MidRound r;
        mid_rows(p, l_row, l_slot, row0, nb, e0, r);
        mid_load(p, k0, r);
        if (!have_base) {  // block-uniform: every thread takes this branch together, once
          unsigned long long pre = 0;
          for (int64_t q = threadIdx.x; q < b; q += kMidThreads) {
            unsigned long long v = ld_relaxed(m.agg + q);  // relaxed polls (acquire per poll is a fence each)
            while (v == 0ull) v = ld_relaxed(m.agg + q);
            pre += v - 1;
          }
          // no fence here: it would wait for the gathers in flight; the polls are complete
          // (their values are consumed) before this block counts itself done below
          base = mid_block_sum(pre, s_red);
          have_base = true;
          if (threadIdx.x == 0) {
            if (tr) tr[5] = gtimer();
            // the last block past its base read resets the table for the next launch (all its
            // threads: one thread clearing ~600 words serially made it the step's last block)
            s_last = atomicAdd(m.done, 1ull) == (unsigned long long)m.n_blocks - 1;
          }
          __syncthreads();
          if (s_last) {
            for (int64_t q = threadIdx.x; q < m.n_blocks; q += kMidThreads) __stcg(m.agg + q, 0ull);
            if (threadIdx.x == 0) {
              __stcg(m.ticket, 0ull);
              __stcg(m.done, 0ull);
              if (early) __stcg(m.scan_done, 0ull);
            }
          }
        }
        mid_store(p, k0, r, base + first, e0, cap);
      }
    }
    __syncthreads();
    sb = se;
    if (sb >= nseg) break;
  }
  if (tr) tr[6] = gtimer();
}

// ------------------------------------------------------------------------------------------
// streamed compaction of dense tiles: TMA stages the tile's bitmap words, segment offsets and
// projected columns (+ null bytes) into a shared-memory ring; consumer warps write each hit
// straight to its final position (contiguous across the lanes of a word).
// ------------------------------------------------------------------------------------------
struct StreamParams {
  const uint32_t* bitmap;
  const unsigned long long* seg_offsets;
  const uint32_t* dense_list;
  const uint32_t* n_dense;
  int32_t seg_rows;        // 128*C
  int32_t segs_per_tile;   // 2, 4, 8
  int32_t tile_rows;       // seg_rows * segs_per_tile
  int32_t stages;
  uint32_t stage_bytes;
  uint32_t tma_bytes;      // bytes the bulk copies of a full tile deliver
  uint32_t meta_bytes;     // ... of the tail tile (bitmap words + offsets only)
  int64_t n_full_tiles;    // tiles below this are staged whole; the tail tile reads HBM directly
  uint32_t off_bitmap;     // stage offset of the tile's bitmap words
  uint32_t off_offsets;    // stage offset of the tile's segment offsets
  int32_t n_proj;
  int32_t width[ESC_MAX_PROJ];
  const uint8_t* data[ESC_MAX_PROJ];
  const uint8_t* nulls[ESC_MAX_PROJ];  // staged null bytes when the output wants them, else nullptr
  uint32_t off_val[ESC_MAX_PROJ];
  uint32_t off_null[ESC_MAX_PROJ];
  esc_outputs_t outs;
  // what the consumers copy, as byte streams grouped by width: streams [cls[c], cls[c+1]) are
  // 8, 4, 2, 1 bytes wide for c = 0..3 (values and staged null bytes alike), then `n_zero` null
  // outputs without a source (written 0)
  int32_t cls[5];
  int32_t n_zero;
  int32_t consumers;       // consumer warps (<= kStreamConsumers; the block is 1 + consumers warps)
  uint32_t s_off[2 * ESC_MAX_PROJ];         // stage offset of the stream's tile
  const uint8_t* s_src[2 * ESC_MAX_PROJ];   // its column in HBM (the tail tile)
  uint8_t* s_dst[2 * ESC_MAX_PROJ];         // its output buffer
  uint8_t* zero_dst[ESC_MAX_PROJ];
};

constexpr int kStreamConsumers = 16;

// Write the hits of up to 4 consecutive bitmap words of one warp segment, for the streams of one
// width class: lane l of word j owns tile row lr + 32j; bit j of `h` says it writes that row (a hit
// inside the output capacity) to output base + of[j].  Each stream loads its (up to) 4 values
// first, then stores them, so a lane keeps 4 loads in flight; the store of a word is contiguous
// across its hit lanes.  Staged tiles read shared memory, the tail tile the column in HBM.
template <typename T, bool STAGED>
__device__ __forceinline__ void stream_class(const StreamParams& p, int k0, int k1, const uint8_t* st,
                                             int64_t row_base, unsigned long long base, uint32_t h,
                                             const uint32_t (&of)[4], int lr) {
  for (int k = k0; k < k1; ++k) {
    const T* src = STAGED ? reinterpret_cast<const T*>(st + p.s_off[k])
                          : reinterpret_cast<const T*>(p.s_src[k]) + row_base;
    T* dst = reinterpret_cast<T*>(p.s_dst[k]) + base;
    T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = ((h >> j) & 1u) ? src[lr + 32 * j] : T(0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((h >> j) & 1u) dst[of[j]] = v[j];
  }
}

template <bool STAGED>
__device__ __forceinline__ void stream_words(const StreamParams& p, const uint8_t* st, int64_t row_base,
                                             unsigned long long base, uint32_t h, const uint32_t (&of)[4],
                                             int lr) {
  stream_class<unsigned long long, STAGED>(p, p.cls[0], p.cls[1], st, row_base, base, h, of, lr);
  stream_class<uint32_t, STAGED>(p, p.cls[1], p.cls[2], st, row_base, base, h, of, lr);
  stream_class<uint16_t, STAGED>(p, p.cls[2], p.cls[3], st, row_base, base, h, of, lr);
  stream_class<uint8_t, STAGED>(p, p.cls[3], p.cls[4], st, row_base, base, h, of, lr);
  for (int k = 0; k < p.n_zero; ++k) {
    uint8_t* dst = p.zero_dst[k] + base;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((h >> j) & 1u) dst[of[j]] = 0;
  }
  if (p.outs.out_row_ids != nullptr) {
    int64_t* ro = p.outs.out_row_ids + base;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((h >> j) & 1u) ro[of[j]] = row_base + lr + 32 * j;
  }
}

__global__ void __launch_bounds__((1 + kStreamConsumers) * 32, 1) sel_stream_kernel(const __grid_constant__ StreamParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  pdl_wait();
  pdl_trigger();
  const uint32_t nd = *p.n_dense;
  if (blockIdx.x >= nd) return;  // a CTA without a dense tile to stream leaves at once
  const int S = p.stages;
  uint8_t* ring = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  long long* tile_of = reinterpret_cast<long long*>(empty_bar + kMaxStages);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], p.consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t policy = evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      for (uint32_t k = blockIdx.x;; k += gridDim.x, s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
        mbar_wait(&empty_bar[s], ph ^ 1u);
        if (k >= nd) {
          tile_of[s] = -1;
          mbar_arrive(&full_bar[s]);
          break;
        }
        const int64_t tile = p.dense_list[k];
        const bool full = tile < p.n_full_tiles;  // the tail tile's columns are read from HBM directly
        tile_of[s] = tile;
        uint8_t* dst = ring + (size_t)s * p.stage_bytes;
        const int64_t row0 = tile * p.tile_rows;
        mbar_arrive_expect_tx(&full_bar[s], full ? p.tma_bytes : p.meta_bytes);
        bulk_g2s(dst + p.off_bitmap, p.bitmap + row0 / 32, (uint32_t)p.tile_rows / 8, &full_bar[s], policy);
        bulk_g2s(dst + p.off_offsets, p.seg_offsets + tile * p.segs_per_tile, (uint32_t)p.segs_per_tile * 8,
                 &full_bar[s], policy);
        if (full) {
          for (int k2 = 0; k2 < p.n_proj; ++k2) {
            const int w = p.width[k2];
            bulk_g2s(dst + p.off_val[k2], p.data[k2] + (size_t)row0 * w, (uint32_t)p.tile_rows * w, &full_bar[s],
                     policy);
            if (p.nulls[k2] != nullptr)
              bulk_g2s(dst + p.off_null[k2], p.nulls[k2] + row0, (uint32_t)p.tile_rows, &full_bar[s], policy);
          }
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int wps = p.consumers / p.segs_per_tile;  // warps per segment (host: <= words per segment)
  const int seg = cw / wps;
  const int W = p.seg_rows / 32;
  const int wpart = W / wps;                            // words this warp writes
  const int w0 = (cw % wps) * wpart;
  const uint32_t lt = (1u << lane) - 1u;
  const long long cap = p.outs.capacity;
  int s = 0;
  uint32_t ph = 0;
  for (;; s = (s + 1 == S) ? 0 : s + 1, ph ^= (s == 0)) {
    mbar_wait(&full_bar[s], ph);
    const int64_t tile = tile_of[s];
    if (tile < 0) break;
    const uint8_t* st = ring + (size_t)s * p.stage_bytes;
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(st + p.off_bitmap) + seg * W;
    const unsigned long long base = reinterpret_cast<const unsigned long long*>(st + p.off_offsets)[seg];
    // hits before this warp's words, and in the whole segment (one reduction each, no scan)
    const uint32_t pc = lane < W ? __popc(bm[lane]) : 0u;
    uint32_t pre = __reduce_add_sync(0xFFFFFFFFu, lane < w0 ? pc : 0u);
    const uint32_t seg_hits = __reduce_add_sync(0xFFFFFFFFu, pc);
    // outputs [base, base + seg_hits) of this segment; past the capacity nothing is written
    const bool fits = (long long)(base + seg_hits) <= cap;
    const long long room_ll = cap - (long long)base;
    const uint32_t room = room_ll <= 0 ? 0u : (room_ll >= (1ll << 32) ? 0xFFFFFFFFu : (uint32_t)room_ll);
    const bool full = tile < p.n_full_tiles;
    const int64_t row_base = tile * p.tile_rows;
    for (int i0 = w0; i0 < w0 + wpart; i0 += 4) {
      uint32_t of[4], h = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t word = i0 + j < w0 + wpart ? bm[i0 + j] : 0u;  // broadcast read
        of[j] = pre + __popc(word & lt);
        pre += __popc(word);
        if (((word >> lane) & 1u) && (fits || of[j] < room)) h |= 1u << j;
      }
      if (__ballot_sync(0xFFFFFFFFu, h != 0) == 0) continue;
      const int lr = seg * p.seg_rows + 32 * i0 + lane;
      if (full) stream_words<true>(p, st, row_base, base, h, of, lr);
      else stream_words<false>(p, st, row_base, base, h, of, lr);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }
}

// ---- batched region copy (esc_copy_regions): blockIdx.y = region -----------------------------
struct CopyRegions {
  int32_t n;
  uint8_t* dst[ESC_MAX_REGIONS];
  const uint8_t* src[ESC_MAX_REGIONS];
  long long bytes[ESC_MAX_REGIONS];
};

__global__ void __launch_bounds__(256) copy_regions_kernel(const __grid_constant__ CopyRegions p) {
  const int r = blockIdx.y;
  uint8_t* d = p.dst[r];
  const uint8_t* s = p.src[r];
  const long long nb = p.bytes[r];
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (((reinterpret_cast<unsigned long long>(d) | reinterpret_cast<unsigned long long>(s)) & 15ull) == 0) {
    const long long nv = nb >> 4;
    for (long long i = t0; i < nv; i += stride)
      reinterpret_cast<uint4*>(d)[i] = __ldg(reinterpret_cast<const uint4*>(s) + i);
    for (long long i = (nv << 4) + t0; i < nb; i += stride) d[i] = s[i];
  } else {
    for (long long i = t0; i < nb; i += stride) d[i] = s[i];
  }
}

// ---- multi-GPU count gate (esc_count_gate): one warp folds the all-gathered per-rank counts ----
__global__ void __launch_bounds__(32) count_gate_kernel(const int64_t* __restrict__ counts, int world, int rank,
                                                        long long capacity, int64_t* __restrict__ out) {
  const int lane = threadIdx.x;
  unsigned long long total = 0, before = 0;
  for (int r = lane; r < world; r += 32) {
    const unsigned long long c = (unsigned long long)counts[r];
    total += c;
    if (r < rank) before += c;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    total += __shfl_xor_sync(0xFFFFFFFFu, total, d);
    before += __shfl_xor_sync(0xFFFFFFFFu, before, d);
  }
  if (lane == 0) {
    out[0] = (int64_t)total;
    out[1] = (int64_t)before;
    out[2] = total <= (unsigned long long)capacity ? 0 : (int64_t)(1ull << 62);
  }
}

// packed NULL bitmap of a bool mask (esc_pack_nulls): one word per thread
__global__ void pack_nulls_kernel(const uint8_t* __restrict__ nulls, int64_t n, int64_t words,
                                  uint32_t* __restrict__ out) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    const int64_t r0 = w * 32;
    if (r0 + 32 <= n) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // 4 bytes at a time (the mask is only byte-aligned)
        const uint32_t x = (uint32_t)nulls[r0 + 4 * q] | ((uint32_t)nulls[r0 + 4 * q + 1] << 8) |
                           ((uint32_t)nulls[r0 + 4 * q + 2] << 16) | ((uint32_t)nulls[r0 + 4 * q + 3] << 24);
        const uint32_t nz = ((x & 0x01010101u) | ((x >> 1) & 0x01010101u) | ((x >> 2) & 0x01010101u) |
                             ((x >> 3) & 0x01010101u) | ((x >> 4) & 0x01010101u) | ((x >> 5) & 0x01010101u) |
                             ((x >> 6) & 0x01010101u) | ((x >> 7) & 0x01010101u));
        v |= (((nz * 0x01020408u) >> 24) & 0xFu) << (4 * q);
      }
    } else {
      for (int64_t r = r0; r < n && r < r0 + 32; ++r) v |= (nulls[r] != 0 ? 1u : 0u) << (r - r0);
    }
    out[w] = v;
  }
}

// gather: out[i] = col[idx[i]]
template <typename T>
__global__ void gather_kernel(const T* __restrict__ src, const uint8_t* __restrict__ nulls,
                              const int64_t* __restrict__ idx, int64_t n, T* __restrict__ out,
                              uint8_t* __restrict__ out_nulls) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = __ldg(idx + i);
    out[i] = __ldg(src + r);
    if (out_nulls != nullptr) out_nulls[i] = nulls != nullptr ? __ldg(nulls + r) : 0;
  }
}

}  // namespace esc
