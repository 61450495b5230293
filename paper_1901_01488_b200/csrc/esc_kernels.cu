// esc_kernels.cu — sm_100a kernels for the ESC selectivity sub-query, behind the C ABI in
// include/esc.h.
//
//   K1 esc_scan_count : fused predicate evaluation + exact count        (executor.py:218-224)
//   K2 esc_compact    : fused predicate + count + order-preserving
//                       compaction with decoupled look-back            (executor.py:202-215,
//                                                                       optimizer.py:180-194)
//   esc_gather        : Column.take                                    (storage.py:176-184)
//
// Design: one persistent CTA per SM. Warp 0 is a TMA producer that streams the
// predicate columns of each tile (T rows x the staged columns, native widths) into an S-stage
// shared-memory ring with cp.async.bulk + mbarrier complete_tx. 16 consumer warps evaluate a
// flat boolean program (compiled on the host from the resolved expr tree, passed by value as a
// __grid_constant__ kernel parameter) over the tile. Each lane owns C chunks of 4 consecutive
// rows, so the smem reads of a chunk are one conflict-free 128-bit access per lane; each
// opcode is dispatched once per lane per tile and evaluated on 4*C rows into a bit mask, so the
// interpreter cost is amortised over the rows. Counting is popc; compaction packs per-chunk
// lane counts into 8-bit fields so ONE warp scan ranks all chunks, then a block scan across
// warps and a decoupled look-back across tiles (tickets from an atomic counter give forward
// progress) place the tile's rows in global order.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/esc.h"

namespace {

constexpr int kConsumerWarps = 16;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kChunkRows = 128;  // one warp chunk: 32 lanes x 4 consecutive rows
constexpr int kMaxStages = 4;
constexpr uint32_t kSmemBudget = 200 * 1024;  // dynamic smem for the stage ring
constexpr int kStatusValueBits = 46;
constexpr uint64_t kStatusValueMask = (1ull << kStatusValueBits) - 1;
constexpr uint64_t kFlagAggregate = 1;
constexpr uint64_t kFlagPrefix = 2;

// ------------------------------------------------------------------------------------------
// workspace layout
// ------------------------------------------------------------------------------------------
struct WsHeader {
  unsigned long long count;   // running count (atomicAdd per CTA)
  unsigned long long ticket;  // tile ticket counter (compaction)
  unsigned long long done;    // CTAs finished (last-CTA detection)
  unsigned long long pad0;
  unsigned long long fail[ESC_MAX_UDFS];  // first failing row per UDF (packed), ~0 = none
  unsigned long long pad1[4];
};
static_assert(sizeof(WsHeader) == 128, "header is one 128-byte line");

struct KCol {
  const uint8_t* data;
  const uint8_t* nulls;
  int32_t dtype;
  int32_t width;
  int32_t staged;       // values staged in smem for full tiles
  int32_t nulls_staged; // null bytes staged in smem for full tiles
  uint32_t smem_off;
  uint32_t smem_null_off;
};

struct KParams {
  esc_program_t prog;
  KCol cols[ESC_MAX_COLS];
  int32_t ncols;
  int32_t chunks;       // C
  int32_t tile_rows;    // T = kConsumerWarps * 128 * C
  int32_t stages;
  uint32_t stage_bytes;
  uint32_t epoch;
  int64_t nrows;
  int64_t n_tiles;
  int64_t n_full_tiles;  // tiles [0, n_full_tiles) are staged with TMA
  const int64_t* row_ids;
  WsHeader* hdr;
  unsigned long long* status;
  esc_result_t* result;
  esc_outputs_t outs;
};

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
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
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
// per-lane tile view
// ------------------------------------------------------------------------------------------
struct LaneTile {
  const uint8_t* stage;  // smem stage base, nullptr when the tile is read directly from HBM
  int64_t grow0;         // logical row of this lane's chunk-0 first row
  int32_t local0;        // row of chunk 0 within the tile
  int64_t nrows;
  const int64_t* ids;    // gather mode: physical row of logical row i
};

template <typename T>
__device__ __forceinline__ T ldg_t(const uint8_t* base, int64_t row) {
  return __ldg(reinterpret_cast<const T*>(base) + row);
}

// 4 consecutive staged values of type T starting at 4-aligned local row
template <typename T>
__device__ __forceinline__ void lds4(const uint8_t* p, T (&v)[4]) {
  if constexpr (sizeof(T) == 1) {
    uint32_t x = *reinterpret_cast<const uint32_t*>(p);
    memcpy(v, &x, 4);
  } else if constexpr (sizeof(T) == 2) {
    uint2 x = *reinterpret_cast<const uint2*>(p);
    memcpy(v, &x, 8);
  } else if constexpr (sizeof(T) == 4) {
    uint4 x = *reinterpret_cast<const uint4*>(p);
    memcpy(v, &x, 16);
  } else {
    uint4 x = reinterpret_cast<const uint4*>(p)[0];
    uint4 y = reinterpret_cast<const uint4*>(p)[1];
    memcpy(&v[0], &x, 16);
    memcpy(&v[2], &y, 16);
  }
}

__device__ __forceinline__ int64_t phys_row(const LaneTile& lt, int64_t r) {
  return lt.ids ? __ldg(lt.ids + r) : r;
}

// Load chunk c (4 rows) of column `col` as T, converted to D.
template <typename T, typename D, int C>
__device__ __forceinline__ void fetch_t(const KCol& col, const LaneTile& lt, D (&out)[4 * C]) {
#pragma unroll
  for (int c = 0; c < C; ++c) {
    T v[4];
    if (lt.stage != nullptr && col.staged) {
      lds4<T>(lt.stage + col.smem_off + (size_t)(lt.local0 + kChunkRows * c) * sizeof(T), v);
    } else {
      const int64_t r0 = lt.grow0 + kChunkRows * c;
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = (r0 + j < lt.nrows) ? ldg_t<T>(col.data, phys_row(lt, r0 + j)) : T(0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) out[4 * c + j] = static_cast<D>(v[j]);
  }
}

// exact conversions where numpy's are exact; RN where numpy rounds (int64 -> f64, f64 -> f32 never used)
template <typename D, int C>
__device__ __forceinline__ void fetch(const KCol& col, const LaneTile& lt, D (&out)[4 * C]) {
  switch (col.dtype) {
    case ESC_I8: fetch_t<int8_t, D, C>(col, lt, out); break;
    case ESC_I16: fetch_t<int16_t, D, C>(col, lt, out); break;
    case ESC_I32: fetch_t<int32_t, D, C>(col, lt, out); break;
    case ESC_I64: fetch_t<long long, D, C>(col, lt, out); break;
    case ESC_U8: fetch_t<uint8_t, D, C>(col, lt, out); break;
    case ESC_U16: fetch_t<uint16_t, D, C>(col, lt, out); break;
    case ESC_U32: fetch_t<uint32_t, D, C>(col, lt, out); break;
    case ESC_F32: fetch_t<float, D, C>(col, lt, out); break;
    default: fetch_t<double, D, C>(col, lt, out); break;
  }
}

// 4*C null bits of a column (bit set = NULL)
template <int C>
__device__ __forceinline__ uint32_t null_bits(const KCol& col, const LaneTile& lt) {
  if (col.nulls == nullptr) return 0u;
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    uint32_t x;
    if (lt.stage != nullptr && col.nulls_staged) {
      x = *reinterpret_cast<const uint32_t*>(lt.stage + col.smem_null_off + lt.local0 + kChunkRows * c);
    } else {
      const int64_t r0 = lt.grow0 + kChunkRows * c;
      x = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (r0 + j < lt.nrows) x |= (uint32_t)(__ldg(col.nulls + phys_row(lt, r0 + j)) != 0) << (8 * j);
    }
    // gather bit 0 of each byte into 4 bits
    const uint32_t nb = (((x & 0x01010101u) * 0x01020408u) >> 24) & 0xFu;
    bits |= nb << (4 * c);
  }
  return bits;
}

template <typename D, int CMP>
__device__ __forceinline__ bool cmp1(D v, D k) {
  if constexpr (CMP == ESC_CMP_EQ) return v == k;
  else if constexpr (CMP == ESC_CMP_NE) return v != k;
  else if constexpr (CMP == ESC_CMP_LT) return v < k;
  else if constexpr (CMP == ESC_CMP_LE) return v <= k;
  else if constexpr (CMP == ESC_CMP_GT) return v > k;
  else return v >= k;
}

template <typename D, int CMP, int C>
__device__ __forceinline__ uint32_t cmp_bits(const D (&v)[4 * C], D k) {
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 4 * C; ++b) r |= (uint32_t)cmp1<D, CMP>(v[b], k) << b;
  return r;
}

template <typename D, int C>
__device__ __forceinline__ uint32_t cmp_dispatch(int cmp, const D (&v)[4 * C], D k) {
  switch (cmp) {
    case ESC_CMP_EQ: return cmp_bits<D, ESC_CMP_EQ, C>(v, k);
    case ESC_CMP_NE: return cmp_bits<D, ESC_CMP_NE, C>(v, k);
    case ESC_CMP_LT: return cmp_bits<D, ESC_CMP_LT, C>(v, k);
    case ESC_CMP_LE: return cmp_bits<D, ESC_CMP_LE, C>(v, k);
    case ESC_CMP_GT: return cmp_bits<D, ESC_CMP_GT, C>(v, k);
    default: return cmp_bits<D, ESC_CMP_GE, C>(v, k);
  }
}

template <typename D, int C>
__device__ __forceinline__ uint32_t range_bits(const D (&v)[4 * C], D lo, D hi) {
  uint32_t r = 0;
#pragma unroll
  for (int b = 0; b < 4 * C; ++b) r |= (uint32_t)((v[b] >= lo) & (v[b] <= hi)) << b;
  return r;
}

template <typename D>
__device__ __forceinline__ D kconst(const esc_const_t& k);
template <>
__device__ __forceinline__ long long kconst<long long>(const esc_const_t& k) { return k.i; }
template <>
__device__ __forceinline__ double kconst<double>(const esc_const_t& k) { return k.f; }
template <>
__device__ __forceinline__ float kconst<float>(const esc_const_t& k) { return static_cast<float>(k.f); }

template <typename D, int C>
__device__ __forceinline__ uint32_t atom_cmp_d(const esc_instr_t& I, const KCol& col, const LaneTile& lt) {
  D v[4 * C];
  fetch<D, C>(col, lt, v);
  if (I.op == ESC_OP_RANGE) return range_bits<D, C>(v, kconst<D>(I.k0), kconst<D>(I.k1));
  return cmp_dispatch<D, C>(I.cmp, v, kconst<D>(I.k0));
}

template <int C>
__device__ __noinline__ uint32_t atom_cmp(const esc_instr_t& I, const KCol& col, const LaneTile& lt) {
  switch (I.domain) {
    case ESC_DOM_I64: return atom_cmp_d<long long, C>(I, col, lt);
    case ESC_DOM_F32: return atom_cmp_d<float, C>(I, col, lt);
    default: return atom_cmp_d<double, C>(I, col, lt);
  }
}

template <typename D, int C>
__device__ __forceinline__ uint32_t atom_colcmp_d(const esc_instr_t& I, const KCol& a, const KCol& b,
                                                  const LaneTile& lt) {
  D va[4 * C], vb[4 * C];
  fetch<D, C>(a, lt, va);
  fetch<D, C>(b, lt, vb);
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 4 * C; ++i) {
    bool t;
    switch (I.cmp) {
      case ESC_CMP_EQ: t = va[i] == vb[i]; break;
      case ESC_CMP_NE: t = va[i] != vb[i]; break;
      case ESC_CMP_LT: t = va[i] < vb[i]; break;
      case ESC_CMP_LE: t = va[i] <= vb[i]; break;
      case ESC_CMP_GT: t = va[i] > vb[i]; break;
      default: t = va[i] >= vb[i]; break;
    }
    r |= (uint32_t)t << i;
  }
  return r;
}

template <int C>
__device__ __noinline__ uint32_t atom_colcmp(const esc_instr_t& I, const KCol& a, const KCol& b,
                                             const LaneTile& lt) {
  switch (I.domain) {
    case ESC_DOM_I64: return atom_colcmp_d<long long, C>(I, a, b, lt);
    case ESC_DOM_F32: return atom_colcmp_d<float, C>(I, a, b, lt);
    default: return atom_colcmp_d<double, C>(I, a, b, lt);
  }
}

template <int C>
__device__ __noinline__ uint32_t atom_lut(const esc_instr_t& I, const KCol& col, const LaneTile& lt,
                                          const uint32_t* lut) {
  long long v[4 * C];
  fetch<long long, C>(col, lt, v);
  uint32_t r = 0;
  const long long n = (long long)I.aux2;
#pragma unroll
  for (int b = 0; b < 4 * C; ++b) {
    const long long code = v[b];
    bool t = false;
    if (code >= 0 && code < n) t = (__ldg(lut + I.aux + (code >> 5)) >> (code & 31)) & 1u;
    r |= (uint32_t)t << b;
  }
  return r;
}

// ---- UDF: CPython float semantics ----------------------------------------------------------
__device__ __forceinline__ double load_f64(const KCol& col, const LaneTile& lt, int bit) {
  const int c = bit >> 2, j = bit & 3;
  const int64_t grow = lt.grow0 + kChunkRows * c + j;
  const uint8_t* p;
  if (lt.stage != nullptr && col.staged) {
    p = lt.stage + col.smem_off + (size_t)(lt.local0 + kChunkRows * c + j) * col.width;
    switch (col.dtype) {
      case ESC_I8: return (double)*reinterpret_cast<const int8_t*>(p);
      case ESC_I16: return (double)*reinterpret_cast<const int16_t*>(p);
      case ESC_I32: return (double)*reinterpret_cast<const int32_t*>(p);
      case ESC_I64: return __ll2double_rn(*reinterpret_cast<const long long*>(p));
      case ESC_U8: return (double)*reinterpret_cast<const uint8_t*>(p);
      case ESC_U16: return (double)*reinterpret_cast<const uint16_t*>(p);
      case ESC_U32: return (double)*reinterpret_cast<const uint32_t*>(p);
      case ESC_F32: return (double)*reinterpret_cast<const float*>(p);
      default: return *reinterpret_cast<const double*>(p);
    }
  }
  const int64_t r = phys_row(lt, grow);
  switch (col.dtype) {
    case ESC_I8: return (double)ldg_t<int8_t>(col.data, r);
    case ESC_I16: return (double)ldg_t<int16_t>(col.data, r);
    case ESC_I32: return (double)ldg_t<int32_t>(col.data, r);
    case ESC_I64: return __ll2double_rn(ldg_t<long long>(col.data, r));
    case ESC_U8: return (double)ldg_t<uint8_t>(col.data, r);
    case ESC_U16: return (double)ldg_t<uint16_t>(col.data, r);
    case ESC_U32: return (double)ldg_t<uint32_t>(col.data, r);
    case ESC_F32: return (double)ldg_t<float>(col.data, r);
    default: return ldg_t<double>(col.data, r);
  }
}

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

// Evaluate UDF `u` on one row; returns the value, sets *fail to a ESC_FAIL_* code on error.
__device__ double udf_eval(const esc_program_t& prog, const esc_udf_t& u, const KCol* cols, const LaneTile& lt,
                           int bit, uint32_t* fail) {
  double stk[16];
  int sp = 0;
  double args[ESC_MAX_UDF_ARGS];
  for (int a = 0; a < u.n_args; ++a) {
    double x = load_f64(cols[u.arg_col[a]], lt, bit);
    if (u.arg_div[a] != 0.0) x = __ddiv_rn(x, u.arg_div[a]);
    args[a] = x;
  }
  for (int i = 0; i < u.n_ops; ++i) {
    const esc_udf_op_t& o = prog.udf_ops[u.first_op + i];
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
          default:  // FLOORDIV
            if (b == 0.0) { *fail = ESC_FAIL_FLOORDIV; return 0.0; }
            r = py_floordiv(a, b);
            break;
        }
        stk[sp - 1] = r;
      }
    }
  }
  return stk[0];
}

__device__ __forceinline__ bool cmp_f64(int cmp, double v, double k) {
  switch (cmp) {
    case ESC_CMP_EQ: return v == k;
    case ESC_CMP_NE: return v != k;
    case ESC_CMP_LT: return v < k;
    case ESC_CMP_LE: return v <= k;
    case ESC_CMP_GT: return v > k;
    default: return v >= k;
  }
}

template <int C>
__device__ __noinline__ uint32_t atom_udf(const KParams& p, const esc_instr_t& I, const LaneTile& lt,
                                          uint32_t care, uint32_t valid) {
  const esc_udf_t& u = p.prog.udfs[I.aux];
  uint32_t todo = (u.dense ? valid : (care & valid));
  uint32_t r = 0;
  while (todo) {
    const int bit = __ffs(todo) - 1;
    todo &= todo - 1;
    uint32_t fail = 0;
    const double v = udf_eval(p.prog, u, p.cols, lt, bit, &fail);
    if (fail) {
      const int64_t grow = lt.grow0 + kChunkRows * (bit >> 2) + (bit & 3);
      atomicMin(&p.hdr->fail[I.aux], (unsigned long long)(grow << 3) | fail);
    } else if (cmp_f64(I.cmp, v, I.k0.f)) {
      r |= 1u << bit;
    }
  }
  // false when any argument is NULL (executor.py:146)
  uint32_t nn = 0;
  for (int a = 0; a < u.n_args; ++a) nn |= null_bits<C>(p.cols[u.arg_col[a]], lt);
  return r & ~nn;
}

__device__ __forceinline__ uint32_t combine(int mode, uint32_t acc, uint32_t r) {
  return mode == ESC_COMB_AND ? (acc & r) : mode == ESC_COMB_OR ? (acc | r) : r;
}
__device__ __forceinline__ uint32_t care_for(int mode, uint32_t acc, uint32_t care) {
  return mode == ESC_COMB_AND ? (care & acc) : mode == ESC_COMB_OR ? (care & ~acc) : care;
}

// Evaluate the boolean program on this lane's 4*C rows of the tile.
template <int C>
__device__ __forceinline__ uint32_t eval_program(const KParams& p, const LaneTile& lt, uint32_t valid) {
  const esc_program_t& prog = p.prog;
  uint32_t acc = 0, care = valid;
  uint32_t stk_acc[ESC_MAX_STACK], stk_care[ESC_MAX_STACK];
  int sp = 0;
  const int n = prog.n_instrs;
  for (int pc = 0; pc < n; ++pc) {
    const esc_instr_t& I = prog.instrs[pc];
    uint32_t r;
    switch (I.op) {
      case ESC_OP_PUSH:
        stk_acc[sp] = acc;
        stk_care[sp] = care;
        ++sp;
        care = care_for(I.combine, acc, care);
        acc = 0;
        continue;
      case ESC_OP_POP:
        --sp;
        acc = combine(I.combine, stk_acc[sp], acc);
        care = stk_care[sp];
        continue;
      case ESC_OP_NOT:
        acc = ~acc;
        continue;
      case ESC_OP_CMP:
      case ESC_OP_RANGE: {
        const KCol& col = p.cols[I.col_a];
        r = atom_cmp<C>(I, col, lt) & ~null_bits<C>(col, lt);
        break;
      }
      case ESC_OP_LUT: {
        const KCol& col = p.cols[I.col_a];
        r = atom_lut<C>(I, col, lt, prog.lut) & ~null_bits<C>(col, lt);
        break;
      }
      case ESC_OP_COLCMP: {
        const KCol& a = p.cols[I.col_a];
        const KCol& b = p.cols[I.col_b];
        r = atom_colcmp<C>(I, a, b, lt) & ~(null_bits<C>(a, lt) | null_bits<C>(b, lt));
        break;
      }
      case ESC_OP_NOTNULL:
        r = ~null_bits<C>(p.cols[I.col_a], lt);
        break;
      case ESC_OP_UDF:
        r = atom_udf<C>(p, I, lt, care_for(I.combine, acc, care), valid);
        break;
      default:  // ESC_OP_FALSE
        r = 0;
        break;
    }
    if (I.neg) r = ~r;
    acc = combine(I.combine, acc, r);
  }
  return acc & valid;
}

__device__ __forceinline__ uint32_t valid_bits(int64_t grow0, int64_t nrows, int C) {
  uint32_t v = 0;
  for (int c = 0; c < C; ++c)
    for (int j = 0; j < 4; ++j) v |= (uint32_t)(grow0 + kChunkRows * c + j < nrows) << (4 * c + j);
  return v;
}

// Decoupled look-back: publish the tile aggregate, accumulate predecessors until an inclusive
// prefix is found, publish the inclusive prefix; returns the exclusive prefix of this tile.
__device__ unsigned long long lookback(unsigned long long* status, int64_t tile, unsigned long long agg,
                                       uint32_t epoch) {
  const unsigned long long tag = (unsigned long long)epoch << 48;
  if (tile == 0) {
    st_release(&status[0], tag | (kFlagPrefix << kStatusValueBits) | agg);
    return 0;
  }
  st_release(&status[tile], tag | (kFlagAggregate << kStatusValueBits) | agg);
  unsigned long long excl = 0;
  int64_t q = tile - 1;
  while (true) {
    const unsigned long long w = ld_acquire(&status[q]);
    if ((w >> 48) != epoch) continue;  // predecessor has not published yet
    excl += w & kStatusValueMask;
    if (((w >> kStatusValueBits) & 3ull) == kFlagPrefix) break;
    --q;
  }
  st_release(&status[tile], tag | (kFlagPrefix << kStatusValueBits) | (excl + agg));
  return excl;
}

template <int C>
__device__ __forceinline__ void write_hits(const KParams& p, const LaneTile& lt, uint32_t bits, int chunk,
                                           unsigned long long pos) {
  const esc_outputs_t& o = p.outs;
  for (int j = 0; j < 4; ++j) {
    if (!((bits >> (4 * chunk + j)) & 1u)) continue;
    if ((int64_t)pos < o.capacity) {
      const int64_t grow = lt.grow0 + kChunkRows * chunk + j;
      const int32_t local = lt.local0 + kChunkRows * chunk + j;
      const int64_t prow = phys_row(lt, grow);
      for (int k = 0; k < o.n_proj; ++k) {
        const KCol& col = p.cols[o.slot[k]];
        const int w = col.width;
        const uint8_t* src = (lt.stage != nullptr && col.staged) ? lt.stage + col.smem_off + (size_t)local * w
                                                                 : col.data + (size_t)prow * w;
        uint8_t* dst = static_cast<uint8_t*>(o.out_values[k]) + (size_t)pos * w;
        switch (w) {
          case 1: *dst = *src; break;
          case 2: *reinterpret_cast<uint16_t*>(dst) = *reinterpret_cast<const uint16_t*>(src); break;
          case 4: *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src); break;
          default: *reinterpret_cast<uint64_t*>(dst) = *reinterpret_cast<const uint64_t*>(src); break;
        }
        if (o.out_nulls[k] != nullptr) {
          uint8_t nb = 0;
          if (col.nulls != nullptr)
            nb = (lt.stage != nullptr && col.nulls_staged) ? lt.stage[col.smem_null_off + local]
                                                            : __ldg(col.nulls + prow);
          o.out_nulls[k][pos] = nb;
        }
      }
      if (o.out_row_ids != nullptr) o.out_row_ids[pos] = lt.ids != nullptr ? phys_row(lt, grow) : grow;
    }
    ++pos;
  }
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------
template <int C, bool COMPACT>
__global__ void __launch_bounds__(kThreads, 1) esc_scan_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = p.stages;
  uint8_t* ring = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + (size_t)S * p.stage_bytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  long long* tile_of = reinterpret_cast<long long*>(empty_bar + kMaxStages);
  uint32_t* s_warp_tot = reinterpret_cast<uint32_t*>(tile_of + kMaxStages);
  uint32_t* s_warp_off = s_warp_tot + kConsumerWarps;
  unsigned long long* s_misc = reinterpret_cast<unsigned long long*>(s_warp_off + kConsumerWarps);
  // s_misc[0] = tile base (compaction), s_misc[1..16] per-warp counts, s_misc[17] = last flag

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ===================== producer =====================
    if (lane == 0) {
      const uint64_t policy = evict_first_policy();
      int64_t static_next = blockIdx.x;
      for (int64_t k = 0;; ++k) {
        const int s = (int)(k % S);
        const uint32_t ph = (uint32_t)((k / S) & 1);
        int64_t tile;
        if constexpr (COMPACT) {
          tile = (int64_t)atomicAdd(&p.hdr->ticket, 1ull);
        } else {
          tile = static_next;
          static_next += gridDim.x;
        }
        mbar_wait(&empty_bar[s], ph ^ 1u);
        if (tile >= p.n_tiles) {
          tile_of[s] = -1;
          mbar_arrive(&full_bar[s]);
          break;
        }
        tile_of[s] = tile;
        if (tile < p.n_full_tiles) {
          mbar_arrive_expect_tx(&full_bar[s], p.stage_bytes);
          uint8_t* dst = ring + (size_t)s * p.stage_bytes;
          const int64_t row0 = tile * p.tile_rows;
          for (int i = 0; i < p.ncols; ++i) {
            const KCol& col = p.cols[i];
            if (col.staged)
              bulk_g2s(dst + col.smem_off, col.data + (size_t)row0 * col.width, (uint32_t)p.tile_rows * col.width,
                       &full_bar[s], policy);
            if (col.nulls_staged)
              bulk_g2s(dst + col.smem_null_off, col.nulls + row0, (uint32_t)p.tile_rows, &full_bar[s], policy);
          }
        } else {
          mbar_arrive(&full_bar[s]);
        }
      }
    }
    return;
  }

  // ===================== consumers =====================
  const int cw = warp - 1;
  unsigned long long my_count = 0;
  for (int64_t k = 0;; ++k) {
    const int s = (int)(k % S);
    const uint32_t ph = (uint32_t)((k / S) & 1);
    mbar_wait(&full_bar[s], ph);
    const int64_t tile = tile_of[s];
    if (tile < 0) break;

    LaneTile lt;
    lt.stage = (tile < p.n_full_tiles) ? ring + (size_t)s * p.stage_bytes : nullptr;
    lt.local0 = cw * (kChunkRows * C) + 4 * lane;
    lt.grow0 = tile * p.tile_rows + lt.local0;
    lt.nrows = p.nrows;
    lt.ids = p.row_ids;
    const uint32_t valid = (lt.stage != nullptr) ? ((4 * C == 32) ? 0xFFFFFFFFu : ((1u << (4 * C)) - 1u))
                                                 : valid_bits(lt.grow0, p.nrows, C);
    const uint32_t bits = eval_program<C>(p, lt, valid);

    if constexpr (!COMPACT) {
      my_count += __popc(bits);
    } else {
      // per-chunk lane counts packed in 8-bit fields -> one warp scan ranks every chunk
      uint32_t packed = 0;
#pragma unroll
      for (int c = 0; c < C; ++c) packed |= (uint32_t)__popc((bits >> (4 * c)) & 0xFu) << (8 * c);
      uint32_t incl = packed;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t wtot_packed = __shfl_sync(0xFFFFFFFFu, incl, 31);
      uint32_t wtot = 0;
#pragma unroll
      for (int c = 0; c < C; ++c) wtot += (wtot_packed >> (8 * c)) & 0xFFu;
      if (lane == 0) s_warp_tot[cw] = wtot;
      consumer_bar();
      if (cw == 0) {
        uint32_t v = lane < kConsumerWarps ? s_warp_tot[lane] : 0u;
        uint32_t sc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, sc, d);
          if (lane >= d) sc += t;
        }
        if (lane < kConsumerWarps) s_warp_off[lane] = sc - v;
        const uint32_t tile_total = __shfl_sync(0xFFFFFFFFu, sc, 31);
        if (lane == 0) {
          s_misc[0] = lookback(p.status, tile, tile_total, p.epoch);
          my_count += tile_total;
        }
      }
      consumer_bar();
      const unsigned long long warp_base = s_misc[0] + s_warp_off[cw];
      const uint32_t excl = incl - packed;
      uint32_t chunk_base = 0;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t lane_excl = (excl >> (8 * c)) & 0xFFu;
        if ((bits >> (4 * c)) & 0xFu) write_hits<C>(p, lt, bits, c, warp_base + chunk_base + lane_excl);
        chunk_base += (wtot_packed >> (8 * c)) & 0xFFu;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);
  }

  // ---- CTA reduction, global accumulation, last-CTA finalisation ----
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) my_count += __shfl_down_sync(0xFFFFFFFFu, my_count, d);
  if (lane == 0) s_misc[1 + cw] = my_count;
  consumer_bar();
  if (threadIdx.x == 32) {
    unsigned long long tot = 0;
    for (int w = 0; w < kConsumerWarps; ++w) tot += s_misc[1 + w];
    if (tot) atomicAdd(&p.hdr->count, tot);
    __threadfence();
    const unsigned long long prev = atomicAdd(&p.hdr->done, 1ull);
    s_misc[17] = (prev == gridDim.x - 1) ? 1ull : 0ull;
    if (prev == gridDim.x - 1) {
      __threadfence();
      volatile WsHeader* h = p.hdr;
      p.result->count = h->count;
      for (int i = 0; i < ESC_MAX_UDFS; ++i) {
        p.result->udf_fail[i] = h->fail[i];
        h->fail[i] = ~0ull;
      }
      h->count = 0;
      h->ticket = 0;
      h->done = 0;
      __threadfence_system();
    }
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

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int dtype_width(int dt) {
  switch (dt) {
    case ESC_I8: case ESC_U8: return 1;
    case ESC_I16: case ESC_U16: return 2;
    case ESC_I32: case ESC_U32: case ESC_F32: return 4;
    case ESC_I64: case ESC_F64: return 8;
    default: return 0;
  }
}

int sm_count_cached() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n;
  return n;
}

// per-workspace epoch for the look-back status words (host side; guarded)
std::mutex g_epoch_mu;
std::unordered_map<const void*, uint32_t> g_epochs;

size_t status_words(int64_t nrows) {
  // smallest tile is kConsumerWarps * 128 rows
  const int64_t t = (int64_t)kConsumerWarps * kChunkRows;
  return (size_t)((nrows + t - 1) / t) + 1;
}

int validate_program(const esc_program_t* prog, int32_t ncols) {
  if (prog == nullptr) return fail(ESC_ERR_INVALID, "null program");
  if (prog->abi_version != ESC_ABI_VERSION) return fail(ESC_ERR_INVALID, "program ABI version mismatch");
  if (prog->n_instrs > ESC_MAX_INSTRS || prog->n_udfs > ESC_MAX_UDFS || prog->n_udf_ops > ESC_MAX_UDF_OPS)
    return fail(ESC_ERR_INVALID, "program exceeds limits");
  if (prog->max_depth > ESC_MAX_STACK) return fail(ESC_ERR_INVALID, "program nesting too deep");
  int depth = 0;
  for (int i = 0; i < prog->n_instrs; ++i) {
    const esc_instr_t& I = prog->instrs[i];
    if (I.op < ESC_OP_CMP || I.op > ESC_OP_NOT) return fail(ESC_ERR_INVALID, "bad opcode");
    if (I.op == ESC_OP_PUSH && ++depth > ESC_MAX_STACK) return fail(ESC_ERR_INVALID, "stack overflow");
    if (I.op == ESC_OP_POP && --depth < 0) return fail(ESC_ERR_INVALID, "stack underflow");
    const bool uses_col = I.op == ESC_OP_CMP || I.op == ESC_OP_RANGE || I.op == ESC_OP_LUT ||
                          I.op == ESC_OP_COLCMP || I.op == ESC_OP_NOTNULL;
    if (uses_col && I.col_a >= ncols) return fail(ESC_ERR_INVALID, "column slot out of range");
    if (I.op == ESC_OP_COLCMP && I.col_b >= ncols) return fail(ESC_ERR_INVALID, "column slot out of range");
    if (I.op == ESC_OP_LUT && (prog->lut == nullptr || (uint64_t)I.aux + (I.aux2 + 31) / 32 > prog->lut_words))
      return fail(ESC_ERR_INVALID, "LUT out of range");
    if (I.op == ESC_OP_UDF) {
      if (I.aux >= prog->n_udfs) return fail(ESC_ERR_INVALID, "UDF index out of range");
      const esc_udf_t& u = prog->udfs[I.aux];
      if (u.n_args > ESC_MAX_UDF_ARGS || u.first_op + u.n_ops > prog->n_udf_ops)
        return fail(ESC_ERR_INVALID, "UDF out of range");
      for (int a = 0; a < u.n_args; ++a)
        if (u.arg_col[a] >= ncols) return fail(ESC_ERR_INVALID, "UDF argument slot out of range");
      int sp = 0;
      for (int k = 0; k < u.n_ops; ++k) {
        const esc_udf_op_t& o = prog->udf_ops[u.first_op + k];
        if (o.op == ESC_UDF_ARG) {
          if (o.arg >= u.n_args) return fail(ESC_ERR_INVALID, "UDF ARG index out of range");
          ++sp;
        } else if (o.op == ESC_UDF_CONST) {
          ++sp;
        } else if (o.op == ESC_UDF_NEG || o.op == ESC_UDF_ABS || o.op == ESC_UDF_SQUARE) {
          if (sp < 1) return fail(ESC_ERR_INVALID, "UDF stack underflow");
        } else if (o.op >= ESC_UDF_ADD && o.op <= ESC_UDF_FLOORDIV) {
          if (sp < 2) return fail(ESC_ERR_INVALID, "UDF stack underflow");
          --sp;
        } else {
          return fail(ESC_ERR_INVALID, "bad UDF opcode");
        }
        if (sp > 16) return fail(ESC_ERR_INVALID, "UDF stack overflow");
      }
      if (sp != 1) return fail(ESC_ERR_INVALID, "UDF program must leave one value");
    }
  }
  if (depth != 0) return fail(ESC_ERR_INVALID, "unbalanced PUSH/POP");
  return ESC_OK;
}

struct Geometry {
  int chunks = 1;
  int tile_rows = 0;
  int stages = 0;
  uint32_t stage_bytes = 0;
};

// Decide which columns are staged and the tile geometry.
// Slots the boolean program (or its UDFs) reads.
uint64_t program_slots(const esc_program_t* prog) {
  uint64_t m = 0;
  for (int i = 0; i < prog->n_instrs; ++i) {
    const esc_instr_t& I = prog->instrs[i];
    switch (I.op) {
      case ESC_OP_CMP: case ESC_OP_RANGE: case ESC_OP_LUT: case ESC_OP_NOTNULL: m |= 1ull << I.col_a; break;
      case ESC_OP_COLCMP: m |= (1ull << I.col_a) | (1ull << I.col_b); break;
      case ESC_OP_UDF: {
        const esc_udf_t& u = prog->udfs[I.aux];
        for (int a = 0; a < u.n_args; ++a) m |= 1ull << u.arg_col[a];
        break;
      }
      default: break;
    }
  }
  return m;
}

Geometry plan_geometry(KParams& kp, const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                       bool gather, int64_t nrows) {
  Geometry g;
  const uint64_t used = program_slots(prog);
  // bytes per row of stageable columns
  uint32_t per_row = 0;
  for (int i = 0; i < ncols; ++i) {
    KCol& c = kp.cols[i];
    const bool want = ((used >> i) & 1ull) || (cols[i].flags & ESC_COL_STAGE);
    c.staged = want && !gather && (reinterpret_cast<uintptr_t>(c.data) % 16 == 0);
    c.nulls_staged = want && !gather && c.nulls != nullptr && (reinterpret_cast<uintptr_t>(c.nulls) % 16 == 0);
    per_row += (c.staged ? c.width : 0) + (c.nulls_staged ? 1 : 0);
  }
  // choose C so that >= 3 stages fit (prefer larger tiles for small per-row bytes)
  int chunks = 4;
  while (chunks > 1 && (uint64_t)kConsumerWarps * kChunkRows * chunks * per_row * 3 > kSmemBudget) chunks >>= 1;
  int tile_rows = kConsumerWarps * kChunkRows * chunks;
  // if even C=1 cannot hold 2 stages, drop columns from staging (largest first) until it does
  while ((uint64_t)tile_rows * per_row * 2 > kSmemBudget) {
    int best = -1;
    for (int i = 0; i < ncols; ++i)
      if (kp.cols[i].staged && (best < 0 || kp.cols[i].width > kp.cols[best].width)) best = i;
    if (best < 0) break;
    kp.cols[best].staged = 0;
    per_row -= kp.cols[best].width;
    if (kp.cols[best].nulls_staged) {
      kp.cols[best].nulls_staged = 0;
      per_row -= 1;
    }
  }
  g.chunks = chunks;
  g.tile_rows = tile_rows;
  uint32_t off = 0;
  for (int i = 0; i < ncols; ++i) {
    KCol& c = kp.cols[i];
    if (c.staged) { c.smem_off = off; off += (uint32_t)tile_rows * c.width; }
    if (c.nulls_staged) { c.smem_null_off = off; off += (uint32_t)tile_rows; }
  }
  g.stage_bytes = off;
  if (off == 0 || nrows < tile_rows) {
    g.stages = 1;  // nothing staged (or no full tile): the ring only carries tile ids
    g.stage_bytes = 0;
    for (int i = 0; i < ncols; ++i) kp.cols[i].staged = kp.cols[i].nulls_staged = 0;
  } else {
    g.stages = (int)(kSmemBudget / off);
    if (g.stages > kMaxStages) g.stages = kMaxStages;
    if (g.stages < 1) g.stages = 1;
  }
  return g;
}

int build_params(KParams& kp, const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                 const int64_t* row_ids, void* d_ws, size_t ws_bytes, esc_result_t* result) {
  if (ncols < 0 || ncols > ESC_MAX_COLS) return fail(ESC_ERR_INVALID, "ncols out of range");
  if (nrows < 0) return fail(ESC_ERR_INVALID, "negative nrows");
  if (nrows >= (1ll << kStatusValueBits)) return fail(ESC_ERR_INVALID, "nrows exceeds 2^46");
  if (result == nullptr) return fail(ESC_ERR_INVALID, "null result");
  int rc = validate_program(prog, ncols);
  if (rc != ESC_OK) return rc;
  if (d_ws == nullptr || (reinterpret_cast<uintptr_t>(d_ws) % 128) != 0)
    return fail(ESC_ERR_WORKSPACE, "workspace must be 128-byte aligned");
  if (ws_bytes < esc_workspace_bytes(nrows)) return fail(ESC_ERR_WORKSPACE, "workspace too small");
  std::memset(&kp, 0, sizeof(kp));
  std::memcpy(&kp.prog, prog, sizeof(esc_program_t));
  for (int i = 0; i < ncols; ++i) {
    const int w = dtype_width(cols[i].dtype);
    if (w == 0) return fail(ESC_ERR_INVALID, "bad column dtype");
    if (cols[i].data == nullptr && nrows > 0) return fail(ESC_ERR_INVALID, "null column data");
    kp.cols[i].data = static_cast<const uint8_t*>(cols[i].data);
    kp.cols[i].nulls = cols[i].nulls;
    kp.cols[i].dtype = cols[i].dtype;
    kp.cols[i].width = w;
  }
  kp.ncols = ncols;
  kp.nrows = nrows;
  kp.row_ids = row_ids;
  Geometry g = plan_geometry(kp, prog, cols, ncols, row_ids != nullptr, nrows);
  kp.chunks = g.chunks;
  kp.tile_rows = g.tile_rows;
  kp.stages = g.stages;
  kp.stage_bytes = g.stage_bytes;
  kp.n_tiles = (nrows + g.tile_rows - 1) / g.tile_rows;
  kp.n_full_tiles = (g.stage_bytes == 0) ? 0 : nrows / g.tile_rows;
  kp.hdr = static_cast<WsHeader*>(d_ws);
  kp.status = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(d_ws) + sizeof(WsHeader));
  kp.result = result;
  return ESC_OK;
}

size_t smem_bytes_for(const KParams& kp) {
  return (size_t)kp.stages * kp.stage_bytes + 2 * kMaxStages * sizeof(uint64_t) + kMaxStages * sizeof(long long) +
         2 * kConsumerWarps * sizeof(uint32_t) + 20 * sizeof(unsigned long long);
}

template <int C, bool COMPACT>
int launch_c(const KParams& kp, cudaStream_t stream) {
  auto kern = esc_scan_kernel<C, COMPACT>;
  const size_t smem = smem_bytes_for(kp);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t grid = kp.n_tiles < sms ? kp.n_tiles : sms;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(kp);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

template <bool COMPACT>
int launch(const KParams& kp, cudaStream_t stream) {
  switch (kp.chunks) {
    case 4: return launch_c<4, COMPACT>(kp, stream);
    case 2: return launch_c<2, COMPACT>(kp, stream);
    default: return launch_c<1, COMPACT>(kp, stream);
  }
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

size_t esc_workspace_bytes(int64_t nrows) {
  if (nrows < 0) nrows = 0;
  return sizeof(WsHeader) + status_words(nrows) * sizeof(unsigned long long);
}

int esc_workspace_init(void* d_ws, size_t ws_bytes, void* stream) {
  if (d_ws == nullptr || ws_bytes < sizeof(WsHeader)) return fail(ESC_ERR_WORKSPACE, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_ws, 0, ws_bytes, st);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(static_cast<uint8_t*>(d_ws) + offsetof(WsHeader, fail), 0xFF,
                        sizeof(unsigned long long) * ESC_MAX_UDFS, st);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("workspace init: ") + cudaGetErrorString(e));
  std::lock_guard<std::mutex> g(g_epoch_mu);
  g_epochs[d_ws] = 0;
  return ESC_OK;
}

int esc_scan_count(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                   const int64_t* d_row_ids, esc_result_t* result, void* d_ws, size_t ws_bytes, void* stream) {
  static thread_local KParams kp;
  int rc = build_params(kp, prog, cols, ncols, nrows, d_row_ids, d_ws, ws_bytes, result);
  if (rc != ESC_OK) return rc;
  return launch<false>(kp, static_cast<cudaStream_t>(stream));
}

int esc_compact(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                const int64_t* d_row_ids, const esc_outputs_t* outs, esc_result_t* result, void* d_ws,
                size_t ws_bytes, void* stream) {
  static thread_local KParams kp;
  int rc = build_params(kp, prog, cols, ncols, nrows, d_row_ids, d_ws, ws_bytes, result);
  if (rc != ESC_OK) return rc;
  if (outs == nullptr) return fail(ESC_ERR_INVALID, "null outputs");
  if (outs->n_proj < 0 || outs->n_proj > ESC_MAX_PROJ) return fail(ESC_ERR_INVALID, "n_proj out of range");
  if (outs->capacity < 0) return fail(ESC_ERR_INVALID, "negative capacity");
  for (int k = 0; k < outs->n_proj; ++k) {
    if (outs->slot[k] < 0 || outs->slot[k] >= ncols) return fail(ESC_ERR_INVALID, "projection slot out of range");
    if (outs->out_values[k] == nullptr && outs->capacity > 0) return fail(ESC_ERR_INVALID, "null output buffer");
  }
  kp.outs = *outs;
  {
    std::lock_guard<std::mutex> g(g_epoch_mu);
    uint32_t& ep = g_epochs[d_ws];
    ep = (ep + 1) & 0xFFFFu;
    if (ep == 0) {
      // epoch wrapped: stale status words could alias, clear them
      cudaError_t e = cudaMemsetAsync(kp.status, 0, status_words(nrows) * sizeof(unsigned long long),
                                      static_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("status clear: ") + cudaGetErrorString(e));
      ep = 1;
    }
    kp.epoch = ep;
  }
  return launch<true>(kp, static_cast<cudaStream_t>(stream));
}

int esc_gather(const esc_column_t* col, const int64_t* d_idx, int64_t n, void* out_values, uint8_t* out_nulls,
               void* stream) {
  if (col == nullptr || n < 0) return fail(ESC_ERR_INVALID, "bad gather arguments");
  if (n == 0) return ESC_OK;
  if (d_idx == nullptr || out_values == nullptr || col->data == nullptr)
    return fail(ESC_ERR_INVALID, "null gather buffer");
  const int w = dtype_width(col->dtype);
  if (w == 0) return fail(ESC_ERR_INVALID, "bad column dtype");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int threads = 256;
  int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  switch (w) {
    case 1:
      gather_kernel<uint8_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint8_t*>(col->data), col->nulls,
                                                                   d_idx, n, static_cast<uint8_t*>(out_values),
                                                                   out_nulls);
      break;
    case 2:
      gather_kernel<uint16_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint16_t*>(col->data),
                                                                    col->nulls, d_idx, n,
                                                                    static_cast<uint16_t*>(out_values), out_nulls);
      break;
    case 4:
      gather_kernel<uint32_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint32_t*>(col->data),
                                                                    col->nulls, d_idx, n,
                                                                    static_cast<uint32_t*>(out_values), out_nulls);
      break;
    default:
      gather_kernel<unsigned long long><<<(unsigned)blocks, threads, 0, st>>>(
          static_cast<const unsigned long long*>(col->data), col->nulls, d_idx, n,
          static_cast<unsigned long long*>(out_values), out_nulls);
      break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("gather launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

const char* esc_last_error(void) { return g_last_error.c_str(); }

int esc_abi_version(void) { return ESC_ABI_VERSION; }

int esc_device_sm_count(void) { return sm_count_cached(); }

int esc_struct_size(int which) {
  switch (which) {
    case 0: return (int)sizeof(esc_program_t);
    case 1: return (int)sizeof(esc_instr_t);
    case 2: return (int)sizeof(esc_udf_t);
    case 3: return (int)sizeof(esc_udf_op_t);
    case 4: return (int)sizeof(esc_column_t);
    case 5: return (int)sizeof(esc_result_t);
    case 6: return (int)sizeof(esc_outputs_t);
    default: return -1;
  }
}

int esc_tile_rows(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols) {
  static thread_local KParams kp;
  if (ncols < 0 || ncols > ESC_MAX_COLS) return 0;
  std::memset(&kp, 0, sizeof(kp));
  for (int i = 0; i < ncols; ++i) {
    kp.cols[i].data = static_cast<const uint8_t*>(cols[i].data);
    kp.cols[i].nulls = cols[i].nulls;
    kp.cols[i].dtype = cols[i].dtype;
    kp.cols[i].width = dtype_width(cols[i].dtype);
  }
  if (prog == nullptr) return 0;
  return plan_geometry(kp, prog, cols, ncols, false, 1ll << 40).tile_rows;
}

}  // extern "C"
