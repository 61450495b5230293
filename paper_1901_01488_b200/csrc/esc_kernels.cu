// esc_kernels.cu — sm_100a kernels for the ESC selectivity sub-query, behind the C ABI in
// include/esc.h.
//
//   K1 esc_scan_count : fused predicate evaluation + exact count        (executor.py:218-224)
//   K2 esc_compact    : fused predicate + count + order-preserving
//                       compaction with decoupled look-back            (executor.py:202-215,
//                                                                       optimizer.py:180-194)
//   esc_gather        : Column.take                                    (storage.py:176-184)
//
// Design: one persistent CTA per SM.
//   warp 0  TMA producer: streams the predicate columns of each tile (T rows x staged columns,
//           native widths) into an S-stage shared-memory ring (cp.async.bulk + mbarrier
//           complete_tx; L2 evict-first, every byte is read once).
//   warp 1  (K2 only) look-back warp: per tile, combines the consumer warps' counts and runs a
//           warp-parallel decoupled look-back over the tile status words (tickets from an atomic
//           counter give forward progress), publishing the tile's global base.
//   16 consumer warps: evaluate the compiled predicate over the tile. Each lane owns C chunks of
//           4 consecutive rows, so a chunk of a staged column is one conflict-free LDS.128 (4-byte
//           types). The host lowers every comparison to an inclusive (optionally negated) range
//           in one of four domains, so the hot opcodes are ~10 tight smem-only loops: 2 ALU ops
//           per row for integers ((u)(v-lo) <= span), 2 for floats. The result of each opcode is
//           a 4*C-bit mask merged into an accumulator (AND/OR/SET + PUSH/POP groups); the
//           dispatch cost is paid once per lane per tile. In K2 the scatter of tile k is deferred
//           to iteration k+1 so the look-back latency never stalls the consumers.
// Tiles that are not staged (tail tile, row-id selections, unaligned columns) run a separate,
// cold, bounds-checked evaluator.
#include <cuda_runtime.h>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <sstream>
#include <atomic>
#include <vector>

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <utility>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/esc.h"
#include "esc_device.cuh"

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
namespace {
using namespace esc;

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};  // kernels this library has launched (esc_launch_count)
unsigned long long* g_trace = nullptr;           // esc_debug_trace stamps (diagnostics only)

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

bool dtype_int_range(int dt, long long* lo, long long* hi) {
  switch (dt) {
    case ESC_I8: *lo = -128; *hi = 127; return true;
    case ESC_U8: *lo = 0; *hi = 255; return true;
    case ESC_I16: *lo = -32768; *hi = 32767; return true;
    case ESC_U16: *lo = 0; *hi = 65535; return true;
    case ESC_I32: *lo = INT32_MIN; *hi = INT32_MAX; return true;
    case ESC_U32: *lo = 0; *hi = 4294967295ll; return true;
    case ESC_I64: *lo = INT64_MIN; *hi = INT64_MAX; return true;
    default: return false;
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

// K1 L2 prefetch of the whole scan when its staged bytes are at most this (ESC_PREFETCH_L2_BYTES;
// 0 = off): the 126 MB L2 holds a mid-size table's predicate columns
std::atomic<long long> g_prefetch_max_bytes{[] {
  const char* e = getenv("ESC_PREFETCH_L2_BYTES");
  return e ? atoll(e) : 0ll;  // measured slower on config 2 (43 -> 47 us): off by default
}()};

// per-workspace epoch for the look-back status words (host side; guarded), and the most status
// words any one-pass launch on that workspace has used (all of them end at the workspace's end)
std::mutex g_epoch_mu;
struct EpochState {
  uint32_t epoch = 0;
  size_t max_words = 0;
};
std::unordered_map<const void*, EpochState> g_epochs;

size_t status_words(int64_t nrows) {
  const int64_t t = (int64_t)kConsumerWarps * kChunkRows;  // smallest tile
  return (size_t)((nrows + t - 1) / t) + 1;
}

// Workspace layout: [header][mid-kernel block sums u64 x kMidMaxBlocks][segment offsets u64]
//                   [scan partials u64][segment counts u32][selection bitmap u32]
//                   [dense-tile counter + list u32] ... [tile status u64]
// The one-pass kernel's tile status words sit at the END of the workspace, whatever its size
// (status_base): every other region is a prefix whose extent grows with nrows, the status words a
// suffix that does too, and esc_workspace_bytes(n) covers both, so for any two launches of
// n_a, n_b <= the workspace's capacity the prefix regions of one never overlap the status words of
// the other — a smaller table's offsets/bitmap can never leave words that a later look-back
// might take for a published status (they carry a 16-bit epoch tag, see next_epoch).
struct WsLayout {
  size_t mid, offsets, partials, counts, bitmap, dense, total;
  int64_t max_tiles, bitmap_words;
};
WsLayout ws_layout(int64_t nrows) {
  WsLayout L;
  if (nrows < 0) nrows = 0;
  const int64_t t_min = (int64_t)kConsumerWarps * kChunkRows;        // smallest tile (C = 1)
  const int64_t t_max = 8 * t_min;                                   // largest tile (C = 8)
  L.max_tiles = ((nrows + t_min - 1) / t_min + 1) * kConsumerWarps;  // warp segments
  L.bitmap_words = ((nrows + t_max - 1) / t_max + 1) * (t_max / 32);  // covers every C's last tile
  const int64_t segs = L.max_tiles / kScanSeg + 2;
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  // [header][one line: sel_mid_kernel's early-start flag, away from the header's atomics]
  L.mid = sizeof(WsHeader) + 128;  // sel_mid_kernel block sums: a FIXED place (every launch size sees the
                                   // same words, which its last block leaves zero)
  L.offsets = up(L.mid + kMidMaxBlocks * sizeof(unsigned long long));
  L.partials = up(L.offsets + (size_t)L.max_tiles * 8);
  L.counts = up(L.partials + (size_t)segs * 8);
  L.bitmap = up(L.counts + (size_t)L.max_tiles * 4);
  L.dense = up(L.bitmap + (size_t)L.bitmap_words * 4);
  L.total = up(L.dense + 256 + (size_t)L.max_tiles * 4) + up(status_words(nrows) * 8);
  return L;
}

unsigned long long* status_base(void* d_ws, size_t ws_bytes, int64_t nrows) {
  uint8_t* end = static_cast<uint8_t*>(d_ws) + (ws_bytes & ~(size_t)7);
  return reinterpret_cast<unsigned long long*>(end - status_words(nrows) * 8);
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
    if (I.combine > ESC_COMB_OR) return fail(ESC_ERR_INVALID, "bad combine mode");
    if (I.op == ESC_OP_PUSH && ++depth > ESC_MAX_STACK) return fail(ESC_ERR_INVALID, "stack overflow");
    if (I.op == ESC_OP_POP && --depth < 0) return fail(ESC_ERR_INVALID, "stack underflow");
    const bool uses_col = I.op == ESC_OP_CMP || I.op == ESC_OP_RANGE || I.op == ESC_OP_LUT ||
                          I.op == ESC_OP_COLCMP || I.op == ESC_OP_NOTNULL;
    if (uses_col && I.col_a >= ncols) return fail(ESC_ERR_INVALID, "column slot out of range");
    if ((I.op == ESC_OP_CMP || I.op == ESC_OP_COLCMP || I.op == ESC_OP_UDF) && I.cmp > ESC_CMP_GE)
      return fail(ESC_ERR_INVALID, "bad comparison operator");
    if ((I.op == ESC_OP_CMP || I.op == ESC_OP_RANGE || I.op == ESC_OP_COLCMP) && I.domain > ESC_DOM_F64)
      return fail(ESC_ERR_INVALID, "bad comparison domain");
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
      // stack heights along every path (jumps only go forward, so one pass in op order visits each
      // op after all of its predecessors): a branch merge must see one height, the end exactly 1
      int height[ESC_MAX_UDF_OPS + 1];
      for (int k = 0; k <= u.n_ops; ++k) height[k] = -1;
      height[0] = 0;
      for (int k = 0; k < u.n_ops; ++k) {
        const esc_udf_op_t& o = prog->udf_ops[u.first_op + k];
        int sp = height[k];
        if (sp < 0) continue;  // unreachable
        int jump = -1;  // extra successor
        bool falls = true;
        if (o.op == ESC_UDF_ARG) {
          if (o.arg >= u.n_args) return fail(ESC_ERR_INVALID, "UDF ARG index out of range");
          ++sp;
        } else if (o.op == ESC_UDF_CONST) {
          ++sp;
        } else if (o.op == ESC_UDF_NEG || o.op == ESC_UDF_ABS || o.op == ESC_UDF_SQUARE ||
                   (o.op >= ESC_UDF_FLOOR && o.op <= ESC_UDF_RINT)) {
          if (sp < 1) return fail(ESC_ERR_INVALID, "UDF stack underflow");
        } else if ((o.op >= ESC_UDF_ADD && o.op <= ESC_UDF_FLOORDIV) || (o.op >= ESC_UDF_LT && o.op <= ESC_UDF_NE)) {
          if (sp < 2) return fail(ESC_ERR_INVALID, "UDF stack underflow");
          --sp;
        } else if (o.op == ESC_UDF_JMPF || o.op == ESC_UDF_JMP) {
          if (o.op == ESC_UDF_JMPF && sp-- < 1) return fail(ESC_ERR_INVALID, "UDF stack underflow");
          jump = k + 1 + o.arg;
          if (jump > u.n_ops) return fail(ESC_ERR_INVALID, "UDF jump out of range");
          falls = o.op == ESC_UDF_JMPF;
        } else {
          return fail(ESC_ERR_INVALID, "bad UDF opcode");
        }
        if (sp > 16) return fail(ESC_ERR_INVALID, "UDF stack overflow");
        for (int t : {falls ? k + 1 : -1, jump}) {
          if (t < 0) continue;
          if (height[t] >= 0 && height[t] != sp) return fail(ESC_ERR_INVALID, "UDF branches leave different stacks");
          height[t] = sp;
        }
      }
      if (height[u.n_ops] != 1) return fail(ESC_ERR_INVALID, "UDF program must leave one value");
    }
  }
  if (depth != 0) return fail(ESC_ERR_INVALID, "unbalanced PUSH/POP");
  return ESC_OK;
}

// ---- lowering: every CMP/RANGE becomes an inclusive range (optionally negated) --------------
// constant atom on non-NULL rows: NOTNULL (true) or FALSE; the user's NOT (K.neg) still applies
void set_const_atom(KInstr& K, bool value_on_nonnull) {
  K.inv = 0;
  K.op = value_on_nonnull ? K_NOTNULL : K_FALSE;
}

// Every CMP/RANGE becomes an inclusive range [lo, hi] in the column's compare domain; "<>" is the
// inverted equality range (inv: applied before the NULL floor, unlike the user's NOT = neg).
void lower_range(const esc_instr_t& I, int dtype, KInstr& K) {
  const bool is_range = I.op == ESC_OP_RANGE;
  const int cmp = I.cmp;
  const bool inv = !is_range && cmp == ESC_CMP_NE;
  K.inv = inv ? 1 : 0;
  if (I.domain == ESC_DOM_I64) {
    long long dmin, dmax;
    if (!dtype_int_range(dtype, &dmin, &dmax)) {  // float column with an int-domain const: compare as f64
      K.op = K_RANGE_F64;
      const double k = (double)I.k0.i;
      K.lo.f = k;
      K.hi.f = is_range ? (double)I.k1.i : k;
      if (!is_range && cmp != ESC_CMP_EQ && cmp != ESC_CMP_NE) {
        K.lo.f = (cmp == ESC_CMP_GT) ? nextafter(k, INFINITY) : (cmp == ESC_CMP_GE) ? k : -INFINITY;
        K.hi.f = (cmp == ESC_CMP_LT) ? nextafter(k, -INFINITY) : (cmp == ESC_CMP_LE) ? k : INFINITY;
      }
      return;
    }
    __int128 lo, hi;
    const __int128 k = I.k0.i;
    if (is_range) {
      lo = I.k0.i;
      hi = I.k1.i;
    } else {
      switch (cmp) {
        case ESC_CMP_EQ: case ESC_CMP_NE: lo = hi = k; break;
        case ESC_CMP_LT: lo = dmin; hi = k - 1; break;
        case ESC_CMP_LE: lo = dmin; hi = k; break;
        case ESC_CMP_GT: lo = k + 1; hi = dmax; break;
        default: lo = k; hi = dmax; break;
      }
    }
    if (lo < dmin) lo = dmin;
    if (hi > dmax) hi = dmax;
    if (lo > hi) return set_const_atom(K, inv);                     // empty range
    if (lo == dmin && hi == dmax) return set_const_atom(K, !inv);  // every value
    K.lo.i = (long long)lo;
    K.hi.i = (long long)hi;
    switch (dtype) {
      case ESC_I8: K.op = K_RANGE_S8; break;
      case ESC_U8: K.op = K_RANGE_U8; break;
      case ESC_I16: K.op = K_RANGE_S16; break;
      case ESC_U16: K.op = K_RANGE_U16; break;
      case ESC_I32: K.op = K_RANGE_S32; break;
      case ESC_U32: K.op = K_RANGE_U32; break;
      default: K.op = K_RANGE_S64; break;
    }
    return;
  }
  // floating domains: strict comparisons become the adjacent representable bound; NaN bounds
  // make every comparison false (and "<>" true), exactly like IEEE compares
  const bool f32 = I.domain == ESC_DOM_F32;
  K.op = (f32 && dtype == ESC_F32) ? K_RANGE_F32 : K_RANGE_F64;  // f32 domain on small ints: exact in f64
  if (is_range) {
    K.lo.f = I.k0.f;
    K.hi.f = I.k1.f;
    return;
  }
  const double k = I.k0.f;
  const double inf = INFINITY;
  switch (cmp) {
    case ESC_CMP_EQ: case ESC_CMP_NE: K.lo.f = K.hi.f = k; break;
    case ESC_CMP_LT:
      if (k == -inf) return set_const_atom(K, false);
      K.lo.f = -inf;
      K.hi.f = f32 ? (double)nextafterf((float)k, -INFINITY) : nextafter(k, -inf);
      break;
    case ESC_CMP_LE: K.lo.f = -inf; K.hi.f = k; break;
    case ESC_CMP_GT:
      if (k == inf) return set_const_atom(K, false);
      K.lo.f = f32 ? (double)nextafterf((float)k, INFINITY) : nextafter(k, inf);
      K.hi.f = inf;
      break;
    default: K.lo.f = k; K.hi.f = inf; break;
  }
}

int lower_program(const esc_program_t* prog, KParams& kp) {
  kp.n_ins = prog->n_instrs;
  for (int i = 0; i < prog->n_instrs; ++i) {
    const esc_instr_t& I = prog->instrs[i];
    KInstr& K = kp.ins[i];
    std::memset(&K, 0, sizeof(K));
    K.combine = I.combine;
    K.neg = I.neg;
    K.col = I.col_a;
    K.col_b = I.col_b;
    K.cmp = I.cmp;
    K.domain = I.domain;
    K.aux = I.aux;
    K.aux2 = I.aux2;
    switch (I.op) {
      case ESC_OP_CMP:
      case ESC_OP_RANGE: lower_range(I, kp.cols[I.col_a].dtype, K); break;
      case ESC_OP_LUT: K.op = K_LUT; break;
      case ESC_OP_COLCMP: K.op = K_COLCMP; break;
      case ESC_OP_NOTNULL: K.op = K_NOTNULL; break;
      case ESC_OP_FALSE: K.op = K_FALSE; break;
      case ESC_OP_UDF: K.op = K_UDF; K.lo.f = I.k0.f; break;
      case ESC_OP_PUSH: K.op = K_PUSH; break;
      case ESC_OP_POP: K.op = K_POP; break;
      default: K.op = K_NOT; break;
    }
  }
  return ESC_OK;
}

#include "esc_jit.cuh"

struct Geometry {
  int chunks = 1;
  int tile_rows = 0;
  int stages = 0;
  uint32_t stage_bytes = 0;  // stage stride (TMA data + compaction regions)
  uint32_t tma_bytes = 0;    // bytes the producer's bulk copies deliver per stage
};

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

// Which columns are staged, the compaction regions, and the tile geometry: the largest C whose
// stage ring still has `min_stages` stages in the smem budget.  For K2 (outs != nullptr) every
// projection gets a per-stage region its warps compact hits into (in place for staged columns,
// scratch filled by gathering only the hit rows otherwise) + a u16 row-index scratch for row-id
// outputs; the stage count is a multiple of the writer-warp count.
Geometry plan_geometry(KParams& kp, const esc_program_t* prog, const esc_column_t* cols, int32_t ncols,
                       bool gather, int64_t nrows, int min_stages, const esc_outputs_t* outs) {
  Geometry g;
  const uint64_t used = program_slots(prog);
  uint32_t per_row = 0;
  for (int i = 0; i < ncols; ++i) {
    KCol& c = kp.cols[i];
    const bool want = ((used >> i) & 1ull) || (cols[i].flags & ESC_COL_STAGE);
    c.staged = want && !gather && (reinterpret_cast<uintptr_t>(c.data) % 16 == 0);
    c.nulls_staged = want && !gather && c.nulls != nullptr && (reinterpret_cast<uintptr_t>(c.nulls) % 16 == 0);
    // count / selection scans stage a packed bitmap when the column has one: N/8 bytes of NULL
    // state instead of N (the one-pass compaction keeps bytes: it copies them out as outputs)
    if (want && !gather && c.nulls != nullptr && outs == nullptr && c.null_bits != nullptr &&
        reinterpret_cast<uintptr_t>(c.null_bits) % 16 == 0)
      c.nulls_staged = 2;
    per_row += (c.staged ? c.width : 0) + (c.nulls_staged == 1 ? 1 : 0);
  }
  // compaction regions (bytes per row of scratch)
  uint32_t scratch_row = 0;
  const bool compact = outs != nullptr && !gather;
  if (compact) {
    for (int k = 0; k < outs->n_proj; ++k) {
      int first = k;
      for (int j = 0; j < k; ++j)
        if (outs->slot[j] == outs->slot[k]) { first = j; break; }
      const KCol& c = kp.cols[outs->slot[k]];
      kp.proj_mode[k] = first != k ? 2 : (c.staged ? 0 : 1);
      if (kp.proj_mode[k] == 1) scratch_row += c.width;
      if (outs->out_nulls[k] == nullptr || c.nulls == nullptr) kp.proj_nmode[k] = 3;
      else if (first != k) kp.proj_nmode[k] = 2;
      else if (c.nulls_staged) kp.proj_nmode[k] = 0;
      else { kp.proj_nmode[k] = 1; scratch_row += 1; }
    }
    if (outs->out_row_ids != nullptr) scratch_row += 2;
  }
  // C = 8 (32 rows per lane) only for count/selection scans: narrow tables need big tiles to
  // stream at full bandwidth; the one-pass compaction packs per-chunk counts in 8-bit fields
  int chunks = compact || outs != nullptr ? 4 : 8;
  while (chunks > 1 &&
         (uint64_t)kConsumerWarps * kChunkRows * chunks * (per_row + scratch_row) * min_stages > kSmemBudget)
    chunks >>= 1;
  // small tables are latency-bound: smaller tiles spread them over more SMs (a 30K-row one-pass
  // compaction: 25 us at C = 4 on 8 CTAs, 17 us at C = 1 on 30)
  {
    const int sms = sm_count_cached() > 0 ? sm_count_cached() : 148;
    while (chunks > 1 && nrows < (int64_t)sms * 2 * kConsumerWarps * kChunkRows * chunks) chunks >>= 1;
  }
  if (const char* e = getenv("ESC_CHUNKS")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4 || (v == 8 && outs == nullptr)) chunks = v;
  }
  const int tile_rows = kConsumerWarps * kChunkRows * chunks;
  bool fast = compact;
  if (fast && (uint64_t)tile_rows * (per_row + scratch_row) * 2 > kSmemBudget) {
    fast = false;  // compaction regions do not fit: consumers scatter directly (slow path)
    scratch_row = 0;
  }
  // if even C=1 cannot hold two stages, drop columns from staging (largest first)
  while ((uint64_t)tile_rows * (per_row + scratch_row) * 2 > kSmemBudget) {
    int best = -1;
    for (int i = 0; i < ncols; ++i)
      if (kp.cols[i].staged && (best < 0 || kp.cols[i].width > kp.cols[best].width)) best = i;
    if (best < 0) break;
    kp.cols[best].staged = 0;
    per_row -= kp.cols[best].width;
    if (kp.cols[best].nulls_staged) {
      if (kp.cols[best].nulls_staged == 1) per_row -= 1;
      kp.cols[best].nulls_staged = 0;
    }
    fast = false;
  }
  g.chunks = chunks;
  g.tile_rows = tile_rows;
  uint32_t off = 0;
  for (int i = 0; i < ncols; ++i) {
    KCol& c = kp.cols[i];
    if (c.staged) { c.smem_off = off; off += (uint32_t)tile_rows * c.width; }
    if (c.nulls_staged) { c.smem_null_off = off; off += c.nulls_staged == 2 ? (uint32_t)tile_rows / 8 : (uint32_t)tile_rows; }
  }
  const uint32_t tma_bytes = off;  // what the producer's bulk copies fill per stage
  if (fast) {
    for (int k = 0; k < outs->n_proj; ++k) {
      const KCol& c = kp.cols[outs->slot[k]];
      int first = k;
      for (int j = 0; j < k; ++j)
        if (outs->slot[j] == outs->slot[k]) { first = j; break; }
      if (kp.proj_mode[k] == 0) kp.proj_off[k] = c.smem_off;
      else if (kp.proj_mode[k] == 1) { kp.proj_off[k] = off; off += (uint32_t)tile_rows * c.width; }
      else kp.proj_off[k] = kp.proj_off[first];
      if (kp.proj_nmode[k] == 0) kp.proj_noff[k] = c.smem_null_off;
      else if (kp.proj_nmode[k] == 1) { kp.proj_noff[k] = off; off += (uint32_t)tile_rows; }
      else if (kp.proj_nmode[k] == 2) kp.proj_noff[k] = kp.proj_noff[first];
    }
    if (outs->out_row_ids != nullptr) {
      off = (off + 15u) & ~15u;
      kp.rows_off = off;
      off += (uint32_t)tile_rows * 2;
    }
    off = (off + 127u) & ~127u;
  }
  kp.all_fast = fast ? 1 : 0;
  g.stage_bytes = off;
  g.tma_bytes = tma_bytes;
  if (tma_bytes == 0 || nrows < tile_rows) {
    g.stages = 2;  // nothing staged (or no full tile): the ring only carries tile ids
    g.stage_bytes = 0;
    g.tma_bytes = 0;
    kp.all_fast = 0;
    for (int i = 0; i < ncols; ++i) kp.cols[i].staged = kp.cols[i].nulls_staged = 0;
  } else {
    g.stages = (int)(kSmemBudget / off);
    if (g.stages > kMaxStages) g.stages = kMaxStages;
    const int max_stages = g.stages;
    // ~96 KB of TMA in flight per SM (at least 3 stages) streams best: a 1-column int32 scan
    // (32 KB stages) runs at 5.9 TB/s with 3 stages and 5.4 TB/s with 6 (tools/stage_sweep.py)
    {
      const int want = (int)((96u * 1024u + off - 1) / off);
      const int cap = want < 3 ? 3 : want;
      if (outs == nullptr && g.stages > cap) g.stages = cap;
    }
    if (const char* e = getenv("ESC_STAGES")) {  // tuning override (experiments only)
      const int v = atoi(e);
      if (v >= 1 && v <= max_stages) g.stages = v;
    }
    if (g.stages < 1) g.stages = 1;
  }
  if (outs != nullptr && g.stages > kMaxWriters) g.stages = kMaxWriters;  // one writer warp per slot
  if (outs != nullptr && g.stages < 2) g.stages = 2;  // K2 holds a stage for its writer warp
  return g;
}

int build_params(KParams& kp, const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                 const int64_t* row_ids, void* d_ws, size_t ws_bytes, esc_result_t* result,
                 const esc_outputs_t* outs) {
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
  for (int i = 0; i < ncols; ++i) {
    const int w = dtype_width(cols[i].dtype);
    if (w == 0) return fail(ESC_ERR_INVALID, "bad column dtype");
    if (cols[i].data == nullptr && nrows > 0) return fail(ESC_ERR_INVALID, "null column data");
    kp.cols[i].data = static_cast<const uint8_t*>(cols[i].data);
    kp.cols[i].nulls = cols[i].nulls;
    kp.cols[i].null_bits = cols[i].null_bits;
    kp.cols[i].dtype = cols[i].dtype;
    kp.cols[i].width = w;
  }
  kp.ncols = ncols;
  kp.nrows = nrows;
  kp.row_ids = row_ids;
  if (outs != nullptr) {
    if (outs->n_proj < 0 || outs->n_proj > ESC_MAX_PROJ) return fail(ESC_ERR_INVALID, "n_proj out of range");
    if (outs->capacity < 0) return fail(ESC_ERR_INVALID, "negative capacity");
    for (int k = 0; k < outs->n_proj; ++k) {
      if (outs->slot[k] < 0 || outs->slot[k] >= ncols) return fail(ESC_ERR_INVALID, "projection slot out of range");
      if (outs->out_values[k] == nullptr && outs->capacity > 0) return fail(ESC_ERR_INVALID, "null output buffer");
    }
    kp.outs = *outs;
  }
  const Geometry g = plan_geometry(kp, prog, cols, ncols, row_ids != nullptr, nrows, 3, outs);
  kp.chunks = g.chunks;
  kp.tile_rows = g.tile_rows;
  kp.stages = g.stages;
  kp.stage_bytes = g.stage_bytes;
  kp.tma_bytes = g.tma_bytes;
  kp.n_tiles = (nrows + g.tile_rows - 1) / g.tile_rows;
  kp.n_full_tiles = (g.tma_bytes == 0) ? 0 : nrows / g.tile_rows;
  {  // K1 tile tickets: >= 128 KB of staged data per ticket, at most 8 tiles
    const int64_t per = g.tma_bytes > 0 ? g.tma_bytes : (int64_t)g.tile_rows * 4;
    int64_t kb = (131072 + per - 1) / per;
    const int sms = sm_count_cached() > 0 ? sm_count_cached() : 148;
    // small and mid scans keep one tile per ticket: >= ~8 tickets per CTA, so the last wave of
    // tickets is short (config 2, 732 tiles: 2-tile tickets left CTAs ending 4 or 6 tiles deep)
    int64_t spread = kp.n_tiles / (8 * (int64_t)sms);
    if (const char* e = getenv("ESC_TICKET_SPREAD")) {  // tuning override (experiments only)
      const int v = atoi(e);
      if (v > 0) spread = kp.n_tiles / ((int64_t)v * sms);
    }
    if (kb > spread) kb = spread;
    kp.ticket_tiles = (int32_t)(kb < 1 ? 1 : (kb > 8 ? 8 : kb));
    // tables whose staged bytes fit comfortably in L2: prefetch them all up front (DRAM ramp)
    const long long staged = (long long)kp.n_full_tiles * g.tma_bytes;
    kp.prefetch_l2 = (staged > 0 && staged <= g_prefetch_max_bytes.load()) ? 1 : 0;
  }
  rc = lower_program(prog, kp);
  if (rc != ESC_OK) return rc;
  // smem offsets into the lowered instructions; fast evaluation needs every program column staged
  const uint64_t used = program_slots(prog);
  kp.all_staged = 1;
  for (int i = 0; i < ncols; ++i)
    if (((used >> i) & 1ull) && (!kp.cols[i].staged || (kp.cols[i].nulls != nullptr && !kp.cols[i].nulls_staged)))
      kp.all_staged = 0;
  for (int i = 0; i < kp.n_ins; ++i) {
    KInstr& K = kp.ins[i];
    const KCol& c = kp.cols[K.col];
    K.soff = c.smem_off;
    K.noff = c.nulls != nullptr ? (c.smem_null_off | (c.nulls_staged == 2 ? kPackedNulls : 0u)) : kNoNulls;
    const KCol& b = kp.cols[K.col_b];
    K.soff_b = b.smem_off;
    K.noff_b = b.nulls != nullptr ? b.smem_null_off : kNoNulls;
  }
  std::memcpy(kp.udfs, prog->udfs, sizeof(kp.udfs));
  std::memcpy(kp.udf_ops, prog->udf_ops, sizeof(kp.udf_ops));
  kp.lut = prog->lut;
  kp.hdr = static_cast<WsHeader*>(d_ws);
  kp.status = status_base(d_ws, ws_bytes, nrows);
  kp.result = result;
  kp.trace = g_trace;
  return ESC_OK;
}

size_t smem_bytes_for(const KParams& kp) {
  return (size_t)kp.stages * kp.stage_bytes + 4 * kMaxStages * sizeof(uint64_t) + kMaxStages * sizeof(long long) +
         kMaxStages * sizeof(unsigned long long) + kConsumerWarps * sizeof(unsigned long long) +
         2 * kMaxStages * kConsumerWarps * sizeof(uint32_t) + kMaxStages * sizeof(uint32_t) +
         2 * sizeof(uint32_t) + sizeof(unsigned long long);  // s_writers_done[2], s_cta_count
}

// A resolved scan launch (kernel, geometry, cooperative flag): prepared once, issued any number
// of times with the same KParams (esc_step_plan_* re-issues it without rebuilding anything).
struct ScanLaunch {
  const void* func = nullptr;  // JIT cudaKernel_t or the ahead-of-time interpreter instantiation
  unsigned grid = 1;
  unsigned block = 0;
  size_t smem = 0;
  bool coop = false;
};

template <int C, bool COMPACT>
int prepare_c(const KParams& kp, ScanLaunch* L) {
  const size_t smem = smem_bytes_for(kp);
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t grid = kp.n_tiles < sms ? kp.n_tiles : sms;
  if (grid < 1) grid = 1;
  L->grid = (unsigned)grid;
  L->block = Layout<COMPACT>::kThreads;
  L->smem = smem;
  L->coop = COMPACT;  // the one-pass look-back relies on every CTA being resident
  // JIT tier: large scans whose tiles run the fast (staged) evaluator
  const int mode = jit::g_mode.load();
  if (mode == 2 || (mode == 1 && kp.nrows >= jit::g_min_rows.load())) {
    if (kp.all_staged && kp.n_full_tiles > 0) {
      std::string why;
      cudaKernel_t k = jit::get_kernel(kp, COMPACT, smem, &why);
      if (k != nullptr) {
        L->func = reinterpret_cast<const void*>(k);
        return ESC_OK;
      }
    }
  }
  auto kern = esc_scan_kernel<C, COMPACT, InterpPred>;
  static std::atomic<size_t> configured{0};
  if (smem > configured.load()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    configured = smem;
  }
  L->func = reinterpret_cast<const void*>(kern);
  return ESC_OK;
}

int issue_scan(const ScanLaunch& L, const KParams& kp, cudaStream_t stream) {
  void* args[] = {const_cast<KParams*>(&kp)};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(L.block);
  cfg.dynamicSmemBytes = L.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = L.coop ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  cudaError_t e = cudaLaunchKernelExC(&cfg, L.func, args);
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

template <bool COMPACT>
int prepare(const KParams& kp, ScanLaunch* L) {
  switch (kp.chunks) {
    case 8:
      if constexpr (!COMPACT) return prepare_c<8, false>(kp, L);
      return fail(ESC_ERR_INVALID, "internal: C=8 tiles are for count/selection scans only");
    case 4: return prepare_c<4, COMPACT>(kp, L);
    case 2: return prepare_c<2, COMPACT>(kp, L);
    default: return prepare_c<1, COMPACT>(kp, L);
  }
}

template <bool COMPACT>
int launch(const KParams& kp, cudaStream_t stream) {
  ScanLaunch L;
  const int rc = prepare<COMPACT>(kp, &L);
  return rc != ESC_OK ? rc : issue_scan(L, kp, stream);
}

// ---- streamed compaction of dense tiles ------------------------------------------------------
// A stream tile is dense when it holds at least tile_rows / ESC_STREAM_DIV hits (default 32: one
// hit per bitmap word on average, ~3% selectivity): from there on, reading the tile's projected
// columns whole through TMA beats sector-granular gathers of the hit rows.
std::atomic<int> g_stream_div{[] {
  const char* e = getenv("ESC_STREAM_DIV");
  return e ? atoi(e) : 32;
}()};

// selections over at most this many rows compact with ONE sel_mid_kernel launch (ESC_MID_MAX_ROWS;
// 0 turns it off): below it the chain's launch + ramp costs dominate, above it the streamed
// (TMA) compaction of dense tiles reads less than per-hit gathers
// early start of the mid-size compaction on the scan's completion flag (ESC_MID_EARLY=0: PDL wait)
std::atomic<int> g_mid_early{[] {
  const char* e = getenv("ESC_MID_EARLY");
  return e ? atoi(e) : 1;
}()};
// lean selection bitmaps in step plans (ESC_BITMAP_LEAN=0: every segment's words written)
std::atomic<int> g_bitmap_lean{[] {
  const char* e = getenv("ESC_BITMAP_LEAN");
  return e ? atoi(e) : 1;
}()};
// warp hit lists in the gathered compaction (ESC_HIT_LISTS: 0 off, 1 auto = sparse selections of
// tables whose segment groups fill the GPU, 2 always)
std::atomic<int> g_hit_lists{[] {
  const char* e = getenv("ESC_HIT_LISTS");
  return e ? atoi(e) : 1;
}()};
std::atomic<long long> g_mid_max_rows{[] {
  const char* e = getenv("ESC_MID_MAX_ROWS");
  return e ? atoll(e) : (32ll << 20);
}()};

uint32_t stream_dense_min(int tile_rows) {
  const int div = g_stream_div.load();
  if (div <= 0) return 0xFFFFFFFFu;  // streaming off
  const uint32_t m = (uint32_t)(tile_rows / div);
  return m > 0 ? m : 1u;
}

// Stage layout of sel_stream_kernel; false when streaming does not apply (row-id chaining, an
// unaligned column, nothing fits).  Tiles of 8 segments shrink to 4 or 2 until >= 3 stages fit.
bool plan_stream(StreamParams& tp, const SelParams& sp, const esc_column_t* cols, const esc_outputs_t* outs,
                 const esc_selection_t* sel, int64_t nrows, const int64_t* d_row_ids) {
  std::memset(&tp, 0, sizeof(tp));
  if (d_row_ids != nullptr || nrows <= 0) return false;
  if (stream_dense_min(1 << 20) == 0xFFFFFFFFu) return false;
  if (reinterpret_cast<uintptr_t>(sel->bitmap) % 16 != 0) return false;
  uint32_t per_row = 0;
  for (int k = 0; k < outs->n_proj; ++k) {
    const esc_column_t& c = cols[outs->slot[k]];
    const int w = dtype_width(c.dtype);
    if (reinterpret_cast<uintptr_t>(c.data) % 16 != 0) return false;
    const bool want_nulls = outs->out_nulls[k] != nullptr && c.nulls != nullptr;
    if (want_nulls && reinterpret_cast<uintptr_t>(c.nulls) % 16 != 0) return false;
    per_row += w + (want_nulls ? 1 : 0);
  }
  tp.seg_rows = sel->seg_rows;
  int spt = kConsumerWarps < 8 ? kConsumerWarps : 8;  // the dense-tile rule handles 2, 4 or 8 segments
  auto stage_for = [&](int s) {
    const uint32_t rows = (uint32_t)s * (uint32_t)tp.seg_rows;
    uint32_t b = rows / 8;                 // bitmap words
    b = (b + 15u) & ~15u;
    b += 64;                               // <= 8 segment offsets
    for (int k = 0; k < outs->n_proj; ++k) {
      const esc_column_t& c = cols[outs->slot[k]];
      b += rows * dtype_width(c.dtype);
      if (outs->out_nulls[k] != nullptr && c.nulls != nullptr) b += rows;
      b = (b + 15u) & ~15u;
    }
    return (b + 127u) & ~127u;
  };
  const int W = tp.seg_rows / 32;
  auto warps_ok = [&](int s) { return kStreamConsumers / s <= W; };  // >= 1 word per consumer warp
  // >= 3 stages in the ring, unless at most ~1/3 of the rows can be written (the output capacity
  // bounds it): then the consumers' fixed cost per tile dominates and twice-larger tiles in two
  // stages stream faster (600M-row config-5 shape, s = 0.05-0.3: 2.71 -> 2.48 ms; at s = 0.5 the
  // two stages lose, 3.33 -> 3.64 ms; tools/diag_stream_ab.py)
  const int min_stages = outs->capacity <= nrows / 3 ? 2 : 3;
  while (spt > 2 && warps_ok(spt >> 1) && stage_for(spt) * min_stages > kSmemBudget) spt >>= 1;
  if (const char* e = getenv("ESC_STREAM_SPT")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if ((v == 2 || v == 4 || v == 8) && warps_ok(v)) spt = v;
  }
  if (!warps_ok(spt) || stage_for(spt) * 2 > kSmemBudget) return false;
  (void)per_row;
  tp.segs_per_tile = spt;
  tp.tile_rows = spt * tp.seg_rows;
  const uint32_t rows = (uint32_t)tp.tile_rows;
  uint32_t off = 0;
  tp.off_bitmap = off;
  off += (rows / 8 + 15u) & ~15u;
  tp.off_offsets = off;
  off += 64;
  tp.tma_bytes = rows / 8 + (uint32_t)spt * 8;
  tp.meta_bytes = tp.tma_bytes;
  tp.n_proj = outs->n_proj;
  for (int k = 0; k < outs->n_proj; ++k) {
    const esc_column_t& c = cols[outs->slot[k]];
    const int w = dtype_width(c.dtype);
    tp.width[k] = w;
    tp.data[k] = static_cast<const uint8_t*>(c.data);
    tp.off_val[k] = off;
    off += rows * w;
    off = (off + 15u) & ~15u;
    tp.tma_bytes += rows * w;
    if (outs->out_nulls[k] != nullptr && c.nulls != nullptr) {
      tp.nulls[k] = c.nulls;
      tp.off_null[k] = off;
      off += rows;
      off = (off + 15u) & ~15u;
      tp.tma_bytes += rows;
    }
  }
  // the consumers' byte streams, grouped by width (8, 4, 2, 1)
  int ns = 0;
  for (int c = 0; c < 4; ++c) {
    tp.cls[c] = ns;
    const int cw = 8 >> c;
    for (int k = 0; k < outs->n_proj; ++k) {
      if (tp.width[k] == cw) {
        tp.s_off[ns] = tp.off_val[k];
        tp.s_src[ns] = tp.data[k];
        tp.s_dst[ns++] = static_cast<uint8_t*>(outs->out_values[k]);
      }
      if (cw == 1 && tp.nulls[k] != nullptr) {
        tp.s_off[ns] = tp.off_null[k];
        tp.s_src[ns] = tp.nulls[k];
        tp.s_dst[ns++] = outs->out_nulls[k];
      }
    }
  }
  tp.cls[4] = ns;
  tp.n_zero = 0;
  for (int k = 0; k < outs->n_proj; ++k)
    if (outs->out_nulls[k] != nullptr && tp.nulls[k] == nullptr) tp.zero_dst[tp.n_zero++] = outs->out_nulls[k];
  tp.stage_bytes = (off + 127u) & ~127u;
  tp.stages = (int)(kSmemBudget / tp.stage_bytes);
  if (tp.stages > kMaxStages) tp.stages = kMaxStages;
  if (const char* e = getenv("ESC_STREAM_STAGES")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if (v >= 2 && v < tp.stages) tp.stages = v;
  }
  tp.consumers = kStreamConsumers;
  if (const char* e = getenv("ESC_STREAM_WARPS")) {  // tuning override (experiments only)
    const int v = atoi(e);
    if ((v == 4 || v == 8 || v == 16) && v / spt >= 1 && v / spt <= W) tp.consumers = v;
  }
  (void)sp;
  return tp.stages >= 2;
}

// ---- selection compaction: prepared once, issued any number of times ---------------------------
struct MatLaunch {
  SelParams sp;
  StreamParams tp;
  MidParams mp;
  bool mid = false;        // one sel_mid_kernel launch instead of the scan + compaction chain
  bool hit_list = false;   // sel_compact_kernel<true>: sparse hits gathered through warp hit lists
  size_t mid_smem = 0;
  bool streaming = false;
  bool empty = true;
  unsigned segs = 0;
  const uint32_t* seg_counts = nullptr;
  unsigned long long* partials = nullptr;
  unsigned long long* offsets = nullptr;
  size_t stream_smem = 0;
  unsigned stream_grid = 1;
  unsigned compact_grid = 1;
};

int prepare_mat(const esc_selection_t* sel, int64_t nrows, const esc_column_t* cols, int32_t ncols,
                const int64_t* d_row_ids, const esc_outputs_t* outs, void* d_ws, size_t ws_bytes, MatLaunch* M) {
  SelParams& sp = M->sp;
  if (sel == nullptr || sel->bitmap == nullptr || sel->seg_counts == nullptr || outs == nullptr)
    return fail(ESC_ERR_INVALID, "null selection argument");
  if (nrows < 0 || ncols < 0 || ncols > ESC_MAX_COLS) return fail(ESC_ERR_INVALID, "bad sizes");
  if (sel->seg_rows <= 0 || sel->seg_rows % 128 != 0 || sel->seg_rows > 1024)
    return fail(ESC_ERR_INVALID, "selection was not filled by esc_scan_select");
  if (outs->n_proj < 0 || outs->n_proj > ESC_MAX_PROJ || outs->capacity < 0)
    return fail(ESC_ERR_INVALID, "bad outputs");
  const WsLayout L = ws_layout(nrows);
  if (d_ws == nullptr || ws_bytes < L.total) return fail(ESC_ERR_WORKSPACE, "workspace too small");
  M->mid = false;  // M may be a reused (thread-local) launch: every route flag is re-decided here
  M->hit_list = false;
  M->streaming = false;
  M->empty = true;
  std::memset(&sp, 0, sizeof(sp));
  sp.bitmap = sel->bitmap;
  sp.seg_counts = sel->seg_counts;
  sp.row_ids = d_row_ids;
  sp.nrows = nrows;
  sp.seg_rows = sel->seg_rows;
  sp.cap_per_seg = sel->cap_per_seg;
  sp.cap_stride = sel->cap_stride;
  // segments cover whole tiles: tile = kConsumerWarps segments
  const int64_t tile_rows = (int64_t)sel->seg_rows * kConsumerWarps;
  sp.n_segs = ((nrows + tile_rows - 1) / tile_rows) * kConsumerWarps;
  sp.n_proj = outs->n_proj;
  sp.need_bitmap_captured = outs->out_row_ids != nullptr;
  for (int k = 0; k < outs->n_proj; ++k) {
    if (outs->slot[k] < 0 || outs->slot[k] >= ncols) return fail(ESC_ERR_INVALID, "projection slot out of range");
    const esc_column_t& c = cols[outs->slot[k]];
    const int w = dtype_width(c.dtype);
    if (w == 0) return fail(ESC_ERR_INVALID, "bad column dtype");
    if (outs->out_values[k] == nullptr && outs->capacity > 0) return fail(ESC_ERR_INVALID, "null output buffer");
    sp.cols[k].data = static_cast<const uint8_t*>(c.data);
    sp.cols[k].nulls = c.nulls;
    sp.cols[k].dtype = c.dtype;
    sp.cols[k].width = w;
    sp.cap_index[k] = -1;
    for (int j = 0; j < sel->n_cap; ++j)
      if (sel->cap_slot[j] == outs->slot[k] && (outs->out_nulls[k] == nullptr || c.nulls == nullptr ||
                                                sel->cap_nulls[j] != nullptr)) {
        sp.cap_index[k] = j;
        sp.cap_values[j] = sel->cap_values[j];
        sp.cap_nulls[j] = sel->cap_nulls[j];
        break;
      }
    if (sp.cap_index[k] < 0) sp.need_bitmap_captured = 1;
  }
  sp.outs = *outs;
  M->empty = sp.n_segs == 0;
  if (M->empty) return ESC_OK;
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  M->offsets = reinterpret_cast<unsigned long long*>(ws + L.offsets);
  M->partials = reinterpret_cast<unsigned long long*>(ws + L.partials);
  M->seg_counts = sel->seg_counts;
  sp.seg_offsets = M->offsets;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  sp.rule.dense_min = 0xFFFFFFFFu;
  sp.rule.skip_count = nullptr;
  sp.rule.skip_capacity = outs->capacity;
  if (outs->flags & ESC_OUT_SKIP_OVER_CAPACITY) {
    if (sel->d_count == nullptr && sel->d_gate == nullptr)
      return fail(ESC_ERR_INVALID, "ESC_OUT_SKIP_OVER_CAPACITY needs sel->d_count or sel->d_gate");
    sp.rule.skip_count = reinterpret_cast<const unsigned long long*>(sel->d_gate != nullptr ? sel->d_gate
                                                                                             : sel->d_count);
  }
  // mid-size selections: ONE kernel (sel_mid_kernel) — offsets and compaction without the chain —
  // when the output can hold at most a quarter of the rows (an ESC step's capacity is the push-down
  // threshold, 20% by default; an exact materialisation's is its count): it gathers hit by hit,
  // which beats the chain up to ~10-20% density and loses to the chain's TMA-streamed dense tiles
  // beyond (tools/diag_mid_sweep.py: 4M-48M rows, s = 0.001 .. 0.5)
  const long long mid_max = g_mid_max_rows.load();  // >= 2^40: forced for every size and density (tests)
  if (nrows <= mid_max && (outs->capacity <= nrows / 4 || mid_max >= (1ll << 40))) {
    static const int mid_resident = [] {
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sel_mid_kernel, kMidThreads, 4096);
      return b > 0 ? b : 4;
    }();
    const int64_t target = (int64_t)sms * mid_resident;
    int64_t spb = (sp.n_segs + target - 1) / target;
    if (spb < 1) spb = 1;
    if ((sp.n_segs + spb - 1) / spb > kMidMaxBlocks) spb = (sp.n_segs + kMidMaxBlocks - 1) / kMidMaxBlocks;
    if (spb * sel->seg_rows < (1ll << 31) && spb <= 4096) {
      MidParams& mp = M->mp;
      std::memset(&mp, 0, sizeof(mp));
      mp.segs_per_block = (int32_t)spb;
      mp.n_blocks = (sp.n_segs + spb - 1) / spb;
      uint8_t* ws = static_cast<uint8_t*>(d_ws);
      mp.agg = reinterpret_cast<unsigned long long*>(ws + L.mid);  // fixed place: zero between launches
      mp.trace = g_trace;
      WsHeader* hdr = static_cast<WsHeader*>(d_ws);
      mp.ticket = &hdr->mid_ticket;
      mp.done = &hdr->mid_done;
      M->mid = true;
      M->mid_smem = (size_t)spb * sizeof(uint32_t);
      return ESC_OK;
    }
  }
  // dense stream tiles (no row-id chaining: the staged tile must be the physical rows)
  StreamParams& tp = M->tp;
  M->streaming = plan_stream(tp, sp, cols, outs, sel, nrows, d_row_ids);
  sp.rule.segs_per_tile = 8;
  sp.rule.n_tiles = 0;
  sp.rule.n_dense = reinterpret_cast<uint32_t*>(ws + L.dense);
  sp.rule.dense_list = reinterpret_cast<uint32_t*>(ws + L.dense + 256);
  if (M->streaming) {
    sp.rule.dense_min = stream_dense_min(tp.tile_rows);
    sp.rule.segs_per_tile = tp.segs_per_tile;
    sp.rule.n_tiles = (nrows + tp.tile_rows - 1) / tp.tile_rows;
    tp.n_full_tiles = nrows / tp.tile_rows;
    tp.dense_list = sp.rule.dense_list;
    tp.n_dense = sp.rule.n_dense;
    tp.bitmap = sel->bitmap;
    tp.seg_offsets = M->offsets;
    tp.outs = *outs;
    M->stream_smem = (size_t)tp.stages * tp.stage_bytes + 2 * kMaxStages * sizeof(uint64_t) +
                     kMaxStages * sizeof(long long);
    static std::atomic<size_t> configured{0};
    if (M->stream_smem > configured.load()) {
      cudaError_t e = cudaFuncSetAttribute(sel_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)M->stream_smem);
      if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      configured = M->stream_smem;
    }
    const int64_t tiles = sp.rule.n_tiles;
    M->stream_grid = (unsigned)(tiles < sms ? (tiles > 0 ? tiles : 1) : sms);
  }
  M->segs = (unsigned)((sp.n_segs + kScanSeg - 1) / kScanSeg);
  // phase A: 32 segments per warp; when those groups alone give every SM 4+ CTAs, phase A also
  // writes the sparse segments; otherwise phase B spreads 128-row chunks (32 per warp)
  const int64_t groups_ctas = (sp.n_segs + 32 * kSelWarps - 1) / (32 * kSelWarps);
  const int hl_mode = g_hit_lists.load();
  sp.sparse_in_a = (groups_ctas >= 4LL * sms || hl_mode == 2) ? 1 : 0;
  const int64_t chunks = sp.n_segs * (sp.seg_rows / kChunkRows);
  const int64_t want = sp.sparse_in_a ? groups_ctas : (chunks + 32 * kSelWarps - 1) / (32 * kSelWarps);
  // warp hit lists for sparse selections (capacity <= 1 row in 500): a few hits per 32 segments,
  // so lanes gathering their own chunk's hits would leave most of the warp idle (config-5 shape,
  // 600M rows: s = 1e-4 98 -> 52 us, 1e-3 170 -> 141 us; at 3e-3 the lanes win, 228 vs 262 us)
  M->hit_list = nrows < (1ll << 31) && (hl_mode == 2 || (hl_mode == 1 && sp.sparse_in_a && outs->capacity * 500 <= nrows));
  // one wave of resident CTAs: warps loop over groups with the next group's loads in flight
  static const int resident_lanes = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sel_compact_kernel<false>, kSelWarps * 32, 0);
    return b > 0 ? b : 4;
  }();
  static const int resident_list = [] {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sel_compact_kernel<true>, kSelWarps * 32, 0);
    return b > 0 ? b : 3;
  }();
  const int resident = M->hit_list ? resident_list : resident_lanes;
  const int64_t cap_grid = (int64_t)sms * resident;
  M->compact_grid = (unsigned)(want < cap_grid ? want : cap_grid);
  sp.a_split = 1;
  if (!sp.sparse_in_a) {
    const int64_t groups = (sp.n_segs + 31) / 32, warps = (int64_t)M->compact_grid * kSelWarps;
    while (sp.a_split < 8 && groups * sp.a_split * 2 <= warps) sp.a_split *= 2;
  }
  return ESC_OK;
}

// launch with programmatic stream serialization (the kernel waits for its predecessor itself)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int issue_mat(const MatLaunch& M, cudaStream_t st) {
  if (M.empty) return ESC_OK;
  const SelParams& sp = M.sp;
  if (M.mid) {
    cudaError_t e = launch_pdl(sel_mid_kernel, (unsigned)M.mp.n_blocks, kMidThreads, M.mid_smem, st, sp, M.mp);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("mid-size compaction launch: ") + cudaGetErrorString(e));
    return ESC_OK;
  }
  cudaError_t e = launch_pdl(tile_scan_partials, M.segs, kScanThreads, 0, st, M.seg_counts, sp.n_segs, M.partials,
                             sp.rule.n_dense, sp.rule.skip_count, sp.rule.skip_capacity);
  if (e == cudaSuccess)
    e = launch_pdl(tile_scan_apply, M.segs, kScanThreads, 0, st, M.seg_counts, sp.n_segs,
                   static_cast<const unsigned long long*>(M.partials), M.offsets, sp.rule);
  if (e == cudaSuccess && M.streaming)
    e = launch_pdl(sel_stream_kernel, M.stream_grid, (1 + M.tp.consumers) * 32, M.stream_smem, st, M.tp);
  if (e == cudaSuccess)
    e = M.hit_list ? launch_pdl(sel_compact_kernel<true>, M.compact_grid, kSelWarps * 32, 0, st, sp)
                   : launch_pdl(sel_compact_kernel<false>, M.compact_grid, kSelWarps * 32, 0, st, sp);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("selection compaction launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

size_t esc_workspace_bytes(int64_t nrows) { return ws_layout(nrows).total; }

int esc_selection_sizes(int64_t nrows, int64_t* bitmap_words, int64_t* max_segments, int64_t* cap_entries) {
  const WsLayout L = ws_layout(nrows);
  if (bitmap_words) *bitmap_words = L.bitmap_words;
  if (max_segments) *max_segments = L.max_tiles;
  // capture slots: 4*C per segment of 128*C rows (C <= 4), i.e. n/32 plus the tail tile's slack
  if (cap_entries) *cap_entries = (nrows < 0 ? 0 : nrows) / 32 + 4 * 4 * (int64_t)kConsumerWarps * 2;
  return ESC_OK;
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
  g_epochs[d_ws] = EpochState();
  return ESC_OK;
}

int esc_scan_count(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                   const int64_t* d_row_ids, esc_result_t* result, void* d_ws, size_t ws_bytes, void* stream) {
  static thread_local KParams kp;
  int rc = build_params(kp, prog, cols, ncols, nrows, d_row_ids, d_ws, ws_bytes, result, nullptr);
  if (rc != ESC_OK) return rc;
  return launch<false>(kp, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {
int prepare_select(KParams& kp, const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                   const int64_t* d_row_ids, esc_selection_t* sel, esc_result_t* result, void* d_ws,
                   size_t ws_bytes) {
  if (sel == nullptr || sel->bitmap == nullptr || sel->seg_counts == nullptr)
    return fail(ESC_ERR_INVALID, "null selection output");
  if (sel->n_cap < 0 || sel->n_cap > ESC_MAX_PROJ) return fail(ESC_ERR_INVALID, "n_cap out of range");
  for (int k = 0; k < sel->n_cap; ++k)
    if (sel->cap_slot[k] < 0 || sel->cap_slot[k] >= ncols || sel->cap_values[k] == nullptr)
      return fail(ESC_ERR_INVALID, "bad capture slot / buffer");
  int rc = build_params(kp, prog, cols, ncols, nrows, d_row_ids, d_ws, ws_bytes, result, nullptr);
  if (rc != ESC_OK) return rc;
  sel->seg_rows = kChunkRows * kp.chunks;
  sel->cap_per_seg = 4 * kp.chunks;  // segments with <= 4*C hits (~3% of 128*C rows) are captured
  if (kp.chunks > 4) sel->cap_per_seg = 0;  // (no capture with C = 8 tiles)
  const int64_t n_segs = kp.n_tiles * kConsumerWarps;
  if (n_segs > INT32_MAX) sel->cap_per_seg = 0;  // slot-major index would overflow the stride
  sel->cap_stride = (int32_t)(n_segs > INT32_MAX ? 0 : n_segs);
  kp.sel_on = 1;
  kp.sel = *sel;
  return ESC_OK;
}

// A queued ESC step (esc_step_plan_*): the scan and the compaction fully prepared.
struct StepPlanImpl {
  KParams kp;
  ScanLaunch scan;
  MatLaunch mat;
  bool onepass = false;  // one launch of the look-back kernel (no selection, no queued compaction)
  bool scan_pending = false;  // part 1 issued, its part 2 not yet (early-start compactions)
  // queued plans: the launches of parts 1, 2 and 3 captured once into CUDA graphs (their
  // parameters never change), so a re-issue is one graph launch instead of up to five kernel
  // launches with kilobytes of parameters each
  cudaGraphExec_t graph[4] = {nullptr, nullptr, nullptr, nullptr};
  int graph_kernels[4] = {0, 0, 0, 0};
  bool graph_failed[4] = {false, false, false, false};
  ~StepPlanImpl() {
    for (auto& g : graph)
      if (g != nullptr) cudaGraphExecDestroy(g);
  }
};

std::atomic<int> g_graphs{[] {
  const char* e = getenv("ESC_GRAPHS");  // 0 turns the step-plan graphs off (experiments)
  return e ? atoi(e) : 1;
}()};

// issue a queued plan's parts on `st` directly
int issue_parts(StepPlanImpl* p, int parts, cudaStream_t st) {
  int rc = (parts & 1) ? issue_scan(p->scan, p->kp, st) : ESC_OK;
  return (rc != ESC_OK || !(parts & 2)) ? rc : issue_mat(p->mat, st);
}

// capture a queued plan's parts into an executable graph (on a private stream, thread-local
// capture mode); false leaves the plan on direct launches
bool capture_parts(StepPlanImpl* p, int parts) {
  cudaStream_t cs = nullptr;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return false;
  const long long before = g_launches.load();
  bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  const int rc = ok ? issue_parts(p, parts, cs) : ESC_ERR_CUDA;
  cudaGraph_t g = nullptr;
  const cudaError_t e = ok ? cudaStreamEndCapture(cs, &g) : cudaErrorUnknown;
  ok = ok && rc == ESC_OK && e == cudaSuccess && g != nullptr;
  cudaGraphExec_t x = nullptr;
  if (ok) ok = cudaGraphInstantiate(&x, g, 0) == cudaSuccess;
  if (g != nullptr) cudaGraphDestroy(g);
  cudaStreamDestroy(cs);
  cudaGetLastError();  // a failed capture must not leave a sticky launch error behind
  const long long issued = g_launches.load() - before;
  g_launches -= issued;  // captured, not launched: counted per graph launch instead
  if (!ok) return false;
  p->graph[parts] = x;
  p->graph_kernels[parts] = (int)issued;
  return true;
}

// next look-back epoch of a workspace (status words carry it, so they need no clearing per launch)
int next_epoch(KParams& kp, int64_t nrows, void* d_ws, cudaStream_t stream) {
  std::lock_guard<std::mutex> g(g_epoch_mu);
  EpochState& es = g_epochs[d_ws];
  const size_t words = status_words(nrows);
  if (words > es.max_words) es.max_words = words;
  es.epoch = (es.epoch + 1) & 0xFFFFu;
  if (es.epoch == 0) {
    // epoch wrapped: a word left by ANY earlier one-pass launch on this workspace (of any table
    // size: they all end at the workspace's end) could alias the new epoch — clear all of them
    unsigned long long* end = kp.status + words;
    cudaError_t e = cudaMemsetAsync(end - es.max_words, 0, es.max_words * sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("status clear: ") + cudaGetErrorString(e));
    es.epoch = 1;
  }
  kp.epoch = es.epoch;
  return ESC_OK;
}
}  // namespace

extern "C" {

int esc_scan_select(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                    const int64_t* d_row_ids, esc_selection_t* sel, esc_result_t* result, void* d_ws,
                    size_t ws_bytes, void* stream) {
  static thread_local KParams kp;
  int rc = prepare_select(kp, prog, cols, ncols, nrows, d_row_ids, sel, result, d_ws, ws_bytes);
  return rc != ESC_OK ? rc : launch<false>(kp, static_cast<cudaStream_t>(stream));
}

int esc_step_plan_create(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                         esc_selection_t* sel, const esc_column_t* mat_cols, int32_t mat_ncols,
                         const esc_outputs_t* outs, esc_result_t* result, void* d_ws, size_t ws_bytes,
                         void** out_plan) {
  if (out_plan == nullptr) return fail(ESC_ERR_INVALID, "null plan output");
  *out_plan = nullptr;
  StepPlanImpl* plan = new (std::nothrow) StepPlanImpl();
  if (plan == nullptr) return fail(ESC_ERR_INVALID, "out of host memory");
  if (sel == nullptr) {  // one-pass plan: the look-back kernel compacts `outs` directly
    if (outs == nullptr) {
      delete plan;
      return fail(ESC_ERR_INVALID, "null outputs");
    }
    int rc = build_params(plan->kp, prog, cols, ncols, nrows, nullptr, d_ws, ws_bytes, result, outs);
    if (rc == ESC_OK) rc = prepare<true>(plan->kp, &plan->scan);
    if (rc != ESC_OK) {
      delete plan;
      return rc;
    }
    plan->onepass = true;
    *out_plan = plan;
    return ESC_OK;
  }
  int rc = prepare_select(plan->kp, prog, cols, ncols, nrows, nullptr, sel, result, d_ws, ws_bytes);
  if (rc == ESC_OK) rc = prepare<false>(plan->kp, &plan->scan);
  if (rc == ESC_OK) rc = prepare_mat(sel, nrows, mat_cols, mat_ncols, nullptr, outs, d_ws, ws_bytes, &plan->mat);
  if (rc != ESC_OK) {
    delete plan;
    return rc;
  }
  // the plan's selection lives only for its own compaction: when that reads no bitmap for
  // captured segments (every projection captured, no row ids), K1 skips the bitmap words of
  // captured and empty segments and the dense-tile rule keeps their tiles off the streamed path
  if (!plan->mat.empty && !plan->mat.sp.need_bitmap_captured && sel->n_cap > 0 && g_bitmap_lean.load()) {
    plan->kp.bitmap_lean = 1;
    plan->mat.sp.rule.lean = 1;
  }
  // a mid-size compaction in the same plan as its scan starts on the scan's completion flag (set
  // by its last CTA) instead of the grid's completion
  if (plan->mat.mid && !plan->mat.empty && g_mid_early.load()) {
    auto* flag = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(d_ws) + sizeof(WsHeader));
    plan->kp.scan_done = flag;
    plan->mat.mp.scan_done = flag;
  }
  *out_plan = plan;
  return ESC_OK;
}

int esc_step_plan_launch(void* plan, int32_t parts, void* stream) {
  if (plan == nullptr) return fail(ESC_ERR_INVALID, "null plan");
  const bool force_graph = (parts & ESC_PLAN_GRAPH) != 0;
  parts &= ~ESC_PLAN_GRAPH;
  if (parts < 1 || parts > 3) return fail(ESC_ERR_INVALID, "parts must be 1 (scan), 2 (compaction) or 3");
  StepPlanImpl* p = static_cast<StepPlanImpl*>(plan);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  p->kp.trace = g_trace;
  if (p->onepass) {
    const int rc = next_epoch(p->kp, p->kp.nrows, p->kp.hdr, st);
    return rc != ESC_OK ? rc : issue_scan(p->scan, p->kp, st);
  }
  if (p->mat.mp.scan_done != nullptr) {  // an early-start compaction follows its own scan only
    if (parts == 2 && !p->scan_pending) return fail(ESC_ERR_INVALID, "compaction part issued without its scan");
    p->scan_pending = parts == 1;
  }
  // graphs for whole steps, or for a part when asked (ESC_PLAN_GRAPH): the profiling split
  // (parts 1 / 2 with events between) launches directly — as two graphs it measured 30-40 us
  // longer on a 6M-row table, since the PDL overlap of the scan and the compaction chain does not
  // cross graph boundaries; the multi-GPU step, whose count exchange sits between the parts
  // anyway, asks for graphs (no kilobyte parameter blocks marshalled per launch)
  if ((parts == 3 || force_graph) && g_graphs.load() && g_trace == nullptr && !p->graph_failed[parts]) {
    if (p->graph[parts] == nullptr && !capture_parts(p, parts)) {
      p->graph_failed[parts] = true;
      return issue_parts(p, parts, st);
    }
    const cudaError_t e = cudaGraphLaunch(p->graph[parts], st);
    if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("step graph launch: ") + cudaGetErrorString(e));
    g_launches += p->graph_kernels[parts];
    return ESC_OK;
  }
  return issue_parts(p, parts, st);
}

int esc_step_plan_rebind(void* plan, const esc_outputs_t* outs) {
  if (plan == nullptr || outs == nullptr) return fail(ESC_ERR_INVALID, "null plan or outputs");
  StepPlanImpl* p = static_cast<StepPlanImpl*>(plan);
  if (!p->onepass) return fail(ESC_ERR_INVALID, "only one-pass plans take new outputs");
  const esc_outputs_t& o = p->kp.outs;
  bool same = outs->n_proj == o.n_proj && outs->capacity == o.capacity && outs->flags == o.flags &&
              (outs->out_row_ids == nullptr) == (o.out_row_ids == nullptr);
  for (int k = 0; same && k < o.n_proj; ++k)
    same = outs->slot[k] == o.slot[k] && (outs->out_nulls[k] == nullptr) == (o.out_nulls[k] == nullptr) &&
           (outs->out_values[k] == nullptr) == (o.out_values[k] == nullptr);
  if (!same) return fail(ESC_ERR_INVALID, "outputs differ in shape from the plan's");
  p->kp.outs = *outs;
  return ESC_OK;
}

int esc_step_plan_destroy(void* plan) {
  delete static_cast<StepPlanImpl*>(plan);
  return ESC_OK;
}

int esc_materialize_selection(const esc_selection_t* sel, int64_t nrows, const esc_column_t* cols, int32_t ncols,
                              const int64_t* d_row_ids, const esc_outputs_t* outs, void* d_ws, size_t ws_bytes,
                              void* stream) {
  static thread_local MatLaunch M;
  const int rc = prepare_mat(sel, nrows, cols, ncols, d_row_ids, outs, d_ws, ws_bytes, &M);
  return rc != ESC_OK ? rc : issue_mat(M, static_cast<cudaStream_t>(stream));
}

int esc_compact(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                const int64_t* d_row_ids, const esc_outputs_t* outs, esc_result_t* result, void* d_ws,
                size_t ws_bytes, void* stream) {
  // K1 with selection outputs into the workspace, then the bitmap compaction (no look-back)
  if (outs == nullptr) return fail(ESC_ERR_INVALID, "null outputs");
  const WsLayout L = ws_layout(nrows);
  if (d_ws == nullptr || ws_bytes < L.total) return fail(ESC_ERR_WORKSPACE, "workspace too small");
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  esc_selection_t sel;
  std::memset(&sel, 0, sizeof(sel));
  sel.bitmap = reinterpret_cast<uint32_t*>(ws + L.bitmap);
  sel.seg_counts = reinterpret_cast<uint32_t*>(ws + L.counts);
  int rc = esc_scan_select(prog, cols, ncols, nrows, d_row_ids, &sel, result, d_ws, ws_bytes, stream);
  if (rc != ESC_OK) return rc;
  return esc_materialize_selection(&sel, nrows, cols, ncols, d_row_ids, outs, d_ws, ws_bytes, stream);
}

int esc_compact_onepass(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols, int64_t nrows,
                        const int64_t* d_row_ids, const esc_outputs_t* outs, esc_result_t* result, void* d_ws,
                        size_t ws_bytes, void* stream) {
  static thread_local KParams kp;
  if (outs == nullptr) return fail(ESC_ERR_INVALID, "null outputs");
  int rc = build_params(kp, prog, cols, ncols, nrows, d_row_ids, d_ws, ws_bytes, result, outs);
  if (rc != ESC_OK) return rc;
  rc = next_epoch(kp, nrows, d_ws, static_cast<cudaStream_t>(stream));
  if (rc != ESC_OK) return rc;
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
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  switch (w) {
    case 1:
      ++g_launches;
      gather_kernel<uint8_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint8_t*>(col->data), col->nulls,
                                                                   d_idx, n, static_cast<uint8_t*>(out_values),
                                                                   out_nulls);
      break;
    case 2:
      ++g_launches;
      gather_kernel<uint16_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint16_t*>(col->data),
                                                                    col->nulls, d_idx, n,
                                                                    static_cast<uint16_t*>(out_values), out_nulls);
      break;
    case 4:
      ++g_launches;
      gather_kernel<uint32_t><<<(unsigned)blocks, threads, 0, st>>>(static_cast<const uint32_t*>(col->data),
                                                                    col->nulls, d_idx, n,
                                                                    static_cast<uint32_t*>(out_values), out_nulls);
      break;
    default:
      ++g_launches;
      gather_kernel<unsigned long long><<<(unsigned)blocks, threads, 0, st>>>(
          static_cast<const unsigned long long*>(col->data), col->nulls, d_idx, n,
          static_cast<unsigned long long*>(out_values), out_nulls);
      break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("gather launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int64_t esc_null_bits_words(int64_t n) { return n < 0 ? 0 : ((n + 31) / 32 + 3) / 4 * 4 + 4; }

int esc_pack_nulls(const uint8_t* nulls, int64_t n, uint32_t* out, void* stream) {
  if (n < 0 || out == nullptr || (n > 0 && nulls == nullptr)) return fail(ESC_ERR_INVALID, "bad pack arguments");
  const int64_t words = esc_null_bits_words(n);
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  int64_t blocks = (words + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  ++g_launches;
  pack_nulls_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(nulls, n, words, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ESC_OK : fail(ESC_ERR_CUDA, std::string("pack nulls: ") + cudaGetErrorString(e));
}

int esc_copy_regions(int32_t n, void* const* dst, const void* const* src, const int64_t* bytes, void* stream) {
  if (n < 0 || n > ESC_MAX_REGIONS) return fail(ESC_ERR_INVALID, "region count out of range");
  if (n == 0) return ESC_OK;
  if (dst == nullptr || src == nullptr || bytes == nullptr) return fail(ESC_ERR_INVALID, "null region arrays");
  static thread_local CopyRegions cr;
  cr.n = n;
  long long most = 0;
  for (int i = 0; i < n; ++i) {
    if (bytes[i] < 0) return fail(ESC_ERR_INVALID, "negative region size");
    if (bytes[i] > 0 && (dst[i] == nullptr || src[i] == nullptr)) return fail(ESC_ERR_INVALID, "null region");
    cr.dst[i] = static_cast<uint8_t*>(dst[i]);
    cr.src[i] = static_cast<const uint8_t*>(src[i]);
    cr.bytes[i] = bytes[i];
    most = std::max(most, (long long)bytes[i]);
  }
  if (most == 0) return ESC_OK;
  const int sms = sm_count_cached();
  if (sms <= 0) return fail(ESC_ERR_CUDA, "no CUDA device");
  long long bx = (most / 16 + 255) / 256;
  const long long cap = std::max(1ll, (long long)sms * 8 / n);
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  ++g_launches;
  copy_regions_kernel<<<dim3((unsigned)bx, (unsigned)n), 256, 0, static_cast<cudaStream_t>(stream)>>>(cr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("copy launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

int esc_count_gate(const int64_t* counts, int32_t world, int32_t rank, int64_t capacity, int64_t* out,
                   void* stream) {
  if (counts == nullptr || out == nullptr) return fail(ESC_ERR_INVALID, "null count gate buffer");
  if (world < 1 || rank < 0 || rank >= world) return fail(ESC_ERR_INVALID, "bad world / rank");
  if (capacity < 0) return fail(ESC_ERR_INVALID, "negative capacity");
  ++g_launches;
  count_gate_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(counts, world, rank, capacity, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ESC_ERR_CUDA, std::string("count gate launch: ") + cudaGetErrorString(e));
  return ESC_OK;
}

const char* esc_last_error(void) { return g_last_error.c_str(); }

int64_t esc_launch_count(void) { return (int64_t)g_launches.load(); }

int esc_abi_version(void) { return ESC_ABI_VERSION; }

int esc_device_sm_count(void) { return sm_count_cached(); }

int esc_set_jit(int mode, int64_t min_rows) {
  if (mode < 0 || mode > 2) return fail(ESC_ERR_INVALID, "JIT mode must be 0, 1 or 2");
  jit::g_mode = mode;
  if (min_rows >= 0) jit::g_min_rows = min_rows;
  return ESC_OK;
}

int esc_jit_selftest(void) {
  const std::string log = jit::selftest();
  if (!log.empty()) return fail(ESC_ERR_UNSUPPORTED, log);
  return ESC_OK;
}

int esc_jit_stats(int64_t* out) {
  if (out == nullptr) return fail(ESC_ERR_INVALID, "null output");
  out[0] = jit::g_compiled.load();
  out[1] = jit::g_hits.load();
  out[2] = jit::g_failures.load();
  out[3] = jit::g_compile_us.load();
  out[4] = jit::nvrtc().ok ? 1 : 0;
  return ESC_OK;
}

int esc_debug_trace(void* d_stamps) {
  g_trace = static_cast<unsigned long long*>(d_stamps);
  return ESC_OK;
}

int esc_set_stream_div(int div) {
  const int prev = g_stream_div.load();
  g_stream_div = div;
  return prev;
}

int esc_set_hit_lists(int mode) {
  const int prev = g_hit_lists.load();
  if (mode >= 0 && mode <= 2) g_hit_lists = mode;
  return prev;
}

int64_t esc_set_mid_max_rows(int64_t max_rows) {
  const long long prev = g_mid_max_rows.load();
  if (max_rows >= 0) g_mid_max_rows = max_rows;
  return prev;
}

int esc_struct_size(int which) {
  switch (which) {
    case 0: return (int)sizeof(esc_program_t);
    case 1: return (int)sizeof(esc_instr_t);
    case 2: return (int)sizeof(esc_udf_t);
    case 3: return (int)sizeof(esc_udf_op_t);
    case 4: return (int)sizeof(esc_column_t);
    case 5: return (int)sizeof(esc_result_t);
    case 6: return (int)sizeof(esc_outputs_t);
    case 7: return (int)sizeof(esc_selection_t);
    case 8: return (int)sizeof(esc_join_step_t);
    case 9: return (int)sizeof(esc_join_t);
    default: return -1;
  }
}

int esc_tile_rows(const esc_program_t* prog, const esc_column_t* cols, int32_t ncols) {
  static thread_local KParams kp;
  if (prog == nullptr || ncols < 0 || ncols > ESC_MAX_COLS) return 0;
  std::memset(&kp, 0, sizeof(kp));
  for (int i = 0; i < ncols; ++i) {
    kp.cols[i].data = static_cast<const uint8_t*>(cols[i].data);
    kp.cols[i].nulls = cols[i].nulls;
    kp.cols[i].null_bits = cols[i].null_bits;
    kp.cols[i].dtype = cols[i].dtype;
    kp.cols[i].width = dtype_width(cols[i].dtype);
  }
  return plan_geometry(kp, prog, cols, ncols, false, 1ll << 40, 3, nullptr).tile_rows;
}

}  // extern "C"

#include "esc_sort.cuh"
#include "esc_join.cuh"
#include "esc_csv.cuh"
