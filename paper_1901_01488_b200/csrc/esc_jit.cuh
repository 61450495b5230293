// esc_jit.cuh — JIT tier of the ESC kernels (host code, included by esc_kernels.cu).
//
// The ahead-of-time kernels interpret the lowered program: every opcode costs a dispatch per
// lane per tile, and UDFs run on a small stack machine.  For large scans the same hand-written
// kernel skeleton (esc_device.cuh: TMA ring, look-back warp, deferred scatter) is instantiated
// with a GENERATED predicate evaluator: one straight-line function per program shape, where
// every atom is a direct call of its smem range loop and every UDF is inlined SSA arithmetic.
// Query constants stay in the kernel parameters (one module serves all constants of a shape);
// UDF constants (part of the registered function) are baked in, which lets UDFs whose values
// provably stay integral and below 2^53 run in exact int64 arithmetic (division by literal
// constants becomes multiply-high) — bit-identical to CPython's float results.
//
// Compilation: NVRTC (dlopen'ed, so the library loads without it) -> CUBIN for sm_100a ->
// cudaLibraryLoadData.  Modules are cached per generated source.  A shape that fails to compile
// is remembered and served by the interpreter (still on the GPU).
#pragma once

// (system headers are included by esc_kernels.cu: this file is included inside its namespace)
#include "esc_embedded.inc"  // kEscHeaderSrc (include/esc.h), kEscDeviceSrc (esc_device.cuh)

namespace jit {

struct Nvrtc {
  bool ok = false;
  void* h = nullptr;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcAddNameExpression) add_name = nullptr;
  decltype(&nvrtcGetLoweredName) lowered = nullptr;
  std::string why;
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* cands[] = {getenv("ESC_NVRTC_LIB"), "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                           "libnvrtc.so"};
    for (const char* c : cands) {
      if (c == nullptr) continue;
      n.h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) {
      n.why = "libnvrtc.so.12 not found";
      return;
    }
#define ESC_SYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.h, name))
    ESC_SYM(create, "nvrtcCreateProgram");
    ESC_SYM(compile, "nvrtcCompileProgram");
    ESC_SYM(cubin_size, "nvrtcGetCUBINSize");
    ESC_SYM(cubin, "nvrtcGetCUBIN");
    ESC_SYM(log_size, "nvrtcGetProgramLogSize");
    ESC_SYM(log, "nvrtcGetProgramLog");
    ESC_SYM(destroy, "nvrtcDestroyProgram");
    ESC_SYM(add_name, "nvrtcAddNameExpression");
    ESC_SYM(lowered, "nvrtcGetLoweredName");
#undef ESC_SYM
    n.ok = n.create && n.compile && n.cubin_size && n.cubin && n.log_size && n.log && n.destroy && n.add_name &&
           n.lowered;
    if (!n.ok) n.why = "libnvrtc is missing symbols";
  });
  return n;
}

// ---- settings and statistics ----------------------------------------------------------------
int env_mode() {
  const char* e = getenv("ESC_JIT");
  return (e != nullptr && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 1;
}
std::atomic<int> g_mode{env_mode()};        // 0 off, 1 auto (nrows >= min_rows), 2 always
std::atomic<long long> g_min_rows{1ll << 22};
std::atomic<long long> g_compiled{0}, g_hits{0}, g_failures{0};
std::atomic<long long> g_compile_us{0};

struct Entry {
  bool ok = false;
  cudaKernel_t kernel = nullptr;
  int smem_configured = 0;
  std::string log;
};
std::mutex g_mu;
std::unordered_map<std::string, Entry> g_cache;   // generated source -> module
std::unordered_map<std::string, Entry*> g_shape;  // shape bytes -> its module (fast path: no codegen)

// Everything the generated evaluator bakes in (opcodes, flags, smem offsets, dtypes, UDF
// programs) — but not the query constants, which it reads from the kernel parameters.
std::string shape_key(const KParams& kp, bool compact) {
  std::string k;
  k.reserve(64 + sizeof(KInstr) * kp.n_ins + sizeof(kp.udfs) + sizeof(kp.udf_ops) + 16 * kp.ncols);
  const int hdr[4] = {kp.chunks, compact ? 1 : 0, kp.n_ins, kp.ncols};
  k.append(reinterpret_cast<const char*>(hdr), sizeof(hdr));
  for (int i = 0; i < kp.n_ins; ++i) {
    KInstr K = kp.ins[i];
    K.lo.i = K.hi.i = 0;
    k.append(reinterpret_cast<const char*>(&K), sizeof(K));
  }
  k.append(reinterpret_cast<const char*>(kp.udfs), sizeof(kp.udfs));
  k.append(reinterpret_cast<const char*>(kp.udf_ops), sizeof(kp.udf_ops));
  for (int i = 0; i < kp.ncols; ++i) {
    const KCol& c = kp.cols[i];
    const uint32_t v[6] = {(uint32_t)c.dtype, c.smem_off, c.smem_null_off, c.nulls != nullptr ? 1u : 0u,
                           (uint32_t)c.staged, (uint32_t)c.nulls_staged};
    k.append(reinterpret_cast<const char*>(v), sizeof(v));
  }
  // the scan-time capture is baked in too (which columns, where their nulls go)
  const int ncap = kp.sel_on ? kp.sel.n_cap : 0;
  k.append(reinterpret_cast<const char*>(&ncap), sizeof(ncap));
  for (int j = 0; j < ncap; ++j) {
    const int32_t v[2] = {kp.sel.cap_slot[j], kp.sel.cap_nulls[j] != nullptr ? 1 : 0};
    k.append(reinterpret_cast<const char*>(v), sizeof(v));
  }
  return k;
}

// ---- code generation -------------------------------------------------------------------------
const char* ctype_of(int dtype) {
  switch (dtype) {
    case ESC_I8: return "int8_t";
    case ESC_I16: return "int16_t";
    case ESC_I32: return "int32_t";
    case ESC_I64: return "long long";
    case ESC_U8: return "uint8_t";
    case ESC_U16: return "uint16_t";
    case ESC_U32: return "uint32_t";
    case ESC_F32: return "float";
    default: return "double";
  }
}

bool int_dtype(int dt) { return dt != ESC_F32 && dt != ESC_F64; }

const char* comb_stmt(int mode) { return mode == ESC_COMB_AND ? "&=" : mode == ESC_COMB_OR ? "|=" : "="; }

std::string dlit(double v) {  // exact double literal
  if (std::isnan(v)) return "__longlong_as_double(0x7ff8000000000000ll)";
  if (std::isinf(v)) return v > 0 ? "__longlong_as_double(0x7ff0000000000000ll)" : "__longlong_as_double(0xfff0000000000000ll)";
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  std::string s = b;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

const char* cmp_op(int cmp) {
  switch (cmp) {
    case ESC_CMP_EQ: return "==";
    case ESC_CMP_NE: return "!=";
    case ESC_CMP_LT: return "<";
    case ESC_CMP_LE: return "<=";
    case ESC_CMP_GT: return ">";
    default: return ">=";
  }
}

// integer interval of an SSA value (exact integer arithmetic while |v| < 2^53)
struct Val {
  std::string name;
  bool is_int = false;  // held as long long
  double lo = 0, hi = 0;
};
constexpr double kExact = 9007199254740992.0;  // 2^53

std::string as_double(const Val& v) { return v.is_int ? "(double)" + v.name : v.name; }

// the staged NULL flag of tile row `lr` of column c (a byte, or a bit of the packed bitmap)
std::string staged_null_expr(const KCol& c, const std::string& lr) {
  if (c.nulls_staged == 2)
    return "((reinterpret_cast<const uint32_t*>(st + " + std::to_string(c.smem_null_off) + "u)[(" + lr + ") >> 5] >> ((" +
           lr + ") & 31)) & 1u)";
  return "(st[" + std::to_string(c.smem_null_off) + "u + " + lr + "] != 0)";
}
const char* nulls_fn(uint32_t noff) { return (noff & kPackedNulls) ? "null_bits_packed" : "null_bits_staged"; }

// UDFs gen_udf_body turns into straight-line code: arithmetic only (no branches, comparisons
// or math functions — those run through the interpreter's atom_udf)
bool straight_line_udf(const KParams& kp, int ui) {
  const esc_udf_t& u = kp.udfs[ui];
  for (int i = 0; i < u.n_ops; ++i)
    if (kp.udf_ops[u.first_op + i].op > ESC_UDF_SQUARE) return false;
  return true;
}

// UDF `ui` of the program -> statements computing `double`/`long long` result; returns its Val
Val gen_udf_body(const KParams& kp, int ui, std::ostringstream& o, const std::string& pfx) {
  const esc_udf_t& u = kp.udfs[ui];
  std::vector<Val> stk;
  int tmp = 0;
  auto fresh = [&]() { return pfx + "t" + std::to_string(tmp++); };
  std::vector<Val> args(u.n_args);
  for (int a = 0; a < u.n_args; ++a) {
    const KCol& c = kp.cols[u.arg_col[a]];
    Val v;
    v.name = pfx + "a" + std::to_string(a);
    const std::string load = std::string("*reinterpret_cast<const ") + ctype_of(c.dtype) + "*>(st + " +
                             std::to_string(c.smem_off) + "u + (size_t)lr * " + std::to_string(c.width) + ")";
    if (int_dtype(c.dtype) && u.arg_div[a] == 0.0) {
      long long lo, hi;
      dtype_int_range(c.dtype, &lo, &hi);
      v.is_int = true;
      v.lo = (double)lo;
      v.hi = (double)hi;
      if (hi > (long long)kExact || lo < -(long long)kExact) v.is_int = false;  // int64 args: stay float
    }
    if (v.is_int) {
      o << "      const long long " << v.name << " = (long long)" << load << ";\n";
    } else {
      o << "      double " << v.name << " = ";
      if (c.dtype == ESC_I64) o << "__ll2double_rn(" << load << ")";
      else o << "(double)" << load;
      o << ";\n";
      if (u.arg_div[a] != 0.0) o << "      " << v.name << " = __ddiv_rn(" << v.name << ", " << dlit(u.arg_div[a]) << ");\n";
    }
    args[a] = v;
  }
  for (int i = 0; i < u.n_ops; ++i) {
    const esc_udf_op_t& op = kp.udf_ops[u.first_op + i];
    switch (op.op) {
      case ESC_UDF_ARG: stk.push_back(args[op.arg]); break;
      case ESC_UDF_CONST: {
        Val v;
        v.name = fresh();
        const double k = op.k;
        if (std::isfinite(k) && k == std::floor(k) && std::fabs(k) < kExact) {
          v.is_int = true;
          v.lo = v.hi = k;
          char b[64];
          std::snprintf(b, sizeof b, "%lldll", (long long)k);
          o << "      const long long " << v.name << " = " << b << ";\n";
        } else {
          o << "      const double " << v.name << " = " << dlit(k) << ";\n";
        }
        stk.push_back(v);
        break;
      }
      case ESC_UDF_NEG: case ESC_UDF_ABS: case ESC_UDF_SQUARE: {
        Val x = stk.back();
        stk.pop_back();
        Val v;
        v.name = fresh();
        if (op.op == ESC_UDF_NEG) {
          v.is_int = x.is_int;
          v.lo = -x.hi;
          v.hi = -x.lo;
          o << "      const " << (v.is_int ? "long long " : "double ") << v.name << " = -" << x.name << ";\n";
        } else if (op.op == ESC_UDF_ABS) {
          v.is_int = x.is_int;
          v.lo = 0;
          v.hi = std::max(std::fabs(x.lo), std::fabs(x.hi));
          o << "      const " << (v.is_int ? "long long " : "double ") << v.name << " = "
            << (v.is_int ? "llabs(" : "fabs(") << x.name << ");\n";
        } else {
          const double m = std::max(std::fabs(x.lo), std::fabs(x.hi));
          if (x.is_int && m * m < kExact) {
            v.is_int = true;
            v.lo = 0;
            v.hi = m * m;
            o << "      const long long " << v.name << " = " << x.name << " * " << x.name << ";\n";
          } else {
            o << "      const double " << v.name << " = __dmul_rn(" << as_double(x) << ", " << as_double(x) << ");\n";
            o << "      if (isinf(" << v.name << ") && isfinite(" << as_double(x) << ")) { failed = "
              << ESC_FAIL_POW << "u; break; }\n";
          }
        }
        stk.push_back(v);
        break;
      }
      default: {
        Val b = stk.back();
        stk.pop_back();
        Val a = stk.back();
        stk.pop_back();
        Val v;
        v.name = fresh();
        const int o_ = op.op;
        bool done = false;
        if (a.is_int && b.is_int && (o_ == ESC_UDF_ADD || o_ == ESC_UDF_SUB || o_ == ESC_UDF_MUL)) {
          double c[4];
          if (o_ == ESC_UDF_ADD) { c[0] = a.lo + b.lo; c[1] = a.hi + b.hi; c[2] = c[0]; c[3] = c[1]; }
          else if (o_ == ESC_UDF_SUB) { c[0] = a.lo - b.hi; c[1] = a.hi - b.lo; c[2] = c[0]; c[3] = c[1]; }
          else { c[0] = a.lo * b.lo; c[1] = a.lo * b.hi; c[2] = a.hi * b.lo; c[3] = a.hi * b.hi; }
          const double lo = std::min(std::min(c[0], c[1]), std::min(c[2], c[3]));
          const double hi = std::max(std::max(c[0], c[1]), std::max(c[2], c[3]));
          if (lo > -kExact && hi < kExact) {
            v.is_int = true;
            v.lo = lo;
            v.hi = hi;
            const char* sym = o_ == ESC_UDF_ADD ? "+" : o_ == ESC_UDF_SUB ? "-" : "*";
            o << "      const long long " << v.name << " = " << a.name << " " << sym << " " << b.name << ";\n";
            done = true;
          }
        }
        if (!done && a.is_int && b.is_int && b.lo == b.hi && b.lo != 0.0 &&
            (o_ == ESC_UDF_MOD || o_ == ESC_UDF_FLOORDIV)) {
          // exact integers: CPython's float % and // equal the floored integer operations;
          // a literal divisor lets the compiler use multiply-high
          char k[64];
          std::snprintf(k, sizeof k, "%lldll", (long long)b.lo);
          const double d = std::fabs(b.lo);
          v.is_int = true;
          if (o_ == ESC_UDF_MOD) {
            v.lo = b.lo > 0 ? 0 : b.lo + 1;
            v.hi = b.lo > 0 ? b.lo - 1 : 0;
            o << "      long long " << v.name << " = " << a.name << " % " << k << ";\n";
            o << "      if (" << v.name << " != 0 && ((" << v.name << " < 0) != (" << k << " < 0))) " << v.name
              << " += " << k << ";\n";
          } else {
            const double m = std::max(std::fabs(a.lo), std::fabs(a.hi)) / d + 1;
            v.lo = -m;
            v.hi = m;
            o << "      long long " << v.name << " = " << a.name << " / " << k << ";\n";
            o << "      if ((" << a.name << " % " << k << ") != 0 && ((" << a.name << " < 0) != (" << k
              << " < 0))) --" << v.name << ";\n";
          }
          done = true;
        }
        if (!done) {
          const std::string x = as_double(a), y = as_double(b);
          switch (o_) {
            case ESC_UDF_ADD: o << "      const double " << v.name << " = __dadd_rn(" << x << ", " << y << ");\n"; break;
            case ESC_UDF_SUB: o << "      const double " << v.name << " = __dsub_rn(" << x << ", " << y << ");\n"; break;
            case ESC_UDF_MUL: o << "      const double " << v.name << " = __dmul_rn(" << x << ", " << y << ");\n"; break;
            case ESC_UDF_DIV:
              o << "      if (" << y << " == 0.0) { failed = " << ESC_FAIL_DIV << "u; break; }\n";
              o << "      const double " << v.name << " = __ddiv_rn(" << x << ", " << y << ");\n";
              break;
            case ESC_UDF_MOD:
              o << "      if (" << y << " == 0.0) { failed = " << ESC_FAIL_MOD << "u; break; }\n";
              o << "      const double " << v.name << " = py_mod(" << x << ", " << y << ");\n";
              break;
            default:
              o << "      if (" << y << " == 0.0) { failed = " << ESC_FAIL_FLOORDIV << "u; break; }\n";
              o << "      const double " << v.name << " = py_floordiv(" << x << ", " << y << ");\n";
              break;
          }
        }
        stk.push_back(v);
      }
    }
  }
  return stk.back();
}

// Scan-time capture with the captured columns' types and stage offsets baked in: staged tiles
// copy each hit's values straight from shared memory; tail tiles keep the generic path.
void gen_capture(const KParams& kp, std::ostringstream& o) {
  o << "  template <int C>\n  static __device__ __forceinline__ void capture(const KParams& p, const RowRef& rr, "
       "uint32_t bits, uint32_t excl, uint32_t wtp, int64_t seg) {\n";
  const int ncap = kp.sel_on ? kp.sel.n_cap : 0;
  if (ncap == 0) {
    o << "    capture_generic<C>(p, rr, bits, excl, wtp, seg);\n  }\n";
    return;
  }
  o << "    if (rr.stage == nullptr) { capture_generic<C>(p, rr, bits, excl, wtp, seg); return; }\n"
    << "    const uint8_t* st = rr.stage;\n"
    << "    const size_t base = (size_t)seg, stride = (size_t)p.sel.cap_stride;  // slot-major\n";
  for (int k = 0; k < ncap; ++k) {
    const KCol& c = kp.cols[kp.sel.cap_slot[k]];
    o << "    " << ctype_of(c.dtype) << "* cv" << k << " = static_cast<" << ctype_of(c.dtype) << "*>(p.sel.cap_values["
      << k << "]) + base;\n";
    if (kp.sel.cap_nulls[k] != nullptr) o << "    uint8_t* cn" << k << " = p.sel.cap_nulls[" << k << "] + base;\n";
  }
  o << "    uint32_t cb = 0;\n#pragma unroll\n    for (int c = 0; c < C; ++c) {\n"
    << "      uint32_t r = cb + ((excl >> (8 * c)) & 0xFFu);\n      cb += (wtp >> (8 * c)) & 0xFFu;\n"
    << "      uint32_t m = (bits >> (4 * c)) & 0xFu;\n      while (m) {\n"
    << "        const int j = __ffs(m) - 1;\n        m &= m - 1;\n"
    << "        const int lr = rr.local0 + " << kChunkRows << " * c + j;\n";
  for (int k = 0; k < ncap; ++k) {
    const int slot = kp.sel.cap_slot[k];
    const KCol& c = kp.cols[slot];
    if (c.staged)
      o << "        cv" << k << "[(size_t)r * stride] = *reinterpret_cast<const " << ctype_of(c.dtype) << "*>(st + " << c.smem_off
        << "u + (size_t)lr * " << c.width << ");\n";
    else
      o << "        cv" << k << "[(size_t)r * stride] = *reinterpret_cast<const " << ctype_of(c.dtype) << "*>(value_ptr(p.cols[" << slot
        << "], rr, 4 * c + j));\n";
    if (kp.sel.cap_nulls[k] != nullptr) {
      if (c.nulls == nullptr) o << "        cn" << k << "[(size_t)r * stride] = 0;\n";
      else if (c.nulls_staged) o << "        cn" << k << "[(size_t)r * stride] = " << staged_null_expr(c, "lr") << " ? 1 : 0;\n";
      else o << "        cn" << k << "[(size_t)r * stride] = is_null(p.cols[" << slot << "], rr, 4 * c + j) ? 1 : 0;\n";
    }
  }
  o << "        ++r;\n      }\n    }\n  }\n";
}

// The generated evaluator.  Returns false when the program uses something the generator does
// not specialise (the caller then keeps the interpreter).
bool gen_pred(const KParams& kp, int C, std::ostringstream& o) {
  o << "struct JitPred {\n  template <int C>\n  static __device__ __forceinline__ uint32_t eval(const KParams& p, "
       "const RowRef& rr, uint32_t valid) {\n";
  o << "    const uint8_t* st = rr.stage;\n    const int l0 = rr.local0;\n    (void)st; (void)l0;\n";
  o << "    uint32_t acc0 = 0, care0 = valid;\n";
  std::vector<int> stack{0};
  int next = 1;
  for (int i = 0; i < kp.n_ins; ++i) {
    const KInstr& K = kp.ins[i];
    const std::string acc = "acc" + std::to_string(stack.back());
    const std::string care = "care" + std::to_string(stack.back());
    const std::string I = "p.ins[" + std::to_string(i) + "]";
    if (K.op == K_PUSH) {
      const int d = next++;
      const std::string nc = K.combine == ESC_COMB_AND ? (care + " & " + acc)
                             : K.combine == ESC_COMB_OR ? (care + " & ~" + acc) : care;
      o << "    uint32_t acc" << d << " = 0, care" << d << " = " << nc << ";\n";
      stack.push_back(d);
      continue;
    }
    if (K.op == K_POP) {
      const std::string inner = acc;
      stack.pop_back();
      o << "    acc" << stack.back() << " " << comb_stmt(K.combine) << " " << inner << ";\n";
      continue;
    }
    if (K.op == K_NOT) {
      o << "    " << acc << " = ~" << acc << ";\n";
      continue;
    }
    o << "    {\n      uint32_t r;\n";
    const std::string sub = "(uint32_t)(" + I + ".hi.i - " + I + ".lo.i)";
    const std::string sub64 = "(unsigned long long)" + I + ".hi.i - (unsigned long long)" + I + ".lo.i";
    const std::string colp = "st + " + std::to_string(K.soff) + "u";
    switch (K.op) {
      case K_FALSE: o << "      r = 0u;\n"; break;
      case K_NOTNULL:
        if (K.noff != kNoNulls) o << "      r = ~" << nulls_fn(K.noff) << "<C>(st + " << (K.noff & ~kPackedNulls) << "u, l0);\n";
        else o << "      r = 0xFFFFFFFFu;\n";
        break;
      case K_RANGE_S8: case K_RANGE_U8: case K_RANGE_S16: case K_RANGE_U16: case K_RANGE_S32: {
        const char* t = K.op == K_RANGE_S8 ? "int8_t" : K.op == K_RANGE_U8 ? "uint8_t" : K.op == K_RANGE_S16 ? "int16_t"
                        : K.op == K_RANGE_U16 ? "uint16_t" : "int32_t";
        o << "      r = range_i32<" << t << ", C>(" << colp << ", l0, (int32_t)" << I << ".lo.i, " << sub << ");\n";
        break;
      }
      case K_RANGE_S64:
        o << "      r = range_i64<long long, C>(" << colp << ", l0, " << I << ".lo.i, " << sub64 << ");\n";
        break;
      case K_RANGE_U32:
        o << "      r = range_i64<uint32_t, C>(" << colp << ", l0, " << I << ".lo.i, " << sub64 << ");\n";
        break;
      case K_RANGE_F32:
        o << "      r = range_f32<C>(" << colp << ", l0, (float)" << I << ".lo.f, (float)" << I << ".hi.f);\n";
        break;
      case K_UDF: {
        const esc_udf_t& u = kp.udfs[K.aux];
        const std::string ce = K.combine == ESC_COMB_AND ? (care + " & " + acc)
                               : K.combine == ESC_COMB_OR ? (care + " & ~" + acc) : care;
        if (!straight_line_udf(kp, K.aux)) {
          // branches / math: the interpreter's atom (a jump-aware stack machine) on the staged tile
          o << "      r = atom_udf(p, " << I << ", rr, " << ce << ", valid);\n";
          break;
        }
        o << "      r = 0u;\n      uint32_t todo = " << (u.dense ? std::string("valid") : "(" + ce + ") & valid")
          << ";\n      while (todo) {\n        const int bit = __ffs(todo) - 1;\n        todo &= todo - 1;\n"
          << "        const int lr = l0 + " << kChunkRows << " * (bit >> 2) + (bit & 3);\n"
          << "        uint32_t failed = 0u;\n        double v = 0.0;\n        do {\n";
        std::ostringstream body;
        const Val res = gen_udf_body(kp, K.aux, body, "u" + std::to_string(i) + "_");
        o << body.str() << "      v = " << as_double(res) << ";\n        } while (0);\n";
        o << "        if (failed) {\n          atomicMin(&p.hdr->fail[" << K.aux
          << "], (unsigned long long)(logical_row(rr, bit) << 3) | failed);\n          continue;\n        }\n";
        std::string nulls;
        for (int a = 0; a < u.n_args; ++a) {
          const KCol& c = kp.cols[u.arg_col[a]];
          if (c.nulls != nullptr) nulls += " || " + staged_null_expr(c, "lr");
        }
        o << "        if (!(false" << nulls << ") && v " << cmp_op(K.cmp) << " " << I << ".lo.f) r |= 1u << bit;\n"
          << "      }\n";
        break;
      }
      default:  // K_RANGE_F64, K_LUT, K_COLCMP: the generic per-row path (nulls handled inside)
        o << "      r = atom_generic(p, " << I << ", rr, valid);\n";
        break;
    }
    if (K.op <= K_RANGE_F32) {
      if (K.inv) o << "      r = ~r;\n";
      if (K.noff != kNoNulls) o << "      r &= ~" << nulls_fn(K.noff) << "<C>(st + " << (K.noff & ~kPackedNulls) << "u, l0);\n";
    }
    if (K.neg) o << "      r = ~r;\n";
    o << "      " << acc << " " << comb_stmt(K.combine) << " r;\n    }\n";
  }
  o << "    return acc0 & valid;\n  }\n";
  gen_capture(kp, o);
  o << "};\n";
  (void)C;
  return true;
}

// Compile (or fetch) the JIT kernel for this program shape; nullptr when unavailable.
cudaKernel_t get_kernel(const KParams& kp, bool compact, size_t smem, std::string* why) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) {
    *why = nv.why;
    return nullptr;
  }
  const std::string inst = "esc::esc_scan_kernel<" + std::to_string(kp.chunks) + ", " + (compact ? "true" : "false") +
                           ", esc::JitPred>";
  std::lock_guard<std::mutex> g(g_mu);
  const std::string shape = shape_key(kp, compact);
  auto serve = [&](Entry& en) -> cudaKernel_t {
    if (!en.ok) {
      *why = en.log;
      return nullptr;
    }
    if (en.smem_configured < (int)smem) {
      if (cudaFuncSetAttribute(reinterpret_cast<const void*>(en.kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) == cudaSuccess)
        en.smem_configured = (int)smem;
    }
    ++g_hits;
    return en.kernel;
  };
  auto sh = g_shape.find(shape);
  if (sh != g_shape.end()) return serve(*sh->second);
  std::ostringstream pred;
  if (!gen_pred(kp, kp.chunks, pred)) return nullptr;
  const std::string src = std::string("#include \"esc_device.cuh\"\nnamespace esc {\n") + pred.str() + "}\n";
  const std::string key = inst + "\n" + src;
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    g_shape.emplace(shape, &it->second);
    return serve(it->second);
  }
  Entry e;
  const auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  const char* headers[] = {kEscHeaderSrc, kEscDeviceSrc};
  const char* names[] = {"esc.h", "esc_device.cuh"};
  if (nv.create(&prog, src.c_str(), "esc_jit.cu", 2, headers, names) != NVRTC_SUCCESS) {
    e.log = "nvrtcCreateProgram failed";
  } else {
    nv.add_name(prog, inst.c_str());
    const std::string warps = "-DESC_CONSUMER_WARPS=" + std::to_string(kConsumerWarps);
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-fmad=false", "-lineinfo",
                          "--device-as-default-execution-space", "-DESC_JIT=1", warps.c_str()};
    const nvrtcResult rc = nv.compile(prog, 7, opts);
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    if (rc != NVRTC_SUCCESS) {
      e.log = "NVRTC: " + log;
    } else {
      const char* lowered = nullptr;
      nv.lowered(prog, inst.c_str(), &lowered);
      size_t n = 0;
      nv.cubin_size(prog, &n);
      std::string cubin(n, '\0');
      nv.cubin(prog, &cubin[0]);
      cudaLibrary_t lib;
      cudaError_t ce = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
      if (ce == cudaSuccess) ce = cudaLibraryGetKernel(&e.kernel, lib, lowered);
      if (ce == cudaSuccess)
        ce = cudaFuncSetAttribute(reinterpret_cast<const void*>(e.kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem);
      if (ce != cudaSuccess) {
        e.log = std::string("module load: ") + cudaGetErrorString(ce);
      } else {
        e.ok = true;
        e.smem_configured = (int)smem;
      }
    }
    nv.destroy(&prog);
  }
  g_compile_us += std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count();
  if (e.ok) ++g_compiled;
  else ++g_failures;
  auto& slot = g_cache[key] = e;
  g_shape.emplace(shape, &slot);
  if (!slot.ok) {
    *why = slot.log;
    return nullptr;
  }
  return slot.kernel;
}

// Compile the embedded device sources with a trivial evaluator for every kernel instantiation
// the JIT tier emits (no device needed: NVRTC only).  Returns "" on success, else the log.
std::string selftest() {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) return nv.why.empty() ? "NVRTC unavailable" : nv.why;
  const char* src =
      "#include \"esc_device.cuh\"\nnamespace esc {\nstruct JitPred {\n"
      "  template <int C> static __device__ __forceinline__ uint32_t eval(const KParams& p, const RowRef& rr, "
      "uint32_t valid) { return eval_program<C, true>(p, rr, valid); }\n"
      "  template <int C> static __device__ __forceinline__ void capture(const KParams& p, const RowRef& rr, "
      "uint32_t bits, uint32_t excl, uint32_t wtp, int64_t seg) { capture_generic<C>(p, rr, bits, excl, wtp, seg); }\n"
      "};\n}\n";
  nvrtcProgram prog;
  const char* headers[] = {kEscHeaderSrc, kEscDeviceSrc};
  const char* names[] = {"esc.h", "esc_device.cuh"};
  if (nv.create(&prog, src, "esc_jit_selftest.cu", 2, headers, names) != NVRTC_SUCCESS) return "nvrtcCreateProgram failed";
  const char* insts[] = {"esc::esc_scan_kernel<1, false, esc::JitPred>", "esc::esc_scan_kernel<4, false, esc::JitPred>",
                         "esc::esc_scan_kernel<8, false, esc::JitPred>", "esc::esc_scan_kernel<4, true, esc::JitPred>"};
  for (const char* i : insts) nv.add_name(prog, i);
  const std::string warps = "-DESC_CONSUMER_WARPS=" + std::to_string(kConsumerWarps);
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-fmad=false", "-lineinfo",
                        "--device-as-default-execution-space", "-DESC_JIT=1", warps.c_str()};
  const nvrtcResult rc = nv.compile(prog, 7, opts);
  std::string out;
  if (rc != NVRTC_SUCCESS) {
    size_t ls = 0;
    nv.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) nv.log(prog, &log[0]);
    out = "NVRTC: " + log;
  }
  nv.destroy(&prog);
  return out;
}

}  // namespace jit
