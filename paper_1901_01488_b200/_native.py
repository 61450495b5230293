"""ctypes binding of the sm_100a C ABI (``include/esc.h``) + per-stream workspaces.

This is the only module that touches the shared library. Loading is lazy and loud: if the
extension is missing, or a kernel is asked to run on CPU tensors / without a CUDA device, a
:class:`~paper_1901_01488_b200.errors.NativeUnavailable` is raised — there is no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from .errors import ExecutionError, NativeUnavailable

LIB_NAME = "_esc_native.so"
LIB_PATH = os.environ.get("ESC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

ABI_VERSION = 2
MAX_COLS, MAX_INSTRS, MAX_UDFS, MAX_UDF_OPS, MAX_UDF_ARGS, MAX_STACK, MAX_PROJ = 32, 96, 8, 128, 8, 16, 32

# dtypes
I8, I16, I32, I64, F32, F64, U8, U16, U32 = range(9)
# opcodes
OP_CMP, OP_RANGE, OP_LUT, OP_COLCMP, OP_NOTNULL, OP_FALSE, OP_UDF, OP_PUSH, OP_POP, OP_NOT = range(1, 11)
COMB_SET, COMB_AND, COMB_OR = 0, 1, 2
CMP_EQ, CMP_NE, CMP_LT, CMP_LE, CMP_GT, CMP_GE = range(6)
DOM_I64, DOM_F32, DOM_F64 = 0, 1, 2
(UDF_ARG, UDF_CONST, UDF_ADD, UDF_SUB, UDF_MUL, UDF_DIV, UDF_MOD, UDF_FLOORDIV, UDF_NEG, UDF_ABS,
 UDF_SQUARE, UDF_LT, UDF_LE, UDF_GT, UDF_GE, UDF_EQ, UDF_NE, UDF_JMPF, UDF_JMP, UDF_FLOOR, UDF_CEIL, UDF_TRUNC,
 UDF_SQRT, UDF_RINT) = range(1, 25)
FAIL_DIV, FAIL_MOD, FAIL_FLOORDIV, FAIL_POW, FAIL_NAN_INT, FAIL_INF_INT, FAIL_DOMAIN = 1, 2, 3, 4, 5, 6, 7
COL_STAGE = 1

CMP_CODE = {"=": CMP_EQ, "<>": CMP_NE, "<": CMP_LT, "<=": CMP_LE, ">": CMP_GT, ">=": CMP_GE}

TORCH_DTYPE_CODE = {
    torch.int8: I8, torch.int16: I16, torch.int32: I32, torch.int64: I64,
    torch.float32: F32, torch.float64: F64, torch.uint8: U8, torch.uint16: U16, torch.uint32: U32,
}


class EscConst(C.Union):
    _fields_ = [("i", C.c_int64), ("f", C.c_double)]


class EscInstr(C.Structure):
    _fields_ = [("op", C.c_uint8), ("combine", C.c_uint8), ("cmp", C.c_uint8), ("domain", C.c_uint8),
                ("col_a", C.c_uint8), ("col_b", C.c_uint8), ("neg", C.c_uint8), ("pad0", C.c_uint8),
                ("aux", C.c_uint32), ("aux2", C.c_uint32), ("k0", EscConst), ("k1", EscConst)]


class EscUdfOp(C.Structure):
    _fields_ = [("op", C.c_uint8), ("arg", C.c_uint8), ("pad", C.c_uint8 * 6), ("k", C.c_double)]


class EscUdf(C.Structure):
    _fields_ = [("first_op", C.c_uint16), ("n_ops", C.c_uint8), ("n_args", C.c_uint8), ("dense", C.c_uint8),
                ("pad", C.c_uint8 * 3), ("arg_col", C.c_uint8 * MAX_UDF_ARGS),
                ("arg_div", C.c_double * MAX_UDF_ARGS)]


class EscProgram(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("n_instrs", C.c_uint16), ("n_udfs", C.c_uint16),
                ("n_udf_ops", C.c_uint16), ("max_depth", C.c_uint16), ("lut_words", C.c_uint32),
                ("lut", C.c_void_p), ("instrs", EscInstr * MAX_INSTRS), ("udfs", EscUdf * MAX_UDFS),
                ("udf_ops", EscUdfOp * MAX_UDF_OPS)]


class EscColumn(C.Structure):
    _fields_ = [("data", C.c_void_p), ("nulls", C.c_void_p), ("dtype", C.c_int32), ("flags", C.c_int32),
                ("null_bits", C.c_void_p)]


class EscResult(C.Structure):
    _fields_ = [("count", C.c_uint64), ("udf_fail", C.c_uint64 * MAX_UDFS)]


class EscOutputs(C.Structure):
    _fields_ = [("n_proj", C.c_int32), ("flags", C.c_int32), ("slot", C.c_int32 * MAX_PROJ),
                ("out_values", C.c_void_p * MAX_PROJ), ("out_nulls", C.c_void_p * MAX_PROJ),
                ("out_row_ids", C.c_void_p), ("capacity", C.c_int64)]


class EscSelection(C.Structure):
    _fields_ = [("bitmap", C.c_void_p), ("seg_counts", C.c_void_p), ("seg_rows", C.c_int32),
                ("cap_per_seg", C.c_int32), ("n_cap", C.c_int32), ("cap_stride", C.c_int32),
                ("cap_slot", C.c_int32 * MAX_PROJ), ("cap_values", C.c_void_p * MAX_PROJ),
                ("cap_nulls", C.c_void_p * MAX_PROJ), ("d_count", C.c_void_p), ("d_gate", C.c_void_p)]


MAX_STEPS = 8
JOIN_DENSE, JOIN_HASH, JOIN_PAIRS = 0, 1, 2


class EscJoinStep(C.Structure):
    _fields_ = [("key_data", C.c_void_p), ("key_nulls", C.c_void_p), ("key_dtype", C.c_int32), ("mode", C.c_int32),
                ("dense_min", C.c_int64), ("dense_len", C.c_int64), ("factor", C.c_void_p),
                ("factor_bits", C.c_int32), ("pad", C.c_int32), ("slots", C.c_void_p), ("capacity", C.c_int64),
                ("unique_keys", C.c_void_p), ("weight", C.c_void_p * (MAX_STEPS + 1))]


class EscJoin(C.Structure):
    _fields_ = [("n_steps", C.c_int32), ("n_stages", C.c_int32), ("star", C.c_int32), ("pad", C.c_int32),
                ("nrows", C.c_int64), ("bitmap", C.c_void_p), ("stage_of", C.c_int32 * MAX_STEPS),
                ("steps", EscJoinStep * MAX_STEPS)]


SEG_CAPTURED = 0x80000000
OUT_SKIP_OVER_CAPACITY = 1
PLAN_GRAPH = 4  # esc_step_plan_launch: a single part as a cached CUDA graph
STRUCTS = [EscProgram, EscInstr, EscUdf, EscUdfOp, EscColumn, EscResult, EscOutputs, EscSelection, EscJoinStep,
           EscJoin]

# every symbol include/esc.h declares, with its ctypes signature
_SIGNATURES = {
    "esc_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "esc_workspace_init": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_scan_count": (C.c_int, [C.POINTER(EscProgram), C.POINTER(EscColumn), C.c_int32, C.c_int64,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_compact": (C.c_int, [C.POINTER(EscProgram), C.POINTER(EscColumn), C.c_int32, C.c_int64,
                              C.c_void_p, C.POINTER(EscOutputs), C.c_void_p, C.c_void_p, C.c_size_t,
                              C.c_void_p]),
    "esc_compact_onepass": (C.c_int, [C.POINTER(EscProgram), C.POINTER(EscColumn), C.c_int32, C.c_int64,
                                      C.c_void_p, C.POINTER(EscOutputs), C.c_void_p, C.c_void_p, C.c_size_t,
                                      C.c_void_p]),
    "esc_selection_sizes": (C.c_int, [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    "esc_scan_select": (C.c_int, [C.POINTER(EscProgram), C.POINTER(EscColumn), C.c_int32, C.c_int64, C.c_void_p,
                                  C.POINTER(EscSelection), C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_materialize_selection": (C.c_int, [C.POINTER(EscSelection), C.c_int64, C.POINTER(EscColumn), C.c_int32,
                                            C.c_void_p, C.POINTER(EscOutputs), C.c_void_p, C.c_size_t,
                                            C.c_void_p]),
    "esc_gather": (C.c_int, [C.POINTER(EscColumn), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                             C.c_void_p]),
    "esc_count_gate": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]),
    "esc_null_bits_words": (C.c_int64, [C.c_int64]),
    "esc_pack_nulls": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "esc_last_error": (C.c_char_p, []),
    "esc_launch_count": (C.c_int64, []),
    "esc_abi_version": (C.c_int, []),
    "esc_device_sm_count": (C.c_int, []),
    "esc_struct_size": (C.c_int, [C.c_int]),
    "esc_tile_rows": (C.c_int, [C.POINTER(EscProgram), C.POINTER(EscColumn), C.c_int32]),
    "esc_set_jit": (C.c_int, [C.c_int, C.c_int64]),
    "esc_jit_stats": (C.c_int, [C.POINTER(C.c_int64)]),
    "esc_jit_selftest": (C.c_int, []),
    "esc_set_stream_div": (C.c_int, [C.c_int]),
    "esc_set_mid_max_rows": (C.c_int64, [C.c_int64]),
    "esc_set_hit_lists": (C.c_int, [C.c_int]),
    "esc_debug_trace": (C.c_int, [C.c_void_p]),
    "esc_copy_regions": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "esc_sort_temp_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32]),
    "esc_sort_pairs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_runs": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_order_keys": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]),
    "esc_rank_values": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "esc_hist_buckets": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p]),
    "esc_dict_temp_bytes": (C.c_size_t, [C.c_int64]),
    "esc_dict_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_hash_insert": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
    "esc_factor_array": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                   C.c_size_t, C.c_void_p]),
    "esc_pairs_bytes": (C.c_size_t, [C.c_int64]),
    "esc_pairs_build": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
    "esc_hash_build_temp_bytes": (C.c_int, [C.c_int64, C.POINTER(C.c_size_t)]),
    "esc_hash_build": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_hash_probe": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "esc_expand": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_void_p]),
    "esc_join_count": (C.c_int, [C.POINTER(EscJoin), C.c_void_p, C.c_void_p]),
    "esc_step_plan_create": (C.c_int, [C.POINTER(EscProgram), C.c_void_p, C.c_int32, C.c_int64,
                                       C.POINTER(EscSelection), C.c_void_p, C.c_int32, C.POINTER(EscOutputs),
                                       C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "esc_step_plan_launch": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "esc_step_plan_destroy": (C.c_int, [C.c_void_p]),
    "esc_step_plan_rebind": (C.c_int, [C.c_void_p, C.c_void_p]),
    "esc_csv_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "esc_csv_count": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "esc_csv_fields": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                 C.c_void_p]),
    "esc_csv_parse": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "esc_csv_check": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "esc_csv_verify_text": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load (once) and type the extension; raise NativeUnavailable when it is absent."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        try:
            lib = C.CDLL(path)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.esc_abi_version() != ABI_VERSION:
            raise NativeUnavailable("C ABI version mismatch between the library and the binding")
        for i, st in enumerate(STRUCTS):
            if lib.esc_struct_size(i) != C.sizeof(st):
                raise NativeUnavailable(f"struct {st.__name__} size mismatch: "
                                        f"C={lib.esc_struct_size(i)} ctypes={C.sizeof(st)}")
        _lib = lib
        return lib


# tuning generation: bumped by every setting change, so prepared launch plans are re-prepared
TUNING = [0]


def set_jit(mode: int, min_rows: int = -1):
    """0 = interpreter only, 1 = JIT scans of >= min_rows rows, 2 = always JIT."""
    check(load_library().esc_set_jit(int(mode), int(min_rows)), "esc_set_jit")
    TUNING[0] += 1


def set_mid_max_rows(rows: int) -> int:
    """Largest selection (rows) compacted by the one-launch mid-size kernel (0: never); returns
    the previous setting."""
    TUNING[0] += 1
    return int(load_library().esc_set_mid_max_rows(int(rows)))


def set_hit_lists(mode: int) -> int:
    """Warp hit lists in the gathered compaction (0 off, 1 auto, 2 always); returns the previous
    setting."""
    TUNING[0] += 1
    return int(load_library().esc_set_hit_lists(int(mode)))


def set_stream_div(div: int) -> int:
    """Dense-tile rule of the selection compaction (tile streamed when hits >= rows/div; <= 0 off);
    returns the previous setting."""
    TUNING[0] += 1
    return int(load_library().esc_set_stream_div(int(div)))


def jit_stats() -> dict:
    out = (C.c_int64 * 5)()
    check(load_library().esc_jit_stats(out), "esc_jit_stats")
    return {"compiled": out[0], "hits": out[1], "failures": out[2], "compile_ms": out[3] / 1e3,
            "nvrtc": bool(out[4])}


def check(rc: int, what: str):
    if rc != 0:
        msg = load_library().esc_last_error().decode(errors="replace")
        raise ExecutionError(f"{what} failed (code {rc}): {msg}")


def require_cuda(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise NativeUnavailable(f"{what} lives on {t.device}; the ESC kernels run on CUDA devices only")


def dtype_code(t: torch.Tensor) -> int:
    try:
        return TORCH_DTYPE_CODE[t.dtype]
    except KeyError:
        raise ExecutionError(f"unsupported column dtype {t.dtype}") from None


# --------------------------------------------------------------------------------------------
# per-(device, stream) workspace and result slot
# --------------------------------------------------------------------------------------------
RESULT_SLOTS = 64


class _Workspace:
    def __init__(self, device: torch.device):
        self.device = device
        self.buf: torch.Tensor | None = None
        self.nbytes = 0
        self.ptr = 0
        self.covers = 0  # largest row count known to fit (workspace size grows with rows)
        # result block written by the last CTA of every launch: pinned host memory is mapped
        # into the device address space under UVA, so no D2H copy is issued
        self.result = torch.zeros(C.sizeof(EscResult), dtype=torch.uint8, pin_memory=True)
        # more result blocks for steps queued together before one host wait (slots 1..RESULT_SLOTS)
        self.results = torch.zeros(RESULT_SLOTS * C.sizeof(EscResult), dtype=torch.uint8, pin_memory=True)
        # device-side result block (for NCCL reductions of counts)
        # device words initialised by host copies (no fill kernels in the launch list)
        self.dresult = torch.zeros(C.sizeof(EscResult), dtype=torch.uint8).to(device)
        # device copy of the last selection count (queued compactions check it on the device)
        self.dcount = torch.zeros(1, dtype=torch.int64).to(device)
        # the queued ESC step's cached launch plan (executor._step_plan)
        self.scratch: dict = {}

    def ensure(self, nrows: int, stream_ptr: int) -> tuple[int, int]:
        if self.buf is not None and nrows <= self.covers:
            return self.ptr, self.nbytes
        lib = load_library()
        need = int(lib.esc_workspace_bytes(max(int(nrows), 1)))
        if self.buf is None or self.nbytes < need:
            size = max(need, 1 << 20, self.nbytes * 2 if self.buf is not None else 0)
            self.buf = torch.empty(size, dtype=torch.uint8, device=self.device)
            self.nbytes = size
            check(lib.esc_workspace_init(C.c_void_p(self.buf.data_ptr()), C.c_size_t(size),
                                         C.c_void_p(stream_ptr)), "esc_workspace_init")
            self.ptr = self.buf.data_ptr()
        self.covers = max(self.covers, int(nrows)) if need <= self.nbytes else self.covers
        return self.ptr, self.nbytes

    def result_ptr(self, slot: int = 0) -> int:
        if slot == 0:
            return self.result.data_ptr()
        if not 1 <= slot <= RESULT_SLOTS:
            raise ValueError(f"result slot {slot} out of range")
        return self.results.data_ptr() + (slot - 1) * C.sizeof(EscResult)

    def read_result(self, n_udfs: int = 0, slot: int = 0) -> tuple[int, list[int]]:
        r = EscResult.from_address(self.result_ptr(slot))
        return int(r.count), [int(r.udf_fail[i]) for i in range(n_udfs)]


_workspaces: dict = {}
_ws_lock = threading.Lock()


def workspace(device: torch.device, stream: torch.cuda.Stream) -> _Workspace:
    key = (device.index, stream.cuda_stream, threading.get_ident())
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None:
            ws = _workspaces[key] = _Workspace(device)
        return ws
