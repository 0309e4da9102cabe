"""ctypes binding of libmmjoin_b200.so (the C ABI in include/mmjoin_b200.h).

There is no CPU fallback: importing this module without the built library,
or calling into it without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import MatrixOverflowError

# MMJ_LIB_VARIANT=check loads the bounds-checked build (MMJ_DCHECK compiled
# in, build.py --check) instead of the product library
_LIB_PATH = Path(__file__).resolve().parent / "_lib" / (
    "libmmjoin_b200_check.so" if os.environ.get("MMJ_LIB_VARIANT") == "check" else "libmmjoin_b200.so")

MMJ_OK = 0
MMJ_ERR_ARG = 1
MMJ_ERR_CUDA = 2
MMJ_ERR_OVERFLOW = 3
MMJ_ERR_UNSUPPORTED = 4
MMJ_ERR_CAPACITY = 5

MODE_BITMAP = 0
MODE_COUNT32 = 1
MODE_ACC64 = 2
MODE_BITMAP_U8 = 3
MODE_BITMAP_PAIR = 4
MODE_COUNT16 = 5
MODE_UPPER = 16

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
INT = C.c_int
SZ = C.c_size_t

_SIGS = {
    "mmj_abi_version": (INT, []),
    "mmj_last_error": (C.c_char_p, []),
    "mmj_set_device": (INT, [INT]),
    "mmj_sm_count": (INT, []),
    "mmj_launch_count": (C.c_longlong, []),
    "mmj_scan_workspace_bytes": (C.c_size_t, [I64]),
    "mmj_exclusive_scan_i32": (INT, [P, P, I64, P, P]),
    "mmj_code_checksum": (INT, [P, I64, I64, P, P]),
    "mmj_heavy_y_positions": (INT, [P, P, I64, I64, P, P, P, P, P]),
    "mmj_build_operand": (INT, [P, P, I64, P, I64, P, P, I64, I64, I64, P]),
    "mmj_ingest_workspace_bytes": (SZ, [I64]),
    "mmj_ingest_dedup": (INT, [P, I64, P, P, P, SZ, P]),
    "mmj_ingest_first_seen": (INT, [P, I64, I64, P, P, P, P, SZ, P]),
    "mmj_ingest_distinct": (INT, [P, I64, I64, P, P, P, SZ, P]),
    "mmj_ingest_intersect": (INT, [P, I64, P, I64, P, P, P, SZ, P]),
    "mmj_ingest_repr_order": (INT, [P, I64, P, P, P, SZ, P]),
    "mmj_ingest_lookup": (INT, [P, P, I64, P, I64, I64, P, P]),
    "mmj_ingest_filter": (INT, [P, P, I64, P, P, P, P, SZ, P]),
    "mmj_ingest_sort_ids": (INT, [P, I64, P, P, P, SZ, P]),
    "mmj_ingest_remap": (INT, [P, I64, P, P, P]),
    "mmj_ingest_gather": (INT, [P, INT, P, I64, P, P]),
    "mmj_ingest_histogram": (INT, [P, I64, I64, P, P]),
    "mmj_ingest_csr": (INT, [P, P, I64, I64, I64, P, P, P, P, P, SZ, P]),
    "mmj_compact_rows": (INT, [P, P, P, P, P, P, I64, I64, I64, I64] + [P] * 11 + [SZ, P]),
    "mmj_decode_compact_codes": (INT, [P, I64, I64, P, P, I64, P, P]),
    "mmj_split_codes": (INT, [P, I64, I64, P, P, P]),
    "mmj_build_operand_pairs": (INT, [P, P, I64, P, I64, P, P, I64, I64, I64, P]),
    "mmj_light_z_csr": (INT, [P, P, I64, I64, P, I64, P, P, P, P, P, P]),
    "mmj_light_lengths": (INT, [P, P, I64, I64, P, I64, P, P, P, P, P, I64, INT, P, P, P, P]),
    "mmj_light_expand": (INT, [P, P, I64, I64, P, I64, P, P, P, P, P, I64, INT, P, I64, INT, I64, P, I64, P]),
    "mmj_heavy_mma": (INT, [P, I64, P, I64, I64, I64, I64, I64, I64, INT, INT, P, I64, P, INT, P]),
    "mmj_digit_plane": (INT, [P, I64, I64, INT, INT, P, I64, P]),
    "mmj_tile_count": (I64, [I64, I64]),
    "mmj_tile_merge": (INT, [P, INT, I64, I64, I64, I64, P, P, P, I64, P, P, P, P, P, P, P, P, P, P]),
    "mmj_emit_codes": (INT, [P, P, I64, I64, I64, I64, P, P]),
    "mmj_merge_emit_workspace_size": (SZ, [I64, I64]),
    "mmj_merge_emit": (INT, [P, INT, I64, I64, I64, I64, P, P, P, I64, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P]),
    "mmj_build_heavy_rows": (INT, [P, P, I64, P, I64, P, P, I64, I64, P]),
    "mmj_heavy_row_stats": (INT, [P, P, I64, P, I64, I64, P, P, P]),
    "mmj_merge_emit_col_blocks": (INT, [I64]),
    "mmj_debug_timing_buffer": (None, [P]),
    "mmj_list_splits": (INT, [P, P, I64, I64, P, P]),
    "mmj_bsi_degree_histogram": (INT, [P, P, I64, I64, I64, INT, INT, P, P]),
    "mmj_bsi_record_words": (INT, [INT]),
    "mmj_bsi_records": (INT, [P, P, I64, P, INT, P, P, P]),
    "mmj_bsi_answer": (INT, [P, P, I64, P, P, I64, P, I64, I64, P, P, I64, P, I64, I64, P, P, P, P, INT, P, P]),
    "mmj_bsi_direct_table": (INT, [P, P, I64, I64, I64, P, P]),
    "mmj_bsi_span_table": (INT, [P, P, I64, I64, I64, P, P, P, I64, INT, P, P]),
    "mmj_bsi_answer_spans": (INT, [P, P, I64, P, I64, I64, INT, P, I64, P, P, I64, I64, INT, P, I64, P, P, P]),
    "mmj_format_keys": (INT, [P, P, I64, INT, P, P, P, P, P, P]),
    "mmj_format_lengths": (INT, [P, P, P, I64, INT, P, P, P, P]),
    "mmj_format_write": (INT, [P, P, P, I64, INT, P, P, P, P, P, P]),
    "mmj_bsi_answer_lists": (INT, [P, P, I64, P, P, I64, P, I64, I64, P, P, I64, P, I64, I64, P, P, P, P, P, P]),
    "mmj_star_split": (INT, [INT, P, I64, C.c_double, P, P, P, P, P, P, P, P]),
    "mmj_star_operand": (INT, [INT, P, P, I64, I64, I64, P, P]),
    "mmj_star_light_workspace_bytes": (SZ, [I64]),
    "mmj_star_light": (INT, [INT, P, P, P, P, I64, I64, I64, INT, P, I64, P, P, P]),
    "mmj_bitmap_segment_count": (I64, [I64]),
    "mmj_bitmap_segments": (INT, [P, I64, P, P, P, P]),
    "mmj_bitmap_emit": (INT, [P, I64, I64, P, I64, I64, P, P]),
    "mmj_count_segment_count": (I64, [I64]),
    "mmj_count_segments": (INT, [P, INT, I64, I64, I64, I64, I32, P, INT, P, P, P, P]),
    "mmj_count_emit": (INT, [P, INT, I64, I64, I64, I64, I64, I32, P, INT, P, P, P, P]),
}

_lib = None


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load (once) and return the ctypes library object."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build the CUDA extension first "
            "(python -m paper_2002_12459_b200.build); there is no CPU fallback")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mmj_abi_version() != 1:
        raise ImportError("libmmjoin_b200.so ABI mismatch")
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS)


class NativeError(RuntimeError):
    pass


def check(status: int, what: str = ""):
    if status == MMJ_OK:
        return
    msg = load().mmj_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == MMJ_ERR_ARG:
        raise ValueError(text)
    if status == MMJ_ERR_OVERFLOW:
        raise MatrixOverflowError(text)
    if status == MMJ_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    raise NativeError(text)


def call(name: str, *args):
    """Invoke ``name`` from the library and raise the mapped exception on failure."""
    fn = getattr(load(), name)
    check(fn(*args), name)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the mmjoin B200 engine needs a CUDA device (no CPU fallback)")
    lib = load()
    dev = torch.cuda.current_device()
    check(lib.mmj_set_device(dev), "mmj_set_device")
    return dev


def ptr(t) -> int:
    """Device pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_handle():
    import torch
    return torch.cuda.current_stream().cuda_stream


if os.environ.get("MMJ_EAGER_LOAD"):
    load()
