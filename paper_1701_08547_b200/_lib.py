"""ctypes binding of liboccx.so (the C ABI in include/occx.h).

This is the binding a maintainer would add to occmix.  The
library must have been built for sm_100a (``__graft_entry__.build()`` or
``python -m paper_1701_08547_b200.build``); there is no CPU fallback --
importing the device API without the library or without a GPU raises.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

import numpy as np

from .errors import DeviceError, raise_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# OCCX_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("OCCX_LIB") or os.path.join(_HERE, "liboccx.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "occx.h")

# --- struct layouts (must match include/occx.h) -----------------------------
CAND = np.dtype([("variant", "<u4"), ("smem", "<u4"), ("threads", "<u2"),
                 ("blocks", "<u2"), ("regs", "<u2"), ("arch", "u1"), ("aux", "u1")])
OCC = np.dtype([("wpb", "u1"), ("limit_warps", "u1"), ("active_blocks", "u1"),
                ("active_warps", "u1"), ("limiter", "u1"), ("status", "u1"),
                ("r0", "u1"), ("r1", "u1"), ("limit_regs", "<u4"),
                ("limit_smem", "<u4"), ("reg_warp_limit", "<u4"), ("r2", "<u4"),
                ("occupancy", "<f8")])
MIX = np.dtype([("counts", "<u4", 16), ("first_key", "<u4", 16),
                ("reg_operands", "<u8"), ("n_instr", "<u4"), ("reserved", "<u4")])
MIXSUM = np.dtype([("intensity", "<f8"), ("flops", "<u8"), ("mem", "<u8"),
                   ("ctrl", "<u8"), ("unclassified", "<u8"), ("total", "<u8")])
FEAT = np.dtype([("cost", "<f8"), ("coef", "<f8", 4), ("cycles", "<f8", 4),
                 ("shares", "<f8", 4), ("per_class", "<f8", 16),
                 ("status", "<i4"), ("pc_status", "<i4")])
VENT = np.dtype([("member", "<u4", 4), ("seg", "<u4"), ("key_hi", "<u4"),
                 ("rank_bits", "<u4"), ("reserved", "<u4")])
SEGDESC = np.dtype([("start", "<u8"), ("size", "<u8"), ("arch", "<u4"),
                    ("var_base", "<u4"), ("dim_off", "<u4", 7), ("dim_len", "<u4", 7)])
SUGG_IN = np.dtype([("arch", "<u4"), ("regs", "<u4"), ("smem", "<u4"), ("reserved", "<u4")])
SUGG = np.dtype([("status", "<i4"), ("best_threads", "<u4"), ("best_blocks", "<u4"),
                 ("best_warps", "<u4"), ("smem_budget", "<u4"),
                 ("register_headroom", "<u4"), ("best_occupancy", "<f8")])
for _dt, _size in ((CAND, 16), (OCC, 32), (MIX, 144), (MIXSUM, 48), (FEAT, 240),
                   (VENT, 32), (SEGDESC, 80), (SUGG_IN, 16), (SUGG, 32)):
    assert _dt.itemsize == _size, (_dt, _size)

_P, _I, _U32, _U64, _D = (ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32,
                          ctypes.c_uint64, ctypes.c_double)
SIGNATURES = {
    "occx_abi_version": ([], _I),
    "occx_status_string": ([_I], ctypes.c_char_p),
    "occx_ctx_create": ([_I, _P], _I),
    "occx_ctx_create_ex": ([_I, _U32, _P], _I),
    "occx_ctx_options": ([_P], _U32),
    "occx_ctx_destroy": ([_P], _I),
    "occx_ctx_sm_count": ([_P], _I),
    "occx_check_archs": ([_P, _I, _P], _I),
    "occx_occupancy_batch": ([_P, _P, _I, _P, _U64, _I, _P, _P], _I),
    "occx_suggest_batch": ([_P, _P, _I, _P, _U32, _I, _P, _P], _I),
    "occx_mix_reduce": ([_P, _P, _P, _U32, _P, _U32, _P, _P], _I),
    "occx_feature_score": ([_P, _P, _U32, _P, _U32, _P, _D, _I, _P, _P, _P], _I),
    "occx_build_vtab": ([_P, _P, _P, _U32, _U32, _P, _P, _P, _P], _I),
    "occx_score_workspace_bytes": ([_P, _U32, _U32, _P], _I),
    "occx_score_lists": ([_P], _I),
    "occx_stream_sync": ([_P], _I),
    "occx_score_workspace_init": ([_P, _P, _U32, _U32, _P], _I),
    "occx_space_buf_bytes": ([_P, _U64, _U32, _U32, _U32, _U32, _P, _P], _I),
    "occx_score_space_host": ([_P, _P, _I, _P, _U64, _P, _U32, _U32, _U32, _P, _D, _I, _U64,
                               _U64, _U64, _I, _U32, _U32, _P, _U64, _P, _P], _I),
    "occx_score_topk": ([_P, _P, _I, _P, _U64, _U64, _I, _P, _U32, _U32, _U32, _P, _U64,
                         _P, _P], _I),
    "occx_topk_merge": ([_P, _P, _U32, _U32, _U32, _P, _P], _I),
    "occx_gen_space": ([_P, _P, _U32, _P, _U64, _U64, _P, _P], _I),
    "occx_sass_parse": ([ctypes.c_char_p, _U64, _P, _P], _I),
    "occx_sass_parse_ex": ([ctypes.c_char_p, _U64, _U64, _P, _P], _I),
    "occx_sass_n_kernels": ([_P], _U32),
    "occx_sass_n_instr": ([_P], _U64),
    "occx_sass_records": ([_P], _P),
    "occx_sass_offsets": ([_P], _P),
    "occx_sass_kernel_name": ([_P, _U32], ctypes.c_char_p),
    "occx_sass_n_sigs": ([_P], _U32),
    "occx_sass_signature": ([_P, _U32], ctypes.c_char_p),
    "occx_sass_error_text": ([_P], ctypes.c_char_p),
    "occx_sass_names_blob": ([_P, _P], _P),
    "occx_sass_signatures_blob": ([_P, _P], _P),
    "occx_sass_free": ([_P], None),
    "occx_sass_classify": ([_P, _P, _U32], _I),
    "occx_score_space": ([_P, _P, _I, _P, _U32, _P, _U32, _U64, _U64, _U64, _I, _U32, _P, _U32,
                          _U32, _U32, _P, _U64, _P, _P], _I),
}


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Function names declared in include/occx.h."""
    text = open(path, encoding="utf-8").read()
    return sorted(set(re.findall(
        r"^\s*(?:int|void|uint32_t|uint64_t|const char\*|const uint32_t\*|const uint64_t\*)"
        r"\s+(occx_\w+)\s*\(", text, re.M)))


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load liboccx.so and declare every signature; raises when missing."""
    global _lib
    with _lock:
        if _lib is None:
            import torch  # noqa: F401  -- loads the libcudart.so.12 liboccx links
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is not built; run `python -m paper_1701_08547_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status:
        msg = load().occx_status_string(status).decode()
        raise_status(status, f"{what}: {msg}")


# context options (include/occx.h): implementation choices, same results
CTX_K2_FEED_LDG = 0x1
CTX_K2_ONE_SLICE = 0x2
CTX_K2_NO_STEAL = 0x4
SCORE_EVERY_KEY = 0x1           # occx_score_space flag: no block-bound pruning

_ctx: dict[tuple[int, int], int] = {}


def ctx(device: int | None = None, options: int = 0) -> int:
    """Per-(device, options) context handle (created once, immutable)."""
    import torch
    if not _ctx and not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the occx backend runs on the GPU only")
    dev = torch.cuda.current_device() if device is None else device
    with _lock:
        h = _ctx.get((dev, options))
    if h is None:
        out = ctypes.c_void_p()
        check(load().occx_ctx_create_ex(dev, options, ctypes.byref(out)), "occx_ctx_create_ex")
        with _lock:
            h = _ctx.setdefault((dev, options), out.value)
        if h != out.value:          # another thread won the race: drop ours
            load().occx_ctx_destroy(out)
    return h


def ptr(t) -> int:
    """Device pointer of a torch tensor, or host pointer of a numpy array."""
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
