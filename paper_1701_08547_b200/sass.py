"""Native disassembly tokenizer -> K0 instruction records.

``tokenize(text)`` runs ``occx_sass_parse`` (host C++ in liboccx.so, a
restatement of occmix/sass.py:216-339) and returns per-function names, CSR
offsets, 4-byte OCCX_INSTR records and the interned signature table; errors
are raised as the reference raises them (``ParseError`` with the same line
and message, ``EmptyInputError``, and ``AttributeError`` where the reference
trips over its own opcode regex).  ``aggregate_text(text)`` feeds the records
to the K0 reducer on the GPU: the equivalent of
``[(name, aggregate(instrs)) for name, instrs in parse_disassembly(text)]``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EmptyInputError, ParseError
from .mix import DEFAULT_OPCLASSES, DEVICE_ID, OpClass, classify_signature


@dataclass
class SassRecords:
    names: list            # function names, in file order (duplicates kept)
    offsets: np.ndarray    # u64 [n + 1]
    records: np.ndarray    # u32 OCCX_INSTR records
    signatures: list       # (opcode, modifiers) per signature id

    def class_lut(self, table=DEFAULT_OPCLASSES) -> np.ndarray:
        """classify() of every signature (mix.py:176-187) as device class ids."""
        lut = [DEVICE_ID[classify_signature(op, mods, table)] for op, mods in self.signatures]
        return np.asarray(lut or [DEVICE_ID[OpClass.UNCLASSIFIED]], np.uint8)


_AS_UTF8 = ctypes.pythonapi.PyUnicode_AsUTF8AndSize
_AS_UTF8.restype = ctypes.c_void_p
_AS_UTF8.argtypes = [ctypes.py_object, ctypes.POINTER(ctypes.c_ssize_t)]


def _utf8(text: str):
    """The listing's UTF-8 bytes without a copy where CPython has them: an
    ASCII str stores exactly those bytes, and PyUnicode_AsUTF8AndSize hands
    out that buffer (kept alive by ``text``).  A str with lone surrogates is
    encoded with 'surrogatepass' (the bytes the tokenizer expects).
    Returns (char pointer or bytes, length)."""
    n = ctypes.c_ssize_t(0)
    try:
        p = _AS_UTF8(text, ctypes.byref(n))
        return ctypes.cast(p, ctypes.c_char_p), n.value
    except UnicodeEncodeError:
        data = text.encode("utf-8", "surrogatepass")
        return data, len(data)


def _blob(fn, h) -> list:
    """One call for all names / signatures: the library joins them by 0x1E."""
    n = ctypes.c_uint64(0)
    ptr = fn(h, ctypes.byref(n))
    return ctypes.string_at(ptr, n.value).decode("utf-8", "surrogatepass").split("\x1e")


def tokenize(text: str, chunk_bytes: int = 0, table=None) -> SassRecords:
    """``chunk_bytes``: minimum bytes per worker-thread chunk (0 = library
    default); only the split changes, never the result.  ``table`` (an
    opcode-class table): emit class records -- each record's signature id
    replaced by classify() of its signature (occx_sass_classify), for K0 with
    the identity class table ``CLASS_LUT``; ``signatures`` still lists the
    interned signatures."""
    lib = _lib.load()
    data, n_bytes = _utf8(text)
    h = ctypes.c_void_p()
    line = ctypes.c_int64(0)
    st = lib.occx_sass_parse_ex(data, n_bytes, int(chunk_bytes), ctypes.byref(h),
                                ctypes.byref(line))
    try:
        if st:
            err = lib.occx_sass_error_text(h).decode("utf-8", "surrogatepass")
            if st == 12:
                raise EmptyInputError(err)
            if st == 11:
                if err.startswith("\x01"):
                    err = f"instruction {err[1:]!r} missing terminating ';'"
                raise ParseError(err, int(line.value))
            if st == 13:
                raise AttributeError(err)
            _lib.check(st, f"occx_sass_parse (line {line.value}): {err}")
        n_k = lib.occx_sass_n_kernels(h)
        n_i = lib.occx_sass_n_instr(h)
        names = _blob(lib.occx_sass_names_blob, h) if n_k else []
        off = np.ctypeslib.as_array(ctypes.cast(lib.occx_sass_offsets(h),
                                                ctypes.POINTER(ctypes.c_uint64)),
                                    shape=(n_k + 1,)).copy() if n_k else np.zeros(1, np.uint64)
        sigs = []
        if lib.occx_sass_n_sigs(h):
            for s in _blob(lib.occx_sass_signatures_blob, h):
                parts = s.split("\x1f")
                sigs.append((parts[0], tuple("." + m for m in parts[1:])))
        out = SassRecords(names, off, None, sigs)
        if table is not None and n_i:
            lut = out.class_lut(table)
            _lib.check(lib.occx_sass_classify(h, lut.ctypes.data, len(lut)), "occx_sass_classify")
        out.records = np.ctypeslib.as_array(
            ctypes.cast(lib.occx_sass_records(h), ctypes.POINTER(ctypes.c_uint32)),
            shape=(n_i,)).copy() if n_i else np.zeros(0, np.uint32)
        return out
    finally:
        lib.occx_sass_free(h)


def aggregate_text(text: str, table=DEFAULT_OPCLASSES) -> list:
    """[(name, InstructionMix)] for every function of a listing: native
    tokenizer + K0 on the GPU."""
    from .batch import CLASS_LUT, _to_device, _to_host, mix_from_record, mix_reduce
    r = tokenize(text, table=table)
    if not r.names:
        return []
    d = mix_reduce(_to_device(r.records if len(r.records) else np.zeros(1, np.uint32)),
                   _to_device(r.offsets), len(r.names), _to_device(CLASS_LUT), len(CLASS_LUT))
    out = _to_host(d, _lib.MIX, len(r.names))
    return [(n, mix_from_record(m)) for n, m in zip(r.names, out)]
