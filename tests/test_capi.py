"""The C-ABI library loads on a CPU-only host, exports every symbol that
include/occx.h declares, and its host-only entry points behave (no GPU
compute is attempted here)."""

import ctypes

import pytest

from paper_1701_08547_b200 import _lib, workloads
from paper_1701_08547_b200.arch import ARCH_DTYPE, pack_archs


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_exports_every_header_function(lib):
    names = _lib.header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "binding and header disagree"


def test_abi_version_and_status_strings(lib):
    assert lib.occx_abi_version() == 2
    for code in range(14):
        assert lib.occx_status_string(code) != b"unknown status", code
    assert lib.occx_status_string(14) == b"unknown status"
    assert b"IllegalLaunchError" in lib.occx_status_string(2)
    assert b"ParseError" in lib.occx_status_string(11)
    assert b"EmptyInputError" in lib.occx_status_string(12)
    assert b"AttributeError" in lib.occx_status_string(13)


def test_ctx_options_validated_before_device(lib):
    out = ctypes.c_void_p()
    assert lib.occx_ctx_create_ex(0, 0x10, ctypes.byref(out)) == 1      # unknown option bit
    assert lib.occx_ctx_create_ex(0, 0, None) == 1
    assert lib.occx_ctx_options(None) == 0


def test_library_reads_no_environment():
    """Implementation switches are explicit arguments (ctx options, score
    flags, tokenizer chunk size), not environment variables."""
    import os
    import re
    csrc = os.path.join(os.path.dirname(_lib.__file__), "csrc")
    for f in os.listdir(csrc):
        text = open(os.path.join(csrc, f), encoding="utf-8").read()
        assert not re.search(r"\bgetenv\s*\(", text), f


def test_struct_sizes_match_header():
    # sizes asserted in _lib against the C layout; re-check the arch row
    assert ARCH_DTYPE.itemsize == 40
    assert _lib.CAND.itemsize == 16 and _lib.OCC.itemsize == 32
    assert _lib.VENT.itemsize == 32 and _lib.SEGDESC.itemsize == 80


def test_check_archs_host_only(lib):
    a = pack_archs(workloads.all_archs())
    bad = ctypes.c_int(7)
    assert lib.occx_check_archs(a.ctypes.data, len(a), ctypes.byref(bad)) == 0
    assert bad.value == -1
    b = a.copy()
    b[2]["max_warps_per_mp"] = 200          # 7-bit key field
    assert lib.occx_check_archs(b.ctypes.data, len(b), ctypes.byref(bad)) == 8
    assert bad.value == 2
    assert lib.occx_check_archs(a.ctypes.data, 0, ctypes.byref(bad)) == 8


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    out = ctypes.c_void_p()
    assert lib.occx_ctx_create(0, ctypes.byref(out)) == 6      # OCCX_ERR_CUDA
    from paper_1701_08547_b200 import DeviceError, occupancy_batch
    with pytest.raises(DeviceError):
        occupancy_batch(workloads.all_archs()[1], [(128, 27, 0)])


def test_null_arguments_rejected(lib):
    assert lib.occx_occupancy_batch(None, None, 0, None, 0, 0, None, None) == 1
    assert lib.occx_score_topk(None, None, 0, None, 0, 0, 0, None, 0, 0, 0, None, 0,
                               None, None) == 1
    assert lib.occx_topk_merge(None, None, 0, 0, 0, None, None) == 1


def _spec(**kw):
    from dataclasses import replace
    base = workloads.all_archs()[4]            # sm_100 INI table
    return replace(base, **kw)


@pytest.mark.parametrize("field,value", [
    ("max_threads_per_block", 4096),            # T = 4096 (warp size 64) outside the 64-bit masks
    ("register_file_size", 1 << 20),
    ("register_alloc_granularity", 1 << 20),
    ("max_blocks_per_mp", 256),
    ("shared_mem_per_block", 1 << 24),
])
def test_host_and_device_limits_agree(lib, field, value):
    """arch.device_limits_ok and occx_check_archs enforce one set of limits:
    an arch the device tables cannot hold fails in pack_archs with
    ArchSpecError naming it, and the C check rejects the same row."""
    from paper_1701_08547_b200.arch import device_limits_ok
    from paper_1701_08547_b200.errors import ArchSpecError
    kw = {field: value}
    if field == "max_threads_per_block":
        kw.update(warp_size=64, max_warps_per_mp=64, max_threads_per_mp=64 * 64)
    try:
        s = _spec(**kw)
    except Exception:                            # the reference's own invariants reject it
        pytest.skip("not a valid ArchSpec")
    assert device_limits_ok(s)
    with pytest.raises(ArchSpecError):
        pack_archs([s])
    ok = _spec()
    row = pack_archs([ok])
    for f, v in kw.items():
        if f in row.dtype.names:
            row[0][f] = v
    bad = ctypes.c_int(0)
    assert lib.occx_check_archs(row.ctypes.data, 1, ctypes.byref(bad)) == 8 and bad.value == 0
    assert device_limits_ok(ok) is None
    assert lib.occx_check_archs(pack_archs([ok]).ctypes.data, 1, ctypes.byref(bad)) == 0


def test_t2048_arch_accepted(lib):
    """64 warps of 32 threads (max_threads_per_block 2048) is inside the
    device tables: T = 2048 is mask bit 63."""
    from paper_1701_08547_b200.arch import device_limits_ok
    s = _spec(max_threads_per_block=2048, max_threads_per_mp=2048, max_warps_per_mp=64)
    assert device_limits_ok(s) is None
    bad = ctypes.c_int(0)
    assert lib.occx_check_archs(pack_archs([s]).ctypes.data, 1, ctypes.byref(bad)) == 0
