"""The C-ABI library loads and exports every symbol include/cgbn.h declares (no GPU
needed: nothing here launches a kernel)."""

import ctypes
import os
import re

import pytest

from paper_1711_07240_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cgbn.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|size_t|const char\*)\s+(cgbn_\w+)\(", text, re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for name in ("cgbn_fwd_stats", "cgbn_fwd_normalize", "cgbn_fwd_train_local",
                 "cgbn_bwd_reduce", "cgbn_bwd_dx", "cgbn_bwd_local", "cgbn_fwd_eval",
                 "cgbn_fold_sum", "cgbn_workspace_bytes", "cgbn_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_constants_match_header():
    text = open(HEADER).read()

    def define(name):
        return int(re.search(rf"#define {name}\s+(\d+)", text).group(1))

    assert define("CGBN_LAYOUT_NCHW") == _lib.LAYOUT_NCHW
    assert define("CGBN_LAYOUT_NHWC") == _lib.LAYOUT_NHWC
    assert define("CGBN_MAX_GROUP") == _lib.MAX_GROUP
    assert define("CGBN_ERR_INVALID") == _lib.ERR_INVALID
    assert define("CGBN_ERR_UNSUPPORTED") == _lib.ERR_UNSUPPORTED
    assert define("CGBN_STATUS_NONFINITE") == _lib.STATUS_NONFINITE
    assert define("CGBN_STATUS_SMALL_COUNT") == _lib.STATUS_SMALL_COUNT


def test_abi_version_and_argument_validation_without_gpu():
    lib = _lib.load()
    assert lib.cgbn_abi_version() == 7
    assert b"sm_100a" in lib.cgbn_build_info()
    # invalid shapes are rejected on the host before any CUDA call
    rc = lib.cgbn_fwd_stats(None, 2, 3, 4, 0, None, None, 0, None)
    assert rc == _lib.ERR_INVALID
    assert b"NULL" in lib.cgbn_last_error()
    rc = lib.cgbn_fwd_stats(1, 0, 3, 4, 0, 1, None, 0, None)
    assert rc == _lib.ERR_INVALID
    assert b"positive" in lib.cgbn_last_error()
    rc = lib.cgbn_fwd_stats(1, 2, 70000, 4, 0, 1, None, 0, None)
    assert rc == _lib.ERR_INVALID
    assert b"65535" in lib.cgbn_last_error()


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.CGBNLibraryError, match="no CPU fallback"):
        _lib.load()


def test_producer_conv_argument_validation_without_gpu():
    """The producer entry points reject bad arguments on the host, before any CUDA call,
    with the shared thread-local message (the conv lives in a second translation unit)."""
    lib = _lib.load()
    rc = lib.cgbn_conv1x1(None, None, None, 2, 64, 128, 64, 0, None, None, 0, None)
    assert rc == _lib.ERR_INVALID and b"null" in lib.cgbn_last_error()
    rc = lib.cgbn_conv_nhwc(16, 16, None, 2, 64, 128, 8, 8, 2, 1, 0, 16, None, 0, None)
    assert rc == _lib.ERR_INVALID and b"ksize" in lib.cgbn_last_error()
    rc = lib.cgbn_conv_nhwc(16, 16, None, 2, 60, 128, 8, 8, 3, 1, 0, 16, None, 0, None)
    assert rc == _lib.ERR_UNSUPPORTED and b"Cin" in lib.cgbn_last_error()
    rc = lib.cgbn_conv1x1(16, 16, None, 2, 64, 128, 49, 0, 16, None, 0, None)
    assert rc == _lib.ERR_UNSUPPORTED and b"H*W" in lib.cgbn_last_error()
    rc = lib.cgbn_conv1x1(16, 16, None, 2, 64, 128, 64, 0x20, 16, None, 0, None)
    assert rc == _lib.ERR_INVALID and b"dtype" in lib.cgbn_last_error()
    rc = lib.cgbn_conv1x1_stats(16, 16, None, 2, 64, 128, 64, 0, 16, None, None, 0, None)
    assert rc == _lib.ERR_INVALID and b"workspace" in lib.cgbn_last_error()
    rc = lib.cgbn_fwd_normalize_slots(16, 2, 8, 16, 0, None, 16, 16, 1e-5, 0.1, 16, 16, 16, 0,
                                      16, 16, 16, 1 << 20, None)
    assert rc == _lib.ERR_INVALID and b"slot table" in lib.cgbn_last_error()
    rc = lib.cgbn_conv_nhwc_stats(16, 16, None, 2, 64, 128, 8, 8, 3, 2, 0, 16, 16, 16, 0, None)
    assert rc == _lib.ERR_INVALID and b"workspace" in lib.cgbn_last_error()


def test_stale_build_rejected(monkeypatch):
    """load() checks the ABI version and every bound symbol before use."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "ABI_VERSION", 5)
    with pytest.raises(_lib.CGBNLibraryError, match="ABI v7"):
        _lib.load()
    monkeypatch.setattr(_lib, "ABI_VERSION", 7)
    monkeypatch.setitem(_lib.SIGNATURES, "cgbn_not_there", (_lib._i, []))
    with pytest.raises(_lib.CGBNLibraryError, match="cgbn_not_there"):
        _lib.load()


@pytest.mark.parametrize("act", [_lib.ACT_F32, _lib.ACT_BF16, _lib.ACT_F16])
def test_dtype_units_share_the_error_message(act):
    """Each activation dtype is its own translation unit (cgbn.cu, cgbn_bf16.cu,
    cgbn_f16.cu); the public entry points route on the dtype bits of `layout` and every
    unit reports through the one thread-local message."""
    lib = _lib.load()
    rc = lib.cgbn_fwd_stats(None, 2, 3, 4, act, None, None, 0, None)
    assert rc == _lib.ERR_INVALID and b"NULL" in lib.cgbn_last_error()
    rc = lib.cgbn_bwd_local(1, 1, 2, 3, 4, act, 1, 1, 1, -1.0, 0, 1, None, None, None, None,
                            0, None)
    assert rc == _lib.ERR_INVALID and b"eps" in lib.cgbn_last_error()
    rc = lib.cgbn_fwd_stats(1, 2, 3, 4, 0x30, 1, None, 0, None)  # unknown dtype -> unit 0
    assert rc == _lib.ERR_INVALID and b"dtype" in lib.cgbn_last_error()
    for name in ("cgbn_fwd_stats_a0", "cgbn_fwd_stats_a1", "cgbn_fwd_stats_a2"):
        assert hasattr(lib, name)


def test_conv_workspace_plan_without_gpu():
    """The conv workspace (ABI v7) sizes itself from the host-side plan: statistics slots,
    then split-K partials for layers the plan splits (the 3x3 512-channel layers: 52 tiles
    of 128 pixels, 72 k-steps), then the 16 KB ticket region every layer keeps."""
    lib = _lib.load()
    slots_only = lib.cgbn_conv_nhwc_ws_bytes(32, 256, 256, 14, 14, 3, 1)  # not split
    split = lib.cgbn_conv_nhwc_ws_bytes(32, 512, 512, 7, 7, 3, 1)
    assert slots_only > 16384 and split > slots_only
    # 52 tiles x (2 - 1) partials x 128 x 128 fp32 beyond the slot table
    slots_512 = lib.cgbn_conv_nhwc_ws_bytes(32, 64, 512, 7, 7, 1, 1)  # Cin 64: never split
    assert split - slots_512 == 52 * 128 * 128 * 4
    assert lib.cgbn_conv_nhwc_ws_bytes(32, 64, 64, 7, 7, 2, 1) == 0  # ksize 2: invalid
    assert lib.cgbn_conv1x1_ws_bytes(0, 64, 64, 49) == 0
