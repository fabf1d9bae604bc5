"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "flashsplat_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_08270_b200 import _native
    if not _native.LIB_PATH.exists():
        import __graft_entry__
        __graft_entry__.build()
    return _native.load()


def test_header_declares_expected_entry_points():
    from paper_2409_08270_b200 import _native
    assert declared_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_library_is_sm100a_only(lib):
    import subprocess
    from paper_2409_08270_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version_and_error_strings(lib):
    from paper_2409_08270_b200 import _native
    assert b"sm_100a" in lib.fs_version()
    # argument validation happens before any CUDA call
    rc = lib.fs_assign(None, None, 5, 3, 0.0, _native.MODE_BINARY, None, 0)
    assert rc == _native.FS_EINVAL
    assert b"" != lib.fs_last_error()


def test_compute_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2409_08270_b200 import _native
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0)


def test_multi_entry_points_validate_before_touching_contexts(lib):
    """fs_accumulate_multi / fs_finalize_multi reject a context listed twice (one host
    thread per context) and bad counts before dereferencing anything (no GPU needed)."""
    import ctypes
    from paper_2409_08270_b200 import _native
    dummy = ctypes.c_void_p(0x1000)
    two = (ctypes.c_void_p * 2)(dummy, dummy)
    accs = (ctypes.c_void_p * 2)(ctypes.c_void_p(0x2000), ctypes.c_void_p(0x3000))
    rc = lib.fs_accumulate_multi(two, 2, 0, None, None, 2, 1 / 255, 1e-4, _native.ACC_FIXED,
                                 accs, None, None)
    assert rc == _native.FS_EINVAL and b"listed twice" in lib.fs_last_error()
    rc = lib.fs_finalize_multi(two, 2, _native.ACC_FIXED, accs, 10, 2, None, 0.0, -1, None)
    assert rc == _native.FS_EINVAL and b"listed twice" in lib.fs_last_error()
    rc = lib.fs_accumulate_multi(two, 0, 0, None, None, 2, 1 / 255, 1e-4, _native.ACC_FIXED,
                                 accs, None, None)
    assert rc == _native.FS_EINVAL
    rc = lib.fs_finalize_multi(two, 1, 7, accs, 10, 2, None, 0.0, -1, None)
    assert rc == _native.FS_EINVAL and b"accumulator kind" in lib.fs_last_error()
