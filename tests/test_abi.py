"""The C-ABI library loads without a GPU and exports every declared symbol (CPU)."""

import os
import re

from paper_1812_00282_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "vate.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vate_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("vate_pool_create", "vate_scan_pairs", "vate_scan_packed", "vate_advance",
                 "vate_count_inactive", "vate_host_g0", "vate_estimate_begin",
                 "vate_estimate_finish", "vate_snapshot", "vate_load", "vate_hosts_active",
                 "vate_merge_dirty"):
        assert must in names


def test_library_exports_every_declared_symbol():
    missing = [n for n in _declared() if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_binding_covers_the_header():
    assert sorted(_lib.EXPORTED) == _declared()


def test_abi_version_and_error_text():
    assert _lib.lib.vate_abi_version() == 1
    assert isinstance(_lib.last_error(), str)


def test_null_handles_fail_cleanly_without_a_gpu():
    import ctypes as C
    n = C.c_uint64()
    assert _lib.lib.vate_pool_launches(None, C.byref(n)) == _lib.VATE_EVALUE
    assert "null" in _lib.last_error()
    assert _lib.lib.vate_hosts_size(None, C.byref(n)) == _lib.VATE_EVALUE
