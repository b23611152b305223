"""CPU checks of the drop-in boundary: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/hkv_b200.h declares (no compute
calls — there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hkv_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(hkv_[a-z_0-9]+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_17168_b200 import _lib, build

    build.build()
    return _lib.load()


def test_header_declares_api():
    syms = declared_symbols()
    for s in ("hkv_create", "hkv_destroy", "hkv_find", "hkv_contains", "hkv_find_ptr", "hkv_upsert",
              "hkv_assign", "hkv_erase", "hkv_export", "hkv_size", "hkv_import_state", "hkv_export_state",
              "hkv_route", "hkv_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_python_binding_covers_header(lib):
    from paper_2603_17168_b200 import _lib

    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a(lib):
    from paper_2603_17168_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_config_validation_without_gpu(lib):
    """Host-side validation runs before any CUDA call (table.py:108-127 messages)."""
    from paper_2603_17168_b200 import _lib

    def create(**kw):
        base = dict(capacity=1024, value_dim=4, mode=0, score_policy=0, fast_tier_budget=-1, digest_filter=1,
                    admit_ties_unified=0, overflow_in_hbm=0, device=0)
        base.update(kw)
        cfg = _lib.HkvConfig(**base)
        h = ctypes.c_void_p()
        return lib.hkv_create(ctypes.byref(cfg), ctypes.byref(h)), lib.hkv_last_error().decode()

    assert create(capacity=1000) == (1, "capacity must be a positive multiple of 128")
    assert create(capacity=128 * 3) == (1, "bucket count must be a power of two")
    assert create(value_dim=0) == (1, "value_dim must be >= 1")
    assert create(fast_tier_budget=9) == (1, "fast_tier_budget out of range")
    assert create(score_policy=7) == (1, "unknown policy")
