"""The C-ABI library loads on a CPU-only host, exports every entry point
include/wavecast_b200.h declares, and fails loudly (no CPU fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wavecast_b200.h")
LIB = os.path.join(ROOT, "paper_2309_10212_b200", "libwavecast_b200.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wc_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__

        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("wc_volume_create", "wc_session_create", "wc_session_pass", "wc_session_framebuffer",
                 "wc_decode_blocks", "wc_reference_render", "wc_exclusive_scan", "wc_sort_by_key"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2309_10212_b200 import _lib

    assert set(declared_functions()) == set(_lib._SIGS), set(declared_functions()) ^ set(_lib._SIGS)


def test_no_gpu_fails_loudly(lib):
    import paper_2309_10212_b200._lib as L

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    L._initialised = False
    with pytest.raises(RuntimeError, match="CUDA"):
        L.ensure_device(0)
    lib.wc_build_info.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.wc_build_info()


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out
