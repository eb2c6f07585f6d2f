"""CPU checks of the C-ABI boundary (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "geoshoot_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1907_04834_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes signature table covers exactly the header
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == names


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_1907_04834_b200", "libgeoshoot_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_host_only_entry_points():
    from paper_1907_04834_b200 import _lib
    lib = _lib.load()
    assert lib.gs_abi_version() == 1
    c = lib.gs_default_config()  # reference defaults, core.hpp:204-213
    assert (c.sigma, c.lambda_, c.timesteps, c.backend, c.threshold_multiplier) == (2.0, 1.0, 40, 0, 3.0)
    bad = _lib.gs_config(-1.0, 0.0, 0, 0, 0.0, 0, 0)
    mask = C.c_uint32()
    assert lib.gs_validate_config(C.byref(bad), C.byref(mask)) == _lib.GS_CONFIG_ERROR
    assert mask.value == 0b1111  # every violation reported (core.cpp:5-17)
    ok = lib.gs_default_config()
    assert lib.gs_validate_config(C.byref(ok), C.byref(mask)) == _lib.GS_OK and mask.value == 0


def test_no_cpu_fallback_without_device():
    """Without a B200 the context refuses to exist: there is no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1907_04834_b200 import DeviceError, Geoshoot
    with pytest.raises(DeviceError):
        Geoshoot(0)


def test_config_error_mirrors_reference(ref):
    from paper_1907_04834_b200 import _lib
    lib = _lib.load()
    for args in [(-1.0, 1.0, 5, 3.0), (1.0, 0.0, 0, 3.0), (1.0, 1.0, 5, -2.0), (0.0, -1.0, 0, 0.0)]:
        cfg = _lib.gs_config(args[0], args[1], args[2], 0, args[3], 0, 0)
        mask = C.c_uint32()
        lib.gs_validate_config(C.byref(cfg), C.byref(mask))
        assert mask.value == ref.validate_config(*args)
