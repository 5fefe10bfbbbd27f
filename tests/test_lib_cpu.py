"""CPU-side checks of the C-ABI library (no GPU): it is built for sm_100a, loads, and exports every
entry point include/pas.h declares; argument validation that needs no device fails cleanly."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pas.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2502_06798_b200 import build
    build.build()
    from paper_2502_06798_b200 import pas
    return pas


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pas_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("pas_cache_load", "pas_set_fractions", "pas_route_batch", "pas_plan_stats",
                 "pas_create", "pas_destroy", "pas_set_bands"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    for name in _declared():
        assert hasattr(so, name), name
    assert set(_declared()) == set(lib.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in _declared():
        assert re.search(r"\bT " + name + r"\b", out), name


def test_built_for_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)", out)
    sass = subprocess.run(["cuobjdump", "-sass", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass   # tcgen05 + TMA + TMEM loads


def test_version_and_clean_failures_without_gpu(lib):
    assert "sm_100a" in lib.pas_version()
    with pytest.raises(lib.PasError) as ei:
        lib.pas_create(device=0)          # no CUDA device in this container
    assert ei.value.status in (-1, -8)
    with pytest.raises(lib.PasError):
        lib.pas_create(d=100)             # d must be a multiple of 64
    st = lib.lib.pas_route_batch(None, None, 0, 0, None, None)
    assert st == -1                       # null context -> PAS_ERR_ARG, nothing enqueued


def test_binding_fails_loudly_without_library(tmp_path):
    """No silent CPU fallback: importing the binding with no library raises ImportError."""
    code = ("import os, sys; os.environ['PAS_LIB'] = %r; sys.path.insert(0, %r)\n"
            "try:\n    import paper_2502_06798_b200.pas\nexcept ImportError as e:\n    print('raised', e)\n")
    out = subprocess.run([sys.executable, "-c", code % (str(tmp_path / "missing.so"), ROOT)],
                         capture_output=True, text=True)
    assert "raised" in out.stdout, out.stdout + out.stderr


def test_binding_rejects_bad_embedding_layouts(lib):
    """the binding checks the rows K1 will read with vector loads -- width d, contiguous,
    on the right side of the PCIe bus -- before any pointer crosses the ABI."""
    import torch
    fake = ctypes.c_void_p(12345)
    lib._CTX_D[fake.value] = 768
    try:
        with pytest.raises(ValueError):
            lib._rows(fake, torch.zeros(4, 512), device=False)           # wrong d
        with pytest.raises(ValueError):
            lib._rows(fake, torch.zeros(768, 4).t(), device=False)       # strided view
        with pytest.raises(ValueError):
            lib._rows(fake, torch.zeros(4, 768), device=True)            # host tensor on a device path
        assert lib._rows(fake, torch.zeros(4, 768), device=False).value is not None
    finally:
        lib._CTX_D.pop(fake.value)


def test_nvtx_stage_ranges_built_in(lib, tmp_path):
    """The six stage range names are in the library (SURVEY 5 tracing row; exercised on the GPU by
    tests/test_gpu_nvtx.py) and the test-only injection probe builds and exports its entry point."""
    data = open(lib.LIB_PATH, "rb").read()
    for name in ("K1 normalise", "K2 similarity + top-k", "K3/K4 merge + optimal-K", "K5 plan", "K6 redirect",
                 "K7 route-and-batch"):
        assert b"pas " + name.encode() + b"\0" in data, name
    probe = str(tmp_path / "probe.so")
    subprocess.run(["gcc", "-shared", "-fPIC", "-O2", "-o", probe, os.path.join(ROOT, "tests", "native", "nvtx_probe.c")],
                   check=True)
    out = subprocess.run(["nm", "-D", "--defined-only", probe], capture_output=True, text=True).stdout
    assert re.search(r"\bT InitializeInjectionNvtx2\b", out)
