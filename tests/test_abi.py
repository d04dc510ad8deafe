"""The C-ABI library: built for sm_100a, loads, exports every symbol
include/cavac_b200.h declares, and fails loudly (no CPU fallback) without a
GPU.  CPU only -- no compute calls."""
import ctypes
import os
import subprocess

import pytest

from conftest import ROOT, has_gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2112_00087_b200 import _lib, build
    build.build()
    return _lib


def test_exports_every_declared_symbol(lib):
    L = lib.load()
    names = lib.declared_symbols()
    assert len(names) >= 30
    missing = [s for s in names if not hasattr(L, s)]
    assert not missing, missing


def test_sm100a_cubin_and_no_fma(lib):
    out = subprocess.check_output(["cuobjdump", "-lelf", lib.LIB_PATH], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", "-fun", "k_inv_diag", lib.LIB_PATH], text=True)
    assert "DFMA" not in sass  # --fmad=false: the reference object code has no FMA


def test_names_and_codes(lib):
    L = lib.load()
    assert L.cvk_abi_version() == 2
    assert L.cvk_solver_name(2) == b"tfqmr"
    assert L.cvk_solver_from_name(b"bicgstab_l") == 1
    assert L.cvk_solver_from_name(b"gmres2") == -6
    assert b"allowed" in L.cvk_last_error()
    assert L.cvk_breakdown_name(3) == b"omega breakdown"


def test_cvk_opts_layout(lib):
    """cvk_opts as declared in include/cavac_b200.h (ABI 2 adds warm)."""
    import ctypes as C
    assert C.sizeof(lib.CvkOpts) == 48
    assert lib.CvkOpts.warm.offset == 40
    assert set(lib.OPTIONS.values()) == set(range(1, 14))


def test_no_environment_switches_in_native_code():
    """Execution paths are chosen by cvk_ctx_set_option, never by getenv."""
    src = os.path.join(ROOT, "paper_2112_00087_b200", "csrc")
    for f in os.listdir(src):
        assert "getenv" not in open(os.path.join(src, f)).read(), f


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_fails_loudly_without_gpu(lib):
    L = lib.load()
    h = ctypes.c_void_p()
    assert L.cvk_ctx_create(0, ctypes.byref(h)) == -2
    import paper_2112_00087_b200 as P
    with pytest.raises(Exception):
        P.Device(0)


def test_product_does_not_import_oracle():
    """The product never loads the checker (oracle/, oracle/_ref)."""
    import re
    pat = re.compile(r"(from\s+oracle|import\s+oracle|liboracle|libcavac_ref|oracle/_ref)")
    pkg = os.path.join(ROOT, "paper_2112_00087_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(root, f)).read()
                assert not pat.search(txt), f
