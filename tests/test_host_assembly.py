"""The C++ host assembly (cpp/helmholtz_host.cpp, reference helmholtz.cpp:14-168)
against helmholtz.py, which test_helmholtz.py pins to the golden system and
to the oracle: bitwise CSR, values and right-hand sides, with and without
wall admittance, plus the manufactured problem.  Runs on CPU: the host
library only loads the CUDA library, it makes no device call here."""
import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2112_00087_b200 import helmholtz as H

PKG = os.path.join(ROOT, "paper_2112_00087_b200")


@pytest.fixture(scope="module")
def dumper(tmp_path_factory):
    if not os.path.exists(os.path.join(PKG, "libcavac_host.so")):
        pytest.skip("libcavac_host.so not built")
    exe = tmp_path_factory.mktemp("dump") / "dump_assembly"
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "dump_assembly.cpp"), "-L" + PKG, "-lcavac_host",
                           "-lcavac_b200", "-Wl,-rpath," + PKG, "-o", str(exe)])
    return exe


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("h,f,adm,mn", [(0.1, 13.0, 0j, (1, 1)), (0.05, 100.0, 0.01 + 0j, (2, 3)),
                                        (0.013, 250.0, 0.02 - 0.005j, (3, 1))])
def test_host_assembly_bitwise(dumper, tmp_path, h, f, adm, mn):
    pre = str(tmp_path / "d")
    out = subprocess.run([str(dumper), pre, repr(h), repr(f), repr(adm.real), repr(adm.imag), str(mn[0]), str(mn[1])],
                         capture_output=True, text=True, check=True).stdout.split()
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    assert [int(v) for v in out] == [g.nx, g.ny, g.roof_begin, g.roof_end]
    om = 2 * math.pi * f
    i = np.arange(g.roof_size())
    dirichlet = (1.0 + 0.01 * i) + 1j * (-0.5 * i)
    p = H.assemble(g, om, 340.0, dirichlet)
    mp = H.manufactured_problem(g, mn[0], mn[1], om, 340.0)
    load = lambda s, t: np.fromfile(pre + s, t)  # noqa: E731
    for tag, A, b in (("_asm", p.A, p.b), ("_man", mp.problem.A, mp.problem.b)):
        assert np.array_equal(load(tag + "_rp.bin", np.int64), A.row_offsets.astype(np.int64))
        assert np.array_equal(load(tag + "_ci.bin", np.int64), A.col_indices.astype(np.int64))
        assert np.array_equal(bits(load(tag + "_v.bin", np.complex128)), bits(A.values))
        assert np.array_equal(bits(load(tag + "_b.bin", np.complex128)), bits(b))
    assert np.array_equal(bits(load("_man_exact.bin", np.complex128)), bits(mp.exact))
