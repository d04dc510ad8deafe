"""The C++ host API (namespace cavac over the C ABI) on the device, and the
reference's own acceptance gate linked against it (tools/dropin)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_host_api(cvk, tmp_path):
    exe = tmp_path / "test_host_api"
    pkg = os.path.join(ROOT, "paper_2112_00087_b200")
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp"), "-L" + pkg, "-lcavac_host",
                           "-lcavac_b200", "-Wl,-rpath," + pkg, "-o", str(exe)])
    r = subprocess.run([str(exe), os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


ACCEPT = os.path.join(ROOT, "dropin", "_bin", "acceptance_b200")


@pytest.mark.skipif(not os.path.exists(ACCEPT), reason="drop-in acceptance binary not built here")
def test_reference_acceptance_gate_on_b200(cvk):
    """proj/tests/acceptance.cpp with the B200 numkit/krylov/schwarz: every
    criterion must pass, including 7 (bench_solvers, pipeline.cpp:227-293),
    which throws unless both ExecModes give identical iteration counts and
    asserts Parallel >= Sequential speed at the finest ladder point.  On the
    device both modes give the reference's iterates bit for bit (Sequential:
    one thread per reduction; Parallel: the terms formed by a whole CTA)."""
    r = subprocess.run([ACCEPT], cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout
    status = dict((m.group(2), m.group(1)) for m in re.finditer(r"\[(PASS|FAIL)\] (.+?) \(", out))
    assert len(status) == 8, out
    assert all(v == "PASS" for v in status.values()), out
    assert r.returncode == 0, out + r.stderr
