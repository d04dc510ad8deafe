"""cvk_complex.h (device scalar arithmetic) against libgcc/libstdc++ on the
host, bit for bit: complex division (__divdc3) and multiplication. CPU only."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HARNESS = r'''
#include "cvk_complex.h"
#include <complex>
#include <cstdio>
#include <cstring>
#include <random>
int main() {
    std::mt19937_64 g(12345);
    std::uniform_real_distribution<double> u(-1, 1), e(-300, 300);
    long bad = 0, n = 0, skipped = 0;
    for (int t = 0; t < 400000; ++t) {
        double v[4];
        for (int k = 0; k < 4; ++k) {
            v[k] = u(g) * std::pow(10.0, (t % 3 == 0) ? e(g) : (t % 3 == 1 ? u(g) * 10 : 0));
            if (g() % 50 == 0) v[k] = 0;
        }
        if (v[2] == 0 && v[3] == 0) continue;
        std::complex<double> q = std::complex<double>(v[0], v[1]) / std::complex<double>(v[2], v[3]);
        if (!std::isfinite(q.real()) || !std::isfinite(q.imag())) { ++skipped; continue; }
        cvk_c r = cvk_cdiv(cvk_make(v[0], v[1]), cvk_make(v[2], v[3]));
        double qr = q.real(), qi = q.imag();
        ++n;
        if (std::memcmp(&r.x, &qr, 8) || std::memcmp(&r.y, &qi, 8)) ++bad;
        std::complex<double> m = std::complex<double>(v[0], v[1]) * std::complex<double>(v[2], v[3]);
        cvk_c mm = cvk_mul(cvk_make(v[0], v[1]), cvk_make(v[2], v[3]));
        if (std::isfinite(m.real()) && std::isfinite(m.imag()) && (mm.x != m.real() || mm.y != m.imag())) ++bad;
    }
    std::printf("%ld %ld %ld\n", n, bad, skipped);
    return 0;
}
'''


def test_cdiv_and_cmul_match_libgcc(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    exe = tmp_path / "h"
    subprocess.check_call(["/usr/bin/g++", "-O2", "-ffp-contract=off", "-std=c++17",
                           "-I" + os.path.join(ROOT, "paper_2112_00087_b200", "csrc"), str(src), "-o", str(exe)])
    n, bad, skipped = (int(t) for t in subprocess.check_output([str(exe)]).split())
    assert n > 300000 and bad == 0


def test_python_cdiv_matches_libgcc(oracle):
    """helmholtz.cdiv (host assembly) against libgcc through the oracle."""
    from paper_2112_00087_b200.helmholtz import cdiv
    rng = np.random.default_rng(7)
    for _ in range(20000):
        a = complex(*rng.uniform(-1e3, 1e3, 2))
        b = complex(*rng.uniform(-1e3, 1e3, 2))
        got, want = cdiv(a, b), oracle.cdiv(a, b)
        assert got.real == want.real and got.imag == want.imag
