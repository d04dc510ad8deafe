import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")  # the reference's own fixtures, byte for byte
FIXTURES = os.path.join(ROOT, "tests", "fixtures")  # fixtures made here from the reference (tools/)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def golden(oracle):
    rp, ci, v = oracle.read_matrix_market(os.path.join(GOLDEN, "system.mtx"))
    b = oracle.read_vector_csv(os.path.join(GOLDEN, "rhs.csv"))
    sol_text = open(os.path.join(GOLDEN, "solution.csv")).read()
    return {"rp": rp, "ci": ci, "v": v, "b": b, "solution_csv": sol_text,
            "x": oracle.read_vector_csv(os.path.join(GOLDEN, "solution.csv"))}


@pytest.fixture(scope="session")
def cvk():
    if not has_gpu():
        pytest.skip("no GPU")
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import build
    build.build()
    return P


@pytest.fixture
def knobs(cvk):
    """knobs(phased_min_n=0, stream=0, ...): execution-path options of the
    default device context (cvk_ctx_set_option), restored after the test."""
    entered = []

    def set_(**kw):
        cm = cvk.path_options(**kw)
        cm.__enter__()
        entered.append(cm)

    yield set_
    for cm in reversed(entered):
        cm.__exit__(None, None, None)
