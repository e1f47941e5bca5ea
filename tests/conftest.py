import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2311_04499_b200", "libcovap_b200.so")
    if not os.path.exists(lib):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2311_04499_b200", "csrc")],
                       check=True)
    from oracle import oracle as o
    if not os.path.exists(o.ORACLE_SO) or (os.path.isdir(o.REF_SRC) and not os.path.exists(o.REF_SO)):
        o.build(ref=True)


_ensure_built()


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("reference library (oracle/_ref) not built here")
    return Ref()


@pytest.fixture(scope="session")
def covap():
    import paper_2311_04499_b200 as c
    return c


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
