import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: longer parity cases")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the oracle (and the product library when missing) once."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    if os.path.isdir("/root/reference/proj"):  # the reference's own build (oracle/_ref), here only
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "-f", "Makefile.ref"], check=True)
    lib = os.path.join(ROOT, "paper_2510_02382_b200", "libctfiss.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2510_02382_b200", "csrc")], check=True)
    yield


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    return oracle
