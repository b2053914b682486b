import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def orc():
    """The C restatement (oracle/chebfd_oracle.c); built on demand."""
    import oracle
    if not os.path.exists(oracle.ORACLE_SO):
        subprocess.run(["make", "-s", "-C", oracle.HERE, "oracle"], check=True)
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), skipped where it was not built."""
    import oracle
    if not oracle.ref_available():
        if os.path.isdir("/root/reference/proj"):
            subprocess.run(["make", "-s", "-C", oracle.HERE, "ref"], check=True)
        else:
            pytest.skip("oracle/_ref/libchebfd_ref.so not built here")
    return oracle.Ref(threads=1)


@pytest.fixture(scope="session")
def lib_built():
    so = os.path.join(ROOT, "paper_1510_04895_b200", "libchebfd_b200.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1510_04895_b200", "csrc")],
                       check=True)
    return so


@pytest.fixture(scope="session")
def ctx(lib_built):
    import paper_1510_04895_b200 as cf
    c = cf.Context(0)
    yield c
    c.close()
