import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libsv.so")
    config.addinivalue_line("markers", "slow: long CPU test (oracle at the 7B shape)")


@pytest.fixture(scope="session")
def svlib():
    """libsv.so, built in-tree if missing (the CUDA path has no fallback)."""
    from paper_2505_21594_b200 import sv
    if not os.path.exists(sv.LIB_PATH):
        import subprocess
        subprocess.check_call([os.path.join(ROOT, "paper_2505_21594_b200", "csrc", "build.sh")])
    return sv.lib()
