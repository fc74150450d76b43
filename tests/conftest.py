import glob
import os
import subprocess
import sys
import time

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running oracle case")
    _wait_for_cuda()


def _has_gpu_node():
    return bool(glob.glob("/dev/nvidia[0-9]*"))


def _wait_for_cuda(tries=6, pause=10.0):
    """On a GPU box, CUDA can fail to initialise in the first seconds after the box is handed over;
    the failure is cached per process.  Probe in child processes (before this one touches CUDA)
    until it comes up, so GPU tests never skip on a box that has a GPU."""
    if not _has_gpu_node():
        return
    probe = [sys.executable, "-c", "import sys, torch; sys.exit(0 if torch.cuda.is_available() else 1)"]
    for _ in range(tries):
        if subprocess.run(probe).returncode == 0:
            return
        time.sleep(pause)


@pytest.fixture(scope="session")
def cuda_lib():
    """The built C-ABI library through its Python binding (GPU tests only)."""
    import torch
    if not torch.cuda.is_available():
        if _has_gpu_node():
            pytest.fail("a GPU device node exists but CUDA did not initialise")
        pytest.skip("no CUDA device")
    import paper_2304_14021_b200 as pd
    return pd
