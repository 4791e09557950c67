import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # a fresh checkout has no built artefacts: build the library (nvcc cross-compiles
    # without a GPU) and the oracle checkers before anything imports them
    lib = os.path.join(ROOT, "paper_2512_05516_b200", "libsoaforge_b200.so")
    oracle_lib = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        from paper_2512_05516_b200 import build as B
        B.build()
    if not os.path.exists(oracle_lib):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
