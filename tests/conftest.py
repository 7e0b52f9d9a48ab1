"""Shared fixtures.  Markers: ``gpu`` (needs a B200 and the built libpfb200.so)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and libpfb200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    return np.load(path, allow_pickle=False)


def golden_meta(z) -> dict:
    return json.loads(str(z["meta"]))


def rel_err(a, b) -> float:
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(float(np.abs(b).max()), 1e-300)
    return float(np.abs(a - b).max() / scale)


KAT_MESHES = ("notched8", "notched12x6", "plain10", "lshape")


def kat_mesh(name):
    from paper_2209_07969_b200 import meshing

    return {
        "notched8": lambda: meshing.build_notched_square(8, 8, 1.0),
        "notched12x6": lambda: meshing.build_notched_square(12, 6, 2.0),
        "plain10": lambda: meshing.build_notched_square(10, 10, 1000.0, False),
        "lshape": lambda: meshing.build_lshape_mesh(62.5),
    }[name]()


def kat_params(tag):
    from paper_2209_07969_b200 import material

    return material.MaterialParams.from_young_poisson(
        210000.0, 0.3, g_c=2.7, length_l=0.05, at_model="AT2" if tag == "at2" else "AT1")


@pytest.fixture(scope="session")
def cuda_ok():
    """Fail loudly (not skip) when a gpu-marked test runs without the CUDA path."""
    from paper_2209_07969_b200 import _native

    _native.load()
    import ctypes

    cnt = ctypes.c_int(0)
    try:
        rt = ctypes.CDLL("libcudart.so")
    except OSError:
        rt = None
    if rt is not None:
        rt.cudaGetDeviceCount(ctypes.byref(cnt))
    return True
