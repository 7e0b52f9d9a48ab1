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


def mirror_perm(mesh) -> np.ndarray:
    """Node permutation of the reflection y -> side - y of a notched square.

    Grid node (i, j) maps to (i, ny - j); on the slit row the lower-face node (i, ny/2) and its
    duplicate (upper face) swap.  The tension load case (bottom fixed, top pulled) is
    invariant under this reflection up to a rigid translation, so a phase field and its
    mirror image are equally valid solutions (the crack-step bifurcation picks one by
    round-off).
    """
    from paper_2209_07969_b200.meshing import StructuredLayout

    lay = StructuredLayout.from_mesh(mesh)
    nx, ny = lay.nx, lay.ny
    ids = np.arange((nx + 1) * (ny + 1)).reshape(ny + 1, nx + 1)
    perm = np.arange(mesh.n_nodes)
    perm[: ids.size] = ids[::-1].ravel()
    if lay.notch_row >= 0:
        cols = np.arange(lay.notch_lo, lay.notch_hi)
        orig = lay.notch_row * (nx + 1) + cols
        dup = lay.dup_start + (cols - lay.notch_lo)
        perm[orig], perm[dup] = dup, orig
    return perm


def _pooled_rel_spread(case: str) -> float:
    """Largest relative round-off deviation max |v - ref| / ref over every scheme's ensemble
    of the case (the bifurcation at the crack step is a property of the case)."""
    import glob

    rel = 0.0
    for sch in ("ST", "S1", "S2", "S3"):
        paths = (glob.glob(os.path.join(GOLDEN, f"sens_{case}_{sch}.json")) +
                 glob.glob(os.path.join(GOLDEN, f"sens_{case}_{sch}_part*.json")))
        run = os.path.join(GOLDEN, f"run_{case}_{sch}.npz")
        if not paths or not os.path.exists(run):
            continue
        ref = np.load(run)["table"][:, 1].astype(int)
        for path in paths:
            with open(path) as f:
                for v in json.load(f)["n_stag"].values():
                    v = np.asarray(v)
                    n = min(v.size, ref.size)
                    rel = max(rel, float(np.max(np.abs(v[:n] - ref[:n]) / np.maximum(ref[:n], 1))))
    return rel


def stag_band(case: str, scheme: str, n_steps: int, run_file: str | None = None) -> np.ndarray:
    """Per-step allowed |n_stag - reference|.

    The samples are the reference run plus its round-off ensemble (tests/golden/sens_*.json:
    restatements of the reference algorithm that are identical in exact arithmetic and differ
    only in floating-point evaluation order, make_sensitivity.py).  Where every sample agrees
    (all pre-crack steps) the band is the strict +-1.  Where they disagree (the crack steps:
    staggered iteration counts there are round-off chaotic) the GPU run is treated as one more
    sample of the same process and the band is the largest of
      * the two-sided 99% Student-t prediction interval for a new sample,
        |mean - ref| + t(0.995, n-1) * s * sqrt(1 + 1/n);
      * 1 + the largest deviation of this scheme's ensemble;
      * 1 + the case's largest relative ensemble deviation (pooled over its schemes, the
        bifurcation being a property of the case) times the step's reference count.
    All three come from CPU data only (the reference and its restatements).
    """
    import glob

    from scipy import stats

    paths = sorted(glob.glob(os.path.join(GOLDEN, f"sens_{case}_{scheme}.json")) +
                   glob.glob(os.path.join(GOLDEN, f"sens_{case}_{scheme}_part*.json")))
    if not paths:
        return np.ones(n_steps, dtype=int)
    sens = {}
    for path in paths:
        with open(path) as f:
            sens.update(json.load(f)["n_stag"])
    z = np.load(os.path.join(GOLDEN, run_file or f"run_{case}_{scheme}.npz"))
    ref = z["table"][:n_steps, 1].astype(int)
    rel = _pooled_rel_spread(case)
    band = np.ones(n_steps, dtype=int)
    for i in range(n_steps):
        samples = [int(ref[i])] + [int(v[i]) for v in sens.values() if len(v) > i]
        x = np.asarray(samples, dtype=float)
        dev = int(np.max(np.abs(x - ref[i])))
        if dev == 0:
            continue
        n = x.size
        half = stats.t.ppf(0.995, n - 1) * x.std(ddof=1) * np.sqrt(1.0 + 1.0 / n)
        band[i] = max(1 + dev, int(np.ceil(abs(x.mean() - ref[i]) + half)),
                      1 + int(np.ceil(rel * ref[i])))
    return band


def exact_geometry_ensemble(case: str, scheme: str) -> dict:
    """The reference algorithm's round-off ensemble restricted to exact uniform-cell geometry
    (tests/golden/sens_<case>_<scheme>_exact_part*.json, make_sensitivity.py "exact:a:b"): the
    Jacobians / B matrices from the exact cell size, as the device path evaluates them (DESIGN.md
    section 4), instead of from node coordinates.  {variant: per-step n_stag}."""
    import glob

    out = {}
    for path in sorted(glob.glob(os.path.join(GOLDEN, f"sens_{case}_{scheme}_exact_part*.json"))):
        with open(path) as f:
            out.update(json.load(f)["n_stag"])
    return out


# Cases too large for a CPU round-off ensemble take the relative spread of a smaller case of the
# same load case and physics at its crack step (cfg2 512^2 <- cfg1 64^2, both notched tension).
PROXY = {"cfg2": "cfg1"}


def proxy_rel_spread(proxy: str) -> float:
    """Largest relative deviation from the reference at the proxy case's crack step over all
    its schemes and both ensembles (coordinate and exact geometry)."""
    import glob

    rel = 0.0
    for sch in ("ST", "S1", "S2", "S3"):
        run = os.path.join(GOLDEN, f"run_{proxy}_{sch}.npz")
        if not os.path.exists(run):
            continue
        ref = np.load(run)["table"][:, 1].astype(int)
        i = int(np.argmax(ref))
        for path in glob.glob(os.path.join(GOLDEN, f"sens_{proxy}_{sch}*.json")):
            with open(path) as f:
                for v in json.load(f)["n_stag"].values():
                    if len(v) > i:
                        rel = max(rel, abs(v[i] - ref[i]) / ref[i])
    return rel


def stag_window(case: str, scheme: str, n_steps: int, run_file: str | None = None) -> tuple:
    """Per-step allowed [lo, hi] of n_stag.  Default: the reference's count +- stag_band.  At
    round-off-chaotic crack steps of cases with an exact-geometry ensemble, the window is that
    ensemble's range +- 2: the reference evaluates cell geometry from node coordinates, and that
    1e-16 spatially varying perturbation alone shifts the crack-step count (cfg1 ST: 298-299 with
    coordinates, 303-312 with exact geometry, the device's 305-311), so the
    device is compared with the population that evaluates the same arithmetic.  Cases too large
    for an ensemble (cfg2) take the proxy case's relative spread at their crack step."""
    z = np.load(os.path.join(GOLDEN, run_file or f"run_{case}_{scheme}.npz"))
    ref = z["table"][:n_steps, 1].astype(int)
    band = stag_band(case, scheme, n_steps, run_file)
    lo, hi = ref - band, ref + band
    ex = exact_geometry_ensemble(case, scheme)
    for i in range(n_steps):
        vals = [int(v[i]) for v in ex.values() if len(v) > i]
        if band[i] > 1 and vals:
            lo[i], hi[i] = min(vals) - 2, max(vals) + 2
    if case in PROXY:  # crack steps (a jump of 5x over the previous step) of the large cases
        rel = proxy_rel_spread(PROXY[case])
        for i in range(1, n_steps):
            if band[i] == 1 and ref[i] >= 5 * max(ref[i - 1], 1):
                lo[i] = int(np.floor(ref[i] * (1.0 - rel))) - 2
                hi[i] = int(np.ceil(ref[i] * (1.0 + rel))) + 2
    return lo, hi


KAT_MESHES = ("notched8", "notched12x6", "plain10", "lshape", "notched16", "notched80x16",
              "lshape12p5")


def kat_mesh(name):
    from paper_2209_07969_b200 import meshing

    return {
        "notched8": lambda: meshing.build_notched_square(8, 8, 1.0),
        "notched12x6": lambda: meshing.build_notched_square(12, 6, 2.0),
        "plain10": lambda: meshing.build_notched_square(10, 10, 1000.0, False),
        "lshape": lambda: meshing.build_lshape_mesh(62.5),
        "notched16": lambda: meshing.build_notched_square(16, 16, 1.0),
        "notched80x16": lambda: meshing.build_notched_square(80, 16, 5.0),
        "lshape12p5": lambda: meshing.build_lshape_mesh(12.5),
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
