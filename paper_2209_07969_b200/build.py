"""In-tree build of ``libpfb200.so`` for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "pf_api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in (
    "pf_device.cuh", "pf_kernels.cuh", "pf_cg.cuh", "pf_march.cuh", "pf_mg.cuh", "pf_mgs.cuh", "pf_mgd.cuh", "pf_st.cuh",
    "pf_comm.h")] + [
    os.path.join(ROOT, "include", "pf_b200.h")]
OUT = os.path.join(HERE, "libpfb200.so")

NCCL_INCLUDE = None
for _cand in ("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include",
              "/usr/include"):
    if os.path.exists(os.path.join(_cand, "nccl.h")):
        NCCL_INCLUDE = _cand
        break

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile libpfb200.so.  `defines`/`out`: experiment variants (e.g. -DPFB_USE_RING=1 into
    another file, loaded through PFB200_LIB); the default library never uses them."""
    if out is None and not defines and not force and up_to_date():
        return OUT
    target = out or OUT
    inc = ["-I", NCCL_INCLUDE] if NCCL_INCLUDE else []
    cmd = [nvcc(), *NVCC_FLAGS, *inc, *[f"-D{d}" for d in defines], "-ldl", "-lpthread",
           "-o", target + ".tmp", *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}): {' '.join(cmd)}")
    os.replace(target + ".tmp", target)
    if out is not None:
        return target
    log = os.path.join(HERE, "csrc", "ptxas_sm100a.log")
    with open(log, "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    return OUT


if __name__ == "__main__":
    argv = sys.argv[1:]
    defs = [a[2:] for a in argv if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in argv if a.startswith("--out=")]
    print(build(force="--force" in argv, verbose=True, defines=defs,
                out=outs[0] if outs else None))
