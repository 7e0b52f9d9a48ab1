"""Fixed-length PCG launches on the cfg5 layout (8192^2) for ncu captures (one launch each)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200 import meshing  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
case = C.get_case(name)
if name == "cfg5":
    lay = meshing.StructuredLayout.rectangle(8192, 8192, 1000.0 / 8192, 1000.0 / 8192)
else:
    lay = meshing.StructuredLayout.from_mesh(C.build_mesh(case, C.b200_api()))
s = DeviceSession(lay, C.material(case, C.b200_api()),
                  C.b200_api().SolverConfig(tol_st=case.tol_st), device=0)
rng = np.random.default_rng(7)
nn = lay.n_nodes
s.push(u=1e-4 * rng.standard_normal(2 * nn), d=0.5 * rng.random(nn), d_prev=np.zeros(nn))
s.refresh_gp()
for phys in ("momentum", "evolution"):
    ms, it = s.bench_cg(phys, iters)
    print(phys, it, "iterations", round(1e3 * ms / it, 2), "us/iter", flush=True)
