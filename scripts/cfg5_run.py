"""BASELINE configs[4] (8192^2 cells, 67.1 M nodes, 201 M DOFs, 256 seeded pre-cracks, biaxial
loading) on ONE B200 through the device session, without materialising the reference's element
arrays: the row-compact layout of the plain square (StructuredLayout.rectangle), boundary dofs
from the layout, the zero state and the pre-cracks built on the device (DeviceSession.init_state,
configs.precrack_segments).  Prints one JSON line per load step (n_stag, Newton counts, PCG iterations, step ms,
reactions).

    python scripts/cfg5_run.py [n_steps] [scheme]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200 import meshing  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scheme = sys.argv[2] if len(sys.argv) > 2 else "S1"
case = C.get_case("cfg5")
_, nx, ny, side, _ = case.mesh
h = side / nx
t0 = time.perf_counter()
lay = meshing.StructuredLayout.rectangle(nx, ny, h, h)
ids = np.arange(lay.n_nodes, dtype=np.int64).reshape(ny + 1, nx + 1)
segs, radius = C.precrack_segments(case)
api = C.b200_api()
params = C.material(case, api)
config = api.SolverConfig(tol_st=case.tol_st)
left, right, bottom, top = ids[:, 0], ids[:, -1], ids[0, :], ids[-1, :]
bcs = [(2 * left, 0.0), (2 * bottom + 1, 0.0), (2 * right, case.inc), (2 * top + 1, case.inc)]
setup_s = time.perf_counter() - t0
s = DeviceSession(lay, params, config, device=0)
nn, ne = lay.n_nodes, lay.n_elems
t1 = time.perf_counter()
s.init_state(segs, radius, side, side)  # zero state + pre-cracks built on the device
init_s = time.perf_counter() - t1
print(json.dumps({"case": "cfg5", "n_nodes": nn, "n_cells": ne, "dofs": 3 * nn,
                  "precrack_segments": int(segs.shape[0]), "host_setup_s": round(setup_s, 2),
                  "device_init_s": round(init_s, 3),
                  "mg": s.mg_info()}), flush=True)
for k in range(1, n_steps + 1):
    st = s.step(scheme, bcs)
    fx = s.reaction_force(right, 0)
    fy = s.reaction_force(top, 1)
    print(json.dumps({"step": k, "n_stag": st.n_stag, "n_nr_u": st.n_nr_u, "n_nr_d": st.n_nr_d,
                      "cg_iters_u": st.cg_iters_u, "cg_iters_d": st.cg_iters_d,
                      "step_ms": round(st.step_ms, 1), "F_right_x": fx, "F_top_y": fy,
                      "dof_iter_per_s": 3 * nn * st.n_stag / (st.step_ms / 1e3)}), flush=True)
s.close()
