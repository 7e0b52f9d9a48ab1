"""cfg2 (512^2 tension, S1) through all 65 load steps on the device: per-step n_stag and top
reaction, wall time; run with PFB200_MG=0 / 1 to compare the Jacobi and multigrid momentum
solvers through the crack step."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200.session import DeviceSession
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
scheme = sys.argv[2] if len(sys.argv) > 2 else "S1"
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else None
pb = C.setup(C.get_case(name), C.b200_api())
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
s.push_state(pb.state)
_, nodes, comp = pb.reactions[0]
rows, t0 = [], time.perf_counter()
for k in range(nsteps or pb.case.n_steps):
    st = s.step(scheme, pb.bcs, pb.pins)
    rows.append((st.n_stag, round(s.reaction_force(nodes, comp), 9), round(st.step_ms, 2)))
wall = time.perf_counter() - t0
print(json.dumps({"case": name, "scheme": scheme, "mg": s.mg_info(), "wall_s": round(wall, 2),
                  "total_n_stag": sum(r[0] for r in rows), "n_stag": [r[0] for r in rows],
                  "F": [r[1] for r in rows], "step_ms": [r[2] for r in rows]}))
