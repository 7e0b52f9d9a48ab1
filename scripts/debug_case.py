"""Per-step comparison GPU vs golden reference vs oracle (debug helper)."""
import sys, os, numpy as np, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C
from oracle.phasefield_oracle import oracle_api
case, scheme = sys.argv[1], sys.argv[2]
z = np.load(f"tests/golden/run_{case}_{scheme}.npz")
tab = z["table"]
pb = C.setup(C.get_case(case), C.b200_api())
from paper_2209_07969_b200.session import DeviceSession
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
s.push_state(pb.state)
oc = C.setup(C.get_case(case), oracle_api("cg"))
od = C.setup(C.get_case(case), oracle_api())
for k, row in enumerate(tab, 1):
    st = s.step(scheme, pb.bcs, pb.pins)
    f = s.reaction_force(pb.mesh.boundary_sets["top"] if "top" in pb.mesh.boundary_sets else pb.mesh.boundary_sets["load_zone"], 1 if case != "shear32" else 0)
    r1 = oc.api.staggered_step(oc.disc, oc.state, scheme, oc.bcs, oc.params, oc.config, oc.pins)
    r2 = od.api.staggered_step(od.disc, od.state, scheme, od.bcs, od.params, od.config, od.pins)
    g = s.pull()
    print(f"step {k:3d} gpu ({st.n_stag},{st.n_nr_u},{st.n_nr_d},{st.spd_fallbacks}) ref {tuple(int(x) for x in row[1:5])} "
          f"ocg ({r1.n_stag},{r1.n_nr_u},{r1.n_nr_d},{r1.spd_fallbacks}) odir ({r2.n_stag},{r2.n_nr_u},{r2.n_nr_d},{r2.spd_fallbacks}) "
          f"F {f:.6f} ref {row[7]:.6f} | dgpu-docg {np.abs(g['d']-oc.state.d).max():.2e} dgpu-dodir {np.abs(g['d']-od.state.d).max():.2e} "
          f"cgit u/d {st.cg_iters_u}/{st.cg_iters_d} ocg_it {r1.cg_iters_u}/{r1.cg_iters_d}", flush=True)
g = s.pull()
dd = np.abs(g["d"] - z["final_d"]); i = int(dd.argmax())
print("max |d - ref| at node", i, pb.mesh.nodes[i], g["d"][i], z["final_d"][i], "n_nodes", pb.mesh.n_nodes)
print("gpu hist last step", s.last_history[:5], s.last_history[-5:])
n = C.get_case(case).mesh[1]
if C.get_case(case).mesh[0] == "notched":
    for j in (n//2-1, n//2, n//2+1):
        print("gpu row", j, np.round(g["d"][j*(n+1):(j+1)*(n+1)], 3))
    print("gpu dups", np.round(g["d"][(n+1)*(n+1):], 3))
