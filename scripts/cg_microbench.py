"""Per-iteration time of the persistent PCG kernels on a given case (perf experiments)."""
import sys, os, json, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200.session import DeviceSession
case = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pb = C.setup(C.get_case(case), C.b200_api())
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
s.push_state(pb.state)
s.step("ST", pb.bcs, pb.pins)
info = s.device_info()
for k in range(steps):
    s.flush_l2()
    st = s.step("ST", pb.bcs, pb.pins)
    nn = pb.mesh.n_nodes
    us_u = 1e3 * st.kernel_ms_u / max(st.cg_iters_u, 1)
    us_d = 1e3 * st.kernel_ms_d / max(st.cg_iters_d, 1)
    print(json.dumps({"lib": os.environ.get("PFB200_LIB", "default"), "case": case, "n_nodes": nn,
        "step_ms": round(st.step_ms, 2), "n_stag": st.n_stag, "iters_u": st.cg_iters_u, "iters_d": st.cg_iters_d,
        "us_per_iter_u": round(us_u, 2), "us_per_iter_d": round(us_d, 2),
        "GBs_u": round(168 * nn / us_u / 1e3, 1), "GBs_d": round((72 * nn + 32 * pb.mesh.n_elems) / us_d / 1e3, 1),
        "launches": st.launches, **info}), flush=True)
