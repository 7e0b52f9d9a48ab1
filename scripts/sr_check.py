import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200.session import DeviceSession
res = {}
for flag in ("0", "1"):
    os.environ["PFB200_SR"] = flag
    for case, sch, n in (("tension16", "S1", 12), ("lpanel25", "ST", 6), ("cfg2", "S1", 3)):
        pb = C.setup(C.get_case(case), C.b200_api())
        s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
        s.push_state(pb.state)
        st = [s.step(sch, pb.bcs, pb.pins) for _ in range(n)]
        g = s.pull()
        res[(flag, case)] = ([(x.n_stag, x.cg_iters_u) for x in st], g["u"], g["d"],
                             sum(x.kernel_ms_u for x in st) / max(1, sum(x.cg_iters_u for x in st)) * 1e3)
        s.close()
for case in ("tension16", "lpanel25", "cfg2"):
    a, b = res[("0", case)], res[("1", case)]
    du = np.max(np.abs(a[1] - b[1])) / np.max(np.abs(a[1])); dd = np.max(np.abs(a[2] - b[2]))
    print(case, "HS", a[0], f"{a[3]:.2f} us/it")
    print(case, "SR", b[0], f"{b[3]:.2f} us/it", f"du {du:.2e} dd {dd:.2e}")
