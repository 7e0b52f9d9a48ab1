"""Per-iteration and setup cost of the multigrid momentum PCG (pf_bench_cg physics 2) on a
seeded synthetic cracked state of a BASELINE mesh; env PFB200_MG_* knobs are read at create.

    python scripts/mg_timing.py cfg2 [cfg3 ...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402


def state(pb, case):
    X = np.asarray(pb.mesh.nodes)
    side = case.mesh[3] if case.mesh[0] == "notched" else 500.0
    l = case.material["length_l"]
    tip = 0.8 * side
    dist = np.where(X[:, 0] < tip, np.abs(X[:, 1] - 0.5 * side),
                    np.hypot(X[:, 0] - tip, X[:, 1] - 0.5 * side))
    d = np.exp(-dist / l)
    u = np.zeros(2 * X.shape[0])
    u[1::2] = 6e-3 * X[:, 1] / side * (1 + 0.3 * np.sin(7 * X[:, 0] / side))
    u[0::2] = -1e-3 * X[:, 0] / side
    return u, d


def main():
  for name in sys.argv[1:] or ["cfg2"]:
      case = C.get_case(name)
      pb = C.setup(case, C.b200_api())
      s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
      u, d = state(pb, case)
      s.push(u=u, d=d, d_prev=np.zeros_like(d))
      s.refresh_gp()
      info = s.mg_info(with_omega=True)
      out = {"case": name, "levels": info["n_levels"], "n_grid": info["n_grid"],
             "omega": [round(float(x), 3) for x in info.get("omega", [])]}
      for phys, ns in (("momentum_mg", (1, 21)), ("momentum", (1, 201))):
          t = {}
          for n in ns:
              s.bench_cg(phys, n)
              best = min(s.bench_cg(phys, n)[0] for _ in range(3))
              t[n] = best
          per = (t[ns[1]] - t[ns[0]]) / (ns[1] - ns[0])
          out[phys] = {"ms_first": round(t[ns[0]], 4), "us_per_iter": round(1e3 * per, 2),
                       "setup_ms": round(t[ns[0]] - per, 4)}
      print(json.dumps(out), flush=True)
      s.close()


if __name__ == "__main__":
    main()
