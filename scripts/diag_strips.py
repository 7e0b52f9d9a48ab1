"""Diagnostic: N host-emulated strips of a case for a few load steps (trace on)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200.dist import HostGroup, StripSession
case, scheme, nranks, steps = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
pb = C.setup(C.get_case(case), C.b200_api())
group = HostGroup(nranks)
out = [None] * nranks
def worker(rank):
  try:
      ss = StripSession(pb.disc.layout, pb.params, pb.config, rank, nranks, group, device=0)
      print(rank, "created", ss.sess.solver_kinds(), ss.strip.jlo, ss.strip.jhi, flush=True)
      s = pb.state
      ss.push_global(s.u, s.d, s.d_prev, s.gp.tr_eps_plus, s.gp.dev_dot_dev, s.gp.psi_plus, s.gp.psi_max)
      for k in range(steps):
          t = time.time()
          st = ss.step(scheme, pb.bcs, pb.pins)
          print(rank, "step", k + 1, st.n_stag, st.n_nr_u, st.n_nr_d, st.cg_iters_u, st.cg_iters_d, round(time.time() - t, 2), flush=True)
      ss.close()
  except Exception:
      import traceback
      traceback.print_exc()
      sys.stdout.flush()
ths = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(nranks)]
for t in ths: t.start()
for t in ths: t.join(timeout=120)
print("alive", [t.is_alive() for t in ths], flush=True)
os._exit(0)
