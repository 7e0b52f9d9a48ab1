"""Per-solve PCG iteration counts of the bench workload (PFB200_TRACE=1 prints one line per
Newton/PCG solve to stderr): where the iterations of a load step go."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PFB200_TRACE"] = "1"
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
scheme = sys.argv[2] if len(sys.argv) > 2 else "S1"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 6
pb = C.setup(C.get_case(case), C.b200_api())
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
s.push_state(pb.state)
for k in range(n):
    st = s.step(scheme, pb.bcs, pb.pins)
    print(f"step {k + 1}: n_stag {st.n_stag} cg_u {st.cg_iters_u} cg_d {st.cg_iters_d} "
          f"ms {st.step_ms:.1f}", file=sys.stderr, flush=True)
