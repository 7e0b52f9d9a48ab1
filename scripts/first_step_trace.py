"""One load step of a case on the device (default cfg3, scheme ST) -- with PFB200_TRACE=1 it prints every inner solve (e.g. the single-reduction phase-field stall and its two-barrier redo on cfg3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C
from paper_2209_07969_b200.session import DeviceSession
pb = C.setup(C.get_case(sys.argv[1] if len(sys.argv) > 1 else "cfg3"), C.b200_api())
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
s.push_state(pb.state)
st = s.step("ST", pb.bcs, pb.pins)
print("n_stag", st.n_stag, "cg_d", st.cg_iters_d, "cg_u", st.cg_iters_u)
