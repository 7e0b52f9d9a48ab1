"""One multigrid momentum solve of fixed length on cfg2's synthetic cracked state (for the ncu
launch list: per-kernel durations of the setup and solve graphs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mg_timing import state  # noqa: E402
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
case = C.get_case(name)
pb = C.setup(case, C.b200_api())
s = DeviceSession(pb.disc.layout, pb.params, pb.config, device=0)
u, d = state(pb, case)
s.push(u=u, d=d, d_prev=d * 0)
s.refresh_gp()
print(s.bench_cg("momentum_mg", n))
