"""cfg5 multigrid kernels for ncu (launch list / --set full) and per-kernel CUDA-event timings:
session A runs W real load steps (state with grown damage, built hierarchies), session B (created
with PFB200_MG_UNROLL=N: the solve graphs hold N unconditional iterations, so ncu sees every kernel)
gets A's state and runs N-iteration momentum and phase-field MG solves; then the fine-level
marches are re-launched on their own (pf_bench_mg_kernel).

    python scripts/prof_mg_cfg5.py [W] [N] [case]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_07969_b200 import configs as C  # noqa: E402
from paper_2209_07969_b200.session import DeviceSession  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
N = int(sys.argv[2]) if len(sys.argv) > 2 else 2
case = C.get_case(sys.argv[3] if len(sys.argv) > 3 else "cfg5")
dp = C.device_problem(case)
segs, radius = C.precrack_segments(case)
lay = dp.layout
a = DeviceSession(lay, dp.params, dp.config, device=0)
a.init_state(segs if len(segs) else None, radius, lay.nx * lay.hx, lay.ny * lay.hy)
for _ in range(W):
    a.step("S1", dp.bcs, dp.pins)
state = a.pull()
a.close()
os.environ["PFB200_MG_UNROLL"] = str(N)
b = DeviceSession(lay, dp.params, dp.config, device=0)
b.push(**state)
out = {"case": case.name, "unroll": N}
out["momentum_mg_ms"] = b.bench_cg("momentum_mg", N)[0]
out["phase_field_mg_ms"] = b.bench_cg("phase_field_mg", N)[0]
kernels = {}
for which in (0, 1, 2, 10, 11, 12):
    ms, nb, desc = b.bench_mg_kernel(which, 10)
    kernels[which] = {"ms": ms, "bytes": nb, "gbs": nb / (ms * 1e-3) / 1e9}
out["kernels"] = kernels
print(json.dumps(out), flush=True)
b.close()
