cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kat2.log 2>&1; tail -3 gpurun_out/kat2.log
timeout 600 python scripts/debug_case.py tension16 ST > gpurun_out/dbg_t16_ST.log 2>&1
grep "step  12" gpurun_out/dbg_t16_ST.log; tail -5 gpurun_out/dbg_t16_ST.log
timeout 900 python -m pytest tests/test_gpu_solver.py -q -k "end_to_end or cfg1" > gpurun_out/solver2.log 2>&1; grep -E "Error|passed|failed" gpurun_out/solver2.log | tail -20
