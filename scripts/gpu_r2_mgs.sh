# Scalar phase-field multigrid: correctness tests, then cfg5 load steps (scalar vs packed).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/mgs
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_dropin_reference.py -q -x -k "phase_field or reference or helpers" > gpurun_out/mgs/tests.log 2>&1; echo "tests exit $?"; tail -n 3 gpurun_out/mgs/tests.log
PFB200_TRACE=1 timeout 600 python scripts/cfg5_run.py 3 S1 > gpurun_out/mgs/cfg5_scalar.log 2>&1; echo "cfg5 scalar exit $?"; grep '^{' gpurun_out/mgs/cfg5_scalar.log
PFB200_MG_EVO=packed timeout 600 python scripts/cfg5_run.py 3 S1 > gpurun_out/mgs/cfg5_packed.log 2>&1; echo "cfg5 packed exit $?"; grep '^{' gpurun_out/mgs/cfg5_packed.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/mgs/gpu_all.log 2>&1; echo "gpu all exit $?"; tail -n 3 gpurun_out/mgs/gpu_all.log
