cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mg.py -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -15 gpurun_out/mg_tests.log
timeout 2400 python -m pytest tests -m gpu -q --durations=6 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -10 gpurun_out/gpu_all.log
timeout 900 python scripts/cfg5_run.py 3 S1 > gpurun_out/cfg5_run2.jsonl 2>&1; echo "cfg5 exit $?"; cut -c1-300 gpurun_out/cfg5_run2.jsonl
