cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_strips.py -q -x > gpurun_out/strips.log 2>&1; echo "strips exit $?"; tail -25 gpurun_out/strips.log
timeout 1800 python -m pytest tests -m gpu -q -k "not strips" --durations=10 > gpurun_out/gpu_all.log 2>&1; echo "gpu all exit $?"; grep -E "passed|failed|^E  .*Assert|FAILED" gpurun_out/gpu_all.log | head -30
