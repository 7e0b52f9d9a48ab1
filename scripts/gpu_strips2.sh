cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_strips.py -q -x > gpurun_out/strips2.log 2>&1; echo "strips exit $?"; tail -25 gpurun_out/strips2.log
