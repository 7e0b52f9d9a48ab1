cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -30 gpurun_out/mg_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mg.log 2>&1; echo "bench exit $?"; tail -2 gpurun_out/bench_mg.log
