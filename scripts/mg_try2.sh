cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for T in 1200 300; do PFB200_MG_TAIL=$T timeout 300 python scripts/mg_timing.py cfg2 cfg3 2>&1 | tail -3 | sed "s/^/tail=$T /"; done
timeout 600 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -5 gpurun_out/mg_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mg.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_mg.log | cut -c1-700
