cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python scripts/mg_timing.py cfg2 cfg3 2>&1 | tail -2 | cut -c1-330; echo
timeout 600 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -3 gpurun_out/mg_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mg.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_mg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pcg_iters'], d['kernel_ms'], d['e2e']['value'])"
export PFB200_MG_UNROLL=3
python scripts/mg_launches.py cfg2 3 > gpurun_out/plain_mgl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/mg_launches_cfg2_warm.csv python scripts/mg_launches.py cfg2 3 > gpurun_out/ncu_mgl.log 2>&1
echo "ncu exit $?"
