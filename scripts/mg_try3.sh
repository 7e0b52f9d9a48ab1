cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -3 gpurun_out/mg_tests.log
for W in 1 0; do
PFB200_MG_WARM=$W PFB200_TRACE=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w$W.log 2>&1; echo "bench warm=$W exit $?"; grep "mg solve" gpurun_out/bench_w$W.log | tail -4; tail -1 gpurun_out/bench_w$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pcg_iters'], d['kernel_ms'], d['e2e']['value'])"
done
