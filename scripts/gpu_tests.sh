cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
PFB200_TRACE=1 timeout 300 python scripts/sr_evo_debug.py cfg3 2>&1 | grep -v "mg solve\|momentum pass" | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_tr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pcg_iters'], d['kernel_ms'], d['e2e']['value'])"
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -12 gpurun_out/gpu_all.log
