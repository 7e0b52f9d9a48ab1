cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for F in 1 0; do PFB200_MG_FUSE=$F timeout 300 python scripts/mg_timing.py cfg2 cfg3 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('fuse=$F', d['case'], d['momentum_mg'])"; done
timeout 600 python -m pytest tests/test_gpu_mg.py -x -q > gpurun_out/mg_tests.log 2>&1; echo "mg tests exit $?"; tail -2 gpurun_out/mg_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f.log 2>&1; tail -1 gpurun_out/bench_f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['momentum_solver'], d['kernel_ms'], d['e2e']['value'])"
