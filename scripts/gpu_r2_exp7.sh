cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e7
for rows in 1 0; do
PFB200_MG_ROWS=$rows PFB200_TRACE=1 timeout 300 python scripts/cfg5_run.py 6 S1 > gpurun_out/e7/cfg5_$rows.log 2>&1; echo "mom rows $rows"; grep '^{"step"' gpurun_out/e7/cfg5_$rows.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print([r['cg_iters_u'] for r in rows], [r['cg_iters_d'] for r in rows], [round(r['step_ms']) for r in rows], sum(r['step_ms'] for r in rows[2:])/len(rows[2:]))"; grep " mg solve:" gpurun_out/e7/cfg5_$rows.log | tail -n 2
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/e7/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 gpurun_out/e7/gpu_all.log
timeout 300 python bench.py --case cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e7/cfg2.log 2>&1; tail -n 1 gpurun_out/e7/cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'], d['momentum_solver']['us_per_iteration'], d['pcg_iters'])"
