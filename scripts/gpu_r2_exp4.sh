cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e4
for pw in 8 4; do
  PFB200_MG_POW=$pw timeout 300 python scripts/cfg5_run.py 6 S1 > gpurun_out/e4/pow$pw.log 2>&1; echo "mom pow $pw"; grep '^{"step"' gpurun_out/e4/pow$pw.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print([r['cg_iters_u'] for r in rows], [r['cg_iters_d'] for r in rows], [round(r['step_ms']) for r in rows], sum(r['step_ms'] for r in rows[2:])/len(rows[2:]))"
  PFB200_MG_POW=$pw timeout 300 python bench.py --case cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e4/cfg2_$pw.log 2>&1; tail -n 1 gpurun_out/e4/cfg2_$pw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['value'], d['ms_per_step'], d['momentum_solver']['us_per_iteration'], d['pcg_iters'])"
done
timeout 900 python -m pytest tests/test_gpu_mg.py -q -x > gpurun_out/e4/mg.log 2>&1; echo "mg tests $?"; tail -n 2 gpurun_out/e4/mg.log
