cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e5
PFB200_TRACE=1 timeout 300 python scripts/cfg5_run.py 6 S1 > gpurun_out/e5/cfg5.log 2>&1; grep '^{"step"' gpurun_out/e5/cfg5.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print([r['cg_iters_u'] for r in rows], [r['cg_iters_d'] for r in rows], [round(r['step_ms']) for r in rows], sum(r['step_ms'] for r in rows[2:])/len(rows[2:]))"; grep -c "safe hierarchy" gpurun_out/e5/cfg5.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/e5/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 16 gpurun_out/e5/gpu_all.log
