cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e6
for rows in 1 0; do
PFB200_MGS_ROWS=$rows PFB200_TRACE=1 timeout 300 python scripts/cfg5_run.py 6 S1 > gpurun_out/e6/cfg5_$rows.log 2>&1; echo "rows $rows"; grep '^{"step"' gpurun_out/e6/cfg5_$rows.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print([r['cg_iters_u'] for r in rows], [r['cg_iters_d'] for r in rows], [round(r['step_ms']) for r in rows], sum(r['step_ms'] for r in rows[2:])/len(rows[2:]))"; grep "scalar phase-field" gpurun_out/e6/cfg5_$rows.log | tail -n 2
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e6/launches.csv python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/e6/ncu_launch.log 2>&1; echo "ncu exit $?"
timeout 600 python -m pytest tests/test_gpu_mg.py -q -x -k "phase_field" > gpurun_out/e6/t.log 2>&1; echo "tests $?"; tail -n 1 gpurun_out/e6/t.log
