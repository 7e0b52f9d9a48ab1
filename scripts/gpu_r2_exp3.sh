cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e3
for pw in 3 4 6; do
  PFB200_MGS_POW=$pw timeout 300 python scripts/cfg5_run.py 6 S1 > gpurun_out/e3/pow$pw.log 2>&1; echo "pow $pw"; grep '^{"step"' gpurun_out/e3/pow$pw.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
print([r['cg_iters_d'] for r in rows], [r['n_nr_d'] for r in rows], [round(r['step_ms']) for r in rows], sum(r['step_ms'] for r in rows[2:])/len(rows[2:]))"
done
for pw in 3 4; do
  PFB200_MGS_POW=$pw PFB200_MG_EVO=1 timeout 600 python -m pytest tests/test_gpu_mg.py -q -x -k "phase_field and scalar" > gpurun_out/e3/t$pw.log 2>&1; echo "tests pow $pw exit $?"; tail -n 2 gpurun_out/e3/t$pw.log
done
