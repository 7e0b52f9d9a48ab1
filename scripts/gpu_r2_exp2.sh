cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e2
timeout 300 python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/e2/prof.log 2>&1; tail -n 1 gpurun_out/e2/prof.log
for pw in 8 4; do
  PFB200_TRACE=1 PFB200_MGS_POW=$pw timeout 300 python scripts/cfg5_run.py 5 S1 > gpurun_out/e2/pow$pw.log 2>&1; echo "pow $pw"; grep '^{"step"' gpurun_out/e2/pow$pw.log | cut -c1-140
  grep "scalar phase-field" gpurun_out/e2/pow$pw.log | tail -n 3
done
timeout 300 python bench.py --case cfg2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e2/cfg2.log 2>&1; tail -n 1 gpurun_out/e2/cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['momentum_solver'], d['pcg_iters'], d['kernel_ms'])"
