# A/B timing of the cfg5 fine marches across build variants (exp/lib_*.so via PFB200_LIB), and the
# warm power-step count.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/e1
timeout 300 python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/e1/default.log 2>&1; tail -n 1 gpurun_out/e1/default.log
for v in noprol noprol_skip minb2 minb4; do
  PFB200_LIB=exp/lib_$v.so timeout 300 python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/e1/$v.log 2>&1; echo "$v exit $?"; tail -n 1 gpurun_out/e1/$v.log
done
for pw in 1 2 4; do
  PFB200_MGS_POW_WARM=$pw timeout 300 python scripts/cfg5_run.py 4 S1 > gpurun_out/e1/pow$pw.log 2>&1; echo "pow $pw"; grep '^{"step"' gpurun_out/e1/pow$pw.log | cut -c1-170
done
