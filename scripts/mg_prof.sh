cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PFB200_MG_UNROLL=3
python scripts/mg_launches.py cfg2 3 > gpurun_out/plain_mgl.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/mg_launches_cfg2_warm.csv python scripts/mg_launches.py cfg2 3 > gpurun_out/ncu_mgl.log 2>&1
echo "ncu exit $?"
