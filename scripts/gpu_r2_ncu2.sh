cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/n2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n2/launches.csv python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/n2/ncu_launch.log 2>&1; echo "ncu exit $?"
