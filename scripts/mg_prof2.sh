cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PFB200_MG_UNROLL=3
ncu --set full --clock-control none --import-source on -k regex:"k_mg_resid|k_mg_restrict" -s 6 -c 2 -o gpurun_out/prof_mgk python scripts/mg_launches.py cfg2 3 > gpurun_out/ncu_mgk.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_mgk.log
