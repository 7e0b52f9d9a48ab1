cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/dg
PFB200_TRACE=1 timeout 200 python scripts/diag_strips.py tension16 S1 3 2 > gpurun_out/dg/t16_3.log 2>&1; echo "exit $?"; grep -v "^\[pfb200\] evolution\|mg solve:" gpurun_out/dg/t16_3.log | tail -n 30
PFB200_TRACE=1 timeout 200 python scripts/diag_strips.py multicrack32 ST 2 2 > gpurun_out/dg/mc32_2.log 2>&1; echo "exit $?"; tail -n 12 gpurun_out/dg/mc32_2.log
