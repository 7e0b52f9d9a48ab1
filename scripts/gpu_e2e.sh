cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nproc
timeout 300 python scripts/e2e_breakdown.py cfg2 2>&1 | tail -8
