# march form of k_evo_prepare: KATs and end-to-end on reduced cases (forced), full suite, cfg5
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/batch4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -x -k "kernels_match or evo_prepare_march" > $O/tests.log 2>&1; echo "tests exit $?"; tail -n 5 $O/tests.log
for em in 1 0; do
PFB200_EVO_MARCH=$em timeout 900 python scripts/cfg5_run.py 6 S1 > $O/cfg5_$em.log 2>&1; echo "exit $?"
grep '^{"step"' $O/cfg5_$em.log | cut -c1-200 | tail -n 3
done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 $O/gpu_all.log
