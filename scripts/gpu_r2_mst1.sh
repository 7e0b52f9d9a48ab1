# Staged (TMA bulk copy) fine marches: correctness (multigrid tests + solver goldens), then cfg5
# per-kernel timings of the default library against exp/lib_mst0.so (PFB_MST=0: register-
# prefetched marches).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/mst1
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_kernels.py -m gpu -q -x > $O/tests_mg.log 2>&1; echo "mg tests exit $?"; tail -n 3 $O/tests_mg.log
for lib in default exp/lib_mst0.so; do
  if [ $lib = default ]; then unset PFB200_LIB; else export PFB200_LIB=$PWD/$lib; fi
  timeout 600 python scripts/prof_mg_cfg5.py 2 2 > $O/prof_$(basename $lib).log 2>&1; echo "prof $lib exit $?"; tail -n 1 $O/prof_$(basename $lib).log
done
unset PFB200_LIB
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 $O/gpu_all.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1; echo "bench exit $?"; tail -n 1 $O/bench.log | cut -c1-1500
