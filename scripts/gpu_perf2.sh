cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "kernels or symmetry or spd or solver_level or determinism or errors or tension16" > gpurun_out/t_quick.log 2>&1; tail -3 gpurun_out/t_quick.log
for lib in default m1e2; do
  if [ $lib = default ]; then unset PFB200_LIB; else export PFB200_LIB=$PWD/paper_2209_07969_b200/libpfb200_$lib.so; fi
  for c in cfg2 cfg3 cfg4; do timeout 300 python scripts/cg_microbench.py $c 2 2>&1 | tail -1; done
done
