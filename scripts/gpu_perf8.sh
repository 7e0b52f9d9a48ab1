cd $GRAFT_REPO_ROOT
for lib in default nt128; do
  if [ $lib = default ]; then unset PFB200_LIB; else export PFB200_LIB=$PWD/paper_2209_07969_b200/libpfb200_$lib.so; fi
  for c in cfg1 cfg2 cfg3 cfg4; do PFB200_WARM=0 timeout 300 python scripts/cg_microbench.py $c 2 > gpurun_out/mb_${lib}_$c.log 2>&1; tail -1 gpurun_out/mb_${lib}_$c.log | cut -c1-230; done
done
