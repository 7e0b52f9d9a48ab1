cd $GRAFT_REPO_ROOT
for lib in default m3; do
  if [ $lib = default ]; then unset PFB200_LIB; else export PFB200_LIB=$PWD/paper_2209_07969_b200/libpfb200_$lib.so; fi
  for c in cfg2 cfg3 cfg4; do timeout 300 python scripts/cg_microbench.py $c 2 > gpurun_out/mb_${lib}_$c.log 2>&1; tail -1 gpurun_out/mb_${lib}_$c.log | cut -c1-250; done
done
unset PFB200_LIB
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench exit $?"; tail -c 1200 gpurun_out/bench_n1.log
