cd $GRAFT_REPO_ROOT
for c in cfg2 cfg3; do timeout 300 python scripts/cg_microbench.py $c 4 > gpurun_out/mb_$c.log 2>&1; tail -3 gpurun_out/mb_$c.log | cut -c1-200; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_warm.log 2>&1; echo "bench exit $?"; tail -c 900 gpurun_out/bench_warm.log
