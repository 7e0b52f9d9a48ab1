cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -k "not strips" > gpurun_out/gpu_all.log 2>&1; echo "gpu exit $?"; grep -E "passed|failed|^E  .*Assert|FAILED" gpurun_out/gpu_all.log | head -20
for c in cfg2 cfg3; do timeout 300 python scripts/cg_microbench.py $c 3 > gpurun_out/mb_$c.log 2>&1; tail -2 gpurun_out/mb_$c.log | cut -c1-260; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_warm.log 2>&1; echo "bench exit $?"; tail -c 1500 gpurun_out/bench_warm.log
