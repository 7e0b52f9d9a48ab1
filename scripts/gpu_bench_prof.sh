cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"
tail -c 3000 gpurun_out/bench_full.log
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
tail -c 1500 gpurun_out/bench_ref.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
python scripts/cg_microbench.py cfg2 1 > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o gpurun_out/prof_cg_cfg2_v3 python scripts/cg_microbench.py cfg2 1 > gpurun_out/ncu_cfg2.log 2>&1
echo "ncu cfg2 exit $?"
python scripts/cg_microbench.py cfg3 1 > gpurun_out/plain_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o gpurun_out/prof_cg_cfg3_v3 python scripts/cg_microbench.py cfg3 1 > gpurun_out/ncu_cfg3.log 2>&1
echo "ncu cfg3 exit $?"
