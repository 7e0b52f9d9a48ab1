# full verification + measurement pass (run via gpurun)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; grep -E "passed|failed|FAILED|^E  .*Assert" gpurun_out/gpu_all.log | head -30
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"; tail -c 2500 gpurun_out/bench_full.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -c 600 gpurun_out/bench_ref.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
PFB200_TRACE=1 python scripts/cg_microbench.py cfg2 1 > gpurun_out/plain_cfg2.log 2>&1 && \
PFB200_TRACE=1 ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o gpurun_out/prof_cg_cfg2_v5 python scripts/cg_microbench.py cfg2 1 > gpurun_out/ncu_cfg2.log 2>&1
echo "ncu cfg2 exit $?"
PFB200_TRACE=1 python scripts/cg_microbench.py cfg3 1 > gpurun_out/plain_cfg3.log 2>&1 && \
PFB200_TRACE=1 ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o gpurun_out/prof_cg_cfg3_v5 python scripts/cg_microbench.py cfg3 1 > gpurun_out/ncu_cfg3.log 2>&1
echo "ncu cfg3 exit $?"
