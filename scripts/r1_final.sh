# Round-1 closing measurement (v10: final code): GPU test suite, smoke, bench line + reference arm,
# bench launch list.  The k_cg_st ncu capture of v9 (gpu_final3.sh) is of the same kernel.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-v15}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -2 gpurun_out/gpu_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref_line.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
