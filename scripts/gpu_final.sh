# Full verification + measurement pass (run through gpurun from the repo root):
#   smoke, GPU test suite, bench line + reference arm, launch list of the bench command,
#   ncu --set full of the momentum PCG on cfg2 (bench), cfg3 and cfg5 (largest mesh),
#   per-size per-iteration sweep.  Every ncu command runs after the same command exited 0.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-v6}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; grep -E "passed|failed|FAILED|^E  .*Assert" gpurun_out/gpu_all.log | head -30
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref_line.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
for C in cfg2 cfg3; do
  python scripts/cg_microbench.py $C 1 > gpurun_out/plain_$C.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o gpurun_out/prof_cg_${C}_$TAG python scripts/cg_microbench.py $C 1 > gpurun_out/ncu_$C.log 2>&1
  echo "ncu $C exit $?"
done
python scripts/prof_cfg5.py cfg5 20 > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg -c 2 -o gpurun_out/prof_cg_cfg5_$TAG python scripts/prof_cfg5.py cfg5 20 > gpurun_out/ncu_cfg5.log 2>&1
echo "ncu cfg5 exit $?"
timeout 900 python scripts/roofline_sizes.py > gpurun_out/roofline_sizes.jsonl 2> gpurun_out/roofline_sizes.err; echo "sizes exit $?"
