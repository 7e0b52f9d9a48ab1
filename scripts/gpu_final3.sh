# Round-1 measurement pass (v9: assembled-stencil phase-field PCG k_cg_st is the dominant single
# kernel at cfg2), run through gpurun from the repo root: smoke, bench line + reference arm, launch
# list, ncu --set full of k_cg_st, MG per-kernel launch list, per-size sweep, cfg5 and cfg2 runs.
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-v9}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref_line.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
python scripts/cg_microbench.py cfg2 3 > gpurun_out/plain_evo.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'^k_cg_st$' -s 2 -c 1 -o gpurun_out/prof_evo_cfg2_$TAG python scripts/cg_microbench.py cfg2 3 > gpurun_out/ncu_evo.log 2>&1
echo "ncu evo exit $?"
PFB200_MG_UNROLL=3 python scripts/mg_launches.py cfg2 3 > gpurun_out/plain_mgl.log 2>&1 && \
PFB200_MG_UNROLL=3 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/mg_launches_cfg2_warm.csv python scripts/mg_launches.py cfg2 3 > gpurun_out/ncu_mgl.log 2>&1
echo "ncu mg exit $?"
timeout 1500 python scripts/roofline_sizes.py > gpurun_out/roofline_sizes.jsonl 2> gpurun_out/roofline_sizes.err; echo "sizes exit $?"; tail -3 gpurun_out/roofline_sizes.err
timeout 900 python scripts/cfg5_run.py 3 S1 > gpurun_out/cfg5_run.jsonl 2>&1; echo "cfg5 exit $?"
timeout 600 python scripts/cfg2_full.py cfg2 S1 > gpurun_out/cfg2_full_mg.json 2> gpurun_out/cfg2_full_mg.err; echo "cfg2 full exit $?"
