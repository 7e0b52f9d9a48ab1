# Round 2 closing measurement on the final tree: GPU test suite, smoke, the cfg5 bench line, the
# reference arm, the secondary cfg2 line, the bench launch list, the unrolled-MG launch list and
# the --set full capture of the dominant kernel (roofline traffic).
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${TAG:-v1}
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > $O/gpu_tests.log 2>&1; echo "gpu tests exit $?"; tail -n 3 $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -n 1 $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "bench exit $?"; tail -n 1 $O/bench.log > $O/bench_cfg5.json
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.log 2>&1; echo "ref exit $?"; tail -n 1 $O/bench_ref.log > $O/bench_reference.json
timeout 600 python bench.py --case cfg2 --steps 20 --warmup 5 > $O/bench_cfg2.log 2>&1; echo "cfg2 exit $?"; tail -n 1 $O/bench_cfg2.log > $O/bench_cfg2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mg.csv python scripts/prof_mg_cfg5.py 2 2 > $O/ncu_mg.log 2>&1; echo "ncu mg exit $?"
for k in k_mgs_fine_smooth k_mgs_fine_resid k_mgs_pcg k_mg_fine_smooth k_evo_prepare_march; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$" -c 1 -o $O/$k python scripts/prof_mg_cfg5.py 2 2 > $O/ncu_$k.log 2>&1; echo "ncu $k exit $?"
  ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
  # gpurun_out is capped at 64 MiB: only the dominant kernel's report travels back
  [ $k = k_mgs_fine_smooth ] || rm -f $O/$k.ncu-rep
done
