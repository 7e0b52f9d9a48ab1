# First cfg5 bench line + multigrid kernel profile (launch list of an unrolled MG solve pair).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/b1
free -g > gpurun_out/b1/free.txt; nproc >> gpurun_out/b1/free.txt
timeout 600 python -m pytest tests/test_gpu_dropin_reference.py -q -x > gpurun_out/b1/dropin.log 2>&1; echo "dropin exit $?"; tail -n 2 gpurun_out/b1/dropin.log
timeout 900 python bench.py --steps 4 --warmup 3 > gpurun_out/b1/bench.log 2>&1; echo "bench exit $?"; tail -n 1 gpurun_out/b1/bench.log | head -c 3000; echo
timeout 600 python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/b1/prof.log 2>&1; echo "prof exit $?"; tail -n 1 gpurun_out/b1/prof.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/b1/launches.csv python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/b1/ncu_launch.log 2>&1; echo "ncu exit $?"
