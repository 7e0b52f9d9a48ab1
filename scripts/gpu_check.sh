set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "kernels or symmetry" > gpurun_out/pytest_kern.log 2>&1; echo "pytest kern exit $?"
tail -30 gpurun_out/pytest_kern.log
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -k "not kernels and not symmetry" > gpurun_out/pytest_solver.log 2>&1; echo "pytest solver exit $?"
tail -60 gpurun_out/pytest_solver.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench exit $?"
tail -5 gpurun_out/bench1.log
