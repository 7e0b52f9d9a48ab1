cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "kernels or symmetry or spd or solver_level or determinism or errors" > gpurun_out/t_quick.log 2>&1; tail -1 gpurun_out/t_quick.log
for c in cfg1 cfg2 cfg3 cfg4; do timeout 300 python scripts/cg_microbench.py $c 2 > gpurun_out/mb_$c.log 2>&1; tail -1 gpurun_out/mb_$c.log | cut -c1-300; done
