cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "kernels or symmetry or spd or solver_level or determinism or errors" > gpurun_out/t_quick.log 2>&1; tail -2 gpurun_out/t_quick.log
for mode in split persistent; do
  export PFB200_CG=$mode
  for c in cfg1 cfg2 cfg3 cfg4; do timeout 300 python scripts/cg_microbench.py $c 2 2>&1 | tail -1 | sed "s/^/$mode /"; done
done
export PFB200_CG=split
for ch in 8 64; do export PFB200_CG_CHUNK=$ch; timeout 300 python scripts/cg_microbench.py cfg2 2 2>&1 | tail -1 | sed "s/^/chunk$ch /"; done
