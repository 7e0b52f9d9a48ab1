# L2 prefetch hints rows ahead in the fine marches (PFB_L2PF): cfg5 per-kernel timings of the
# default library (6 rows) against 0 / 3 / 12 rows, after the multigrid tests on the default.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/l2pf
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_mg.py -m gpu -q -x > $O/tests_mg.log 2>&1; echo "mg tests exit $?"; tail -n 2 $O/tests_mg.log
for lib in default exp/lib_pf0.so exp/lib_pf3.so exp/lib_pf12.so; do
  if [ $lib = default ]; then unset PFB200_LIB; else export PFB200_LIB=$PWD/$lib; fi
  timeout 600 python scripts/prof_mg_cfg5.py 2 2 > $O/prof_$(basename $lib).log 2>&1; echo "prof $lib exit $?"
  tail -n 1 $O/prof_$(basename $lib).log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:round(v['ms'],3) for k,v in d['kernels'].items()}, round(d['momentum_mg_ms'],1), round(d['phase_field_mg_ms'],1))"
done
