cd $GRAFT_REPO_ROOT
for r in 2 4 6 8 12; do for c in cfg2 cfg3; do PFB200_WARM=0 PFB200_MIN_ROWS=$r timeout 300 python scripts/cg_microbench.py $c 1 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('rows>=$r', d['case'], d['us_per_iter_u'], d['us_per_iter_d'])"; done; done
