cd "${GRAFT_REPO_ROOT:-.}"
for E in "" "PFB200_WARM_DEPTH=5" "PFB200_SR_EVO=1" "PFB200_WARM_DEPTH=2"; do
env $E timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', round(d['value']/1e6,1), d['pcg_iters'], {k: round(v,2) for k,v in d['kernel_ms'].items()})"
done
