cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for cfg in "1 libpfb200.so" "1 libpfb200_l1.so" "0 libpfb200.so" "1 libpfb200.so" "1 libpfb200_l1.so"; do
set -- $cfg
PFB200_LIB=$PWD/paper_2209_07969_b200/$2 PFB200_ST_EVO=$1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('st=$1 $2', d['value'], d['e2e']['value'], d['ms_per_step'], 'pf us/it', 1e3*d['kernel_ms']['phase_field_pcg']/d['pcg_iters']['phase_field'])"
done
