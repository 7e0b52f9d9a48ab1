cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -4 gpurun_out/gpu_all.log
for k in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], 'pf us/it', 1e3*d['kernel_ms']['phase_field_pcg']/d['pcg_iters']['phase_field'], d['pcg_iters'], d['roofline']['frac'])"
done
