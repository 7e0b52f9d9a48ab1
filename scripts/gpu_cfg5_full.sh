# BASELINE configs[4], all 50 load steps, S1 and the standard scheme (per-step JSON lines)
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/cfg5full
mkdir -p $O
for sc in S1 ST; do
  timeout 1500 python scripts/cfg5_run.py 50 $sc > $O/cfg5_$sc.jsonl 2> $O/cfg5_$sc.err; echo "$sc exit $?"
  grep -c '^{"step"' $O/cfg5_$sc.jsonl
  python - $O/cfg5_$sc.jsonl <<'P'
import json,sys
rows=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{"step"')]
print('n_stag', [r['n_stag'] for r in rows]); print('sum n_stag', sum(r['n_stag'] for r in rows), 'step ms (mean of 6..)', sum(r['step_ms'] for r in rows[5:])/max(1,len(rows[5:])))
print('F_right_x last', rows[-1]['F_right_x'], 'pcg u/d', sum(r['cg_iters_u'] for r in rows), sum(r['cg_iters_d'] for r in rows))
P
done
