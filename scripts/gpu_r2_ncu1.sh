# ncu --set full of the three largest fine-level multigrid marches at cfg5 (unrolled solves).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/n1
for k in k_mgs_fine_smooth k_mgs_fine_resid k_mg_fine_smooth k_mg_pcg; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^${k}\$" -c 1 \
    -o gpurun_out/n1/$k python scripts/prof_mg_cfg5.py 2 2 > gpurun_out/n1/$k.log 2>&1
  echo "$k exit $?"
done
ls -la gpurun_out/n1
