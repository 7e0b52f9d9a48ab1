# Round-2 parity tables on the device: cfg1 crack-step counts per solver variant (plain
# Hestenes-Stiefel Jacobi PCG from x0 = 0 and each acceleration on its own), cfg2 65-step
# tables for all four schemes (restart state after step 54 for the reference crack step),
# a short cfg5 trace.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/tables
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/gpu.txt
PLAIN="PFB200_MG=0 PFB200_WARM=0 PFB200_SR=0 PFB200_SR_EVO=0 PFB200_ST_EVO=0"
run() { # tag env...
  tag=$1; shift
  for sch in ST S1; do
    env "$@" timeout 600 python scripts/gpu_tables.py cfg1 $sch --out gpurun_out/tables/cfg1_${sch}_${tag}.npz >> gpurun_out/tables/cfg1_variants.log 2>&1
  done
}
run default PFB200_DUMMY=1
run plain $PLAIN
run mg      PFB200_MG=1 PFB200_WARM=0 PFB200_SR=0 PFB200_SR_EVO=0 PFB200_ST_EVO=0
run warm    PFB200_MG=0 PFB200_WARM=1 PFB200_SR=0 PFB200_SR_EVO=0 PFB200_ST_EVO=0
run sr      PFB200_MG=0 PFB200_WARM=0 PFB200_SR=1 PFB200_SR_EVO=0 PFB200_ST_EVO=0
run srevo   PFB200_MG=0 PFB200_WARM=0 PFB200_SR=0 PFB200_SR_EVO=1 PFB200_ST_EVO=0
run stevo   PFB200_MG=0 PFB200_WARM=0 PFB200_SR=0 PFB200_SR_EVO=1 PFB200_ST_EVO=1
echo "cfg1 variants done"
for sch in S1 ST S2 S3; do
  ss=""; [ $sch = S1 ] && ss="--state-snap 54"
  timeout 900 python scripts/gpu_tables.py cfg2 $sch --snap 25,54,55 $ss --out gpurun_out/tables/cfg2_${sch}.npz >> gpurun_out/tables/cfg2.log 2>&1
done
echo "cfg2 done"
PFB200_TRACE=1 timeout 600 python scripts/cfg5_run.py 3 S1 > gpurun_out/tables/cfg5_trace.log 2>&1
echo "cfg5 exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gpu_all.log 2>&1; echo "gpu tests exit $?"; tail -n 3 gpurun_out/gpu_all.log
