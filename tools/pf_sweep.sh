# GPU box: L2 prefetch distance sweep of the plane passes (clusters ahead), c3 stage times
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/pf_sweep.txt
for inv in 0 33 48 66; do
  echo "HOMFE_PF_INV=$inv" >> gpurun_out/pf_sweep.txt
  HOMFE_PF_INV=$inv REPS=20 python tools/profile_step.py c3 2>&1 | tail -1 >> gpurun_out/pf_sweep.txt
done
for fwd in 48 64 96; do
  echo "HOMFE_PF_FWD=$fwd" >> gpurun_out/pf_sweep.txt
  HOMFE_PF_FWD=$fwd REPS=20 python tools/profile_step.py c3 2>&1 | tail -1 >> gpurun_out/pf_sweep.txt
done
cat gpurun_out/pf_sweep.txt
