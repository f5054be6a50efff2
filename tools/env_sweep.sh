# GPU box: c3 stage times of the in-tree library under environment settings, one per line of $1 (";"-separated)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/env_sweep.txt
IFS=';' read -ra SETS <<< "$1"
for e in "${SETS[@]}"; do
  echo "$e" >> gpurun_out/env_sweep.txt
  env $e REPS=20 HOMFE_FFT_OCC=1 python tools/profile_step.py ${CFG:-c3} 2>&1 | grep -E "^c[1-5] [0-9]|plane kernel" >> gpurun_out/env_sweep.txt
done
cat gpurun_out/env_sweep.txt
