# GPU box: c3 stage times (tools/profile_step.py, 20 repetitions) of the in-tree library and of every
# variants/*/libhomfe_gpu.so; optional pytest selection afterwards ($1 = files, $2 = -k expression)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/var_sweep.txt
for lib in paper_2203_02962_b200/_lib/libhomfe_gpu.so variants/*/libhomfe_gpu.so; do
  [ -f "$lib" ] || continue
  echo "$lib" >> gpurun_out/var_sweep.txt
  HOMFE_LIB=$PWD/$lib REPS=20 python tools/profile_step.py ${CFG:-c3} 2>&1 | tail -1 >> gpurun_out/var_sweep.txt
done
cat gpurun_out/var_sweep.txt
if [ -n "$1" ]; then
  timeout 1500 python -m pytest $1 -q -x -k "${2:-fused or hex or operator}" > gpurun_out/qtests.log 2>&1; echo rc=$?
  tail -3 gpurun_out/qtests.log
fi
