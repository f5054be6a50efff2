# GPU box: where the fused-pass time goes (stage times with phases switched
# off through HOMFE_FFT_DBG; results are garbage, only the timings count),
# fp64 ceilings, one ncu --set full capture of each fused pass
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
for d in 0 1 2 4 5 8 128 136 16 32 48 64 256; do
  echo "dbg $d" >> gpurun_out/passes.txt
  HOMFE_FFT_DBG=$d MAX_CG=40 timeout 300 python tools/profile_step.py c3 >> gpurun_out/passes.txt 2>&1
done
MAX_CG=3 timeout 900 ncu --set full --import-source on --clock-control none -k "regex:k_plane_fwd|k_plane_inv|k_pencil" -s 6 -c 3 -o gpurun_out/full_passes_r2 python tools/profile_step.py c3 > gpurun_out/ncu_passes.log 2>&1; echo ncu=$?
