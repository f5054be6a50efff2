# ncu --set full of the cuFFT-path kernels: c4 (512^3 elasticity) and c5 (8192^2)
set -x
MAX_CG=2 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_hex_z|k_spectral|k_update" -c 12 -o gpurun_out/full_c4 python tools/profile_step.py c4 > gpurun_out/ncu_c4.log 2>&1
echo ncu_c4=$?
MAX_CG=2 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_elem2d|k_spectral|k_update" -c 12 -o gpurun_out/full_c5 python tools/profile_step.py c5 > gpurun_out/ncu_c5.log 2>&1
echo ncu_c5=$?
