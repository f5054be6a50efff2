set -x

MAX_CG=3 timeout 300 ncu --set full --import-source on --clock-control none -k "regex:k_plane_fwd|k_plane_inv|k_hex_z|k_pencil" -c 20 -o gpurun_out/full_c3d python tools/profile_step.py c3 > gpurun_out/ncu_full.log 2>&1
echo ncu=$?
