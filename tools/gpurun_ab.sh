# GPU box: K/pass timings of the current build, parity smoke of the changed
# kernels, one ncu --set full capture of the four iteration kernels
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_kernels.py paper_2203_02962_b200/_lib/libhomfe_gpu.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py -q -x -k "fused or c3_c4 or hex or seams or newton" > gpurun_out/ktests.log 2>&1; echo rc=$?
timeout 300 python -m pytest tests/test_gpu_j2.py -q -x > gpurun_out/j2tests.log 2>&1; echo rc=$?
MAX_CG=3 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_plane_fwd|k_plane_inv|k_hex_z|k_pencil" -s 4 -c 4 -o gpurun_out/full_c3_r2b python tools/profile_step.py c3 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
