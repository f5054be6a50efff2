# GPU box: A/B kernel timing of variants, new feature tests, one ncu capture
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_kernels.py variants/base/libhomfe_gpu.so paper_2203_02962_b200/_lib/libhomfe_gpu.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -k "2d or multi or seams" > gpurun_out/newtests.log 2>&1; echo rc=$?
timeout 300 python tools/j2_mgr_debug.py > gpurun_out/j2dbg.log 2>&1
MAX_CG=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hex_z -s 1 -c 1 -o gpurun_out/hexz_r2a python tools/profile_step.py c3 > gpurun_out/ncu_hexz.log 2>&1; echo ncu=$?
