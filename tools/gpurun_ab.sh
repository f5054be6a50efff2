# GPU box: A/B stage timings of the library variants (variants/*/ + in-tree),
# then the K / PCG parity tests on the in-tree build.
# usage: bash tools/gpurun_ab.sh [pytest -k expression]
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_kernels.py > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
K="${1:-fused or c3_c4 or hex or seams or newton or operator or determin or slab}"
timeout 1500 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dist.py tests/test_gpu_j2.py -q -x -k "$K" > gpurun_out/ktests.log 2>&1; echo rc=$?
tail -3 gpurun_out/ktests.log
