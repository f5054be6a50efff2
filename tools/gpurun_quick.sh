# GPU box: stage timings of variants/*/ + in-tree build, then a quick parity subset
# usage: bash tools/gpurun_quick.sh "<pytest files>" "<-k expr>"
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/ab_kernels.py > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
timeout 1200 python -m pytest ${1:-tests/test_gpu_fused.py tests/test_gpu_baseline_parity.py} -q -x -k "${2:-fused}" > gpurun_out/qtests.log 2>&1; echo rc=$?
tail -3 gpurun_out/qtests.log
