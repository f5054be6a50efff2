# GPU box: full -m gpu suite with the parity log, smoke, fp64 ceilings
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
HOMFE_PARITY_LOG=gpurun_out/parity.jsonl timeout 3000 python -m pytest tests -m gpu -q -s --durations=30 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
