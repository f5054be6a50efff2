set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
HOMFE_PARITY_LOG=gpurun_out/parity.jsonl timeout 3000 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_parity.py -q -s --durations=40 > gpurun_out/parity.log 2>&1; echo parity_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref_rc=$?
