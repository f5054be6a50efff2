cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_baseline_parity.py tests/test_gpu_dist.py -q -x -k "two-triangles or bilinear or c5 or c1 or 2d or two_d or rows" > gpurun_out/qtests.log 2>&1; echo rc=$?; tail -2 gpurun_out/qtests.log
python bench.py --config c1 --steps 3000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for n in 1024 2048 4096 8192; do
  python bench.py --config c5 --n $n --steps $((8192 * 8192 * 20 / (n * n) + 20)) --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$n.json 2> gpurun_out/bench_c5_$n.err
done
