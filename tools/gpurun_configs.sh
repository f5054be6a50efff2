# GPU box: bench lines (with clock records) for every BASELINE configuration
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --config c1 --steps 3000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for n in 1024 2048 4096 8192; do
  python bench.py --config c5 --n $n --steps $((8192 * 8192 * 20 / (n * n) + 20)) --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$n.json 2> gpurun_out/bench_c5_$n.err
done
