# GPU box: smoke, full -m gpu suite (parity log), c3 bench both arms, stage timings,
# launch list of the bench command, one ncu --set full of the four iteration kernels
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_rc=$?
python tools/ab_kernels.py paper_2203_02962_b200/_lib/libhomfe_gpu.so > gpurun_out/ab.jsonl 2> gpurun_out/ab.err
HOMFE_PARITY_LOG=gpurun_out/parity.jsonl timeout 3000 python -m pytest tests -m gpu -q -s --durations=30 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
HOMFE_NO_WHILE_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncul=$?
MAX_CG=3 timeout 600 ncu --set full --import-source on --clock-control none -k "regex:k_plane_fwd|k_plane_inv|k_hex_z|k_pencil" -c 20 -o gpurun_out/full_c3_r2 python tools/profile_step.py c3 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
