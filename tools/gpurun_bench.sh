# usage (on the GPU box, from the repo root): bash tools/gpurun_bench.sh
# full measurement pass (GPU box): bench lines, launch lists, ncu --set full captures
set -x
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > $O/gpu.txt
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
python bench.py --workload target --steps 20 --e2e-steps 2 --no-cpu-baseline > $O/bench_target.json 2>&1
python bench.py --workload target --dtype f64 --steps 5 --e2e-steps 0 --no-cpu-baseline > $O/bench_target_f64.json 2>&1
python bench.py --workload sst --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_sst.json 2>&1
python bench.py --workload kdv --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/bench_kdv.json 2>&1
python bench.py --dtype f64 --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_lorenz_f64.json 2>&1
python bench.py --dtype f32c64 --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_lorenz_f32c64.json 2>&1
SMNN_KERNEL=resident python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_lorenz_checkpoint.json 2>&1
SMNN_KERNEL=stream python bench.py --workload target --steps 5 --e2e-steps 0 --no-cpu-baseline > $O/bench_target_stream.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_lorenz.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_target.csv python bench.py --workload target --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rf_kernel" -s 6 -c 2 -o $O/prof_lorenz python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pipe_" -s 9 -c 6 -o $O/prof_target python bench.py --workload target --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $O
