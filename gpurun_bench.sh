set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/bench_lorenz_f32.json 2> gpurun_out/bench_lorenz_f32.err; tail -c 3000 gpurun_out/bench_lorenz_f32.json
python bench.py --dtype f32c64 --no-cpu-baseline > gpurun_out/bench_lorenz_f32c64.json 2>&1; tail -c 1500 gpurun_out/bench_lorenz_f32c64.json
python bench.py --dtype f64 --no-cpu-baseline > gpurun_out/bench_lorenz_f64.json 2>&1; tail -c 1500 gpurun_out/bench_lorenz_f64.json
python bench.py --workload target --steps 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_target_f32.json 2>&1; tail -c 1500 gpurun_out/bench_target_f32.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_lorenz.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 2 -o gpurun_out/prof_lorenz_f32 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1; tail -5 gpurun_out/ncu_full.log
