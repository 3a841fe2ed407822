nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -1 gpurun_out/bench_reference.json
python bench.py --workload target --steps 20 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_target.json 2>&1; tail -1 gpurun_out/bench_target.json
python bench.py --workload target --dtype f64 --steps 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_target_f64.json 2>&1; tail -1 gpurun_out/bench_target_f64.json
python bench.py --workload kdv --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_kdv.json 2>&1; tail -1 gpurun_out/bench_kdv.json
python bench.py --workload sst --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_sst.json 2>&1; tail -1 gpurun_out/bench_sst.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lorenz.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"resident|fused" --csv --log-file gpurun_out/launches_lorenz_dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"resident|fused" -s 6 -c 2 -o gpurun_out/prof_r1_lorenz python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"resident|fused" -s 6 -c 2 -o gpurun_out/prof_r1_target python bench.py --workload target --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out
