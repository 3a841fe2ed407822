# usage (GPU box, repo root): bash tools/gpurun_probe.sh  -- quick state check of the x64 path
O=gpurun_out/probe; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp_rates tools/fp_rates.cu && /tmp/fp_rates > $O/fp_rates.txt 2>&1
timeout 600 python tools/x64_check.py > $O/x64_check.txt 2>&1
for d in f32c64 f32 f64; do
  timeout 300 python bench.py --workload target --dtype $d --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/bench_target_$d.json 2>&1
done
timeout 300 python bench.py --workload lorenz --dtype f32c64 --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_lorenz_f32c64.json 2>&1
timeout 300 python bench.py --workload kdv --dtype f32c64 --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/bench_kdv_f32c64.json 2>&1
timeout 300 python bench.py --workload sst --dtype f32c64 --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/bench_sst_f32c64.json 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_target_f32c64.csv python bench.py --workload target --dtype f32c64 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"x64" -s 6 -c 2 -o $O/prof_x64_target python bench.py --workload target --dtype f32c64 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $O
