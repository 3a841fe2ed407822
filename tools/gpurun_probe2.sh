# x64 vs pipeline in f32c64 on every workload (GPU box)
O=gpurun_out/probe2; mkdir -p $O
for wl in target lorenz sst kdv; do
  timeout 300 python bench.py --workload $wl --dtype f32c64 --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/x64_$wl.json 2>&1
  SMNN_KERNEL=pipe timeout 300 python bench.py --workload $wl --dtype f32c64 --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/pipe_$wl.json 2>&1
done
timeout 300 python bench.py --workload target --dtype f64 --steps 5 --e2e-steps 0 --no-cpu-baseline > $O/x64_target_f64.json 2>&1
SMNN_KERNEL=pipe timeout 300 python bench.py --workload target --dtype f64 --steps 5 --e2e-steps 0 --no-cpu-baseline > $O/pipe_target_f64.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"x64" -s 6 -c 2 -o $O/prof_x64_lorenz python bench.py --workload lorenz --dtype f32c64 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pipe_" -s 9 -c 6 -o $O/prof_pipe_target python bench.py --workload target --dtype f32c64 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $O
