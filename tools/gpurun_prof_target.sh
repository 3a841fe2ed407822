# GPU box: bench + launch list + ncu --set full of the pipeline kernels, f32c64 target
O=gpurun_out/prof_target; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_" -s 18 -c 6 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la $O; tail -c 600 $O/bench.json
