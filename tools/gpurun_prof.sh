# usage (on the GPU box, from the repo root): bash tools/gpurun_prof.sh <tag> [workload]
tag=${1:-rf}; wl=${2:-lorenz}
python bench.py --workload $wl --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_bench.json 2>gpurun_out/${tag}_bench.err; tail -1 gpurun_out/${tag}_bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rf_kernel|resident|fused|pipe_" --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"rf_kernel|resident|fused|pipe_" -s 9 -c 3 -o gpurun_out/${tag}_prof python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out | grep $tag
