SMNN_CHUNK=8 ncu --set full --clock-control none --import-source on -k regex:resident -s 2 -c 2 -o gpurun_out/prof_lorenz_res3 python bench.py --workload lorenz --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
for m in 4 6 8 12; do
SMNN_CHUNK=$m python bench.py --workload lorenz --steps 20 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('m=$m lorenz f32', '%.3g' % d['value'], d['kernels_ms'], '%.3f' % d['roofline']['frac'])"
done
for m in 8 16 24; do
SMNN_CHUNK=$m python bench.py --workload target --steps 10 --no-cpu-baseline --e2e-steps 0 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('m=$m target f32', '%.3g' % d['value'], d['kernels_ms'], '%.3f' % d['roofline']['frac'])"
done
