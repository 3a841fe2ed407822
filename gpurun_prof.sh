python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SMNN_KERNEL=stream python -m pytest tests -m gpu -q -x -k "fused or full" 2>&1 | tail -2
for wl in lorenz sst target; do
for m in 8 16; do
SMNN_CHUNK=$m python bench.py --workload $wl --steps 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b.json 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('m=$m $wl', '%.3g' % d['value'], d['kernels_ms'], '%.3f' % d['roofline']['frac'])" 2>&1 | tail -1
done; done
