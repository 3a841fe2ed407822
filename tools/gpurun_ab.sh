# GPU box: A/B of the main build against variant builds (interleaved), f32c64 pipeline
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  timeout 600 python tools/path_sweep.py --T 1461,3000,10000 --paths pipe > $O/main_$rep.jsonl 2>&1
  for v in paper_2410_06074_b200/lib/variants/*.so; do
    timeout 600 python tools/path_sweep.py --T 1461,3000,10000 --paths pipe --lib $v > $O/$(basename $v .so)_$rep.jsonl 2>&1
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pipe_p" -s 12 -c 4 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob('gpurun_out/ab/*.jsonl')):
    out=[]
    for l in open(f):
        try: r=json.loads(l)
        except Exception: continue
        p=r['pipe']; out.append('T=%d f%.3f b%.3f'%(r['T'],p['fwd_ms'],p['bwd_ms']))
    print(os.path.basename(f), ' | '.join(out))
PY
