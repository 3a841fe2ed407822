# GPU box: f32c64 pipeline timing, main build vs variants (target horizon and two shorter ones)
O=gpurun_out/variants; mkdir -p $O
timeout 600 python tools/path_sweep.py --T 1000,3000,10000 --paths pipe > $O/main.jsonl 2>&1
for v in paper_2410_06074_b200/lib/variants/*.so; do
  t=$(basename $v .so)
  timeout 600 python tools/path_sweep.py --T 1000,3000,10000 --paths pipe --lib $v > $O/$t.jsonl 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2>&1
tail -c 400 $O/bench.json; for f in $O/*.jsonl; do echo $f; cat $f; done
