# GPU box: f32c64 pipeline timing, main build vs variants
O=gpurun_out/variants2; mkdir -p $O
timeout 600 python tools/path_sweep.py --T 1000,1461,3000,10000 --paths pipe,x64 > $O/main.jsonl 2>&1
for v in paper_2410_06074_b200/lib/variants/*.so; do
  t=$(basename $v .so)
  timeout 600 python tools/path_sweep.py --T 1000,1461,3000,10000 --paths pipe --lib $v > $O/$t.jsonl 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pipe_p2" -s 6 -c 2 -o $O/prof_p2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
tail -c 400 $O/bench.json; for f in $O/*.jsonl; do echo $f; cat $f; done
