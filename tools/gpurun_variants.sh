# GPU box: f32c64 pipeline timing, main build vs variants (interleaved twice to see box noise)
O=gpurun_out/variants13; mkdir -p $O
for rep in 1 2; do
  timeout 600 python tools/path_sweep.py --T 1000,1461,10000 --paths pipe > $O/main_$rep.jsonl 2>&1
  for v in paper_2410_06074_b200/lib/variants/*.so; do
    timeout 600 python tools/path_sweep.py --T 1000,1461,10000 --paths pipe --lib $v > $O/$(basename $v .so)_$rep.jsonl 2>&1
  done
done
for f in $O/*.jsonl; do echo $f; cat $f | cut -c1-200; done
