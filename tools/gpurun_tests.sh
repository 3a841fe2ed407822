# GPU box: the parity suite + default bench + smoke
O=gpurun_out/r2tests; mkdir -p $O
rm -f gpurun_out/parity/errors.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cp gpurun_out/parity/errors.jsonl $O/ 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -3 $O/pytest.log; tail -c 1500 $O/bench_default.json
timeout 900 python tools/path_sweep.py > $O/path_sweep_f32c64.jsonl 2>&1
timeout 600 python tools/path_sweep.py --dtype f64 --T 1000,3000,10000 > $O/path_sweep_f64.jsonl 2>&1
