# GPU box: the parity suite + default bench + smoke (+ extras)
O=gpurun_out/r2tests; mkdir -p $O
rm -f gpurun_out/parity/errors.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 --durations=25 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cp gpurun_out/parity/errors.jsonl $O/ 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for wl in sweep_t1e5 sweep_t1e6 sweep_o3_t1e5; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${wl}_f32c64.json 2>&1
done
tail -3 $O/pytest.log; tail -c 300 $O/bench_default.json
