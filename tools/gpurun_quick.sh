# GPU box: parity suite + target bench + path sweep (quick iteration loop)
O=gpurun_out/quick; mkdir -p $O
rm -f gpurun_out/parity/errors.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cp gpurun_out/parity/errors.jsonl $O/ 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2>&1
timeout 600 python tools/path_sweep.py --T 1000,1461,3000,10000,100000 --paths pipe > $O/sweep.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pipe_" -s 18 -c 6 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
tail -3 $O/pytest.log; tail -c 250 $O/bench.json; cat $O/sweep.jsonl | cut -c1-200
