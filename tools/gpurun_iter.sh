# GPU box: quick iteration -- selected parity tests, target bench (both bwd modes), launch list
O=gpurun_out/iter; mkdir -p $O
rm -f gpurun_out/parity/errors.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "${K:-not nothing}" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cp gpurun_out/parity/errors.jsonl $O/ 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-ylo > $O/bench_noylo.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_target.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
${EXTRA:-true}
tail -3 $O/pytest.log; for f in $O/bench*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f',d['value'],d['ms_per_step'],d['kernels_ms'],d['roofline']['frac'],d['roofline']['step_frac'],d.get('e2e',{}).get('value') if d.get('e2e') else None)"; done
