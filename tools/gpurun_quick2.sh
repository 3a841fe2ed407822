# GPU box: quick check -- selected tests (K), target bench, launch list
O=gpurun_out/q2; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "${K:-ylo or benched_mode}" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
${EXTRA:-true}
tail -2 $O/pytest.log; python -c "
import json;d=json.load(open('$O/bench.json'));print(d['value'],d['ms_per_step'],d['kernels_ms'],d['roofline']['frac'],d['roofline']['step_frac'])"
python tools/launches.py $O/launches.csv ${NL:-6}
