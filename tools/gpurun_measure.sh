# GPU box: full round-2 pass -- parity suite, smoke, bench lines, launch list, ncu --set full
O=gpurun_out/measure6; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv,noheader > $O/gpu.txt
rm -f gpurun_out/parity/errors.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 --durations=15 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
cp gpurun_out/parity/errors.jsonl $O/parity_errors.jsonl 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_default.json 2> $O/bench_default.err
python bench.py --no-ylo --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_target_f32c64_noylo.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
for wl in lorenz sst kdv; do
  python bench.py --workload $wl --steps 20 --e2e-steps 3 --no-cpu-baseline > $O/bench_${wl}_f32c64.json 2>&1
done
for wl in target lorenz sst; do
  python bench.py --workload $wl --dtype f32 --steps 20 --e2e-steps 0 --no-cpu-baseline > $O/bench_${wl}_f32.json 2>&1
done
python bench.py --workload target --dtype f64 --steps 10 --e2e-steps 0 --no-cpu-baseline > $O/bench_target_f64.json 2>&1
for wl in sweep_t1e2 sweep_wide sweep_t1e5 sweep_t1e6 sweep_o3_t1e5; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${wl}_f32c64.json 2>&1
  timeout 900 python bench.py --workload $wl --dtype f64 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_${wl}_f64.json 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_target.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pipe_" -s 18 -c 6 -o $O/prof_target python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
tail -3 $O/pytest.log; cat $O/smoke.log; ls $O
