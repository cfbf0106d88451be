# round 2 (final): measurement set — bench lines for every BASELINE config (+ reference arm), launch
# list of the headline bench (ncu captures: ncu_captures.sh)
mkdir -p gpurun_out/measure
python -c "import __graft_entry__ as g; g.build()"
python bench.py --steps 20 --warmup 5 > gpurun_out/measure/bench_cfg3.json 2> gpurun_out/measure/bench_cfg3.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/measure/bench_cfg3_reference.json 2> gpurun_out/measure/bench_cfg3_reference.err
for c in cfg1 cfg2 cfg4; do  # (cfg4: e2e is wall clock over whole fits — 3 of them)
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --e2e-steps 3 > gpurun_out/measure/bench_$c.json 2> gpurun_out/measure/bench_$c.err
  timeout 600 python bench.py --config $c --impl reference --steps 20 --warmup 5 > gpurun_out/measure/bench_${c}_reference.json 2> gpurun_out/measure/bench_${c}_reference.err
done
timeout 1200 python bench.py --config cfg5 --steps 20 --warmup 3 --e2e-steps 1 --max-reps 5 --cpu-seconds 20 > gpurun_out/measure/bench_cfg5.json 2> gpurun_out/measure/bench_cfg5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/measure/launches_cfg3.csv python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu --max-reps 1 > gpurun_out/measure/ncu_launch.log 2>&1
