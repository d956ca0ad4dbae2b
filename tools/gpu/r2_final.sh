python -m pytest tests -m gpu -q -x --durations=40 > gpurun_out/r2_suite.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_suite.log
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?" >> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-extras --skip-configs --no-cpu-baseline > gpurun_out/r2_ncu_bench.log 2>&1
