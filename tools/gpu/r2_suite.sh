python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2_gputest_suite.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2_gputest_suite.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench3.log 2> gpurun_out/r2_bench3.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_bench3.err
