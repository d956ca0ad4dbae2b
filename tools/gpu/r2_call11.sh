python -m pytest tests/test_structural_gpu.py -k canary -q -x > gpurun_out/r2_t11a.log 2>&1; python -m pytest tests/test_structural_gpu.py -k "write_only" -q -x >> gpurun_out/r2_t11a.log 2>&1; echo "canary rc=$?"; tail -3 gpurun_out/r2_t11a.log
python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/r2_gputest_suite2.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r2_gputest_suite2.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench4.log 2> gpurun_out/r2_bench4.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_bench4.err
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
