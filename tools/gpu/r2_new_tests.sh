set -x
python -m pytest tests/test_contract_gpu.py -q -x -k "rank28 or ill_scaled" > gpurun_out/r2_t_c1.log 2>&1; echo "c1 rc=$?"; tail -3 gpurun_out/r2_t_c1.log
python -m pytest tests/test_configs_full_gpu.py -q -x --durations=0 > gpurun_out/r2_t_cfg.log 2>&1; echo "cfg rc=$?"; tail -15 gpurun_out/r2_t_cfg.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench2.log 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench2.err
