python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_mps_ops_gpu.py tests/test_configs_full_gpu.py -x -q -k "not c1 and not c3" > gpurun_out/t_svd_final.log 2>&1; echo rc=$? >> gpurun_out/t_svd_final.log
for rep in 1 2; do python tools/run_mps.py > gpurun_out/c4_final_$rep.json 2>&1; done
python tools/bench_svd.py 8x2048x1024 > gpurun_out/svd_final.txt 2>&1
python tools/pcie_probe.py > gpurun_out/pcie.txt 2>&1
