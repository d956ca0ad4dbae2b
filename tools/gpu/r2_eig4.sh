python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_configs_full_gpu.py -x -q -k "not c1 and not c3" > gpurun_out/t_eig4.log 2>&1; echo rc=$? >> gpurun_out/t_eig4.log
python tools/run_mps.py > gpurun_out/c4_eig4.json 2>&1
python tools/bench_svd.py 8x2048x1024 > gpurun_out/svd_eig4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_svd_eigen --launch-skip 300 -c 1 -o gpurun_out/ncu_eig4 env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 > /dev/null 2>&1
