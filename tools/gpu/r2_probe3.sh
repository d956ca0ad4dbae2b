python -m pytest tests/test_gate_gpu.py -x -q -k "bit_reversal" > gpurun_out/t_bitrev2.log 2>&1; echo rc=$? >> gpurun_out/t_bitrev2.log
python tools/run_rcs_tn.py --no-statevector > gpurun_out/c3_run.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/run_rcs_tn.py --no-statevector > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qft\|bitrev --csv --log-file gpurun_out/qft33_launches.csv python tools/run_qft.py --n 33 > /dev/null 2>&1
QTNH_SVD_B=32 python tools/bench_svd.py 8x2048x1024 > gpurun_out/svd_b32.json 2>&1
QTNH_SVD_INNER=2 python tools/bench_svd.py 8x2048x1024 > gpurun_out/svd_inner2.json 2>&1
QTNH_SVD_SORT=1 python tools/bench_svd.py 8x2048x1024 > gpurun_out/svd_sort.json 2>&1
