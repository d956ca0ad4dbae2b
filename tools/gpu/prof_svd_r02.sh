set -x
python tools/run_mps.py > gpurun_out/c4_run.json 2> gpurun_out/c4_run.err
QTNH_SVD_DEBUG=1 python tools/bench_svd.py 8x2048x1024 1x2048x1024 > gpurun_out/svd_bench.json 2> gpurun_out/svd_debug.err
QTNH_SVD_DEBUG=1 QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 >> gpurun_out/svd_bench.json 2>> gpurun_out/svd_debug_g1.err
QTNH_SVD_GROUPS=2 python tools/bench_svd.py 8x2048x1024 >> gpurun_out/svd_bench.json 2>&1
QTNH_SVD_GROUPS=8 python tools/bench_svd.py 8x2048x1024 >> gpurun_out/svd_bench.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -c 1600 --csv --log-file gpurun_out/svd_launches.csv env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 > gpurun_out/ncu_svd.log 2>&1
