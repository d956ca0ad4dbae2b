BENCH_SVD_SPECTRUM=two QTNH_SVD_DEBUG=1 python tools/bench_svd.py 8x2048x1024 > gpurun_out/split_two.txt 2> gpurun_out/split_two.err
BENCH_SVD_SPECTRUM=two ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split_launches.csv env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 > /dev/null 2>&1
QTNH_SVD_DEBUG=1 python tools/run_mps.py > gpurun_out/c4_dbg.json 2> gpurun_out/c4_dbg.err
grep "split path" gpurun_out/c4_dbg.err > gpurun_out/c4_split_lines.txt
rm -f gpurun_out/c4_dbg.err
