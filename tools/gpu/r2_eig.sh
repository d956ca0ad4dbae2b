python -m pytest tests/test_svd_gpu.py -x -q > gpurun_out/t_svd.log 2>&1; echo rc=$? >> gpurun_out/t_svd.log
for t in 64 128 256; do QTNH_SVD_EIG_T=$t python tools/bench_svd.py 8x2048x1024 1x2048x1024 | sed "s/^/T$t /" >> gpurun_out/svd_eig.txt 2>&1; done
for t in 64 256; do QTNH_SVD_EIG_T=$t ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_svd_eigen --launch-skip 300 -c 20 --csv env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 2>/dev/null | grep gpu__time | awk -F'","' -v t=$t '{s+=$NF; n++} END {print "T" t " eigen avg ns", s/n}' >> gpurun_out/svd_eig.txt; done
python tools/run_mps.py > gpurun_out/c4_eig64.json 2>&1
