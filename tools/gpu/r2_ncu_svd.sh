for k in k_svd_eigen_t k_svd_update_v2 k_svd_gram_mma_t; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 300 -c 1 -o gpurun_out/ncu_$k env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 > gpurun_out/ncu_$k.log 2>&1
done
