for cfg in "QTNH_SVD_EIG=3" "QTNH_SVD_EIG=1" "QTNH_SVD_EIG=3 QTNH_SVD_EIG_T=128" "QTNH_SVD_EIG=3 QTNH_SVD_GRAM_CTAS=4" "QTNH_SVD_EIG=3 QTNH_SVD_GRAM_CTAS=6" "QTNH_SVD_EIG=1 QTNH_SVD_GRAM_CTAS=4"; do
  for rep in 1 2; do
  env $cfg python tools/bench_svd.py 8x2048x1024 12x2048x1024 | sed "s/^/[$cfg] /" >> gpurun_out/svd_eig3b.txt 2>&1
  done
done
