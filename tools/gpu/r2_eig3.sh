python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_configs_full_gpu.py -x -q -k "not c1 and not c3" > gpurun_out/t_eig3.log 2>&1; echo rc=$? >> gpurun_out/t_eig3.log
for cfg in "QTNH_SVD_EIG=3" "QTNH_SVD_EIG=1" "QTNH_SVD_EIG=3 QTNH_SVD_EIG_T=128"; do
  env $cfg python tools/bench_svd.py 8x2048x1024 1x1024x512 | sed "s/^/[$cfg] /" >> gpurun_out/svd_eig3.txt 2>&1
done
for cfg in "QTNH_SVD_EIG=3" "QTNH_SVD_EIG=1" "QTNH_SVD_EIG=3 QTNH_SVD_EIG_T=128"; do
  env $cfg python tools/run_mps.py > gpurun_out/c4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('[$cfg]', round(d['total_s'],3), d['fidelity'], [round(x,3) for x in d['per_layer_s'][9:]])" >> gpurun_out/svd_eig3.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_svd_eigen --launch-skip 300 -c 10 --csv env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 2>/dev/null | grep gpu__time | awk -F'","' '{s+=$NF; n++} END {print "eig3 eigen avg ns", s/n}' >> gpurun_out/svd_eig3.txt
