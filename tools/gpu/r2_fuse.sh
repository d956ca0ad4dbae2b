QTNH_SVD_ORDER=xor python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py -x -q > gpurun_out/t_svd_xor.log 2>&1; echo rc=$? >> gpurun_out/t_svd_xor.log
for cfg in "QTNH_SVD_EIG_T=256" "QTNH_SVD_EIG_T=64" "QTNH_SVD_ORDER=xor QTNH_SVD_FUSE=0" "QTNH_SVD_ORDER=xor" "QTNH_SVD_ORDER=xor QTNH_SVD_EIG_T=256"; do
  env $cfg python tools/bench_svd.py 8x2048x1024 1x1024x512 | sed "s/^/[$cfg] /" >> gpurun_out/svd_fuse.txt 2>&1
done
for cfg in "QTNH_SVD_EIG_T=256" "QTNH_SVD_ORDER=xor" "QTNH_SVD_EIG_T=256 QTNH_SVD_ORDER=xor"; do
  env $cfg python tools/run_mps.py > gpurun_out/c4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('[$cfg]', round(d['total_s'],3), d['fidelity'], [round(x,3) for x in d['per_layer_s'][9:]])" >> gpurun_out/svd_fuse.txt
done
QTNH_SVD_ORDER=xor ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_svd --launch-skip 300 -c 30 --csv env QTNH_SVD_GROUPS=1 python tools/bench_svd.py 8x2048x1024 > gpurun_out/ncu_fuse.csv 2>/dev/null
