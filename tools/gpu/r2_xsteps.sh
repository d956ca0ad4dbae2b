QTNH_SVD_CROSS_STEPS=1 python -m pytest tests/test_svd_gpu.py -x -q > gpurun_out/t_xsteps.log 2>&1; echo rc=$? >> gpurun_out/t_xsteps.log
for cfg in "QTNH_SVD_CROSS_STEPS=0" "QTNH_SVD_CROSS_STEPS=1"; do
  env $cfg python tools/bench_svd.py 8x2048x1024 8x2048x1024 | sed "s/^/[$cfg] /" >> gpurun_out/svd_xsteps.txt 2>&1
  env $cfg python tools/run_mps.py > gpurun_out/c4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('[$cfg]', round(d['total_s'],3), d['fidelity'], [round(x,3) for x in d['per_layer_s'][9:]])" >> gpurun_out/svd_xsteps.txt
done
