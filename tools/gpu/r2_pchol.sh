QTNH_SVD_DEBUG=1 python -m pytest tests/test_svd_gpu.py -x -q -k "split" > gpurun_out/t_pchol.log 2> gpurun_out/t_pchol.err; echo rc=$? >> gpurun_out/t_pchol.log
python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_mps_ops_gpu.py tests/test_configs_full_gpu.py -x -q -k "not c1 and not c3" >> gpurun_out/t_pchol.log 2>&1; echo rc=$? >> gpurun_out/t_pchol.log
for cfg in "QTNH_SVD_SPLIT_BASIS=pchol" "QTNH_SVD_SPLIT_BASIS=jacobi"; do
  env $cfg BENCH_SVD_SPECTRUM=two python tools/bench_svd.py 8x2048x1024 | sed "s/^/[$cfg] /" >> gpurun_out/pchol.txt 2>&1
  env $cfg python tools/run_mps.py > gpurun_out/c4.json 2>&1; python -c "
import json;d=json.load(open('gpurun_out/c4.json'));print('[$cfg]', round(d['total_s'],3), d['fidelity'], [round(x,3) for x in d['per_layer_s'][9:]], d['amp_first'][:2])" >> gpurun_out/pchol.txt
done
QTNH_SVD_DEBUG=1 BENCH_SVD_SPECTRUM=two python tools/bench_svd.py 8x2048x1024 2>&1 | grep "basis" | head -20 >> gpurun_out/pchol.txt
