python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_mps_ops_gpu.py -m gpu -q -x > gpurun_out/r2_t12.log 2>&1; echo "svd tests rc=$?"; tail -2 gpurun_out/r2_t12.log
python -m pytest tests/test_structural_gpu.py -m gpu -q -x --durations=5 > gpurun_out/r2_t12b.log 2>&1; echo "structural rc=$?"; tail -9 gpurun_out/r2_t12b.log
QTNH_SVD_DEBUG=1 python tools/c4_theta_study.py > gpurun_out/r2_theta_g.json 2> gpurun_out/r2_theta_g.err; echo "study rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/r2_theta_g.json'));print({k:d[k] for k in ('ours_batch1','ours_batch8')})"; grep "polish" gpurun_out/r2_theta_g.err | tail -3
QTNH_SVD_SPLIT_BASIS=jacobi python tools/c4_theta_study.py > gpurun_out/r2_theta_j.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_theta_j.json'));print('jacobi basis', {k:d[k] for k in ('ours_batch1','ours_batch8')})"
python tools/run_mps.py > gpurun_out/r2_run_mps5.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_run_mps5.json'));print(d['total_s'],d['fidelity'],[round(x,3) for x in d['per_layer_s']])"
