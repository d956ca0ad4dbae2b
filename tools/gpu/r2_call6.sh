python -m pytest tests/test_svd_gpu.py tests/test_mps_gpu.py tests/test_mps_ops_gpu.py -m gpu -q -x > gpurun_out/r2_t6.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_t6.log
QTNH_SVD_DEBUG=1 python tools/c4_theta_study.py > gpurun_out/r2_theta_study2.json 2> gpurun_out/r2_theta_study2.err; echo "study rc=$?"; cat gpurun_out/r2_theta_study2.json; grep "split path" gpurun_out/r2_theta_study2.err | tail -3
python tools/run_mps.py > gpurun_out/r2_run_mps2.json 2> gpurun_out/r2_run_mps2.err; echo "mps rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r2_run_mps2.json'));print(d['total_s'],d['fidelity'],[round(x,3) for x in d['per_layer_s']])"
python tools/run_rcs_tn.py --no-statevector > gpurun_out/r2_rcs_tn.json 2>&1; echo "rcs rc=$?"; tail -c 600 gpurun_out/r2_rcs_tn.json
