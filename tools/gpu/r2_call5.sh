python -m pytest tests/test_nccl_gpu.py tests/test_gate_gpu.py tests/test_contract_gpu.py -m gpu -q -x > gpurun_out/r2_t5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_t5.log
QTNH_SVD_DEBUG=1 python tools/c4_theta_study.py > gpurun_out/r2_theta_study.json 2> gpurun_out/r2_theta_study.err; echo "study rc=$?"; cat gpurun_out/r2_theta_study.json
grep -c "svd sweep" gpurun_out/r2_theta_study.err
