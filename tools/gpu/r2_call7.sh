python tools/prof_rcs_tn.py > gpurun_out/r2_prof_rcs.json 2>&1; echo "prof rc=$?"
QTNH_ZGEMM_NARROW_GAUSS=0 python tools/run_rcs_tn.py --no-statevector > gpurun_out/r2_rcs_tn_nog.json 2>&1; tail -c 300 gpurun_out/r2_rcs_tn_nog.json
python tools/run_rcs_tn.py --no-statevector > gpurun_out/r2_rcs_tn2.json 2>&1; tail -c 300 gpurun_out/r2_rcs_tn2.json
QTNH_SVD_DEBUG=1 python tools/run_mps.py > gpurun_out/r2_run_mps3.json 2> gpurun_out/r2_run_mps3.err; echo "mps rc=$?"; grep -c "svd sweep" gpurun_out/r2_run_mps3.err; grep "split path" gpurun_out/r2_run_mps3.err | sort | uniq -c | head
