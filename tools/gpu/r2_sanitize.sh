# compute-sanitizer memcheck (one tool per call) over the multi-rank peer-memory
# kernels (push remap, pairwise in-place swaps, fused distributed gates / QFT), the
# pipelined exchange-form swap, and a 2-process CUDA-IPC world.
SEL='distributed_swaps or tensor_to_tensor or asymmetric or scatter_and_gather or dense_gates_on_distributed or distributed_qft or fused_qft_distributed or inplace_distributed_swap'
python -m pytest tests/test_structural_gpu.py tests/test_gate_gpu.py -k "$SEL" -q -x > gpurun_out/r2_san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2_san_plain.log
timeout 2400 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 99 --log-file gpurun_out/r2_memcheck_%p.log \
  python -m pytest tests/test_structural_gpu.py tests/test_gate_gpu.py tests/test_ipc_gpu.py -k "$SEL or 2-None" -q -x -p no:cacheprovider > gpurun_out/r2_san.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2_san.log
grep -h "ERROR SUMMARY" gpurun_out/r2_memcheck_*.log | sort | uniq -c
