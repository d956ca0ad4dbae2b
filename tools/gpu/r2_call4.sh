python -m pytest tests/test_nccl_gpu.py tests/test_structural_gpu.py tests/test_ipc_gpu.py tests/test_abi.py -m gpu -q -x > gpurun_out/r2_t4.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_t4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2_bench_n2.log 2> gpurun_out/r2_bench_n2.err; echo "torchrun rc=$?"; tail -5 gpurun_out/r2_bench_n2.err
python tools/run_mps.py > gpurun_out/r2_run_mps.json 2> gpurun_out/r2_run_mps.err; echo "mps rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --skip-extras --skip-configs --no-cpu-baseline"
$CMD > gpurun_out/r2_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv $CMD > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu1 rc=$?"
$CMD > gpurun_out/r2_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_zgemm_even -s 3 -c 1 -o gpurun_out/r2_zgemm_full $CMD > gpurun_out/r2_ncu_full.log 2>&1; echo "ncu2 rc=$?"
