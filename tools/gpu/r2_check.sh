set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest1.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gputest1.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench1.log
