python -m pytest tests/test_gate_gpu.py -x -q -k "bit_reversal or blocked_qft or qft_norm or qft16" > gpurun_out/t_bitrev.log 2>&1; echo rc=$? >> gpurun_out/t_bitrev.log
python tools/qft_time.py --help > /dev/null 2>&1
for v in 1 0; do QTNH_BITREV_TMA=$v python tools/run_qft.py --n 33 > gpurun_out/qft33_tma$v.json 2>&1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bitrev --csv --log-file gpurun_out/bitrev_ncu.csv python tools/run_qft.py --n 30 > /dev/null 2>&1
QTNH_BITREV_TMA=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bitrev --csv --log-file gpurun_out/bitrev_ncu_old.csv python tools/run_qft.py --n 30 > /dev/null 2>&1
