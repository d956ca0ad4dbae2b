for cfg in "QTNH_QFT_LOW_S=11 QTNH_QFT_LOW_MINB=3" "QTNH_QFT_LOW_S=10 QTNH_QFT_LOW_MINB=4" "QTNH_QFT_LOW_S=10 QTNH_QFT_LOW_MINB=5" "QTNH_QFT_LOW_S=10 QTNH_QFT_LOW_MINB=3" "QTNH_QFT_LOW_S=9 QTNH_QFT_LOW_MINB=5"; do
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qft_low --csv python tools/run_qft.py --n 33 2>/dev/null | grep -E "qft_low" | awk -F'","' -v v="$cfg" '{print v, $(NF-2), $NF}' >> gpurun_out/low4.txt
done
QTNH_QFT_LOW_S=10 QTNH_QFT_LOW_MINB=4 python -m pytest tests/test_gate_gpu.py -x -q -k "blocked_qft or qft_norm" > gpurun_out/t_low4.log 2>&1; echo rc=$? >> gpurun_out/t_low4.log
