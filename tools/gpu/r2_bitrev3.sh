python -m pytest tests/test_gate_gpu.py -x -q -k "bit_reversal" > gpurun_out/t_bitrev3.log 2>&1; echo rc=$? >> gpurun_out/t_bitrev3.log
for cfg in "QTNH_BITREV_TMA=0" "QTNH_BITREV_TMA=2 QTNH_BITREV_NB=3 QTNH_BITREV_CTAS=2" "QTNH_BITREV_TMA=2 QTNH_BITREV_NB=4 QTNH_BITREV_CTAS=1" "QTNH_BITREV_TMA=2 QTNH_BITREV_NB=3 QTNH_BITREV_CTAS=1" "QTNH_BITREV_TMA=2 QTNH_BITREV_NB=4 QTNH_BITREV_CTAS=2"; do
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bitrev --csv python tools/run_qft.py --n 33 2>/dev/null | grep -E "bitrev" | awk -F'","' -v v="$cfg" '{print v, $(NF-2), $NF}' >> gpurun_out/bitrev3.txt
done
