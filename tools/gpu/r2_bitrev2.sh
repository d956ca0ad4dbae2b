for c in "6,512,1" "3,256,2" "2,256,3" "4,256,2" "3,512,2" "2,128,6" "6,256,1" "4,384,1"; do
  QTNH_BITREV_CFG=$c ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bitrev --csv python tools/run_qft.py --n 30 2>/dev/null | grep gpu__time | tail -1 | sed "s/^/$c /" >> gpurun_out/bitrev_sweep.txt
done
QTNH_BITREV_TMA=0 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bitrev --csv python tools/run_qft.py --n 30 2>/dev/null | grep gpu__time | tail -1 | sed "s/^/old /" >> gpurun_out/bitrev_sweep.txt
