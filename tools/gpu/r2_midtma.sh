python -m pytest tests/test_gate_gpu.py -x -q -k "qft" > gpurun_out/t_midtma.log 2>&1; echo rc=$? >> gpurun_out/t_midtma.log
for v in 1 0; do QTNH_QFT_MID_TMA=$v python tools/run_qft.py --n 33 > gpurun_out/q33.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/q33.json').read().strip().splitlines()[-1]);print('midtma=$v', d['qft_blocked_s'], d['norm_after'], d['spot_max_abs_err'])" >> gpurun_out/midtma.txt; done
for v in 1 0; do QTNH_QFT_MID_TMA=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qft_mid --csv python tools/run_qft.py --n 33 2>/dev/null | grep -E "qft_mid" | awk -F'","' -v v=$v '{print "midtma=" v, $(NF-2), $NF}' >> gpurun_out/midtma.txt; done
