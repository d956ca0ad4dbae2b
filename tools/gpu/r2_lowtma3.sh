QTNH_QFT_LOW_NB=1 python -m pytest tests/test_gate_gpu.py -x -q -k "blocked_qft or bit_reversal or qft_norm" > gpurun_out/t_lowtma3.log 2>&1; echo rc=$? >> gpurun_out/t_lowtma3.log
for nb in 1 2 3; do QTNH_QFT_LOW_NB=$nb python tools/run_qft.py --n 33 > gpurun_out/q33.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/q33.json').read().strip().splitlines()[-1]);print('nb=$nb', d['qft_blocked_s'], d['norm_after'], d['spot_max_abs_err'])" >> gpurun_out/lowtma3.txt; done
for nb in 1 2 3; do QTNH_QFT_LOW_NB=$nb ncu --metrics gpu__time_duration.sum --clock-control none -k regex:qft_low --csv python tools/run_qft.py --n 33 2>/dev/null | grep -E "qft_low" | awk -F'","' -v v=$nb '{print "nb=" v, $(NF-2), $NF}' >> gpurun_out/lowtma3.txt; done
