#!/bin/bash
# Profile where the wall time of a (small) GPU test goes: cProfile around pytest.
out=gpurun_out/prof_test.log; : > $out
for sel in "tests/test_svd_gpu.py -k 8-6-0" "tests/test_gate_gpu.py -k blocked_qft_and_7-3-8"; do
  sel2=${sel//_and_/ and }
  echo "=== $sel2" >> $out
  python -m cProfile -o /tmp/p.prof -m pytest $( echo "${sel2%% -k*}" ) -k "${sel2##*-k }" -q -m gpu --durations=5 >> $out 2>&1
  python - >> $out 2>&1 <<'P'
import pstats
s = pstats.Stats('/tmp/p.prof'); s.sort_stats('cumulative').print_stats(45)
s.sort_stats('tottime').print_stats(15)
P
done
