#!/bin/bash
# cProfile around the whole GPU suite: where the host wall time goes.
out=gpurun_out/prof_suite.log; : > $out
python -m cProfile -o /tmp/suite.prof -m pytest tests -q -m gpu -x --durations=15 >> $out 2>&1
python - >> $out 2>&1 <<'P'
import pstats
s = pstats.Stats('/tmp/suite.prof')
s.sort_stats('tottime').print_stats(40)
s.sort_stats('tottime').print_callers('acquire', 12)
P
