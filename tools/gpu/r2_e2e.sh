for c in 16 32 64; do QTNH_HOST_CHUNKS=$c python bench.py --skip-configs --skip-extras --no-cpu-baseline > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err; python -c "
import json;d=json.loads(open('gpurun_out/e2e_$c.json').read().strip().splitlines()[-1]);print('chunks $c', d['value'], d['e2e'])" >> gpurun_out/e2e.txt; done
