python tools/c4_theta_study.py --layer 19 --pairs 5 > gpurun_out/r2_theta_l19.json 2> gpurun_out/r2_theta_l19.err; echo "rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/r2_theta_l19.json'))
for s in d['spectra']: print(s)
print({k:v for k,v in d.items() if k!='spectra' and k!='hist' and k!='hist_edges'})"
