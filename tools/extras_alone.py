import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2505_06119_b200.qtnh import World
stream = torch.cuda.Stream()
def body(rk):
    rk.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        ex = bench.measure_extras(rk, stream, torch)
    print(json.dumps({k: v for k, v in ex.items() if 'svd' in k}))
World(1, [0]).run(body)
