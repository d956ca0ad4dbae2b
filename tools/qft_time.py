import sys, os, time
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import torch, numpy as np
from paper_2505_06119_b200 import qtnh, circuits
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World
n = int(sys.argv[1])
def body(rk):
    st = torch.cuda.Stream(); rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2]*n, 0), None, None)
    qtnh.qft(t); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); qtnh.qft(t); e1.record(st); e1.synchronize()
    print('n', n, 'qft ms', e0.elapsed_time(e1), 'G', os.environ.get('QTNH_QFT_G'))
World(1).run(body)
