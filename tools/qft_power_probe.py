"""QFT-33 on a zero state and on seeded random amplitudes, with nvidia-smi sampling
(clocks, power, throttle reasons) every 20 ms: is the ~10 % difference a clock effect?"""
import ctypes as C, os, subprocess, sys, threading, time
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2505_06119_b200 import qtnh
from paper_2505_06119_b200.qtnh import IndexTuple, Tensor, World
n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
samples = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown",
                         "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [samples.append((time.time(), l.strip())) for l in proc.stdout], daemon=True).start()
def body(rk):
    st = torch.cuda.Stream(); rk.set_stream(st.cuda_stream)
    t = Tensor.dense(rk, IndexTuple([2] * n, 0), None, None)
    for label in ("zero", "random", "zero", "random"):
        if label == "random":
            qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(st.cuda_stream), 7, 0, 2**n, C.c_void_p(t.device_ptr())))
        else:
            torch.cuda.memset = None
            qtnh.check(qtnh.lib.qtnh_counter_complex_normals_device(C.c_void_p(st.cuda_stream), 7, 0, 16, C.c_void_p(t.device_ptr())))
            import torch as _t
            from paper_2505_06119_b200.mps import _DevView
            _t.as_tensor(_DevView(t.device_ptr(), 2**n), device="cuda").zero_()
        torch.cuda.synchronize(); time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time(); e0.record(st)
        for _ in range(3): qtnh.qft(t)
        e1.record(st); e1.synchronize(); t1 = time.time()
        win = [s for ts, s in samples if t0 <= ts <= t1]
        print(label, "qft ms", e0.elapsed_time(e1) / 3, "samples", len(win))
        for s in win[:: max(1, len(win) // 6)]: print("   ", s)
World(1).run(body)
proc.terminate()
