"""Whole distributed QFT in a process-per-GPU IPC world (N processes; on a 1-GPU
box they share the device). usage: python tools/ipc_qft_time.py n nproc [peer 0|1]
Launches nproc copies of itself; rank 0 prints the max-over-ranks device time."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(n, peer):
    import torch

    from paper_2505_06119_b200 import qtnh
    from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World, check, lib

    check(lib.qtnh_set_option(b"peer_direct", float(peer)))
    world = World.from_env_ipc()
    k = world.size().bit_length() - 1

    def body(rk):
        t = Tensor.dense(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), None)
        st = torch.cuda.Stream()
        rk.set_stream(st.cuda_stream)
        best = None
        for rep in range(3):
            rk.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            qtnh.qft(t)
            e1.record(st)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        t.free()
        rk.barrier()
        return best

    ms = world.run(body)[0]
    print(f"RANKTIME {os.environ['RANK']} {ms:.3f}", flush=True)


def main():
    if os.environ.get("QTNH_IPC_WORKER"):
        worker(int(sys.argv[1]), int(sys.argv[3]) if len(sys.argv) > 3 else 1)
        return
    n, nproc = int(sys.argv[1]), int(sys.argv[2])
    peer = sys.argv[3] if len(sys.argv) > 3 else "1"
    d = tempfile.mkdtemp(prefix="qtnh_ipc_")
    procs = [subprocess.Popen([sys.executable, __file__, str(n), str(nproc), peer],
                              env=dict(os.environ, QTNH_IPC_WORKER="1", RANK=str(r), LOCAL_RANK=str(r),
                                       WORLD_SIZE=str(nproc), QTNH_IPC_DIR=d),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(nproc)]
    times = []
    for p in procs:
        out, _ = p.communicate(timeout=600)
        for line in out.splitlines():
            if line.startswith("RANKTIME"):
                times.append(float(line.split()[2]))
        if p.returncode != 0:
            print(out[-2000:])
    print(f"qft n={n} ipc world of {nproc} processes peer_direct={peer}: {max(times):.2f} ms (max over ranks)")


if __name__ == "__main__":
    main()
