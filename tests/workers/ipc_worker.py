"""One rank of a process-per-GPU IPC world (launched by tests/test_ipc_gpu.py):
distributed structural ops, fused peer kernels and a contraction, each checked
against the oracle, with peer kernels on and off (pull-copy exchange)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2505_06119_b200 import circuits, qtnh  # noqa: E402
from paper_2505_06119_b200.qtnh import DistParams, IndexTuple, Tensor, World  # noqa: E402


def bits(x):
    return np.ascontiguousarray(x, dtype=np.complex128).view(np.uint64)


def main():
    P = oracle.port()
    world = World.from_env_ipc()
    size = world.size()
    k = size.bit_length() - 1
    n = 12
    g = circuits.counter_state(3, 2**n)
    g[::5] = complex(-0.0, -0.0)
    st = g / np.linalg.norm(g)

    def body(rk):
        for mode in (1, 0):
            qtnh.check(qtnh.lib.qtnh_set_option(b"peer_direct", float(mode)))
            # permute (push remap / pack-exchange-unpack)
            perm = list(reversed(range(n)))
            t = Tensor.from_global(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), g)
            u = qtnh.ops.permute(t, perm, k)
            got = u.to_global_vector()
            inside = t.in_span()  # with a non-power-of-two world some ranks hold nothing
            if inside:
                assert np.array_equal(bits(got), bits(P.permute([2] * n, g, perm))), ("permute", mode)
            # in-place distributed <-> local swap
            qtnh.swap_indices(t, 0, n - 1)
            sp = list(range(n))
            sp[0], sp[n - 1] = sp[n - 1], sp[0]
            v = t.to_global_vector()
            if inside:
                assert np.array_equal(bits(v), bits(P.permute([2] * n, g, sp))), ("swap", mode)
            # dense gate on a distributed qubit (fused peer gate)
            s = Tensor.from_global(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), st)
            qtnh.apply_gate(s, [0, 5], circuits.FSIM)
            want = P.gate([2] * n, st, [0, 5], circuits.FSIM.reshape(-1))
            v = s.to_global_vector()
            if inside:
                assert np.linalg.norm(v - want) < 1e-12, ("gate", mode)
            # whole QFT (fused distributed layers + distributed bit reversal)
            q = Tensor.from_global(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), st)
            qtnh.qft(q, swaps=True)
            v = q.to_global_vector()
            if inside:
                assert np.linalg.norm(v - P.qft(n, st)) < 1e-12, ("qft", mode)
            # contraction with A sharded on open indices and a contracted one
            a = circuits.rng_normals(5, 2**n)
            b = circuits.rng_normals(6, 2**5)
            ap, bp = [1, 4, 9], [2, 0, 4]
            ta = Tensor.from_global(rk, IndexTuple([2] * n, k), DistParams(1, 1, 0), a)
            tb = Tensor.from_global(rk, IndexTuple([2] * 5, 0), DistParams(size, 1, 0), b)
            c = qtnh.contract(ta, tb, ap, bp)
            want = P.contract([2] * n, a, [2] * 5, b, ap, bp)
            got = c.to_global_vector()
            if c.in_span():  # the result spans the ranks of a's open distributed indices
                assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12, ("contract", mode)
            for x in (t, u, s, q, ta, tb, c):
                x.free()
            rk.barrier()
        return True

    world.run(body)
    print("ipc rank ok", flush=True)


if __name__ == "__main__":
    main()
