"""Tensor storage variants on the device (tensor.hpp:28-164; ops.hpp:54-161): compact
storage in HBM, variant-keeping ops, and gates given as variant tensors. Parity
with the reference itself is tests/test_abi.py's tensor drop-in (every record of
tests/cpp/test_tensor_dropin.cpp against the golden the reference wrote)."""
import numpy as np
import pytest

import oracle
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import (DENSE, DIAGONAL, IDENTITY, SWAP, SYMMETRIC, DistParams, IndexTuple,
                                        InvalidArgument, Tensor, World, apply_gate, apply_gate_tensor, contract, ops)

pytestmark = pytest.mark.gpu


def test_compact_storage_and_variant_tags():
    """A diagonal tensor keeps only its slice of the diagonal in HBM, identity and swap
    nothing; the dense value appears only through to_dense (tensor.hpp:45-52)."""
    n_in = 1 << 10
    diag = circuits.rng_normals(5, 2 * n_in)

    def body(rk):
        dg = Tensor.diagonal(rk, IndexTuple([2, 2, n_in, n_in], 2), DistParams(1, 1, 0), diag)
        idt = Tensor.identity(rk, IndexTuple([2, 2, n_in, n_in], 2), DistParams(1, 1, 0), [0, 2], [1, 3])
        sw = Tensor.swap_tensor(rk, IndexTuple([4, 4, 4, 4], 0), DistParams(4, 1, 0), [0, 1], [2, 3])
        sy = Tensor.symmetric_from_global(rk, IndexTuple([2, 2, 3, 3], 2), DistParams(1, 1, 0), np.arange(36.0))
        on_diag = rk.rank() in (0, 3)
        assert dg.variant() == DIAGONAL and dg.local_data().size == (n_in if on_diag else 0)
        assert dg.local_size() == n_in * n_in  # the metadata still describes the full block
        assert idt.variant() == IDENTITY and idt.local_data().size == 0 and idt.device_ptr() == 0
        assert sw.variant() == SWAP and sw.equality_pairs() == ([0, 1], [2, 3])
        assert sy.variant() == SYMMETRIC and sy.to_dense().variant() == DENSE
        if on_diag:
            b = 0 if rk.rank() == 0 else 1
            assert np.array_equal(dg.local_data(), diag[b * n_in:(b + 1) * n_in])
        d = dg.to_dense()
        assert d.variant() == DENSE and d.local_data().size == n_in * n_in
        blk = d.local_data().reshape(n_in, n_in)
        want = np.diag(diag[(0 if rk.rank() == 0 else 1) * n_in:][:n_in]) if on_diag else np.zeros((n_in, n_in))
        assert np.array_equal(blk, want)
        # element lookup without materialising
        assert dg.local_element([0, 0, 5, 6]) == 0
        if rk.rank() == 3:
            assert dg.local_element([1, 1, 7, 7]) == diag[n_in + 7]
        assert idt.local_element([1, 1, 9, 9]) == 1 and idt.local_element([1, 0, 9, 9]) == 0
        return True

    assert all(World(4).run(body))


@pytest.mark.parametrize("peer", [1, 0])
def test_variant_keeping_ops_against_dense(peer):
    """rebcast / conj / scale keep the variant (ops.hpp:54-161) and agree with the same
    op on the dense value; everything else yields dense tensors."""
    from paper_2505_06119_b200 import lib
    lib.qtnh_set_option(b"peer_direct", float(peer))
    diag = circuits.rng_normals(6, 2 * 6)
    try:
        def body(rk):
            dg = Tensor.diagonal(rk, IndexTuple([2, 2, 2, 3, 2, 3], 2), DistParams(1, 1, 0), diag)
            out = {}
            for name, f in (("rebcast", lambda t: ops.rebcast(t, DistParams(2, 1, 0))),
                            ("rebcast_cyc", lambda t: ops.rebcast(t, DistParams(1, 2, 0))),
                            ("conj", ops.conj), ("scale", lambda t: ops.scale(t, 1.5 - 2j))):
                a, b = f(dg), f(dg.to_dense())
                assert a.variant() == DIAGONAL and b.variant() == DENSE, name
                assert a.local_data().size in (0, 6)
                if a.in_span():
                    out[name] = (a.to_global_vector(), b.to_global_vector())
            p = ops.permute(dg, [1, 0, 3, 2, 5, 4], 2)
            assert p.variant() == DENSE
            return out

        for o in World(8).run(body):
            for name, (a, b) in o.items():
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), name
    finally:
        lib.qtnh_set_option(b"peer_direct", 1.0)


@pytest.mark.parametrize("world,split", [(1, 0), (4, 2), (8, 3)])
def test_diagonal_variant_gate_needs_no_exchange(world, split):
    """A CP gate given as a DIAGONAL tensor on distributed qubits: same values as the dense
    gate through contract + permute back (the reference's path), no swap of the state
    (tensor.hpp:114-142)."""
    n = 12
    P = oracle.port()
    g = circuits.counter_state(9, 2**n)
    theta = 2 * np.pi / 8
    d4 = np.array([1, 1, 1, np.exp(1j * theta)])
    dense = np.diag(d4)
    targets = [0, max(split, 1)]  # qubit 0 is distributed whenever split > 0

    def body(rk):
        st = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        st2 = Tensor.from_global(rk, IndexTuple([2] * n, split), DistParams(1, 1, 0), g)
        gate = Tensor.diagonal(rk, IndexTuple([2, 2, 2, 2], 0), DistParams(1, world, 0), d4)
        apply_gate_tensor(st, targets, gate)
        apply_gate(st2, targets, dense)
        idt = Tensor.identity(rk, IndexTuple([2, 2, 2, 2], 0), DistParams(1, world, 0), [2, 3], [0, 1])
        before = st.to_global_vector()
        apply_gate_tensor(st, targets, idt)
        assert np.array_equal(before, st.to_global_vector())
        return before, st2.to_global_vector()

    for a, b in World(world).run(body):
        want = P.gate([2] * n, g, targets, dense)
        assert np.linalg.norm(a - want) <= 1e-14 * np.linalg.norm(want)
        assert np.linalg.norm(a - b) <= 1e-14 * np.linalg.norm(want)


def test_swap_variant_gate_and_dense_gate_tensor():
    n = 10
    g = circuits.counter_state(3, 2**n)

    def body(rk):
        st = Tensor.from_global(rk, IndexTuple([2] * n, 1), DistParams(1, 1, 0), g)
        sw = Tensor.swap_tensor(rk, IndexTuple([2, 2, 2, 2], 0), DistParams(1, 2, 0), [2, 3], [0, 1])
        apply_gate_tensor(st, [0, 7], sw)
        a = st.to_global_vector()
        st3 = Tensor.from_global(rk, IndexTuple([2] * n, 1), DistParams(1, 1, 0), g)
        fs = Tensor.from_global(rk, IndexTuple([2, 2, 2, 2], 0), DistParams(1, 2, 0), circuits.FSIM.reshape(-1))
        apply_gate_tensor(st3, [3, 8], fs)
        st4 = Tensor.from_global(rk, IndexTuple([2] * n, 1), DistParams(1, 1, 0), g)
        apply_gate(st4, [3, 8], circuits.FSIM)
        with pytest.raises(InvalidArgument):
            apply_gate_tensor(st4, [3], fs)
        return a, st3.to_global_vector(), st4.to_global_vector()

    for a, b, c in World(2).run(body):
        want = g.reshape([2] * n).swapaxes(0, 7).reshape(-1)
        assert np.array_equal(a, want)
        assert np.array_equal(b, c)


def test_contraction_with_variant_operands():
    """contract() reads any variant through its dense value (remap.hpp:75-95 visits the
    non-zeros): a diagonal operand scales, an identity operand copies."""
    P = oracle.port()
    a = circuits.rng_normals(2, 2**8)
    diag = circuits.rng_normals(7, 4)

    def body(rk):
        ta = Tensor.from_global(rk, IndexTuple([2] * 8, 0), None, a)
        dg = Tensor.diagonal(rk, IndexTuple([2, 2, 2, 2], 0), None, diag)
        idt = Tensor.identity(rk, IndexTuple([2, 2, 2, 2], 0), None, [0, 1], [2, 3])
        return (contract(ta, dg, [2, 5], [0, 1]).to_global_vector(),
                contract(ta, idt, [2, 5], [0, 1]).to_global_vector())

    c1, c2 = World(1).run(body)[0]
    dd = np.zeros((4, 4), complex)
    dd[np.arange(4), np.arange(4)] = diag
    w1 = P.contract([2] * 8, a, [2] * 4, dd.reshape(-1), [2, 5], [0, 1])
    w2 = P.contract([2] * 8, a, [2] * 4, np.eye(4, dtype=complex).reshape(-1), [2, 5], [0, 1])
    assert np.linalg.norm(c1 - w1) <= 1e-13 * np.linalg.norm(w1)
    assert np.array_equal(c2, w2)


def test_variant_files_round_trip(tmp_path):
    diag = circuits.rng_normals(8, 6)

    def body(rk):
        out = []
        for name, t in (("dg", Tensor.diagonal(rk, IndexTuple([2, 2, 3, 3], 2), DistParams(1, 1, 0), diag)),
                        ("sw", Tensor.swap_tensor(rk, IndexTuple([3, 3, 3, 3], 1), DistParams(1, 1, 0), [0, 1], [2, 3])),
                        ("sy", Tensor.symmetric_from_global(rk, IndexTuple([2, 2, 2, 2], 2), DistParams(1, 1, 0),
                                                            np.arange(16.0) * (1 - 1j)))):
            p = str(tmp_path / (name + ".qtt"))
            t.save(p)
            rk.barrier()
            r = Tensor.load(rk, p)
            assert r.variant() == t.variant() and r.shape().dims == t.shape().dims
            assert np.array_equal(r.local_data(), t.local_data())
            if t.in_span():
                assert np.array_equal(r.to_global_vector(), t.to_global_vector())
            out.append(r.variant())
        return out

    assert World(4).run(body)[0] == [DIAGONAL, SWAP, SYMMETRIC]
    # a diagonal file holds the diagonal only: header (8 + 12 + 24 + 4*8 + 8) + 6 * 16 bytes
    assert (tmp_path / "dg.qtt").stat().st_size == 84 + 96
