"""QTNHTEN1 serialization (tensor.hpp:373-446) interoperating with the unmodified
reference in both directions."""
import os

import numpy as np
import pytest

import oracle
from conftest import bits
from paper_2505_06119_b200 import circuits
from paper_2505_06119_b200.qtnh import DistParams, Error, IndexTuple, Tensor, World

pytestmark = pytest.mark.gpu


def test_reference_file_round_trip(tmp_path):
    if not oracle.ref_available():
        pytest.skip("reference build absent")
    R = oracle.ref()
    dims, split = [2, 3, 4, 2], 2
    g = np.array([complex(0.5 * i, 1.0 / (1 + i)) for i in range(48)])  # test_tensor.cpp:197-198
    ref_file = str(tmp_path / "ref.qtt")
    R.save(6, dims, split, (1, 1, 0), g, ref_file)

    def body(rk):
        t = Tensor.load(rk, ref_file)
        assert t.shape().dims == dims and t.shape().split == split
        v = t.to_global_vector()
        rk.barrier()
        t.save(str(tmp_path / "ours.qtt"))
        rk.barrier()
        return v

    got = World(6).run(body)[0]
    assert np.array_equal(bits(got), bits(g))
    d, s, dist, back = R.load(6, str(tmp_path / "ours.qtt"))
    assert d == dims and s == split and dist == (1, 1, 0)
    assert np.array_equal(bits(back), bits(g))
    # byte-identical files
    assert open(ref_file, "rb").read() == open(str(tmp_path / "ours.qtt"), "rb").read()


def test_bad_stream(tmp_path):
    p = tmp_path / "bad.qtt"
    p.write_bytes(b"NOTQTNH!")

    def body(rk):
        with pytest.raises(Error):
            Tensor.load(rk, str(p))
        return True

    assert World(1).run(body)[0]


@pytest.mark.parametrize("dims,split,dist,world", [
    ([2] * 22, 3, (1, 1, 0), 8),      # 64 MiB, 8 blocks written in parallel (multi-chunk per block)
    ([3, 2, 4, 7, 2], 1, (2, 1, 1), 7),  # stretched copies + offset: only canonical holders write
    ([4, 4, 4], 1, (1, 2, 0), 8),        # cyclic copies
    ([6, 5], 0, (1, 1, 2), 3),           # one block on rank 2
])
def test_device_save_load_matches_reference(tmp_path, dims, split, dist, world):
    """Device-side save (each canonical holder pwrites its block) produces the
    reference's bytes, signed zeros included; device-side load (each rank preads
    its block) round-trips bit-exactly on every copy."""
    g = circuits.counter_state(77, int(np.prod(dims)))
    g[::7] = complex(-0.0, -0.0)
    g[1::11] = complex(0.0, -0.0)
    g[2::13] = complex(-0.0, 1.5)
    ours = str(tmp_path / "ours.qtt")

    def body(rk):
        t = Tensor.from_global(rk, IndexTuple(dims, split), DistParams(*dist), g)
        t.save(ours)
        rk.barrier()  # save is span-collective; ranks outside the span must not read early
        u = Tensor.load(rk, ours)
        out = u.to_global_vector() if u.in_span() else None
        return out

    outs = [o for o in World(world).run(body) if o is not None]
    for o in outs:
        assert np.array_equal(bits(o), bits(g))
    if oracle.ref_available():
        R = oracle.ref()
        ref_file = str(tmp_path / "ref.qtt")
        R.save(world, dims, split, dist, g, ref_file)
        assert open(ref_file, "rb").read() == open(ours, "rb").read()


def test_truncated_file_is_an_error(tmp_path):
    dims = [2] * 10
    g = circuits.counter_state(5, 2**10)
    p = str(tmp_path / "t.qtt")

    def body(rk):
        Tensor.from_global(rk, IndexTuple(dims, 0), None, g).save(p)
        data = open(p, "rb").read()
        open(p, "wb").write(data[:-100])
        with pytest.raises(Error):
            Tensor.load(rk, p)
        return True

    assert World(1).run(body)[0]
