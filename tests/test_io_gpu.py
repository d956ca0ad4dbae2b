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
