"""CPU: pin the C restatement (oracle/qtnh_oracle.c) against the reference's golden
vectors, its own known-answer tests (proj/tests/test_ops.cpp) and -- where the
reference build is present -- live calls into the unmodified reference."""
import numpy as np
import pytest

import oracle
from conftest import bits, golden, rel_l2

P = oracle.port()


def ref_or_skip():
    if not oracle.ref_available():
        pytest.skip("reference build (oracle/_ref) not present")
    return oracle.ref()


def test_hash_counter_and_rng_match_reference():
    R = ref_or_skip()
    for seed in [0, 1, 7, 2**63 + 5]:
        for k in [(0, 0, 0), (1, 2, 3), (5, 0, 9)]:
            assert P.hash_counter(seed, *k) == R.hash_counter(seed, *k)
        assert np.array_equal(bits(P.rng_complex_normals(seed, 513)), bits(R.rng_complex_normals(seed, 513)))


def test_product_rng_matches_oracle():
    # the product's host input generators must reproduce the reference stream bit for bit
    from paper_2505_06119_b200 import circuits

    assert np.array_equal(bits(circuits.rng_normals(3, 1000)), bits(P.rng_complex_normals(3, 1000)))
    assert np.array_equal(bits(circuits.counter_state(9, 70000)), bits(P.counter_normals(9, 0, 70000)))
    assert np.array_equal(bits(circuits.counter_state(9, 1000, start=5000)), bits(P.counter_normals(9, 5000, 1000)))
    assert circuits.hash_counter(4, 1, 2, 3) == P.hash_counter(4, 1, 2, 3)


def test_transpose_known_answer():
    # test_ops.cpp:77-85
    out = P.permute([2, 2], np.array([1, 2, 3, 4], complex), [1, 0])
    assert np.array_equal(out, np.array([1, 3, 2, 4], complex))


def test_permute_golden_bit_exact():
    meta, z = golden("permute")
    for i, m in enumerate(meta):
        out = P.permute(m["dims"], z[f"in{i}"], m["perm"])
        assert np.array_equal(bits(out), bits(z[f"out{i}"])), f"case {i}: {m}"
        assert m["out_dims"] == [m["dims"][p] for p in m["perm"]]


def test_signed_zero_canonicalisation():
    # remap.hpp:69-70 + :125-127: (-0,-0) -> (+0,+0); partial zeros keep their sign
    meta, z = golden("permute")
    idx = [i for i, m in enumerate(meta) if m["dims"] == [2, 2, 2] and m["perm"] == [2, 1, 0]][0]
    out = z[f"out{idx}"]
    inp = z[f"in{idx}"]
    perm_in = inp.reshape(2, 2, 2).transpose(2, 1, 0).reshape(-1)
    for a, b in zip(out, perm_in):
        if a.real == 0 and a.imag == 0:
            assert not np.signbit(a.real) and not np.signbit(a.imag)
        else:
            assert np.signbit(a.real) == np.signbit(b.real) and np.signbit(a.imag) == np.signbit(b.imag)


def test_contract_golden():
    meta, z = golden("contract")
    for i, m in enumerate(meta):
        out = P.contract(m["da"], z[f"a{i}"], m["db"], z[f"b{i}"], m["apos"], m["bpos"])
        assert rel_l2(out, z[f"out{i}"]) < 1e-13, m


def test_gate_golden():
    meta, z = golden("gate")
    dims = [2] * meta["n"]
    for i, g in enumerate(meta["gates"]):
        out = P.gate(dims, z["state"], g["targets"], z[f"g{i}"])
        assert rel_l2(out, z[f"out{i}"]) < 1e-14


def test_qft_golden_and_dft():
    meta, z = golden("qft10")
    n = meta["n"]
    out = P.qft(n, z["state"], swaps=True)
    assert rel_l2(out, z["out"]) < 1e-13
    # analytic QFT = unitary inverse-sign DFT
    dft = np.fft.ifft(z["state"]) * np.sqrt(2**n)
    assert rel_l2(out, dft) < 1e-13
    assert rel_l2(P.qft(n, z["state"], swaps=False), z["out_noswap"]) < 1e-13


def test_svd_golden_properties():
    meta, z = golden("svd")
    a, u, s, vh = z["a"], z["u"], z["s"], z["vh"]
    # absorb left: a ~= u @ vh with the discarded weight as the only error
    sv = np.linalg.svd(a, compute_uv=False)
    err = np.linalg.norm(a - u @ vh) ** 2
    assert abs(err - np.sum(sv[16:] ** 2)) < 1e-9 * np.sum(sv**2)
    assert np.all(np.diff(s) <= 0)
    # zero padding to chi above the rank (linalg.hpp:488-501)
    assert z["s_pad"].shape == (64,) and np.all(z["s_pad"][40:] == 0)
    assert np.all(z["u_pad"][:, 40:] == 0) and np.all(z["vh_pad"][40:, :] == 0)


def test_live_reference_random_permutes():
    R = ref_or_skip()
    rng = np.random.default_rng(1)
    for trial in range(6):
        r = int(rng.integers(1, 7))
        dims = [int(d) for d in rng.integers(1, 4, size=r)]
        data = rng.standard_normal(int(np.prod(dims))) + 1j * rng.standard_normal(int(np.prod(dims)))
        data[::3] = 0
        perm = [int(p) for p in rng.permutation(r)]
        out, d, s, _ = R.permute(1, dims, 0, None, data, perm, 0)
        assert np.array_equal(bits(out), bits(P.permute(dims, data, perm)))


def test_live_reference_contract_general_dims():
    R = ref_or_skip()
    da, db = [2, 3, 4, 3], [3, 5, 4]
    a = P.rng_complex_normals(1, int(np.prod(da)))
    b = P.rng_complex_normals(2, int(np.prod(db)))
    out, d, s = R.contract(1, da, 0, None, a, db, 0, None, b, [1, 2], [0, 2])
    assert d == [2, 3, 5]
    assert rel_l2(P.contract(da, a, db, b, [1, 2], [0, 2]), out) < 1e-14


def test_resource_error_on_small_world():
    # test_ops.cpp:102-109: asymmetric permute on a 2-rank world
    R = ref_or_skip()
    g = np.arange(32, dtype=complex)
    with pytest.raises(oracle.OracleError) as e:
        R.permute(2, [2, 2, 4, 2], 1, (1, 1, 0), g, [2, 0, 1, 3], 1)
    assert e.value.code == 2 and e.value.info == 4


def test_bench_c1_sample_is_a_slice_of_the_rank28_contraction():
    """bench.py's CPU arms time 1/64 slices of the C1 contraction (first six open
    indices of the rank-28 A fixed). The reference's output for a slice must equal
    the definition-level brute force of those rows of the rank-28 result."""
    import bench

    if not oracle.ref_available():
        pytest.skip("reference build absent")
    P = oracle.port()
    _, _, _, _, outs = bench.cpu_reference_c1(budget_s=0.0, blocks=[37], keep_outputs=True)
    rows = bench.C1Sample.rows(37)
    idx = np.arange(rows.start, rows.stop)[::997]
    bf = bench.c1_brute_force(P, idx)
    ref = outs[37][idx - rows.start]
    assert np.linalg.norm(bf - ref) <= 1e-13 * np.linalg.norm(ref)
