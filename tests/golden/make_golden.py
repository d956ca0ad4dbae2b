"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libqtnh_ref.so).

Run in the build container (needs the reference build): ``python tests/golden/make_golden.py``.
Each fixture stores its inputs, the reference's output and the exact call, so the
CPU suite can pin the C restatement (oracle/qtnh_oracle.c) and the GPU suite can
check the CUDA path without /root/reference.

Cases follow the reference's own tests where they exist (proj/tests/test_ops.cpp,
test_tensor.cpp) and SURVEY.md section 8 for the contraction / gate / QFT / SVD paths,
which the reference leaves untested (test_linalg.cpp:1 is empty).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R = oracle.ref()
H = R.hash_counter


def iota_global(n):  # test_ops.cpp:28-32
    return np.array([complex(i + 1, 0.1 * i) for i in range(n)])


def random_dims(seed, max_rank):  # test_ops.cpp:51-56
    r = 1 + H(seed, 1) % max_rank
    return [1 + H(seed, 2, i) % 3 for i in range(r)]


def fy_perm(seed, tag, r):  # test_ops.cpp:124-129
    p = list(range(r))
    for i in range(r - 1, 0, -1):
        j = H(seed, tag, i) % (i + 1)
        p[i], p[j] = p[j], p[i]
    return p


def save(name, meta, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), meta=json.dumps(meta), **arrays)


def main():
    cases = []
    # 1. transpose known answer (test_ops.cpp:77-85)
    g = np.array([1, 2, 3, 4], dtype=complex)
    out, d, s, _ = R.permute(1, [2, 2], 0, None, g, [1, 0], 0)
    cases.append(dict(world=1, dims=[2, 2], split=0, dist=[1, 1, 0], perm=[1, 0], new_split=0,
                      out_dims=d, out_split=s, inp=g, out=out))
    # 2. asymmetric permutation (test_ops.cpp:87-110)
    g = iota_global(32)
    out, d, s, dist = R.permute(4, [2, 2, 4, 2], 1, (1, 1, 0), g, [2, 0, 1, 3], 1)
    cases.append(dict(world=4, dims=[2, 2, 4, 2], split=1, dist=[1, 1, 0], perm=[2, 0, 1, 3], new_split=1,
                      out_dims=d, out_split=s, inp=g, out=out))
    # 3. round trip / composition seeds (test_ops.cpp:112-159), forward permutation only
    for seed in range(8):
        dims = random_dims(seed, 5)
        r = len(dims)
        split = H(seed, 3) % (r + 1)
        while int(np.prod(dims[:split])) > 4:
            split -= 1
        p = fy_perm(seed, 4, r)
        ns = H(seed, 6) % (r + 1)
        while int(np.prod([dims[p[i]] for i in range(ns)])) > 4:
            ns -= 1
        g = iota_global(int(np.prod(dims)))
        out, d, s, _ = R.permute(4, dims, split, (1, 1, 0), g, p, ns)
        cases.append(dict(world=4, dims=dims, split=split, dist=[1, 1, 0], perm=p, new_split=ns,
                          out_dims=d, out_split=s, inp=g, out=out))
    # 4. signed zeros (remap.hpp:69-70): (-0,-0) -> (+0,+0); (-0,1), (1,-0) keep signs
    g = np.array([complex(-0.0, -0.0), complex(-0.0, 1.0), complex(1.0, -0.0), complex(0.0, -0.0),
                  complex(2, 3), complex(-0.0, 0.0), complex(5, 0), complex(0, 0)])
    out, d, s, _ = R.permute(2, [2, 2, 2], 1, (1, 1, 0), g, [2, 1, 0], 1)
    cases.append(dict(world=2, dims=[2, 2, 2], split=1, dist=[1, 1, 0], perm=[2, 1, 0], new_split=1,
                      out_dims=d, out_split=s, inp=g, out=out))
    # 5. random qubit permutations, distributed (world 8, split 3 -> other splits)
    for seed in range(4):
        n = 12
        g = oracle.port().counter_normals(100 + seed, 0, 2 ** n)
        p = fy_perm(100 + seed, 7, n)
        ns = [0, 1, 2, 3][seed]
        out, d, s, _ = R.permute(8, [2] * n, 3, (1, 1, 0), g, p, ns)
        cases.append(dict(world=8, dims=[2] * n, split=3, dist=[1, 1, 0], perm=p, new_split=ns,
                          out_dims=d, out_split=s, inp=g, out=out))
    arr = {}
    meta = []
    for i, c in enumerate(cases):
        arr[f"in{i}"] = c.pop("inp")
        arr[f"out{i}"] = c.pop("out")
        meta.append(c)
    save("permute", meta, **arr)

    # rebcast (test_ops.cpp:161-192)
    g = iota_global(4)
    rb = []
    arr = {}
    for i, nd in enumerate([(2, 1, 0), (1, 2, 0), (1, 1, 0), (1, 1, 2)]):
        arr[f"out{i}"] = R.rebcast(4, [2, 2], 1, (1, 1, 0), g, nd)
        rb.append(dict(world=4, dims=[2, 2], split=1, dist=[1, 1, 0], new_dist=list(nd)))
    arr["inp"] = g
    save("rebcast", rb, **arr)

    # scatter / gather (test_ops.cpp:218-248)
    g = iota_global(4)
    s_out, sd, ss = R.scatter_gather(2, 0, [2, 2], 0, None, g, 0)
    g_out, gd, gs = R.scatter_gather(2, 1, [2, 2], 1, None, s_out, 0)
    save("scatter_gather", dict(scatter=dict(dims=sd, split=ss), gather=dict(dims=gd, split=gs)),
         inp=g, scatter=s_out, gather=g_out)

    # contraction (SPEC.md:361-369 composed as t2m -> pgemm -> m2t), seeded
    cc = []
    arr = {}
    for i, (na, nb, k, world, sa) in enumerate([(10, 6, 3, 1, 0), (12, 8, 4, 4, 2), (9, 9, 5, 2, 1)]):
        a = R.rng_complex_normals(200 + i, 2 ** na)
        b = R.rng_complex_normals(300 + i, 2 ** nb)
        ap = sorted(fy_perm(200 + i, 8, na)[:k])
        bp = sorted(fy_perm(300 + i, 8, nb)[:k])
        out, d, s = R.contract(world, [2] * na, sa, (1, 1, 0), a, [2] * nb, 0, (1, 1, 0), b, ap, bp)
        arr[f"a{i}"], arr[f"b{i}"], arr[f"out{i}"] = a, b, out
        cc.append(dict(world=world, da=[2] * na, sa=sa, db=[2] * nb, sb=0, apos=ap, bpos=bp, out_dims=d, out_split=s))
    # general dims (3, 5)
    da, db = [3, 2, 5, 2], [5, 3, 4]
    a = R.rng_complex_normals(400, int(np.prod(da)))
    b = R.rng_complex_normals(401, int(np.prod(db)))
    out, d, s = R.contract(1, da, 0, None, a, db, 0, None, b, [0, 2], [1, 0])
    i = len(cc)
    arr[f"a{i}"], arr[f"b{i}"], arr[f"out{i}"] = a, b, out
    cc.append(dict(world=1, da=da, sa=0, db=db, sb=0, apos=[0, 2], bpos=[1, 0], out_dims=d, out_split=s))
    save("contract", cc, **arr)

    # gate application (contract + permute back) and QFT
    n = 8
    st = oracle.port().counter_normals(11, 0, 2 ** n)
    st /= np.linalg.norm(st)
    r2 = 1 / np.sqrt(2)
    hgate = np.array([r2, r2, r2, -r2], dtype=complex)
    th = 2 * np.pi / 8
    cp = np.diag([1, 1, 1, np.exp(1j * th)]).reshape(-1)
    rnd = R.rng_complex_normals(12, 16)
    gates = [([3], hgate), ([0], hgate), ([7], hgate), ([5, 2], cp), ([1, 6], rnd), ([7, 0], rnd)]
    gg = []
    arr = {"state": st}
    for i, (t, gm) in enumerate(gates):
        arr[f"g{i}"] = gm
        arr[f"out{i}"] = R.gate(1, n, 0, None, st, t, gm)
        gg.append(dict(targets=t))
    arr["out_dist"] = R.gate(4, n, 2, (1, 1, 0), st, [1, 6], rnd)
    save("gate", dict(n=n, gates=gg, dist_case=dict(world=4, split=2, targets=[1, 6], gate=4)), **arr)

    n = 10
    st = oracle.port().counter_normals(5, 0, 2 ** n)
    st /= np.linalg.norm(st)
    save("qft10", dict(n=n, seed=5), state=st, out=R.qft(n, st, swaps=True), out_noswap=R.qft(n, st, swaps=False))

    # SVD + truncation + absorption (linalg.hpp:441-523)
    m = R.rng_complex_normals(21, 48 * 40).reshape(48, 40)
    u, s, vh = R.svd(m, chi=16, absorb=1)
    u2, s2, vh2 = R.svd(m, chi=64, absorb=0)  # zero-pad above rank
    save("svd", dict(m=48, n=40), a=m, u=u, s=s, vh=vh, u_pad=u2, s_pad=s2, vh_pad=vh2)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
