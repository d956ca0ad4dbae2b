import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path of libqtnh_b200.so)")
    config.addinivalue_line("markers", "slow: long-running parity case")


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    import json

    import numpy as np

    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:  # materialise: NpzFile is not thread-safe
        arrays = {k: z[k] for k in z.files}
    return json.loads(str(arrays.pop("meta"))), arrays


def bits(x):
    """Bit pattern view (exact equality including signed zeros)."""
    import numpy as np

    return np.ascontiguousarray(x, dtype=np.complex128).view(np.uint64)


def rel_l2(a, b):
    import numpy as np

    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(params=[1, 0], ids=["peer", "exchange"])
def peer_mode(request):
    """Run a multi-rank test through both redistribution forms of the local
    world: peer-memory kernels (push remap, pairwise in-place swap) and the
    pack -> exchange -> unpack path the NCCL world uses."""
    from paper_2505_06119_b200.qtnh import check, lib

    check(lib.qtnh_set_option(b"peer_direct", float(request.param)))
    yield request.param
    check(lib.qtnh_set_option(b"peer_direct", 1.0))


@pytest.fixture(autouse=True)
def _restore_process_wide_options():
    """Options set through qtnh_set_option are process-wide; a test that leaves
    "pool_reserve_gb" set makes every later world map (and trim) that much HBM."""
    yield
    mod = sys.modules.get("paper_2505_06119_b200.qtnh")
    if mod is not None:
        mod.lib.qtnh_set_option(b"pool_reserve_gb", 0.0)
