"""Process-per-GPU world over CUDA IPC: N processes (sharing this box's GPU) run
the distributed ops through cross-process peer memory and the pull-copy exchange,
each checking parity against the oracle (tests/workers/ipc_worker.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("nproc,legacy_min", [(2, None), (3, None), (4, None), (2, "0")])
def test_ipc_world_ops(tmp_path, nproc, legacy_min):
    """legacy_min "0": every block goes through legacy IPC handles (the path of
    multi-GiB shards)."""
    env_base = dict(os.environ, WORLD_SIZE=str(nproc), QTNH_IPC_DIR=str(tmp_path / "rdv"),
                    QTNH_COLLECTIVE_TIMEOUT_MS="60000")
    if legacy_min is not None:
        env_base["QTNH_IPC_LEGACY_MIN"] = legacy_min
    procs = []
    for r in range(nproc):
        env = dict(env_base, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "workers", "ipc_worker.py")],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append((p.returncode, out))
    bad = [f"rank {r} rc={rc}:\n{out[-2500:]}" for r, (rc, out) in enumerate(outs) if rc != 0 or "ipc rank ok" not in out]
    assert not bad, "\n".join(bad)
