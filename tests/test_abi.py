"""CPU: the C-ABI library loads, exports every symbol include/qtnh_b200.h declares,
and its host-side validation maps to the reference's error classes (no GPU needed)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "qtnh_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qtnh_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2505_06119_b200 import lib

    names = declared_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_sass_is_sm100a_with_dmma():
    import shutil
    import subprocess

    from paper_2505_06119_b200 import LIB_PATH

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # complex128 GEMM on the FP64 tensor cores


def test_version_and_error_mapping():
    from paper_2505_06119_b200 import qtnh

    assert b"sm_100a" in qtnh.lib.qtnh_version()
    with pytest.raises(qtnh.InvalidArgument):
        qtnh.World(0)
    with pytest.raises(qtnh.InvalidArgument):
        qtnh.IndexTuple([2, 0], 0)
    with pytest.raises(qtnh.InvalidArgument):
        qtnh.IndexTuple([2, 2], 3)
    assert qtnh.IndexTuple([2, 3, 4, 2], 2).str() == "(2,3;4,2)"
    assert qtnh.IndexTuple([], 0).total_size() == 1


def test_world_creation_is_host_only():
    from paper_2505_06119_b200 import qtnh

    w = qtnh.World(3)
    assert w.size() == 3
    w.close()


def _build_cpp_example(tmp_path):
    import subprocess

    exe = tmp_path / "test_api"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/test_api.cpp",
                    f"-L{ROOT}/paper_2505_06119_b200", "-l:libqtnh_b200.so",
                    f"-Wl,-rpath,{ROOT}/paper_2505_06119_b200", "-lpthread", "-o", str(exe)], check=True)
    return exe


def test_cpp_header_layer_compiles(tmp_path):
    """include/qtnh_b200.hpp (the reference-shaped C++ API) builds against the ABI."""
    assert _build_cpp_example(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_header_layer_runs(tmp_path):
    import subprocess

    exe = _build_cpp_example(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "cpp api ok" in out.stdout


def _read_dropin(path):
    out, lines, i = {}, open(path).read().splitlines(), 0
    import numpy as np

    while i < len(lines):
        name, rest = lines[i].split(" ", 1)
        if name in ("a2a_error", "u_chi3_absorbed"):
            out[name] = rest
            i += 1
            continue
        n = int(rest)
        vals = [complex(*map(float, ln.split())) for ln in lines[i + 1:i + 1 + n]]
        out[name] = np.array(vals, dtype=complex)
        i += 1 + n
    return out


def _build_dropin(tmp_path):
    import subprocess

    exe = tmp_path / "test_linalg_dropin"
    subprocess.run(["g++", "-std=c++17", "-O2", "-DQTNH_B200", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/test_linalg_dropin.cpp", f"-L{ROOT}/paper_2505_06119_b200",
                    "-l:libqtnh_b200.so", f"-Wl,-rpath,{ROOT}/paper_2505_06119_b200", "-lpthread", "-o", str(exe)],
                   check=True)
    return exe


def test_reference_call_sequence_compiles_by_namespace_swap(tmp_path):
    """tests/cpp/test_linalg_dropin.cpp -- t2m -> pgemm -> m2t -> psvd -> truncate_svd ->
    absorb(power), Tensor value semantics, Group collectives -- is the same source the
    reference headers compile (oracle/Makefile `dropin`, golden committed); here it
    builds against include/qtnh_b200.hpp with only the namespace alias switched."""
    assert _build_dropin(tmp_path).exists()
    assert os.path.exists(os.path.join(ROOT, "tests", "golden", "linalg_dropin_ref.txt"))


@pytest.mark.gpu
def test_reference_call_sequence_matches_reference_output(tmp_path):
    import subprocess

    import numpy as np

    exe = _build_dropin(tmp_path)
    out = tmp_path / "b200.txt"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = _read_dropin(out)
    want = _read_dropin(os.path.join(ROOT, "tests", "golden", "linalg_dropin_ref.txt"))
    assert set(got) == set(want)

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

    for k in ("contract", "s", "s_pad12", "recon_chi3", "recon_chi12", "copy_scaled", "original_after_copy"):
        assert got[k].shape == want[k].shape, k
        assert rel(got[k], want[k]) < 1e-10, (k, rel(got[k], want[k]))
    assert np.array_equal(got["collectives"], want["collectives"])
    assert got["a2a_error"] == want["a2a_error"]
    assert got["u_chi3_absorbed"] == want["u_chi3_absorbed"]
    assert np.allclose(got["copy_scaled"], 2j * got["original_after_copy"])


def _build_tensor_dropin(tmp_path):
    import subprocess

    exe = tmp_path / "test_tensor_dropin"
    subprocess.run(["g++", "-std=c++17", "-O2", "-DQTNH_B200", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/test_tensor_dropin.cpp", f"-L{ROOT}/paper_2505_06119_b200",
                    "-l:libqtnh_b200.so", f"-Wl,-rpath,{ROOT}/paper_2505_06119_b200", "-lpthread", "-o", str(exe)],
                   check=True)
    return exe


def test_tensor_variant_sequences_compile_by_namespace_swap(tmp_path):
    """tests/cpp/test_tensor_dropin.cpp -- layout arithmetic (indexing.hpp), dense
    distribution and element lookup, the symmetric / diagonal / identity / swap
    variants, to_dense, variant-keeping rebcast / conj / scale, every structural op
    on every variant, QTNHTEN1 files of every variant, error classes -- is the same
    source the reference headers compile (oracle/Makefile `dropin`, golden
    committed); here it builds against include/qtnh_b200.hpp by namespace swap."""
    assert _build_tensor_dropin(tmp_path).exists()
    assert os.path.exists(os.path.join(ROOT, "tests", "golden", "tensor_dropin_ref.txt"))


@pytest.mark.gpu
def test_tensor_variant_sequences_match_reference_output_exactly(tmp_path):
    """Every record (values at %.17g, variant tags, stored sizes, homes, the BYTES of
    the six saved files, error classes and messages) equals the reference's."""
    import subprocess

    exe = _build_tensor_dropin(tmp_path)
    out, scratch = tmp_path / "b200.txt", tmp_path / "scratch"
    scratch.mkdir()
    r = subprocess.run([str(exe), str(out), str(scratch)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr

    def read(p):
        return dict(ln.split(" = ", 1) for ln in open(p).read().splitlines())

    got, want = read(out), read(os.path.join(ROOT, "tests", "golden", "tensor_dropin_ref.txt"))
    assert set(got) == set(want)
    bad = [k for k in sorted(want) if got[k] != want[k]]
    assert not bad, [(k, got[k][:200], want[k][:200]) for k in bad[:5]]
    assert len(want) > 2000
