"""The C-ABI boundary (include/dndc.h) without a GPU: the library loads, exports
every declared symbol, and its host-only entry points behave like the
reference functions they replace."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2007_13552_b200 import _lib


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # the binding table covers the header exactly
    assert sorted(_lib._SIGS) == declared


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_chunk_map_host(oracle):
    for n, p in [(5, 3), (3, 5), (200_000, 8), (0, 2)]:
        off = np.empty(p, np.int64)
        ext = np.empty(p, np.int64)
        assert _lib.lib().dndc_chunk_map(n, p, off.ctypes.data, ext.ctypes.data) == 0
        o2, e2 = oracle.chunk_map(n, p)
        assert np.array_equal(off, o2) and np.array_equal(ext, e2)
    assert _lib.lib().dndc_chunk_map(5, 0, None, None) == _lib.DNDC_EVALUE
    assert b"rank count" in _lib.lib().dndc_last_error()


@pytest.mark.parametrize("n,k,s", [(100, 8, 21), (6, 6, 77), (100_000_000, 8, 42), (50_000_000, 64, 42)])
def test_init_indices_host(golden, n, k, s):
    out = np.empty(k, np.int64)
    assert _lib.lib().dndc_kmeans_init_indices(n, k, s, out.ctypes.data) == 0
    assert np.array_equal(out, golden[f"init_{n}_{k}_{s}"])


def test_value_errors_map_to_python():
    out = np.empty(4, np.int64)
    with pytest.raises(ValueError, match="out of range"):
        _lib.check(_lib.lib().dndc_kmeans_init_indices(3, 4, 1, out.ctypes.data))


def test_create_rejects_bad_rank_without_touching_cuda():
    h = C.c_void_p()
    rc = _lib.lib().dndc_create(0, 3, 2, None, C.byref(h))
    assert rc == _lib.DNDC_EVALUE
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_product_package_never_uses_the_oracle():
    """The oracle is the checker only: no import, link or symbol use in the product."""
    import pathlib
    import re
    import subprocess

    pkg = pathlib.Path(_lib.HERE)
    bad = re.compile(r"(from|import)\s+oracle|liboracle|libdndref|\bdno_|\bref_(kmeans|cdist|bench)")
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert not bad.search(f.read_text()), f
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "dndref" not in deps


def test_cpp_dropin_compiles_against_the_c_abi():
    """cpp/include/dnd (the reference's C++ API names) builds over include/dndc.h
    and links libdndc.so only -- no CUDA headers on the host side."""
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["make", "-C", os.path.join(root, "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(os.path.join(root, "cpp", "build", "test_dnd"))
    assert os.path.exists(os.path.join(root, "cpp", "build", "dnd"))
    for h in ("ndarray.hpp", "pairwise.hpp", "cluster.hpp", "moments.hpp", "transport.hpp", "chunking.hpp",
              "dataio.hpp", "regression.hpp"):
        src = open(os.path.join(root, "cpp", "include", "dnd", h)).read()
        assert "cuda_runtime" not in src and "#include <cuda" not in src


def test_cli_usage_errors_and_no_cpu_fallback():
    """`dnd` (F3, tools/main.cpp:12-83): bad command lines exit 2 with the
    usage line; a runtime dnd::Error exits 2 with "error: " (main.cpp:78-82);
    a valid command on a host without a GPU fails loudly, it never computes on
    the CPU; `convert` writes a DNB container without any GPU."""
    import subprocess
    import tempfile

    import torch

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["make", "-C", os.path.join(root, "cpp")], capture_output=True, check=True)
    exe = os.path.join(root, "cpp", "build", "dnd")
    for args in (["frobnicate"], ["bench", "svm"], ["bench", "kmeans", "--synthetic", "12"], ["bench", "kmeans", "--k"],
                 ["bench", "load"], ["bench"], ["verify", "kmeans", "--split", "2"], ["convert", "a.csv"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and "usage: dnd" in r.stderr, (args, r.stderr)
    with tempfile.TemporaryDirectory() as d:
        csv = os.path.join(d, "x.csv")
        open(csv, "w").write("a,b,c\n1,2,3\n4,5,6.5\n")
        r = subprocess.run([exe, "convert", csv, os.path.join(d, "x.dnb"), "--dtype", "f32", "--skip-header"],
                           capture_output=True, text=True, timeout=60)
        assert r.returncode == 0 and "wrote" in r.stderr and "2x3" in r.stderr, r.stderr
        raw = open(os.path.join(d, "x.dnb"), "rb").read()
        assert raw[:4] == b"DNB1" and np.array_equal(np.frombuffer(raw[-24:], "<f4"), [1, 2, 3, 4, 5, 6.5])
        r = subprocess.run([exe, "convert", os.path.join(d, "missing.csv"), os.path.join(d, "y.dnb")],
                           capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and r.stderr.startswith("error: ")
    if not torch.cuda.is_available():
        r = subprocess.run([exe, "bench", "kmeans", "--synthetic", "100x4"], capture_output=True,
                           text=True, timeout=60)
        assert r.returncode == 2 and r.stderr.startswith("error: ")
