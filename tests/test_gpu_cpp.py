"""The C++ drop-in API (cpp/include/dnd) on the GPU: the reference's own test
cases (test_pairwise/test_cluster/test_moments/test_chunking) written against
it, one rank per visible GPU up to 2 (cpp/tests/test_dnd.cpp)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_reference_cases():
    subprocess.run(["make", "-C", os.path.join(ROOT, "cpp")], check=True, capture_output=True)
    r = subprocess.run([os.path.join(ROOT, "cpp", "build", "test_dnd")], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-3000:]
    assert " 0 failed" in r.stdout


def _run(*args):
    subprocess.run(["make", "-C", os.path.join(ROOT, "cpp")], check=True, capture_output=True)
    return subprocess.run([os.path.join(ROOT, "cpp", "build", "dnd"), *args], capture_output=True, text=True,
                          timeout=600)


def _dnd(*args):
    r = _run(*args)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def _ranks():
    import torch
    return min(2, torch.cuda.device_count())


@pytest.mark.parametrize("algo", ["kmeans", "cdist", "moments"])
def test_cli_bench_report_shape(algo):
    """`dnd bench` keeps the reference report keys (tools/bench.cpp:118-128)."""
    rep = _dnd("bench", algo, "--synthetic", "20000x18", "--runs", "3", "--ranks", str(_ranks()))
    for key in ("algo", "ranks", "split", "params", "warmup_runs", "timed_runs", "mean_seconds", "std_seconds"):
        assert key in rep
    assert rep["algo"] == algo and rep["timed_runs"] == 3
    assert rep["mean_seconds"] > 0 and rep["std_seconds"] >= 0


@pytest.mark.parametrize("algo", ["kmeans", "cdist", "moments", "lasso"])
@pytest.mark.parametrize("ranks", [2, 3])
def test_cli_verify_distributed_vs_single(algo, ranks):
    """`dnd verify ALGO`: P ranks against one rank, the reference's gate lines
    (tools/verify.cpp:283-300); 3 ranks share GPUs on a 1-2 GPU box."""
    r = _run("verify", algo, "--synthetic", "3000x18", "--ranks", str(ranks))
    print(r.stdout)
    assert r.returncode == 0 and r.stdout.strip().splitlines()[-1] == "result: OK", r.stdout + r.stderr[-2000:]


def test_cli_verify_catches_an_injected_combiner_fault():
    """verify --inject-combiner-fault (verify.cpp:57-73): the corrupted moments
    combiner must FAIL the gate (exit 1) -- the gate is not vacuous."""
    r = _run("verify", "moments", "--synthetic", "3000x18", "--ranks", "3", "--inject-combiner-fault")
    print(r.stdout)
    assert r.returncode == 1 and "FAIL" in r.stdout, r.stdout + r.stderr[-2000:]


def test_cli_bench_from_dnb_file(tmp_path):
    """`dnd bench --data FILE.dnb`: the container is loaded straight into HBM
    (dataio.hpp:102-142) and gives the same fit as the in-memory array."""
    import numpy as np

    x = np.random.default_rng(3).random((20000, 18), dtype=np.float32)
    path = tmp_path / "x.dnb"
    with open(path, "wb") as f:
        f.write(b"DNB1" + bytes([1, 2]) + np.array(x.shape, "<u8").tobytes() + x.tobytes())
    rep = _dnd("bench", "kmeans", "--data", str(path), "--runs", "2", "--ranks", str(_ranks()))
    assert rep["params"]["rows"] == 20000 and rep["params"]["cols"] == 18
    r = _run("bench", "kmeans", "--data", str(tmp_path / "nope.dnb"))
    assert r.returncode == 2 and "cannot open" in r.stderr
