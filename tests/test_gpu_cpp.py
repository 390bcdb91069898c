"""The C++ drop-in API (cpp/include/dnd) on the GPU: the reference's own test
cases (test_pairwise/test_cluster/test_moments/test_chunking) written against
it, one rank per visible GPU up to 2 (cpp/tests/test_dnd.cpp)."""
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
