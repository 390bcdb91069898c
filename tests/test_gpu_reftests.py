"""The reference's OWN unit tests, unchanged, against the B200 drop-in.

cpp/reftests/Makefile compiles /root/reference/proj/tests/test_pairwise.cpp,
test_cluster.cpp and test_moments.cpp as they are -- the same TEST_CASEs,
run_world(1..5) worlds, oracles (tests/support/oracles.hpp) and tolerances --
against cpp/include/dnd (this repo's headers over libdndc.so) instead of the
reference library.  Worlds larger than the box's GPU count share GPUs through
libdndc's host loopback group (dndc_create_in_group).  Every case must pass.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["pairwise", "cluster", "moments"])
def test_reference_unit_tests_pass_unchanged(name):
    exe = os.path.join(ROOT, "cpp", "build", f"ref_test_{name}")
    if not os.path.exists(exe):
        pytest.skip("built only where /root/reference exists (cpp/reftests/Makefile)")
    env = dict(os.environ, DND_TIMEOUT_SECS="120")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
