"""Parity at BASELINE.json's configuration sizes.

Every check runs the full-size GPU path and compares it with the unmodified
reference (committed fixtures from oracle/_ref: tests/golden/cfg_golden.npz,
made by tests/golden/make_golden_cfg.py) or with the oracle restatement run on
this box's host at the same size:

  cfg1  5M x 18, k=8, 20 iterations: labels and per-cluster counts, exact
        (cluster.cpp:44-56, :112-122)
  cfg3  the survey's 5M x 64, k=64 slice: centroids/trace at 1e-5, labels and
        counts exact (cluster.cpp:83-153); delta == full accumulation
  cfg4  100k x 1024 vs 100k x 1024 cdist_xy: sampled row panels at 1e-5
        (pairwise.cpp:87-100)
  cfg5  100M x 32 moments at 1e-12 against the reference's single-rank
        Welford chain (moments.cpp:100-134), and k-means++ (k=8) against the
        oracle's restatement (A16: no k-means++ in the reference)
Gate metric: |a - b| / max(1, |ref|) (tools/verify.cpp:24-28).
"""
import os

import numpy as np
import pytest
import torch

import paper_2007_13552_b200.api as dnd
from _parity import label_digest, rel_dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def cfg_golden():
    return np.load(os.path.join(HERE, "golden", "cfg_golden.npz"))


def _host_ram_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


def _labels(model, x):
    return dnd.gather(dnd.kmeans_predict(model, x)).astype(np.int64)


def test_cfg1_labels_and_counts_match_reference(comm, oracle, golden, cfg_golden):
    n, m, k = 5_000_000, 18, 8
    x = dnd.random_uniform((n, m), 0, 42, comm)
    model = dnd.kmeans_fit(x, k, 20, 0.0, 42)
    assert rel_dev(model.centroids, golden["cfg1_centroids"]) <= 1e-5
    lab = _labels(model, x)
    # (1) the GPU decision is the reference's decision for the same centroids
    want = oracle.kmeans_predict(x.tile.cpu().numpy().astype(np.float64), model.centroids)
    assert np.array_equal(lab, want), int(np.sum(lab != want))
    # (2) the whole trajectory is the reference's: same labels, same counts
    counts = np.bincount(lab, minlength=k)
    assert np.array_equal(counts, cfg_golden["cfg1_counts"]), (counts, cfg_golden["cfg1_counts"])
    assert label_digest(lab) == int(cfg_golden["cfg1_label_digest"][0])
    print(f"cfg1: centroids rel {rel_dev(model.centroids, golden['cfg1_centroids']):.2e}, counts {counts.tolist()}")


def test_cfg3_slice_matches_reference(comm, oracle, cfg_golden):
    """the 5M x 64, k=64 slice of config 3 (the 50M array needs
    ~100 GB of host f64 for the reference).  Runs the tcgen05 k-means kernel
    (k*d >= 1024) including its delta iterations."""
    n, m, k = 5_000_000, 64, 64
    x = dnd.random_uniform((n, m), 0, 42, comm)
    m1 = dnd.kmeans_fit(x, k, 1, 0.0, 42)
    assert rel_dev(m1.centroids, cfg_golden["cfg3s_centroids_it1"]) <= 1e-5
    model = dnd.kmeans_fit(x, k, 20, 0.0, 42)
    dev = rel_dev(model.centroids, cfg_golden["cfg3s_centroids_it20"])
    assert dev <= 1e-5, dev
    assert rel_dev(model.inertia_trace, cfg_golden["cfg3s_trace_it20"]) <= 1e-5
    lab = _labels(model, x)
    counts = np.bincount(lab, minlength=k)
    assert np.array_equal(counts, cfg_golden["cfg3s_counts"]), np.nonzero(counts - cfg_golden["cfg3s_counts"])
    assert label_digest(lab) == int(cfg_golden["cfg3s_label_digest"][0])
    # the predict kernel's decision equals the oracle's for the same centroids
    want = oracle.kmeans_predict(x.tile.cpu().numpy().astype(np.float64), model.centroids)
    assert np.array_equal(lab, want), int(np.sum(lab != want))
    print(f"cfg3 slice: centroids rel {dev:.2e}, refined rows {model.refined_rows}")


def test_cfg3_slice_delta_equals_full_accumulation(comm, monkeypatch):
    """The tcgen05 kernel's delta iterations (+x/-x of the rows whose label
    changed into running f64 sums) against summing every row every iteration."""
    n, m, k = 5_000_000, 64, 64
    x = dnd.random_uniform((n, m), 0, 42, comm)
    a = dnd.kmeans_fit(x, k, 20, 0.0, 42)
    monkeypatch.setenv("DNDC_TC_NO_DELTA", "1")
    xb = dnd.DndArray(x.shape, 0, comm, x.tile.clone())  # new buffers: a new fit graph
    b = dnd.kmeans_fit(xb, k, 20, 0.0, 42)
    assert rel_dev(a.centroids, b.centroids) <= 1e-12
    assert rel_dev(a.inertia_trace, b.inertia_trace) <= 1e-12
    assert np.array_equal(_labels(a, x), _labels(b, x))


def test_cfg4_panels_full_size(comm, oracle):
    """BASELINE config 4 on one GPU: X(100k x 1024, seed 42) vs Y(100k x 1024,
    seed 43) through the tcgen05 3xTF32 kernel, 40 GB of output; 64 sampled
    rows spread over X checked against the oracle at the 1e-5 gate."""
    n, m = 100_000, 1024
    if torch.cuda.mem_get_info()[0] < n * n * 4 + (4 << 30):
        pytest.skip("not enough HBM for the 40 GB output")
    x = dnd.random_uniform((n, m), 0, 42, comm)
    y = dnd.random_uniform((n, m), 0, 43, comm)
    d = dnd.cdist_xy(x, dnd.DndArray((n, m), None, comm, y.tile))
    rows = np.unique(np.concatenate([np.arange(0, n, n // 48), [1, 127, 128, 255, 256, 12345, n - 2, n - 1]]))
    ref = oracle.cdist_xy(x.tile[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64),
                          y.tile.cpu().numpy().astype(np.float64))
    got = d.tile[torch.from_numpy(rows).cuda()].cpu().numpy()
    dev = rel_dev(got, ref)
    print(f"cfg4 panels: {rows.size} rows x {n} columns, max rel dev {dev:.3e}")
    assert dev <= 1e-5
    assert float(d.tile.min()) >= 0.0
    del d
    torch.cuda.empty_cache()


def test_cfg5_moments_full_size(comm, oracle):
    """BASELINE config 5 moments: 100M x 32 fp32 (12.8 GB) at full size against
    the reference's single-rank sequential Welford chain (moments.cpp:100-114,
    the oracle fed the same rows block by block) at 1e-12."""
    n, m = 100_000_000, 32
    a = dnd.random_uniform((n, m), 0, 42, comm)
    st = dnd.moments_axis0(a)
    assert st.count == n
    step = 5_000_000
    cnt, mean, m2 = oracle.welford_stream((a.tile[i:i + step].cpu().numpy() for i in range(0, n, step)), m)
    assert cnt == n
    assert rel_dev(st.mean, mean) <= 1e-12, rel_dev(st.mean, mean)
    assert rel_dev(st.m2 / n, m2 / n) <= 1e-12, rel_dev(st.m2 / n, m2 / n)
    print(f"cfg5 moments: mean rel {rel_dev(st.mean, mean):.2e}, var rel {rel_dev(st.m2 / n, m2 / n):.2e}")


def test_cfg5_kmeanspp_full_size(comm, oracle):
    """BASELINE config 5 k-means++ seeding (k=8) on 100M x 32 against the
    oracle's restatement of the definition in DESIGN.md section 6."""
    n, m, k, seed = 100_000_000, 32, 8, 42
    if _host_ram_gb() < 24:
        pytest.skip("needs ~13 GB of host RAM for the fp32 copy")
    a = dnd.random_uniform((n, m), 0, 42, comm)
    got = dnd.kmeanspp_indices(a, k, seed)
    xh = a.tile.cpu().numpy()
    want = oracle.kmeanspp_indices(xh, k, seed)
    assert np.array_equal(got, want), (got, want)


def test_cfg1_fit_is_bitwise_repeatable(comm):
    """the fit must not depend on run-to-run scheduling.  The
    persistent kernel hands out part of its tiles dynamically, so its sums are
    integer fixed point (order-independent); two fits at cfg1 size, and one on
    data with tiny magnitudes (bits far below the fixed-point step), must agree
    to the last bit."""
    n, m, k = 5_000_000, 18, 8
    x = dnd.random_uniform((n, m), 0, 42, comm)
    a = dnd.kmeans_fit(x, k, 20, 0.0, 42)
    b = dnd.kmeans_fit(x, k, 20, 0.0, 42)
    assert np.array_equal(a.centroids, b.centroids) and a.inertia_trace == b.inertia_trace
    xs = dnd.DndArray(x.shape, 0, comm, x.tile * 1e-6)
    c = dnd.kmeans_fit(xs, k, 10, 0.0, 42)
    d = dnd.kmeans_fit(xs, k, 10, 0.0, 42)
    assert np.array_equal(c.centroids, d.centroids) and c.inertia_trace == d.inertia_trace
