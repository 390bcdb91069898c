"""World-size-2 checks of the N>1 host logic on CPU (gloo over 127.0.0.1).

The GPU path exchanges data with NCCL (csrc/runtime.cu, csrc/cdist.cu); what
these tests pin on CPU is the distributed *decomposition* that path implements,
run with real processes and a real collective backend:

* the NCCL unique-id handshake of Communicator.from_torch_distributed;
* gather(): rank-order concatenation of the row shards (ndarray.hpp:389-393);
* the cdist ring schedule of cdist_ring (pairwise.cpp:54-83): round t computes
  against the block that originated at (rank - t) mod p, fills that origin's
  column window, and forwards the block to rank + 1 -- assembled with gloo
  send/recv and checked bit-for-bit against the oracle's cdist;
* the k-means stats exchange (cluster.cpp:105-133): per-rank sums/counts,
  allgather, fold in rank order 0..p-1 from the zero identity, update --
  checked bit-for-bit against the oracle's p = 2 simulation.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn_name, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        globals()[fn_name](rank, world)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # surfaced by the parent
        import traceback

        q.put((rank, traceback.format_exc()))


def _spawn(fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, fn_name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(WORLD):
        assert res.get(r) == "ok", f"rank {r}:\n{res.get(r)}"


# --------------------------------------------------------------- rank bodies
def _body_unique_id(rank, world):
    from paper_2007_13552_b200.api import Communicator

    obj = [Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    assert isinstance(uid, bytes) and len(uid) == 128
    everyone = [None] * world
    dist.all_gather_object(everyone, uid)
    assert all(u == everyone[0] for u in everyone)


class _StubComm:
    def __init__(self, world):
        self._w = world

    def size(self):
        return self._w


def _body_gather(rank, world):
    from oracle.bind import Oracle
    from paper_2007_13552_b200 import api

    n, m = 11, 3
    off, ext = api.chunk_map(n, world)
    o_off, o_ext = Oracle().chunk_map(n, world)
    assert list(off) == list(o_off) and list(ext) == list(o_ext)
    full = np.arange(n * m, dtype=np.float64).reshape(n, m)
    tile = torch.from_numpy(full[off[rank]: off[rank] + ext[rank]].copy())
    a = api.DndArray((n, m), 0, _StubComm(world), tile)
    assert np.array_equal(api.gather(a), full)


def _body_ring(rank, world):
    from oracle.bind import Oracle

    O = Oracle()
    n, m = 37, 5
    x = O.uniform_f32(n, m, 7).astype(np.float64)
    off, ext = O.chunk_map(n, world)
    mine = x[off[rank]: off[rank] + ext[rank]]
    out = np.full((ext[rank], n), np.nan)
    block, origin = mine.copy(), rank
    for t in range(world):
        # compute against the block in hand, into its origin's column window
        out[:, off[origin]: off[origin] + ext[origin]] = O.cdist_xy(mine, block)
        if t + 1 < world:
            src_origin = (origin - 1) % world
            recv = np.empty((ext[src_origin], m), np.float64)
            send_t = torch.from_numpy(np.ascontiguousarray(block))
            recv_t = torch.from_numpy(recv)
            reqs = [dist.isend(send_t, (rank + 1) % world), dist.irecv(recv_t, (rank - 1) % world)]
            for r in reqs:
                r.wait()
            block, origin = recv_t.numpy().copy(), src_origin
    ref = O.cdist(x, p=world)[off[rank]: off[rank] + ext[rank]]
    assert np.array_equal(out, ref)


def _seq_dot(a, b):
    """Sequential f64 dot products along the feature axis, one rounding per op
    (pairwise.cpp:22-33 order, no FMA)."""
    g = np.zeros(a.shape[0] if a.ndim == 2 else 1)
    for f in range(a.shape[-1]):
        g = g + a[..., f] * b[..., f]
    return g


def _body_kmeans_fold(rank, world):
    from oracle.bind import Oracle

    O = Oracle()
    n, m, k, iters = 240, 4, 5, 6
    x = O.uniform_f32(n, m, 11).astype(np.float64)
    init = x[O.kmeans_init_indices(n, k, 3)].copy()
    off, ext = O.chunk_map(n, world)
    mine = x[off[rank]: off[rank] + ext[rank]]
    c = init.copy()
    xn = _seq_dot(mine, mine)
    for _ in range(iters):
        # assign_local: nearest centroid, strict < keeps the lowest index
        cn = np.array([_seq_dot(c[j][None, :], c[j][None, :])[0] for j in range(k)])
        d = np.stack([np.sqrt(np.maximum((xn + cn[j]) - 2.0 * _seq_dot(mine, np.broadcast_to(c[j], mine.shape)),
                                         0.0)) for j in range(k)], axis=1)
        lab = np.argmin(d, axis=1)
        stats = np.zeros(k * m + k)
        for i in range(mine.shape[0]):  # row order, as the reference's loop
            j = lab[i]
            stats[j * m: (j + 1) * m] = stats[j * m: (j + 1) * m] + mine[i]
            stats[k * m + j] += 1.0
        parts = [torch.zeros(k * m + k, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(stats))
        tot = np.zeros(k * m + k)
        for r in range(world):  # allreduce(plus_vec): rank order from the identity
            tot = tot + parts[r].numpy()
        for j in range(k):
            if tot[k * m + j] > 0:
                c[j] = tot[j * m: (j + 1) * m] / tot[k * m + j]
    ref, _, _ = O.kmeans_lloyd(x, init, iters, 0.0, p=world)
    assert np.max(np.abs(c - ref)) <= 1e-15 * np.max(np.abs(ref)), np.max(np.abs(c - ref))


# -------------------------------------------------------------------- tests
@pytest.mark.timeout(300)
def test_unique_id_handshake():
    _spawn("_body_unique_id")


@pytest.mark.timeout(300)
def test_gather_rank_order():
    _spawn("_body_gather")


@pytest.mark.timeout(300)
def test_cdist_ring_schedule():
    _spawn("_body_ring")


@pytest.mark.timeout(300)
def test_kmeans_stats_exchange_and_fold():
    _spawn("_body_kmeans_fold")
