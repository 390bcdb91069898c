"""Python mirror of the reference's C++ API for the hot path.

Names, argument meaning and error behaviour follow proj/include/dnd/*.hpp so
the parity tests read like the reference's own tests (tests/test_pairwise.cpp,
test_cluster.cpp, test_moments.cpp).  Every compute call goes through the
C-ABI of include/dndc.h (libdndc.so, CUDA kernels for sm_100a + NCCL); shards
live in HBM as torch CUDA tensors, which are used only as device memory.

  reference                                   here
  ------------------------------------------  -----------------------------------
  Communicator / run_world (transport.hpp)    Communicator (one per GPU / rank)
  chunk_map (chunking.hpp:27)                 chunk_map
  DndArray<T> (ndarray.hpp:58-91)             DndArray (any split, resplit)
  random_uniform / from_global / gather       random_uniform / from_global / gather
  detail::row_norms / distance_block          row_norms / distance_block
  cdist / cdist_xy (pairwise.hpp:15-19)       cdist / cdist_xy
  kmeans_* (cluster.hpp:25-42)                kmeans_init_indices / _centroids / fit / predict
  mean_axis / var_axis / stddev_axis          same names (axis 0 = the split axis)
  resplit (ndarray.hpp:340-386)               resplit (dndc_resplit, NCCL send/recv)
  lasso_fit / lasso_predict (regression.hpp)  same names (dndc_lasso_*_f64)
  dnb_read_header / dnb_save / dnb_load       same names (payload file <-> HBM, dndc_file_*)
  (not in the reference)                      kmeanspp_indices (BASELINE config 5)
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import DataError, TransportError, check, lib

__all__ = [
    "Communicator", "DndArray", "KMeansModel", "MomentState", "TransportError", "chunk_map",
    "random_uniform", "from_global", "gather", "resplit", "row_norms", "distance_block", "cdist", "cdist_xy",
    "kmeans_init_indices", "kmeans_init_centroids", "kmeans_fit", "kmeans_predict", "mean_axis",
    "var_axis", "stddev_axis", "moments_axis0", "kmeanspp_indices", "LassoModel", "soft_threshold",
    "lasso_fit", "lasso_predict", "DataError", "dnb_read_header", "dnb_save", "dnb_load",
]

_SUFFIX = {torch.float32: "f32", torch.float64: "f64"}


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class Communicator:
    """Rank handle over one GPU (dnd::Communicator, transport.hpp:85-217).

    world == 1 needs nothing; world > 1 shares an NCCL unique id, normally via
    `Communicator.from_torch_distributed()` (one process per GPU, torchrun).
    """

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None):
        self.device = int(device)
        self._rank, self._world = int(rank), int(world)
        h = C.c_void_p()
        uid = None
        if unique_id is not None:
            uid = C.create_string_buffer(bytes(unique_id), _lib.UNIQUE_ID_BYTES)
        torch.cuda.set_device(self.device)
        check(lib().dndc_create(self.device, self._rank, self._world, uid, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(_lib.UNIQUE_ID_BYTES)
        check(lib().dndc_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, device: int | None = None) -> "Communicator":
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            device = torch.cuda.current_device()
        obj = [cls.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return cls(device, rank, world, obj[0] if world > 1 else None)

    # -- handle plumbing
    @property
    def handle(self):
        lib().dndc_set_stream(self._h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        return self._h

    def rank(self) -> int:
        return self._rank

    def size(self) -> int:
        return self._world

    def counters(self) -> dict:
        c = _lib.Counters()
        check(lib().dndc_get_counters(self._h, C.byref(c)))
        return {n: getattr(c, n) for n, _ in c._fields_}

    @property
    def transport(self) -> str:
        """How the k-means stats exchange travels (NVLink peer stores or NCCL)."""
        return lib().dndc_transport_status(self._h).decode()

    @property
    def launches(self) -> int:
        return int(lib().dndc_launch_count(self._h))

    def synchronize(self) -> None:
        check(lib().dndc_synchronize(self.handle))

    def barrier(self) -> None:
        """Communicator::barrier (transport.hpp:86-88)."""
        check(lib().dndc_barrier(self.handle))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().dndc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def chunk_map(n: int, p: int) -> tuple[np.ndarray, np.ndarray]:
    """Balanced split of n rows over p ranks (chunking.cpp:9-30)."""
    off = np.empty(max(p, 1), np.int64)
    ext = np.empty(max(p, 1), np.int64)
    check(lib().dndc_chunk_map(int(n), int(p), off.ctypes.data, ext.ctypes.data))
    return off, ext


@dataclass
class DndArray:
    """An N-D array split along one axis (or replicated, split=None); the
    hot-path ops take row shards and resplit other layouts first."""

    shape: tuple
    split: int | None
    comm: Communicator
    tile: torch.Tensor  # this rank's rows, contiguous, on the rank's GPU

    def ndim(self) -> int:
        return len(self.shape)

    def lshape(self) -> tuple:
        return tuple(self.tile.shape)

    def split_chunks(self):
        if self.split is None:
            raise ValueError("split_chunks: array is not split")
        return chunk_map(self.shape[self.split], self.comm.size())

    def row_offset(self) -> int:
        return int(self.split_chunks()[0][self.comm.rank()]) if self.split == 0 else 0


def _check_split(shape, split):
    if any(e < 0 for e in shape):
        raise ValueError(f"negative extent in shape {tuple(shape)}")
    if split is not None and not 0 <= split < len(shape):
        raise ValueError(f"split axis {split} out of range for shape {tuple(shape)}")


def _local_shape(shape, split, comm):
    if split is None:
        return tuple(shape)
    off, ext = chunk_map(shape[split], comm.size())
    return tuple(int(ext[comm.rank()]) if d == split else e for d, e in enumerate(shape))


def resplit(a: DndArray, new_split) -> DndArray:
    """dnd::resplit (ndarray.hpp:340-386): same global content on another
    split axis or replicated, moved between the HBM shards by dndc_resplit
    (one grouped NCCL exchange of the intersection blocks)."""
    _check_split(a.shape, new_split)
    if a.split == new_split:
        return a
    tile = torch.empty(_local_shape(a.shape, new_split, a.comm), dtype=a.tile.dtype, device=a.tile.device)
    if int(np.prod(a.shape)) > 0:
        shp = np.asarray(a.shape, np.int64)
        src = a.tile.contiguous()
        check(lib().dndc_resplit(a.comm.handle, _ptr(src), len(a.shape), shp.ctypes.data, src.element_size(),
                                 -1 if a.split is None else int(a.split), -1 if new_split is None else int(new_split),
                                 _ptr(tile)))
    return DndArray(a.shape, new_split, a.comm, tile)


def _rows(x: DndArray) -> DndArray:
    """x as row shards or replicated (pairwise.cpp:41, cluster.cpp:91)."""
    return resplit(x, 0) if x.split not in (None, 0) else x


def random_uniform(shape, split, seed: int, comm: Communicator, dtype=torch.float32) -> DndArray:
    """dnd::random_uniform<T> (ndarray.hpp:154-169), generated on the GPU."""
    shape = tuple(int(s) for s in shape)
    _check_split(shape, split)
    if split not in (None, 0):  # generated as row shards, then moved
        return resplit(random_uniform(shape, 0, seed, comm, dtype), split)
    n = shape[0]
    m = int(np.prod(shape[1:])) if len(shape) > 1 else 1
    if split is None:
        row0, rows = 0, n
    else:
        off, ext = chunk_map(n, comm.size())
        row0, rows = int(off[comm.rank()]), int(ext[comm.rank()])
    tile = torch.empty((rows,) + shape[1:], dtype=dtype, device=f"cuda:{comm.device}")
    fn = getattr(lib(), f"dndc_fill_uniform_{_SUFFIX[dtype]}")
    check(fn(comm.handle, int(seed) & 0xFFFFFFFFFFFFFFFF, row0, rows, m, _ptr(tile)))
    return DndArray(shape, split, comm, tile)


def from_global(data, shape, split, comm: Communicator, dtype=None) -> DndArray:
    """dnd::from_global (ndarray.hpp:173-188): every rank passes the same data."""
    shape = tuple(int(s) for s in shape)
    _check_split(shape, split)
    arr = np.asarray(data)
    if dtype is None:
        dtype = torch.float64 if arr.dtype == np.float64 else torch.float32
    if arr.size != int(np.prod(shape)):
        raise ValueError(f"from_global: data holds {arr.size} elements, shape {shape} needs "
                         f"{int(np.prod(shape))}")
    arr = arr.reshape(shape)
    if split is not None:
        off, ext = chunk_map(shape[split], comm.size())
        sl = [slice(None)] * len(shape)
        sl[split] = slice(int(off[comm.rank()]), int(off[comm.rank()] + ext[comm.rank()]))
        arr = arr[tuple(sl)]
    np_dtype = np.float64 if dtype == torch.float64 else (np.int32 if dtype == torch.int32 else np.float32)
    tile = torch.from_numpy(np.ascontiguousarray(arr, dtype=np_dtype)).to(f"cuda:{comm.device}")
    return DndArray(shape, split, comm, tile)


def gather(a: DndArray) -> np.ndarray:
    """Full global content on every rank (dnd::gather, ndarray.hpp:389-393)."""
    if a.split not in (None, 0):
        a = resplit(a, None)
    local = a.tile.detach().cpu().numpy()
    if a.split is None or a.comm.size() == 1:
        return local.reshape(a.shape)
    import torch.distributed as dist

    parts = [None] * a.comm.size()
    dist.all_gather_object(parts, local)
    return np.concatenate(parts, axis=0).reshape(a.shape)


def _fn(name: str, t: torch.Tensor):
    if t.dtype not in _SUFFIX:
        raise ValueError(f"{name[5:]}: float32 or float64 input required, got {t.dtype}")
    return getattr(lib(), f"{name}_{_SUFFIX[t.dtype]}")


def row_norms(tile: torch.Tensor) -> torch.Tensor:
    """detail::row_norms (pairwise.cpp:10-20)."""
    tile = tile.contiguous()
    comm_dev = tile.device.index
    out = torch.empty(tile.shape[0], dtype=tile.dtype, device=tile.device)
    ctx = _device_ctx(comm_dev)
    check(_fn("dndc_row_norms", tile)(ctx.handle, _ptr(tile), tile.shape[0], tile.shape[1], _ptr(out)))
    return out


def distance_block(a: torch.Tensor, na: torch.Tensor, b: torch.Tensor, nb: torch.Tensor) -> torch.Tensor:
    """detail::distance_block (pairwise.cpp:22-33)."""
    out = torch.empty((a.shape[0], b.shape[0]), dtype=a.dtype, device=a.device)
    ctx = _device_ctx(a.device.index)
    check(_fn("dndc_cdist_tile", a)(ctx.handle, _ptr(a), _ptr(na), a.shape[0], _ptr(b), _ptr(nb), b.shape[0],
                                    a.shape[1], _ptr(out), b.shape[0], 0, -1))
    return out


_DEVICE_CTX: dict[int, Communicator] = {}


def _device_ctx(device: int) -> Communicator:
    """A world-1 handle per device for communication-free helpers."""
    if device not in _DEVICE_CTX:
        _DEVICE_CTX[device] = Communicator(device)
    return _DEVICE_CTX[device]


def _require_2d(x: DndArray, who: str):
    if x.ndim() != 2:
        raise ValueError(f"{who}: input must be 2-D")


def cdist(x: DndArray) -> DndArray:
    """Ring self-distance (pairwise.cpp:37-85): world-1 exchanges per rank."""
    _require_2d(x, "cdist")
    if x.shape[0] == 0:
        raise ValueError("cdist: input has no rows")
    if x.split != 0:
        x = resplit(x, 0)  # pairwise.cpp:41
    n, m = x.shape
    out = torch.empty((x.tile.shape[0], n), dtype=x.tile.dtype, device=x.tile.device)
    check(_fn("dndc_cdist", x.tile)(x.comm.handle, _ptr(x.tile), x.tile.shape[0], n, m, _ptr(out)))
    return DndArray((n, n), 0, x.comm, out)


def cdist_xy(x: DndArray, y: DndArray) -> DndArray:
    """cdist_xy (pairwise.cpp:87-100).  y replicated: communication-free;
    y split=0: its shards travel the ring (BASELINE config 2)."""
    if x.ndim() != 2 or y.ndim() != 2:
        raise ValueError("cdist_xy: inputs must be 2-D")
    if x.shape[1] != y.shape[1]:
        raise ValueError(f"cdist_xy: feature counts {x.shape[1]} and {y.shape[1]} do not match")
    x = _rows(x)  # pairwise.cpp:93-94
    if y.split not in (None, 0):
        y = resplit(y, None)
    m = x.shape[1]
    nx_local = x.tile.shape[0] if x.split == 0 else x.shape[0]
    out = torch.empty((nx_local, y.shape[0]), dtype=x.tile.dtype, device=x.tile.device)
    if y.split is None:
        check(_fn("dndc_cdist_xy", x.tile)(x.comm.handle, _ptr(x.tile), nx_local, _ptr(y.tile), y.shape[0], m,
                                           _ptr(out)))
    else:
        check(_fn("dndc_cdist_xy_ring", x.tile)(x.comm.handle, _ptr(x.tile), nx_local, _ptr(y.tile),
                                                y.tile.shape[0], y.shape[0], m, _ptr(out)))
    return DndArray((x.shape[0], y.shape[0]), x.split, x.comm, out)


@dataclass
class KMeansModel:
    """cluster.hpp:14-21."""

    k: int = 0
    n_features: int = 0
    centroids: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    inertia_trace: list = field(default_factory=list)
    iterations_run: int = 0
    seed: int = 0
    refined_rows: int = 0  # rows re-decided in f64 during the last iteration set


def kmeans_init_indices(n: int, k: int, seed: int) -> np.ndarray:
    """cluster.cpp:60-75."""
    out = np.empty(max(k, 1), np.int64)
    check(lib().dndc_kmeans_init_indices(int(n), int(k), int(seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out[:k]


def _shard(x: DndArray):
    """(handle owner, local rows, global rows).  A replicated input is
    processed whole by every rank on a world-1 handle (the reference
    resplits it first, cluster.cpp:91; results are identical)."""
    n_local = x.tile.shape[0]
    if x.split == 0:
        return x.comm, n_local, x.shape[0]
    return (_device_ctx(x.comm.device) if x.comm.size() > 1 else x.comm), n_local, n_local


def kmeans_init_centroids(x: DndArray, k: int, seed: int) -> np.ndarray:
    """cluster.cpp:77-81 (rows replicated to every rank, f64)."""
    _require_2d(x, "kmeans_init_centroids")
    x = _rows(x)
    comm, n_local, n_global = _shard(x)
    m = x.shape[1]
    out = np.empty((max(k, 1), m), np.float64)
    if x.tile.dtype != torch.float32:
        idx = kmeans_init_indices(n_global, k, seed)
        full = gather(x)
        return full[idx].astype(np.float64)
    check(lib().dndc_kmeans_init_centroids_f32(comm.handle, _ptr(x.tile), n_local, n_global, m, int(k),
                                               int(seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out[:k]


def kmeans_fit(x: DndArray, k: int, max_iter: int, tol: float, seed: int, init=None) -> KMeansModel:
    """Lloyd's algorithm (cluster.cpp:83-153) on the fused GPU kernels."""
    _require_2d(x, "kmeans_fit")
    x = _rows(x)
    comm, n_local, n_global = _shard(x)
    m = x.shape[1]
    if k < 1:
        raise ValueError(f"kmeans_fit: k must be positive, got {k}")
    if k > n_global:
        raise ValueError(f"kmeans_fit: k={k} exceeds the {n_global} available samples")
    if max_iter < 1:
        raise ValueError(f"kmeans_fit: max_iter must be positive, got {max_iter}")
    cent = np.empty((k, m), np.float64)
    trace = np.zeros(max_iter, np.float64)
    iters = C.c_int(0)
    init_ptr = None
    if init is not None:
        init = np.ascontiguousarray(init, np.float64).reshape(k, m)
        init_ptr = init.ctypes.data
    check(_fn("dndc_kmeans_fit", x.tile)(comm.handle, _ptr(x.tile), n_local, n_global, m, int(k), int(max_iter),
                                         float(tol), int(seed) & 0xFFFFFFFFFFFFFFFF, init_ptr, cent.ctypes.data,
                                         trace.ctypes.data, C.byref(iters)))
    refined = C.c_int64(0)
    lib().dndc_kmeans_last_refined(comm._h, C.byref(refined))
    return KMeansModel(k, m, cent, list(trace[: iters.value]), iters.value, seed, refined.value)


def kmeans_predict(model: KMeansModel, x: DndArray) -> DndArray:
    """cluster.cpp:155-172 (ties to the lowest centroid index)."""
    _require_2d(x, "kmeans_predict")
    if x.split not in (None, 0):
        raise ValueError("kmeans_predict: input must be split=0 or replicated")  # cluster.cpp:160-161
    if x.shape[1] != model.n_features:
        raise ValueError(f"kmeans_predict: input has {x.shape[1]} features, model expects {model.n_features}")
    n_local = x.tile.shape[0]
    labels = torch.empty(n_local, dtype=torch.int32, device=x.tile.device)
    c = np.ascontiguousarray(model.centroids, np.float64)
    check(_fn("dndc_kmeans_predict", x.tile)(x.comm.handle, _ptr(x.tile), n_local, x.shape[1], c.ctypes.data,
                                             int(model.k), _ptr(labels)))
    return DndArray((x.shape[0],), x.split, x.comm, labels)


@dataclass
class MomentState:
    """moments.hpp:14-24 (count, per-slot mean and M2)."""

    count: int
    mean: np.ndarray
    m2: np.ndarray


def moments_axis0(a: DndArray) -> MomentState:
    """local_moments_axis + rank-order combine (moments.cpp:41-52)."""
    _require_2d(a, "moments")
    a = _rows(a)
    m = a.shape[1]
    cnt = np.zeros(1, np.int64)
    mean = np.zeros(max(m, 1), np.float64)
    m2 = np.zeros(max(m, 1), np.float64)
    fn_ctx = _shard(a)[0]
    check(_fn("dndc_moments_axis0", a.tile)(fn_ctx.handle, _ptr(a.tile), a.tile.shape[0], m, cnt.ctypes.data,
                                            mean.ctypes.data, m2.ctypes.data))
    return MomentState(int(cnt[0]), mean[:m].copy(), m2[:m].copy())


def _variance_from(s: MomentState, ddof: int, who: str) -> np.ndarray:
    if s.count - ddof <= 0:
        raise ValueError(f"{who}: need more than ddof={ddof} samples, got {s.count}")
    return s.m2 / float(s.count - ddof)


def _replicated(values: np.ndarray, comm: Communicator) -> DndArray:
    return DndArray((values.shape[0],), None, comm, torch.from_numpy(values).to(f"cuda:{comm.device}"))


def mean_axis(a: DndArray, axis: int = 0) -> DndArray:
    if axis != 0:
        raise ValueError("mean_axis: the B200 path reduces along the split axis 0")
    return _replicated(moments_axis0(a).mean, a.comm)


def var_axis(a: DndArray, axis: int = 0, ddof: int = 0) -> DndArray:
    if axis != 0:
        raise ValueError("var_axis: the B200 path reduces along the split axis 0")
    return _replicated(_variance_from(moments_axis0(a), ddof, "var_axis"), a.comm)


def stddev_axis(a: DndArray, axis: int = 0, ddof: int = 0) -> DndArray:
    if axis != 0:
        raise ValueError("stddev_axis: the B200 path reduces along the split axis 0")
    return _replicated(np.sqrt(_variance_from(moments_axis0(a), ddof, "stddev_axis")), a.comm)


def kmeanspp_indices(x: DndArray, k: int, seed: int) -> np.ndarray:
    """k-means++ seeding (BASELINE config 5; definition in DESIGN.md)."""
    _require_2d(x, "kmeanspp")
    x = _rows(x)
    comm, n_local, n_global = _shard(x)
    out = np.empty(max(k, 1), np.int64)
    check(_fn("dndc_kmeanspp_indices", x.tile)(comm.handle, _ptr(x.tile), n_local, n_global, x.shape[1], int(k),
                                               int(seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data))
    return out[:k]


del math


@dataclass
class LassoModel:
    """regression.hpp:10-19 (weights[0] is the unpenalised bias)."""

    weights: np.ndarray = field(default_factory=lambda: np.zeros(0))
    lambda_: float = 0.0
    objective_trace: list = field(default_factory=list)
    sweeps_run: int = 0


def soft_threshold(rho: float, threshold: float) -> float:
    """regression.cpp:19-23."""
    if rho > threshold:
        return rho - threshold
    if rho < -threshold:
        return rho + threshold
    return 0.0


def lasso_fit(x: DndArray, y: DndArray, lam: float, sweeps: int, tol: float = 0.0) -> LassoModel:
    """Cyclic coordinate descent (regression.cpp:25-102): one GPU kernel per
    coordinate, the cross-GPU sum over NVLink inside it (dndc_lasso_fit_f64)."""
    if x.ndim() != 2:
        raise ValueError("lasso_fit: design matrix must be 2-D")
    if y.ndim() != 1:
        raise ValueError("lasso_fit: targets must be 1-D")
    if x.shape[0] != y.shape[0]:
        raise ValueError(f"lasso_fit: {x.shape[0]} rows vs {y.shape[0]} targets")
    if x.tile.dtype != torch.float64 or y.tile.dtype != torch.float64:
        raise ValueError("lasso_fit: float64 arrays (the reference's DndArray<double>)")
    if x.split != 0:
        x = resplit(x, 0)
    if y.split != 0:
        y = resplit(y, 0)
    m = x.shape[1]
    w = np.zeros(max(m, 1), np.float64)
    trace = np.zeros(max(int(sweeps), 1), np.float64)
    run = C.c_int(0)
    check(lib().dndc_lasso_fit_f64(x.comm.handle, _ptr(x.tile), x.tile.shape[0], x.shape[0], m, _ptr(y.tile),
                                   float(lam), int(sweeps), float(tol), w.ctypes.data, trace.ctypes.data,
                                   C.byref(run)))
    return LassoModel(w[:m].copy(), float(lam), list(trace[: run.value]), run.value)


def lasso_predict(model: LassoModel, x: DndArray) -> DndArray:
    """Xw per local row (regression.cpp:105-127), bit-identical to the reference."""
    if x.ndim() != 2:
        raise ValueError("lasso_predict: input must be 2-D")
    if x.shape[1] != len(model.weights):
        raise ValueError(f"lasso_predict: input has {x.shape[1]} columns, model expects {len(model.weights)}")
    if x.split not in (None, 0):
        raise ValueError("lasso_predict: input must be split=0 or replicated")
    w = np.ascontiguousarray(model.weights, np.float64)
    out = torch.empty(x.tile.shape[0], dtype=torch.float64, device=x.tile.device)
    check(lib().dndc_lasso_predict_f64(x.comm.handle, _ptr(x.tile), x.tile.shape[0], x.shape[1], w.ctypes.data,
                                       _ptr(out)))
    return DndArray((x.shape[0],), x.split, x.comm, out)


_DNB_DTYPES = {1: (torch.float32, 4), 2: (torch.float64, 8)}


def dnb_read_header(path: str):
    """dataio.cpp:57-88: (dtype, extents, header_bytes); DataError on a missing
    file, bad magic, unknown dtype_code, ndim 0 or truncated extents."""
    import os

    if not os.path.exists(path):
        raise DataError(f"dnb_read_header: cannot open {path}")
    with open(path, "rb") as f:
        fixed = f.read(6)
        if len(fixed) != 6:
            raise DataError(f"dnb_read_header: {path} is shorter than the fixed header")
        if fixed[:4] != b"DNB1":
            raise DataError(f'dnb_read_header: bad magic in {path}, expected "DNB1"')
        if fixed[4] not in _DNB_DTYPES:
            raise DataError(f"dnb_read_header: unknown dtype_code {fixed[4]} in {path}")
        if fixed[5] == 0:
            raise DataError(f"dnb_read_header: ndim must be at least 1 in {path}")
        raw = f.read(8 * fixed[5])
        if len(raw) != 8 * fixed[5]:
            raise DataError(f"dnb_read_header: truncated extents in {path}")
    ext = tuple(int(e) for e in np.frombuffer(raw, "<u8"))
    return _DNB_DTYPES[fixed[4]][0], ext, 6 + 8 * len(ext)


def dnb_save(a: DndArray, path: str) -> None:
    """Collective save (dataio.hpp:61-100): rank 0 writes the header (and a
    replicated payload); split=0 ranks write their rows from HBM at their offset."""
    if a.split not in (None, 0):
        a = resplit(a, 0)
    code = {torch.float32: 1, torch.float64: 2}.get(a.tile.dtype)
    if code is None:
        raise ValueError("dnb_save: float32 or float64 arrays")
    head = b"DNB1" + bytes([code, len(a.shape)]) + np.asarray(a.shape, "<u8").tobytes()
    esz = a.tile.element_size()
    if a.comm.rank() == 0:
        with open(path, "wb") as f:
            f.write(head)
        if a.split is None and a.tile.numel():
            check(lib().dndc_file_write_from_device(a.comm.handle, path.encode(), len(head), _ptr(a.tile),
                                                    a.tile.numel() * esz))
    a.comm.barrier()
    if a.split == 0 and a.tile.numel():
        row = a.tile.numel() // a.tile.shape[0]
        check(lib().dndc_file_write_from_device(a.comm.handle, path.encode(), len(head) + a.row_offset() * row * esz,
                                                _ptr(a.tile), a.tile.numel() * esz))
    a.comm.barrier()


def dnb_load(path: str, split, comm: Communicator) -> DndArray:
    """Collective load (dataio.hpp:102-142): split=0 ranks read only their byte
    range, straight into HBM; other splits load as split=0 and resplit."""
    import os

    dtype, shape, hb = dnb_read_header(path)
    esz = _DNB_DTYPES[{torch.float32: 1, torch.float64: 2}[dtype]][1]
    want = hb + int(np.prod(shape)) * esz
    have = os.path.getsize(path)
    if have != want:
        raise DataError(f"dnb_load: truncated payload in {path}: expected {want} bytes, file has {have}")
    _check_split(shape, split)
    if split not in (None, 0):
        return resplit(dnb_load(path, 0, comm), split)
    tile = torch.empty(_local_shape(shape, split, comm), dtype=dtype, device=f"cuda:{comm.device}")
    if tile.numel():
        row = tile.numel() // tile.shape[0]
        off = hb + (int(chunk_map(shape[0], comm.size())[0][comm.rank()]) * row * esz if split == 0 else 0)
        check(lib().dndc_file_read_to_device(comm.handle, path.encode(), off, tile.numel() * esz, _ptr(tile)))
    return DndArray(shape, split, comm, tile)

