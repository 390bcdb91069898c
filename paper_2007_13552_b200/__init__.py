"""B200-native hot path of HeAT (arXiv 2007.13552): distributed cdist,
k-means Lloyd iterations and split-axis moments on row-split arrays.

The compute lives in libdndc.so (CUDA for sm_100a + NCCL), behind the C ABI
of include/dndc.h; `api` mirrors the reference's C++ API (proj/include/dnd).
"""
from ._lib import LIB_PATH, TransportError, header_symbols  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # the compute API loads libdndc.so on first use and raises if it is absent
    import importlib

    api = importlib.import_module(__name__ + ".api")
    return api if name == "api" else getattr(api, name)
