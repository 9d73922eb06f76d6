"""B200-native (sm_100a) memory-layer hot path of "Memory Layers at Scale"
(arXiv 2412.09764): product-key top-k and the EmbeddingBag forward/backward,
exposed as the C-ABI library libmemlayer.so (include/memlayer.h) with this
thin torch binding.  The CUDA extension is mandatory: importing `ops`
without the built library raises.
"""
from ._lib import LIB_PATH, MemlayerError, lib  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # lazy import of the torch binding so `import paper_2412_09764_b200`
    # works (e.g. for build()) before torch / the library is needed
    if name in ("ops", "group", "graph"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
