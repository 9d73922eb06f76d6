"""ctypes declarations of libmemlayer (include/memlayer.h).

Loading fails loudly: there is no fallback path.  The library is built
in-tree by `python -m paper_2412_09764_b200._build` (or
`__graft_entry__.build()`).
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmemlayer.so")

ML_OK, ML_ERR_ARG, ML_ERR_CONFIG, ML_ERR_INDEX, ML_ERR_WORKSPACE, ML_ERR_CUDA = 0, 1, 2, 3, 4, 5
ML_ERR_NCCL, ML_ERR_UNSUPPORTED = 6, 7
ML_F32, ML_BF16 = 0, 1
STATUS_NAMES = {0: "ML_OK", 1: "ML_ERR_ARG", 2: "ML_ERR_CONFIG", 3: "ML_ERR_INDEX",
                4: "ML_ERR_WORKSPACE", 5: "ML_ERR_CUDA", 6: "ML_ERR_NCCL", 7: "ML_ERR_UNSUPPORTED"}


class PkmShape(C.Structure):
    _fields_ = [("T", C.c_int32), ("H", C.c_int32), ("S", C.c_int32), ("Dk", C.c_int32),
                ("k", C.c_int32), ("dtype", C.c_int), ("qk_norm", C.c_int32)]


class BagShape(C.Structure):
    _fields_ = [("N", C.c_int64), ("dv", C.c_int32), ("T", C.c_int32), ("B", C.c_int32),
                ("dtype", C.c_int), ("grad_dtype", C.c_int)]


class LayerShape(C.Structure):
    _fields_ = [("pkm", PkmShape), ("N", C.c_int64), ("dv", C.c_int32), ("D", C.c_int32),
                ("gated", C.c_int32), ("grad_dtype", C.c_int)]


class PeerShape(C.Structure):
    _fields_ = [("pkm", PkmShape), ("N", C.c_int64), ("D", C.c_int32)]


class AdamParams(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float)]


class MemlayerError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


P = C.c_void_p
SZ = C.c_size_t
I64 = C.c_int64

# name -> argtypes (restype is c_int status unless listed in _RESTYPES)
SIGNATURES = {
    "ml_last_error": [],
    "ml_version": [],
    "ml_launch_count": [],
    "ml_device_info": [C.POINTER(C.c_int)] * 3,
    "ml_timing_enable": [C.c_int],
    "ml_set_serial": [C.c_int],
    "ml_timing_reset": [],
    "ml_timing_report": [C.c_char_p, SZ],
    "ml_synth_fill": [P, I64, I64, I64, C.c_uint64, C.c_uint32, C.c_float, C.c_int, C.c_int, I64, P],
    "pkm_topk_workspace": [C.POINTER(PkmShape), C.POINTER(SZ)],
    "pkm_topk": [C.POINTER(PkmShape), P, P, P, P, P, P, P, SZ, P],
    "pkm_topk_bwd_workspace": [C.POINTER(PkmShape), C.POINTER(SZ)],
    "pkm_topk_bwd": [C.POINTER(PkmShape), P, P, P, P, P, P, P, P, P, P, SZ, P],
    "embbag_fwd": [C.POINTER(BagShape), P, P, P, P, P, P, P],
    "embbag_bwd_workspace": [C.POINTER(BagShape), C.POINTER(SZ)],
    "embbag_bwd": [C.POINTER(BagShape), P, P, P, P, P, P, P, P, P, SZ, P],
    "embbag_grad_apply": [C.POINTER(BagShape), P, P, P, P, P],
    "embbag_bwd_state_bytes": [C.POINTER(BagShape), C.POINTER(SZ)],
    "embbag_bwd_prepare": [C.POINTER(BagShape), P, P, SZ, P],
    "embbag_bwd_state": [C.POINTER(BagShape), P, P, P, P, SZ, P, P, P, P, P, SZ, P],
    "embbag_bwd_atomics": [C.POINTER(BagShape), P, P, P, P, P],
    "embbag_bwd_lock": [C.POINTER(BagShape), P, P, P, P, P, P],
    "embbag_bwd_lock_count": [C.POINTER(BagShape)],
    "ml_sparse_adam": [C.POINTER(BagShape), P, P, P, P, P, P, P, P, C.POINTER(AdamParams), P],
    "memory_layer_fwd_workspace": [C.POINTER(LayerShape), C.POINTER(SZ)],
    "memory_layer_fwd": [C.POINTER(LayerShape)] + [P] * 13 + [SZ, P],
    "memory_layer_bwd_workspace": [C.POINTER(LayerShape), C.POINTER(SZ)],
    "memory_layer_bwd": [C.POINTER(LayerShape)] + [P] * 23 + [SZ, P],
    "memory_layer_state_bytes": [C.POINTER(LayerShape), C.POINTER(SZ)],
    "memory_layer_state_wait": [P, P],
    "peer_fwd_workspace": [C.POINTER(PeerShape), C.POINTER(SZ)],
    "peer_fwd": [C.POINTER(PeerShape)] + [P] * 11 + [SZ, P],
    "peer_bwd_workspace": [C.POINTER(PeerShape), C.POINTER(SZ)],
    "peer_bwd": [C.POINTER(PeerShape)] + [P] * 20 + [SZ, P],
    "memory_layer_fwd_state": [C.POINTER(LayerShape)] + [P] * 13 + [SZ, P, SZ, P],
    "memory_layer_bwd_state": [C.POINTER(LayerShape)] + [P] * 13 + [SZ] + [P] * 11 + [SZ, P],
    "ml_group_unpack": [P, C.c_int32, C.c_int32, C.c_int32, P, P, P, C.c_int, P],
    "ml_group_pack": [P, C.c_int32, C.c_int32, C.c_int32, P, C.c_int, P],
    "ml_gate_bwd": [P, P, P, P, P, P, I64, C.c_int, P],
    "ml_gemm": [C.c_int, C.c_int, I64, I64, I64, P, I64, P, I64, P, I64, C.c_int, C.c_int, P, SZ, P],
    # memory group (a7 / a12)
    "ml_group_unique_id": [P],
    "ml_group_init": [P, C.c_int, C.c_int, C.POINTER(P)],
    "ml_group_hub_create": [C.c_int, C.POINTER(P)],
    "ml_group_hub_destroy": [P],
    "ml_group_init_hub": [P, C.c_int, C.POINTER(P)],
    "ml_group_init_loopback": [C.c_int, C.c_int, P, P, C.c_int, C.POINTER(P)],
    "ml_group_destroy": [P],
    "ml_group_info": [P, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    "ml_group_set_p2p": [P, C.c_int],
    "embbag_fwd_group_workspace": [P, C.POINTER(BagShape), C.c_int, C.POINTER(SZ)],
    "embbag_fwd_group": [P, C.POINTER(BagShape), P, P, P, P, P, C.c_int, P, P, SZ, P],
    "embbag_bwd_group_state_bytes": [P, C.POINTER(BagShape), C.POINTER(SZ)],
    "embbag_bwd_group_prepare": [P, C.POINTER(BagShape), P, P, SZ, P],
    "embbag_bwd_group_sort_local_workspace": [C.POINTER(BagShape), C.POINTER(SZ)],
    "embbag_bwd_group_sort_local": [C.POINTER(BagShape), C.c_int, P, P, P, SZ, P],
    "embbag_bwd_group_merge": [C.POINTER(BagShape), C.c_int, P, P, SZ, P],
    "embbag_bwd_group_workspace": [P, C.POINTER(BagShape), C.c_int, C.POINTER(SZ)],
    "embbag_bwd_group": [P, C.POINTER(BagShape), P, P, P, P, C.c_int, P, SZ, P, P, P, P, P, SZ, P],
    "memory_layer_fwd_group_workspace": [P, C.POINTER(LayerShape), C.c_int, C.POINTER(SZ)],
    "memory_layer_fwd_group": [P, C.POINTER(LayerShape), C.c_int] + [P] * 16 + [SZ, P, SZ, P],
    "memory_layer_bwd_group_workspace": [P, C.POINTER(LayerShape), C.POINTER(SZ)],
    "memory_layer_bwd_group": [P, C.POINTER(LayerShape)] + [P] * 15 + [SZ] + [P] * 11 + [SZ, P],
}
_RESTYPES = {"ml_group_hub_destroy": C.c_int, "ml_last_error": C.c_char_p, "ml_version": C.c_int, "ml_launch_count": C.c_uint64,
             "ml_device_info": C.c_int, "ml_timing_enable": None, "ml_set_serial": None, "ml_timing_reset": None,
             "ml_timing_report": C.c_size_t, "embbag_bwd_lock_count": C.c_int64}

_lib = None


def lib():
    """The loaded CDLL; raises if the extension has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libmemlayer.so not found at {LIB_PATH}: build it with "
                "`python -m paper_2412_09764_b200._build` (no CPU fallback exists)")
        l = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = _RESTYPES[name] if name in _RESTYPES else C.c_int
        _lib = l
    return _lib


def check(status):
    if status != ML_OK:
        raise MemlayerError(status, lib().ml_last_error().decode(errors="replace"))
