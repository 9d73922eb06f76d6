"""The C-ABI library builds/loads and exports every symbol include/memlayer.h
declares; host-side validation works without a GPU (no compute calls)."""
import ctypes as C
import os
import re

import pytest

from paper_2412_09764_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "memlayer.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_parsed():
    names = declared_functions()
    for n in ("pkm_topk", "pkm_topk_bwd", "embbag_fwd", "embbag_bwd", "memory_layer_fwd",
              "memory_layer_bwd", "memory_layer_state_bytes", "memory_layer_fwd_state",
              "memory_layer_bwd_state", "peer_fwd", "peer_bwd", "embbag_bwd_prepare",
              "embbag_bwd_state", "ml_last_error",
              "ml_synth_fill", "ml_group_init", "ml_group_destroy", "ml_group_unique_id",
              "embbag_fwd_group", "embbag_bwd_group", "memory_layer_fwd_group",
              "memory_layer_bwd_group"):
        assert n in names


def test_every_declared_symbol_exported():
    lib = _lib.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding declares a signature for each of them
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                       capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", r.stdout))
    assert archs == {"100a"}, archs


def _pkm(T=16, H=2, S=32, Dk=32, k=4, dt=_lib.ML_F32):
    return _lib.PkmShape(T, H, S, Dk, k, dt)


def _size(fn, shape):
    n = C.c_size_t(0)
    st = fn(C.byref(shape), C.byref(n))
    return st, n.value


def test_workspace_queries_on_host():
    lib = _lib.lib()
    st, n = _size(lib.pkm_topk_workspace, _pkm())
    assert st == _lib.ML_OK and n >= 16 * 2 * 2 * 32 * 4
    st, n = _size(lib.embbag_bwd_workspace, _lib.BagShape(1024, 64, 16, 8, _lib.ML_F32))
    assert st == _lib.ML_OK and n > 0
    sh = _lib.LayerShape(_pkm(), 1024, 64, 64, 1)
    for fn in (lib.memory_layer_fwd_workspace, lib.memory_layer_bwd_workspace):
        st, n = _size(fn, sh)
        assert st == _lib.ML_OK and n > 0


@pytest.mark.parametrize("shape,status", [
    (_pkm(k=33, S=64), _lib.ML_ERR_UNSUPPORTED),   # k > 32 (warp select)
    (_pkm(k=5, S=4), _lib.ML_ERR_CONFIG),          # k > S
    (_pkm(Dk=31), _lib.ML_ERR_CONFIG),             # odd Dk
    (_pkm(Dk=6), _lib.ML_ERR_CONFIG),              # half row of 12 B: not 16-B vectors
    (_pkm(S=1 << 16), _lib.ML_ERR_CONFIG),         # N = S^2 >= 2^31
])
def test_pkm_validation(shape, status):
    st, _ = _size(_lib.lib().pkm_topk_workspace, shape)
    assert st == status
    assert _lib.lib().ml_last_error()


def test_bag_and_layer_validation():
    lib = _lib.lib()
    st, _ = _size(lib.embbag_bwd_workspace, _lib.BagShape(1024, 3, 16, 8, _lib.ML_F32))
    assert st == _lib.ML_ERR_CONFIG          # 12-byte rows
    st, _ = _size(lib.embbag_bwd_workspace, _lib.BagShape(1024, 64, 16, 0, _lib.ML_F32))
    assert st == _lib.ML_ERR_CONFIG          # empty bag size
    st, _ = _size(lib.memory_layer_fwd_workspace, _lib.LayerShape(_pkm(), 1000, 64, 64, 1))
    assert st == _lib.ML_ERR_CONFIG          # N != S^2
    st, _ = _size(lib.memory_layer_fwd_workspace, _lib.LayerShape(_pkm(), 1024, 64, 32, 0))
    assert st == _lib.ML_ERR_CONFIG          # ungated needs D == dv


def test_null_pointer_rejected_before_any_launch():
    lib = _lib.lib()
    sh = _lib.BagShape(1024, 64, 16, 8, _lib.ML_F32)
    st = lib.embbag_fwd(C.byref(sh), None, None, None, None, None, None, None)
    assert st == _lib.ML_ERR_ARG


def test_state_and_peer_queries_and_validation():
    """The state / PEER entry points validate on the host (no device needed)."""
    lib = _lib.lib()
    bag = _lib.BagShape(1024, 64, 16, 8, _lib.ML_F32)
    st, n = _size(lib.embbag_bwd_state_bytes, bag)
    assert st == _lib.ML_OK and n > 16 * 8 * 4
    st, n = _size(lib.memory_layer_state_bytes, _lib.LayerShape(_pkm(), 1024, 64, 64, 1))
    assert st == _lib.ML_OK and n > 0
    peer = _lib.PeerShape(_pkm(), 1024, 64)
    for fn in (lib.peer_fwd_workspace, lib.peer_bwd_workspace):
        st, n = _size(fn, peer)
        assert st == _lib.ML_OK and n > 0
    st, _ = _size(lib.peer_fwd_workspace, _lib.PeerShape(_pkm(), 1000, 64))
    assert st == _lib.ML_ERR_CONFIG          # N != S^2
    st, _ = _size(lib.peer_fwd_workspace, _lib.PeerShape(_pkm(), 1024, 3))
    assert st == _lib.ML_ERR_CONFIG          # 12-byte rows
    # a too-small state is refused before any launch
    buf = (C.c_char * 16)()
    st = lib.embbag_bwd_prepare(C.byref(bag), C.cast(buf, C.c_void_p), C.cast(buf, C.c_void_p), 16,
                                None)
    assert st == _lib.ML_ERR_WORKSPACE
    assert lib.memory_layer_state_wait(None, None) == _lib.ML_ERR_ARG


def test_group_bootstrap_on_host():
    """The NCCL unique id (the group bootstrap, P:167's process group) is made
    without a GPU, or ML_ERR_NCCL names a missing libnccl; the in-process hub
    is created and destroyed on the host."""
    lib = _lib.lib()
    buf = C.create_string_buffer(128)
    st = lib.ml_group_unique_id(buf)
    assert st in (_lib.ML_OK, _lib.ML_ERR_NCCL), st
    if st == _lib.ML_OK:
        assert any(buf.raw)
    hub = C.c_void_p()
    assert lib.ml_group_hub_create(2, C.byref(hub)) == _lib.ML_OK and hub.value
    assert lib.ml_group_hub_destroy(hub) == _lib.ML_OK
    assert lib.ml_group_hub_create(0, C.byref(hub)) == _lib.ML_ERR_ARG
    out = C.c_void_p()
    assert lib.ml_group_init(buf, 2, 5, C.byref(out)) in (_lib.ML_ERR_CONFIG, _lib.ML_ERR_NCCL)
