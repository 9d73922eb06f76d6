"""The inverse index map's sort (§3.1.4: "preprocessing to
inverse the token_id to embedding_id mapping") through the C ABI
(embbag_bwd_group_sort_local at rank 0: the positions of idx sorted stably by
row).  A stable sort has exactly one result, so the expectation is numpy's
stable argsort of the clamped rows (an index outside [0, N) sorts as row 0
with kClampedPos = bit 31 on its position; include/memlayer.h).

Both device algorithms are covered: the counting sort (key range 2^ceil(log2
N) <= 2 * positions and >= 2 radix passes, i.e. N > 2048) with its three run
regimes (one thread <= 32, one CTA's shared memory <= 8192, CTA merge passes
beyond), and the radix sort (larger key ranges)."""
import numpy as np
import pytest
import torch


pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_09764_b200 import ops  # noqa: F401  (fails loudly without the .so)
    yield


def _expected(idx, N):
    k = idx.astype(np.int64).ravel()
    clamped = (k < 0) | (k >= N)
    k = np.where(clamped, 0, k)
    order = np.argsort(k, kind="stable")
    pos = order.astype(np.int64) | (clamped[order].astype(np.int64) << 31)
    return k[order].astype(np.int32), pos.astype(np.uint32).view(np.int32)


def _rows(seed, N, P, kind):
    rng = np.random.default_rng([seed, N, P, len(kind)])
    idx = rng.integers(0, N, P, dtype=np.int64)
    if kind == "hot":             # one ~5k run (shared-memory chunk), many 33..200 runs
        idx[rng.random(P) < 0.3] = 7
        med = rng.integers(0, N, 60)
        sel = rng.random(P) < 0.25
        idx[sel] = med[rng.integers(0, 60, int(sel.sum()))]
    elif kind == "one":           # a single run of every position (merge passes)
        idx[:] = N - 1
    elif kind == "two_big":       # two runs > 8192, interleaved
        idx = np.where(rng.random(P) < 0.5, 3, N - 2)
    elif kind == "all_clamped":   # every index out of range: one run of row 0
        idx = np.where(rng.random(P) < 0.5, -7, N + 3)
    elif kind == "clamped":       # out-of-range indices join row 0's run
        bad = rng.random(P) < 0.05
        idx[bad] = np.where(rng.random(int(bad.sum())) < 0.5, -1 - rng.integers(0, 9, int(bad.sum())),
                            N + rng.integers(0, 9, int(bad.sum())))
        idx[rng.random(P) < 0.02] = 0
    return idx.astype(np.int32)


@pytest.mark.parametrize("N,P,kind", [
    (5000, 16384, "uniform"),       # counting sort, short runs
    (5000, 16384 + 77, "hot"),      # ragged count; long runs in shared memory
    (4097, 3 * 8192 + 5, "one"),    # one run of 24581: chunk sorts + 2 merge passes
    (8000, 40000, "two_big"),
    (6000, 9000, "clamped"),
    (4500, 4096, "all_clamped"),    # a single 4096-position run of clamped positions
    (2049, 2048 * 3 + 1, "uniform"),  # smallest counting-sort key range (2 passes), ragged
    (1 << 20, 1 << 21, "uniform"),  # the C2 value-row sort (2^20 rows, 2.1M positions)
    (1 << 20, 1 << 18, "uniform"),  # key range > 2 * count: radix sort
    (1 << 20, 1 << 18, "hot"),
    (1000, 5000, "uniform"),        # one radix pass (bits <= 11)
])
def test_sort_local_is_the_stable_sort(N, P, kind):
    from paper_2412_09764_b200 import ops
    idx = _rows(11, N, P, kind)
    lst = ops.group_sort_local(N, torch.from_numpy(idx).cuda().view(P, 1), 0)
    torch.cuda.synchronize()
    got = lst.cpu().numpy()
    rows, pos = _expected(idx, N)
    assert np.array_equal(got[0], rows), kind
    assert np.array_equal(got[1], pos), kind


def _bag_bwd_in_subprocess(arrays, env):
    import os
    import subprocess
    import sys
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        for n, a in arrays.items():
            np.save(os.path.join(d, n + ".npy"), a)
        code = (
            "import numpy as np, torch\n"
            "from paper_2412_09764_b200 import ops\n"
            f"d = {d!r}\n"
            "L = lambda n: torch.from_numpy(np.load(d + '/' + n + '.npy')).cuda()\n"
            "rows, dV, dw = ops.embbag_bwd(L('V').to(torch.bfloat16), L('idx'), L('w'),\n"
            "                              L('dy').to(torch.bfloat16))\n"
            "for n, t in (('rows', rows), ('dV', dV), ('dw', dw)):\n"
            "    np.save(d + '/o_' + n + '.npy', t.cpu().numpy())\n")
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return [np.load(os.path.join(d, f"o_{n}.npy")) for n in ("rows", "dV", "dw")]


@pytest.mark.parametrize("N,T,B,kind,dv", [
    (1 << 16, 1024, 128, "uniform", 1024),   # C2-like: 2 positions per row; the pipelined pass
    (5000, 300, 64, "hot", 64),              # runs > 32 positions (pieces), one of ~5.8k
    (6000, 160, 64, "clamped", 64),
])
def test_runs_from_counting_sort_bit_identical(N, T, B, kind, dv):
    """The runs of the counting sort taken from its per-row counts (row scan,
    ML_RUNS_ROWSCAN=1) give the segmented backward exactly the inputs the pass
    over the sorted positions (find_runs, the default) and the radix sort
    (ML_SORT_COUNTING=0) give: rows, dV and dw bit for bit."""
    P = T * B
    idx = _rows(12, N, P, kind).reshape(T, B)
    rng = np.random.default_rng(5)
    arrays = dict(V=rng.standard_normal((N, dv)).astype(np.float32), idx=idx,
                  w=rng.random((T, B)).astype(np.float32),
                  dy=rng.standard_normal((T, dv)).astype(np.float32))
    base = _bag_bwd_in_subprocess(arrays, {"ML_RUNS_ROWSCAN": "1", "ML_SORT_COUNTING": "1"})
    for env in ({"ML_RUNS_ROWSCAN": "0", "ML_SORT_COUNTING": "1"}, {"ML_SORT_COUNTING": "0"}):
        other = _bag_bwd_in_subprocess(arrays, env)
        for a, b, n in zip(base, other, ("rows", "dV", "dw")):
            assert a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8)), (env, n)


def _pkm_bwd_in_subprocess(arrays, env):
    import os
    import subprocess
    import sys
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        for n, a in arrays.items():
            np.save(os.path.join(d, n + ".npy"), a)
        code = (
            "import numpy as np, torch\n"
            "from paper_2412_09764_b200 import ops\n"
            f"d = {d!r}\n"
            "L = lambda n: torch.from_numpy(np.load(d + '/' + n + '.npy')).cuda()\n"
            "b = lambda n: L(n).to(torch.bfloat16)\n"
            "dq, dK1, dK2 = ops.pkm_topk_bwd(b('q'), b('K1'), b('K2'), L('idx'), L('w'), L('dw'))\n"
            "for n, t in (('dq', dq), ('dK1', dK1), ('dK2', dK2)):\n"
            "    np.save(d + '/o_' + n + '.npy', t.float().cpu().numpy())\n")
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=root,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return [np.load(os.path.join(d, f"o_{n}.npy")) for n in ("dq", "dK1", "dK2")]


@pytest.mark.parametrize("T,H,S,Dk,k", [(512, 4, 4096, 256, 32), (1500, 2, 4096, 128, 16),
                                       (2048, 4, 4096, 256, 32)])   # 16 slots per key: warp-sorted runs
def test_sparse_key_backward_counting_sort_bit_identical(T, H, S, Dk, k):
    """The sparse key backward (S > 2048) sorts its half-key slots with the
    counting sort when the key range 2^ceil(log2(H*S + 1)) is at most twice
    the slot count and the slots at most ML_SORT_COUNTING_MAX_PER_KEY per key
    (default 8; 64 here, so the third case's runs go through the warp sort);
    the deduplication sentinel's run (most slots) stays unordered, which the
    segmented pass skips: dq, dK1, dK2 equal the radix path's bit for bit."""
    from oracle import pkm as opkm
    from synthetic import gen
    sc = gen.scale_for("K1", Dk=Dk)
    q = gen.tensor(44, "q", (T, H, Dk), dtype="bf16")
    K1 = gen.tensor(44, "K1", (H, S, Dk // 2), scale=sc, dtype="bf16")
    K2 = gen.tensor(44, "K2", (H, S, Dk // 2), scale=sc, dtype="bf16")
    ridx, _, rw = opkm.pkm_lookup(q.astype(np.float64), K1.astype(np.float64), K2.astype(np.float64), k)
    dw = gen.tensor(44, "dout", (T, H, k), dtype="f32")
    arrays = dict(q=q.astype(np.float32), K1=K1.astype(np.float32), K2=K2.astype(np.float32),
                  idx=ridx.astype(np.int32), w=rw.astype(np.float32), dw=dw.astype(np.float32))
    a = _pkm_bwd_in_subprocess(arrays, {"ML_SORT_COUNTING": "1", "ML_SORT_COUNTING_MAX_PER_KEY": "64"})
    b = _pkm_bwd_in_subprocess(arrays, {"ML_SORT_COUNTING": "0"})
    for x, y, n in zip(a, b, ("dq", "dK1", "dK2")):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), n
