"""Parity at BASELINE.json's full size (config[1], the bench.py workload):
N = 1024^2 values x 2048, 4 heads, k = 32, 16K tokens, bf16, Memory+ gate,
run through the same C-ABI entry points bench.py times.  The oracle checks
sampled outputs it can compute one by one:

* idx / w / y / out / dw / dq of sampled tokens (oracle per token, rows of
  the 4 GiB value table regenerated on demand);
* dV of sampled rows: every (token, head) whose half top-k lists contain the
  row's two sub-keys is found from the oracle's full half-score matrices and
  re-run through the exact two-stage lookup, so the row's complete
  contributor set is the oracle's own;
* the key gradients via an identity that holds at any size:
  sum_a <dK1[h,a], K1[h,a]> = sum_t <dq1[t,h], q1[t,h]> (both equal
  sum_{t,j} ds_j s1_j).
"""
import numpy as np
import pytest
import torch

from oracle import bag as obag, gate as ogate, pkm as opkm
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SEED = 0
S, dv, D, Dk, H, k, T = 1024, 2048, 2048, 1024, 4, 32, 16384
Dh = Dk // 2


@pytest.fixture(scope="module")
def run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench
    from paper_2412_09764_b200 import ops
    cfg = bench.CONFIGS["c2"]
    assert (cfg["S"], cfg["dv"], cfg["H"], cfg["k"], cfg["T"]) == (S, dv, H, k, T)
    t = bench.make_inputs(cfg, torch.device("cuda", 0), 1, 0, ops, torch)
    out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"], k)
    g = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"],
                             saved, want_dw=True)
    torch.cuda.synchronize()
    res = dict(out=out, idx=host(saved["idx"]), w=host(saved["w"]), y=saved["y"], g=saved["g"],
               dq=g["dq"], dK1=g["dK1"], dK2=g["dK2"], dw=host(g["dw"]), U=int(g["U"].item()))
    res["rows"] = g["rows"][:res["U"]].cpu().numpy()
    res["dV"] = g["dV"][:res["U"]]
    del t
    return res


@pytest.fixture(scope="module")
def host_tables():
    f64 = lambda a: a.astype(np.float64)
    K1 = f64(gen.tensor(SEED, "K1", (H, S, Dh), scale=gen.scale_for("K1", Dk=Dk), dtype="bf16"))
    K2 = f64(gen.tensor(SEED, "K2", (H, S, Dh), scale=gen.scale_for("K2", Dk=Dk), dtype="bf16"))
    W1 = f64(gen.tensor(SEED, "W1", (D, dv), scale=gen.scale_for("W1", D=D), dtype="bf16"))
    W2 = f64(gen.tensor(SEED, "W2", (dv, D), scale=gen.scale_for("W2", dv=dv), dtype="bf16"))
    return dict(K1=K1, K2=K2, W1=W1, W2=W2)


def Vrows(ids):
    return gen.rows(SEED, "V", np.asarray(ids), dv, dtype="bf16").astype(np.float64)


def q_of(tokens):
    tokens = np.asarray(tokens)
    rows = (tokens[:, None] * H + np.arange(H)[None, :]).reshape(-1)
    return gen.rows(SEED, "q", rows, Dk, dtype="bf16").astype(np.float64).reshape(-1, H, Dk)


def token_oracle(tokens, tb):
    """Oracle forward + the token-local backward pieces for `tokens`."""
    q = q_of(tokens)
    idx, score, w = opkm.pkm_lookup(q, tb["K1"], tb["K2"], k)
    x = gen.rows(SEED, "x", tokens, D, dtype="bf16").astype(np.float64)
    dout = gen.rows(SEED, "dout", tokens, D, dtype="bf16").astype(np.float64)
    n = len(tokens)
    bidx, bw = idx.reshape(n, H * k), w.reshape(n, H * k)
    y = np.stack([bw[i] @ Vrows(bidx[i]) for i in range(n)])
    out, gpre, z = ogate.gate_fwd(x, y, tb["W1"], tb["W2"])
    gb = ogate.gate_bwd(dout, x, y, gpre, tb["W1"], tb["W2"])
    dy = gb["dy"]
    dw = np.stack([Vrows(bidx[i]) @ dy[i] for i in range(n)])
    dq, _, _, _ = opkm.pkm_bwd(q, tb["K1"], tb["K2"], idx, w, dw.reshape(n, H, k))
    return dict(q=q, idx=idx, w=w, y=y, out=out, dy=dy, dw=dw, dq=dq)


SAMPLE = np.array([0, 1, 2, 127, 128, 4095, 8191, 9000, 12345, 16382, 16383] +
                  list(np.random.default_rng(0).choice(T, 9, replace=False)))


def test_sampled_tokens(run, host_tables):
    r = token_oracle(SAMPLE, host_tables)
    near = compare_topk(run["idx"][SAMPLE], r["idx"], r["q"], host_tables["K1"], host_tables["K2"])
    ok = np.ones((len(SAMPLE), H), bool)
    for i, h, _ in near:
        ok[i, h] = False
    tok_ok = ok.all(1)
    assert tok_ok.sum() >= len(SAMPLE) - 2, f"too many near ties: {near}"
    assert_close(run["w"][SAMPLE][ok], r["w"][ok], TOL["f32"], "w")
    s = SAMPLE[tok_ok]
    assert_close(host(run["y"][torch.as_tensor(s)]), r["y"][tok_ok], TOL["bf16"], "y")
    assert_close(host(run["out"][torch.as_tensor(s)]), r["out"][tok_ok], TOL["bf16"], "out")
    assert_close(run["dw"][s].reshape(len(s), -1), r["dw"][tok_ok], TOL["bf16"], "dw")
    assert_close(host(run["dq"][torch.as_tensor(s)]), r["dq"][tok_ok], TOL["bf16"], "dq")


def test_sampled_value_rows(run, host_tables):
    """dV of rows chosen by the oracle, with their complete contributor sets."""
    tb = host_tables
    r0 = token_oracle(SAMPLE[:3], tb)
    rows = sorted(set(r0["idx"][0, 0, :3].tolist()) | set(r0["idx"][1, 2, :2].tolist())
                  | {int(r0["idx"][2, 3, 5])})
    q_all = q_of(np.arange(T))                      # [T, H, Dk]
    contrib = {rr: [] for rr in rows}
    for h in range(H):
        s1 = q_all[:, h, :Dh] @ tb["K1"][h].T       # [T, S] all half scores (fp64)
        s2 = q_all[:, h, Dh:] @ tb["K2"][h].T
        kth1 = -np.partition(-s1, k - 1, axis=1)[:, k - 1]
        kth2 = -np.partition(-s2, k - 1, axis=1)[:, k - 1]
        for rr in rows:
            a, b = divmod(rr, S)
            cand = np.nonzero((s1[:, a] >= kth1) & (s2[:, b] >= kth2))[0]
            for t in cand:                         # exact two-stage for the candidates
                I, sc = opkm.topk_two_stage(q_all[t, h], tb["K1"][h], tb["K2"][h], k)
                if rr in I.tolist():
                    j = I.tolist().index(rr)
                    contrib[rr].append((int(t), h, j, opkm.softmax(sc)[j]))
    toks = sorted({t for v in contrib.values() for (t, _, _, _) in v})
    ro = token_oracle(np.array(toks), tb)
    dy = {t: ro["dy"][i] for i, t in enumerate(toks)}
    gpu_rows = run["rows"]
    for rr in rows:
        assert contrib[rr], rr
        ref = sum(wj * dy[t] for (t, h, j, wj) in contrib[rr])
        pos = np.searchsorted(gpu_rows, rr)
        assert pos < len(gpu_rows) and gpu_rows[pos] == rr, f"row {rr} missing from the GPU dV rows"
        assert_close(host(run["dV"][pos]), ref, TOL["bf16"], f"dV[{rr}]")


def test_key_gradient_identity(run, host_tables):
    """sum_a <dK_half[h,a], K_half[h,a]> == sum_t <dq_half[t,h], q_half[t,h]>
    (both equal sum_{t,j} ds_j s_half_j); holds at any size."""
    q = q_of(np.arange(T))
    dq = host(run["dq"])
    for half, (dK, K) in enumerate(((run["dK1"], host_tables["K1"]), (run["dK2"], host_tables["K2"]))):
        lhs = (host(dK) * K).sum(axis=(1, 2))
        sl = slice(half * Dh, (half + 1) * Dh)
        rhs = (dq[:, :, sl] * q[:, :, sl]).sum(axis=(0, 2))
        scale = np.abs(host(dK) * K).sum(axis=(1, 2))
        assert np.all(np.abs(lhs - rhs) <= 1e-4 * scale + 1e-6), (half, lhs, rhs)


def test_row_set_properties(run):
    rows = run["rows"]
    assert np.all(np.diff(rows) > 0)                       # ascending, distinct
    flat = run["idx"].reshape(-1)
    assert run["U"] == np.unique(flat).size                # = distinct selected rows
    assert np.array_equal(rows, np.unique(flat))
    w = run["w"]
    np.testing.assert_allclose(w.sum(-1), 1.0, atol=1e-5)  # softmax per head
    assert np.all(np.diff(w, axis=-1) <= 1e-7)             # sorted by descending score
