"""Shared machinery of the full-size parity tests (tests/test_gpu_fullsize*.py):
one BASELINE.json configuration run through the same C-ABI entry points
bench.py times, checked by the oracle on outputs it can compute one by one
(rows of the value table regenerated on demand from the synthetic
generator, so the tables never exist on the host).

* idx / w / y / out / dw / dq of sampled tokens (oracle per token);
* dV of sampled rows: every (token, head) whose half top-k lists contain the
  row's two sub-keys is found from the oracle's full half-score matrices and
  re-run through the exact two-stage lookup, so the row's complete
  contributor set is the oracle's own;
* the key gradients via an identity that holds at any size:
  sum_a <dK1[h,a], K1[h,a]> = sum_t <dq1[t,h], q1[t,h]> (both = sum_{t,j} ds_j s1_j);
* the row set: ascending, distinct, equal to the distinct selected indices.
"""
import numpy as np
import torch

from oracle import gate as ogate, pkm as opkm
from synthetic import gen
from tests.gpu_util import TOL, assert_close, compare_topk, host

SEED = 0


class Full:
    def __init__(self, cfg_name):
        import bench
        self.cfg = bench.CONFIGS[cfg_name]
        c = self.cfg
        self.name = cfg_name
        self.S, self.dv, self.D, self.Dk = c["S"], c["dv"], c["D"], c["Dk"]
        self.H, self.k, self.T = c["H"], c["k"], c["T"]
        self.Dh = self.Dk // 2

    # ------------------------------------------------------------- GPU run
    def run(self):
        import bench
        from paper_2412_09764_b200 import ops
        t = bench.make_inputs(self.cfg, torch.device("cuda", 0), 1, 0, ops, torch, False)
        k = self.k
        out, saved = ops.memory_layer_fwd(t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"], t["W2"], k)
        g = ops.memory_layer_bwd(t["dout"], t["x"], t["q"], t["K1"], t["K2"], t["V"], t["W1"],
                                 t["W2"], saved, want_dw=True)
        torch.cuda.synchronize()
        res = dict(out=out, idx=host(saved["idx"]), w=host(saved["w"]), y=saved["y"],
                   dq=g["dq"], dK1=g["dK1"], dK2=g["dK2"], dw=host(g["dw"]), U=int(g["U"].item()))
        res["rows"] = g["rows"][:res["U"]].cpu().numpy()
        res["dV"] = g["dV"][:res["U"]].clone()
        del t, g, saved
        torch.cuda.empty_cache()
        return res

    # ---------------------------------------------------------- host side
    def host_tables(self):
        f64 = lambda a: a.astype(np.float64)
        S, Dh, Dk, D, dv, H = self.S, self.Dh, self.Dk, self.D, self.dv, self.H
        return dict(
            K1=f64(gen.tensor(SEED, "K1", (H, S, Dh), scale=gen.scale_for("K1", Dk=Dk), dtype="bf16")),
            K2=f64(gen.tensor(SEED, "K2", (H, S, Dh), scale=gen.scale_for("K2", Dk=Dk), dtype="bf16")),
            W1=f64(gen.tensor(SEED, "W1", (D, dv), scale=gen.scale_for("W1", D=D), dtype="bf16")),
            W2=f64(gen.tensor(SEED, "W2", (dv, D), scale=gen.scale_for("W2", dv=dv), dtype="bf16")))

    def Vrows(self, ids):
        return gen.rows(SEED, "V", np.asarray(ids), self.dv, dtype="bf16").astype(np.float64)

    def q_of(self, tokens):
        tokens = np.asarray(tokens)
        H = self.H
        rows = (tokens[:, None] * H + np.arange(H)[None, :]).reshape(-1)
        return gen.rows(SEED, "q", rows, self.Dk, dtype="bf16").astype(np.float64).reshape(-1, H, self.Dk)

    def token_oracle(self, tokens, tb):
        """Oracle forward + the token-local backward pieces for `tokens`."""
        H, k, D = self.H, self.k, self.D
        q = self.q_of(tokens)
        idx, score, w = opkm.pkm_lookup(q, tb["K1"], tb["K2"], k)
        x = gen.rows(SEED, "x", tokens, D, dtype="bf16").astype(np.float64)
        dout = gen.rows(SEED, "dout", tokens, D, dtype="bf16").astype(np.float64)
        n = len(tokens)
        bidx, bw = idx.reshape(n, H * k), w.reshape(n, H * k)
        y = np.stack([bw[i] @ self.Vrows(bidx[i]) for i in range(n)])
        out, gpre, z = ogate.gate_fwd(x, y, tb["W1"], tb["W2"])
        gb = ogate.gate_bwd(dout, x, y, gpre, tb["W1"], tb["W2"])
        dy = gb["dy"]
        dw = np.stack([self.Vrows(bidx[i]) @ dy[i] for i in range(n)])
        dq, _, _, _ = opkm.pkm_bwd(q, tb["K1"], tb["K2"], idx, w, dw.reshape(n, H, k))
        # rounding-model magnitudes sum|terms| (tests/gpu_util.py assert_close mag=)
        A = np.abs
        sg = A(ogate.silu(gpre))
        mdy = (A(dout) @ A(tb["W2"]).T) * sg
        mw = np.stack([A(self.Vrows(bidx[i])) @ mdy[i] for i in range(n)])
        mds = (w * (mw.reshape(n, H, k) + (w * mw.reshape(n, H, k)).sum(-1, keepdims=True)))
        S, Dh = self.S, self.Dh
        mdq = np.zeros(q.shape)
        for hh in range(H):
            for j in range(k):
                a, b = idx[:, hh, j] // S, idx[:, hh, j] % S
                mdq[:, hh, :Dh] += mds[:, hh, j, None] * A(tb["K1"][hh, a])
                mdq[:, hh, Dh:] += mds[:, hh, j, None] * A(tb["K2"][hh, b])
        mag = dict(y=np.stack([bw[i] @ A(self.Vrows(bidx[i])) for i in range(n)]),
                   out=(A(y) * sg) @ A(tb["W2"]), dy=mdy, dw=mw, dq=mdq)
        return dict(q=q, idx=idx, w=w, y=y, out=out, dy=dy, dw=dw, dq=dq, mag=mag)

    def sample(self):
        T = self.T
        return np.array([0, 1, 2, 127, 128, 4095, 8191, 9000, 12345, T - 2, T - 1] +
                        list(np.random.default_rng(0).choice(T, 9, replace=False)))

    # --------------------------------------------------------------- checks
    def check_sampled_tokens(self, run, tb):
        SAMPLE = self.sample()
        H = self.H
        r = self.token_oracle(SAMPLE, tb)
        near = compare_topk(run["idx"][SAMPLE], r["idx"], r["q"], tb["K1"], tb["K2"])
        ok = np.ones((len(SAMPLE), H), bool)
        for i, h, _ in near:
            ok[i, h] = False
        tok_ok = ok.all(1)
        assert tok_ok.sum() >= len(SAMPLE) - 2, f"too many near ties: {near}"
        assert_close(run["w"][SAMPLE][ok], r["w"][ok], TOL["f32"], "w")
        s = SAMPLE[tok_ok]
        m = r["mag"]
        assert_close(host(run["y"][torch.as_tensor(s)]), r["y"][tok_ok], TOL["bf16"], "y",
                     mag=m["y"][tok_ok])
        assert_close(host(run["out"][torch.as_tensor(s)]), r["out"][tok_ok], TOL["bf16"], "out",
                     mag=m["out"][tok_ok])
        assert_close(run["dw"][s].reshape(len(s), -1), r["dw"][tok_ok], TOL["bf16"], "dw",
                     mag=m["dw"][tok_ok])
        assert_close(host(run["dq"][torch.as_tensor(s)]), r["dq"][tok_ok], TOL["bf16"], "dq",
                     mag=m["dq"][tok_ok])

    def check_sampled_value_rows(self, run, tb, n_rows=6):
        """dV of rows chosen by the oracle, with their complete contributor sets."""
        S, H, k, Dh, T = self.S, self.H, self.k, self.Dh, self.T
        SAMPLE = self.sample()
        r0 = self.token_oracle(SAMPLE[:3], tb)
        rows = sorted(set(r0["idx"][0, 0, :3].tolist()) | set(r0["idx"][1, 2, :2].tolist())
                      | {int(r0["idx"][2, 3, 5])})[:n_rows]
        q_all = self.q_of(np.arange(T))                     # [T, H, Dk]
        contrib = {rr: [] for rr in rows}
        for h in range(H):
            s1 = q_all[:, h, :Dh] @ tb["K1"][h].T           # [T, S] all half scores (fp64)
            s2 = q_all[:, h, Dh:] @ tb["K2"][h].T
            kth1 = -np.partition(-s1, k - 1, axis=1)[:, k - 1]
            kth2 = -np.partition(-s2, k - 1, axis=1)[:, k - 1]
            for rr in rows:
                a, b = divmod(rr, S)
                cand = np.nonzero((s1[:, a] >= kth1) & (s2[:, b] >= kth2))[0]
                for t in cand:                             # exact two-stage for the candidates
                    I, sc = opkm.topk_two_stage(q_all[t, h], tb["K1"][h], tb["K2"][h], k)
                    if rr in I.tolist():
                        j = I.tolist().index(rr)
                        contrib[rr].append((int(t), h, j, opkm.softmax(sc)[j]))
        toks = sorted({t for v in contrib.values() for (t, _, _, _) in v})
        ro = self.token_oracle(np.array(toks), tb)
        dy = {t: ro["dy"][i] for i, t in enumerate(toks)}
        mdy = {t: ro["mag"]["dy"][i] for i, t in enumerate(toks)}
        gpu_rows = run["rows"]
        for rr in rows:
            assert contrib[rr], rr
            ref = sum(wj * dy[t] for (t, h, j, wj) in contrib[rr])
            mag = sum(wj * mdy[t] for (t, h, j, wj) in contrib[rr])
            pos = np.searchsorted(gpu_rows, rr)
            assert pos < len(gpu_rows) and gpu_rows[pos] == rr, f"row {rr} missing from the GPU dV rows"
            assert_close(host(run["dV"][pos]), ref, TOL["bf16"], f"dV[{rr}]", mag=mag)

    def check_key_gradient_identity(self, run, tb):
        Dh, T = self.Dh, self.T
        q = self.q_of(np.arange(T))
        dq = host(run["dq"])
        for half, (dK, K) in enumerate(((run["dK1"], tb["K1"]), (run["dK2"], tb["K2"]))):
            lhs = (host(dK) * K).sum(axis=(1, 2))
            sl = slice(half * Dh, (half + 1) * Dh)
            rhs = (dq[:, :, sl] * q[:, :, sl]).sum(axis=(0, 2))
            scale = np.abs(host(dK) * K).sum(axis=(1, 2))
            assert np.all(np.abs(lhs - rhs) <= 1e-4 * scale + 1e-6), (half, lhs, rhs)

    @staticmethod
    def check_row_set(run):
        rows = run["rows"]
        assert np.all(np.diff(rows) > 0)                       # ascending, distinct
        flat = run["idx"].reshape(-1)
        assert run["U"] == np.unique(flat).size                # = distinct selected rows
        assert np.array_equal(rows, np.unique(flat))
        w = run["w"]
        np.testing.assert_allclose(w.sum(-1), 1.0, atol=1e-5)  # softmax per head
        assert np.all(np.diff(w, axis=-1) <= 1e-7)             # sorted by descending score
