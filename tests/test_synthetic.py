"""Pins of the shared counter-based generator."""
import numpy as np
import torch

from synthetic import gen, streams


def test_splitmix64_published_sequence():
    # SplitMix64 seeded with 0: the published first outputs of the sequence
    # (state advanced by the golden gamma before each mix).
    g = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    got = gen.splitmix64(np.array([0, g, (2 * g) % 2**64], dtype=np.uint64))
    assert [int(v) for v in got] == want


def test_round_bf16_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32),
                        np.float32([1 + 2**-8, 1 + 3 * 2**-8, -1 - 2**-8, 0.0])])
    ours = gen.round_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(ours, ref)
    # ties to even, by hand: 1+2^-8 -> 1.0 ; 1+3*2^-8 -> 1+2^-6
    assert ours[-4] == 1.0 and ours[-3] == np.float32(1 + 2**-6)


def test_value_classes():
    u = gen.counter_u64(3, 1, np.arange(4096, dtype=np.uint64))
    c = gen.unit_values(u, gen.CLS_CONTINUOUS)
    assert c.min() >= -1.0 and c.max() < 1.0
    e = gen.unit_values(u, gen.CLS_EXACT)
    assert set(np.unique(e * 8).astype(int)) <= set(range(-8, 8))
    d = gen.unit_values(u, gen.CLS_DYADIC)
    assert np.all(d * 64 == np.round(d * 64)) and d.max() < 1


def test_rows_on_demand_equal_full_tensor():
    full = gen.tensor(7, "V", (64, 48), dtype="bf16")
    ids = np.array([5, 0, 63, 5])
    assert np.array_equal(gen.rows(7, "V", ids, 48, dtype="bf16"), full[ids])
    part = gen.rows(7, "V", ids, 48, dtype="bf16", col_lo=16, col_hi=32)
    assert np.array_equal(part, full[ids, 16:32])


def test_bf16_values_are_representable():
    v = gen.tensor(1, "K1", (100,), scale=gen.scale_for("K1", Dk=1024), dtype="bf16")
    assert np.array_equal(gen.round_bf16(v), v)


def test_streams_shapes_and_ranges():
    N = 1 << 12
    for idx in (streams.uniform_indices(0, 16, 8, N),
                streams.zipf_indices(0, 16, 8, N, 1.1),
                streams.collision_indices(0, 16, 8, N, 50)):
        assert idx.shape == (16, 8) and idx.min() >= 0 and idx.max() < N
    c0 = streams.collision_indices(0, 16, 8, N, 0)
    assert np.unique(c0).size == 128
    c100 = streams.collision_indices(0, 16, 8, N, 100)
    assert np.unique(c100).size == 1
