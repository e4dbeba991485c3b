"""The shared input generator: numpy and torch backends are bit-identical,
values are in range, index ranges compose (a rank draws exactly its shard)."""
import numpy as np
import torch

import gen

P30 = 998244353
P32 = 3221225473
PG = (1 << 64) - (1 << 32) + 1


def test_numpy_torch_identical():
    for p in (P30, P32, PG, 7, 1108307720798209, (1 << 50) - 27, (1 << 40) + 15):
        a = gen.residues(gen.config_seed(3), 1, 100_003, p)
        t = gen.residues_torch(gen.config_seed(3), 1, 100_003, p, "cpu")
        t = t.numpy().view(np.uint32 if p < (1 << 32) else np.uint64)
        assert np.array_equal(a, t)
        assert int(a.max()) < p
    l = gen.limbs16(5, 2, 4099)
    assert np.array_equal(l, gen.limbs16_torch(5, 2, 4099, "cpu").numpy().view(np.uint16))


def test_shards_compose():
    full = gen.residues(11, 2, 1 << 16, P30)
    parts = [gen.residues(11, 2, 1 << 14, P30, start=r << 14) for r in range(4)]
    assert np.array_equal(full, np.concatenate(parts))
    tparts = [gen.residues_torch(11, 2, 1 << 14, P30, "cpu", start=r << 14).numpy().view(np.uint32) for r in range(4)]
    assert np.array_equal(full, np.concatenate(tparts))


def test_streams_and_seeds_differ():
    a = gen.residues(1, 1, 1000, P30)
    b = gen.residues(1, 2, 1000, P30)
    c = gen.residues(2, 1, 1000, P30)
    assert (a != b).mean() > 0.99 and (a != c).mean() > 0.99


def test_roughly_uniform():
    a = gen.residues(gen.config_seed(2), 1, 1 << 20, P32).astype(np.float64) / P32
    hist, _ = np.histogram(a, bins=16, range=(0, 1))
    assert hist.min() > 0.9 * (1 << 20) / 16 and hist.max() < 1.1 * (1 << 20) / 16
