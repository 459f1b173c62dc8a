"""bench.py host logic without a GPU: both arms print the same config keys; the rank-row cost model the strong-
scaling shards use equals the C ABI's ttc_pair_cost; the partition covers every pair exactly once."""
import numpy as np

import bench
import paper_2109_00626_b200 as ttc
import ttgen


def test_config_dict_same_keys_for_both_arms():
    a = bench.config_dict("C2", 4096, 1, 7)
    b = bench.config_dict("C2", 4096, 1, 7)
    assert a == b
    assert a["global_pairs"] == 4096 and a["parallelism"] == "dp1" and a["workload"] == "C2"
    assert bench.config_dict("C5", 100, 8, 7)["global_pairs"] == 800


def test_pair_macs_matches_ttc_pair_cost():
    X, Y = ttgen.config_batch("C5", B=37)
    mac, _ = ttc.ttc_pair_cost(ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y))
    got = bench.pair_macs(X.ranks, Y.ranks, X.dims)
    np.testing.assert_allclose(got, mac, rtol=0, atol=0)


def test_strong_scaling_shards_cover_the_batch():
    c = ttgen.CONFIGS["C5"]
    G = 1000
    xr = ttgen.random_ranks(1, 5, 0, 0, G, c["N"], c["rank_choices"])
    yr = ttgen.random_ranks(1, 5, 1, 0, G, c["N"], c["rank_choices"])
    cost = bench.pair_macs(xr, yr, (c["I"],) * c["N"])
    for world in (1, 2, 4, 8):
        b = ttc.ttc_partition(cost, world)
        assert b[0] == 0 and b[-1] == G and np.all(np.diff(b) >= 0)
        parts = [cost[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(parts) <= cost.sum() / world + cost.max()
