"""Pins for oracle a1 (layout), a2/a4 (gathers, secondary copy): CPU only.

Each test ties the oracle to something other than itself: SPEC.md worked
examples (tests/golden/spec_examples.json), the Eq. (1) size bound, brute-force
round trips against plain slicing, and hand-derived BASELINE numbers.
"""
import json
import os

import numpy as np
import pytest

from oracle import hpz_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["partition"])
def test_partition_spec_examples(ex):
    # A=1 and P'=P reproduce SPEC's own padding rule exactly (reading R2)
    lay = O.LayerLayout(ex["N"], ex["P"], ex["P"], 1)
    full = O.pad_full(np.arange(ex["N"], dtype=np.float32), lay)
    sh = O.partition_primary(full, lay, ex["rank"])
    n_real = len(ex["elements"])
    assert list(sh[:n_real]) == ex["elements"]
    assert sh.size == n_real + ex["pad"]
    assert np.all(sh[n_real:] == 0)


@pytest.mark.parametrize("ex", GOLD["secondary"])
def test_eq1_secondary_size_examples(ex):
    lay = O.LayerLayout(ex["N"], ex["P_prime"], ex["P_prime"], 1)
    assert lay.sec_shard == ex["sec_shard"]
    full = O.pad_full(np.arange(1, ex["N"] + 1, dtype=np.float32), lay)
    secs = [O.secondary_copy(full, lay, r) for r in range(ex["P_prime"])]
    # "equal to full_params[local*s' .. local*s'+s']"
    for r, s in enumerate(secs):
        assert np.array_equal(s, full[r * lay.sec_shard:(r + 1) * lay.sec_shard])
    if "last_local_pad" in ex:
        assert np.count_nonzero(secs[-1] == 0) == ex["last_local_pad"]


@pytest.mark.parametrize("ex", GOLD["secondary_group"])
def test_secondary_group_examples(ex):
    assert O.node_group(ex["rank"], ex["per_node"]) == ex["group"]


def test_gather_constant_shards():
    ex = GOLD["gather_constant_shards"]
    shards = [np.full(ex["shard_len"], c, dtype=np.float32) for c in ex["constants"]]
    F = O.all_gather(shards)
    expect = np.repeat(np.array(ex["constants"], dtype=np.float32), ex["shard_len"])
    assert np.array_equal(F, expect)


def test_layout_baseline_numbers():
    ex = GOLD["layout_baseline"]
    lay = O.LayerLayout(ex["N"], ex["P"], ex["P_prime"], ex["A"])
    assert (lay.numel_pad, lay.shard, lay.sec_shard) == (ex["numel_pad"], ex["shard"], ex["sec_shard"])


def test_topology_errors():
    with pytest.raises(ValueError):
        O.check_topology(8, 3)
    with pytest.raises(ValueError):
        O.check_topology(2, 4)
    with pytest.raises(ValueError):
        O.check_topology(0, 1)


def test_round_trip_bruteforce():
    """Concatenating the P primary shards (truncated) reconstructs the layer."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        N = int(rng.integers(1, 1001))
        P = int(rng.integers(1, 17))
        divs = [d for d in range(1, P + 1) if P % d == 0]
        Pp = int(rng.choice(divs))
        A = int(rng.choice([1, 2, 8, 256]))
        lay = O.LayerLayout(N, P, Pp, A)
        w = rng.standard_normal(N).astype(np.float32)
        full = O.pad_full(w, lay)
        prims = [O.partition_primary(full, lay, r) for r in range(P)]
        assert all(p.size == lay.shard for p in prims)
        F = O.fwd_gather(prims)
        assert np.array_equal(F[:N], w) and np.all(F[N:] == 0)
        # plain-slicing brute force of each shard
        for r in range(P):
            assert np.array_equal(prims[r], np.concatenate([w, np.zeros(lay.numel_pad - N, np.float32)])[r * lay.shard:(r + 1) * lay.shard])


def test_eq1_property_random():
    """Eq. (1): |L_i,second| = N / P', padded: s' >= ceil(N/P'), and the
    P' secondaries of any node reconstruct the layer."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        N = int(rng.integers(1, 100_001))
        Pp = int(rng.integers(1, 17))
        k = int(rng.integers(1, 4))
        P = Pp * k
        lay = O.LayerLayout(N, P, Pp, 256)
        assert lay.sec_shard * Pp == lay.numel_pad
        assert lay.sec_shard >= -(-N // Pp)
        assert lay.sec_shard == k * lay.shard
        w = rng.standard_normal(N).astype(np.float32)
        full = O.pad_full(w, lay)
        for node in range(k):
            secs = {q: O.secondary_copy(full, lay, q) for q in range(node * Pp, (node + 1) * Pp)}
            r = node * Pp
            B = O.bwd_gather([secs.get(q) for q in range(P)], lay, r)
            assert np.array_equal(B[:N], w)


def test_secondary_nests_primary_and_replicates():
    """Secondary of rank r == concat of the primaries l(r)*k .. l(r)*k+k-1 (R2), and it is
    replicated on each node: sec_r == sec_{r+P'} (PAPER.md:73 'replicated on each node')."""
    for (P, Pp) in [(8, 4), (8, 2), (4, 2), (8, 1), (8, 8), (2, 1), (1, 1)]:
        lay = O.LayerLayout(5000, P, Pp, 16)
        full = O.pad_full(np.arange(5000, dtype=np.float32) + 1, lay)
        prims = [O.partition_primary(full, lay, r) for r in range(P)]
        k = P // Pp
        for r in range(P):
            sec = O.secondary_copy(O.fwd_gather(prims), lay, r)
            l = O.local_of(r, Pp)
            assert np.array_equal(sec, np.concatenate(prims[l * k:(l + 1) * k]))
            if r + Pp < P:
                assert np.array_equal(sec, O.secondary_copy(O.fwd_gather(prims), lay, r + Pp))
        if Pp == P:   # single node: secondary == primary shard
            for r in range(P):
                assert np.array_equal(O.secondary_copy(full, lay, r), prims[r])
