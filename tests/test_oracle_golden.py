"""Pin the C restatement (oracle/) against the reference's golden fixtures
(tests/golden/, generated from the unmodified reference by make_golden.py)
and its literal known-answer tests."""
import numpy as np
import pytest

import oracle as O
from helpers import SCENARIOS, load_scenario, oracle_from_scenario, replay


@pytest.mark.parametrize("name", SCENARIOS)
def test_oracle_replays_reference_scenario(name):
    sc = load_scenario(name)
    ix = oracle_from_scenario(sc)
    bad = replay(ix, sc)
    assert not bad, bad[:10]


def test_interleaved_offsets_kat():
    # test_block_store.cpp:112-122
    L = O.oracle_lib()
    got = [L.orc_interleaved_offset(s, d, 4, 32) for (s, d) in
           [(0, 0), (0, 1), (1, 0), (1, 1), (32, 0), (32, 1)]]
    assert got == [0, 32, 1, 33, 128, 160]
    # dim=2 block of 64 slots: slot 32 starts the second group (offset 64)
    assert L.orc_interleaved_offset(32, 0, 2, 32) == 64
    assert L.orc_interleaved_offset(33, 1, 2, 32) == 97


def test_distance_kat_and_order():
    # test_ivf_index.cpp:164-171: distance 25 = 9 + 16
    assert O.oracle_l2([1, 2], [4, 6]) == 25.0
    rng = np.random.default_rng(0)
    for _ in range(50):
        a = rng.normal(size=37).astype(np.float32) * 30
        b = rng.normal(size=37).astype(np.float32) * 30
        acc = np.float32(0)
        for d in range(37):
            t = np.float32(a[d] - b[d])
            acc = np.float32(acc + np.float32(t * t))
        assert np.float32(O.oracle_l2(a, b)).view(np.uint32) == acc.view(np.uint32)
        s = np.float32(0)
        for d in range(37):
            s = np.float32(s + np.float32(a[d] * b[d]))
        assert np.float32(O.oracle_ip(a, b)).view(np.uint32) == s.view(np.uint32)


def test_five_inserts_two_blocks_kat():
    # test_ivf_index.cpp:102-123 (blocks of 4 and 1, hops 1) and auto id 2 (:91-100)
    cent = np.array([[0, 0], [10, 10]], np.float32)
    ix = O.OracleIndex(cent, cent, np.array([0, 1], np.uint32), 4, 256)
    ids, rc, ins = ix.insert(np.array([[0.01 * i, 0] for i in range(5)], np.float32))
    assert rc == 0 and ins == 5 and ids[0] == 2
    k = ix.assign([0, 0])
    assert ix.list_length(k) == 5 and ix.hop_count(k) == 1
    h = ix.online_head(k)
    assert ix.block_header(h)[2] == 4
    nxt = ix.block_header(h)[1]
    assert ix.block_header(nxt)[2] == 1 and ix.block_header(nxt)[1] == -1


def test_pool_exhaustion_kat():
    # test_ivf_index.cpp:291-313: 2 blocks of 2 slots -> inserted == 4, poisoned list
    cent = np.array([[0, 0], [10, 10]], np.float32)
    ix = O.OracleIndex(cent, cent, np.array([0, 1], np.uint32), 2, 2)
    _, rc, ins = ix.insert(np.array([[0, 0.1 * i] for i in range(6)], np.float32))
    assert rc == O.ORC_EPOOL and ins == 4
    k = ix.assign([0, 0])
    assert ix.list_length(k) == 4
    _, rc, ins = ix.insert(np.array([[0.0, 0.9]], np.float32))
    assert rc == O.ORC_EPOOL and ins == 0 and ix.list_length(k) == 4


def test_exceed_strict_kat():
    # test_ivf_index.cpp:200-214
    cent = np.array([[0, 0], [10, 10]], np.float32)
    ix = O.OracleIndex(cent, cent, np.array([0, 1], np.uint32), 4, 256, rearrange_threshold=4)
    k = ix.assign([0, 0])
    assert not ix.exceed(k)
    ix.insert(np.array([[0, 0], [0, 0.1], [0, 0.2], [0, 0.3]], np.float32))
    assert not ix.exceed(k)
    ix.insert(np.array([[0, 0.4]], np.float32))
    assert ix.exceed(k)


def test_remove_semantics():
    """Delete restatement (parity unpinned: the reference has no delete)."""
    cent = np.array([[0, 0], [10, 10]], np.float32)
    off = np.array([[0, 0], [0, 1], [0, 2], [10, 10]], np.float32)
    ix = O.OracleIndex(cent, off, np.array([0, 0, 0, 1], np.uint32), 2, 16)
    ids, _, _ = ix.insert(np.array([[0, 3 + i] for i in range(5)], np.float32))  # 4..8 in list 0
    # remove an offline id (hole filled by the segment's last), an online id
    # (filled by the list's last), an unknown id, and a duplicate request
    rem, found = ix.remove([1, 5, 999, 5, 8])
    assert rem == 3 and found.tolist() == [True, True, False, False, True]
    ids0, vecs0 = ix.cluster_contents(0)
    assert ids0.tolist() == [0, 2, 4, 7, 6]
    assert vecs0[1].tolist() == [0, 2] and vecs0[3].tolist() == [0, 6]
    assert ix.offline_count(0) == 2 and ix.list_length(0) == 3
    assert ix.size == 6
    # the emptied tail block stays linked and is reused by the next insert
    nb = ix.allocated_blocks()
    ix.insert(np.array([[0, 9]], np.float32))
    assert ix.allocated_blocks() == nb and ix.list_length(0) == 4
