"""Row-sharded step, host side (world_size 2, gloo on CPU): the owner work lists
partition every candidate and anchor contribution exactly once across ranks,
CSR rows are the owners' local rows, and the host-staged collectives compute
all-gather / reduce-scatter / all-to-all / all-reduce."""
import pickle
import socket

import numpy as np
import pytest

import paper_2602_21597_b200 as m

torch = pytest.importorskip("torch")
ALL = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni", "inp"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def plans(tmp_path_factory):
    import torch.multiprocessing as mp

    import shard_workers
    out = tmp_path_factory.mktemp("shard")
    mp.spawn(shard_workers.host_plan_worker, args=(2, _port(), str(out), "small", ALL, 48, 8, 16),
             nprocs=2, join=True)
    return [pickle.load(open(out / f"plan{r}.pkl", "rb")) for r in range(2)]


def test_collectives_host_staged(plans):
    x = [np.arange(6, dtype=np.float32) + 10 * r for r in range(2)]
    for r, p in enumerate(plans):
        c = p["coll"]
        assert np.array_equal(c["ag"], np.concatenate(x))
        assert np.array_equal(c["rs"], (x[0] + x[1])[3 * r:3 * r + 3])
        assert np.array_equal(c["a2a"], np.concatenate([x[0][3 * r:3 * r + 3], x[1][3 * r:3 * r + 3]]))
        assert np.array_equal(c["ar"], x[0] + x[1])


def test_metadata_identical_on_all_ranks(plans):
    for key in ("anchor_ids", "unit_k", "unit_slots", "cand"):
        assert np.array_equal(plans[0][key], plans[1][key])


def test_owned_candidates_partition(plans):
    G = 2
    p0 = plans[0]
    U, nc = G * p0["batch"], p0["nc"]
    cand = p0["cand"].reshape(U, nc)
    seen = np.zeros((U, nc), np.int32)
    for r, p in enumerate(plans):
        for u in range(U):
            for j in p["owned"][p["unit_off"][u]:p["unit_off"][u + 1]]:
                assert cand[u, j] % G == r
                seen[u, j] += 1
    live = p0["unit_k"] > 0
    assert (seen[live] == 1).all() and (seen[~live] == 0).all()


def test_owner_csr_partitions_contributions(plans):
    G = 2
    p0 = plans[0]
    A, S, B, nc = p0["A"], p0["S"], p0["batch"], p0["nc"]
    codes = []
    for r, p in enumerate(plans):
        rows, seg, con = p["rows"], p["seg"], p["contrib"]
        assert np.all(np.diff(rows) > 0)  # ascending local rows
        for i, lr in enumerate(rows):
            ent = lr * G + r  # local row -> global entity
            for code in con[seg[i]:seg[i + 1]]:
                if code < 0:
                    q, a = divmod(-code - 1, A)
                    assert p0["anchor_ids"][q * A + a] == ent
                else:
                    gslot, j = divmod(code, nc)
                    q, slot = divmod(gslot, S)
                    units = np.where((p0["unit_slots"].reshape(G * B, 3)[q * B:(q + 1) * B] == slot).any(1))[0]
                    assert len(units) == 1
                    assert p0["cand"].reshape(G * B, nc)[q * B + units[0], j] == ent
                codes.append(code)
    assert len(codes) == len(set(codes))
    n_anchor = int((p0["anchor_ids"] >= 0).sum())
    n_cand = int(sum(p0["unit_k"][u] * nc for u in range(G * B)))
    assert len(codes) == n_anchor + n_cand
