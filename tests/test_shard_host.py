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


@pytest.fixture(scope="module", params=[("q2b", False, 2), ("betae", True, 2), ("q2b", False, 3)],
                ids=["q2b", "betae-fused", "q2b-world3"])
def plans(tmp_path_factory, request):
    # (the FuseSemantic plan puts FuseSemantic nodes where EmbedAnchor was:
    # their anchors must enter the lookup exchange the same way)
    import torch.multiprocessing as mp

    import shard_workers
    backbone, semantic, world = request.param
    out = tmp_path_factory.mktemp("shard")
    mp.spawn(shard_workers.host_plan_worker,
             args=(world, _port(), str(out), "small", ALL, 48, 8, 16, backbone, semantic),
             nprocs=world, join=True)
    return [pickle.load(open(out / f"plan{r}.pkl", "rb")) for r in range(world)]


def test_collectives_host_staged(plans):
    if len(plans) != 2:
        pytest.skip("collective expectations are written for two ranks")
    x = [np.arange(6, dtype=np.float32) + 10 * r for r in range(2)]
    for r, p in enumerate(plans):
        c = p["coll"]
        assert np.array_equal(c["ag"], np.concatenate(x))
        assert np.array_equal(c["rs"], (x[0] + x[1])[3 * r:3 * r + 3])
        # rank q sends [q+1, 2-q] elements (rank-major) -> rank r gets q's block r
        blocks = [np.split(x[q][:3], [q + 1]) for q in range(2)]
        assert np.array_equal(c["a2a"], np.concatenate([blocks[q][r] for q in range(2)]))
        assert np.array_equal(c["ar"], x[0] + x[1])


def test_metadata_identical_on_all_ranks(plans):
    for key in ("anchor_ids", "unit_k", "unit_slots", "cand"):
        for p in plans[1:]:
            assert np.array_equal(plans[0][key], p[key])


def test_owned_candidates_partition(plans):
    G = len(plans)
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
    G = len(plans)
    p0 = plans[0]
    A, S, B, nc = p0["A"], p0["S"], p0["batch"], p0["nc"]
    codes = []
    for r, p in enumerate(plans):
        rows, seg, con = p["rows"], p["seg"], p["contrib"]
        assert np.all(np.diff(rows) > 0)  # ascending local rows
        for i, lr in enumerate(rows):
            ent = lr * G + r  # local row -> global entity
            for code in con[seg[i]:seg[i + 1]]:
                if code < 0:  # anchor row sent at lookup position -code-1
                    assert p["send_rows"][-code - 1] == lr
                else:
                    gslot, j = divmod(code, nc)
                    q, slot = divmod(gslot, S)
                    units = np.where((p0["unit_slots"].reshape(G * B, 3)[q * B:(q + 1) * B] == slot).any(1))[0]
                    assert len(units) == 1
                    assert p0["cand"].reshape(G * B, nc)[q * B + units[0], j] == ent
                codes.append((r, code) if code < 0 else code)  # send positions are per rank
    assert len(codes) == len(set(codes))
    n_anchor = int((p0["anchor_ids"] >= 0).sum())
    n_cand = int(sum(p0["unit_k"][u] * nc for u in range(G * B)))
    assert len(codes) == n_anchor + n_cand


def test_lookup_exchange_lists(plans):
    # the uneven all-to-all carries exactly the owned rows: owner q's block for
    # rank r lists r's anchors owned by q in slot order; r places them by
    # recv_slot / anchor_pos; counts agree on both sides
    G = len(plans)
    p0 = plans[0]
    A = p0["A"]
    anc = p0["anchor_ids"].reshape(G, A)
    for q in range(G):
        for r in range(G):
            assert plans[q]["send_cnt"][r] == plans[r]["recv_cnt"][q]
    for r, p in enumerate(plans):
        assert len(p["send_rows"]) == p["send_cnt"].sum()
        assert len(p["recv_slot"]) == p["recv_cnt"].sum()
        mine = anc[r][anc[r] >= 0]
        assert len(p["recv_slot"]) == len(mine)
        # anchor_pos inverts recv_slot
        for pos, slot in enumerate(p["recv_slot"]):
            assert p["anchor_pos"][slot] == pos
        # receive order = owner-major, slots ascending within an owner
        off = 0
        for q in range(G):
            n = p["recv_cnt"][q]
            slots = p["recv_slot"][off:off + n]
            assert np.all(np.diff(slots) > 0)
            assert np.all(anc[r][slots] % G == q)
            # owner q sends the same rows in the same order
            soff = int(plans[q]["send_cnt"][:r].sum())
            rows = plans[q]["send_rows"][soff:soff + n]
            assert np.array_equal(rows * G + q, anc[r][slots])
            off += n
    # only owned rows travel: total rows sent = anchors of all ranks
    assert sum(len(p["send_rows"]) for p in plans) == int((anc >= 0).sum())
