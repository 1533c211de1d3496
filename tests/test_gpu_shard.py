"""Row-sharded step on the GPU: two ranks share GPU 0 over gloo
(host-staged collectives; NCCL needs one GPU per rank). Every per-query loss,
the summed gradients and the post-Adam parameters must match the oracle's
"G sub-batches" mode — each rank's batch scheduled independently, gradients
summed, one Adam step (SURVEY §8(e) parity) — at the 1e-4 bar."""
import pickle
import socket

import numpy as np
import pytest

import paper_2602_21597_b200 as m
from parity import check_all, tie_free

pytestmark = pytest.mark.gpu
ALL = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni", "inp"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("backbone,dim,b,k,steps,sdim,G", [
    ("q2b", 32, 64, 16, 1, 0, 2), ("gqe", 16, 48, 8, 2, 0, 2), ("q2b", 400, 128, 32, 2, 0, 2),
    ("betae", 16, 64, 16, 2, 0, 2), ("betae", 400, 64, 32, 1, 0, 2),
    # FuseSemantic: store rows sharded with the entity rows, fused rows exchanged
    ("gqe", 16, 64, 16, 2, 24, 2), ("q2b", 400, 64, 32, 1, 768, 2), ("betae", 16, 48, 16, 2, 24, 2),
    # three ranks: every exchange has two remote peers
    ("q2b", 32, 48, 16, 2, 0, 3), ("gqe", 16, 48, 16, 1, 24, 3)])
def test_sharded_step_matches_oracle_sub_batches(small_graph, tmp_path, backbone, dim, b, k, steps,
                                                 sdim, G):
    import torch.multiprocessing as mp

    import oracle as O
    import shard_workers
    info = small_graph.info()
    ne, nr = info["n_entities"], info["n_relations"]
    w = m.pattern_weights(ALL)
    store = m.semantic_store(ne, sdim, seed=5) if sdim else None
    om = O.OracleModel(backbone, ne, nr, dim, k, precision=64)
    if sdim:
        om.set_semantic(store)
    om.init(2)
    batches = []
    for step in range(1, steps + 1):
        per_rank = []
        for r in range(G):
            bt = m.Batch.sample(small_graph, w, b, k, seed=3, tag=step * G + r)
            if step == 1:  # certify kink-free queries at the initial parameters
                probe = O.OracleModel(backbone, ne, nr, dim, k, precision=64)
                if sdim:
                    probe.set_semantic(store)
                probe.init(2)
                bt, _ = tie_free(bt, probe, 512, 1)
            arr = bt.arrays()
            per_rank.append(arr)
            with open(tmp_path / f"batch_{step}_{r}.pkl", "wb") as f:
                pickle.dump(arr, f)
        batches.append(per_rank)
    mp.spawn(shard_workers.gpu_step_worker,
             args=(G, _port(), str(tmp_path), "small", ALL, b, k, dim, steps, backbone, sdim),
             nprocs=G, join=True)
    outs = [pickle.load(open(tmp_path / f"gpu{r}.pkl", "rb")) for r in range(G)]

    res = {"loss": [], "grads": {}, "params": {}, "weak": {}}
    for step in range(1, steps + 1):
        refs = om.step_multi(batches[step - 1], step=step)
        for r in range(G):
            res["loss"].append((outs[r]["loss"][step - 1], refs[r]))
    specs = m.param_specs(backbone, ne, nr, dim, sdim)
    for name, rows, cols, sparse in specs:
        def full(key):
            if name != "entity":
                return outs[0][key][name]
            t = np.zeros((rows, cols), np.float32)
            for r in range(G):
                t[r::G] = outs[r][key][name]
            return t
        res["grads"][name] = (full("grads"), om.get("g:" + name, (rows, cols)))
        res["params"][name] = (full("params"), om.get(name, (rows, cols)))
        if name != "entity":  # replicated tensors are identical on every rank
            for o in outs[1:]:
                assert np.array_equal(outs[0]["params"][name], o["params"][name]), name
    check_all(res, allow_frac=0.0, steps=steps)


@pytest.mark.parametrize("backbone,dim,sdim", [("q2b", 32, 0), ("gqe", 16, 0), ("betae", 32, 0),
                                              ("gqe", 32, 24), ("betae", 16, 24)])
def test_sharded_graph_replay_matches_eager(tmp_path, backbone, dim, sdim):
    # the resident sharded step (stages + NCCL collectives captured in one CUDA
    # graph, bench.py --config c5) updates the parameters bit-identically to the
    # eager stage-by-stage run
    import torch.multiprocessing as mp

    import shard_workers
    mp.spawn(shard_workers.graph_replay_worker,
             args=(1, _port(), str(tmp_path), "small", ALL, 64, 16, dim, 3, backbone, sdim),
             nprocs=1, join=True)
    out = pickle.load(open(tmp_path / "graph0.pkl", "rb"))
    for name, v in out["eager"].items():
        assert np.array_equal(v, out["graph"][name]), name


@pytest.mark.parametrize("backbone,sdim", [("q2b", 0), ("gqe", 24)])
def test_sharded_train_loop_matches_steps(tmp_path, backbone, sdim):
    # ShardedEngine.train (bench.py --config c5 e2e) = the same batches run
    # step by step: identical parameters and per-step losses
    import torch.multiprocessing as mp

    import shard_workers
    mp.spawn(shard_workers.train_loop_worker,
             args=(1, _port(), str(tmp_path), "small", ALL, 64, 16, 32, 4, backbone, sdim),
             nprocs=1, join=True)
    out = pickle.load(open(tmp_path / "loop0.pkl", "rb"))
    for name, v in out["seq"].items():
        assert np.array_equal(v, out["loop"][name]), name
        assert np.array_equal(v, out["native"][name]), name  # ngdb_shard_train_run
    np.testing.assert_allclose(out["loop_sums"], out["seq_sums"], rtol=1e-12)
    np.testing.assert_allclose(out["native_sums"], out["seq_sums"], rtol=1e-12)


@pytest.mark.parametrize("backbone,dim,sdim", [("q2b", 400, 0), ("gqe", 32, 0), ("betae", 32, 0),
                                              ("q2b", 32, 24)])
def test_nccl_transport_matches_host_transport(tmp_path, backbone, dim, sdim):
    # the libngdb NCCL path (ngdb_shard_step_exec) and the host-staged path run
    # the same stages over the same exchange layouts: bit-identical results
    import torch.multiprocessing as mp

    import shard_workers
    mp.spawn(shard_workers.transport_worker,
             args=(1, _port(), str(tmp_path), "small", ALL, 64, 16, dim, 3, backbone, sdim),
             nprocs=1, join=True)
    out = pickle.load(open(tmp_path / "transport0.pkl", "rb"))
    for a, b in zip(out["host"]["loss"], out["nccl"]["loss"]):
        assert np.array_equal(a, b)
    for name, v in out["host"]["params"].items():
        assert np.array_equal(v, out["nccl"]["params"][name]), name


def test_cpp_driver_matches_python_engine(tmp_path):
    # tools/cpp/sharded_train.cpp drives the whole sharded step from C++ alone
    # (libngdb's NCCL communicator, packed metadata all-gather over NCCL, owner
    # lists, ngdb_shard_step_exec): the same per-step losses as ShardedEngine
    import subprocess
    from pathlib import Path

    import torch.multiprocessing as mp

    import shard_workers
    exe = Path(m.__file__).parent / "_lib" / "sharded_train"
    assert exe.exists(), "make examples"
    r = subprocess.run([str(exe), "1", "0", "0", str(tmp_path / "nccl.id"), "small", "3", "64",
                        "16", "32"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    cpp = [float(line.split()[2]) for line in r.stdout.splitlines() if line.startswith("step")]
    mp.spawn(shard_workers.python_sums_worker,
             args=(1, _port(), str(tmp_path), "small", ALL, 64, 16, 32, 3, "q2b"),
             nprocs=1, join=True)
    py = pickle.load(open(tmp_path / "pysums0.pkl", "rb"))
    assert len(cpp) == 3 and cpp == py, (cpp, py)


def test_c5_wikikg2_sharded_step_vs_oracle(tmp_path):
    # the C5 row-sharded step (one NCCL rank, libngdb
    # collectives) on the wikikg2-shaped graph (2.5 M entities) at the
    # benchmark's per-rank shape (B = 512, K = 128, d = 400) against the oracle
    # (f32, same seeds): every per-query loss of two steps within 1e-4 (step 2
    # carries step 1's Adam update of the 2.5 M-row table), and the replicated
    # relation table after the second update
    import torch.multiprocessing as mp

    import oracle as O
    import shard_workers
    from parity import rel_close
    b, k, dim, steps = 512, 128, 400, 2
    mp.spawn(shard_workers.wikikg2_worker, args=(1, _port(), str(tmp_path), b, k, dim, steps),
             nprocs=1, join=True)
    out = pickle.load(open(tmp_path / "wiki0.pkl", "rb"))
    info = O.synth_info("wikikg2")
    om = O.OracleModel("q2b", info["n_entities"], info["n_relations"], dim, k, precision=32)
    om.init(2)
    for s in range(steps):
        a = out["arrays"][s]
        ref = om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, step=s + 1)
        ok, nbad, worst = rel_close(out["loss"][s], ref)
        assert ok, f"step {s + 1}: {nbad} of {b} losses beyond 1e-4 (worst {worst:.3e})"
    rel = om.get("relation", out["relation"].shape)
    ok, nbad, worst = rel_close(out["relation"], rel)
    assert ok, f"relation: {nbad} beyond 1e-4 (worst {worst:.3e})"


def test_packed_shard_begin_rejects_wrong_sizes(small_graph, tmp_path):
    # ngdb_shard_begin_packed validates the caller's packed blob sizes against
    # the plans (ShapeMismatch), and a correctly packed step runs like
    # ngdb_shard_begin (same losses)
    import ctypes as C

    import torch.multiprocessing as mp

    import shard_workers
    mp.spawn(shard_workers.packed_begin_worker, args=(1, _port(), str(tmp_path)), nprocs=1,
             join=True)
    out = pickle.load(open(tmp_path / "packed0.pkl", "rb"))
    assert out["bad_kind"] == "ShapeMismatch"
    assert np.array_equal(out["loss_packed"], out["loss_plain"])
