"""Worker processes of the sharded-step tests (spawned, world_size 2, gloo on
127.0.0.1). Each returns its results through a file in `out_dir`."""
import os
import pickle


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def host_plan_worker(rank, world, port, out_dir, shape, mix, b, k, dim, backbone="q2b",
                     semantic=False):
    """CPU only: plan this rank's batch, exchange metadata, build the owner lists;
    also exercise the host-staged collectives on CPU tensors."""
    dist = _init(rank, world, port)
    import numpy as np
    import torch

    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, plan_shard_step

    comm = Comm()
    g = m.Graph.synthetic(shape, 1)
    batch = m.Batch.sample(g, m.pattern_weights(mix), b, k, seed=3, tag=rank)
    st = plan_shard_step(comm, batch, backbone, dim, semantic=semantic)
    v, s = st.views()
    U = s.world * s.batch
    n_owned = s.unit_off[U]
    plan = {
        "world": s.world, "rank": s.rank, "batch": s.batch, "A": s.max_anchors,
        "S": s.max_slots, "nc": s.n_candidates,
        "anchor_ids": np.ctypeslib.as_array(s.anchor_ids, (s.world * s.max_anchors,)).copy(),
        "unit_k": np.ctypeslib.as_array(s.unit_k, (U,)).copy(),
        "unit_slots": np.ctypeslib.as_array(s.unit_slots, (U * 3,)).copy(),
        "cand": np.ctypeslib.as_array(s.cand, (U * s.n_candidates,)).copy(),
        "unit_off": np.ctypeslib.as_array(s.unit_off, (U + 1,)).copy(),
        "owned": np.ctypeslib.as_array(s.owned, (max(n_owned, 1),))[:n_owned].copy(),
        "rows": np.ctypeslib.as_array(s.rows, (max(s.n_rows, 1),))[: s.n_rows].copy(),
        "seg": np.ctypeslib.as_array(s.seg, (s.n_rows + 1,)).copy(),
    }
    plan["contrib"] = np.ctypeslib.as_array(s.contrib, (max(int(plan["seg"][-1]), 1),))[
        : int(plan["seg"][-1])].copy()
    from paper_2602_21597_b200.sharded import _arr
    plan["send_cnt"], plan["recv_cnt"] = _arr(s.send_cnt, s.world), _arr(s.recv_cnt, s.world)
    plan["send_rows"] = _arr(s.send_rows, s.n_send)
    plan["recv_slot"] = _arr(s.recv_slot, s.n_recv)
    plan["anchor_pos"] = _arr(s.anchor_pos, s.n_anchor_pos)
    plan["n_score_slots"] = v.n_score_slots
    # collectives (host-staged path) on CPU tensors (their expectations are
    # written for two ranks)
    if world != 2:
        with open(os.path.join(out_dir, f"plan{rank}.pkl"), "wb") as f:
            pickle.dump(plan, f)
        dist.barrier()
        dist.destroy_process_group()
        return
    x = torch.arange(6, dtype=torch.float32) + 10 * rank
    ag = torch.zeros(6 * world)
    comm.all_gather(ag, x)
    rs = torch.zeros(6 // world)
    comm.reduce_scatter(rs, x)
    # uneven all-to-all: rank r sends r+1 elements to rank 0 and 2-r to rank 1
    sc = [rank + 1, 2 - rank]
    rc = [q + 1 if rank == 0 else 2 - q for q in range(world)]
    a2a = torch.zeros(sum(rc))
    comm.all_to_all_v(a2a, x, sc, rc)
    ar = x.clone()
    comm.all_reduce(ar)
    plan["coll"] = {"ag": ag.numpy(), "rs": rs.numpy(), "a2a": a2a.numpy(), "ar": ar.numpy()}
    with open(os.path.join(out_dir, f"plan{rank}.pkl"), "wb") as f:
        pickle.dump(plan, f)
    dist.barrier()
    dist.destroy_process_group()


def gpu_step_worker(rank, world, port, out_dir, shape, mix, b, k, dim, steps, backbone, sdim=0):
    """Two ranks sharing GPU 0: the row-sharded step through ngdb_shard_*
    (sdim > 0: FuseSemantic over the synthetic store of that width)."""
    dist = _init(rank, world, port)
    import numpy as np

    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine

    comm = Comm()
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    eng = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=k,
                        max_queries=b, device=0, debug=True, semantic=store)
    w = m.pattern_weights(mix)
    res = {"loss": [], "batches": []}
    for step in range(1, steps + 1):
        batch = m.Batch.from_arrays(_load_batch(out_dir, step, rank))
        res["loss"].append(eng.train_step(batch))
    specs = m.param_specs(backbone, info["n_entities"], info["n_relations"], dim, sdim)
    res["params"] = {n: eng.download(n) for n, *_ in specs}
    res["grads"] = {n: eng.download("g:" + n) for n, *_ in specs}
    with open(os.path.join(out_dir, f"gpu{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def _load_batch(out_dir, step, rank):
    with open(os.path.join(out_dir, f"batch_{step}_{rank}.pkl"), "rb") as f:
        return pickle.load(f)


def graph_replay_worker(rank, world, port, out_dir, shape, mix, b, k, dim, steps, backbone,
                        sdim=0):
    """One NCCL rank on GPU 0: the same steps run eagerly on one engine and as
    captured CUDA graphs (stages + collectives) replayed on another."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine, plan_shard_step

    comm = Comm(transport="nccl")  # the context's own NCCL communicator
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    w = m.pattern_weights(mix)
    batches = [m.Batch.sample(g, w, b, k, seed=3, tag=s * world + rank) for s in range(steps + 1)]
    plans = [plan_shard_step(comm, bt, backbone, dim, semantic=sdim > 0) for bt in batches]
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    out = {}
    for mode in ("eager", "graph"):
        eng = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                            n_neg=k, max_queries=b, semantic=store)
        eng.run(plans[0], 1)  # communicator warm-up (eager)
        if mode == "eager":
            for s in range(1, steps + 1):
                eng.run(plans[s], s + 1)
        else:
            graphs = eng.capture(plans[1:])
            for s in range(1, steps + 1):
                graphs[s - 1].replay(s + 1)
        torch.cuda.synchronize()
        out[mode] = {n: eng.download(n) for n, *_ in m.param_specs(backbone, info["n_entities"],
                                                                  info["n_relations"], dim, sdim)}
    with open(os.path.join(out_dir, f"graph{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.destroy_process_group()


def train_loop_worker(rank, world, port, out_dir, shape, mix, b, k, dim, steps, backbone,
                      sdim=0):
    """One NCCL rank on GPU 0: ShardedEngine.train (pipelined: planning
    threads, async loss read-back) vs the same batches step by step."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np

    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine, plan_shard_step

    comm = Comm(transport="nccl")
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    w = m.pattern_weights(mix)
    tag = lambda s: (s + 1) * world + rank  # noqa: E731
    out = {}
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    specs = m.param_specs(backbone, info["n_entities"], info["n_relations"], dim, sdim)
    eng = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                        n_neg=k, max_queries=b, semantic=store)
    seq = []
    for s in range(steps):
        batch = m.Batch.sample(g, w, b, k, seed=3, tag=tag(s))
        seq.append(float(np.sum(eng.run(plan_shard_step(comm, batch, backbone, dim,
                                                         semantic=sdim > 0)),
                                dtype=np.float64)))
    out["seq"] = {n: eng.download(n) for n, *_ in specs}
    eng2 = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                         n_neg=k, max_queries=b, semantic=store)
    sums = eng2.train(g, w, steps, b, k, tag, producers=3)
    torch.cuda.synchronize()
    out["loop"] = {n: eng2.download(n) for n, *_ in specs}
    out["seq_sums"] = seq
    out["loop_sums"] = sums.tolist()
    # the native loop (libngdb threads + the metadata communicator), same batches:
    # tag((s+1)*world + rank) == (first_tag + s) * world + rank with first_tag = 1
    eng3 = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                         n_neg=k, max_queries=b, semantic=store)
    nsums = eng3.train_native(g, w, steps, b, k, first_tag=1, producers=3)
    torch.cuda.synchronize()
    out["native"] = {n: eng3.download(n) for n, *_ in specs}
    out["native_sums"] = nsums.tolist()
    with open(os.path.join(out_dir, f"loop{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.destroy_process_group()


def transport_worker(rank, world, port, out_dir, shape, mix, b, k, dim, steps, backbone, sdim=0):
    """One rank on GPU 0: the same steps through the context's NCCL transport
    (ngdb_shard_step_exec: uneven all-to-alls, all-gather, reduce-scatter,
    all-reduce inside libngdb) and through the host-staged transport."""
    import torch
    dist = _init(rank, world, port)
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine

    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    w = m.pattern_weights(mix)
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    out = {}
    for transport in ("host", "nccl"):
        comm = Comm(transport=transport)
        eng = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                            n_neg=k, max_queries=b, semantic=store)
        losses = []
        for s in range(steps):
            batch = m.Batch.sample(g, w, b, k, seed=3, tag=(s + 1) * world + rank)
            losses.append(eng.train_step(batch))
        torch.cuda.synchronize()
        out[transport] = {"loss": losses,
                          "params": {n: eng.download(n) for n, *_ in m.param_specs(
                              backbone, info["n_entities"], info["n_relations"], dim, sdim)}}
        del eng
    with open(os.path.join(out_dir, f"transport{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.destroy_process_group()


def python_sums_worker(rank, world, port, out_dir, shape, mix, b, k, dim, steps, backbone):
    """One rank on GPU 0 through ShardedEngine (NCCL transport): per-step loss
    sums of the batches tagged (s+1)*world + rank (the C++ driver's convention)."""
    import numpy as np
    dist = _init(rank, world, port)
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine

    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    w = m.pattern_weights(mix)
    eng = ShardedEngine(Comm(transport="nccl"), backbone, info["n_entities"], info["n_relations"],
                        dim=dim, n_neg=k, max_queries=b)
    sums = [float(np.sum(eng.train_step(m.Batch.sample(g, w, b, k, seed=3,
                                                         tag=(s + 1) * world + rank)),
                         dtype=np.float64)) for s in range(steps)]
    with open(os.path.join(out_dir, f"pysums{rank}.pkl"), "wb") as f:
        pickle.dump(sums, f)
    dist.destroy_process_group()


def wikikg2_worker(rank, world, port, out_dir, b, k, dim, steps):
    """One NCCL rank on GPU 0: the C5 row-sharded step on the wikikg2-shaped
    graph; per-query losses of `steps` steps (batch s: tag (s+1)*world + rank)."""
    import numpy as np
    dist = _init(rank, world, port)
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine

    g = m.Graph.synthetic("wikikg2", 1)
    info = g.info()
    w = m.pattern_weights(m.PATTERNS)
    eng = ShardedEngine(Comm(transport="nccl"), "q2b", info["n_entities"], info["n_relations"],
                        dim=dim, n_neg=k, max_queries=b)
    out = {"loss": [], "arrays": []}
    for s in range(steps):
        bt = m.Batch.sample(g, w, b, k, seed=3, tag=(s + 1) * world + rank)
        out["arrays"].append(bt.arrays())
        out["loss"].append(eng.train_step(bt))
    out["relation"] = eng.download("relation")
    with open(os.path.join(out_dir, f"wiki{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.destroy_process_group()


def packed_begin_worker(rank, world, port, out_dir):
    """One rank: ngdb_shard_begin_packed with a wrong size, then a packed step
    and the same step through ngdb_shard_begin on a fresh engine."""
    import ctypes as C

    import numpy as np
    import torch

    dist = _init(rank, world, port)
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200._native import NgdbError, ShardBuffers, check, lib
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine, plan_shard_step

    g = m.Graph.synthetic("small", 1)
    info = g.info()
    comm = Comm()
    batch = m.Batch.sample(g, m.pattern_weights(["1p", "2i", "2u"]), 48, 8, seed=3, tag=5)
    st = plan_shard_step(comm, batch, "q2b", 16)
    v, s = st.views()
    n_plan = int(lib.ngdb_plan_packed_size(C.byref(v)))
    n_shard = int(lib.ngdb_shard_packed_size(C.byref(s)))
    pk = np.zeros(n_plan + n_shard, np.int32)
    P32 = C.POINTER(C.c_int32)
    check(lib.ngdb_plan_pack(C.byref(v), pk.ctypes.data_as(P32), n_plan))
    check(lib.ngdb_shard_pack(C.byref(s), pk[n_plan:].ctypes.data_as(P32), n_shard))
    out = {}
    eng = ShardedEngine(comm, "q2b", info["n_entities"], info["n_relations"], dim=16, n_neg=8,
                        max_queries=48)
    b = ShardBuffers()
    try:
        check(lib.ngdb_shard_begin_packed(eng.handle, C.byref(v), pk.ctypes.data_as(P32), n_plan + 1,
                                          C.byref(s), pk[n_plan:].ctypes.data_as(P32), n_shard,
                                          C.byref(b)))
        out["bad_kind"] = "accepted"
    except NgdbError as e:
        out["bad_kind"] = e.kind
    # a correct packed begin, then the host-staged stages (world 1)
    from paper_2602_21597_b200.sharded import _host_stages
    with torch.cuda.stream(eng.stream):
        check(lib.ngdb_shard_begin_packed(eng.handle, C.byref(v), pk.ctypes.data_as(P32), n_plan,
                                          C.byref(s), pk[n_plan:].ctypes.data_as(P32), n_shard,
                                          C.byref(b)))
        _host_stages(eng, b, np.array(st.counts()[0]), np.array(st.counts()[1]))
        check(lib.ngdb_shard_optimizer(eng.handle, 1))
    losses = np.zeros(st.n_queries, np.float32)
    tot, bad = C.c_double(), C.c_int32()
    check(lib.ngdb_step_end(eng.handle, losses.ctypes.data_as(C.POINTER(C.c_float)), st.n_queries,
                            C.byref(tot), C.byref(bad)))
    out["loss_packed"] = losses
    eng2 = ShardedEngine(comm, "q2b", info["n_entities"], info["n_relations"], dim=16, n_neg=8,
                         max_queries=48)
    out["loss_plain"] = eng2.run(st, 1)
    with open(os.path.join(out_dir, f"packed{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()
