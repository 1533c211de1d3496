"""Checkpoint blob (resume determinism SPEC.md:576, 755): saving
theta + Adam moments + step and resuming reproduces the uninterrupted run
bit for bit; corrupt / mismatched blobs fail with the SPEC's error kinds."""
import numpy as np
import pytest

import paper_2602_21597_b200 as m
from paper_2602_21597_b200._native import NgdbError

pytestmark = pytest.mark.gpu

ALL = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni", "inp"]


def _names(backbone, info, dim):
    return [s[0] for s in m.param_specs(backbone, info["n_entities"], info["n_relations"], dim)]


@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
def test_resume_is_bit_identical(small_graph, tmp_path, backbone):
    info = small_graph.info()
    dim = 32
    w = m.pattern_weights(ALL)
    steps = [m.PlannedStep(m.Batch.sample(small_graph, w, 64, 8, seed=3, tag=t), backbone, dim)
             for t in range(3)]
    a = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=8,
                 max_queries=64)
    a.run_step(steps[0], 64)
    a.run_step(steps[1], 64)
    path = tmp_path / "ck.ngck"
    a.save_checkpoint(path, config_hash=0xC0FFEE)
    la = a.run_step(steps[2], 64)
    b = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=8,
                 max_queries=64, seed=99)  # different init: everything comes from the blob
    assert b.load_checkpoint(path, config_hash=0xC0FFEE) == 2
    lb = b.run_step(steps[2], 64)
    np.testing.assert_array_equal(la, lb)
    for n in _names(backbone, info, dim):
        for pre in ("", "m:", "v:"):
            np.testing.assert_array_equal(a.download(pre + n), b.download(pre + n))


def test_checkpoint_errors(small_graph, tmp_path):
    info = small_graph.info()
    a = m.Engine("gqe", info["n_entities"], info["n_relations"], dim=16, n_neg=4, max_queries=8)
    path = tmp_path / "ck.ngck"
    a.save_checkpoint(path, config_hash=7)
    with pytest.raises(NgdbError) as e:
        a.load_checkpoint(path, config_hash=8)
    assert e.value.kind == "ConfigError"
    q = m.Engine("q2b", info["n_entities"], info["n_relations"], dim=16, n_neg=4, max_queries=8)
    with pytest.raises(NgdbError) as e:  # BackboneMismatch
        q.load_checkpoint(path)
    assert e.value.kind == "ConfigError"
    raw = bytearray(path.read_bytes())
    raw[100] ^= 0xFF
    bad = tmp_path / "bad.ngck"
    bad.write_bytes(bytes(raw))
    with pytest.raises(NgdbError) as e:
        a.load_checkpoint(bad)
    assert e.value.kind == "DomainError"
    assert a.load_checkpoint(path) == 0  # hash 0: not checked


def test_sharded_blob_loads_only_into_its_rank(tmp_path):
    # a row-sharded context's blob holds only its e mod G rows; it
    # records (world, rank) and refuses any other slot, even when shapes match
    import ctypes as C

    from paper_2602_21597_b200._native import ModelDesc, check, lib

    def ctx(world, rank):
        d = ModelDesc(1, 200, 5, 16, 8, 0, 12.0, 0.02, 1e-4, 0.9, 0.999, 1e-8, 512, 64, world,
                      rank)
        h = C.c_void_p()
        check(lib.ngdb_ctx_create(C.byref(d), 0, C.byref(h)))
        return h

    r0, r1, solo = ctx(2, 0), ctx(2, 1), ctx(1, 0)
    try:
        p = str(tmp_path / "r0.ngck").encode()
        check(lib.ngdb_checkpoint_save(r0, p, 0, 3))
        st = C.c_int64()
        check(lib.ngdb_checkpoint_load(r0, p, 0, C.byref(st)))
        assert st.value == 3
        for other in (r1, solo):  # 200 entities, G = 2: rank 1 has the same 100-row shape
            with pytest.raises(NgdbError, match="rank 0 of 2"):
                check(lib.ngdb_checkpoint_load(other, p, 0, C.byref(st)))
    finally:
        for h in (r0, r1, solo):
            lib.ngdb_ctx_destroy(h)
