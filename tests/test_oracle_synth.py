"""The oracle's own synthetic-KG and PTE-store generators (oracle/src/synth.cpp,
used by bench.py's CPU reference arm so that it never loads the product library)
produce exactly the product's inputs."""
import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m


def _sorted(t):  # the product's graph hands its splits back sorted by (h, r, t)
    t = np.asarray(t)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


@pytest.mark.parametrize("shape", ["tiny", "small", "fb15k-237", "nell995"])
def test_synthetic_triples_identical(shape):
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    assert O.synth_info(shape) == info
    for mine, theirs in zip(O.synth_triples(shape, 1), (g.triples(0), g.triples(1), g.triples(2))):
        assert np.array_equal(_sorted(mine), _sorted(theirs))


@pytest.mark.slow
def test_synthetic_triples_identical_wikikg2():
    g = m.Graph.synthetic("wikikg2", 1)
    for mine, theirs in zip(O.synth_triples("wikikg2", 1), (g.triples(0), g.triples(1),
                                                            g.triples(2))):
        assert np.array_equal(_sorted(mine), _sorted(theirs))


def test_semantic_store_identical():
    assert np.array_equal(O.semantic_store(300, 48, seed=5), m.semantic_store(300, 48, seed=5))
