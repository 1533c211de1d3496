"""ORACLE — test infrastructure only.

ctypes binding of oracle/_build/liboracle.so, the independent CPU restatement of
the reference training step (see oracle/src/oracle_internal.hpp for what pins
it). Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "_build" / "liboracle.so"
if not _LIB.exists():
    raise ImportError(f"{_LIB} missing: run `make -C oracle`")
lib = C.CDLL(str(_LIB))

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER
_SIG = {
    "oracle_last_error": (C.c_char_p, []),
    "oracle_rng_next": (u64, [u64, i64, i32]),
    "oracle_rng_below": (C.c_int, [u64, P(u64), i32, i32, P(u64)]),
    "oracle_rng_uniform": (C.c_int, [u64, i32, f64, f64, P(f64)]),
    "oracle_rng_gaussian": (C.c_int, [u64, i32, P(f64)]),
    "oracle_fnv1a64": (u64, [C.c_char_p, i64]),
    "oracle_graph_create": (C.c_int, [i32, i32, P(i32), i64, P(i32), i64, P(i32), i64,
                                      P(C.c_void_p)]),
    "oracle_graph_answer": (C.c_int, [C.c_void_p, i32, i32, P(i32), P(i32), P(i32), i64, P(i64)]),
    "oracle_graph_destroy": (C.c_int, [C.c_void_p]),
    "oracle_sample_batch": (C.c_int, [C.c_void_p, P(f64), i32, i32, u64, u64, P(i32), P(i32),
                                      P(i32), P(i32), P(i32)]),
    "oracle_build_dag": (C.c_int, [i32, P(i32), P(i32), P(i32), P(i32), i64, P(i32), P(i32),
                                   P(i32), i64, P(i32)]),
    "oracle_model_create": (C.c_int, [i32, i32, i32, i32, i32, f64, f64, f64, i32,
                                      P(C.c_void_p)]),
    "oracle_model_init": (C.c_int, [C.c_void_p, u64]),
    "oracle_model_set": (C.c_int, [C.c_void_p, C.c_char_p, P(C.c_float), i64]),
    "oracle_model_get": (C.c_int, [C.c_void_p, C.c_char_p, P(f64), i64]),
    "oracle_model_step": (C.c_int, [C.c_void_p, i32, P(i32), P(i32), P(i32), P(i32), P(i32), i32,
                                    i64, i32, i32, i32, P(f64)]),
    "oracle_model_trace_json": (C.c_int, [C.c_void_p, i32, C.c_char_p, i64, P(i64)]),
    "oracle_model_destroy": (C.c_int, [C.c_void_p]),
    "oracle_model_margins": (C.c_int, [C.c_void_p, P(f64), i32]),
    "oracle_q2b_distance": (f64, [P(f64), P(f64), P(f64), i32, f64]),
    "oracle_loss": (f64, [f64, f64, P(f64), i32]),
    "oracle_lgamma": (f64, [f64]),
    "oracle_model_step_multi": (C.c_int, [C.c_void_p, i32, P(i32), P(i32), P(i32), P(i32), P(i32),
                                          P(i32), i32, i64, i32, P(f64)]),
    "oracle_model_set_semantic": (C.c_int, [C.c_void_p, i32, P(C.c_float), i64]),
    "oracle_model_qmargins": (C.c_int, [C.c_void_p, P(f64), i32]),
    "oracle_model_set_dev_tau": (C.c_int, [C.c_void_p, f64]),
    "oracle_model_dev": (C.c_int, [C.c_void_p, C.c_char_p, P(f64), i64]),
    "oracle_synth_shape": (C.c_int, [C.c_char_p, P(i32), P(i32), P(i64)]),
    "oracle_synth_triples": (C.c_int, [C.c_char_p, u64, P(i32)]),
    "oracle_semantic_store": (C.c_int, [i32, i32, u64, P(C.c_float)]),
    "oracle_set_threads": (C.c_int, [i32]),
    "oracle_digamma": (f64, [f64]),
    "oracle_trigamma": (f64, [f64]),
    "oracle_beta_kl": (f64, [f64, f64, f64, f64]),
}
for _n, (_r, _a) in _SIG.items():
    _f = getattr(lib, _n)
    _f.restype, _f.argtypes = _r, _a

BACKBONES = {"gqe": 0, "q2b": 1, "betae": 2}


def _p(a, t):
    return a.ctypes.data_as(P(t))


def _check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib.oracle_last_error().decode())


def set_threads(n):
    """OpenMP threads of the oracle's row-parallel loops (results do not depend on it)."""
    lib.oracle_set_threads(int(n))


def synth_info(shape):
    ne, nr, c = i32(), i32(), (i64 * 3)()
    _check(lib.oracle_synth_shape(shape.encode(), C.byref(ne), C.byref(nr), c))
    return {"n_entities": ne.value, "n_relations": nr.value, "n_train": c[0], "n_valid": c[1],
            "n_test": c[2]}


def synth_triples(shape, seed=1):
    """(train, valid, test) [n][3] int32 of the synthetic benchmark KG (oracle/src/synth.cpp)."""
    info = synth_info(shape)
    n = info["n_train"] + info["n_valid"] + info["n_test"]
    out = np.zeros((n, 3), np.int32)
    _check(lib.oracle_synth_triples(shape.encode(), seed, _p(out, i32)))
    a, b = info["n_train"], info["n_train"] + info["n_valid"]
    return out[:a], out[a:b], out[b:]


def semantic_store(n_entities, dim=768, seed=5):
    out = np.zeros((n_entities, dim), np.float32)
    _check(lib.oracle_semantic_store(n_entities, dim, seed, _p(out, C.c_float)))
    return out


class OracleGraph:
    @classmethod
    def synthetic(cls, shape, seed=1):
        info = synth_info(shape)
        return cls(info["n_entities"], info["n_relations"], *synth_triples(shape, seed))

    def __init__(self, n_entities, n_relations, train, valid=None, test=None):
        def arr(x):
            return np.ascontiguousarray(np.zeros((0, 3)) if x is None else x, dtype=np.int32)
        tr, va, te = arr(train), arr(valid), arr(test)
        self.n_entities = n_entities
        self._h = C.c_void_p()
        _check(lib.oracle_graph_create(n_entities, n_relations, _p(tr, i32), len(tr), _p(va, i32),
                                       len(va), _p(te, i32), len(te), C.byref(self._h)))

    def answer(self, pattern_idx, anchors, relations, full=False):
        a = np.array(list(anchors) + [-1] * 3, dtype=np.int32)[:3]
        r = np.array(list(relations) + [-1] * 4, dtype=np.int32)[:4]
        out = np.zeros(self.n_entities, dtype=np.int32)
        n = C.c_int64()
        _check(lib.oracle_graph_answer(self._h, int(full), pattern_idx, _p(a, i32), _p(r, i32),
                                       _p(out, i32), len(out), C.byref(n)))
        return out[: n.value].copy()

    def sample(self, weights, b, n_neg, seed=3, tag=0):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        pat = np.zeros(b, np.int32)
        anc = np.zeros((b, 3), np.int32)
        rel = np.zeros((b, 4), np.int32)
        pos = np.zeros(b, np.int32)
        neg = np.zeros((b, n_neg), np.int32)
        _check(lib.oracle_sample_batch(self._h, _p(w, f64), b, n_neg, seed, tag, _p(pat, i32),
                                       _p(anc, i32), _p(rel, i32), _p(pos, i32), _p(neg, i32)))
        return pat, anc, rel, pos, neg

    def __del__(self):
        if getattr(self, "_h", None):
            lib.oracle_graph_destroy(self._h)


def build_dag(patterns, anchors, relations):
    b = len(patterns)
    cap = 40 * b * 11
    out = np.zeros(cap, np.int32)
    edges = np.zeros(80 * b, np.int32)
    n, nf, ne = C.c_int32(), C.c_int32(), C.c_int32()
    pa = [np.ascontiguousarray(x, dtype=np.int32) for x in (patterns, anchors, relations)]
    _check(lib.oracle_build_dag(b, _p(pa[0], i32), _p(pa[1], i32), _p(pa[2], i32), _p(out, i32),
                                cap, C.byref(n), C.byref(nf), _p(edges, i32), len(edges),
                                C.byref(ne)))
    return out[: n.value * 11].reshape(n.value, 11), nf.value, edges[: 2 * ne.value].reshape(-1, 2)


class OracleModel:
    def __init__(self, backbone, n_entities, n_relations, dim, n_neg, gamma=12.0,
                 alpha_box=0.02, lr=1e-4, precision=64):
        self._h = C.c_void_p()
        self.backbone, self.dim = backbone, dim
        self.n_entities, self.n_relations = n_entities, n_relations
        _check(lib.oracle_model_create(BACKBONES[backbone], n_entities, n_relations, dim, n_neg,
                                       gamma, alpha_box, lr, precision, C.byref(self._h)))

    def set_semantic(self, store):
        """Frozen semantic store [n_entities][d_l] + fusion params (before init)."""
        a = np.ascontiguousarray(store, dtype=np.float32)
        _check(lib.oracle_model_set_semantic(self._h, a.shape[1], _p(a, C.c_float), a.size))

    def init(self, seed=2):
        _check(lib.oracle_model_init(self._h, seed))

    def set(self, name, value):
        a = np.ascontiguousarray(value, dtype=np.float32)
        _check(lib.oracle_model_set(self._h, name.encode(), _p(a, C.c_float), a.size))

    def get(self, name, shape):
        out = np.zeros(shape, dtype=np.float64)
        _check(lib.oracle_model_get(self._h, name.encode(), _p(out, f64), out.size))
        return out

    def step(self, patterns, anchors, relations, positives, negatives, b_max=512, step=1,
             executor=0, adam=0, eager=True):
        b = len(patterns)
        arrs = [np.ascontiguousarray(x, dtype=np.int32)
                for x in (patterns, anchors, relations, positives, negatives)]
        losses = np.zeros(b, np.float64)
        _check(lib.oracle_model_step(self._h, b, *[_p(x, i32) for x in arrs], b_max, step,
                                     executor, adam, int(eager), _p(losses, f64)))
        return losses

    def step_multi(self, batches, b_max=512, step=1, adam=0):
        """Sub-batches (one per rank) scheduled independently, gradients summed,
        one Adam step: the parity reference of the row-sharded step."""
        sizes = np.array([len(x.patterns) for x in batches], np.int32)
        cat = [np.ascontiguousarray(np.concatenate([getattr(x, f) for x in batches]), dtype=np.int32)
               for f in ("patterns", "anchors", "relations", "positives", "negatives")]
        losses = np.zeros(int(sizes.sum()), np.float64)
        _check(lib.oracle_model_step_multi(self._h, len(batches), _p(sizes, i32),
                                           *[_p(x, i32) for x in cat], b_max, step, adam,
                                           _p(losses, f64)))
        return np.split(losses, np.cumsum(sizes)[:-1])

    def margins(self, b):
        out = np.zeros(b, np.float64)
        _check(lib.oracle_model_margins(self._h, _p(out, f64), b))
        return out

    def set_dev_tau(self, tau):
        """precision=65 only: kinks within tau inject fp32 deviation bounds."""
        _check(lib.oracle_model_set_dev_tau(self._h, float(tau)))

    def dev(self, name, shape):
        out = np.zeros(shape, dtype=np.float64)
        _check(lib.oracle_model_dev(self._h, name.encode(), _p(out, f64), out.size))
        return out

    def qmargins(self, b):
        out = np.zeros(b, np.float64)
        _check(lib.oracle_model_qmargins(self._h, _p(out, f64), b))
        return out

    def trace(self, with_nodes=False):
        n = C.c_int64()
        _check(lib.oracle_model_trace_json(self._h, int(with_nodes), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.oracle_model_trace_json(self._h, int(with_nodes), buf, n.value + 1, C.byref(n)))
        return json.loads(buf.value.decode())

    def __del__(self):
        if getattr(self, "_h", None):
            lib.oracle_model_destroy(self._h)


def q2b_distance(v, c, o, alpha=0.02):
    v, c, o = (np.ascontiguousarray(x, dtype=np.float64) for x in (v, c, o))
    return lib.oracle_q2b_distance(_p(v, f64), _p(c, f64), _p(o, f64), len(v), alpha)


def loss(gamma, d_pos, d_neg):
    dn = np.ascontiguousarray(d_neg, dtype=np.float64)
    return lib.oracle_loss(gamma, d_pos, _p(dn, f64), len(dn))


def lgamma(x):
    return lib.oracle_lgamma(float(x))


def digamma(x):
    return lib.oracle_digamma(float(x))


def trigamma(x):
    return lib.oracle_trigamma(float(x))


def beta_kl(a1, b1, a2, b2):
    return lib.oracle_beta_kl(float(a1), float(b1), float(a2), float(b2))


# ---- evaluator (module `evaluator`) -------------------------
# Pure numpy restatement. Distances follow the backbone formulas (GQE ||v-q||_1,
# SURVEY A-7; Q2B SPEC.md:378) in float32 with the dimensions summed in order
# (np.cumsum is a sequential accumulation), i.e. the rounding of a sequential
# fp32 loop; scores are negated distances.

class TargetFiltered(ValueError):
    """SPEC.md:617 errors: TargetFiltered (target inside its filter set)."""


def filtered_rank(scores, target, filt):
    """1 + |{e not in filter+{target}: s(e) > s(t)}| + floor(ties/2)."""
    filt = set(int(f) for f in filt)
    if int(target) in filt:
        raise TargetFiltered(f"target {target} is in its filter set")
    s = np.asarray(scores)
    st = s[target]
    keep = np.ones(len(s), dtype=bool)
    keep[list(filt)] = False
    keep[target] = False
    better = int(np.count_nonzero(s[keep] > st))
    ties = int(np.count_nonzero(s[keep] == st))
    return 1 + better + ties // 2


def filtered_rank_sorted(scores, target, filt):
    """The SPEC's derived check: rank by sorting the filtered list
    (descending score); ties are the run of equal scores, mean-rank rounded down."""
    filt = set(int(f) for f in filt)
    cand = [e for e in range(len(scores)) if e not in filt]
    order = sorted(cand, key=lambda e: -scores[e])
    st = scores[target]
    first = next(i for i, e in enumerate(order) if scores[e] == st)
    n_eq = sum(1 for e in cand if scores[e] == st) - 1  # equal competitors
    return 1 + first + n_eq // 2


def eval_distances(backbone, ent, q, dim, alpha=0.02, consts=None):
    """[n_ent] float32 distances of every entity row to one query (GQE: q [d];
    Q2B: centre | offset [2d]), summed sequentially over the dimensions.
    BetaE: `ent` is the entity side T [n][2d] and `consts` C [n] of the
    linearised KL (beta_eval_table); the compared value is sum_k fl(q_k T_k)
    (sequential) + C — KL minus the query's own lnB(q), the same for every
    entity."""
    if backbone == "betae":
        t = np.asarray(ent, dtype=np.float32)
        q = np.asarray(q, dtype=np.float32)[None, :2 * dim]
        dot = np.cumsum((t * q).astype(np.float32), axis=1, dtype=np.float32)[:, -1]
        return (dot + np.asarray(consts, np.float32)).astype(np.float32)
    ent = np.asarray(ent, dtype=np.float32)[:, :dim]
    q = np.asarray(q, dtype=np.float32)
    t = np.abs(ent - q[None, :dim])
    if backbone == "gqe":
        return np.cumsum(t, axis=1, dtype=np.float32)[:, -1]
    o = q[None, dim:2 * dim]
    out = np.cumsum(np.maximum(t - o, np.float32(0)), axis=1, dtype=np.float32)[:, -1]
    inn = np.cumsum(np.minimum(t, o), axis=1, dtype=np.float32)[:, -1]
    return out + np.float32(alpha) * inn


def eval_ranks(backbone, ent, queries, targets, filters, dim, alpha=0.02, consts=None):
    return np.array([filtered_rank(-eval_distances(backbone, ent, q, dim, alpha, consts), t, f)
                     for q, t, f in zip(queries, targets, filters)], dtype=np.int64)


def eval_ranks_multi(backbone, ent, embeddings, targets, filters, dim, alpha=0.02, consts=None):
    """Union queries: an entity's distance is the nearest branch's."""
    out = []
    for e, t, f in zip(embeddings, targets, filters):
        d = np.min(np.stack([eval_distances(backbone, ent, b, dim, alpha, consts)
                             for b in np.atleast_2d(e)]), axis=0)
        out.append(filtered_rank(-d, t, f))
    return np.array(out, dtype=np.int64)


# ---- adaptive sampling (sampler DESIGN DECISIONS :243-244) ----
# A literal numpy restatement of the sampler's difficulty rule, independent of
# the product's C++ (paper_2602_21597_b200/csrc/host/sampler.cpp).

def record_difficulty(ema, obs, pattern, loss, decay=0.9):
    """ema(p) <- decay*ema(p) + (1-decay)*loss; NonFiniteLoss
    (ValueError here) for a non-finite or negative loss."""
    if not np.isfinite(loss) or loss < 0:
        raise ValueError(f"NonFiniteLoss: {loss}")
    ema[pattern] = decay * ema[pattern] + (1.0 - decay) * loss
    obs[pattern] += 1


def update_distribution(ema, obs, eta=1.0, floor=0.01, base=None):
    """w(p) ∝ exp(η·ema(p)), renormalised, clipped below at ε
    and renormalised again — over the support of `base` (default: all 14
    patterns); cold start (a support pattern never observed) returns `base`."""
    base = np.full(14, 1.0 / 14) if base is None else np.asarray(base, np.float64)
    sup = base > 0
    if (np.asarray(obs)[sup] == 0).any():
        return base.copy()
    e = np.asarray(ema, np.float64)
    w = np.zeros(14)
    w[sup] = np.exp(eta * (e[sup] - e[sup].max()))
    w /= w.sum()
    clipped = np.zeros(14, bool)
    while True:  # clip at ε, renormalise the rest, until no new clip
        new = sup & ~clipped & (w < floor)
        clipped |= new
        free = sup & ~clipped
        w[clipped] = floor
        w[free] *= (1.0 - clipped.sum() * floor) / w[free].sum()
        if not new.any():
            return w


def batch_pattern_losses(patterns, losses):
    """(pattern, mean per-query loss) of every pattern present in a batch, in
    pattern order — what the trainer records after each step."""
    sums, cnt = [0.0] * 14, [0] * 14
    for p, x in zip(np.asarray(patterns).tolist(), np.asarray(losses, np.float64).tolist()):
        sums[p] += x  # sequential, query order
        cnt[p] += 1
    return [(p, sums[p] / cnt[p]) for p in range(14) if cnt[p]]


# ---- evaluator entity tables of BetaE and fusion (f64) -------------------------

def beta_realize(x):
    """clamp(softplus(x), 0.05, 1e9) (SURVEY A-7), f64."""
    x = np.asarray(x, np.float64)
    return np.clip(np.logaddexp(0.0, x), 0.05, 1e9)


def beta_eval_table(raw, dim):
    """Entity side of KL(Beta(a,b) || Beta(A,B)) = lnB(A,B) + C_e + A (psi(s)-psi(a))
    + B (psi(s)-psi(b)), for raw entity rows
    [n][2d] -> T [n][2d], C [n] in f64 (scipy special functions)."""
    from scipy.special import betaln, digamma
    a, b = beta_realize(raw[:, :dim]), beta_realize(raw[:, dim:2 * dim])
    s = a + b
    da, db, ds = digamma(a), digamma(b), digamma(s)
    T = np.concatenate([ds - da, ds - db], axis=1)
    C = np.sum(-betaln(a, b) + a * da + b * db - s * ds, axis=1)
    return T, C


def beta_kl(a, b, A, B):
    """KL(Beta(a,b) || Beta(A,B)) elementwise, f64 (the closed form)."""
    from scipy.special import betaln, digamma
    return (betaln(A, B) - betaln(a, b) + (a - A) * digamma(a) + (b - B) * digamma(b)
            + (A - a + B - b) * digamma(a + b))


def fused_table(entity, store, fus_f, fus_wp, fus_bp):
    """sigma(W_p [h | F s] + b_p) of every entity (Eq. 12), f64."""
    h = np.asarray(entity, np.float64)
    fs = np.asarray(store, np.float64) @ np.asarray(fus_f, np.float64).T
    z = np.concatenate([h, fs], axis=1) @ np.asarray(fus_wp, np.float64).T + \
        np.asarray(fus_bp, np.float64).reshape(1, -1)
    return 1.0 / (1.0 + np.exp(-z))
