/* ORACLE C ABI — test infrastructure only (tests/, __graft_entry__.smoke(),
 * bench.py's CPU-baseline leg). Never linked into the product library.
 * All calls return 0 on success, nonzero on error (message: oracle_last_error). */
#ifndef NGDB_ORACLE_H_
#define NGDB_ORACLE_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* RNG restatement (for golden-vector tests) */
uint64_t oracle_rng_next(uint64_t seed, int64_t fork_tag, int32_t skip);
int oracle_rng_below(uint64_t seed, const uint64_t* ns, int32_t count, int32_t reps, uint64_t* out);
int oracle_rng_uniform(uint64_t seed, int32_t n, double lo, double hi, double* out);
int oracle_rng_gaussian(uint64_t seed, int32_t n, double* out);
uint64_t oracle_fnv1a64(const char* s, int64_t n);

/* graph: triples as [n][3] (h, r, t) */
int oracle_graph_create(int32_t n_entities, int32_t n_relations, const int32_t* train,
                        int64_t n_train, const int32_t* valid, int64_t n_valid,
                        const int32_t* test, int64_t n_test, void** out);
int oracle_graph_answer(void* g, int32_t full, int32_t pattern, const int32_t* anchors,
                        const int32_t* relations, int32_t* out, int64_t cap, int64_t* n);
int oracle_graph_destroy(void* g);

/* sampler: Rng(seed).fork(tag); outputs anchors [b][3], relations [b][4] (-1 pad) */
int oracle_sample_batch(void* g, const double* weights, int32_t b, int32_t n_neg, uint64_t seed,
                        uint64_t tag, int32_t* patterns, int32_t* anchors, int32_t* relations,
                        int32_t* positives, int32_t* negatives);

/* DAG node table of a batch: per node (kind, bwd, n_in, in0, in1, in2, payload, query,
 * mirror, consumer, slot) as 11 int32; returns node count via *n and fwd count *nf */
int oracle_build_dag(int32_t b, const int32_t* patterns, const int32_t* anchors,
                     const int32_t* relations, int32_t* out, int64_t cap, int32_t* n, int32_t* nf,
                     int32_t* edges, int64_t edge_cap, int32_t* n_edges);

/* model: precision 64 or 32 */
int oracle_model_create(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                        int32_t n_neg, double gamma, double alpha_box, double lr,
                        int32_t precision, void** out);
int oracle_model_init(void* m, uint64_t seed);
/* name may carry "m:" or "v:" (Adam moments) */
int oracle_model_set(void* m, const char* name, const float* data, int64_t n);
/* name may carry "g:" (last step gradient), "m:" or "v:" (Adam moments) */
int oracle_model_get(void* m, const char* name, double* out, int64_t n);
/* one training step; executor 0 = Alg. 1 scheduled, 1 = sequential reference;
 * adam 0 = lazy touched rows, 1 = dense, -1 = no optimizer step */
int oracle_model_step(void* m, int32_t b, const int32_t* patterns, const int32_t* anchors,
                      const int32_t* relations, const int32_t* positives,
                      const int32_t* negatives, int32_t b_max, int64_t step, int32_t executor,
                      int32_t adam, int32_t eager, double* losses);
int oracle_model_trace_json(void* m, int32_t with_nodes, char* buf, int64_t cap, int64_t* len);
/* per-query minimum |kink argument| of the last step's forward pass (L1/box
 * signs, inside/outside, ReLU inputs, argmin/min routing gaps) */
int oracle_model_margins(void* m, double* out, int32_t n);
int oracle_model_destroy(void* m);
/* per-query min over query-level kinks only (those that change dL/dq) */
int oracle_model_qmargins(void* m, double* out, int32_t n);
/* precision 65 (f64 values with first-order fp32 deviation bounds, oracle/src/dual.hpp):
 * kinks within tau inject bounds; dev(name) = bound per element ("g:" gradients, "m:"/"v:"
 * moments, plain = parameters). Values via oracle_model_get are the f64 model's. */
int oracle_model_set_dev_tau(void* m, double tau);
int oracle_model_dev(void* m, const char* name, double* out, int64_t n);

/* scalar kernels for the SPEC known-answer tests */
double oracle_q2b_distance(const double* v, const double* c, const double* o, int32_t d,
                           double alpha);
/* sub-batches scheduled independently, gradients summed, one Adam (sharded parity) */
int oracle_model_step_multi(void* model, int32_t n, const int32_t* sizes, const int32_t* patterns,
                            const int32_t* anchors, const int32_t* relations,
                            const int32_t* positives, const int32_t* negatives, int32_t b_max,
                            int64_t step, int32_t adam, double* losses);
/* frozen semantic store [ne][dl] + fusion params (call before oracle_model_init) */
int oracle_model_set_semantic(void* model, int32_t dl, const float* store, int64_t n);
/* synthetic benchmark KGs: shape table; all triples of the shape
 * [n_train + n_valid + n_test][3] (train first, then valid, then test); PTE store */
int oracle_synth_shape(const char* name, int32_t* n_entities, int32_t* n_relations,
                       int64_t* counts /* train, valid, test */);
int oracle_synth_triples(const char* name, uint64_t seed, int32_t* out);
int oracle_semantic_store(int32_t n_entities, int32_t dl, uint64_t seed, float* out);
/* OpenMP threads of the row-parallel GEMVs / KL dims (results independent of it) */
int oracle_set_threads(int32_t n);
double oracle_loss(double gamma, double d_pos, const double* d_neg, int32_t k);
/* BetaE special functions and KL(Beta(a1,b1) || Beta(a2,b2)) */
double oracle_lgamma(double x);
double oracle_digamma(double x);
double oracle_trigamma(double x);
double oracle_beta_kl(double a1, double b1, double a2, double b2);

#ifdef __cplusplus
}
#endif
#endif
