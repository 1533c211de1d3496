// ORACLE (test infrastructure only). Training DAGs from pattern expressions.
//
// Each pattern is written as an expression tree (BetaE-benchmark shapes,
// SPEC.md:168; DNF for unions). Node ids are the post-order of
// the tree (children left to right), the Loss sink last (SURVEY A-1, A-3):
//   E<i> anchor i, P(x,j) project by relation j, I(..) intersect, N(x) negate,
//   S(x) score a union branch, U(..) union of branch scores, L(x) loss sink.
// Gradient mirrors are appended in forward-id order (A-2).
#include <stdexcept>
#include <string>

#include "oracle_internal.hpp"

namespace oracle {
namespace {

const char* kExpr[NPAT] = {
    "L(P(E0,0))",                             // 1p
    "L(P(P(E0,0),1))",                        // 2p
    "L(P(P(P(E0,0),1),2))",                   // 3p
    "L(I(P(E0,0),P(E1,1)))",                  // 2i
    "L(I(P(E0,0),P(E1,1),P(E2,2)))",          // 3i
    "L(I(P(P(E0,0),1),P(E1,2)))",             // pi
    "L(P(I(P(E0,0),P(E1,1)),2))",             // ip
    "L(U(S(P(E0,0)),S(P(E1,1))))",            // 2u  -> DNF [1p, 1p]
    "L(U(S(P(P(E0,0),2)),S(P(P(E1,1),2))))",  // up  -> DNF [2p, 2p]
    "L(I(P(E0,0),N(P(E1,1))))",               // 2in
    "L(I(P(E0,0),P(E1,1),N(P(E2,2))))",       // 3in
    "L(I(P(P(E0,0),1),N(P(E1,2))))",          // pin
    "L(I(N(P(P(E0,0),1)),P(E1,2)))",          // pni
    "L(P(I(P(E0,0),N(P(E1,1))),2))",          // inp
};

struct Parser {
  const std::string s;
  size_t i = 0;
  const OQuery& q;
  int query;
  ODag& d;

  int node(int kind, std::vector<int> in, int payload) {
    ONode n;
    n.kind = kind;
    n.in = in;
    n.payload = payload;
    n.query = query;
    const int id = (int)d.nodes.size();
    for (size_t k = 0; k < in.size(); ++k) {
      d.nodes[in[k]].consumer = id;
      d.nodes[in[k]].slot = (int)k;
      d.edges.push_back({in[k], id});
    }
    d.nodes.push_back(n);
    return id;
  }
  int num() {
    int v = 0;
    while (i < s.size() && isdigit((unsigned char)s[i])) v = v * 10 + (s[i++] - '0');
    return v;
  }
  int parse() {
    const char c = s[i++];
    if (c == 'E') return node(K_EMB, {}, q.a[num()]);
    if (s[i++] != '(') throw std::runtime_error("bad pattern expression");
    std::vector<int> kids;
    int rel = -1;
    for (;;) {
      if (isdigit((unsigned char)s[i])) rel = q.r[num()];
      else kids.push_back(parse());
      if (s[i] == ',') {
        ++i;
        continue;
      }
      ++i;  // ')'
      break;
    }
    switch (c) {
      case 'P': return node(K_PROJ, kids, rel);
      case 'I': return node(K_INTER, kids, -1);
      case 'N': return node(K_NEG, kids, -1);
      case 'S': return node(K_SCORE, kids, -1);
      case 'U': return node(K_UNION, kids, -1);
      case 'L': return node(K_LOSS, kids, -1);
    }
    throw std::runtime_error("bad operator in pattern expression");
  }
};

}  // namespace

ODag o_build_training_dag(const std::vector<OQuery>& batch) {
  ODag d;
  for (size_t qi = 0; qi < batch.size(); ++qi) {
    Parser p{kExpr[batch[qi].pattern], 0, batch[qi], (int)qi, d};
    p.parse();
  }
  d.nf = (int)d.nodes.size();
  for (int i = 0; i < d.nf; ++i) {
    ONode b;
    b.kind = d.nodes[i].kind;
    b.bwd = true;
    b.payload = d.nodes[i].payload;
    b.query = d.nodes[i].query;
    b.mirror = i;
    const int pred = d.nodes[i].consumer >= 0 ? d.nf + d.nodes[i].consumer : i;
    b.in = {pred};
    d.nodes[i].mirror = d.nf + i;
    d.nodes.push_back(b);
    d.edges.push_back({pred, d.nf + i});
  }
  return d;
}

}  // namespace oracle
