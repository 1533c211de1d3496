// ORACLE (test infrastructure only). Special functions BetaE needs
// (SPEC.md:395-403): lgamma by Lanczos g=7 (9 terms), digamma and trigamma by
// upward recurrence to x >= 10 then the asymptotic (Bernoulli) series; and the
// Beta KL divergence with its partial derivatives.
#pragma once

#include <cmath>
#include <stdexcept>

namespace oracle {

template <class R>
R sp_lgamma(R x) {
  if (!(x > R(0))) throw std::domain_error("DomainError: lgamma(x <= 0)");
  static const double p[9] = {0.99999999999980993,     676.5203681218851,
                              -1259.1392167224028,     771.32342877765313,
                              -176.61502916214059,     12.507343278686905,
                              -0.13857109526572012,    9.9843695780195716e-6,
                              1.5056327351493116e-7};
  const double kPi = 3.14159265358979323846;
  double xv = double(x);
  if (xv < 0.5) {  // reflection: Gamma(x) Gamma(1-x) = pi / sin(pi x)
    return R(std::log(kPi / std::fabs(std::sin(kPi * xv))) - double(sp_lgamma<double>(1.0 - xv)));
  }
  xv -= 1.0;
  double a = p[0];
  for (int i = 1; i < 9; ++i) a += p[i] / (xv + i);
  const double t = xv + 7.5;
  return R(0.91893853320467274178 + (xv + 0.5) * std::log(t) - t + std::log(a));
}

template <class R>
R sp_digamma(R x) {
  if (!(x > R(0))) throw std::domain_error("DomainError: digamma(x <= 0)");
  R acc = 0;
  while (x < R(10)) {
    acc -= R(1) / x;
    x += R(1);
  }
  const R i2 = R(1) / (x * x);
  const R series =
      i2 * (R(1) / 12 - i2 * (R(1) / 120 - i2 * (R(1) / 252 - i2 * (R(1) / 240 - i2 * (R(1) / 132)))));
  return acc + std::log(x) - R(0.5) / x - series;
}

template <class R>
R sp_trigamma(R x) {
  if (!(x > R(0))) throw std::domain_error("DomainError: trigamma(x <= 0)");
  R acc = 0;
  while (x < R(10)) {
    acc += R(1) / (x * x);
    x += R(1);
  }
  const R i1 = R(1) / x, i2 = i1 * i1;
  // 1/x + 1/(2x^2) + 1/(6x^3) - 1/(30x^5) + 1/(42x^7) - 1/(30x^9) + 5/(66x^11)
  const R series =
      i1 + i2 / 2 + i1 * i2 * (R(1) / 6 - i2 * (R(1) / 30 - i2 * (R(1) / 42 - i2 * (R(1) / 30 - i2 * R(5) / 66))));
  return acc + series;
}

template <class R>
R sp_lbeta(R a, R b) {
  return sp_lgamma(a) + sp_lgamma(b) - sp_lgamma(a + b);
}

// KL(Beta(a1, b1) || Beta(a2, b2))
template <class R>
R beta_kl(R a1, R b1, R a2, R b2) {
  const R s1 = a1 + b1;
  return sp_lbeta(a2, b2) - sp_lbeta(a1, b1) + (a1 - a2) * sp_digamma(a1) +
         (b1 - b2) * sp_digamma(b1) + (a2 - a1 + b2 - b1) * sp_digamma(s1);
}

// partial derivatives of beta_kl: (d/da1, d/db1, d/da2, d/db2)
template <class R>
void beta_kl_grad(R a1, R b1, R a2, R b2, R* g) {
  const R s1 = a1 + b1, s2 = a2 + b2;
  const R t1 = sp_trigamma(s1);
  g[0] = (a1 - a2) * sp_trigamma(a1) + (s2 - s1) * t1;
  g[1] = (b1 - b2) * sp_trigamma(b1) + (s2 - s1) * t1;
  const R ds1 = sp_digamma(s1), ds2 = sp_digamma(s2);
  g[2] = sp_digamma(a2) - ds2 - sp_digamma(a1) + ds1;
  g[3] = sp_digamma(b2) - ds2 - sp_digamma(b1) + ds1;
}

}  // namespace oracle
