// ORACLE (test infrastructure only). First-order deviation bounds for the
// full-batch parity masks (tests/parity.py `run_masked`).
//
// A Dual carries a value v (plain f64 arithmetic, bit-identical to Model<double>)
// and a bound d on how far an fp32 execution of the same formulas may legitimately
// drift from v because it resolved a kink differently. Sources of d are injected
// only at kinks whose argument is within tau of the switch point (Model::pick and
// friends: L1 / box sign and inside/outside tests, ReLU masks, min / argmin
// routing, realize() and negation clamps); everywhere else d propagates like
// |Jacobian|^T d (sums add bounds, products scale them by the other factor's
// magnitude). Forward values are continuous at every kink, so forward d stays 0.
#pragma once

#include <cmath>

namespace oracle {

struct Dual {
  double v = 0.0, d = 0.0;
  Dual() = default;
  Dual(double x) : v(x) {}  // NOLINT: implicit, so R(1), R(alpha) work unchanged
  Dual(double x, double dd) : v(x), d(dd) {}
  explicit operator double() const { return v; }
  explicit operator float() const { return float(v); }
  Dual operator-() const { return {-v, d}; }
  Dual& operator+=(const Dual& o) { v += o.v; d += o.d; return *this; }
  Dual& operator-=(const Dual& o) { v -= o.v; d += o.d; return *this; }
  Dual& operator*=(const Dual& o) { *this = *this * o; return *this; }
  Dual& operator/=(const Dual& o) { *this = *this / o; return *this; }
  friend Dual operator+(Dual a, const Dual& b) { return a += b; }
  friend Dual operator-(Dual a, const Dual& b) { return a -= b; }
  friend Dual operator*(const Dual& a, const Dual& b) {
    return {a.v * b.v, std::fabs(a.v) * b.d + std::fabs(b.v) * a.d + a.d * b.d};
  }
  friend Dual operator/(const Dual& a, const Dual& b) {
    const double q = a.v / b.v;
    return {q, (a.d + std::fabs(q) * b.d) / std::fabs(b.v)};
  }
  friend bool operator<(const Dual& a, const Dual& b) { return a.v < b.v; }
  friend bool operator>(const Dual& a, const Dual& b) { return a.v > b.v; }
  friend bool operator<=(const Dual& a, const Dual& b) { return a.v <= b.v; }
  friend bool operator>=(const Dual& a, const Dual& b) { return a.v >= b.v; }
  friend bool operator==(const Dual& a, const Dual& b) { return a.v == b.v; }
  friend bool operator!=(const Dual& a, const Dual& b) { return a.v != b.v; }
};

inline double val(double x) { return x; }
inline double val(float x) { return x; }
inline double val(const Dual& x) { return x.v; }
inline double dev(double) { return 0.0; }
inline double dev(float) { return 0.0; }
inline double dev(const Dual& x) { return x.d; }
inline void add_dev(double&, double) {}
inline void add_dev(float&, double) {}
inline void add_dev(Dual& x, double a) { x.d += a; }

// math on R in {float, double, Dual}; the Dual forms scale d by |f'(v)|
inline double mexp(double x) { return std::exp(x); }
inline float mexp(float x) { return std::exp(x); }
inline Dual mexp(const Dual& x) {
  const double e = std::exp(x.v);
  return {e, e * x.d};
}
inline double mlog1p(double x) { return std::log1p(x); }
inline float mlog1p(float x) { return std::log1p(x); }
inline Dual mlog1p(const Dual& x) { return {std::log1p(x.v), x.d / std::fabs(1.0 + x.v)}; }
inline double mfabs(double x) { return std::fabs(x); }
inline float mfabs(float x) { return std::fabs(x); }
inline Dual mfabs(const Dual& x) { return {std::fabs(x.v), x.d}; }
inline double msqrt(double x) { return std::sqrt(x); }
inline float msqrt(float x) { return std::sqrt(x); }
inline Dual msqrt(const Dual& x) {
  const double s = std::sqrt(x.v);
  return {s, s > 0 ? x.d / (2 * s) : x.d};
}

}  // namespace oracle
