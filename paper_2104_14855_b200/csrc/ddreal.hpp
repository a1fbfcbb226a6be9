// ddreal.hpp -- double-double arithmetic (~106-bit significand) for the host setup.
//
// Reading R-exact: an assembled operator entry is the fp64 value nearest to
// the exact value of the discrete bilinear form for the given fp64 inputs.  The library
// evaluates every element quantity in double-double (error-free transformations built
// on fma; compile with -ffp-contract=off) and rounds each entry once.
#pragma once
#include <cmath>

namespace mhdp {

#ifdef MHDP_QUAD_CHECK
#include "quadreal_check.hpp"
#else
struct dd {
    double hi = 0.0, lo = 0.0;
    dd() = default;
    dd(double x) : hi(x), lo(0.0) {}
    dd(double h, double l) : hi(h), lo(l) {}
    double value() const { return hi; }   // normalised: hi = RN(hi + lo)
};

inline dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    return dd(s, e);
}
inline dd fast_two_sum(double a, double b) {
    const double s = a + b;
    return dd(s, b - (s - a));
}
inline dd two_prod(double a, double b) {
    const double p = a * b;
    return dd(p, std::fma(a, b, -p));
}
inline dd operator+(const dd &a, const dd &b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = fast_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return fast_two_sum(s.hi, s.lo);
}
inline dd operator-(const dd &a) { return dd(-a.hi, -a.lo); }
inline dd operator-(const dd &a, const dd &b) { return a + (-b); }
inline dd operator*(const dd &a, const dd &b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return fast_two_sum(p.hi, p.lo);
}
inline dd operator/(const dd &a, const dd &b) {
    const double q1 = a.hi / b.hi;
    dd r = a - b * dd(q1);
    const double q2 = r.hi / b.hi;
    r = r - b * dd(q2);
    const double q3 = r.hi / b.hi;
    return fast_two_sum(q1, q2) + dd(q3);
}
inline dd &operator+=(dd &a, const dd &b) { return a = a + b; }
inline dd &operator-=(dd &a, const dd &b) { return a = a - b; }
inline dd &operator*=(dd &a, const dd &b) { return a = a * b; }
inline bool operator<(const dd &a, const dd &b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
inline bool operator>(const dd &a, const dd &b) { return b < a; }
inline dd fabs(const dd &a) { return (a.hi < 0 || (a.hi == 0 && a.lo < 0)) ? -a : a; }
inline dd sqrt(const dd &a) {
    if (a.hi <= 0) return dd(0.0);
    const double x = std::sqrt(a.hi);
    const dd x2 = two_prod(x, x);
    const dd r = a - x2;                       // residual
    return fast_two_sum(x, r.hi / (2.0 * x)) + dd((r.lo) / (2.0 * x));
}

#endif

// uniform helpers for double and dd
inline double to_double(double x) { return x; }
inline double to_double(const dd &x) { return x.value(); }

}  // namespace mhdp
