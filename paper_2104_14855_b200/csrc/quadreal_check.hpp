// quadreal_check.hpp -- diagnostic only: a __float128 stand-in for dd (build with
// -DMHDP_QUAD_CHECK) used to confirm that double-double is accurate enough for R-exact.
struct dd {
    __float128 q = 0;
    dd() = default;
    dd(double x) : q(x) {}
    dd(double h, double l) : q((__float128)h + l) {}
    static dd of(__float128 v) { dd r; r.q = v; return r; }
    double value() const { return (double)q; }
};
inline dd operator+(const dd &a, const dd &b) { return dd::of(a.q + b.q); }
inline dd operator-(const dd &a) { return dd::of(-a.q); }
inline dd operator-(const dd &a, const dd &b) { return dd::of(a.q - b.q); }
inline dd operator*(const dd &a, const dd &b) { return dd::of(a.q * b.q); }
inline dd operator/(const dd &a, const dd &b) { return dd::of(a.q / b.q); }
inline dd &operator+=(dd &a, const dd &b) { return a = a + b; }
inline dd &operator-=(dd &a, const dd &b) { return a = a - b; }
inline dd &operator*=(dd &a, const dd &b) { return a = a * b; }
inline bool operator<(const dd &a, const dd &b) { return a.q < b.q; }
inline bool operator>(const dd &a, const dd &b) { return a.q > b.q; }
inline dd fabs(const dd &a) { return a.q < 0 ? -a : a; }
extern "C" __float128 sqrtq(__float128);
inline dd sqrt(const dd &a) { return dd::of(sqrtq(a.q)); }

