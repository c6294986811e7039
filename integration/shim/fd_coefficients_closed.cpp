// Build fix for the reference's own host code (used by the drop-in build, integration/Makefile,
// and by the oracle build, oracle/Makefile).
//
// Replacement for the reference's src/fd_coefficients.cpp:40-83, which solves
// the Taylor table over Boost.Multiprecision/Boost.Rational (src/fd_coefficients.cpp:1-2;
// Boost is not vendored, proj/.gitignore:2).  This file computes the same exact
// central weights in closed form with the reference's own stencilc::Rational:
//
//   M = accuracy/2,  p_k = prod_{j=1..k} (M-j+1)/(M+j)
//   d = 2:  c(+-k) = 2(-1)^(k+1) p_k / k^2,   c(0) = -2 sum_k c(k)
//   d = 1:  c(+k)  = (-1)^(k+1) p_k / k,      c(-k) = -c(+k),  c(0) = 0
//
// The result is checked against an independent Fraction-based Gaussian
// elimination of the Taylor system in tests/test_oracle.py (test_weights_equal_taylor_solve).
#include <stdexcept>
#include <utility>
#include <vector>

#include "stencilc/symbolic.hpp"

namespace stencilc::sym {

std::vector<std::pair<int, Rational>> fd_coefficients(int derivative_order,
                                                      int accuracy_order) {
    // Error texts follow src/fd_coefficients.cpp:42-45.
    if (derivative_order < 1 || derivative_order > 2)
        throw std::invalid_argument("fd_coefficients: derivative order must be 1 or 2");
    if (accuracy_order < 2 || accuracy_order % 2 != 0)
        throw std::invalid_argument("fd_coefficients: accuracy order must be even and >= 2");
    const int M = accuracy_order / 2;
    std::vector<Rational> side(static_cast<size_t>(M) + 1);  // side[k] = c(+k)
    Rational p(1);
    Rational sum(0);
    for (int k = 1; k <= M; ++k) {
        p *= Rational(M - k + 1, M + k);
        Rational sign(k % 2 == 1 ? 1 : -1);
        if (derivative_order == 2) {
            side[static_cast<size_t>(k)] = Rational(2) * sign * p / Rational(k * k);
            sum += side[static_cast<size_t>(k)];
        } else {
            side[static_cast<size_t>(k)] = sign * p / Rational(k);
        }
    }
    std::vector<std::pair<int, Rational>> out;
    out.reserve(static_cast<size_t>(2 * M + 1));
    for (int o = -M; o <= M; ++o) {
        Rational w(0);
        if (o == 0)
            w = derivative_order == 2 ? Rational(-2) * sum : Rational(0);
        else if (o > 0)
            w = side[static_cast<size_t>(o)];
        else
            w = derivative_order == 2 ? side[static_cast<size_t>(-o)]
                                      : -side[static_cast<size_t>(-o)];
        out.emplace_back(o, w);
    }
    return out;
}

}  // namespace stencilc::sym
