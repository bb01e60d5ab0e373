// Piecewise-polynomial form of the Kaiser-Bessel window (window.cuh) for the window-block
// precomputation of the cell-group kernels (chunks.cu).  Host-only C++.
//
// A point with grid coordinate u = l0 + f (l0 = floor u, f in [0, 1)) has the 2m taps
// a = 0 .. 2m-1 at distances v = f + m - 1 - a, i.e. tap a only ever sees v in
// [m - 1 - a, m - a).  On that unit interval phi is analytic (an even function of
// s = sqrt(m^2 - v^2)), so a degree-14 polynomial in t = f - 1/2 represents it to ~1e-16
// absolute (phi(0) = 1): measured max error 1.1e-16 (m = 8, sigma = 2) and 2.2e-16
// (m = 6, sigma = 3) against 40-digit values, float64 Horner.  One window row then costs
// 14 FMA per tap instead of a sqrt, an exp and a division.
//
// The coefficients are fitted per plan (b depends on sigma): Chebyshev interpolation at
// kHornerDeg + 1 nodes in long double, converted to the monomial basis in t.
#pragma once
#include <cmath>

namespace uotk {

constexpr int kHornerDeg = 14;
constexpr int kHornerMaxTaps = 16;

struct KBHorner {
    double c[kHornerMaxTaps][kHornerDeg + 1];  // c[a][j]: phi(f + m - 1 - a) = sum_j c[a][j] (f - 1/2)^j
};

// phi normalised to phi(0) = 1 (window.cuh), in long double; 0 outside |v| < m
inline long double kb_phi_ld(long double v, long double b, long double m) {
    const long double s2 = m * m - v * v;
    if (s2 <= 0.0L) return 0.0L;
    const long double s = std::sqrt(s2);
    if (s < 1e-9L) return b * m / std::sinh(b * m);
    // sinh(b s) / s * m / sinh(b m) = m e^{b (s - m)} (1 - e^{-2 b s}) / (s (1 - e^{-2 b m}))
    return m * std::exp(b * (s - m)) * (1.0L - std::exp(-2.0L * b * s)) / (s * (1.0L - std::exp(-2.0L * b * m)));
}

inline KBHorner kb_horner_fit(double b, int m) {
    constexpr int K = kHornerDeg + 1;
    const long double pi = 3.141592653589793238462643383279502884L;
    KBHorner h{};
    for (int a = 0; a < 2 * m && a < kHornerMaxTaps; ++a) {
        // Chebyshev coefficients of g(x) = phi(f + m - 1 - a), x = 2f - 1 = 2t in [-1, 1]
        long double val[K], ch[K];
        for (int k = 0; k < K; ++k) {
            const long double x = std::cos(pi * (k + 0.5L) / K);
            val[k] = kb_phi_ld((x + 1.0L) / 2.0L + m - 1 - a, (long double)b, (long double)m);
        }
        for (int j = 0; j < K; ++j) {
            long double s = 0.0L;
            for (int k = 0; k < K; ++k) s += val[k] * std::cos(pi * j * (k + 0.5L) / K);
            ch[j] = (j == 0 ? 1.0L : 2.0L) * s / K;
        }
        // sum_j ch[j] T_j(2t) -> monomials in t: T_0 = 1, T_1 = 2t, T_{j+1} = 4t T_j - T_{j-1}
        long double Tm[K] = {0}, T0[K] = {0}, T1[K] = {0}, mono[K] = {0};
        T0[0] = 1.0L;
        T1[1] = 2.0L;
        for (int i = 0; i < K; ++i) mono[i] += ch[0] * T0[i];
        for (int i = 0; i < K; ++i) mono[i] += ch[1] * T1[i];
        for (int j = 2; j < K; ++j) {
            long double Tn[K] = {0};
            for (int i = 0; i + 1 < K; ++i) Tn[i + 1] += 4.0L * T1[i];
            for (int i = 0; i < K; ++i) Tn[i] -= T0[i];
            for (int i = 0; i < K; ++i) mono[i] += ch[j] * Tn[i];
            for (int i = 0; i < K; ++i) {
                Tm[i] = T0[i];
                T0[i] = T1[i];
                T1[i] = Tn[i];
            }
        }
        (void)Tm;
        for (int j = 0; j < K; ++j) h.c[a][j] = (double)mono[j];
    }
    return h;
}

}  // namespace uotk
