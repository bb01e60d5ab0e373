// Kaiser-Bessel window of the NFFT (footnote P:653: cutoff m; shape b = pi(2 - 1/sigma)).
#pragma once
#include <cmath>

namespace uotk {

// phi(v) = sinh(b sqrt(m^2 - v^2)) / sqrt(m^2 - v^2) * m / sinh(b m),  |v| < m (grid units),
// i.e. the KB window normalised to phi(0) = 1.  Evaluated as
//   m (E^2 - C2) / (E s (1 - C2)),  s = sqrt(m^2 - v^2), E = exp(b (s - m)), C2 = exp(-2 b m),
// which avoids the 1e16-sized sinh values.  Its Fourier transform (used by the
// deconvolution in nfft_plan.cu) is (pi m/n_g) I0(m sqrt(b^2 - (2 pi k/n_g)^2)) / sinh(b m).
struct KBWindow {
    double b;
    double m;
    double m2;
    double C2;        // exp(-2 b m)
    double inv1mC2;   // 1/(1 - C2)
    double lim0;      // value at s -> 0: b m / sinh(b m)
};

inline KBWindow make_window(double b, int m) {
    KBWindow w;
    w.b = b;
    w.m = m;
    w.m2 = (double)m * m;
    w.C2 = std::exp(-2.0 * b * m);
    w.inv1mC2 = 1.0 / (1.0 - w.C2);
    w.lim0 = 2.0 * b * m * std::exp(-b * m) * w.inv1mC2;
    return w;
}

__device__ __forceinline__ double kb_phi(double v, const KBWindow& w) {
    const double s2 = w.m2 - v * v;
    if (s2 <= 0.0) return 0.0;
    const double s = sqrt(s2);
    if (s < 1e-7) return w.lim0;
    const double E = exp(w.b * (s - w.m));
    return w.m * (E * E - w.C2) * w.inv1mC2 / (s * E);
}

}  // namespace uotk
