// Host-side model helpers exported through the C-ABI (include/swb.h).  They reproduce the
// reference's wave_model.cpp / fd_coefficients.cpp results bit-for-bit so a user of the
// Python or C++ mirror gets the same m, damp, dt and wavelet the reference would build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>

#include "../../include/swb.h"

namespace {

int64_t gcd64(int64_t a, int64_t b) {
    a = a < 0 ? -a : a;
    b = b < 0 ? -b : b;
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a ? a : 1;
}

struct Frac {
    int64_t n = 0, d = 1;
    Frac() = default;
    Frac(int64_t nn, int64_t dd) : n(nn), d(dd) {
        if (d < 0) { n = -n; d = -d; }
        int64_t g = gcd64(n, d);
        n /= g;
        d /= g;
    }
};

Frac mul(Frac a, Frac b) {
    // cross-reduce first to keep int64 headroom (weights up to SO 24 stay small)
    int64_t g1 = gcd64(a.n, b.d), g2 = gcd64(b.n, a.d);
    return Frac((a.n / g1) * (b.n / g2), (a.d / g2) * (b.d / g1));
}
Frac add(Frac a, Frac b) {
    int64_t g = gcd64(a.d, b.d);
    return Frac(a.n * (b.d / g) + b.n * (a.d / g), a.d / g * b.d);
}

}  // namespace

extern "C" {

// Exact central weights of d^order/dx^order at even accuracy `so`
// (same values as the Taylor-table solve of src/fd_coefficients.cpp:40-83):
//   M = so/2, p_k = prod_{j<=k} (M-j+1)/(M+j)
//   d=2: c(+-k) = 2(-1)^(k+1) p_k/k^2, c0 = -2 sum c_k;  d=1: c(+k) = (-1)^(k+1) p_k/k = -c(-k).
int swb_fd_weights(int order, int so, int64_t* num, int64_t* den) {
    if (order < 1 || order > 2 || so < 2 || so % 2 != 0 || so > 24 || !num || !den)
        return SWB_EINVAL;
    const int M = so / 2;
    Frac p(1, 1), sum(0, 1);
    for (int k = 1; k <= M; ++k) {
        p = mul(p, Frac(M - k + 1, M + k));
        Frac ck = order == 2 ? mul(p, Frac(2 * ((k % 2) ? 1 : -1), static_cast<int64_t>(k) * k))
                             : mul(p, Frac((k % 2) ? 1 : -1, k));
        num[M + k] = ck.n;
        den[M + k] = ck.d;
        num[M - k] = order == 2 ? ck.n : -ck.n;
        den[M - k] = ck.d;
        sum = add(sum, ck);
    }
    if (order == 2) {
        Frac c0 = mul(sum, Frac(-2, 1));
        num[M] = c0.n;
        den[M] = c0.d;
    } else {
        num[M] = 0;
        den[M] = 1;
    }
    return SWB_OK;
}

// cfl_dt, src/wave_model.cpp:146-154.
double swb_cfl_dt(int rank, const double* spacing, double max_velocity, int so) {
    double min_h = spacing[0];
    for (int d = 1; d < rank; ++d) min_h = std::min(min_h, spacing[d]);
    double base = (min_h / max_velocity) / std::sqrt(static_cast<double>(rank)) * 0.9;
    int64_t num[25], den[25];
    if (swb_fd_weights(2, so, num, den) != SWB_OK) return -1.0;
    double sum = 0.0;
    for (int i = 0; i <= so; ++i)
        sum += std::abs(static_cast<double>(num[i]) / static_cast<double>(den[i]));
    return base * (4.0 / sum);
}

// ricker_amplitude / ricker_wavelet, src/wave_model.cpp:128-144.
int swb_ricker_wavelet(double f, double dt, int steps, float* out) {
    if (!(f > 0.0) || !(dt > 0.0) || steps < 0 || (steps > 0 && !out)) return SWB_EINVAL;
    const double shift = 1.0 / f;
    for (int i = 0; i < steps; ++i) {
        double a = 3.14159265358979323846 * f * (i * dt - shift);
        a *= a;
        out[i] = static_cast<float>((1.0 - 2.0 * a) * std::exp(-a));
    }
    return SWB_OK;
}

// m_data, src/wave_model.cpp:16-23.
int swb_m_data(const float* velocity, size_t n, float* m) {
    if (!velocity || !m) return SWB_EINVAL;
    for (size_t i = 0; i < n; ++i) {
        float c = velocity[i];
        m[i] = 1.0f / (c * c);
    }
    return SWB_OK;
}

// damp_data, src/wave_model.cpp:25-45 (rank 3).
int swb_damp_data(const int32_t* shape, float damp_max, int width, float* out) {
    if (!shape || !out) return SWB_EINVAL;
    const size_t n = static_cast<size_t>(shape[0]) * shape[1] * shape[2];
    std::memset(out, 0, n * sizeof(float));
    if (damp_max <= 0.0f || width <= 0) return SWB_OK;
    for (int x = 0; x < shape[0]; ++x)
        for (int y = 0; y < shape[1]; ++y)
            for (int z = 0; z < shape[2]; ++z) {
                int dist = std::min({x, shape[0] - 1 - x, y, shape[1] - 1 - y, z, shape[2] - 1 - z});
                if (dist < width)
                    out[(static_cast<size_t>(x) * shape[1] + y) * shape[2] + z] =
                        damp_max * (1.0f - static_cast<float>(dist) / static_cast<float>(width));
            }
    return SWB_OK;
}

}  // extern "C"
