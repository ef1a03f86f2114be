// CPU operator layer behind include/fsvd/kernels.hpp (the reference's kern::Ops
// registry, proj/src/kernels/dispatch.cpp:14-63; semantics of
// proj/src/kernels/kernels_scalar.cpp:11-69). Two variants:
//   scalar -- plain loops;
//   avx2   -- the same loops with 8 (f32) / 4 (f64) output columns per vector,
//             compiled for AVX2 through a target attribute. Multiplies and adds
//             stay separately rounded (no FMA), and every output keeps its
//             in-order accumulation, so avx2 == scalar bit for bit.
// Selection once per process: FSVD_KERNELS=scalar|avx2, else the best the CPU runs.
#include <immintrin.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "fsvd/kernels.hpp"

namespace fsvd::kern {
namespace {

// ------------------------------------------------------------- scalar ----
template <typename T>
void s_gemv(T* y, const T* x, const T* a, size_t m, size_t n) {
    for (size_t j = 0; j < n; ++j) y[j] = T(0);
    for (size_t k = 0; k < m; ++k) {
        const T xk = x[k];
        const T* r = a + k * n;
        for (size_t j = 0; j < n; ++j) y[j] = y[j] + xk * r[j];
    }
}
template <typename T>
T s_dot(const T* a, const T* b, size_t n) {
    T acc = T(0);
    for (size_t i = 0; i < n; ++i) acc = acc + a[i] * b[i];
    return acc;
}
template <typename T>
void s_axpy(T* y, T alpha, const T* x, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = y[i] + alpha * x[i];
}
template <typename T>
void s_scal(T* y, T alpha, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = y[i] * alpha;
}
template <typename T>
void s_add(T* y, const T* x, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = y[i] + x[i];
}
template <typename T>
void s_rot(T* p, T* q, T c, T s, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        const T pi = p[i], qi = q[i];
        p[i] = c * pi - s * qi;
        q[i] = s * pi + c * qi;
    }
}
template <typename T>
void s_rmsnorm(T* y, const T* x, const T* gamma, size_t n, T eps) {
    T ss = T(0);
    for (size_t i = 0; i < n; ++i) ss = ss + x[i] * x[i];
    const T inv = T(1) / std::sqrt(ss / static_cast<T>(n) + eps);
    for (size_t i = 0; i < n; ++i) y[i] = x[i] * inv * gamma[i];
}
template <typename T>
void s_silu_mul(T* y, const T* gate, const T* up, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = gate[i] / (T(1) + std::exp(-gate[i])) * up[i];
}

// --------------------------------------------------------------- avx2 ----
// Only gemv and the column-parallel elementwise ops vectorize; dot, rmsnorm and
// silu_mul reduce or call exp and keep the scalar order.
__attribute__((target("avx2"))) void v_gemv_f32(float* y, const float* x, const float* a, size_t m, size_t n) {
    const size_t nv = n & ~size_t(7);
    for (size_t j = 0; j < n; ++j) y[j] = 0.f;
    for (size_t k = 0; k < m; ++k) {
        const __m256 xk = _mm256_set1_ps(x[k]);
        const float* r = a + k * n;
        for (size_t j = 0; j < nv; j += 8)
            _mm256_storeu_ps(y + j, _mm256_add_ps(_mm256_loadu_ps(y + j), _mm256_mul_ps(xk, _mm256_loadu_ps(r + j))));
        for (size_t j = nv; j < n; ++j) y[j] = y[j] + x[k] * r[j];
    }
}
__attribute__((target("avx2"))) void v_gemv_f64(double* y, const double* x, const double* a, size_t m, size_t n) {
    const size_t nv = n & ~size_t(3);
    for (size_t j = 0; j < n; ++j) y[j] = 0.0;
    for (size_t k = 0; k < m; ++k) {
        const __m256d xk = _mm256_set1_pd(x[k]);
        const double* r = a + k * n;
        for (size_t j = 0; j < nv; j += 4)
            _mm256_storeu_pd(y + j, _mm256_add_pd(_mm256_loadu_pd(y + j), _mm256_mul_pd(xk, _mm256_loadu_pd(r + j))));
        for (size_t j = nv; j < n; ++j) y[j] = y[j] + x[k] * r[j];
    }
}
__attribute__((target("avx2"))) void v_axpy_f32(float* y, float alpha, const float* x, size_t n) {
    const size_t nv = n & ~size_t(7);
    const __m256 al = _mm256_set1_ps(alpha);
    for (size_t i = 0; i < nv; i += 8)
        _mm256_storeu_ps(y + i, _mm256_add_ps(_mm256_loadu_ps(y + i), _mm256_mul_ps(al, _mm256_loadu_ps(x + i))));
    for (size_t i = nv; i < n; ++i) y[i] = y[i] + alpha * x[i];
}
__attribute__((target("avx2"))) void v_axpy_f64(double* y, double alpha, const double* x, size_t n) {
    const size_t nv = n & ~size_t(3);
    const __m256d al = _mm256_set1_pd(alpha);
    for (size_t i = 0; i < nv; i += 4)
        _mm256_storeu_pd(y + i, _mm256_add_pd(_mm256_loadu_pd(y + i), _mm256_mul_pd(al, _mm256_loadu_pd(x + i))));
    for (size_t i = nv; i < n; ++i) y[i] = y[i] + alpha * x[i];
}

template <typename T>
constexpr Ops<T> scalar_ops() {
    return Ops<T>{&s_gemv<T>, &s_dot<T>, &s_axpy<T>, &s_scal<T>, &s_add<T>, &s_rot<T>, &s_rmsnorm<T>, &s_silu_mul<T>};
}
const Ops<float> kScalar32 = scalar_ops<float>();
const Ops<double> kScalar64 = scalar_ops<double>();
const Ops<float> kAvx32{&v_gemv_f32, &s_dot<float>, &v_axpy_f32, &s_scal<float>, &s_add<float>, &s_rot<float>,
                        &s_rmsnorm<float>, &s_silu_mul<float>};
const Ops<double> kAvx64{&v_gemv_f64, &s_dot<double>, &v_axpy_f64, &s_scal<double>, &s_add<double>, &s_rot<double>,
                         &s_rmsnorm<double>, &s_silu_mul<double>};

const Variant kAll[2] = {{"scalar", &kScalar32, &kScalar64}, {"avx2", &kAvx32, &kAvx64}};

size_t usable() { return __builtin_cpu_supports("avx2") ? 2 : 1; }

std::atomic<const Variant*> g_forced{nullptr};

const Variant* pick() {
    const Variant* best = &kAll[usable() - 1];
    if (const char* e = std::getenv("FSVD_KERNELS"))
        for (size_t i = 0; i < usable(); ++i)
            if (std::strcmp(e, kAll[i].name) == 0) return &kAll[i];
    return best;
}

}  // namespace

std::span<const Variant> variants() { return {kAll, usable()}; }

const Variant& active() {
    if (const Variant* f = g_forced.load(std::memory_order_acquire)) return *f;
    static const Variant* chosen = pick();  // thread-safe static init
    return *chosen;
}

bool force_variant(const char* name) {
    for (size_t i = 0; i < usable(); ++i)
        if (name && std::strcmp(name, kAll[i].name) == 0) {
            g_forced.store(&kAll[i], std::memory_order_release);
            return true;
        }
    return false;
}

}  // namespace fsvd::kern
