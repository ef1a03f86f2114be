// Drop-in check of include/fsvd/kernels.hpp + include/fsvd/math.hpp (the
// reference's CPU operator / math API, kernels.hpp:18-62, math.hpp:16-140)
// against values the reference itself produced (tests/golden/primitives.json,
// scalar variant, tests/golden/make_golden.py). Compiled against include/ and
// linked to libfsvd_b200.so by tests/test_abi.py. Prints OK or the failures.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "fsvd/kernels.hpp"
#include "fsvd/math.hpp"

using nlohmann::json;

static int g_fail = 0;
#define CHECK(c, what)                                   \
    do {                                                 \
        if (!(c)) {                                      \
            std::printf("FAIL %s (line %d)\n", what, __LINE__); \
            ++g_fail;                                    \
        }                                                \
    } while (0)

static std::vector<double> hexd(const json& a) {
    std::vector<double> v;
    for (const auto& s : a) v.push_back(std::strtod(s.get<std::string>().c_str(), nullptr));
    return v;
}
static std::vector<float> hexf(const json& a) {
    std::vector<float> v;
    for (double x : hexd(a)) v.push_back(static_cast<float>(x));
    return v;
}

int main(int argc, char** argv) {
    std::ifstream f(argv[1]);
    const json P = json::parse(f);
    CHECK(fsvd::kern::variants().size() >= 1 && std::string(fsvd::kern::variants()[0].name) == "scalar", "variants");
    CHECK(!fsvd::kern::force_variant("no-such-variant"), "force unknown");
    CHECK(fsvd::kern::force_variant("scalar"), "force scalar");

    // rmsnorm, f64 and f32 (kernels_scalar.cpp:55-61), bitwise
    {
        const json& r = P["rmsnorm"];
        const auto x = hexd(r["x"]), g = hexd(r["g"]), y = hexd(r["y64"]);
        const auto got = fsvd::rmsnorm<double>(x, g, r["eps"].get<double>());
        CHECK(got == y, "rmsnorm f64");
        const auto xf = hexf(r["xf"]), gf = hexf(r["gf"]), yf = hexf(r["y32"]);
        const auto gotf = fsvd::rmsnorm<float>(xf, gf, static_cast<float>(r["eps"].get<double>()));
        CHECK(gotf == yf, "rmsnorm f32");
        bool threw = false;
        try {
            fsvd::rmsnorm<double>(std::span<const double>(x.data(), 2), g, 1e-5);
        } catch (const fsvd::ShapeError&) {
            threw = true;
        }
        CHECK(threw, "rmsnorm shape error");
    }
    // rope, interleaved pairs, angles in double (math.hpp:30-44), bitwise
    for (const json& r : P["rope"]) {
        const auto v = hexd(r["v"]), o = hexd(r["out64"]);
        CHECK(fsvd::rope_apply<double>(v, r["pos"].get<double>(), 10000.0) == o, "rope f64");
        auto vf = hexf(r["vf"]);
        fsvd::rope_inplace(vf.data(), vf.size(), r["pos"].get<double>(), 10000.0);
        CHECK(vf == hexf(r["out32"]), "rope f32");
    }
    // online softmax attention in the reference's block partition (bitwise) and
    // partition invariance (<= 1e-12, test_tensor.cpp:173-233)
    for (const json& c : P["online_attend"]) {
        const size_t d = c["d"], rows = c["rows"];
        const auto q = hexd(c["q"]), k = hexd(c["k"]), v = hexd(c["v"]), want = hexd(c["out"]);
        for (int mode = 0; mode < 3; ++mode) {
            std::vector<size_t> blocks = mode == 0 ? c["blocks"].get<std::vector<size_t>>()
                                                   : mode == 1 ? std::vector<size_t>{rows} : std::vector<size_t>(rows, 1);
            std::vector<std::pair<fsvd::Tensor2D<double>, fsvd::Tensor2D<double>>> kv;
            size_t r0 = 0;
            for (size_t b : blocks) {
                std::vector<double> kb(k.begin() + r0 * d, k.begin() + (r0 + b) * d);
                std::vector<double> vb(v.begin() + r0 * d, v.begin() + (r0 + b) * d);
                kv.emplace_back(fsvd::Tensor2D<double>(b, d, kb), fsvd::Tensor2D<double>(b, d, vb));
                r0 += b;
            }
            const auto got = fsvd::online_softmax_attend<double>(q, kv, c["scale"].get<double>());
            double err = 0;
            for (size_t e = 0; e < d; ++e) err = std::max(err, std::abs(got[e] - want[e]));
            if (mode == 0) CHECK(got == want, "online attend (reference partition)");
            CHECK(err <= 1e-12, "online attend partition invariance");
        }
    }
    // argmax ties -> lowest index (math.hpp:132-140)
    for (const json& a : P["argmax"]) {
        const auto x = a["x"].get<std::vector<double>>();
        CHECK(fsvd::argmax_greedy<double>(x) == a["idx"].get<size_t>(), "argmax");
    }
    // gemv per-column in-order accumulation (kernels.hpp:8-11), both variants bitwise
    {
        const json& g = P["gemv_f32"];
        const size_t m = g["m"], n = g["n"];
        const auto x = hexf(g["x"]), a = hexf(g["a"]), y = hexf(g["y"]);
        for (const auto& var : fsvd::kern::variants()) {
            std::vector<float> got(n, -1.f);
            var.f32->gemv(got.data(), x.data(), a.data(), m, n);
            CHECK(got == y, var.name);
            // column j depends only on column j: a sub-range of columns gives the same bits
            std::vector<float> a2(m * 5), y2(5);
            for (size_t i = 0; i < m; ++i)
                for (size_t j = 0; j < 5; ++j) a2[i * 5 + j] = a[i * n + 7 + j];
            var.f32->gemv(y2.data(), x.data(), a2.data(), m, 5);
            for (size_t j = 0; j < 5; ++j) CHECK(y2[j] == y[7 + j], "gemv column independence");
        }
    }
    if (g_fail) return 1;
    std::printf("OK (%zu variants, active %s)\n", fsvd::kern::variants().size(), fsvd::kern::active().name);
    return 0;
}
