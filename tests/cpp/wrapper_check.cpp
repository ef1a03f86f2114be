// Compile-and-run check of the C++ drop-in wrapper (include/fsvd/runtime.hpp)
// without a GPU: the loader-side errors surface as the reference's exception
// types. Built and run by tests/test_abi.py.
#include <cstdio>
#include <string>

#include "fsvd/runtime.hpp"

int main(int argc, char** argv) {
    int fails = 0;
    try {
        fsvd::gpu::Model::load("/nonexistent/model.fsvd");
        std::puts("no exception");
        ++fails;
    } catch (const fsvd::FormatError& e) {
        std::printf("FormatError ok: %s\n", e.what());
    }
    fsvd_ffn_backend f;
    fsvd::gpu::check(fsvd_route_ffn_auto(FSVD_PLAN_EAGER, FSVD_FFN_AUTO, &f));
    if (f != FSVD_FFN_NO_MERGE) ++fails;
    try {
        fsvd::gpu::check(fsvd_session_reset(nullptr));
        ++fails;
    } catch (const std::runtime_error&) {
    }
    std::printf("%s\n", fails ? "FAIL" : "OK");
    return fails;
}
