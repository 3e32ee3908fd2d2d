// C++ drop-in check: a program written against the reference's gridjit API
// (driver.hpp / autolaunch.hpp) compiled against include/tt/gridjit_b200.hpp
// and run on the B200.  Mirrors /root/reference/proj/tests/test_driver.cpp
// ("the manual host flow", :229-280) and test_autolaunch.cpp (:38-62), then
// launches the trace transform through cuda_launch and checks it bit-exactly
// against the oracle's replay (oracle/tt_oracle.h).  Exit code 0 = pass.
#include <cstdio>
#include <cstring>
#include <vector>

#include "tt/gridjit_b200.hpp"
#include "tt_oracle.h"

using namespace gridjit;

static int failures = 0;
#define CHECK(x)                                                            \
    do {                                                                    \
        if (!(x)) {                                                         \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            ++failures;                                                     \
        }                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                   \
    do {                                           \
        bool ok = false;                           \
        try {                                      \
            (void)(expr);                          \
        } catch (const T&) {                       \
            ok = true;                             \
        } catch (...) {                            \
        }                                          \
        CHECK(ok && #T);                           \
    } while (0)

static const char* kVadd =
    ".module vadd$9e81eb78751b412a\n"
    ".kernel vadd(.param ptr.global.f32 a, .param ptr.global.f32 b, .param ptr.global.f32 c) {\n  ret\n}\n";

int main() {
    {  // the manual host flow (paper Listing 2)
        DeviceContext ctx = create_context();
        ModuleHandle md = ctx.module_load(kVadd);
        FunctionHandle vadd_fun = ctx.get_function(md, "vadd");
        std::vector<float> a(12), b(12);
        for (int i = 0; i < 12; ++i) {
            a[i] = float((i * 37) % 100);
            b[i] = float((i * 91) % 100);
        }
        DevicePtr ga = ctx.mem_alloc(48), gb = ctx.mem_alloc(48), gc = ctx.mem_alloc(48);
        ctx.memcpy_htod(ga, a.data(), 48);
        ctx.memcpy_htod(gb, b.data(), 48);
        GridConfig cfg;
        cfg.grid = {12, 1, 1};
        CHECK(ctx.launch(vadd_fun, cfg, {ga, gb, gc}).ok());
        std::vector<float> c(12, 0.0f);
        ctx.memcpy_dtoh(c.data(), gc, 48);
        for (int i = 0; i < 12; ++i) CHECK(c[i] == a[i] + b[i]);
        ctx.mem_free(ga);
        ctx.mem_free(gb);
        ctx.mem_free(gc);
        CHECK_THROWS_AS(ctx.mem_free(ga), DoubleFree);
        CHECK_THROWS_AS(ctx.memcpy_htod(ga, a.data(), 4), UseAfterFree);
        ctx.module_unload(md);
        Counters k = ctx.counters();
        CHECK(k.modules_loaded == 1 && k.functions_resolved == 1 && k.launches == 1);
        CHECK(k.allocs == 3 && k.frees == 3 && k.bytes_h2d == 96 && k.bytes_d2h == 48);
        CHECK(ctx.counters_json().find("\"launch_log\": [{\"kernel\": \"vadd\"") != std::string::npos);
        ctx.destroy();
        CHECK_THROWS_AS(ctx.destroy(), ContextDestroyed);
    }
    {  // the one-call facade
        DeviceContext ctx = create_context();
        KernelAst vadd = parse_kernel("kernel vadd(a, b, c) {\n  c[i] = a[i] + b[i];\n}\n");
        std::vector<float> a(12, 1.0f), b(12, 2.0f), c(12, -1.0f);
        GridConfig cfg;
        cfg.grid = {12, 1, 1};
        LaunchReport r1 = cuda_launch(ctx, vadd, cfg, {cu_in(a), cu_in(b), cu_out(c)});
        LaunchReport r2 = cuda_launch(ctx, vadd, cfg, {cu_in(a), cu_in(b), cu_out(c)});
        CHECK(r1.ok() && !r1.cache_hit && r2.cache_hit);
        CHECK(r1.bytes_h2d == 96 && r1.bytes_d2h == 48);
        for (float v : c) CHECK(v == 3.0f);
        CacheStats st = cache_stats(ctx);
        CHECK(st.entries == 1 && st.hits == 1 && st.misses == 1 && st.compiles == 1);
        CHECK_THROWS_AS(cuda_launch(ctx, vadd, cfg, {cu_in(a)}), ArityError);
    }
    {  // the path: trace_t05 through cuda_launch, bit-exact vs the replay oracle
        DeviceContext ctx = create_context();
        const int n = 192, A = 45;
        std::vector<float> img(size_t(n) * n), ctab(A), stab(A), wtab(8 * size_t(n));
        tt_synth_image(1, 7, n, img.data());
        tt_make_tables(n, A, ctab.data(), stab.data(), wtab.data());
        std::vector<float> out(size_t(A) * 6 * n);
        std::vector<std::int32_t> med(size_t(A) * 2 * n);
        KernelAst tr = parse_kernel("kernel trace_t05(img, n, ctab, stab, wtab, out, med, a0) { }");
        GridConfig cfg;
        cfg.grid = {std::uint32_t(A), 1, 1};
        cfg.block = {std::uint32_t(n), 1, 1};
        LaunchReport r = cuda_launch(ctx, tr, cfg,
                                     {cu_in(img), std::int32_t(n), cu_in(ctab), cu_in(stab), cu_in(wtab),
                                      cu_out(out), cu_out(med), std::int32_t(0)});
        CHECK(r.ok());
        std::vector<float> ref(out.size());
        std::vector<std::int32_t> rmed(med.size());
        tto_transform(img.data(), n, 0, A, A, ctab.data(), stab.data(), wtab.data(), 1, TTO_REPLAY, 0, ref.data(),
                      rmed.data(), nullptr, nullptr, 0);
        CHECK(std::memcmp(out.data(), ref.data(), out.size() * 4) == 0);
        CHECK(med == rmed);
        CHECK(ctx.counters().gpu_kernel_launches == 2);  // pass-2 weight layout of the uploaded wtab + fused kernel

        // the same transform through the pipelined host-to-host plan: identical bits
        b200::TracePlan plan(ctx, n, A, true, false, 0, -1, 1, 5);
        std::vector<float> out2(out.size(), -1.0f);
        std::vector<std::int32_t> med2(med.size(), -1);
        plan.run(img.data(), out2.data(), med2.data());
        CHECK(plan.chunks() == 5);
        CHECK(std::memcmp(out2.data(), out.data(), out.size() * 4) == 0);
        CHECK(med2 == med);
        CHECK(b200::prep_side(480, 640) == 801);
    }
    std::printf("%s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
