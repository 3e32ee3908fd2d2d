// ref_tier2.cpp — runs oracle/trace_t05.krn through the REFERENCE's own
// execution engine (gridjit cuda_launch on its emulated device). TEST
// INFRASTRUCTURE: the tier-2 oracle that pins oracle/tt_oracle.c (mode
// TTO_SEQ32) bit-exactly, and the CPU arm of `bench.py --impl reference`.
//
// Built by oracle/Makefile from the reference headers where they lie
// (/root/reference/proj/include; nothing is copied) into oracle/_ref/.
//
// Usage: tt_tier2 <in.bin> <out.bin> <a0> <a_count> <threads> [krn] [lines]
//   lines: only lines p < lines are launched (bounded benchmark samples)
//   in.bin : int32 n, int32 A, then f32 img[n*n], ctab[A], stab[A], wtab[8n]
//   out.bin: f32 out[a_count][6][n], int32 med[a_count][2][n]
//   stdout : one JSON line {"taps":..., "seconds":..., "threads":...}
//
// One DeviceContext per host thread, created serially: the reference's
// context-id counter is a non-atomic static (driver.hpp:279-282).  Angles are
// split into contiguous chunks per thread; each thread issues one cuda_launch
// per angle (grid = (1, ceil(n/B)), block = (B)).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gridjit/gridjit.hpp"

using namespace gridjit;

#ifndef TT_KRN_PATH
#define TT_KRN_PATH "oracle/trace_t05.krn"
#endif

static std::string slurp(const char* path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) {
        std::fprintf(stderr, "cannot open %s\n", path);
        std::exit(2);
    }
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s in.bin out.bin a0 a_count threads [krn]\n", argv[0]);
        return 2;
    }
    const int a0 = std::atoi(argv[3]);
    const int a_count = std::atoi(argv[4]);
    int nthreads = std::atoi(argv[5]);
    const char* krn = argc > 6 ? argv[6] : TT_KRN_PATH;
    int lines_arg = argc > 7 ? std::atoi(argv[7]) : 0;

    std::string in = slurp(argv[1]);
    const char* q = in.data();
    std::int32_t n, A;
    std::memcpy(&n, q, 4);
    std::memcpy(&A, q + 4, 4);
    q += 8;
    std::vector<float> img(size_t(n) * n), ctab(A), stab(A), wtab(size_t(8) * n);
    std::memcpy(img.data(), q, img.size() * 4);
    q += img.size() * 4;
    std::memcpy(ctab.data(), q, ctab.size() * 4);
    q += ctab.size() * 4;
    std::memcpy(stab.data(), q, stab.size() * 4);
    q += stab.size() * 4;
    std::memcpy(wtab.data(), q, wtab.size() * 4);

    KernelAst kernel = parse_kernel(slurp(krn));
    if (nthreads < 1) nthreads = 1;
    if (nthreads > a_count) nthreads = a_count;

    std::vector<float> out(size_t(a_count) * 6 * n, 0.0f);
    std::vector<std::int32_t> med(size_t(a_count) * 2 * n, 0);

    std::vector<DeviceContext> ctxs;
    for (int i = 0; i < nthreads; ++i) ctxs.push_back(create_context());

    const int lines = (lines_arg <= 0 || lines_arg > n) ? n : lines_arg;
    const std::uint32_t B = lines < 256 ? std::uint32_t(lines) : 256u;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    std::vector<int> failed(nthreads, 0);
    for (int th = 0; th < nthreads; ++th) {
        pool.emplace_back([&, th] {
            const int lo = a_count * th / nthreads, hi = a_count * (th + 1) / nthreads;
            // per-thread copies: KernelArg aliases caller storage (autolaunch.hpp:44-67)
            std::vector<float> img_l = img, ctab_l = ctab, stab_l = stab, wtab_l = wtab;
            std::vector<float> o(size_t(6) * n);
            std::vector<std::int32_t> m(size_t(2) * n);
            for (int ai = lo; ai < hi; ++ai) {
                GridConfig cfg;
                cfg.grid = {1, std::uint32_t((lines + B - 1) / B), 1};
                cfg.block = {B, 1, 1};
                LaunchReport rep = cuda_launch(ctxs[th], kernel, cfg,
                                               {cu_in(img_l), std::int32_t(n), cu_in(ctab_l), cu_in(stab_l),
                                                cu_in(wtab_l), cu_out(o), cu_out(m), std::int32_t(a0 + ai)});
                if (!rep.ok()) {
                    std::fprintf(stderr, "trap: %s\n", rep.trap->to_string().c_str());
                    failed[th] = 1;
                    return;
                }
                std::memcpy(out.data() + size_t(ai) * 6 * n, o.data(), o.size() * 4);
                std::memcpy(med.data() + size_t(ai) * 2 * n, m.data(), m.size() * 4);
            }
        });
    }
    for (auto& t : pool) t.join();
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int f : failed)
        if (f) return 1;

    std::ofstream of(argv[2], std::ios::binary);
    of.write(reinterpret_cast<const char*>(out.data()), std::streamsize(out.size() * 4));
    of.write(reinterpret_cast<const char*>(med.data()), std::streamsize(med.size() * 4));
    std::printf("{\"taps\": %llu, \"lines\": %llu, \"seconds\": %.6f, \"threads\": %d}\n",
                (unsigned long long)(std::uint64_t(a_count) * lines * n), (unsigned long long)(std::uint64_t(a_count) * lines),
                secs, nthreads);
    return 0;
}
