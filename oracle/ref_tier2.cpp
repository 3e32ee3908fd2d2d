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
//        tt_tier2 circus <in.bin> <out.bin> <threads> [circus.krn]
//   in.bin : int32 n, int32 rows, f32 sino[rows*n]; out.bin: f32 circ[rows][3]
//        tt_tier2 bench <n> <A> <angles> <lines> <circus_rows> <threads> <krn_dir>
//   the benchmark arm: generates its own inputs (tto_synth DISK, tto_tables:
//   the oracle's C restatement, linked in), then times ONLY the emulator
//   launches -- trace_t05.krn over `angles` angles x `lines` lines and
//   circus.krn over `circus_rows` rows -- and prints one JSON line.
//
// One DeviceContext per host thread, created serially: the reference's
// context-id counter is a non-atomic static (driver.hpp:279-282).  Angles are
// split into contiguous chunks per thread; each thread issues one cuda_launch
// per angle (grid = (1, ceil(n/B)), block = (B)).
#include <algorithm>
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

extern "C" {
void tto_tables(int n, int a_total, float* ctab, float* stab, float* wtab);
void tto_synth(int kind, std::uint64_t seed, int n, float* img);
}

// One cuda_launch per angle on per-thread contexts (created serially by the caller).
// Returns the launch-only wall time (s), or -1 on a trap.
static double run_trace(std::vector<DeviceContext>& ctxs, const KernelAst& kernel, int n, int a0, int a_count,
                        int lines, const std::vector<float>& img, const std::vector<float>& ctab,
                        const std::vector<float>& stab, const std::vector<float>& wtab, std::vector<float>& out,
                        std::vector<std::int32_t>& med) {
    const int nthreads = int(ctxs.size());
    const std::uint32_t B = lines < 256 ? std::uint32_t(lines) : 256u;
    std::vector<int> failed(nthreads, 0);
    // per-thread copies: KernelArg aliases caller storage (autolaunch.hpp:44-67); made before the clock starts
    std::vector<std::vector<float>> img_l(nthreads, img), ctab_l(nthreads, ctab), stab_l(nthreads, stab),
        wtab_l(nthreads, wtab);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < nthreads; ++th) {
        pool.emplace_back([&, th] {
            const int lo = a_count * th / nthreads, hi = a_count * (th + 1) / nthreads;
            std::vector<float> o(size_t(6) * n);
            std::vector<std::int32_t> m(size_t(2) * n);
            for (int ai = lo; ai < hi; ++ai) {
                GridConfig cfg;
                cfg.grid = {1, std::uint32_t((lines + B - 1) / B), 1};
                cfg.block = {B, 1, 1};
                LaunchReport rep = cuda_launch(ctxs[th], kernel, cfg,
                                               {cu_in(img_l[th]), std::int32_t(n), cu_in(ctab_l[th]),
                                                cu_in(stab_l[th]), cu_in(wtab_l[th]), cu_out(o), cu_out(m),
                                                std::int32_t(a0 + ai)});
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
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int f : failed)
        if (f) return -1.0;
    return secs;
}

// circus.krn over rows [0, rows) of sino (one emulated thread per row), rows split
// into contiguous chunks per host thread.  Returns the launch-only wall time (s).
static double run_circus(std::vector<DeviceContext>& ctxs, const KernelAst& kernel, int n, int rows,
                         const std::vector<float>& sino, std::vector<float>& circ) {
    const int nthreads = int(ctxs.size());
    std::vector<int> failed(nthreads, 0);
    std::vector<std::vector<float>> parts(nthreads);
    for (int th = 0; th < nthreads; ++th) {
        const int lo = rows * th / nthreads, hi = rows * (th + 1) / nthreads;
        parts[th].assign(sino.begin() + size_t(lo) * n, sino.begin() + size_t(hi) * n);
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int th = 0; th < nthreads; ++th) {
        pool.emplace_back([&, th] {
            const int lo = rows * th / nthreads, hi = rows * (th + 1) / nthreads, cnt = hi - lo;
            if (cnt <= 0) return;
            std::vector<float> c(size_t(cnt) * 3);
            const std::uint32_t B = cnt < 256 ? std::uint32_t(cnt) : 256u;
            GridConfig cfg;
            cfg.grid = {std::uint32_t((cnt + B - 1) / B), 1, 1};
            cfg.block = {B, 1, 1};
            LaunchReport rep = cuda_launch(ctxs[th], kernel, cfg,
                                           {cu_in(parts[th]), std::int32_t(n), std::int32_t(cnt), cu_out(c)});
            if (!rep.ok()) {
                std::fprintf(stderr, "trap: %s\n", rep.trap->to_string().c_str());
                failed[th] = 1;
                return;
            }
            std::memcpy(circ.data() + size_t(lo) * 3, c.data(), c.size() * 4);
        });
    }
    for (auto& t : pool) t.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int f : failed)
        if (f) return -1.0;
    return secs;
}

static std::vector<DeviceContext> make_contexts(int nthreads) {
    std::vector<DeviceContext> ctxs;  // serially: the context-id counter is a non-atomic static (driver.hpp:279-282)
    for (int i = 0; i < nthreads; ++i) ctxs.push_back(create_context());
    return ctxs;
}

static int main_circus(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s circus in.bin out.bin threads [circus.krn]\n", argv[0]);
        return 2;
    }
    std::string in = slurp(argv[2]);
    std::int32_t n, rows;
    std::memcpy(&n, in.data(), 4);
    std::memcpy(&rows, in.data() + 4, 4);
    std::vector<float> sino(size_t(rows) * n), circ(size_t(rows) * 3, 0.0f);
    std::memcpy(sino.data(), in.data() + 8, sino.size() * 4);
    int nthreads = std::max(1, std::min(std::atoi(argv[4]), std::max(rows, 1)));
    KernelAst kernel = parse_kernel(slurp(argc > 5 ? argv[5] : "oracle/circus.krn"));
    auto ctxs = make_contexts(nthreads);
    const double secs = run_circus(ctxs, kernel, n, rows, sino, circ);
    if (secs < 0) return 1;
    std::ofstream of(argv[3], std::ios::binary);
    of.write(reinterpret_cast<const char*>(circ.data()), std::streamsize(circ.size() * 4));
    std::printf("{\"rows\": %d, \"seconds\": %.6f, \"threads\": %d}\n", rows, secs, nthreads);
    return 0;
}

static int main_bench(int argc, char** argv) {
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s bench n A angles lines circus_rows threads krn_dir\n", argv[0]);
        return 2;
    }
    const int n = std::atoi(argv[2]), A = std::atoi(argv[3]);
    const int angles = std::max(1, std::min(std::atoi(argv[4]), A));
    const int lines = std::max(1, std::min(std::atoi(argv[5]), n));
    const int crow = std::max(0, std::atoi(argv[6]));
    const int nthreads = std::max(1, std::atoi(argv[7]));
    const std::string dir = argv[8];
    std::vector<float> img(size_t(n) * n), ctab(A), stab(A), wtab(size_t(8) * n);
    tto_synth(0, 20160412ull, n, img.data());  // DISK, the GPU line's image
    tto_tables(n, A, ctab.data(), stab.data(), wtab.data());
    const KernelAst tk = parse_kernel(slurp((dir + "/trace_t05.krn").c_str()));
    const KernelAst ck = parse_kernel(slurp((dir + "/circus.krn").c_str()));
    auto ctxs = make_contexts(std::min(nthreads, angles));
    std::vector<float> out(size_t(angles) * 6 * n, 0.0f);
    std::vector<std::int32_t> med(size_t(angles) * 2 * n, 0);
    const double ts = run_trace(ctxs, tk, n, 0, angles, lines, img, ctab, stab, wtab, out, med);
    if (ts < 0) return 1;
    double cs = 0.0;
    if (crow > 0) {  // circus rows: image rows (the stage's cost is value-independent: fixed-length loops)
        std::vector<float> sino(size_t(crow) * n), circ(size_t(crow) * 3);
        for (int r = 0; r < crow; ++r)
            std::memcpy(sino.data() + size_t(r) * n, img.data() + size_t(r % n) * n, size_t(n) * 4);
        auto cctx = make_contexts(std::min(nthreads, crow));
        cs = run_circus(cctx, ck, n, crow, sino, circ);
        if (cs < 0) return 1;
    }
    double sum = 0.0;  // keeps the outputs observable
    for (int a = 0; a < angles; ++a)
        for (int p = 0; p < lines; ++p) sum += out[size_t(a) * 6 * n + p];
    std::printf("{\"trace_lines\": %llu, \"trace_taps\": %llu, \"trace_seconds\": %.6f, \"circus_rows\": %d, "
                "\"circus_seconds\": %.6f, \"threads\": %d, \"checksum\": %.9g}\n",
                (unsigned long long)(std::uint64_t(angles) * lines),
                (unsigned long long)(std::uint64_t(angles) * lines * n), ts, crow, cs, int(ctxs.size()), sum);
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "circus") == 0) return main_circus(argc, argv);
    if (argc > 1 && std::strcmp(argv[1], "bench") == 0) return main_bench(argc, argv);
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s in.bin out.bin a0 a_count threads [krn] [lines]\n", argv[0]);
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
    auto ctxs = make_contexts(nthreads);
    const int lines = (lines_arg <= 0 || lines_arg > n) ? n : lines_arg;
    const double secs = run_trace(ctxs, kernel, n, a0, a_count, lines, img, ctab, stab, wtab, out, med);
    if (secs < 0) return 1;

    std::ofstream of(argv[2], std::ios::binary);
    of.write(reinterpret_cast<const char*>(out.data()), std::streamsize(out.size() * 4));
    of.write(reinterpret_cast<const char*>(med.data()), std::streamsize(med.size() * 4));
    std::printf("{\"taps\": %llu, \"lines\": %llu, \"seconds\": %.6f, \"threads\": %d}\n",
                (unsigned long long)(std::uint64_t(a_count) * lines * n), (unsigned long long)(std::uint64_t(a_count) * lines),
                secs, nthreads);
    return 0;
}
