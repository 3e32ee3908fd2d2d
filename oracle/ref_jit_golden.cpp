// ref_jit_golden.cpp — golden vectors for the VPTX JIT (tests/test_jit_gpu.py).
// TEST INFRASTRUCTURE.  Each case is a DSL kernel compiled by the REFERENCE's
// own front end (parse_kernel -> specialize -> lower -> disassemble:
// /root/reference/proj/include/gridjit/{parser,specialize,codegen}.hpp) and
// run by its emulator through cuda_launch (autolaunch.hpp:167-245).  Writes
// one JSON document: per case the VPTX text the reference produced, the
// launch geometry, the inputs, the outputs (f32/i32 as uint32 bit patterns,
// f64/i64 as uint64) and the trap, if any.  Built by oracle/Makefile
// (target jit-golden) from the reference headers where they lie.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <iostream>
#include <limits>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "gridjit/gridjit.hpp"

using namespace gridjit;
using json = nlohmann::json;

namespace {

template <class T>
json bits(const std::vector<T>& v) {
    json a = json::array();
    for (const T& x : v) {
        if constexpr (sizeof(T) == 4) {
            std::uint32_t u;
            std::memcpy(&u, &x, 4);
            a.push_back(u);
        } else {
            std::uint64_t u;
            std::memcpy(&u, &x, 8);
            a.push_back(u);
        }
    }
    return a;
}

struct Arr {
    std::string type;  // f32 i32 f64 i64
    std::string dir;   // in out inout
    std::vector<float> f32;
    std::vector<std::int32_t> i32;
    std::vector<double> f64;
    std::vector<std::int64_t> i64;
};

struct Case {
    std::string name, src;
    std::uint32_t grid[3], block[3];
    std::uint64_t shared_extra = 0;
    std::vector<json> scalars;  // {"index", "type", "value"}
    std::vector<std::pair<int, Arr>> arrays;
    int nargs = 0;
};

template <class T>
KernelArg dir_arg(const std::string& d, std::vector<T>& v) {
    if (d == "in") return cu_in(v);
    if (d == "out") return cu_out(v);
    return cu_inout(v);
}

json run_case(Case& c) {
    KernelAst ast = parse_kernel(c.src);
    std::vector<KernelArg> args;
    std::vector<int> slot(c.nargs, -1);
    for (std::size_t i = 0; i < c.arrays.size(); ++i) slot[c.arrays[i].first] = int(i);
    json jin = json::array();
    for (int i = 0; i < c.nargs; ++i) {
        if (slot[i] >= 0) {
            Arr& a = c.arrays[slot[i]].second;
            json e = {{"index", i}, {"type", a.type + "[]"}, {"dir", a.dir}};
            if (a.type == "f32") e["data"] = bits(a.f32), args.push_back(dir_arg(a.dir, a.f32));
            else if (a.type == "i32") e["data"] = bits(a.i32), args.push_back(dir_arg(a.dir, a.i32));
            else if (a.type == "f64") e["data"] = bits(a.f64), args.push_back(dir_arg(a.dir, a.f64));
            else e["data"] = bits(a.i64), args.push_back(dir_arg(a.dir, a.i64));
            jin.push_back(e);
        } else {
            for (const json& s : c.scalars)
                if (s["index"] == i) {
                    jin.push_back(s);
                    const std::string t = s["type"];
                    if (t == "f32") args.emplace_back(float(s["value"].get<double>()));
                    else if (t == "f64") args.emplace_back(s["value"].get<double>());
                    else if (t == "i32") args.emplace_back(std::int32_t(s["value"].get<std::int64_t>()));
                    else args.emplace_back(s["value"].get<std::int64_t>());
                }
        }
    }
    std::vector<ArgType> types;
    for (const auto& a : args) types.push_back(a.arg_type());
    const std::string vptx = disassemble(lower(specialize(ast, types)));
    DeviceContext ctx = create_context();
    GridConfig cfg;
    for (int i = 0; i < 3; ++i) {
        cfg.grid[i] = c.grid[i];
        cfg.block[i] = c.block[i];
    }
    cfg.shared_bytes_extra = c.shared_extra;
    LaunchReport r = cuda_launch(ctx, ast, cfg, args);
    json out = json::object();
    for (auto& [idx, a] : c.arrays) {
        if (a.dir == "in") continue;
        if (a.type == "f32") out[std::to_string(idx)] = bits(a.f32);
        else if (a.type == "i32") out[std::to_string(idx)] = bits(a.i32);
        else if (a.type == "f64") out[std::to_string(idx)] = bits(a.f64);
        else out[std::to_string(idx)] = bits(a.i64);
    }
    json trap = nullptr;
    if (r.trap) {
        trap = {{"kind", int(r.trap->kind)},
                {"thread", {r.trap->thread[0], r.trap->thread[1], r.trap->thread[2]}},
                {"block", {r.trap->block[0], r.trap->block[1], r.trap->block[2]}},
                {"instr_index", r.trap->instr_index},
                {"code", r.trap->code}};
        out = json::object();  // downloads are skipped on a trap (autolaunch.hpp:235-243)
    }
    ctx.destroy();
    return {{"name", c.name},
            {"kernel", ast.name},
            {"source", c.src},
            {"vptx", vptx},
            {"grid", {c.grid[0], c.grid[1], c.grid[2]}},
            {"block", {c.block[0], c.block[1], c.block[2]}},
            {"shared_extra", c.shared_extra},
            {"args", jin},
            {"outputs", out},
            {"trap", trap}};
}

Arr f32(const std::string& dir, std::vector<float> v) { Arr a; a.type = "f32"; a.dir = dir; a.f32 = std::move(v); return a; }
Arr i32(const std::string& dir, std::vector<std::int32_t> v) { Arr a; a.type = "i32"; a.dir = dir; a.i32 = std::move(v); return a; }
Arr f64(const std::string& dir, std::vector<double> v) { Arr a; a.type = "f64"; a.dir = dir; a.f64 = std::move(v); return a; }
Arr i64(const std::string& dir, std::vector<std::int64_t> v) { Arr a; a.type = "i64"; a.dir = dir; a.i64 = std::move(v); return a; }

std::vector<float> ramp(int n, float a, float b) {
    std::vector<float> v(n);
    for (int i = 0; i < n; ++i) v[i] = a + b * float(i) * std::sin(float(i) * 0.37f);
    return v;
}

}  // namespace

// --trace-vptx <krn>: the VPTX the reference front end produces for the trace
// kernel's launch signature trace_t05(f32[], i32, f32[], f32[], f32[], f32[], i32[], i32).
int print_trace_vptx(const char* path) {
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    KernelAst ast = parse_kernel(ss.str());
    std::vector<float> fv(1);
    std::vector<std::int32_t> iv(1);
    std::vector<KernelArg> args = {cu_in(fv), std::int32_t(0), cu_in(fv), cu_in(fv), cu_in(fv),
                                   cu_out(fv), cu_out(iv), std::int32_t(0)};
    std::vector<ArgType> types;
    for (const auto& a : args) types.push_back(a.arg_type());
    std::cout << disassemble(lower(specialize(ast, types)));
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 3 && std::string(argv[1]) == "--trace-vptx") return print_trace_vptx(argv[2]);
    std::vector<Case> cases;
    const float nan = std::numeric_limits<float>::quiet_NaN(), inf = std::numeric_limits<float>::infinity();
    {  // the reference's sample kernels (proj/kernels/*.krn)
        Case c{"vadd_f32",
               "kernel vadd(a, b, c) {\n  i = block_id_x() + (thread_id_x() - 1) * num_blocks_x();\n  c[i] = a[i] + b[i];\n}\n",
               {12, 1, 1}, {1, 1, 1}};
        c.nargs = 3;
        c.arrays = {{0, f32("in", ramp(12, 1.0f, 0.5f))}, {1, f32("in", ramp(12, -2.0f, 0.25f))},
                    {2, f32("out", std::vector<float>(12))}};
        cases.push_back(c);
    }
    {
        Case c{"scale_f32_inout",
               "kernel scale(a, k) {\n  t = (block_id_x() - 1) * num_threads_x() + thread_id_x();\n  a[t] = a[t] * k;\n}\n",
               {4, 1, 1}, {8, 1, 1}};
        c.nargs = 2;
        c.arrays = {{0, f32("inout", ramp(32, 0.3f, 1.7f))}};
        c.scalars = {json{{"index", 1}, {"type", "f32"}, {"value", 2.5}}};
        cases.push_back(c);
    }
    {
        Case c{"reduce_shared_barriers",
               "kernel reduce(input, out) {\n  shared tmp[f32; 256];\n  t = thread_id_x();\n"
               "  g = (block_id_x() - 1) * num_threads_x() + t;\n  tmp[t] = input[g];\n  barrier();\n"
               "  stride = 1;\n  while (stride < num_threads_x()) {\n    if ((t - 1) % (2 * stride) == 0) {\n"
               "      tmp[t] = tmp[t] + tmp[t + stride];\n    }\n    barrier();\n    stride = stride * 2;\n  }\n"
               "  if (t == 1) {\n    out[block_id_x()] = tmp[1];\n  }\n}\n",
               {4, 1, 1}, {256, 1, 1}};
        c.nargs = 2;
        c.arrays = {{0, f32("in", ramp(1024, 0.1f, 0.01f))}, {1, f32("out", std::vector<float>(4))}};
        cases.push_back(c);
    }
    {  // integer / float / cvt corner cases: wrap, INT_MIN / -1, saturating and NaN float->int
        const int n = 16;
        std::vector<std::int32_t> a = {7, -7, 7, -7, INT32_MIN, INT32_MIN, 0, 1, 123456789, -5, 2147483647, 3, 9, -9, 100, 42};
        std::vector<std::int32_t> b = {2, 2, -2, -2, -1, 1, 5, 0, 1000, 0, 2, 3, -4, 4, -7, 1};
        std::vector<float> x = {1.5f, -2.25f, 3e9f, -3e9f, nan, inf, -inf, 0.0f, -0.0f, 1e-40f, 7.0f, 0.1f, 2.0f, -0.5f, 1e30f, 3.3f};
        std::vector<float> y = {0.5f, 4.0f, 1.0f, -1.0f, 2.0f, 1.0f, 0.0f, -0.0f, 0.0f, 3.0f, nan, 0.2f, 2.0f, -0.25f, 1e-30f, -3.3f};
        Case c{"mixed_ops",
               "kernel mixed(a, b, x, y, oi, of, od) {\n"
               "  t = (block_id_x() - 1) * num_threads_x() + thread_id_x();\n"
               "  ai = a[t];\n  bi = b[t];\n  q = 0;\n  r = 0;\n"
               "  if (bi != 0) {\n    q = ai / bi;\n    r = ai % bi;\n  }\n"
               "  oi[t] = q * 3 - r + min(ai, bi) + max(ai, bi) + abs(ai);\n"
               "  xf = x[t];\n  yf = y[t];\n"
               "  v = fma(xf, yf, sqrt(abs(xf))) - min(xf, yf) + max(xf, yf);\n"
               "  if (xf < yf || xf == yf) {\n    v = v * f32(2.0);\n  } else {\n    v = v - f32(1.5);\n  }\n"
               "  of[t] = v / (yf + f32(0.5));\n"
               "  ci = i32(xf * f32(1000.0));\n"
               "  od[t] = f64(ci) + f64(xf) * 0.5 + f64(i64(ai) * i64(bi)) - f64(i64(xf));\n"
               "}\n",
               {2, 1, 1}, {8, 1, 1}};
        c.nargs = 7;
        c.arrays = {{0, i32("in", a)}, {1, i32("in", b)}, {2, f32("in", x)}, {3, f32("in", y)},
                    {4, i32("out", std::vector<std::int32_t>(n))}, {5, f32("out", std::vector<float>(n))},
                    {6, f64("out", std::vector<double>(n))}};
        cases.push_back(c);
    }
    {  // 2-D grid / block, i64 arithmetic, while loop, f64
        Case c{"grid2d_loop_i64",
               "kernel g2(m, acc) {\n"
               "  x = (block_id_x() - 1) * num_threads_x() + thread_id_x();\n"
               "  y = (block_id_y() - 1) * num_threads_y() + thread_id_y();\n"
               "  w = num_blocks_x() * num_threads_x();\n"
               "  k = i64(0);\n  s = 0.0;\n  j = 1;\n"
               "  while (j <= x + y) {\n    k = k + i64(j) * i64(1000003);\n    s = s + f64(m[(y - 1) * w + x]) / f64(j);\n    j = j + 1;\n  }\n"
               "  acc[(y - 1) * w + x] = s + f64(k % i64(977));\n"
               "}\n",
               {2, 3, 1}, {4, 2, 1}};
        c.nargs = 2;
        std::vector<std::int64_t> m(48);
        for (int i = 0; i < 48; ++i) m[i] = std::int64_t(i) * 7919 - 100000;
        c.arrays = {{0, i64("in", m)}, {1, f64("out", std::vector<double>(48))}};
        cases.push_back(c);
    }
    {  // traps: first in the emulator's order (block, barrier phase, thread)
        Case c{"trap_global_oob",
               "kernel oob(a) {\n  t = (block_id_x() - 1) * num_threads_x() + thread_id_x();\n  a[t + 5] = f32(1.0);\n}\n",
               {2, 1, 1}, {8, 1, 1}};
        c.nargs = 1;
        c.arrays = {{0, f32("inout", std::vector<float>(12))}};
        cases.push_back(c);
    }
    {
        Case c{"trap_division_by_zero",
               "kernel dz(a, o) {\n  t = thread_id_x();\n  o[t] = 10 / a[t];\n}\n", {1, 1, 1}, {6, 1, 1}};
        c.nargs = 2;
        c.arrays = {{0, i32("in", {1, 2, 5, 0, 4, 0})}, {1, i32("out", std::vector<std::int32_t>(6))}};
        cases.push_back(c);
    }
    {
        Case c{"trap_shared_oob_after_barrier",
               "kernel sh(o) {\n  shared s[f32; 4];\n  t = thread_id_x();\n  s[t] = f32(t);\n  barrier();\n"
               "  o[t] = s[t + 1];\n}\n",
               {1, 1, 1}, {4, 1, 1}};
        c.nargs = 1;
        c.arrays = {{0, f32("out", std::vector<float>(4))}};
        cases.push_back(c);
    }
    {
        Case c{"trap_later_block",
               "kernel lb(a) {\n  b = block_id_x();\n  t = thread_id_x();\n  if (b >= 2 && t >= 3) {\n"
               "    a[100 * b + t] = f32(2.0);\n  }\n  a[t] = f32(b);\n}\n",
               {3, 1, 1}, {4, 1, 1}};
        c.nargs = 1;
        c.arrays = {{0, f32("inout", std::vector<float>(8))}};
        cases.push_back(c);
    }
    json all = json::array();
    for (Case& c : cases) all.push_back(run_case(c));
    std::cout << all.dump(1) << "\n";
    return 0;
}
