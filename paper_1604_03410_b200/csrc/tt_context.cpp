// tt_context.cpp — the CUDA-backed device context behind the C ABI
// (include/tt_b200.h): device memory manager, module/function handles, the
// native-kernel registry, launch validation/dispatch and exact counters.
//
// It re-implements, B200-first, the contract of the reference's
// DeviceContext (/root/reference/proj/include/gridjit/driver.hpp:112-330):
//   - the same handle rules (stale/foreign handles, poisoned contexts);
//   - the same byte-exact Counters and launch log (driver.hpp:54-96,235-246);
//   - the same allocation semantics: zero-filled buffers, 0-byte allocations
//     distinct and non-null, addresses never reused so UseAfterFree stays
//     detectable (emulator.hpp:104-117) — here a synthetic address table over
//     a stream-ordered cudaMallocAsync pool that DOES recycle HBM;
//   - the same validation order for launches (driver.hpp:221-233 then
//     KernelImage, emulator.hpp:217-272), with kernel faults returned as
//     TrapInfo-shaped values.
// The emulated execution engine (emulator.hpp run_kernel) is replaced by the
// sm_100a kernels in tt_kernels.cu; nothing here computes on the CPU.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <array>
#include <atomic>
#include <cctype>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include <cudaTypedefs.h>
#include <mutex>

#include "tt_context_impl.h"


namespace ttc {

namespace {
std::atomic<std::uint64_t> g_next_ctx_id{0};
thread_local std::string t_last_error;
}  // namespace

tt_status fail(const tt_ctx* ctx, tt_status st, const std::string& msg) {
    if (ctx) const_cast<tt_ctx*>(ctx)->last_error = msg;
    t_last_error = msg;
    return st;
}

tt_status cuda_fail(const tt_ctx* ctx, cudaError_t e, const char* what) {
    return fail(ctx, TT_ERR_CUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace ttc

namespace ttc {
tt_status copy_out_text(const std::string& s, char* buf, std::size_t cap, std::size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (buf == nullptr || cap == 0) return TT_OK;
    if (cap < s.size() + 1) return fail(nullptr, TT_ERR_INVALID, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return TT_OK;
}
}  // namespace ttc

using namespace ttc;

namespace {

const std::vector<NativeKernel>& registry();  // the native sm_100a kernels, defined below

void drop_weights(tt_ctx* ctx, std::uint64_t base) {
    auto it = ctx->w_cache.find(base);
    if (it == ctx->w_cache.end()) return;
    if (it->second.d) cudaFreeAsync(it->second.d, ctx->stream);  // stream-ordered after its readers
    ctx->w_cache.erase(it);
}

void drop_texture(tt_ctx* ctx, std::uint64_t base) {
    auto it = ctx->tex_cache.find(base);
    if (it == ctx->tex_cache.end()) return;
    cudaStreamSynchronize(ctx->stream);
    cudaDestroyTextureObject(it->second.tex);
    if (it->second.arr) cudaFreeArray(it->second.arr);
    ctx->tex_cache.erase(it);
}





void finish_launch_log(tt_ctx* ctx) {  // driver.hpp:322-325
    if (!ctx->launch_log.empty()) ctx->launch_log.back().d2h = ctx->c.bytes_d2h - ctx->d2h_mark;
}

// check_owned + liveness (driver.hpp:291-294, GlobalMemory::is_live).
tt_status lookup(tt_ctx* ctx, const tt_devptr& p, Alloc** out) {
    if (p.ctx_id != ctx->id) return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: device pointer belongs to another context");
    if (p.base == 0) return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: null device pointer");
    auto it = ctx->allocs.find(p.base);
    if (it == ctx->allocs.end() || !it->second.live) return fail(ctx, TT_ERR_USE_AFTER_FREE, "UseAfterFree: device pointer no longer live");
    *out = &it->second;
    return TT_OK;
}

// ------------------------------------------------- VPTX header parsing

struct Line {
    int no = 0;
    std::vector<std::string> toks;
};

std::vector<Line> tokenize(const char* text, std::size_t len) {
    std::vector<Line> lines;
    std::size_t pos = 0;
    int no = 0;
    while (pos <= len) {
        std::size_t eol = pos;
        while (eol < len && text[eol] != '\n') ++eol;
        ++no;
        Line l;
        l.no = no;
        std::size_t i = pos;
        while (i < eol) {
            char ch = text[i];
            if (ch == '#') break;
            if (ch == ' ' || ch == '\t' || ch == '\r') {
                ++i;
                continue;
            }
            if (ch == ',' || ch == '(' || ch == ')' || ch == '[' || ch == ']' || ch == '{' || ch == '}') {
                l.toks.emplace_back(1, ch);
                ++i;
                continue;
            }
            std::size_t s = i;
            while (i < eol && text[i] != ' ' && text[i] != '\t' && text[i] != '\r' && text[i] != ',' &&
                   text[i] != '(' && text[i] != ')' && text[i] != '[' && text[i] != ']' && text[i] != '{' &&
                   text[i] != '}' && text[i] != '#')
                ++i;
            l.toks.emplace_back(text + s, i - s);
        }
        if (!l.toks.empty()) lines.push_back(std::move(l));
        if (eol >= len) break;
        pos = eol + 1;
    }
    return lines;
}

bool parse_scalar(const std::string& s, Scalar& t) {
    if (s == "i32") t = Scalar::I32;
    else if (s == "i64") t = Scalar::I64;
    else if (s == "f32") t = Scalar::F32;
    else if (s == "f64") t = Scalar::F64;
    else return false;
    return true;
}

bool parse_param_type(const std::string& s, Param& p) {  // vptx.hpp:739-752
    if (s.rfind("ptr.global.", 0) == 0) {
        p.ptr = true;
        return parse_scalar(s.substr(11), p.type);
    }
    p.ptr = false;
    return parse_scalar(s, p.type);
}

bool is_name(const std::string& s) {
    if (s.empty()) return false;
    for (char ch : s)
        if (!(std::isalnum((unsigned char)ch) || ch == '_' || ch == '$' || ch == '.' || ch == '%')) return false;
    return !std::isdigit((unsigned char)s[0]);
}

// Parses the module header and kernel signatures (vptx.hpp:398-488); kernel
// bodies are skipped — they are bound to native sm_100a kernels instead.
tt_status parse_module(tt_ctx* ctx, const char* text, std::size_t len, Module& m) {
    auto syntax = [&](int line, const std::string& msg) {
        return fail(ctx, TT_ERR_VPTX_SYNTAX, "VptxSyntaxError at line " + std::to_string(line) + ": " + msg);
    };
    std::vector<Line> lines = tokenize(text, len);
    if (lines.empty()) return syntax(1, "empty module text");
    std::size_t li = 0;
    {
        const Line& l = lines[li++];
        if (l.toks[0] != ".module") return syntax(l.no, "expected '.module', got '" + l.toks[0] + "'");
        if (l.toks.size() < 2 || !is_name(l.toks[1])) return syntax(l.no, "expected module name");
        if (l.toks.size() > 2) return syntax(l.no, "trailing text '" + l.toks[2] + "' after .module");
        m.name = l.toks[1];
    }
    while (li < lines.size()) {
        const Line& h = lines[li++];
        const auto& t = h.toks;
        std::size_t k = 0;
        auto take = [&](const char* what, std::string& out) -> bool {
            if (k >= t.size()) return false;
            out = t[k++];
            (void)what;
            return true;
        };
        std::string tok;
        if (!take("kernel", tok) || tok != ".kernel") return syntax(h.no, "expected '.kernel', got '" + t[0] + "'");
        KernelDecl kd;
        if (!take("name", kd.name) || !is_name(kd.name)) return syntax(h.no, "expected kernel name");
        if (!take("(", tok) || tok != "(") return syntax(h.no, "expected '('");
        if (k < t.size() && t[k] == ")") {
            ++k;
        } else {
            while (true) {
                if (!take("param", tok) || tok != ".param") return syntax(h.no, "expected '.param'");
                Param p;
                std::string ty;
                if (!take("type", ty) || !parse_param_type(ty, p))
                    return syntax(h.no, "bad parameter type '" + ty + "'");
                if (!take("pname", p.name) || !is_name(p.name)) return syntax(h.no, "expected parameter name");
                kd.params.push_back(p);
                if (!take(",", tok)) return syntax(h.no, "unterminated parameter list");
                if (tok == ",") continue;
                if (tok == ")") break;
                return syntax(h.no, "expected ',' or ')', got '" + tok + "'");
            }
        }
        if (!take("{", tok) || tok != "{") return syntax(h.no, "expected '{'");
        if (k != t.size()) return syntax(h.no, "trailing text '" + t[k] + "' after .kernel header");
        bool closed = false;
        while (li < lines.size()) {
            const Line& b = lines[li++];
            if (b.toks[0] == "}") {
                if (b.toks.size() != 1) return syntax(b.no, "trailing text after kernel");
                closed = true;
                break;
            }
            kd.body.push_back(tt::jit::Line{b.no, b.toks});
        }
        if (!closed) return syntax(lines.back().no, "unterminated kernel body");
        for (const auto& other : m.kernels)
            if (other.name == kd.name)
                return fail(ctx, TT_ERR_VALIDATION_FAILED,
                            "ValidationFailed:\n  duplicate kernel name '" + kd.name + "'");
        m.kernels.push_back(std::move(kd));
    }
    return TT_OK;
}

const NativeKernel* find_native(const KernelDecl& d) {
    for (const auto& nk : registry()) {
        if (nk.decl.name != d.name || nk.decl.params.size() != d.params.size()) continue;
        bool same = true;
        for (std::size_t i = 0; i < d.params.size(); ++i) same = same && (nk.decl.params[i] == d.params[i]);
        if (same) return &nk;
    }
    return nullptr;
}

// ------------------------------------------------------- native launchers

tt_trap first_thread_trap(tt_trap_kind kind) {
    tt_trap t{};
    t.trapped = 1;
    t.kind = kind;
    for (int i = 0; i < 3; ++i) t.thread[i] = t.block[i] = 1;
    return t;
}

LaunchOutcome cuda_outcome(cudaError_t e, const char* what) {
    LaunchOutcome o;
    if (e != cudaSuccess) {
        o.status = TT_ERR_CUDA;
        o.error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    }
    return o;
}

std::uint64_t elems(const ResolvedArg& a, std::size_t esz) { return a.bytes / esz; }

// vadd: i = block + thread * blocks over x (0-based form of vadd.krn:3-6).
// The first faulting thread in the emulator's schedule (blocks
// lexicographic, threads linear, emulator.hpp:7-11) is reported.
template <tt::ElemKind K, std::size_t ESZ>
LaunchOutcome run_vadd(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    const std::uint64_t gx = g.grid[0], bx = g.block[0];
    const std::uint64_t need = gx * bx;
    const std::uint64_t len = std::min(elems(a[0], ESZ), std::min(elems(a[1], ESZ), elems(a[2], ESZ)));
    if (need > len) {
        LaunchOutcome o;
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        const std::uint64_t span = (bx - 1) * gx;  // largest thread offset
        const std::uint64_t x = len > span ? len - span : 0;
        const std::uint64_t tx = (len > x) ? (len - x + gx - 1) / gx : 0;
        o.trap.block[0] = std::uint32_t(x + 1);
        o.trap.thread[0] = std::uint32_t(tx + 1);
        return o;
    }
    LaunchOutcome o = cuda_outcome(tt::launch_vadd(K, a[0].dptr, a[1].dptr, a[2].dptr, need, ctx.stream), "vadd");
    o.gpu_launches = need > 0 ? 1 : 0;
    return o;
}

// scale(a, k): a[tid] *= k, tid over block.x (scale.krn:2-5).
LaunchOutcome run_scale(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    const std::uint64_t need = g.block[0];
    if (need > elems(a[0], 4)) {
        LaunchOutcome o;
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        o.trap.thread[0] = std::uint32_t(elems(a[0], 4) + 1);
        return o;
    }
    LaunchOutcome o = cuda_outcome(tt::launch_scale_f32((float*)a[0].dptr, a[1].value.v.f32, need, ctx.stream), "scale");
    o.gpu_launches = 1;
    return o;
}

// copy(a, b): b[tid] = a[tid] (test_autolaunch.cpp:26-28).
LaunchOutcome run_copy(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    const std::uint64_t need = g.block[0];
    if (need > std::min(elems(a[0], 4), elems(a[1], 4))) {
        LaunchOutcome o;
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        o.trap.thread[0] = std::uint32_t(std::min(elems(a[0], 4), elems(a[1], 4)) + 1);
        return o;
    }
    LaunchOutcome o = cuda_outcome(tt::launch_copy_f32((const float*)a[0].dptr, (float*)a[1].dptr, need, ctx.stream), "copy");
    o.gpu_launches = 1;
    return o;
}

// add_to(inp, out): out[t] = inp[t] + out[t] (test_autolaunch.cpp:145).
LaunchOutcome run_add_to(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    const std::uint64_t need = g.block[0];
    if (need > std::min(elems(a[0], 4), elems(a[1], 4))) {
        LaunchOutcome o;
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        o.trap.thread[0] = std::uint32_t(std::min(elems(a[0], 4), elems(a[1], 4)) + 1);
        return o;
    }
    LaunchOutcome o = cuda_outcome(tt::launch_add_to_f32((const float*)a[0].dptr, (float*)a[1].dptr, need, ctx.stream), "add_to");
    o.gpu_launches = 1;
    return o;
}

// Shared validation of the trace kernels' logical launch: grid.x angles
// starting at a0, lines p covered by grid.y * block.x threads (the DSL
// kernel oracle/trace_t05.krn computes p = (block_y-1)*threads_x + thread_x-1).
LaunchOutcome run_trace_common(tt_ctx& ctx, const tt_grid& g, const ResolvedArg& img, int n, const ResolvedArg& ct,
                               const ResolvedArg& st, const ResolvedArg* wt, const ResolvedArg& out,
                               const ResolvedArg* med, int a0, bool full, int batch = 1) {
    LaunchOutcome o;
    const std::int64_t a_count = g.grid[0];
    if (n <= 0 || batch <= 0) return o;  // every thread fails `p < n` (or no image): no work
    if (batch > 1 && std::uint64_t(g.grid[2]) < std::uint64_t(batch)) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: trace_t05_batch requires grid.z >= batch (one z-slice per image)";
        return o;
    }
    if (std::uint64_t(g.grid[1]) * g.block[0] < std::uint64_t(n)) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: native trace kernels require grid.y*block.x >= n (every line covered)";
        return o;
    }
    if (n > (full ? tt::max_full_n() : 32768)) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: n=" + std::to_string(n) + " exceeds the native kernel limit " +
                  std::to_string(full ? tt::max_full_n() : 32768);
        return o;
    }
    const std::uint64_t N = std::uint64_t(n);
    const std::int64_t F = full ? tt::kNumF : 1;
    const std::uint64_t B = std::uint64_t(batch);
    bool oob = a0 < 0 || elems(img, 4) < B * N * N || std::int64_t(elems(ct, 4)) < a0 + a_count ||
               std::int64_t(elems(st, 4)) < a0 + a_count || elems(out, 4) < B * std::uint64_t(a_count * F) * N;
    if (wt) oob = oob || elems(*wt, 4) < 8 * N;
    if (med) oob = oob || elems(*med, 4) < B * std::uint64_t(a_count) * 2 * N;
    if (oob) {
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        return o;
    }
    tt::TraceArgs ta;
    ta.img = (const float*)img.dptr;
    ta.n = n;
    ta.a0 = a0;
    tt::launch_structure(int(a_count), &ta.a_count, &ta.pair_stride);
    ta.ctab = (const float*)ct.dptr;
    ta.stab = (const float*)st.dptr;
    ta.wtab = wt ? (const float*)wt->dptr : nullptr;
    ta.out = (float*)out.dptr;
    ta.med = med ? (std::int32_t*)med->dptr : nullptr;
    ta.full = full;
    ta.batch = batch;
    ta.sampler = tt::Sampler(ctx.sampler == 3 ? 2 : ctx.sampler);  // 3 (auto): tiles only where they pay
    if (ta.sampler == tt::Sampler::Tma && !(ctx.sampler == 3 ? tt::tma_radon_pays(ta) : tt::tma_radon_ok(ta)))
        ta.sampler = tt::Sampler::Texture;
    if (ta.sampler == tt::Sampler::Texture) {
        TexEntry& te = ctx.tex_cache[img.base];
        const bool view = te.tex != 0 && te.arr == nullptr;  // pitch-linear view of the allocation (small n)
        if (te.tex == 0 || te.n != n || te.batch != batch || (view && te.bound != ta.img)) {
            if (te.tex) {
                cudaStreamSynchronize(ctx.stream);
                cudaDestroyTextureObject(te.tex);
                if (te.arr) cudaFreeArray(te.arr);
                te = TexEntry{};
            }
            cudaError_t e = batch > 1 ? tt::make_image_atlas(ta.img, n, batch, (long long)N * N, ctx.stream, &te.arr,
                                                              &te.tex, &te.cols)
                                      : tt::make_image_texture(ta.img, n, ctx.stream, &te.arr, &te.tex);
            if (e != cudaSuccess) {
                ctx.tex_cache.erase(img.base);
                return cuda_outcome(e, "image texture");
            }
            te.n = n;
            te.batch = batch;
            te.gen = img.gen;
            te.bound = ta.img;
        } else if (!view && (te.gen != img.gen || img.exported)) {  // image (maybe) rewritten since the copy: refresh
            cudaError_t e = batch > 1 ? tt::fill_image_atlas(te.arr, ta.img, n, batch, (long long)N * N, te.cols,
                                                              ctx.stream)
                                      : cudaMemcpy2DToArrayAsync(te.arr, 0, 0, ta.img, std::size_t(n) * 4,
                                                                 std::size_t(n) * 4, std::size_t(n),
                                                                 cudaMemcpyDeviceToDevice, ctx.stream);
            if (e != cudaSuccess) return cuda_outcome(e, "texture refresh");
            te.gen = img.gen;
        }
        ta.atlas_cols = te.cols;
        ta.tex = te.tex;
    }
    int extra_launches = 0;
    if (full) {
        WeightEntry& we = ctx.w_cache[wt->base];
        if (we.d == nullptr || we.n != n || we.gen != wt->gen || wt->exported) {
            if (we.d == nullptr || we.n != n) {
                if (we.d) cudaFreeAsync(we.d, ctx.stream);
                we = WeightEntry{};
                cudaError_t e = cudaMallocAsync((void**)&we.d, tt::weights_soa_bytes(n), ctx.stream);
                if (e != cudaSuccess) {
                    ctx.w_cache.erase(wt->base);
                    return cuda_outcome(e, "weight table");
                }
                we.n = n;
            }
            cudaError_t e = tt::launch_weights_soa(ta.wtab, n, we.d, ctx.stream);
            if (e != cudaSuccess) return cuda_outcome(e, "weight table");
            we.gen = wt->gen;
            extra_launches = 1;
        }
        ta.wsoa = we.d;
    }
    o = cuda_outcome(tt::launch_trace(ta, ctx.stream), "trace kernel");
    o.gpu_launches = tt::trace_launch_count(ta) + extra_launches;
    return o;
}

// trace_t05(img, n, ctab, stab, wtab, out, med, a0): the signature of the
// DSL kernel oracle/trace_t05.krn, bound to the fused sm_100a kernel.
LaunchOutcome run_trace_t05(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    return run_trace_common(ctx, g, a[0], a[1].value.v.i32, a[2], a[3], &a[4], a[5], &a[6], a[7].value.v.i32, true);
}

// trace_t05_batch(img, n, ctab, stab, wtab, out, med, a0, batch): the same
// kernel over `batch` images stacked [batch][n][n] (outputs stacked per image;
// logical grid.z = batch) -- batched feature extraction (config C4).
LaunchOutcome run_trace_t05_batch(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    return run_trace_common(ctx, g, a[0], a[1].value.v.i32, a[2], a[3], &a[4], a[5], &a[6], a[7].value.v.i32, true,
                            a[8].value.v.i32);
}

// radon(img, n, ctab, stab, out, a0): T0 only (SURVEY.md Appendix B's kernel
// with an explicit first angle).
LaunchOutcome run_radon(tt_ctx& ctx, const tt_grid& g, const std::vector<ResolvedArg>& a) {
    return run_trace_common(ctx, g, a[0], a[1].value.v.i32, a[2], a[3], nullptr, a[4], nullptr, a[5].value.v.i32, false);
}

// circus(sino, n, rows, circ): P-functionals of `rows` sinogram rows of length
// n -> circ[rows][3]; the consumer stage of trace_t05.
LaunchOutcome run_circus(tt_ctx& ctx, const tt_grid&, const std::vector<ResolvedArg>& a) {
    LaunchOutcome o;
    const int n = a[1].value.v.i32, rows = a[2].value.v.i32;
    if (n <= 0 || rows <= 0) return o;
    if (elems(a[0], 4) < std::uint64_t(n) * std::uint64_t(rows) || elems(a[3], 4) < 3ull * std::uint64_t(rows)) {
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        return o;
    }
    o = cuda_outcome(tt::launch_circus((const float*)a[0].dptr, n, rows, (float*)a[3].dptr, ctx.stream), "circus");
    o.gpu_launches = 1;
    return o;
}

// circus_fft(sino, n, rows, pf): the spectral P-functional sum_k |F(s)_k|^4 of
// each row -> pf[rows] (f64).
LaunchOutcome run_circus_fft(tt_ctx& ctx, const tt_grid&, const std::vector<ResolvedArg>& a) {
    LaunchOutcome o;
    const int n = a[1].value.v.i32, rows = a[2].value.v.i32;
    if (n <= 0 || rows <= 0) return o;
    if (n > tt::max_circus_fft_n()) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: circus_fft row length above 16384";
        return o;
    }
    if (elems(a[0], 4) < std::uint64_t(n) * std::uint64_t(rows) || elems(a[3], 8) < std::uint64_t(rows)) {
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        return o;
    }
    o = cuda_outcome(tt::launch_circus_fft((const float*)a[0].dptr, n, rows, (double*)a[3].dptr, ctx.stream),
                     "circus_fft");
    o.gpu_launches = 1;
    return o;
}

// hermite(sino, n, rows, orders, hp, center): Hermite P-functionals of each row around its weighted
// median -> hp[rows][orders] (f64), center[rows].
LaunchOutcome run_hermite(tt_ctx& ctx, const tt_grid&, const std::vector<ResolvedArg>& a) {
    LaunchOutcome o;
    const int n = a[1].value.v.i32, rows = a[2].value.v.i32, orders = a[3].value.v.i32;
    if (n <= 0 || rows <= 0) return o;
    if (orders < 1 || orders > tt::max_hermite_orders()) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: hermite orders must be 1..8";
        return o;
    }
    if (elems(a[0], 4) < std::uint64_t(n) * std::uint64_t(rows) ||
        elems(a[4], 8) < std::uint64_t(rows) * std::uint64_t(orders) || elems(a[5], 4) < std::uint64_t(rows)) {
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        return o;
    }
    o = cuda_outcome(tt::launch_hermite((const float*)a[0].dptr, n, rows, orders, (double*)a[4].dptr,
                                        (std::int32_t*)a[5].dptr, ctx.stream),
                     "hermite");
    o.gpu_launches = 1;
    return o;
}

// orthonormal(img, h, w, angles, out): the square-sinogram input frame -> out[angles][angles].
LaunchOutcome run_orthonormal(tt_ctx& ctx, const tt_grid&, const std::vector<ResolvedArg>& a) {
    LaunchOutcome o;
    const int h = a[1].value.v.i32, w = a[2].value.v.i32, A = a[3].value.v.i32;
    if (h <= 0 || w <= 0 || A < 2) {
        o.status = TT_ERR_LAUNCH_CONFIG;
        o.error = "LaunchConfigError: orthonormal needs h, w >= 1 and angles >= 2";
        return o;
    }
    if (elems(a[0], 4) < std::uint64_t(h) * std::uint64_t(w) || elems(a[4], 4) < std::uint64_t(A) * std::uint64_t(A)) {
        o.trap = first_thread_trap(TT_TRAP_GLOBAL_OUT_OF_BOUNDS);
        return o;
    }
    o = cuda_outcome(tt::launch_orthonormal((const float*)a[0].dptr, h, w, A, (float*)a[4].dptr, ctx.stream),
                     "orthonormal");
    o.gpu_launches = 1;
    return o;
}

Param P(bool ptr, Scalar t, const char* name, bool written = false) {
    Param p;
    p.ptr = ptr;
    p.type = t;
    p.name = name;
    p.written = written;
    return p;
}

// body_fingerprint() of tests/golden/trace_t05.vptx, the reference front end's compilation of
// oracle/trace_t05.krn (checked by tests/test_jit_cpu.py).
constexpr std::uint64_t kTraceT05BodyFingerprint = 0x64a3da5074adf4b3ull;

const std::vector<NativeKernel>& registry() {
    static const std::vector<NativeKernel> reg = [] {
        std::vector<NativeKernel> r;
        auto add = [&](const char* name, std::vector<Param> ps, LaunchFn fn) {
            NativeKernel nk;
            nk.decl.name = name;
            nk.decl.params = std::move(ps);
            nk.fn = fn;
            if (std::string(name) == "trace_t05") nk.body_fingerprints = {kTraceT05BodyFingerprint};
            r.push_back(std::move(nk));
        };
        const Scalar f = Scalar::F32, d = Scalar::F64, i = Scalar::I32, l = Scalar::I64;
        add("trace_t05",
            {P(true, f, "img"), P(false, i, "n"), P(true, f, "ctab"), P(true, f, "stab"), P(true, f, "wtab"),
             P(true, f, "out", true), P(true, i, "med", true), P(false, i, "a0")},
            run_trace_t05);
        add("trace_t05_batch",
            {P(true, f, "img"), P(false, i, "n"), P(true, f, "ctab"), P(true, f, "stab"), P(true, f, "wtab"),
             P(true, f, "out", true), P(true, i, "med", true), P(false, i, "a0"), P(false, i, "batch")},
            run_trace_t05_batch);
        add("radon",
            {P(true, f, "img"), P(false, i, "n"), P(true, f, "ctab"), P(true, f, "stab"), P(true, f, "out", true),
             P(false, i, "a0")},
            run_radon);
        add("circus", {P(true, f, "sino"), P(false, i, "n"), P(false, i, "rows"), P(true, f, "circ", true)},
            run_circus);
        add("circus_fft", {P(true, f, "sino"), P(false, i, "n"), P(false, i, "rows"), P(true, d, "pf", true)},
            run_circus_fft);
        add("hermite",
            {P(true, f, "sino"), P(false, i, "n"), P(false, i, "rows"), P(false, i, "orders"), P(true, d, "hp", true),
             P(true, i, "center", true)},
            run_hermite);
        add("orthonormal",
            {P(true, f, "img"), P(false, i, "h"), P(false, i, "w"), P(false, i, "angles"), P(true, f, "out", true)},
            run_orthonormal);
        add("vadd", {P(true, f, "a"), P(true, f, "b"), P(true, f, "c", true)}, run_vadd<tt::ElemKind::F32, 4>);
        add("vadd", {P(true, d, "a"), P(true, d, "b"), P(true, d, "c", true)}, run_vadd<tt::ElemKind::F64, 8>);
        add("vadd", {P(true, i, "a"), P(true, i, "b"), P(true, i, "c", true)}, run_vadd<tt::ElemKind::I32, 4>);
        add("vadd", {P(true, l, "a"), P(true, l, "b"), P(true, l, "c", true)}, run_vadd<tt::ElemKind::I64, 8>);
        add("scale", {P(true, f, "a", true), P(false, f, "k")}, run_scale);
        add("copy", {P(true, f, "a"), P(true, f, "b", true)}, run_copy);
        add("add_to", {P(true, f, "inp"), P(true, f, "out", true)}, run_add_to);
        return r;
    }();
    return reg;
}


std::string json_escape(const std::string& s) {
    std::string o;
    for (char ch : s) {
        if (ch == '"' || ch == '\\') {
            o += '\\';
            o += ch;
        } else if ((unsigned char)ch < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", ch);
            o += b;
        } else {
            o += ch;
        }
    }
    return o;
}

}  // namespace

// =================================================================== C ABI

extern "C" {

int tt_abi_version(void) { return TT_ABI_VERSION; }

tt_status tt_device_count(int* out) {
    if (!out) return fail(nullptr, TT_ERR_INVALID, "null out");
    cudaError_t e = cudaGetDeviceCount(out);
    if (e != cudaSuccess) {
        *out = 0;
        return cuda_fail(nullptr, e, "cudaGetDeviceCount");
    }
    return TT_OK;
}

const char* tt_last_error(const tt_ctx* ctx) { return ctx ? ctx->last_error.c_str() : t_last_error.c_str(); }

tt_status tt_native_kernels(char* buf, std::size_t cap, std::size_t* needed) {
    std::string s;
    for (const auto& nk : registry()) s += nk.decl.signature() + "\n";
    return copy_out_text(s, buf, cap, needed);
}

tt_status tt_ctx_create(int device, const tt_caps* caps, tt_ctx** out) {
    if (!out) return fail(nullptr, TT_ERR_INVALID, "null out");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(nullptr, TT_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(nullptr, TT_ERR_INVALID, "bad device ordinal");
    DeviceGuard guard(device);
    auto ctx = std::make_unique<tt_ctx>();
    ctx->device = device;
    if (caps) ctx->caps = *caps;
    if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(nullptr, e, "cudaStreamCreate");
    // Keep freed blocks in the pool: steady-state alloc/free never hits the driver.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t thresh = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    // Default sampler 2: TMA-staged tiles for the T0 (Radon) launches they serve, the texture gather for
    // everything else -- the faster of the two for each (measured, profiles/r02_tma_radon.txt);
    // TT_SAMPLER=ldg selects L1 loads, TT_SAMPLER=tex the texture gather for every launch.
    ctx->sampler = 3;  // auto: TMA tiles for the T0 launches where they pay, the texture gather otherwise
    const char* smp = std::getenv("TT_SAMPLER");
    if (smp && (std::strcmp(smp, "ldg") == 0 || std::strcmp(smp, "0") == 0)) ctx->sampler = 0;
    if (smp && (std::strcmp(smp, "tex") == 0 || std::strcmp(smp, "1") == 0)) ctx->sampler = 1;
    ctx->id = ++g_next_ctx_id;
    *out = ctx.release();
    return TT_OK;
}

tt_status tt_ctx_destroy(tt_ctx* ctx) {
    TT_CHECK_CTX(ctx);
    DeviceGuard guard(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    while (!ctx->tex_cache.empty()) drop_texture(ctx, ctx->tex_cache.begin()->first);
    while (!ctx->w_cache.empty()) drop_weights(ctx, ctx->w_cache.begin()->first);
    if (ctx->jit_trap) cudaFree(ctx->jit_trap);
    if (ctx->jit_rng) cudaFree(ctx->jit_rng);
    ctx->jit_trap = nullptr;
    ctx->jit_rng = nullptr;
    for (auto& kv : ctx->allocs)
        if (kv.second.live && kv.second.dptr) cudaFreeAsync(kv.second.dptr, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    ctx->allocs.clear();
    ctx->modules.clear();
    ctx->functions.clear();
    cudaStreamDestroy(ctx->stream);
    ctx->stream = nullptr;
    ctx->destroyed = true;
    return TT_OK;
}

void tt_ctx_release(tt_ctx* ctx) {
    if (!ctx) return;
    if (!ctx->destroyed) tt_ctx_destroy(ctx);
    delete ctx;
}

tt_status tt_ctx_id(const tt_ctx* ctx, std::uint64_t* out) {
    if (!ctx || !out) return fail(ctx, TT_ERR_INVALID, "null argument");
    *out = ctx->id;
    return TT_OK;
}

tt_status tt_ctx_device(const tt_ctx* ctx, int* out) {
    if (!ctx || !out) return fail(ctx, TT_ERR_INVALID, "null argument");
    *out = ctx->device;
    return TT_OK;
}

tt_status tt_ctx_set_sampler(tt_ctx* ctx, int sampler) {
    TT_CHECK_CTX(ctx);
    if (sampler < 0 || sampler > 3)
        return fail(ctx, TT_ERR_INVALID, "sampler must be 0 (global), 1 (texture), 2 (TMA tiles, T0) or 3 (auto)");
    ctx->sampler = sampler;
    return TT_OK;
}

tt_status tt_ctx_synchronize(tt_ctx* ctx) {
    TT_CHECK_CTX(ctx);
    DeviceGuard guard(ctx->device);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? TT_OK : cuda_fail(ctx, e, "cudaStreamSynchronize");
}

tt_status tt_ctx_stream(tt_ctx* ctx, void** out) {
    TT_CHECK_CTX(ctx);
    if (!out) return fail(ctx, TT_ERR_INVALID, "null out");
    *out = (void*)ctx->stream;
    return TT_OK;
}

// ---- modules ------------------------------------------------------------

tt_status tt_module_load(tt_ctx* ctx, const char* text, std::size_t len, tt_module* out) {
    TT_CHECK_CTX(ctx);
    if (!out || (!text && len)) return fail(ctx, TT_ERR_INVALID, "null argument");
    Module m;
    tt_status st = parse_module(ctx, text ? text : "", len, m);  // counter untouched on failure
    if (st != TT_OK) return st;
    const std::uint64_t h = ctx->next_handle++;
    ctx->modules.emplace(h, std::move(m));
    ++ctx->c.modules_loaded;
    ctx->events.push_back(TT_EV_MODULE_LOAD);
    *out = tt_module{ctx->id, h};
    return TT_OK;
}

tt_status tt_module_unload(tt_ctx* ctx, tt_module m) {
    TT_CHECK_CTX(ctx);
    auto it = ctx->modules.find(m.id);
    if (m.ctx_id != ctx->id || it == ctx->modules.end())
        return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: stale or foreign module handle");
    ctx->modules.erase(it);
    for (auto f = ctx->functions.begin(); f != ctx->functions.end();) {  // driver.hpp:159-163
        if (f->second.module_id == m.id) f = ctx->functions.erase(f);
        else ++f;
    }
    return TT_OK;
}

tt_status tt_get_function(tt_ctx* ctx, tt_module m, const char* name, tt_function* out) {
    TT_CHECK_CTX(ctx);
    if (!name || !out) return fail(ctx, TT_ERR_INVALID, "null argument");
    auto it = ctx->modules.find(m.id);
    if (m.ctx_id != ctx->id || it == ctx->modules.end())
        return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: stale or foreign module handle");
    const KernelDecl* decl = nullptr;
    for (const auto& k : it->second.kernels)
        if (k.name == name) decl = &k;
    if (!decl) return fail(ctx, TT_ERR_FUNCTION_NOT_FOUND, std::string("FunctionNotFound: '") + name + "'");
    // header-only module (no body, or a bare `ret` as the C ABI's own renderers emit)
    const bool header_only =
        decl->body.empty() || (decl->body.size() == 1 && decl->body[0].toks.size() == 1 && decl->body[0].toks[0] == "ret");
    const NativeKernel* nk = find_native(*decl);
    if (nk && !header_only) {  // a real body binds natively only if it is the documented DSL body
        const std::uint64_t fp = body_fingerprint(decl->body);
        if (std::find(nk->body_fingerprints.begin(), nk->body_fingerprints.end(), fp) == nk->body_fingerprints.end())
            nk = nullptr;  // run the module's own body
    }
    std::shared_ptr<JitFunction> jf;
    if (!nk) {
        if (header_only)
            return fail(ctx, TT_ERR_FUNCTION_NOT_FOUND,
                        std::string("FunctionNotFound: '") + name + "' (no native sm_100a kernel for " +
                            decl->signature() + " and no VPTX body to compile; see tt_native_kernels)");
        // No native implementation: compile the VPTX body for sm_100a (tt_jit.h).
        DeviceGuard guard(ctx->device);
        jf = std::make_shared<JitFunction>();
        jf->decl = *decl;
        std::vector<tt::jit::Param> jp;
        for (const Param& p : decl->params)
            jp.push_back(tt::jit::Param{p.ptr, tt::jit::Ty(static_cast<int>(p.type)), p.name});
        std::string err;
        if (!tt::jit::compile(decl->name, jp, decl->body, jf->prog, err))
            return fail(ctx, err.rfind("VPTX JIT, line", 0) == 0 ? TT_ERR_VALIDATION_FAILED : TT_ERR_CUDA,
                        (err.rfind("VPTX JIT, line", 0) == 0 ? "ValidationFailed:\n  " : "") + err);
    }
    const std::uint64_t h = ctx->next_handle++;
    ctx->functions.emplace(h, FunctionEntry{m.id, name, nk, jf});
    ++ctx->c.functions_resolved;
    ctx->events.push_back(TT_EV_FUNCTION_RESOLVE);
    *out = tt_function{ctx->id, h};
    return TT_OK;
}

// ---- memory -------------------------------------------------------------

tt_status tt_mem_alloc(tt_ctx* ctx, std::uint64_t bytes, tt_devptr* out) {
    TT_CHECK_CTX(ctx);
    if (!out) return fail(ctx, TT_ERR_INVALID, "null out");
    DeviceGuard guard(ctx->device);
    void* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, bytes ? bytes : 1, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMallocAsync");
    if (bytes && (e = cudaMemsetAsync(d, 0, bytes, ctx->stream)) != cudaSuccess)  // zero-filled arena
        return cuda_fail(ctx, e, "cudaMemsetAsync");
    const std::uint64_t base = ctx->bump;
    ctx->bump += bytes == 0 ? 256 : (bytes + 255) / 256 * 256;  // emulator.hpp:112-117
    ctx->allocs.emplace(base, Alloc{d, bytes, true});
    ++ctx->c.allocs;
    ctx->events.push_back(TT_EV_ALLOC);
    *out = tt_devptr{base, bytes, ctx->id};
    return TT_OK;
}

tt_status tt_mem_free(tt_ctx* ctx, tt_devptr p) {
    TT_CHECK_CTX(ctx);
    if (p.ctx_id != ctx->id) return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: device pointer belongs to another context");
    if (p.base == 0) return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: null device pointer");
    auto it = ctx->allocs.find(p.base);
    if (it == ctx->allocs.end() || !it->second.live)
        return fail(ctx, TT_ERR_DOUBLE_FREE, "DoubleFree: device pointer already freed");
    DeviceGuard guard(ctx->device);
    drop_texture(ctx, p.base);
    drop_weights(ctx, p.base);
    cudaError_t e = cudaFreeAsync(it->second.dptr, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaFreeAsync");
    it->second.live = false;  // the address stays reserved: never reused
    it->second.dptr = nullptr;
    ++ctx->c.frees;
    ctx->events.push_back(TT_EV_FREE);
    return TT_OK;
}

tt_status tt_memcpy_htod(tt_ctx* ctx, tt_devptr dst, const void* src, std::uint64_t bytes) {
    TT_CHECK_CTX(ctx);
    Alloc* a = nullptr;
    tt_status st = lookup(ctx, dst, &a);
    if (st != TT_OK) return st;
    if (bytes > a->bytes)
        return fail(ctx, TT_ERR_OUT_OF_BOUNDS, "OutOfBounds: copy of " + std::to_string(bytes) +
                                                   " bytes into an allocation of " + std::to_string(a->bytes));
    if (bytes && !src) return fail(ctx, TT_ERR_INVALID, "null source");
    if (bytes) {
        DeviceGuard guard(ctx->device);
        cudaError_t e = cudaMemcpyAsync(a->dptr, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // synchronous like driver.hpp:195
        if (e != cudaSuccess) return cuda_fail(ctx, e, "memcpy_htod");
    }
    ++a->gen;
    ctx->c.bytes_h2d += bytes;
    ctx->events.push_back(TT_EV_H2D);
    return TT_OK;
}

tt_status tt_memcpy_dtoh(tt_ctx* ctx, void* dst, tt_devptr src, std::uint64_t bytes) {
    TT_CHECK_CTX(ctx);
    Alloc* a = nullptr;
    tt_status st = lookup(ctx, src, &a);
    if (st != TT_OK) return st;
    if (bytes > a->bytes)
        return fail(ctx, TT_ERR_OUT_OF_BOUNDS, "OutOfBounds: copy of " + std::to_string(bytes) +
                                                   " bytes out of an allocation of " + std::to_string(a->bytes));
    if (bytes && !dst) return fail(ctx, TT_ERR_INVALID, "null destination");
    if (bytes) {
        DeviceGuard guard(ctx->device);
        cudaError_t e = cudaMemcpyAsync(dst, a->dptr, bytes, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "memcpy_dtoh");
    }
    ctx->c.bytes_d2h += bytes;
    ctx->events.push_back(TT_EV_D2H);
    return TT_OK;
}

tt_status tt_mem_device_pointer(tt_ctx* ctx, tt_devptr p, void** out) {
    TT_CHECK_CTX(ctx);
    if (!out) return fail(ctx, TT_ERR_INVALID, "null out");
    Alloc* a = nullptr;
    tt_status st = lookup(ctx, p, &a);
    if (st != TT_OK) return st;
    ++a->gen;  // the caller may write through the raw pointer, now or later: cached copies are stale,
    a->exported = true;  // and stay suspect for the allocation's lifetime (refreshed per launch)
    *out = a->dptr;
    return TT_OK;
}

tt_status tt_host_alloc(std::uint64_t bytes, void** out) {
    if (!out) return fail(nullptr, TT_ERR_INVALID, "null out");
    cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "cudaHostAlloc");
}

tt_status tt_host_free(void* p) {
    cudaError_t e = cudaFreeHost(p);
    return e == cudaSuccess ? TT_OK : cuda_fail(nullptr, e, "cudaFreeHost");
}

// ---- launch ---------------------------------------------------------------

}  // extern "C"

namespace {

// Launch of a JIT-compiled VPTX kernel: the context's allocation table goes to
// the device for the bounds checks, the trap record is reset, and after the
// launch the first trap (emulator order, tt_jit.h) is read back.
LaunchOutcome run_jit(tt_ctx& ctx, JitFunction& jf, const tt_grid& g, const std::vector<ResolvedArg>& a,
                      std::uint64_t shared_total) {
    LaunchOutcome o;
    auto cuda_err = [&](cudaError_t e, const char* what) {
        o.status = TT_ERR_CUDA;
        o.error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
        return o;
    };
    // allocation table: live ranges, then freed ranges that overlap nothing already listed
    std::vector<std::array<unsigned long long, 3>> rng;
    for (int pass = 0; pass < 2; ++pass)
        for (const auto& kv : ctx.allocs) {
            const Alloc& al = kv.second;
            if (al.live != (pass == 0) || !al.dptr) continue;
            const unsigned long long b = (unsigned long long)al.dptr, e = b + al.bytes;
            bool overlap = false;
            if (pass == 1)
                for (const auto& r : rng) overlap = overlap || (b < r[1] && r[0] < e) || b == r[0];
            if (!overlap) rng.push_back({b, e, al.live ? 1ull : 0ull});
        }
    std::sort(rng.begin(), rng.end());
    cudaError_t e = cudaSuccess;
    if (!ctx.jit_trap && (e = cudaMalloc((void**)&ctx.jit_trap, sizeof(tt::jit::TrapRecord))) != cudaSuccess)
        return cuda_err(e, "JIT trap record");
    if (rng.size() > ctx.jit_rng_cap) {
        if (ctx.jit_rng) cudaFree(ctx.jit_rng);
        ctx.jit_rng_cap = std::max<std::size_t>(64, rng.size() * 2);
        if ((e = cudaMalloc((void**)&ctx.jit_rng, ctx.jit_rng_cap * 24)) != cudaSuccess) {
            ctx.jit_rng = nullptr;
            ctx.jit_rng_cap = 0;
            return cuda_err(e, "JIT allocation table");
        }
    }
    tt::jit::TrapRecord rec0{};
    rec0.key = ~0ull;
    if (!rng.empty() && (e = cudaMemcpyAsync(ctx.jit_rng, rng.data(), rng.size() * 24, cudaMemcpyHostToDevice,
                                            ctx.stream)) != cudaSuccess)
        return cuda_err(e, "JIT allocation table upload");
    if ((e = cudaMemcpyAsync(ctx.jit_trap, &rec0, sizeof rec0, cudaMemcpyHostToDevice, ctx.stream)) != cudaSuccess)
        return cuda_err(e, "JIT trap reset");
    // kernel arguments: the VPTX parameters (pointers as device addresses), then the hidden ones
    std::vector<std::array<unsigned char, 8>> store(a.size() + 4);
    std::vector<void*> argv;
    for (std::size_t i = 0; i < a.size(); ++i) {
        auto& cell = store[i];
        if (a[i].kind == TT_ARG_PTR) {
            const long long v = (long long)a[i].dptr;
            std::memcpy(cell.data(), &v, 8);
        } else if (a[i].kind == TT_ARG_I32) {
            std::memcpy(cell.data(), &a[i].value.v.i32, 4);
        } else if (a[i].kind == TT_ARG_I64) {
            std::memcpy(cell.data(), &a[i].value.v.i64, 8);
        } else if (a[i].kind == TT_ARG_F32) {
            std::memcpy(cell.data(), &a[i].value.v.f32, 4);
        } else {
            std::memcpy(cell.data(), &a[i].value.v.f64, 8);
        }
        argv.push_back(cell.data());
    }
    void* trap_ptr = ctx.jit_trap;
    const unsigned long long* rng_ptr = ctx.jit_rng;
    int nr = int(rng.size());
    unsigned shb = unsigned(shared_total);
    argv.push_back(&trap_ptr);
    argv.push_back(&rng_ptr);
    argv.push_back(&nr);
    argv.push_back(&shb);
    e = cudaLaunchKernel((const void*)jf.prog.kernel, dim3(g.grid[0], g.grid[1], g.grid[2]),
                         dim3(g.block[0], g.block[1], g.block[2]), argv.data(), shared_total, ctx.stream);
    if (e != cudaSuccess) return cuda_err(e, "JIT kernel launch");
    o.gpu_launches = 1;
    tt::jit::TrapRecord rec{};
    if ((e = cudaMemcpyAsync(&rec, ctx.jit_trap, sizeof rec, cudaMemcpyDeviceToHost, ctx.stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(ctx.stream)) != cudaSuccess)
        return cuda_err(e, "JIT kernel");
    if (rec.key != ~0ull) {
        o.trap.trapped = 1;
        o.trap.kind = rec.kind;
        for (int i = 0; i < 3; ++i) {
            o.trap.thread[i] = rec.tid[i] + 1;  // 1-indexed, source-language convention
            o.trap.block[i] = rec.ctaid[i] + 1;
        }
        o.trap.instr_index = std::uint64_t(rec.instr);
        o.trap.code = rec.kind == TT_TRAP_EXPLICIT ? rec.code : 0;
    }
    return o;
}

}  // namespace

extern "C" {

tt_status tt_launch(tt_ctx* ctx, tt_function fn, const tt_grid* cfg, const tt_arg* args, int nargs, tt_trap* trap_out) {
    struct Range {  // NVTX (nvtx3, header-only: a no-op unless a profiler injects itself)
        Range() { nvtxRangePushA("tt_launch"); }
        ~Range() { nvtxRangePop(); }
    } nvtx_range;
    TT_CHECK_CTX(ctx);
    if (!cfg || (nargs > 0 && !args) || nargs < 0) return fail(ctx, TT_ERR_INVALID, "null argument");
    if (trap_out) std::memset(trap_out, 0, sizeof *trap_out);
    auto fit = ctx->functions.find(fn.id);
    if (fn.ctx_id != ctx->id || fit == ctx->functions.end())
        return fail(ctx, TT_ERR_FUNCTION_NOT_FOUND, "FunctionNotFound: 'stale or foreign function handle'");
    if (ctx->modules.find(fit->second.module_id) == ctx->modules.end())
        return fail(ctx, TT_ERR_FUNCTION_NOT_FOUND, "FunctionNotFound: 'function's module was unloaded'");
    const NativeKernel* native = fit->second.native;
    const std::shared_ptr<JitFunction> jit = fit->second.jit;
    const KernelDecl& decl = native ? native->decl : jit->decl;

    // driver.hpp:229-231: convert every argument (ownership, liveness) first.
    std::vector<ResolvedArg> ra(static_cast<std::size_t>(nargs));
    for (int i = 0; i < nargs; ++i) {
        ra[i].kind = tt_arg_kind(args[i].kind);
        ra[i].value = args[i];
        if (args[i].kind == TT_ARG_PTR) {
            Alloc* a = nullptr;
            tt_status st = lookup(ctx, args[i].v.ptr, &a);
            if (st != TT_OK) return st;
            ra[i].dptr = a->dptr;
            ra[i].bytes = a->bytes;
            ra[i].base = args[i].v.ptr.base;
            ra[i].gen = a->gen;
            ra[i].exported = a->exported;
        } else if (args[i].kind < TT_ARG_I32 || args[i].kind > TT_ARG_PTR) {
            return fail(ctx, TT_ERR_INVALID, "bad tt_arg kind");
        }
    }
    // KernelImage checks, emulator.hpp:223-271 (same order).
    for (int i = 0; i < 3; ++i)
        if (cfg->grid[i] == 0 || cfg->block[i] == 0)
            return fail(ctx, TT_ERR_LAUNCH_CONFIG, "LaunchConfigError: grid/block dimensions must be >= 1");
    const std::uint64_t tpb = std::uint64_t(cfg->block[0]) * cfg->block[1] * cfg->block[2];
    if (tpb > ctx->caps.max_block_threads)
        return fail(ctx, TT_ERR_LAUNCH_CONFIG, "LaunchConfigError: block of " + std::to_string(tpb) +
                                                   " threads exceeds the cap of " +
                                                   std::to_string(ctx->caps.max_block_threads));
    if (std::size_t(nargs) != decl.params.size())
        return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: kernel '" + decl.name + "' takes " +
                                                       std::to_string(decl.params.size()) +
                                                       " argument(s), got " + std::to_string(nargs));
    for (int i = 0; i < nargs; ++i) {
        const Param& p = decl.params[i];
        bool ok;
        if (p.ptr) ok = args[i].kind == TT_ARG_PTR;
        else
            ok = (p.type == Scalar::I32 && args[i].kind == TT_ARG_I32) ||
                 (p.type == Scalar::I64 && args[i].kind == TT_ARG_I64) ||
                 (p.type == Scalar::F32 && args[i].kind == TT_ARG_F32) ||
                 (p.type == Scalar::F64 && args[i].kind == TT_ARG_F64);
        if (!ok)
            return fail(ctx, TT_ERR_ARGUMENT_MISMATCH, "ArgumentMismatch: argument " + std::to_string(i + 1) +
                                                           " does not match parameter '" + p.name +
                                                           "' of type " + p.type_text());
    }
    const std::uint64_t shared_total = cfg->shared_bytes_extra + (jit ? jit->prog.static_shared : 0);
    if (shared_total > ctx->caps.max_shared_bytes)
        return fail(ctx, TT_ERR_LAUNCH_CONFIG, "LaunchConfigError: shared memory of " +
                                                   std::to_string(shared_total) +
                                                   " bytes exceeds the cap of " +
                                                   std::to_string(ctx->caps.max_shared_bytes));

    DeviceGuard guard(ctx->device);
    LaunchOutcome o = native ? native->fn(*ctx, *cfg, ra) : run_jit(*ctx, *jit, *cfg, ra, shared_total);
    if (o.status != TT_OK) return fail(ctx, o.status, o.error);

    // Allocations a launch may have written get a new generation (cached texture / weight copies go
    // stale): the native kernels' output parameters; every pointer argument of a JIT kernel.
    for (int i = 0; i < nargs; ++i)
        if (args[i].kind == TT_ARG_PTR && (native ? (!o.trap.trapped && decl.params[i].written) : true))
            ++ctx->allocs[args[i].v.ptr.base].gen;

    // Counting and the launch log, driver.hpp:235-246 (traps count too).
    ++ctx->c.launches;
    ctx->c.gpu_kernel_launches += std::uint64_t(o.gpu_launches);
    ctx->events.push_back(TT_EV_LAUNCH);
    finish_launch_log(ctx);
    LaunchRecord rec;
    rec.kernel = decl.name;
    for (int i = 0; i < 3; ++i) {
        rec.grid[i] = cfg->grid[i];
        rec.block[i] = cfg->block[i];
    }
    rec.h2d = ctx->c.bytes_h2d - ctx->h2d_mark;
    ctx->h2d_mark = ctx->c.bytes_h2d;
    ctx->d2h_mark = ctx->c.bytes_d2h;
    ctx->launch_log.push_back(rec);
    if (trap_out) *trap_out = o.trap;
    return TT_OK;
}

// ---- introspection ---------------------------------------------------------

tt_status tt_counters_get(tt_ctx* ctx, tt_counters* out) {
    TT_CHECK_CTX(ctx);
    if (!out) return fail(ctx, TT_ERR_INVALID, "null out");
    finish_launch_log(ctx);
    *out = ctx->c;
    out->launch_log_size = ctx->launch_log.size();
    out->events_size = ctx->events.size();
    return TT_OK;
}

tt_status tt_counters_json(tt_ctx* ctx, char* buf, std::size_t cap, std::size_t* needed) {
    TT_CHECK_CTX(ctx);
    finish_launch_log(ctx);
    const tt_counters& c = ctx->c;
    std::string s = "{\"modules_loaded\": " + std::to_string(c.modules_loaded) +
                    ", \"functions_resolved\": " + std::to_string(c.functions_resolved) +
                    ", \"launches\": " + std::to_string(c.launches) + ", \"allocs\": " + std::to_string(c.allocs) +
                    ", \"frees\": " + std::to_string(c.frees) + ", \"bytes_h2d\": " + std::to_string(c.bytes_h2d) +
                    ", \"bytes_d2h\": " + std::to_string(c.bytes_d2h) +
                    ", \"gpu_kernel_launches\": " + std::to_string(c.gpu_kernel_launches) + ", \"launch_log\": [";
    for (std::size_t i = 0; i < ctx->launch_log.size(); ++i) {
        const LaunchRecord& r = ctx->launch_log[i];
        if (i) s += ", ";
        s += "{\"kernel\": \"" + json_escape(r.kernel) + "\", \"grid\": [" + std::to_string(r.grid[0]) + ", " +
             std::to_string(r.grid[1]) + ", " + std::to_string(r.grid[2]) + "], \"block\": [" +
             std::to_string(r.block[0]) + ", " + std::to_string(r.block[1]) + ", " + std::to_string(r.block[2]) +
             "], \"h2d_bytes\": " + std::to_string(r.h2d) + ", \"d2h_bytes\": " + std::to_string(r.d2h) + "}";
    }
    s += "]}";
    tt_status st = copy_out_text(s, buf, cap, needed);
    if (st != TT_OK) ctx->last_error = t_last_error;
    return st;
}

tt_status tt_events(tt_ctx* ctx, std::uint8_t* buf, std::size_t cap, std::size_t* needed) {
    TT_CHECK_CTX(ctx);
    if (needed) *needed = ctx->events.size();
    if (!buf || cap == 0) return TT_OK;
    if (cap < ctx->events.size()) return fail(ctx, TT_ERR_INVALID, "buffer too small");
    std::memcpy(buf, ctx->events.data(), ctx->events.size());
    return TT_OK;
}

}  // extern "C"

std::uint64_t ttc::body_fingerprint(const std::vector<tt::jit::Line>& body) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&](unsigned char c) {
        h ^= c;
        h *= 1099511628211ull;
    };
    for (const auto& l : body) {
        for (const auto& t : l.toks) {
            for (unsigned char c : t) mix(c);
            mix(0x1f);
        }
        mix('\n');
    }
    return h;
}

extern "C" tt_status tt_vptx_body_fingerprint(const char* vptx, std::size_t len, const char* kernel,
                                              std::uint64_t* out) {
    if (!vptx || !kernel || !out) return fail(nullptr, TT_ERR_INVALID, "null argument");
    Module m;
    tt_status st = parse_module(nullptr, vptx, len, m);
    if (st != TT_OK) return st;
    for (const auto& k : m.kernels)
        if (k.name == kernel) {
            *out = body_fingerprint(k.body);
            return TT_OK;
        }
    return fail(nullptr, TT_ERR_FUNCTION_NOT_FOUND, std::string("FunctionNotFound: '") + kernel + "'");
}

extern "C" tt_status tt_jit_source(const char* vptx, std::size_t len, const char* kernel, char* buf, std::size_t cap,
                                   std::size_t* needed) {
    if (!vptx || !kernel) return fail(nullptr, TT_ERR_INVALID, "null argument");
    Module m;
    tt_status st = parse_module(nullptr, vptx, len, m);
    if (st != TT_OK) return st;
    for (const auto& k : m.kernels) {
        if (k.name != kernel) continue;
        std::vector<tt::jit::Param> jp;
        for (const Param& p : k.params) jp.push_back(tt::jit::Param{p.ptr, tt::jit::Ty(static_cast<int>(p.type)), p.name});
        std::string src, err;
        std::uint64_t sh = 0;
        if (!tt::jit::translate(k.name, jp, k.body, src, sh, err))
            return fail(nullptr, TT_ERR_VALIDATION_FAILED, "ValidationFailed:\n  " + err);
        return copy_out_text(src, buf, cap, needed);
    }
    return fail(nullptr, TT_ERR_FUNCTION_NOT_FOUND, std::string("FunctionNotFound: '") + kernel + "'");
}
