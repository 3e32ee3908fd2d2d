// gridjit_b200.hpp — the reference's C++ host API, source-compatible, over
// the B200 C ABI (include/tt_b200.h, libtt_b200.so).
//
// A program written against /root/reference/proj/include/gridjit/
// driver.hpp + autolaunch.hpp (DeviceContext, create_context, DevicePtr,
// LaunchArg, GridConfig, LaunchResult/TrapInfo, Counters, cuda_launch,
// cu_in/cu_out/cu_inout, LaunchReport, cache_stats and the errors.hpp
// exception taxonomy) compiles against this header unchanged, except that
// kernels are named by their header (KernelAst{name, params} or
// parse_kernel(src), which reads only `kernel name(params)`) and bound to the
// native sm_100a kernel registered for the launch signature, instead of being
// JIT-compiled from the DSL body.  See INTEGRATION.md.
//
// Header-only; link with -ltt_b200.
#pragma once

#include <array>
#include <cctype>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "tt_b200.h"

namespace gridjit {

// ---- errors.hpp -----------------------------------------------------------
class Error : public std::runtime_error {
  public:
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
#define TT_GRIDJIT_ERROR(Name) \
    class Name : public Error { \
      public: \
        explicit Name(const std::string& m) : Error(m) {} \
    };
TT_GRIDJIT_ERROR(ContextDestroyed)
TT_GRIDJIT_ERROR(VptxSyntaxError)
TT_GRIDJIT_ERROR(ValidationFailed)
TT_GRIDJIT_ERROR(FunctionNotFound)
TT_GRIDJIT_ERROR(OutOfBounds)
TT_GRIDJIT_ERROR(DoubleFree)
TT_GRIDJIT_ERROR(UseAfterFree)
TT_GRIDJIT_ERROR(ArgumentMismatch)
TT_GRIDJIT_ERROR(LaunchConfigError)
TT_GRIDJIT_ERROR(ArityError)
TT_GRIDJIT_ERROR(CudaError)
#undef TT_GRIDJIT_ERROR

namespace detail {
[[noreturn]] inline void raise(tt_status st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case TT_ERR_CONTEXT_DESTROYED: throw ContextDestroyed(m);
        case TT_ERR_VPTX_SYNTAX: throw VptxSyntaxError(m);
        case TT_ERR_VALIDATION_FAILED: throw ValidationFailed(m);
        case TT_ERR_FUNCTION_NOT_FOUND: throw FunctionNotFound(m);
        case TT_ERR_OUT_OF_BOUNDS: throw OutOfBounds(m);
        case TT_ERR_DOUBLE_FREE: throw DoubleFree(m);
        case TT_ERR_USE_AFTER_FREE: throw UseAfterFree(m);
        case TT_ERR_ARGUMENT_MISMATCH: throw ArgumentMismatch(m);
        case TT_ERR_LAUNCH_CONFIG: throw LaunchConfigError(m);
        case TT_ERR_ARITY: throw ArityError(m);
        case TT_ERR_CUDA: throw CudaError(m);
        default: throw Error(m);
    }
}
inline void check(tt_status st, const tt_ctx* ctx) {
    if (st != TT_OK) raise(st, tt_last_error(ctx));
}
}  // namespace detail

// ---- types.hpp / emulator.hpp / driver.hpp value types ------------------------
enum class ScalarType : std::uint8_t { I32, I64, F32, F64, Pred };

inline std::string_view scalar_name(ScalarType t) {
    switch (t) {
        case ScalarType::I32: return "i32";
        case ScalarType::I64: return "i64";
        case ScalarType::F32: return "f32";
        case ScalarType::F64: return "f64";
        default: return "pred";
    }
}

struct GridConfig {
    std::array<std::uint32_t, 3> grid{1, 1, 1};
    std::array<std::uint32_t, 3> block{1, 1, 1};
    std::uint64_t shared_bytes_extra = 0;
};

struct DeviceCaps {
    std::uint32_t max_block_threads = 1024;
    std::uint64_t max_shared_bytes = 48 * 1024;
};

struct TrapInfo {
    enum class Kind : std::uint8_t {
        GlobalOutOfBounds, SharedOutOfBounds, UseOfFreedMemory, DivisionByZero, BarrierDivergence, ExplicitTrap
    };
    Kind kind = Kind::ExplicitTrap;
    std::array<std::uint32_t, 3> thread{1, 1, 1};
    std::array<std::uint32_t, 3> block{1, 1, 1};
    std::size_t instr_index = 0;
    std::int64_t code = 0;
    static std::string_view kind_name(Kind k) {
        static const char* names[] = {"GlobalOutOfBounds", "SharedOutOfBounds", "UseOfFreedMemory",
                                      "DivisionByZero", "BarrierDivergence", "ExplicitTrap"};
        return names[int(k)];
    }
};

struct LaunchResult {
    std::optional<TrapInfo> trap;
    bool ok() const { return !trap.has_value(); }
};

struct ModuleHandle {
    std::uint64_t ctx_id = 0, id = 0;
    friend bool operator==(const ModuleHandle&, const ModuleHandle&) = default;
};
struct FunctionHandle {
    std::uint64_t ctx_id = 0, id = 0;
    friend bool operator==(const FunctionHandle&, const FunctionHandle&) = default;
};
struct DevicePtr {
    std::uint64_t base = 0;
    std::uint64_t length = 0;
    std::uint64_t ctx_id = 0;
};

using LaunchArg = std::variant<std::int32_t, std::int64_t, float, double, DevicePtr>;

struct Counters {
    std::uint64_t modules_loaded = 0, functions_resolved = 0, launches = 0, allocs = 0, frees = 0, bytes_h2d = 0,
                  bytes_d2h = 0;
    std::uint64_t gpu_kernel_launches = 0;  // extension: native CUDA kernels enqueued
};

struct MethodCache {
    struct Entry {
        ModuleHandle module;
        FunctionHandle function;
    };
    std::map<std::string, Entry> entries;
    std::uint64_t hits = 0, misses = 0, compiles = 0;
};

// ---- DeviceContext (driver.hpp:112-330) ------------------------------------------
class DeviceContext {
  public:
    explicit DeviceContext(DeviceCaps caps = {}, int device = 0) {
        tt_caps c{caps.max_block_threads, caps.max_shared_bytes};
        detail::check(tt_ctx_create(device, &c, &ctx_), nullptr);
        detail::check(tt_ctx_id(ctx_, &id_), ctx_);
    }
    DeviceContext(const DeviceContext&) = delete;
    DeviceContext& operator=(const DeviceContext&) = delete;
    DeviceContext(DeviceContext&& o) noexcept { *this = std::move(o); }
    DeviceContext& operator=(DeviceContext&& o) noexcept {
        std::swap(ctx_, o.ctx_);
        std::swap(id_, o.id_);
        std::swap(cache_, o.cache_);
        return *this;
    }
    ~DeviceContext() { tt_ctx_release(ctx_); }

    std::uint64_t id() const { return id_; }
    void destroy() { detail::check(tt_ctx_destroy(ctx_), ctx_); }

    ModuleHandle module_load(std::string_view text) {
        tt_module m{};
        detail::check(tt_module_load(ctx_, text.data(), text.size(), &m), ctx_);
        return {m.ctx_id, m.id};
    }
    void module_unload(ModuleHandle h) { detail::check(tt_module_unload(ctx_, {h.ctx_id, h.id}), ctx_); }
    FunctionHandle get_function(ModuleHandle h, std::string_view name) {
        tt_function f{};
        const std::string s(name);
        detail::check(tt_get_function(ctx_, {h.ctx_id, h.id}, s.c_str(), &f), ctx_);
        return {f.ctx_id, f.id};
    }
    DevicePtr mem_alloc(std::uint64_t bytes) {
        tt_devptr p{};
        detail::check(tt_mem_alloc(ctx_, bytes, &p), ctx_);
        return {p.base, p.length, p.ctx_id};
    }
    void mem_free(DevicePtr p) { detail::check(tt_mem_free(ctx_, {p.base, p.length, p.ctx_id}), ctx_); }
    void memcpy_htod(DevicePtr dst, const void* src, std::uint64_t bytes) {
        detail::check(tt_memcpy_htod(ctx_, {dst.base, dst.length, dst.ctx_id}, src, bytes), ctx_);
    }
    void memcpy_dtoh(void* dst, DevicePtr src, std::uint64_t bytes) {
        detail::check(tt_memcpy_dtoh(ctx_, dst, {src.base, src.length, src.ctx_id}, bytes), ctx_);
    }
    LaunchResult launch(FunctionHandle fn, const GridConfig& cfg, const std::vector<LaunchArg>& args) {
        std::vector<tt_arg> a(args.size());
        for (std::size_t i = 0; i < args.size(); ++i) {
            std::memset(&a[i], 0, sizeof(tt_arg));
            std::visit(
                [&](auto v) {
                    using T = std::decay_t<decltype(v)>;
                    if constexpr (std::is_same_v<T, std::int32_t>) { a[i].kind = TT_ARG_I32; a[i].v.i32 = v; }
                    else if constexpr (std::is_same_v<T, std::int64_t>) { a[i].kind = TT_ARG_I64; a[i].v.i64 = v; }
                    else if constexpr (std::is_same_v<T, float>) { a[i].kind = TT_ARG_F32; a[i].v.f32 = v; }
                    else if constexpr (std::is_same_v<T, double>) { a[i].kind = TT_ARG_F64; a[i].v.f64 = v; }
                    else { a[i].kind = TT_ARG_PTR; a[i].v.ptr = {v.base, v.length, v.ctx_id}; }
                },
                args[i]);
        }
        tt_grid g{};
        for (int i = 0; i < 3; ++i) {
            g.grid[i] = cfg.grid[i];
            g.block[i] = cfg.block[i];
        }
        g.shared_bytes_extra = cfg.shared_bytes_extra;
        tt_trap t{};
        detail::check(tt_launch(ctx_, {fn.ctx_id, fn.id}, &g, a.data(), int(a.size()), &t), ctx_);
        LaunchResult r;
        if (t.trapped) {
            TrapInfo ti;
            ti.kind = TrapInfo::Kind(t.kind);
            for (int i = 0; i < 3; ++i) {
                ti.thread[i] = t.thread[i];
                ti.block[i] = t.block[i];
            }
            ti.instr_index = t.instr_index;
            ti.code = t.code;
            r.trap = ti;
        }
        return r;
    }
    Counters counters() {
        tt_counters c{};
        detail::check(tt_counters_get(ctx_, &c), ctx_);
        return {c.modules_loaded, c.functions_resolved, c.launches, c.allocs, c.frees, c.bytes_h2d, c.bytes_d2h,
                c.gpu_kernel_launches};
    }
    std::string counters_json() {  // Counters::to_json text (driver.hpp:78-95)
        std::size_t need = 0;
        detail::check(tt_counters_json(ctx_, nullptr, 0, &need), ctx_);
        std::string s(need, '\0');
        detail::check(tt_counters_json(ctx_, s.data(), s.size(), &need), ctx_);
        s.resize(need ? need - 1 : 0);
        return s;
    }
    MethodCache& method_cache() {
        tt_counters c{};
        detail::check(tt_counters_get(ctx_, &c), ctx_);  // ContextDestroyed like driver.hpp:263-266
        return cache_;
    }
    tt_ctx* raw() { return ctx_; }

  private:
    tt_ctx* ctx_ = nullptr;
    std::uint64_t id_ = 0;
    MethodCache cache_;
};

inline DeviceContext create_context(DeviceCaps caps = {}) { return DeviceContext(caps); }

// ---- autolaunch.hpp ----------------------------------------------------------------
struct KernelAst {  // launch identity only (the DSL body is bound to a native kernel)
    std::string name;
    std::vector<std::string> params;
};

// Reads the header `kernel name(a, b, ...)` of a gridjit DSL kernel.
inline KernelAst parse_kernel(std::string_view src) {
    KernelAst k;
    std::size_t p = src.find("kernel");
    if (p == std::string_view::npos) throw Error("SyntaxError: no kernel definition found");
    p += 6;
    auto skip = [&] { while (p < src.size() && std::isspace((unsigned char)src[p])) ++p; };
    skip();
    std::size_t s = p;
    while (p < src.size() && (std::isalnum((unsigned char)src[p]) || src[p] == '_')) ++p;
    k.name = std::string(src.substr(s, p - s));
    skip();
    if (p >= src.size() || src[p] != '(') throw Error("SyntaxError: expected '(' after kernel name");
    ++p;
    std::string cur;
    for (; p < src.size() && src[p] != ')'; ++p) {
        if (src[p] == ',') {
            k.params.push_back(cur);
            cur.clear();
        } else if (!std::isspace((unsigned char)src[p])) {
            cur += src[p];
        }
    }
    if (!cur.empty()) k.params.push_back(cur);
    return k;
}

enum class Direction : std::uint8_t { In, Out, InOut };

class KernelArg {
  public:
    template <typename T>
    KernelArg(std::vector<T>& host) : KernelArg(Direction::InOut, host) {}
    template <typename T>
        requires std::is_same_v<T, std::int32_t> || std::is_same_v<T, std::int64_t> ||
                 std::is_same_v<T, float> || std::is_same_v<T, double>
    KernelArg(T scalar) : array_(false), type_(type_of<T>()), scalar_(scalar) {}
    template <typename T>
    KernelArg(Direction d, std::vector<T>& host)
        : array_(true), dir_(d), type_(type_of<T>()), data_(host.data()), bytes_(host.size() * sizeof(T)) {}

    bool is_array() const { return array_; }
    Direction direction() const { return dir_; }
    ScalarType elem_type() const { return type_; }
    void* data() const { return data_; }
    std::uint64_t bytes() const { return bytes_; }
    const LaunchArg& scalar() const { return scalar_; }
    std::string sig() const { return std::string(scalar_name(type_)) + (array_ ? "[]" : ""); }
    std::string vptx_type() const { return (array_ ? "ptr.global." : "") + std::string(scalar_name(type_)); }

  private:
    template <typename T>
    static ScalarType type_of() {
        if constexpr (std::is_same_v<T, std::int32_t>) return ScalarType::I32;
        else if constexpr (std::is_same_v<T, std::int64_t>) return ScalarType::I64;
        else if constexpr (std::is_same_v<T, float>) return ScalarType::F32;
        else if constexpr (std::is_same_v<T, double>) return ScalarType::F64;
        else static_assert(sizeof(T) == 0, "kernel arguments must be i32/i64/f32/f64");
    }
    bool array_ = false;
    Direction dir_ = Direction::InOut;
    ScalarType type_ = ScalarType::I32;
    void* data_ = nullptr;
    std::uint64_t bytes_ = 0;
    LaunchArg scalar_{std::int32_t(0)};
};

template <typename T> KernelArg cu_in(std::vector<T>& h) { return KernelArg(Direction::In, h); }
template <typename T> KernelArg cu_out(std::vector<T>& h) { return KernelArg(Direction::Out, h); }
template <typename T> KernelArg cu_inout(std::vector<T>& h) { return KernelArg(Direction::InOut, h); }

struct LaunchReport {
    std::string kernel, signature;
    bool cache_hit = false;
    std::uint64_t bytes_h2d = 0, bytes_d2h = 0;
    std::optional<TrapInfo> trap;
    bool ok() const { return !trap.has_value(); }
};

struct CacheStats {
    std::uint64_t entries = 0, hits = 0, misses = 0, compiles = 0;
};
inline CacheStats cache_stats(DeviceContext& ctx) {
    const MethodCache& c = ctx.method_cache();
    return {c.entries.size(), c.hits, c.misses, c.compiles};
}

// autolaunch.hpp:167-245: signature -> method cache (bind once per signature)
// -> alloc, upload In/InOut, launch, download Out/InOut unless trapped, free.
inline LaunchReport cuda_launch(DeviceContext& ctx, const KernelAst& kernel, const GridConfig& cfg,
                                const std::vector<KernelArg>& args) {
    if (args.size() != kernel.params.size())
        throw ArityError("ArityError: kernel '" + kernel.name + "' expects " + std::to_string(kernel.params.size()) +
                         " argument(s), got " + std::to_string(args.size()));
    std::string key = kernel.name + "(";
    for (std::size_t i = 0; i < args.size(); ++i) key += (i ? "," : "") + args[i].sig();
    key += ")";
    LaunchReport rep;
    rep.kernel = kernel.name;
    rep.signature = key;
    MethodCache& cache = ctx.method_cache();
    FunctionHandle fn;
    auto hit = cache.entries.find(key);
    if (hit != cache.entries.end()) {
        ++cache.hits;
        rep.cache_hit = true;
        fn = hit->second.function;
    } else {
        ++cache.misses;
        ++cache.compiles;
        std::string text = ".module " + kernel.name + "\n.kernel " + kernel.name + "(";
        for (std::size_t i = 0; i < args.size(); ++i)
            text += (i ? ", " : "") + std::string(".param ") + args[i].vptx_type() + " " + kernel.params[i];
        text += ") {\n  ret\n}\n";
        ModuleHandle mh = ctx.module_load(text);
        fn = ctx.get_function(mh, kernel.name);
        cache.entries.emplace(key, MethodCache::Entry{mh, fn});
    }
    std::vector<std::pair<DevicePtr, const KernelArg*>> bufs;
    std::vector<LaunchArg> raw;
    for (const auto& a : args) {
        if (!a.is_array()) {
            raw.push_back(a.scalar());
            continue;
        }
        DevicePtr p = ctx.mem_alloc(a.bytes());
        if (a.direction() != Direction::Out) {
            ctx.memcpy_htod(p, a.data(), a.bytes());
            rep.bytes_h2d += a.bytes();
        }
        bufs.emplace_back(p, &a);
        raw.push_back(p);
    }
    LaunchResult r = ctx.launch(fn, cfg, raw);
    rep.trap = r.trap;
    if (r.ok())
        for (auto& [p, a] : bufs)
            if (a->direction() != Direction::In) {
                ctx.memcpy_dtoh(a->data(), p, a->bytes());
                rep.bytes_d2h += a->bytes();
            }
    for (auto& [p, a] : bufs) ctx.mem_free(p);
    return rep;
}


// ---- B200 extensions (no reference counterpart) -------------------------------------
namespace b200 {

// Host-to-host pipelined trace transform (tt_plan_*): tables, texture and outputs stay on
// the device; run() overlaps the downloads of finished angle chunks with the remaining
// launches and fills the host buffers (pinned: tt_host_alloc) -- the caller-side loop of
// cuda_launch (autolaunch.hpp:167-245) over many images of one configuration.
class TracePlan {
  public:
    TracePlan(DeviceContext& ctx, int n, int angles, bool full = true, bool features = false, int a0 = 0,
              int a_count = -1, int batch = 1, int chunks = 0, int slots = 0, int pair_stride = 0,
              bool graph = false)
        : ctx_(ctx.raw()) {
        tt_plan_desc d{n, angles, a0, a_count < 0 ? angles - a0 : a_count, full ? 1 : 0, features ? 1 : 0,
                       batch, chunks, slots, pair_stride, graph ? 1 : 0};
        detail::check(tt_plan_create(ctx_, &d, &p_), ctx_);
    }
    TracePlan(const TracePlan&) = delete;
    TracePlan& operator=(const TracePlan&) = delete;
    ~TracePlan() { tt_plan_destroy(p_); }

    // img [batch][n][n]; out [batch][a_count][F][n], med [batch][a_count][2][n],
    // circ [batch][a_count][6][3] -- any output may be nullptr (not downloaded).
    void run(const float* img, float* out, std::int32_t* med = nullptr, float* circ = nullptr) {
        detail::check(tt_plan_run(p_, img, out, med, circ), ctx_);
    }
    // Asynchronous form: buffers must stay valid until wait(); consecutive submissions overlap.
    void submit(const float* img, float* out, std::int32_t* med = nullptr, float* circ = nullptr) {
        detail::check(tt_plan_submit(p_, img, out, med, circ), ctx_);
    }
    void wait() { detail::check(tt_plan_wait(p_), ctx_); }
    int chunks() const {
        int c = 0;
        tt_plan_chunks(p_, &c);
        return c;
    }

  private:
    tt_ctx* ctx_ = nullptr;
    tt_plan* p_ = nullptr;
};

// Side of the square whose inscribed disk holds an h x w picture (tt_prep_side).
inline int prep_side(int h, int w) { return tt_prep_side(h, w); }

}  // namespace b200

}  // namespace gridjit
