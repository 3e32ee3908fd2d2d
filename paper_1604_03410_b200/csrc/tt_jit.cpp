// tt_jit.cpp — VPTX kernel bodies -> CUDA C++ -> NVRTC -> sm_100a cubin.
// Semantics: /root/reference/proj/docs/vptx-isa.md; the emulator that
// defines them: /root/reference/proj/include/gridjit/emulator.hpp:399-740
// (step_thread) and :747-793 (run_kernel).  See tt_jit.h.
#include "tt_jit.h"

#include <dlfcn.h>

#include <cctype>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

namespace tt::jit {
namespace {

// ------------------------------------------------------------------ NVRTC

// NVRTC is loaded on first use (dlopen) so the library has no link-time
// dependency on it; a missing libnvrtc fails the JIT loudly.
struct Nvrtc {
    using Prog = void*;
    int (*create)(Prog*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    int (*compile)(Prog, int, const char* const*) = nullptr;
    int (*log_size)(Prog, std::size_t*) = nullptr;
    int (*log)(Prog, char*) = nullptr;
    int (*cubin_size)(Prog, std::size_t*) = nullptr;
    int (*cubin)(Prog, char*) = nullptr;
    int (*destroy)(Prog*) = nullptr;
    bool ok = false;
    std::string why;
};

const Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void* h = nullptr;
        for (const char* lib : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
            if ((h = dlopen(lib, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
        if (!h) {
            r.why = "libnvrtc not found (dlopen)";
            return r;
        }
        auto sym = [&](auto& f, const char* s) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, s)); };
        sym(r.create, "nvrtcCreateProgram");
        sym(r.compile, "nvrtcCompileProgram");
        sym(r.log_size, "nvrtcGetProgramLogSize");
        sym(r.log, "nvrtcGetProgramLog");
        sym(r.cubin_size, "nvrtcGetCUBINSize");
        sym(r.cubin, "nvrtcGetCUBIN");
        sym(r.destroy, "nvrtcDestroyProgram");
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        if (!r.ok) r.why = "libnvrtc lacks the expected symbols";
        return r;
    }();
    return n;
}

// --------------------------------------------------------------- translator

bool parse_ty(const std::string& s, Ty& t) {
    if (s == "i32") t = Ty::I32;
    else if (s == "i64") t = Ty::I64;
    else if (s == "f32") t = Ty::F32;
    else if (s == "f64") t = Ty::F64;
    else if (s == "pred") t = Ty::Pred;
    else return false;
    return true;
}

const char* cty(Ty t) {
    switch (t) {
        case Ty::I32: return "int";
        case Ty::I64: return "long long";
        case Ty::F32: return "float";
        case Ty::F64: return "double";
        case Ty::Pred: return "bool";
    }
    return "?";
}

const char* uty(Ty t) { return t == Ty::I64 ? "unsigned long long" : "unsigned"; }
bool is_int(Ty t) { return t == Ty::I32 || t == Ty::I64; }
bool is_flt(Ty t) { return t == Ty::F32 || t == Ty::F64; }
int ty_bytes(Ty t) { return (t == Ty::I64 || t == Ty::F64) ? 8 : 4; }

struct Reg {
    Ty type;
    std::string cname;
};

struct Translator {
    const std::string& name;
    const std::vector<Param>& params;
    std::map<std::string, Reg> regs;
    std::map<std::string, std::uint64_t> shared;  // name -> byte offset
    std::map<std::string, std::string> labels;    // vptx label -> C label
    std::map<std::string, std::size_t> param_index;
    std::uint64_t shared_bytes = 0;
    std::ostringstream decl, body;
    std::string err;

    Translator(const std::string& n, const std::vector<Param>& p) : name(n), params(p) {}

    bool fail(int line, const std::string& msg) {
        err = "VPTX JIT, line " + std::to_string(line) + ": " + msg;
        return false;
    }

    // %reg -> C name (type-checked by the caller)
    const Reg* reg(const std::string& s) const {
        auto it = regs.find(s);
        return it == regs.end() ? nullptr : &it->second;
    }

    // A register operand of type t.
    bool R(int line, const std::string& s, Ty t, std::string& out) {
        const Reg* r = reg(s);
        if (!r) return fail(line, "undeclared register '" + s + "'");
        if (r->type != t) return fail(line, "register '" + s + "' has the wrong type");
        out = r->cname;
        return true;
    }

    // mov source: register, immediate, special register, parameter, shared array.
    bool mov_src(int line, const std::string& s, Ty t, std::string& out) {
        if (const Reg* r = reg(s)) {
            if (r->type != t) return fail(line, "mov between different types");
            out = r->cname;
            return true;
        }
        static const char* fam[] = {"%tid.", "%ctaid.", "%ntid.", "%nctaid."};
        static const char* cv[] = {"threadIdx.", "blockIdx.", "blockDim.", "gridDim."};
        for (int f = 0; f < 4; ++f) {
            const std::size_t L = std::strlen(fam[f]);
            if (s.size() == L + 1 && s.compare(0, L, fam[f]) == 0 && s[L] >= 'x' && s[L] <= 'z') {
                if (t != Ty::I32) return fail(line, "special registers are i32");
                out = std::string("(int)") + cv[f] + s[L];
                return true;
            }
        }
        auto pi = param_index.find(s);
        if (pi != param_index.end()) {
            const Param& p = params[pi->second];
            if (p.ptr ? t != Ty::I64 : t != p.type) return fail(line, "parameter '" + s + "' moved as a wrong type");
            out = "(" + std::string(cty(t)) + ")P" + std::to_string(pi->second);
            return true;
        }
        auto si = shared.find(s);
        if (si != shared.end()) {
            if (t != Ty::I64) return fail(line, "shared array base is i64");
            out = std::to_string(si->second) + "LL";
            return true;
        }
        // immediates
        if (s.size() == 10 && s[0] == '0' && s[1] == 'f' && t == Ty::F32) {
            out = "__int_as_float((int)0x" + s.substr(2) + "u)";
            return true;
        }
        if (s.size() == 18 && s[0] == '0' && s[1] == 'd' && t == Ty::F64) {
            out = "__longlong_as_double((long long)0x" + s.substr(2) + "ull)";
            return true;
        }
        if (is_int(t) && !s.empty() && (std::isdigit((unsigned char)s[0]) || (s[0] == '-' && s.size() > 1))) {
            for (std::size_t i = (s[0] == '-'); i < s.size(); ++i)
                if (!std::isdigit((unsigned char)s[i])) return fail(line, "bad integer immediate '" + s + "'");
            out = t == Ty::I32 ? "(int)(" + s + "LL)" : "(long long)(" + s + "LL)";
            if (s == "-9223372036854775808") out = "(long long)(-9223372036854775807LL - 1)";
            return true;
        }
        return fail(line, "bad mov source '" + s + "'");
    }

    static bool split_op(const std::string& op, std::vector<std::string>& parts) {
        parts.clear();
        std::size_t s = 0;
        for (std::size_t i = 0; i <= op.size(); ++i)
            if (i == op.size() || op[i] == '.') {
                parts.push_back(op.substr(s, i - s));
                s = i + 1;
            }
        return !parts.empty();
    }

    bool instr(const Line& l, std::size_t idx) {
        std::vector<std::string> ops;  // operands without punctuation
        for (std::size_t i = 1; i < l.toks.size(); ++i)
            if (l.toks[i] != "," && l.toks[i] != "[" && l.toks[i] != "]") ops.push_back(l.toks[i]);
        std::vector<std::string> p;
        split_op(l.toks[0], p);
        const std::string& op = p[0];
        const std::string I = std::to_string(idx);
        auto need = [&](std::size_t n) { return ops.size() == n ? true : fail(l.no, "wrong operand count"); };
        auto tyat = [&](std::size_t k, Ty& t) {
            return k < p.size() && parse_ty(p[k], t) ? true : fail(l.no, "bad type suffix in '" + l.toks[0] + "'");
        };
        std::string d, a, b, c;
        Ty t;
        if (op == "ret" && p.size() == 1) {
            body << "  return;\n";
            return true;
        }
        if (op == "trap" && p.size() == 1) {
            if (!need(1)) return false;
            body << "  TT_TRAP(5, " << I << ", (" << ops[0] << "LL));\n";
            return true;
        }
        if (op == "bar" && p.size() == 2 && p[1] == "sync") {
            body << "  __syncthreads(); ++tt_phase;\n";
            return true;
        }
        if (op == "bra") {
            if (p.size() == 1) {
                if (!need(1) || !labels.count(ops[0])) return fail(l.no, "bad branch");
                body << "  goto " << labels[ops[0]] << ";\n";
                return true;
            }
            if (p.size() == 2 && p[1] == "p") {
                if (!need(2) || !labels.count(ops[1]) || !R(l.no, ops[0], Ty::Pred, a)) return fail(l.no, "bad branch");
                body << "  if (" << a << ") goto " << labels[ops[1]] << ";\n";
                return true;
            }
        }
        if (op == "mov") {
            if (!tyat(1, t) || !need(2) || !R(l.no, ops[0], t, d) || !mov_src(l.no, ops[1], t, a)) return false;
            body << "  " << d << " = " << a << ";\n";
            return true;
        }
        if (op == "add" || op == "sub" || op == "mul" || op == "div" || op == "rem" || op == "min" ||
            op == "max") {
            if (!tyat(1, t) || !need(3) || !R(l.no, ops[0], t, d) || !R(l.no, ops[1], t, a) || !R(l.no, ops[2], t, b))
                return false;
            const bool f32 = t == Ty::F32;
            std::string e;
            if (is_flt(t)) {
                if (op == "rem") return fail(l.no, "rem is integer-only");
                const char* pre = f32 ? "__f" : "__d";
                if (op == "add") e = std::string(pre) + "add_rn(" + a + ", " + b + ")";
                else if (op == "sub") e = std::string(pre) + "sub_rn(" + a + ", " + b + ")";
                else if (op == "mul") e = std::string(pre) + "mul_rn(" + a + ", " + b + ")";
                else if (op == "div") e = std::string(pre) + "div_rn(" + a + ", " + b + ")";
                else if (op == "min") e = std::string(f32 ? "fminf(" : "fmin(") + a + ", " + b + ")";
                else e = std::string(f32 ? "fmaxf(" : "fmax(") + a + ", " + b + ")";
            } else if (is_int(t)) {
                const std::string U = uty(t), T = cty(t);
                if (op == "add") e = "(" + T + ")((" + U + ")" + a + " + (" + U + ")" + b + ")";
                else if (op == "sub") e = "(" + T + ")((" + U + ")" + a + " - (" + U + ")" + b + ")";
                else if (op == "mul") e = "(" + T + ")((" + U + ")" + a + " * (" + U + ")" + b + ")";
                else if (op == "min") e = "(" + a + " < " + b + " ? " + a + " : " + b + ")";
                else if (op == "max") e = "(" + a + " > " + b + " ? " + a + " : " + b + ")";
                else {  // div / rem: trap on zero; INT_MIN / -1 wraps, INT_MIN % -1 == 0
                    body << "  if (" << b << " == 0) TT_TRAP(3, " << I << ", 0);\n";
                    if (op == "div") e = "(" + b + " == -1 ? (" + T + ")(0 - (" + U + ")" + a + ") : " + a + " / " + b + ")";
                    else e = "(" + b + " == -1 ? (" + T + ")0 : " + a + " % " + b + ")";
                }
            } else {
                return fail(l.no, "arithmetic on predicates");
            }
            body << "  " << d << " = " << e << ";\n";
            return true;
        }
        if (op == "neg" || op == "abs" || op == "sqrt" || op == "sin" || op == "cos" || op == "exp" || op == "log") {
            if (!tyat(1, t) || !need(2) || !R(l.no, ops[0], t, d) || !R(l.no, ops[1], t, a)) return false;
            const bool f32 = t == Ty::F32;
            std::string e;
            if (op == "neg") {
                if (is_int(t)) e = "(" + std::string(cty(t)) + ")(0 - (" + uty(t) + ")" + a + ")";
                else if (is_flt(t)) e = "(-" + a + ")";
                else return fail(l.no, "neg of a predicate");
            } else if (op == "abs") {
                if (is_int(t)) e = "(" + a + " < 0 ? (" + cty(t) + ")(0 - (" + uty(t) + ")" + a + ") : " + a + ")";
                else if (is_flt(t)) e = std::string(f32 ? "fabsf(" : "fabs(") + a + ")";
                else return fail(l.no, "abs of a predicate");
            } else {
                if (!is_flt(t)) return fail(l.no, op + " is float-only");
                if (op == "sqrt") e = std::string(f32 ? "__fsqrt_rn(" : "__dsqrt_rn(") + a + ")";
                else e = (f32 ? op + "f(" : op + "(") + a + ")";
            }
            body << "  " << d << " = " << e << ";\n";
            return true;
        }
        if (op == "fma") {
            if (!tyat(1, t) || !is_flt(t) || !need(4) || !R(l.no, ops[0], t, d) || !R(l.no, ops[1], t, a) ||
                !R(l.no, ops[2], t, b) || !R(l.no, ops[3], t, c))
                return false;
            body << "  " << d << " = " << (t == Ty::F32 ? "__fmaf_rn(" : "__fma_rn(") << a << ", " << b << ", "
                 << c << ");\n";
            return true;
        }
        if (op == "and" || op == "or" || op == "xor" || op == "not") {
            if (!tyat(1, t) || t != Ty::Pred) return fail(l.no, "logic ops are pred-only");
            if (op == "not") {
                if (!need(2) || !R(l.no, ops[0], t, d) || !R(l.no, ops[1], t, a)) return false;
                body << "  " << d << " = !" << a << ";\n";
                return true;
            }
            if (!need(3) || !R(l.no, ops[0], t, d) || !R(l.no, ops[1], t, a) || !R(l.no, ops[2], t, b)) return false;
            const char* o = op == "and" ? " && " : op == "or" ? " || " : " != ";
            body << "  " << d << " = " << a << o << b << ";\n";
            return true;
        }
        if (op == "setp") {
            if (p.size() != 3 || !tyat(2, t) || t == Ty::Pred || !need(3) || !R(l.no, ops[0], Ty::Pred, d) ||
                !R(l.no, ops[1], t, a) || !R(l.no, ops[2], t, b))
                return fail(l.no, "bad setp");
            static const std::map<std::string, std::string> cmp = {{"eq", " == "}, {"ne", " != "}, {"lt", " < "},
                                                                   {"le", " <= "}, {"gt", " > "}, {"ge", " >= "}};
            auto it = cmp.find(p[1]);
            if (it == cmp.end()) return fail(l.no, "bad comparison '" + p[1] + "'");
            body << "  " << d << " = " << a << it->second << b << ";\n";  // C++ float compares are IEEE (NaN: only != true)
            return true;
        }
        if (op == "cvt") {
            Ty td, ts;
            if (p.size() != 3 || !tyat(1, td) || !tyat(2, ts) || td == ts || td == Ty::Pred || ts == Ty::Pred ||
                !need(2) || !R(l.no, ops[0], td, d) || !R(l.no, ops[1], ts, a))
                return fail(l.no, "bad cvt");
            std::string e;
            if (is_int(td) && is_int(ts)) e = "(" + std::string(cty(td)) + ")" + a;  // sign-extend / truncate
            else if (is_flt(td) && is_int(ts))
                e = std::string(td == Ty::F32 ? (ts == Ty::I32 ? "__int2float_rn(" : "__ll2float_rn(")
                                              : (ts == Ty::I32 ? "__int2double_rn(" : "__ll2double_rn(")) + a + ")";
            else if (td == Ty::F64 && ts == Ty::F32) e = "(double)" + a;
            else if (td == Ty::F32 && ts == Ty::F64) e = "__double2float_rn(" + a + ")";
            else  // float -> int: truncation toward zero, saturating, NaN -> 0 (cvt.rzi semantics)
                e = std::string(ts == Ty::F32 ? (td == Ty::I32 ? "__float2int_rz(" : "__float2ll_rz(")
                                              : (td == Ty::I32 ? "__double2int_rz(" : "__double2ll_rz(")) + a + ")";
            body << "  " << d << " = " << e << ";\n";
            return true;
        }
        if (op == "ld" || op == "st") {
            if (p.size() != 3 || (p[1] != "global" && p[1] != "shared") || !tyat(2, t) || t == Ty::Pred || !need(2))
                return fail(l.no, "bad " + op);
            const bool ld = op == "ld";
            std::string addr, data;
            if (!R(l.no, ld ? ops[1] : ops[0], Ty::I64, addr) || !R(l.no, ld ? ops[0] : ops[1], t, data)) return false;
            const std::string nb = std::to_string(ty_bytes(t));
            if (p[1] == "global") {
                // one-entry per-thread cache of the last live allocation hit (the table is
                // fixed for the launch): the binary search runs only on a miss
                body << "  { const unsigned long long a_ = (unsigned long long)" << addr << "; if (!(a_ >= tt_clo && a_ + "
                     << nb << "ull <= tt_chi && a_ + " << nb << "ull >= a_)) { const int c_ = tt_gcheck(tt_rng, tt_nrng, a_, "
                     << nb << ", tt_clo, tt_chi); if (c_ != 2) TT_TRAP(c_ == 1 ? 2 : 0, " << I << ", 0); } ";
                if (ld) body << data << " = tt_ld<" << cty(t) << ">((const unsigned char*)a_); }\n";
                else body << "tt_st<" << cty(t) << ">((unsigned char*)a_, " << data << "); }\n";
            } else {
                body << "  { const unsigned long long a_ = (unsigned long long)" << addr << "; if (a_ + " << nb
                     << "ull > (unsigned long long)tt_shbytes || a_ + " << nb << "ull < a_) TT_TRAP(1, " << I
                     << ", 0); ";
                if (ld) body << data << " = tt_ld<" << cty(t) << ">(tt_sh + a_); }\n";
                else body << "tt_st<" << cty(t) << ">(tt_sh + a_, " << data << "); }\n";
            }
            return true;
        }
        return fail(l.no, "unsupported instruction '" + l.toks[0] + "'");
    }

    bool run(const std::vector<Line>& lines, std::string& src, std::uint64_t& static_shared) {
        for (std::size_t i = 0; i < params.size(); ++i) param_index[params[i].name] = i;
        // declarations first (registers, shared arrays), labels (pseudo-instructions)
        std::size_t nregs = 0, nlab = 0;
        for (const Line& l : lines) {
            const auto& t = l.toks;
            if (t[0] == ".reg") {
                Ty ty;
                if (t.size() != 3 || !parse_ty(t[1], ty)) return fail(l.no, "bad .reg");
                if (regs.count(t[2])) return fail(l.no, "register redeclared");
                regs[t[2]] = Reg{ty, "r" + std::to_string(nregs++)};
            } else if (t[0] == ".shared") {  // .shared <elem> <name>[<count>]: naturally aligned, in order
                Ty ty;
                if (t.size() != 6 || !parse_ty(t[1], ty) || ty == Ty::Pred || t[3] != "[" || t[5] != "]")
                    return fail(l.no, "bad .shared");
                const std::uint64_t al = std::uint64_t(ty_bytes(ty));
                shared_bytes = (shared_bytes + al - 1) / al * al;
                shared[t[2]] = shared_bytes;
                shared_bytes += al * std::stoull(t[4]);
            } else if (t.size() == 1 && t[0].size() > 1 && t[0].back() == ':') {
                labels[t[0].substr(0, t[0].size() - 1)] = "L" + std::to_string(nlab++);
            }
        }
        for (const auto& kv : regs)
            decl << "  " << cty(kv.second.type) << " " << kv.second.cname << " = 0;\n";
        std::size_t idx = 0;  // body index (labels count, as in the emulator's pc)
        for (const Line& l : lines) {
            const auto& t = l.toks;
            if (t[0] == ".reg" || t[0] == ".shared") continue;
            if (t.size() == 1 && t[0].back() == ':') {
                body << labels[t[0].substr(0, t[0].size() - 1)] << ":;\n";
                ++idx;
                continue;
            }
            if (!instr(l, idx)) return false;
            ++idx;
        }
        std::ostringstream s;
        s << "typedef unsigned long long u64;\n"
             "struct TtTrap { u64 key; int lock; int kind; long long code; int instr; unsigned tid[3], ctaid[3]; };\n"
             "__device__ __forceinline__ void tt_report(TtTrap* t, int kind, int instr, long long code, unsigned ph) {\n"
             "  const u64 blk = ((u64)blockIdx.x * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z;\n"
             "  const unsigned lt = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);\n"
             "  const u64 key = (blk << 32) | ((u64)(ph < 2097151u ? ph : 2097151u) << 11) | lt;\n"
             "  while (atomicCAS(&t->lock, 0, 1) != 0) {}\n"
             "  __threadfence();\n"
             "  volatile TtTrap* v = t;\n"
             "  if (key < v->key) { v->key = key; v->kind = kind; v->code = code; v->instr = instr;\n"
             "    v->tid[0] = threadIdx.x; v->tid[1] = threadIdx.y; v->tid[2] = threadIdx.z;\n"
             "    v->ctaid[0] = blockIdx.x; v->ctaid[1] = blockIdx.y; v->ctaid[2] = blockIdx.z; }\n"
             "  __threadfence();\n"
             "  atomicExch(&t->lock, 0);\n"
             "}\n"
             "// 0: outside every allocation, 1: inside a freed one, 2: live (rng: sorted [begin, end, live])\n"
             "__device__ __forceinline__ int tt_gcheck(const u64* rng, int nr, u64 a, unsigned len, u64& clo, u64& chi) {\n"
             "  int lo = 0, hi = nr - 1, f = -1;\n"
             "  while (lo <= hi) { const int m = (lo + hi) >> 1; if (rng[3 * m] <= a) { f = m; lo = m + 1; } else hi = m - 1; }\n"
             "  if (f < 0 || a + len > rng[3 * f + 1] || a + len < a) return 0;\n"
             "  if (!rng[3 * f + 2]) return 1;\n"
             "  clo = rng[3 * f]; chi = rng[3 * f + 1];\n"
             "  return 2;\n"
             "}\n"
             "template <class T> __device__ __forceinline__ T tt_ld(const unsigned char* p) {\n"
             "  if (((u64)p & (sizeof(T) - 1)) == 0) return *(const T*)p;\n"
             "  T v; unsigned char* q = (unsigned char*)&v; for (int i = 0; i < (int)sizeof(T); ++i) q[i] = p[i]; return v;\n"
             "}\n"
             "template <class T> __device__ __forceinline__ void tt_st(unsigned char* p, T v) {\n"
             "  if (((u64)p & (sizeof(T) - 1)) == 0) { *(T*)p = v; return; }\n"
             "  const unsigned char* q = (const unsigned char*)&v; for (int i = 0; i < (int)sizeof(T); ++i) p[i] = q[i];\n"
             "}\n"
             "#define TT_TRAP(kind, instr, code) do { tt_report(tt_trap, (kind), (instr), (long long)(code), tt_phase); return; } while (0)\n";
        s << "extern \"C\" __global__ void tt_jit_kernel(";
        for (std::size_t i = 0; i < params.size(); ++i)
            s << (params[i].ptr ? "long long" : cty(params[i].type)) << " P" << i << ", ";
        s << "TtTrap* tt_trap, const u64* tt_rng, int tt_nrng, unsigned tt_shbytes) {\n"
             "  extern __shared__ __align__(16) unsigned char tt_sh[];\n"
             "  unsigned tt_phase = 0;\n"
             "  u64 tt_clo = 1, tt_chi = 0;  // cached live allocation [lo, hi): empty\n"
          << decl.str() << body.str()
          << "  return;\n"  // control never falls off the end of a valid body
             "}\n";
        src = s.str();
        static_shared = shared_bytes;
        return true;
    }
};

}  // namespace

bool translate(const std::string& name, const std::vector<Param>& params, const std::vector<Line>& lines,
               std::string& source, std::uint64_t& static_shared, std::string& err) {
    Translator tr(name, params);
    if (!tr.run(lines, source, static_shared)) {
        err = tr.err;
        return false;
    }
    return true;
}

bool compile(const std::string& name, const std::vector<Param>& params, const std::vector<Line>& lines,
             Program& out, std::string& err) {
    std::string src;
    if (!translate(name, params, lines, src, out.static_shared, err)) return false;
    out.source = src;
    const Nvrtc& nv = nvrtc();
    if (!nv.ok) {
        err = "VPTX JIT unavailable: " + nv.why;
        return false;
    }
    Nvrtc::Prog prog = nullptr;
    if (nv.create(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != 0) {
        err = "nvrtcCreateProgram failed";
        return false;
    }
    const char* opts[] = {"-arch=sm_100a", "--fmad=false", "-default-device", "-std=c++17"};
    const int rc = nv.compile(prog, 4, opts);
    if (rc != 0) {
        std::size_t n = 0;
        nv.log_size(prog, &n);
        std::string log(n, '\0');
        if (n) nv.log(prog, log.data());
        nv.destroy(&prog);
        err = "VPTX JIT compile failed for '" + name + "': " + log;
        return false;
    }
    std::size_t n = 0;
    nv.cubin_size(prog, &n);
    std::string cubin(n, '\0');
    nv.cubin(prog, cubin.data());
    nv.destroy(&prog);
    cudaError_t e = cudaLibraryLoadData(&out.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&out.kernel, out.lib, "tt_jit_kernel");
    if (e != cudaSuccess) {
        err = std::string("loading the JIT cubin: ") + cudaGetErrorString(e);
        release(out);
        return false;
    }
    return true;
}

void release(Program& p) {
    if (p.lib) cudaLibraryUnload(p.lib);
    p.lib = nullptr;
    p.kernel = nullptr;
}

}  // namespace tt::jit
