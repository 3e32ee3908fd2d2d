// tt_host.cpp — host-side inputs of the trace transform (product side):
// angle/weight tables, the deterministic synthetic images of DESIGN.md
// §2.1-2.4, and the picture formats on the caller side (PNM files, the
// grayscale + circumscribed-square preparation launcher).  These are inputs the caller hands to the device kernels (the
// reference-style DSL kernel takes ctab/stab as array arguments, SURVEY.md
// Appendix B); the independent restatement in oracle/tt_oracle.c checks them
// bit-for-bit (tests/test_host_inputs.py).
//
// Compiled with -ffp-contract=off (like /root/reference/proj/CMakeLists.txt:15-16)
// so every f64 expression rounds exactly as written.
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "tt_b200.h"
#include "tt_kernels.cuh"

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kPi = 3.14159265358979323846;

std::uint64_t mix64(std::uint64_t x) {
    std::uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Uniform [0,1) f64 for parameter k of ellipse i.
double param01(std::uint64_t seed, int i, int k) {
    const std::uint64_t key = seed ^ (0x1000ull + 16ull * std::uint64_t(i) + std::uint64_t(k));
    return double(mix64(key) >> 11) * (1.0 / 9007199254740992.0);
}

struct Ellipse {
    double cx, cy, ra, rb, cphi, sphi, alpha;
};

}  // namespace

extern "C" tt_status tt_make_tables(int n, int a_total, float* ctab, float* stab, float* wtab) {
    if (n < 0 || a_total < 0) return TT_ERR_INVALID;
    for (int a = 0; a < a_total; ++a) {
        const double theta = kTwoPi * double(a) / double(a_total);
        if (ctab) ctab[a] = float(std::cos(theta));
        if (stab) stab[a] = float(std::sin(theta));
    }
    if (wtab == nullptr) return TT_OK;
    for (int r = 0; r < n; ++r) {
        double re3 = 0, im3 = 0, re4 = 0, im4 = 0, re5 = 0, im5 = 0;
        const double rr = double(r);
        if (r > 0) {
            const double lg = std::log(rr);
            const double sq = std::sqrt(rr);
            re3 = rr * std::cos(5.0 * lg);
            im3 = rr * std::sin(5.0 * lg);
            re4 = std::cos(3.0 * lg);
            im4 = std::sin(3.0 * lg);
            re5 = sq * std::cos(4.0 * lg);
            im5 = sq * std::sin(4.0 * lg);
        }
        float* e = wtab + 8 * std::size_t(r);  // [n][8] (spec §2.2)
        e[0] = float(rr);
        e[1] = float(rr * rr);
        e[2] = float(re3);
        e[3] = float(im3);
        e[4] = float(re4);
        e[5] = float(im4);
        e[6] = float(re5);
        e[7] = float(im5);
    }
    return TT_OK;
}

extern "C" tt_status tt_synth_image(int kind, std::uint64_t seed, int n, float* img) {
    if (n < 0 || img == nullptr || kind < 0 || kind > 2) return TT_ERR_INVALID;
    const std::int64_t nm1 = std::int64_t(n) - 1;
    Ellipse el[8];
    if (kind == 1) {
        const double centre = 0.5 * double(nm1);
        for (int i = 0; i < 8; ++i) {
            el[i].cx = centre + (param01(seed, i, 0) - 0.5) * 0.5 * double(n);
            el[i].cy = centre + (param01(seed, i, 1) - 0.5) * 0.5 * double(n);
            el[i].ra = (0.05 + 0.25 * param01(seed, i, 2)) * double(n);
            el[i].rb = (0.05 + 0.25 * param01(seed, i, 3)) * double(n);
            const double phi = kPi * param01(seed, i, 4);
            el[i].cphi = std::cos(phi);
            el[i].sphi = std::sin(phi);
            el[i].alpha = 0.1 + 0.9 * param01(seed, i, 5);
        }
    }
    for (std::int64_t y = 0; y < n; ++y) {
        const std::int64_t ddy = 2 * y - nm1;
        for (std::int64_t x = 0; x < n; ++x) {
            const std::uint64_t h = mix64(seed ^ std::uint64_t(y * n + x));
            const float noise = float(h >> 40) * (1.0f / 16777216.0f);
            const std::int64_t ddx = 2 * x - nm1;
            const bool disk = ddx * ddx + ddy * ddy <= nm1 * nm1;
            float value = 0.0f;
            switch (kind) {
                case 0: value = disk ? noise : 0.0f; break;
                case 2: value = (h & 127u) == 0 ? noise : 0.0f; break;
                default: {
                    double sum = 0.0;
                    for (const Ellipse& e : el) {
                        const double dx = double(x) - e.cx, dy = double(y) - e.cy;
                        const double xr = dx * e.cphi + dy * e.sphi;
                        const double yr = dy * e.cphi - dx * e.sphi;
                        const double q = (xr / e.ra) * (xr / e.ra) + (yr / e.rb) * (yr / e.rb);
                        if (q <= 1.0) sum += e.alpha;
                    }
                    value = disk ? float(sum) : 0.0f;
                }
            }
            img[std::size_t(y) * std::size_t(n) + std::size_t(x)] = value;
        }
    }
    return TT_OK;
}

namespace {

// The kernels' fp32 line geometry (spec §2.1), evaluated on the host.
struct LineGeom {
    float o, hi, u, w, c, s;
    LineGeom(int n, float c_, float s_, int p) : c(c_), s(s_) {
        o = float(n - 1) * 0.5f;
        hi = float(n - 1);
        const float x = float(p) - o;
        u = std::fmaf(x, c, o);
        w = std::fmaf(x, s, o);
    }
    bool inside(int t) const {
        const float y = float(t) - o;
        const float qx = std::fmaf(-y, s, u), qy = std::fmaf(y, c, w);
        return qx >= 0.0f && qx < hi && qy >= 0.0f && qy < hi;
    }
};

// First t in [lo, hi) with pred(t) == want given pred is monotone; hi if none.
template <class P>
int first_switch(int lo, int hi, bool want, P pred) {
    while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        if (pred(mid) == want) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

}  // namespace

extern "C" std::uint64_t tt_count_inbounds_taps(int n, int a0, int a_count, const float* ctab, const float* stab) {
    if (n < 1 || a_count < 1 || !ctab || !stab) return 0;
    std::uint64_t total = 0;
    for (int a = a0; a < a0 + a_count; ++a) {
        for (int p = 0; p < n; ++p) {
            const LineGeom g(n, ctab[a], stab[a], p);
            // Each of the four half-plane tests is monotone in t, so the inside
            // set is one interval [t_lo, t_hi); find a member by sampling, then
            // bisect both ends.
            int member = -1;
            const int probes = 64;
            for (int k = 0; k <= probes && member < 0; ++k) {
                const int t = int((long long)(n - 1) * k / probes);
                if (g.inside(t)) member = t;
            }
            if (member < 0) {  // thin intersection: fall back to a scan
                int cnt = 0;
                for (int t = 0; t < n; ++t) cnt += g.inside(t);
                total += std::uint64_t(cnt);
                continue;
            }
            const int lo = first_switch(0, member, true, [&](int t) { return g.inside(t); });
            const int hi = first_switch(member, n, false, [&](int t) { return g.inside(t); });
            total += std::uint64_t(hi - lo);
        }
    }
    return total;
}

// ---------------------------------------------------------------- formats

extern "C" int tt_prep_side(int h, int w) {
    if (h < 1 || w < 1) return 0;
    const std::uint64_t d2 = std::uint64_t(h) * h + std::uint64_t(w) * w;
    std::uint64_t m = std::uint64_t(std::sqrt(double(d2)));
    while (m * m < d2) ++m;  // m = ceil(sqrt(h^2 + w^2)) exactly
    while (m > 0 && (m - 1) * (m - 1) >= d2) --m;
    return int(m + 1);
}

extern "C" tt_status tt_prep_device(const std::uint8_t* d_pix, int h, int w, int channels, int n, float* d_img,
                                   void* stream) {
    if (!d_pix || !d_img || h < 1 || w < 1 || (channels != 1 && channels != 3) || n < std::max(h, w))
        return TT_ERR_INVALID;
    cudaError_t e = tt::launch_prep(d_pix, h, w, channels, n, d_img, (cudaStream_t)stream);
    return e == cudaSuccess ? TT_OK : TT_ERR_CUDA;
}

namespace {
int pnm_token(std::FILE* f) {  // next decimal header field, skipping whitespace and # comments
    int c = std::fgetc(f);
    for (;;) {
        while (c == ' ' || c == '\t' || c == '\r' || c == '\n') c = std::fgetc(f);
        if (c != '#') break;
        while (c != '\n' && c != EOF) c = std::fgetc(f);
    }
    if (c < '0' || c > '9') return -1;
    long v = 0;
    while (c >= '0' && c <= '9') {
        v = v * 10 + (c - '0');
        if (v > (1 << 28)) return -1;
        c = std::fgetc(f);
    }
    return int(v);  // the single whitespace after maxval is consumed here
}
}  // namespace

extern "C" tt_status tt_pnm_read(const char* path, int* h, int* w, int* channels, std::uint8_t* pix, std::size_t cap) {
    if (!path || !h || !w || !channels) return TT_ERR_INVALID;
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return TT_ERR_INVALID;
    char m[2] = {0, 0};
    tt_status st = TT_ERR_INVALID;
    if (std::fread(m, 1, 2, f) == 2 && m[0] == 'P' && (m[1] == '5' || m[1] == '6')) {
        const int ww = pnm_token(f), hh = pnm_token(f), mx = pnm_token(f);
        const int ch = m[1] == '6' ? 3 : 1;
        if (ww > 0 && hh > 0 && mx == 255) {
            const std::size_t bytes = std::size_t(ww) * hh * ch;
            if (!pix) {
                st = TT_OK;
            } else if (cap >= bytes && std::fread(pix, 1, bytes, f) == bytes) {
                st = TT_OK;
            }
            if (st == TT_OK) {
                *h = hh;
                *w = ww;
                *channels = ch;
            }
        }
    }
    std::fclose(f);
    return st;
}

extern "C" tt_status tt_pgm_write(const char* path, const float* img, int h, int w, float lo, float hi) {
    if (!path || !img || h < 1 || w < 1 || !(hi > lo)) return TT_ERR_INVALID;
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return TT_ERR_INVALID;
    std::fprintf(f, "P5\n%d %d\n255\n", w, h);
    std::vector<std::uint8_t> row(static_cast<std::size_t>(w));
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const double t = (double(img[std::size_t(y) * w + x]) - lo) / (double(hi) - lo);
            row[x] = std::uint8_t(std::lround(std::min(1.0, std::max(0.0, t)) * 255.0));
        }
        std::fwrite(row.data(), 1, row.size(), f);
    }
    const bool ok = std::fflush(f) == 0;
    std::fclose(f);
    return ok ? TT_OK : TT_ERR_INVALID;
}
