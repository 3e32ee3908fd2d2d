/*
 * tt_oracle.c — CPU restatement of the trace transform. TEST INFRASTRUCTURE
 * ONLY (see tt_oracle.h): the checker for the B200 product, never shipped on
 * the product path.
 *
 * Spec: DESIGN.md §2 (frozen from SURVEY.md Appendix A; algorithm shape from
 * per-orientation projections reduced by
 * T-functionals; reference numeric conventions from
 * /root/reference/proj/include/gridjit/emulator.hpp:5-20).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).  The
 * -ffp-contract=off flag mirrors /root/reference/proj/CMakeLists.txt:15-16 so
 * that only the explicit fmaf() calls below are fused.
 */
#include "tt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- tables */

/* wtab layout [n][8] per r: r, r^2, w3re, w3im, w4re, w4im, w5re, w5im */
#define WT(w, r, j) ((w)[8 * (size_t)(r) + 2 + (j)])

/* spec §2.1: theta_a = 2*pi*a/A evaluated in f64, rounded to f32 once. */
void tto_tables(int n, int a_total, float* ctab, float* stab, float* wtab) {
    const double two_pi = 6.283185307179586476925286766559;
    for (int a = 0; a < a_total; ++a) {
        double th = two_pi * (double)a / (double)a_total;
        if (ctab) ctab[a] = (float)cos(th);
        if (stab) stab[a] = (float)sin(th);
    }
    if (!wtab) return;
    /* spec §2.2: w3 = r e^{i5 ln r}, w4 = e^{i3 ln r}, w5 = sqrt(r) e^{i4 ln r}; r=0 -> 0 */
    for (int r = 0; r < n; ++r) {
        double w3r = 0, w3i = 0, w4r = 0, w4i = 0, w5r = 0, w5i = 0;
        if (r >= 1) {
            double lr = log((double)r);
            double rr = (double)r, sr = sqrt((double)r);
            w3r = rr * cos(5.0 * lr); w3i = rr * sin(5.0 * lr);
            w4r = cos(3.0 * lr);      w4i = sin(3.0 * lr);
            w5r = sr * cos(4.0 * lr); w5i = sr * sin(4.0 * lr);
        }
        float* e = wtab + 8 * (size_t)r;
        e[0] = (float)r;
        e[1] = (float)((double)r * (double)r);
        e[2] = (float)w3r; e[3] = (float)w3i;
        e[4] = (float)w4r; e[5] = (float)w4i;
        e[6] = (float)w5r; e[7] = (float)w5i;
    }
}

/* ---------------------------------------------------------------- images */

static uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double draw01(uint64_t seed, int i, int k) {
    return (double)(splitmix64(seed ^ (0x1000ull + 16ull * (uint64_t)i + (uint64_t)k)) >> 11) *
           (1.0 / 9007199254740992.0);
}

/* spec §2.4 */
void tto_synth(int kind, uint64_t seed, int n, float* img) {
    const int64_t n1 = (int64_t)n - 1;
    double cx[8], cy[8], ra[8], rb[8], cp[8], sp[8], al[8];
    if (kind == TTO_PHANTOM) {
        const double o = 0.5 * (double)n1;
        for (int i = 0; i < 8; ++i) {
            cx[i] = o + (draw01(seed, i, 0) - 0.5) * 0.5 * (double)n;
            cy[i] = o + (draw01(seed, i, 1) - 0.5) * 0.5 * (double)n;
            ra[i] = (0.05 + 0.25 * draw01(seed, i, 2)) * (double)n;
            rb[i] = (0.05 + 0.25 * draw01(seed, i, 3)) * (double)n;
            double ph = 3.14159265358979323846 * draw01(seed, i, 4);
            cp[i] = cos(ph);
            sp[i] = sin(ph);
            al[i] = 0.1 + 0.9 * draw01(seed, i, 5);
        }
    }
    for (int row = 0; row < n; ++row) {
        for (int col = 0; col < n; ++col) {
            uint64_t h = splitmix64(seed ^ (uint64_t)((int64_t)row * n + col));
            float u = (float)(h >> 40) * (1.0f / 16777216.0f);
            int64_t dx = 2 * (int64_t)col - n1, dy = 2 * (int64_t)row - n1;
            int in_disk = dx * dx + dy * dy <= n1 * n1;
            float val = 0.0f;
            if (kind == TTO_DISK) {
                val = in_disk ? u : 0.0f;
            } else if (kind == TTO_SPARSE) {
                val = ((h & 127u) == 0) ? u : 0.0f;
            } else {
                double acc = 0.0;
                for (int i = 0; i < 8; ++i) {
                    double ex = (double)col - cx[i], ey = (double)row - cy[i];
                    double xr = ex * cp[i] + ey * sp[i];
                    double yr = ey * cp[i] - ex * sp[i];
                    double q = (xr / ra[i]) * (xr / ra[i]) + (yr / rb[i]) * (yr / rb[i]);
                    if (q <= 1.0) acc += al[i];
                }
                val = in_disk ? (float)acc : 0.0f;
            }
            img[(size_t)row * n + col] = val;
        }
    }
}

/* --------------------------------------------------------------- sampler */

/* spec §2.1: pinned fmaf forms; truncation == floor because the bounds test
 * has already established q >= 0. */
static inline float tap(const float* img, int n, float hi, float qx, float qy) {
    if (!(qx >= 0.0f && qx < hi && qy >= 0.0f && qy < hi)) return 0.0f;
    int ix = (int)qx, iy = (int)qy;
    float fx = qx - (float)ix, fy = qy - (float)iy;
    const float* r0 = img + (size_t)iy * n + ix;
    const float* r1 = r0 + n;
    float top = fmaf(fx, r0[1] - r0[0], r0[0]);
    float bot = fmaf(fx, r1[1] - r1[0], r1[0]);
    return fmaf(fy, bot - top, top);
}

void tto_line_samples(const float* img, int n, float c, float s, int p, float* v) {
    const float o = (float)(n - 1) * 0.5f;
    const float hi = (float)(n - 1);
    const float x = (float)p - o;
    const float u = fmaf(x, c, o);
    const float w = fmaf(x, s, o);
    for (int t = 0; t < n; ++t) {
        float y = (float)t - o;
        float qx = fmaf(-y, s, u);
        float qy = fmaf(y, c, w);
        v[t] = tap(img, n, hi, qx, qy);
    }
}

/* Mirrors tt::schedule_slots (paper_1604_03410_b200/csrc/tt_kernels.cu): the
 * slots per line NS.  n <= 1024: one segment of 8, 16 or 32 lanes (the
 * smallest with ceil(n/NS) <= 32; sub-warp segments need 32/NS | n, else 32);
 * larger n: 32W lanes, W the smallest power of two with ceil(n/32W) <= 32,
 * at most 16; T0-only (full = 0) with n > 1024: 32 (one warp per line). */
int tto_schedule_slots(int n, int full) {
    if (!full && n > 1024) return 32;
    if (n <= 1024) {
        int seg = 8;
        while (seg < 32 && (n + seg - 1) / seg > 32) seg *= 2;
        if (seg < 32 && n % (32 / seg) != 0) seg = 32;
        return seg;
    }
    int w = 1;
    while (w * 1024 < n && w < 16) w *= 2;
    return 32 * w;
}

/* ----------------------------------------------------- f64 truth (§2.5) */

static int median64(const float* v, int n, double S) {
    double P = 0.0;
    for (int t = 0; t < n; ++t) {
        P += (double)v[t];
        if (2.0 * P >= S) return t;
    }
    return 0; /* S == 0 handled by the caller; unreachable otherwise */
}

void tto_line_f64(const float* v, int n, const float* wtab, int m_force, int mp_force,
                  double out[6], double absm[6], int32_t med[2]) {
    float* sv = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    double S = 0.0, Sp = 0.0;
    for (int t = 0; t < n; ++t) {
        sv[t] = sqrtf(v[t]);
        S += (double)v[t];
        Sp += (double)sv[t];
    }
    int m = (S > 0.0) ? median64(v, n, S) : 0;
    int mp = (Sp > 0.0) ? median64(sv, n, Sp) : 0;
    if (m_force >= 0) m = m_force;
    if (mp_force >= 0) mp = mp_force;
    double t1 = 0, t2 = 0, a3r = 0, a3i = 0, a4r = 0, a4i = 0, a5r = 0, a5i = 0;
    double m3 = 0, m4 = 0, m5 = 0;
    for (int t = m; t < n; ++t) {
        int r = t - m;
        double vv = (double)v[t];
        t1 += (double)r * vv;
        t2 += (double)r * (double)r * vv;
        a3r += (double)WT(wtab, r, 0) * vv; a3i += (double)WT(wtab, r, 1) * vv;
        a4r += (double)WT(wtab, r, 2) * vv; a4i += (double)WT(wtab, r, 3) * vv;
        m3 += (fabs((double)WT(wtab, r, 0)) + fabs((double)WT(wtab, r, 1))) * vv;
        m4 += (fabs((double)WT(wtab, r, 2)) + fabs((double)WT(wtab, r, 3))) * vv;
    }
    for (int t = mp; t < n; ++t) {
        int r = t - mp;
        double vv = (double)sv[t];
        a5r += (double)WT(wtab, r, 4) * vv; a5i += (double)WT(wtab, r, 5) * vv;
        m5 += (fabs((double)WT(wtab, r, 4)) + fabs((double)WT(wtab, r, 5))) * vv;
    }
    out[0] = S; out[1] = t1; out[2] = t2;
    out[3] = sqrt(a3r * a3r + a3i * a3i);
    out[4] = sqrt(a4r * a4r + a4i * a4i);
    out[5] = sqrt(a5r * a5r + a5i * a5i);
    if (absm) {
        absm[0] = S; absm[1] = t1; absm[2] = t2; absm[3] = m3; absm[4] = m4; absm[5] = m5;
    }
    if (med) { med[0] = m; med[1] = mp; }
    free(sv);
}

/* ----------------------------------------------- sequential fp32 (§2.3) */

static int median32_seq(const float* v, int n, float S) {
    float P = 0.0f;
    for (int t = 0; t < n; ++t) {
        P = P + v[t];
        if (P + P >= S) return t;
    }
    return 0;
}

static void line_seq32(const float* v, float* sv, int n, const float* wtab, float out[6], int32_t med[2]) {
    float S = 0.0f, Sp = 0.0f;
    for (int t = 0; t < n; ++t) {
        sv[t] = sqrtf(v[t]);
        S = S + v[t];
        Sp = Sp + sv[t];
    }
    int m = median32_seq(v, n, S);
    int mp = median32_seq(sv, n, Sp);
    float a1 = 0, a2 = 0, a3r = 0, a3i = 0, a4r = 0, a4i = 0, a5r = 0, a5i = 0;
    for (int t = m; t < n; ++t) {
        int r = t - m;
        float rf = (float)r, r2 = rf * rf, vv = v[t];
        a1 = fmaf(rf, vv, a1);
        a2 = fmaf(r2, vv, a2);
        a3r = fmaf(WT(wtab, r, 0), vv, a3r); a3i = fmaf(WT(wtab, r, 1), vv, a3i);
        a4r = fmaf(WT(wtab, r, 2), vv, a4r); a4i = fmaf(WT(wtab, r, 3), vv, a4i);
    }
    for (int t = mp; t < n; ++t) {
        int r = t - mp;
        float vv = sv[t];
        a5r = fmaf(WT(wtab, r, 4), vv, a5r); a5i = fmaf(WT(wtab, r, 5), vv, a5i);
    }
    out[0] = S; out[1] = a1; out[2] = a2;
    out[3] = sqrtf(fmaf(a3r, a3r, a3i * a3i));
    out[4] = sqrtf(fmaf(a4r, a4r, a4i * a4i));
    out[5] = sqrtf(fmaf(a5r, a5r, a5i * a5i));
    med[0] = m; med[1] = mp;
}

/* ------------------------------------------- B200 schedule replay (§3.2) */

/* Warp butterfly: x_l <- x_l + x_{l^off}, off = 16..1 (commutative, so every
 * lane ends with the same value). */
/* The kernel's reduction schedule is parameterised by NS, the slots (lanes)
 * per line: LG = min(NS, 32) lanes form one warp or sub-warp segment, and
 * NS / LG such groups (warps) share a line.  n <= 1024 uses one segment of 8,
 * 16 or 32 lanes; larger n uses NS = 32W. */

/* Butterfly over LG lanes: x_l <- x_l + x_{l^off}, off = LG/2..1 (commutative,
 * so every lane ends with the same value). */
static float warp_butterfly(float* x, int LG) {
    for (int off = LG / 2; off >= 1; off >>= 1) {
        float y[32];
        for (int l = 0; l < LG; ++l) y[l] = x[l] + x[l ^ off];
        memcpy(x, y, sizeof(float) * (size_t)LG);
    }
    return x[0];
}

/* Kogge-Stone inclusive scan over LG lanes: x_l <- x_{l-d} + x_l for l >= d. */
static void warp_scan(float* x, int LG) {
    for (int d = 1; d < LG; d <<= 1) {
        float y[32];
        for (int l = 0; l < LG; ++l) y[l] = (l >= d) ? x[l - d] + x[l] : x[l];
        memcpy(x, y, sizeof(float) * (size_t)LG);
    }
}

static int lanes_of(int NS) { return NS < 32 ? NS : 32; }

/* Slot-strided sum over [0,len) with stride NS, butterfly per group,
 * sequential over groups (kernel pass 1 / pass 2 reduction order). */
static float replay_strided_sum(const float* v, int len, int NS) {
    const int LG = lanes_of(NS);
    float total = 0.0f;
    for (int w = 0; w < NS / LG; ++w) {
        float x[32];
        for (int l = 0; l < LG; ++l) {
            float acc = 0.0f;
            for (int t = LG * w + l; t < len; t += NS) acc = acc + v[t];
            x[l] = acc;
        }
        total = total + warp_butterfly(x, LG);
    }
    return total;
}

/* Cooperative rescan of the crossing chunk (kernel: one group of LG lanes,
 * LG elements per block, Kogge-Stone scan per block, ballot). */
static int replay_rescan(const float* u, int n, int start, int K, float exc, float S, int LG) {
    int len = n - start;
    if (len > K) len = K;
    if (LG < 32 && (K == 4 * LG || K == 2 * LG)) {
        /* sub-warp segments: lane q holds E = K/LG consecutive elements, sequential
         * in-lane prefix l_e, Kogge-Stone over the lane totals, P = exc + (X_q + l_e)
         * (kernel rescan_lanes) */
        const int E = K / LG;
        float l[32][4], T[32];
        for (int q = 0; q < LG; ++q) {
            for (int e = 0; e < E; ++e) {
                const int j = q * E + e;
                const float x = (j < len) ? u[start + j] : 0.0f;
                l[q][e] = e == 0 ? x : l[q][e - 1] + x;
            }
            T[q] = l[q][E - 1];
        }
        warp_scan(T, LG);
        for (int q = 0; q < LG; ++q) {
            const float X = q == 0 ? 0.0f : T[q - 1];
            for (int e = 0; e < E; ++e) {
                const int j = q * E + e;
                if (j >= len) continue;
                const float P = exc + (X + l[q][e]);
                if (P + P >= S) return start + j;
            }
        }
        return len > 0 ? start + len - 1 : n - 1;
    }
    float C = 0.0f;
    for (int b = 0; b * LG < len; ++b) {
        float x[32];
        for (int j = 0; j < LG; ++j) x[j] = (b * LG + j < len) ? u[start + b * LG + j] : 0.0f;
        warp_scan(x, LG);
        for (int j = 0; j < LG && b * LG + j < len; ++j) {
            float P = exc + (C + x[j]);
            if (P + P >= S) return start + b * LG + j;
        }
        C = C + x[LG - 1];
    }
    return len > 0 ? start + len - 1 : n - 1;
}

/* Chunk sum rule of the kernel: balanced pairwise tree
 * (left + right) over a full power-of-two chunk, else sequential. */
static float tree_sum(const float* u, int K) {
    if (K == 1) return u[0];
    const float l = tree_sum(u, K / 2);
    const float r = tree_sum(u + K / 2, K / 2);
    return l + r;
}

static float chunk_sum(const float* u, int n, int start, int K) {
    int len = n - start;
    if (len > K) len = K;
    if (len <= 0) return 0.0f;
    if (len == K && (K & (K - 1)) == 0) return tree_sum(u + start, K);
    float acc = 0.0f;
    for (int t = start; t < start + len; ++t) acc = acc + u[t];
    return acc;
}

/* Median chunk length of the kernel (tt_kernels.cu chunk_len): ceil(n/NS),
 * an even K that is not a power of two rounded up to one; trailing slots may
 * own short or empty chunks. */
static int chunk_len(int n, int NS) {
    const int K = (n + NS - 1) / NS;
    if ((K & 1) || (K & (K - 1)) == 0) return K;
    int p = 1;
    while (p < K) p <<= 1;
    return p;
}

/* Weighted median of u under the kernel's schedule. */
static int replay_median(const float* u, int n, float S, int NS) {
    const int LG = lanes_of(NS);
    const int K = chunk_len(n, NS);
    float E = 0.0f;
    for (int w = 0; w < NS / LG; ++w) {
        float c[32], inc[32];
        for (int l = 0; l < LG; ++l) {
            c[l] = chunk_sum(u, n, (LG * w + l) * K, K);
            inc[l] = c[l];
        }
        warp_scan(inc, LG);
        for (int l = 0; l < LG; ++l) {
            float e = (l == 0) ? 0.0f : inc[l - 1];
            float exc = E + e;
            float pend = exc + c[l];
            if (pend + pend >= S) return replay_rescan(u, n, (LG * w + l) * K, K, exc, S, LG);
        }
        E = E + inc[LG - 1];
    }
    return 0;
}

/* Medians + pass 2 for one line direction u (su = sqrt u) with the line's
 * S, S' (shared by both directions of a mirrored pair). */
static void replay_emit(const float* u, const float* su, int n, const float* wtab, int NS, float S, float Sp,
                        float out[6], int32_t med[2]) {
    const int LG = lanes_of(NS);
    int m = replay_median(u, n, S, NS);
    int mp = replay_median(su, n, Sp, NS);
    const int R = n - m, Rp = n - mp, Rmax = R > Rp ? R : Rp;
    float tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int w = 0; w < NS / LG; ++w) {
        float x[8][32];
        for (int l = 0; l < LG; ++l) {
            float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int r = LG * w + l; r < Rmax; r += NS) {
                float rf = (float)r, r2 = rf * rf;
                float vv = (r < R) ? u[m + r] : 0.0f;
                float ss = (r < Rp) ? su[mp + r] : 0.0f;
                a[0] = fmaf(rf, vv, a[0]);
                a[1] = fmaf(r2, vv, a[1]);
                a[2] = fmaf(WT(wtab, r, 0), vv, a[2]);
                a[3] = fmaf(WT(wtab, r, 1), vv, a[3]);
                a[4] = fmaf(WT(wtab, r, 2), vv, a[4]);
                a[5] = fmaf(WT(wtab, r, 3), vv, a[5]);
                a[6] = fmaf(WT(wtab, r, 4), ss, a[6]);
                a[7] = fmaf(WT(wtab, r, 5), ss, a[7]);
            }
            for (int j = 0; j < 8; ++j) x[j][l] = a[j];
        }
        for (int j = 0; j < 8; ++j) tot[j] = tot[j] + warp_butterfly(x[j], LG);
    }
    out[0] = S;
    out[1] = tot[0];
    out[2] = tot[1];
    out[3] = sqrtf(fmaf(tot[2], tot[2], tot[3] * tot[3]));
    out[4] = sqrtf(fmaf(tot[4], tot[4], tot[5] * tot[5]));
    out[5] = sqrtf(fmaf(tot[6], tot[6], tot[7] * tot[7]));
    med[0] = m;
    med[1] = mp;
}

static int mirrored(const float* ctab, const float* stab, int a, int ap) {
    float mc = -ctab[a], ms = -stab[a];
    return memcmp(&mc, &ctab[ap], 4) == 0 && memcmp(&ms, &stab[ap], 4) == 0;
}

static void put(float* out, int32_t* med, int F, int n, int row, int col, const float o[6], const int32_t md[2]) {
    for (int f = 0; f < F; ++f) out[((size_t)row * F + f) * n + col] = o[f];
    if (med && F == TTO_NF) {
        med[((size_t)row * 2 + 0) * n + col] = md[0];
        med[((size_t)row * 2 + 1) * n + col] = md[1];
    }
}

/* One launch unit of the kernel: line (a0+i, p) and, with pairing, its
 * partner angle a0+i+pair_stride (the mirrored line n-1-p of the same
 * samples when the tables are exactly mirrored, else sampled separately). */
static void replay_unit(const float* img, int n, int a0, int units, int pair_stride, const float* ctab,
                        const float* stab, const float* wtab, int full, int NS, int i, int p, float* v, float* sv,
                        float* rv, float* rsv, float* out, int32_t* med) {
    const int F = full ? TTO_NF : 1;
    const int nlines = (pair_stride > 0) ? 2 : 1;
    const int mir = (pair_stride > 0) && mirrored(ctab, stab, a0 + i, a0 + i + pair_stride);
    for (int li = 0; li < (mir ? 1 : nlines); ++li) {
        const int a = a0 + i + li * pair_stride;
        if (n >= 2) tto_line_samples(img, n, ctab[a], stab[a], p, v);
        else for (int t = 0; t < n; ++t) v[t] = 0.0f;
        for (int t = 0; t < n; ++t) sv[t] = sqrtf(v[t]);
        const float S = replay_strided_sum(v, n, NS);
        const float Sp = replay_strided_sum(sv, n, NS);
        float o[6] = {S, 0, 0, 0, 0, 0};
        int32_t md[2] = {0, 0};
        if (full) replay_emit(v, sv, n, wtab, NS, S, Sp, o, md);
        put(out, med, F, n, i + li * units, p, o, md);
        if (mir) {
            for (int t = 0; t < n; ++t) {
                rv[t] = v[n - 1 - t];
                rsv[t] = sv[n - 1 - t];
            }
            float o2[6] = {S, 0, 0, 0, 0, 0};
            int32_t md2[2] = {0, 0};
            if (full) replay_emit(rv, rsv, n, wtab, NS, S, Sp, o2, md2);
            put(out, med, F, n, i + units, n - 1 - p, o2, md2);
        }
    }
}

void tto_replay_launch(const float* img, int n, int a0, int units, int pair_stride, const float* ctab,
                       const float* stab, const float* wtab, int full, int NS, float* out, int32_t* med,
                       int nthreads) {
    if (NS <= 0) NS = tto_schedule_slots(n, full);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const long total = (long)units * n;
#pragma omp parallel
    {
        float* buf = (float*)malloc(sizeof(float) * 4 * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 64)
        for (long L = 0; L < total; ++L)
            replay_unit(img, n, a0, units, pair_stride, ctab, stab, wtab, full, NS, (int)(L / n), (int)(L % n), buf,
                        buf + n, buf + 2 * (size_t)n, buf + 3 * (size_t)n, out, med);
        free(buf);
    }
}

/* Replay of selected units of one launch (large configurations whose full
 * replay is too slow on the host): unit (a0 + ui[k], p[k]) with the launch's
 * pairing, outputs out[k][2][F] (line (a0+ui, p), then its partner line:
 * (a0+ui+pair_stride, n-1-p) when mirrored, (a0+ui+pair_stride, p) otherwise)
 * and med[k][2][2].  Same arithmetic as tto_replay_launch. */
void tto_replay_units(const float* img, int n, int a0, int pair_stride, const float* ctab, const float* stab,
                      const float* wtab, int full, int NS, int count, const int32_t* ui, const int32_t* pl,
                      float* out, int32_t* med, int nthreads) {
    if (NS <= 0) NS = tto_schedule_slots(n, full);
    const int F = full ? TTO_NF : 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        float* buf = (float*)malloc(sizeof(float) * 4 * (size_t)(n > 0 ? n : 1));
        float* o = (float*)calloc((size_t)2 * F * (n > 0 ? n : 1), sizeof(float));
        int32_t* m = (int32_t*)calloc((size_t)2 * 2 * (n > 0 ? n : 1), sizeof(int32_t));
#pragma omp for schedule(dynamic, 4)
        for (int k = 0; k < count; ++k) {
            const int a = a0 + ui[k], p = pl[k];
            replay_unit(img, n, a, 1, pair_stride, ctab, stab, wtab, full, NS, 0, p, buf, buf + n,
                        buf + 2 * (size_t)n, buf + 3 * (size_t)n, o, full ? m : NULL);
            const int mir = pair_stride > 0 && mirrored(ctab, stab, a, a + pair_stride);
            const int cols[2] = {p, mir ? n - 1 - p : p};
            for (int li = 0; li < 2; ++li)
                for (int f = 0; f < F; ++f) {
                    out[((size_t)k * 2 + li) * F + f] = (li == 1 && pair_stride <= 0) ? 0.0f
                                                        : o[((size_t)li * F + f) * n + cols[li]];
                    if (med && full && f < 2)
                        med[((size_t)k * 2 + li) * 2 + f] = (li == 1 && pair_stride <= 0) ? 0
                                                            : m[((size_t)li * 2 + f) * n + cols[li]];
                }
        }
        free(buf);
        free(o);
        free(m);
    }
}

/* The structure the native trace_t05 / radon launcher uses for a launch of
 * a_count angles from a0: pairs (a0+i, a0+i+a_count/2) when a_count is even. */
void tto_launch_structure(int a_count, int* units, int* pair_stride) {
    if (a_count >= 2 && a_count % 2 == 0) {
        *units = a_count / 2;
        *pair_stride = a_count / 2;
    } else {
        *units = a_count;
        *pair_stride = 0;
    }
}

/* ------------------------------------------------------------- transform */

void tto_transform(const float* img, int n, int a0, int a_count, int a_total, const float* ctab,
                   const float* stab, const float* wtab, int full, int mode, int W, float* out, int32_t* med,
                   double* out64, double* absm, int nthreads) {
    (void)a_total;
    const int F = full ? TTO_NF : 1;
    if (W <= 0) W = tto_schedule_slots(n, full);
    if (mode == TTO_REPLAY) {
        int units, stride;
        tto_launch_structure(a_count, &units, &stride);
        tto_replay_launch(img, n, a0, units, stride, ctab, stab, wtab, full, W, out, med, nthreads);
        return;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const long lines = (long)a_count * n;
#pragma omp parallel
    {
        float* v = (float*)malloc(sizeof(float) * (size_t)n);
        float* sv = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 64)
        for (long L = 0; L < lines; ++L) {
            const int ai = (int)(L / n), p = (int)(L % n), a = a0 + ai;
            tto_line_samples(img, n, ctab[a], stab[a], p, v);
            float o32[6] = {0, 0, 0, 0, 0, 0};
            int32_t md[2] = {0, 0};
            if (mode == TTO_F64) {
                double o64[6], am[6];
                if (full) {
                    tto_line_f64(v, n, wtab, -1, -1, o64, am, md);
                } else {
                    double S = 0.0;
                    for (int t = 0; t < n; ++t) S += (double)v[t];
                    o64[0] = S;
                    am[0] = S;
                }
                for (int f = 0; f < F; ++f) {
                    o32[f] = (float)o64[f];
                    if (out64) out64[((size_t)ai * F + f) * n + p] = o64[f];
                    if (absm) absm[((size_t)ai * F + f) * n + p] = am[f];
                }
            } else if (mode == TTO_SEQ32) {
                if (full) {
                    line_seq32(v, sv, n, wtab, o32, md);
                } else {
                    float S = 0.0f;
                    for (int t = 0; t < n; ++t) S = S + v[t];
                    o32[0] = S;
                }
            } else {
                /* REPLAY is dispatched before this loop (launch-unit structure) */
            }
            for (int f = 0; f < F; ++f) out[((size_t)ai * F + f) * n + p] = o32[f];
            if (med && full) {
                med[((size_t)ai * 2 + 0) * n + p] = md[0];
                med[((size_t)ai * 2 + 1) * n + p] = md[1];
            }
        }
        free(v);
        free(sv);
    }
}

/* ----------------------------------------------- P-functionals (§2.7) */

void tto_circus(const float* sino, int n, int rows, float* circ, double* circ64, int32_t* med, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        float* d = (float*)malloc(sizeof(float) * (size_t)(n > 1 ? n : 1));
#pragma omp for schedule(dynamic, 16)
        for (int row = 0; row < rows; ++row) {
            const float* s = sino + (size_t)row * n;
            for (int p = 0; p + 1 < n; ++p) d[p] = fabsf(s[p + 1] - s[p]);
            const float S = replay_strided_sum(s, n, 32);
            const float P1 = replay_strided_sum(d, n - 1 > 0 ? n - 1 : 0, 32);
            const int m = replay_median(s, n, S, 32);
            float mx = 0.0f;
            for (int p = 0; p < n; ++p) mx = fmaxf(mx, s[p]);
            if (circ) {
                circ[(size_t)row * 3 + 0] = P1;
                circ[(size_t)row * 3 + 1] = n > 0 ? s[m] : 0.0f;
                circ[(size_t)row * 3 + 2] = mx;
            }
            if (med) med[row] = m;
            if (circ64) {
                double tv = 0.0, tot = 0.0, P = 0.0;
                for (int p = 0; p + 1 < n; ++p) tv += fabs((double)s[p + 1] - (double)s[p]);
                for (int p = 0; p < n; ++p) tot += (double)s[p];
                int m64 = 0;
                if (tot > 0.0)
                    for (int p = 0; p < n; ++p) {
                        P += (double)s[p];
                        if (2.0 * P >= tot) { m64 = p; break; }
                    }
                circ64[(size_t)row * 3 + 0] = tv;
                circ64[(size_t)row * 3 + 1] = n > 0 ? (double)s[m64] : 0.0;
                circ64[(size_t)row * 3 + 2] = (double)mx;
            }
        }
        free(d);
    }
}

/* --------------------------------------------------------------- checker */
static int is_eps_median(const float* v, int n, int m, double eps);

/* Is m an eps-median of v (f64 prefix)?  spec §2.5 */
int tto_is_eps_median(const float* v, int n, int m, double eps) { return is_eps_median(v, n, m, eps); }

static int is_eps_median(const float* v, int n, int m, double eps) {
    if (m < 0 || m >= n) return 0;
    double S = 0.0;
    for (int t = 0; t < n; ++t) S += (double)v[t];
    if (S == 0.0) return m == 0;
    double P = 0.0, Pprev = 0.0;
    for (int t = 0; t <= m; ++t) {
        Pprev = P;
        P += (double)v[t];
    }
    int reaches = 2.0 * P >= S * (1.0 - eps);
    int not_before = (m == 0) || (2.0 * Pprev < S * (1.0 + eps));
    return reaches && not_before;
}

/* One line (a, p) against the f64 truth: gpu values g[f] (F of them), medians gm[2]
 * (NULL: not checked).  Adds to the counters; returns the worst error ratio. */
static double check_line(const float* img, int n, float c, float s_, int p, const float* wtab, int full,
                         const float* g, int gstride, const int32_t* gm, int mstride, double rtol, double atol_c,
                         double eps, float* v, float* sv, long* fails, long* ties, long* medbad) {
    const int F = full ? TTO_NF : 1;
    tto_line_samples(img, n, c, s_, p, v);
    double o64[6], am[6];
    int32_t md[2] = {0, 0};
    if (full) {
        tto_line_f64(v, n, wtab, -1, -1, o64, am, md);
        if (gm) {
            const int m0 = gm[0], m1 = gm[mstride];
            int ok_m = (m0 == md[0]), ok_mp = (m1 == md[1]);
            if (!ok_m || !ok_mp) {
                for (int t = 0; t < n; ++t) sv[t] = sqrtf(v[t]);
                if (!ok_m) ok_m = is_eps_median(v, n, m0, eps);
                if (!ok_mp) ok_mp = is_eps_median(sv, n, m1, eps);
                if (ok_m && ok_mp) {
                    ++*ties;
                    tto_line_f64(v, n, wtab, m0, m1, o64, am, md);
                } else {
                    ++*medbad;
                    ++*fails;
                    return 1e300;
                }
            }
        }
    } else {
        double S = 0.0;
        for (int t = 0; t < n; ++t) S += (double)v[t];
        o64[0] = S;
        am[0] = S;
    }
    double worst = 0.0;
    for (int f = 0; f < F; ++f) {
        const double gv = (double)g[(size_t)f * gstride];
        const double tol = rtol * fabs(o64[f]) + atol_c * am[f] + 1e-30;
        const double e = fabs(gv - o64[f]) / tol;
        if (!(e <= 1.0)) ++*fails; /* NaN fails too */
        if (e > worst || e != e) worst = (e != e) ? 1e300 : e;
    }
    return worst;
}

static double chain_of(int n, int W, double chain) {
    const int NS = W > 0 ? W : tto_schedule_slots(n, 1);
    const int K = (n + NS - 1) / NS;
    /* fp32 chain length of the GPU schedule: slot partial + butterfly + groups
     * (callers checking a sequential fp32 result pass chain = n) */
    return chain > 0.0 ? chain : (double)K + 5.0 + (double)(NS / 32 + 1) + 4.0;
}

long tto_check(const float* img, int n, int a0, int a_count, int a_total, const float* ctab, const float* stab,
               const float* wtab, int full, const float* gpu_out, const int32_t* gpu_med, double rtol, int W,
               double chain, double* stats, int nthreads) {
    (void)a_total;
    const int F = full ? TTO_NF : 1;
    chain = chain_of(n, W, chain);
    const double u = 1.0 / 16777216.0;
    const double atol_c = 2.0 * chain * u;
    const double eps = 2.0 * chain * u; /* median tie window */
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const long lines = (long)a_count * n;
    long fails = 0, ties = 0, medbad = 0;
    double worst = 0.0;
#pragma omp parallel reduction(+ : fails, ties, medbad) reduction(max : worst)
    {
        float* v = (float*)malloc(sizeof(float) * (size_t)n);
        float* sv = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 64)
        for (long L = 0; L < lines; ++L) {
            const int ai = (int)(L / n), p = (int)(L % n), a = a0 + ai;
            const double e = check_line(img, n, ctab[a], stab[a], p, wtab, full, gpu_out + (size_t)ai * F * n + p, n,
                                        gpu_med ? gpu_med + (size_t)ai * 2 * n + p : NULL, n, rtol, atol_c, eps, v, sv,
                                        &fails, &ties, &medbad);
            if (e > worst) worst = e;
        }
        free(v);
        free(sv);
    }
    if (stats) {
        stats[0] = worst;
        stats[1] = (double)ties;
        stats[2] = (double)medbad;
        stats[3] = (double)lines;
    }
    return fails;
}

long tto_check_lines(const float* img, int n, const float* ctab, const float* stab, const float* wtab, int full,
                     int count, const int32_t* a_list, const int32_t* p_list, const float* gpu_out,
                     const int32_t* gpu_med, double rtol, int W, double chain, double* stats, int nthreads) {
    const int F = full ? TTO_NF : 1;
    chain = chain_of(n, W, chain);
    const double u = 1.0 / 16777216.0;
    const double atol_c = 2.0 * chain * u, eps = 2.0 * chain * u;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    long fails = 0, ties = 0, medbad = 0;
    double worst = 0.0;
#pragma omp parallel reduction(+ : fails, ties, medbad) reduction(max : worst)
    {
        float* v = (float*)malloc(sizeof(float) * (size_t)n);
        float* sv = (float*)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
        for (int k = 0; k < count; ++k) {
            const int a = a_list[k];
            const double e = check_line(img, n, ctab[a], stab[a], p_list[k], wtab, full, gpu_out + (size_t)k * F, 1,
                                        gpu_med ? gpu_med + (size_t)k * 2 : NULL, 1, rtol, atol_c, eps, v, sv, &fails,
                                        &ties, &medbad);
            if (e > worst) worst = e;
        }
        free(v);
        free(sv);
    }
    if (stats) {
        stats[0] = worst;
        stats[1] = (double)ties;
        stats[2] = (double)medbad;
        stats[3] = (double)count;
    }
    return fails;
}

/* ---------------------------------------------------- orthonormal frame */
/* the h x w image resampled bilinearly to s x s (s = ceil(A / sqrt 2)), centred in
 * an A x A frame; src = (dst + 0.5) * (w / s) - 0.5 clamped to [0, w-1], the sampler's bilinear form.
 * Restates tt_kernels.cu orthonormal_kernel. */
int tto_orthonormal_side(int angles) { return angles < 1 ? 0 : (int)ceil(angles / sqrt(2.0)); }

void tto_orthonormal(const float* img, int h, int w, int A, float* out) {
    const int s = tto_orthonormal_side(A), off = (A - s) / 2;
    const float sx = (float)w / (float)s, sy = (float)h / (float)s;
    for (int yy = 0; yy < A; ++yy)
        for (int xx = 0; xx < A; ++xx) {
            const int y = yy - off, x = xx - off;
            float v = 0.0f;
            if (x >= 0 && x < s && y >= 0 && y < s) {
                float fx = ((float)x + 0.5f) * sx - 0.5f;
                float fy = ((float)y + 0.5f) * sy - 0.5f;
                fx = fminf(fmaxf(fx, 0.0f), (float)(w - 1));
                fy = fminf(fmaxf(fy, 0.0f), (float)(h - 1));
                const int x0 = (int)fx, y0 = (int)fy;
                const int x1 = x0 + 1 < w ? x0 + 1 : w - 1, y1 = y0 + 1 < h ? y0 + 1 : h - 1;
                const float ax = fx - (float)x0, ay = fy - (float)y0;
                const float i00 = img[(size_t)y0 * w + x0], i01 = img[(size_t)y0 * w + x1];
                const float i10 = img[(size_t)y1 * w + x0], i11 = img[(size_t)y1 * w + x1];
                const float top = fmaf(ax, i01 - i00, i00);
                const float bot = fmaf(ax, i11 - i10, i10);
                v = fmaf(ay, bot - top, top);
            }
            out[(size_t)yy * A + xx] = v;
        }
}
