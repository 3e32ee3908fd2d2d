/*
 * tt_oracle.h — CPU restatement of the trace transform (TEST INFRASTRUCTURE).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1604_03410_b200/) has no dependency on this directory
 * and fails loudly when its CUDA library is missing.
 *
 * The algorithm is the trace transform of arXiv 1604.03410 §7
 * (/root/reference/PAPER.md:810-829).  The reference artifact (gridjit) has
 * NO code for it (/root/reference/SPEC.md:13 lists it OUT OF SCOPE), so the
 * exact semantics are frozen in DESIGN.md §2 ("the spec"), following
 * SURVEY.md Appendix A; the numeric conventions (binary32 RNE, no
 * contraction outside an explicit fma, float->int truncation) mirror the
 * reference emulator, /root/reference/proj/include/gridjit/emulator.hpp:5-20
 * and /root/reference/proj/docs/vptx-isa.md:69-79.
 *
 * Parity pinning: the spec's arithmetic (sampler + sequential fp32
 * functionals, mode TTO_SEQ32) is pinned bit-exactly against the reference's
 * own execution engine running the same algorithm as a gridjit DSL kernel
 * (oracle/ref_tier2.cpp -> oracle/_ref/tt_tier2, built from the reference's
 * headers, /root/reference/proj/include/gridjit/autolaunch.hpp:167).  The
 * definition of T1-T5 itself is not pinned by any reference code or golden
 * vector (none exists); see DESIGN.md §2.
 *
 * Modes
 *   TTO_F64     truth: fp32 sampler (bit-identical everywhere), f64
 *               accumulation and f64 median prefix.  Tolerance reference.
 *   TTO_SEQ32   plain sequential fp32 (what a thread-per-line kernel on the
 *               reference emulator computes).  Bit-exact vs oracle/_ref.
 *   TTO_REPLAY  replays the B200 kernel's exact reduction schedule (W warps
 *               per line, slot-strided partials, butterfly, chunked median
 *               prefix) in fp32.  Bit-exact vs the GPU.
 */
#ifndef TT_ORACLE_H
#define TT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
/* Orthonormal (square) sinogram input frame, DESIGN.md §2.8 (restates tt_orthonormal_device). */
int tto_orthonormal_side(int angles);
void tto_orthonormal(const float* img, int h, int w, int angles, float* out);

#endif

enum { TTO_F64 = 0, TTO_SEQ32 = 1, TTO_REPLAY = 2 };
enum { TTO_DISK = 0, TTO_PHANTOM = 1, TTO_SPARSE = 2 };
#define TTO_NF 6

/* Host tables (spec §2.1/§2.2): ctab/stab[A] = (float)cos/sin(2*pi*a/A) in
 * f64; wtab [n][8] = r, r^2, w3re, w3im, w4re, w4im, w5re, w5im (f64 -> f32). */
void tto_tables(int n, int a_total, float* ctab, float* stab, float* wtab);

/* Deterministic synthetic images (spec §2.4). */
void tto_synth(int kind, uint64_t seed, int n, float* img);

/* The fp32 sampler for one line (a given by its c, s): v[t], t in [0,n). */
void tto_line_samples(const float* img, int n, float c, float s, int p, float* v);

/* Slots (lanes) per line the B200 kernel uses for side n: the replay schedule
 * (8/16/32: one warp segment; 32W: W warps). */
int tto_schedule_slots(int n, int full);

/*
 * Whole transform over angles [a0, a0+a_count) of a_total.
 *   full=1: out[a][6][n] (T0..T5), med[a][2][n] (m, m') if non-NULL
 *   full=0: out[a][1][n] (T0 only)
 *   mode TTO_F64 also fills out64 (same layout, double) and absm (the
 *   condition numbers M_f of spec §2.5) when non-NULL.
 *   W is the replay schedule NS = slots per line (TTO_REPLAY only; <=0 -> tto_schedule_slots).
 *   nthreads <= 0 -> OpenMP default.
 */
void tto_transform(const float* img, int n, int a0, int a_count, int a_total,
                   const float* ctab, const float* stab, const float* wtab,
                   int full, int mode, int W, float* out, int32_t* med,
                   double* out64, double* absm, int nthreads);

/* Replay of one B200 launch: units (a0+i, p), i < units;
 * with pair_stride > 0 each unit also owns angle a0+i+pair_stride (rows
 * units+i), processed as the mirrored line n-1-p of the same samples when
 * ctab/stab are exactly mirrored, else sampled separately. */
void tto_replay_launch(const float* img, int n, int a0, int units, int pair_stride, const float* ctab,
                       const float* stab, const float* wtab, int full, int NS, float* out, int32_t* med,
                       int nthreads);

/* Replay of selected units (a0+ui[k], p[k]) of a launch with the given pairing:
 * out[k][2][F] = the unit's line and its partner line (zeros when unpaired),
 * med[k][2][2]; bit-identical to the same rows of tto_replay_launch. */
void tto_replay_units(const float* img, int n, int a0, int pair_stride, const float* ctab, const float* stab,
                      const float* wtab, int full, int NS, int count, const int32_t* ui, const int32_t* p,
                      float* out, int32_t* med, int nthreads);

/* Launch structure the native trace_t05/radon launcher uses for a_count
 * angles: pairs (i, i + a_count/2) when a_count is even. */
void tto_launch_structure(int a_count, int* units, int* pair_stride);

/* P-functionals of sinogram rows (spec §2.7): circ[row][3] = P1 (total
 * variation), P2 (value at the weighted median), P3 (max) under the kernel's
 * one-warp schedule (bit-exact replay); circ64 the f64 truth (P2 at the f64
 * median); med[row] the replayed median index.  Any output may be NULL. */
void tto_circus(const float* sino, int n, int rows, float* circ, double* circ64, int32_t* med, int nthreads);

/* 1 if m is an eps-median of v (f64 prefix), the tie rule of spec §2.5. */
int tto_is_eps_median(const float* v, int n, int m, double eps);

/* Per-line truth evaluated at forced medians (tie re-evaluation, §2.5).
 * m_force / mp_force < 0 -> use the f64 medians. */
void tto_line_f64(const float* v, int n, const float* wtab, int m_force, int mp_force,
                  double out[6], double absm[6], int32_t med[2]);

/*
 * Parity checker (spec §2.5) for a GPU result of the full transform.
 * Tolerance per value: rtol*|ref| + 2*chain*2^-24*M_f, where chain is the
 * longest fp32 accumulation chain of the checked schedule (<= 0: derived
 * from the GPU schedule W) and M_f the value's condition number.
 * Returns the number of failing values; fills stats:
 *   stats[0] = max over values of |g-r| / (rtol*|r| + atol)  (<=1 passes)
 *   stats[1] = number of median ties accepted (m != m_ref but eps-median)
 *   stats[2] = number of median mismatches rejected
 *   stats[3] = number of lines checked
 */
long tto_check(const float* img, int n, int a0, int a_count, int a_total,
               const float* ctab, const float* stab, const float* wtab, int full,
               const float* gpu_out, const int32_t* gpu_med, double rtol, int W, double chain,
               double* stats, int nthreads);

/* tto_check for an explicit list of lines (a_list[k], p_list[k]) with GPU values
 * gpu_out[k][F] and medians gpu_med[k][2] (may be NULL). */
long tto_check_lines(const float* img, int n, const float* ctab, const float* stab, const float* wtab, int full,
                     int count, const int32_t* a_list, const int32_t* p_list, const float* gpu_out,
                     const int32_t* gpu_med, double rtol, int W, double chain, double* stats, int nthreads);

#ifdef __cplusplus
}
/* Orthonormal (square) sinogram input frame, DESIGN.md §2.8 (restates tt_orthonormal_device). */
int tto_orthonormal_side(int angles);
void tto_orthonormal(const float* img, int h, int w, int angles, float* out);

#endif
/* Orthonormal (square) sinogram input frame, DESIGN.md §2.8 (restates tt_orthonormal_device). */
int tto_orthonormal_side(int angles);
void tto_orthonormal(const float* img, int h, int w, int angles, float* out);

#endif
