// ntt_f64.cuh -- exact modular NTT butterflies on the FP64 pipe, for limbs with q < 2^50.
//
// Why: on B200 the 64-bit integer Shoup butterfly is IMAD-pipe bound (~20 IMAD per butterfly,
// measured 856 G butterflies/s on all SMs), while an exact FP64 butterfly needs ~11 FP64 ops
// (measured 1310 G/s even with conditional corrections; tools/mb_fp64.cu).  Every config-2 limb
// (50-bit q_i) and every 40-bit limb of configs 1, 3-5 qualifies; 60-bit moduli (the special prime,
// q_0 of configs 1, 3-5) keep the integer engine of ntt.cuh.  Results are the same residues: every
// FP64 step below is exact integer arithmetic (values are integers of magnitude < 2^53).
//
// Representation: a residue class v mod q is held as a double (an integer) of magnitude <= B q,
// signed ("centred lazy").  Primitives (q < 2^50, qinv = fl(1/q)); bounds for the worst case
// q -> 2^50 (smaller q only shrink the error terms):
//   red(v)          = v - rint(v qinv) q                    exact (one FMA); |red(v)| <= (0.5 + B 2^-52) q
//   mulred(a, w)    = a w - qt q with qt = rint(fl(fl(a w) qinv)), computed exactly as
//                     h = fl(a w); l = fma(a, w, -h) (= a w - h exactly); t = fma(-qt, q, h) + l
//                     the FMA result h - qt q is an integer of magnitude < 2^53 (exact) and l is an
//                     integer.  The quotient estimate errs by <= 0.5 + 2^-52 |h| / q and
//                     |l| <= 2^-53 |a w|, so |t| <= q/2 + 1.5 2^-52 |a w|.  Twiddles are stored
//                     centred (|W| <= q/2): |t| <= q/2 + 0.75 2^-52 |a| q, i.e. for |a| <= B q,
//                     q < 2^50: |t| <= (0.5 + 3/16 B) q.  (tests/test_f64_arith.py)
// Forward CT butterfly (X, Y) -> (X' + t, X' - t), t = mulred(Y, W), on a lazy schedule
// (full_stage): a "full" stage re-centres X' = red(X), B' = 1 + 3/16 B; the other stages add X
// unreduced, B' = 19/16 B + 1/2.  Full stages are u % 3 == 0 and the pass's last stage, so from
// any pass input B <= 3.3 (or any |v| <= 2^50, e.g. a lifted wider residue: stage 0 is full) the
// magnitudes stay <= 3.3 q < 2^51.8 and every pass output is <= 1.6 q
// (8 stages: 1.19, 1.91, 2.77 | 1.52, 2.30, 3.23 | 1.61, 1.30 from B = 1): 4 of 8 stages skip
// the 3-op re-centring of X (9.5 instead of 11 FP64 ops per butterfly on average).
// Inverse GS butterfly (X, Y) -> (red(X + Y), mulred(red(X - Y), W)):
//   |red(X - Y)| <= 0.5q (+eps)  =>  |t| <= 0.75 q; B_out <= 0.75 for any number of stages.
//   (Without re-centring the difference, B would grow by q/2 per stage: 16 stages could exceed
//   2^53 / q for q near 2^50.)
// Loads convert [0, q) uint64 -> double exactly (bit trick, x < 2^52); stores reduce fully:
//   r = red(v); r += q if r < 0 -> [0, q), then back to uint64.
#pragma once
#include <cstdint>
#include "ntt.cuh"

namespace hisa {

constexpr uint64_t F64_MAX_Q = 1ull << 50;

__device__ __forceinline__ double u2d(uint64_t x) {   // exact for x < 2^52
    return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), 4503599627370496.0);
}
__device__ __forceinline__ uint64_t d2u(double y) {   // y an integer in [0, 2^52)
    return (uint64_t)__double_as_longlong(__dadd_rn(y, 4503599627370496.0)) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double redd(double v, double q, double qinv) {
    return __fma_rn(-rint(__dmul_rn(v, qinv)), q, v);
}
__device__ __forceinline__ double mulred(double a, double w, double q, double qinv) {
    const double h = __dmul_rn(a, w);
    const double l = __fma_rn(a, w, -h);
    const double qt = rint(__dmul_rn(h, qinv));
    return __dadd_rn(__fma_rn(-qt, q, h), l);
}
// any centred-lazy value -> canonical residue in [0, q) as uint64
__device__ __forceinline__ uint64_t d_canon(double v, double q, double qinv) {
    double r = redd(v, q, qinv);
    r = r < 0.0 ? __dadd_rn(r, q) : r;
    r = r >= q ? __dsub_rn(r, q) : r;
    return d2u(r);
}

// any centred-lazy value -> a uint64 representative in (q/2, 3q/2) (no compares): r = red(v) has
// |r| <= (0.5 + eps) q, so r + q > 0; (r + q + 2^52) is exact (< 2^53) and its low 52 mantissa
// bits are r + q.  Used where any representative < 2q will do (the key inner product's 128-bit
// accumulation).
__device__ __forceinline__ uint64_t d_rep(double v, double q, double qinv, double q_plus_2p52) {
    const double r = redd(v, q, qinv);
    return (uint64_t)__double_as_longlong(__dadd_rn(r, q_plus_2p52)) & 0xFFFFFFFFFFFFFull;
}

// a forward-engine output (|v| <= 2q, the fixed point above) -> uint64 representative in [0, 4q]
// with one add: v + 2q + 2^52 is exact (< 2^53) and its low 52 bits are v + 2q.  For the 128-bit
// key inner-product accumulation (products < 4 q^2 < 2^102, sums of <= 64 of them < 2^108).
__device__ __forceinline__ uint64_t d_rep4(double v, double two_q_plus_2p52) {
    return (uint64_t)__double_as_longlong(__dadd_rn(v, two_q_plus_2p52)) & 0xFFFFFFFFFFFFFull;
}

// the lazy forward schedule: stage u of a pass re-centres X (a "full" butterfly) only when
// u % 3 == 0 or u is the pass's last stage; the other stages add X unreduced (header: bounds)
__host__ __device__ constexpr bool full_stage(int u, int log_m) { return u % 3 == 0 || u == log_m - 1; }
// column passes (whose outputs only feed a row pass, which starts with a full stage) may leave
// the last stage lazy: outputs <= 2.41 q instead of 1.6 q (tests/test_f64_arith.py)
__host__ __device__ constexpr bool full_stage_cols(int u) { return u % 3 == 0; }

// forward CT stages [s0, s0 + LOG_M) on doubles in smem; mirrors fwd_engine (ntt.cuh) with
// the FP64 butterfly; tw = doubles W = psi^brv(k) mod q
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void fwd_engine_f64(double* sm, double q, double qinv, const double* __restrict__ tw,
                                               int s0, uint32_t high, int g, int t) {
    using G = Geo<LOG_M, LOG_R>;
#pragma unroll
    for (int u0 = 0; u0 < LOG_M; u0 += LOG_R) {
        const int w = (LOG_M - u0) < LOG_R ? (LOG_M - u0) : LOG_R;
        const int lo_bit = LOG_M - u0 - w;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            double reg[G::R];
            int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) reg[e] = sm[G::addr(g, base | (e << lo_bit))];
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int u = u0 + uu;
                const int dist = 1 << (w - 1 - uu);
                const uint32_t tbase = (1u << (s0 + u)) + (high << u) + ((uint32_t)ohigh << uu);
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << uu)) break;
                    const double W = __ldg(&tw[tbase + k]);
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        const double X = full_stage(u, LOG_M) ? redd(reg[e], q, qinv) : reg[e];
                        const double T = mulred(reg[e + dist], W, q, qinv);
                        reg[e] = __dadd_rn(X, T);
                        reg[e + dist] = __dsub_rn(X, T);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) sm[G::addr(g, base | (e << lo_bit))] = reg[e];
        }
        __syncthreads();
    }
}

// the same forward stages for ONE row group (row pass, g == 0) whose 2^LOG_M - 1 twiddles were
// staged in shared memory: tws[(1 << u) + m] = psi^brv(2^(s0+u) + (row << u) + m), m < 2^u (the
// key-switch inner product reuses one row's twiddles for every digit)
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void fwd_engine_f64_rowtw(double* sm, double q, double qinv, const double* tws, int t) {
    using G = Geo<LOG_M, LOG_R>;
#pragma unroll
    for (int u0 = 0; u0 < LOG_M; u0 += LOG_R) {
        const int w = (LOG_M - u0) < LOG_R ? (LOG_M - u0) : LOG_R;
        const int lo_bit = LOG_M - u0 - w;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            double reg[G::R];
            int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) reg[e] = sm[G::addr(0, base | (e << lo_bit))];
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int u = u0 + uu;
                const int dist = 1 << (w - 1 - uu);
                const int tbase = (1 << u) + (ohigh << uu);
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << uu)) break;
                    const double W = tws[tbase + k];
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        const double X = full_stage(u, LOG_M) ? redd(reg[e], q, qinv) : reg[e];
                        const double T = mulred(reg[e + dist], W, q, qinv);
                        reg[e] = __dadd_rn(X, T);
                        reg[e + dist] = __dsub_rn(X, T);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) sm[G::addr(0, base | (e << lo_bit))] = reg[e];
        }
        __syncthreads();
    }
}

// two tiles of the same prime and row (two digits of the key-switch inner product) through the
// staged-twiddle engine together: twice the independent FP64 dependency chains per thread
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void fwd_engine_f64_rowtw2(double* sa, double* sb, double q, double qinv,
                                                      const double* tws, int t) {
    using G = Geo<LOG_M, LOG_R>;
#pragma unroll
    for (int u0 = 0; u0 < LOG_M; u0 += LOG_R) {
        const int w = (LOG_M - u0) < LOG_R ? (LOG_M - u0) : LOG_R;
        const int lo_bit = LOG_M - u0 - w;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            double ra[G::R], rb[G::R];
            int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) {
                    ra[e] = sa[G::addr(0, base | (e << lo_bit))];
                    rb[e] = sb[G::addr(0, base | (e << lo_bit))];
                }
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int u = u0 + uu;
                const int dist = 1 << (w - 1 - uu);
                const int tbase = (1 << u) + (ohigh << uu);
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << uu)) break;
                    const double W = tws[tbase + k];
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        const bool fs = full_stage(u, LOG_M);
                        const double Xa = fs ? redd(ra[e], q, qinv) : ra[e], Xb = fs ? redd(rb[e], q, qinv) : rb[e];
                        const double Ta = mulred(ra[e + dist], W, q, qinv), Tb = mulred(rb[e + dist], W, q, qinv);
                        ra[e] = __dadd_rn(Xa, Ta);
                        rb[e] = __dadd_rn(Xb, Tb);
                        ra[e + dist] = __dsub_rn(Xa, Ta);
                        rb[e + dist] = __dsub_rn(Xb, Tb);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) {
                    sa[G::addr(0, base | (e << lo_bit))] = ra[e];
                    sb[G::addr(0, base | (e << lo_bit))] = rb[e];
                }
        }
        __syncthreads();
    }
}

// inverse GS stages, mirrors inv_engine (ntt.cuh)
template <int LOG_M, int LOG_R>
__device__ __forceinline__ void inv_engine_f64(double* sm, double q, double qinv, const double* __restrict__ tw,
                                               int v0, int log_n, uint32_t high, int g, int t) {
    using G = Geo<LOG_M, LOG_R>;
#pragma unroll
    for (int b0 = 0; b0 < LOG_M; b0 += LOG_R) {
        const int w = (LOG_M - b0) < LOG_R ? (LOG_M - b0) : LOG_R;
        const int lo_bit = b0;
        const int per = G::R >> w;
#pragma unroll
        for (int x = 0; x < G::R; x++) {
            if (x >= per) break;
            const int o = t * per + x;
            const int olow = o & ((1 << lo_bit) - 1);
            const int ohigh = o >> lo_bit;
            double reg[G::R];
            const int base = (ohigh << (lo_bit + w)) | olow;
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) reg[e] = sm[G::addr(g, base | (e << lo_bit))];
#pragma unroll
            for (int uu = 0; uu < LOG_R; uu++) {
                if (uu >= w) break;
                const int bit = lo_bit + uu;
                const int v = v0 + bit;
                const int dist = 1 << uu;
                const uint32_t tbase = (1u << (log_n - v - 1)) + (high << (LOG_M - bit - 1)) +
                                       ((uint32_t)ohigh << (w - uu - 1));
#pragma unroll
                for (int k = 0; k < (1 << LOG_R); k++) {
                    if (k >= (1 << (w - uu - 1))) break;
                    const double W = __ldg(&tw[tbase + k]);
#pragma unroll
                    for (int e0 = 0; e0 < G::R; e0++) {
                        if (e0 >= dist) break;
                        const int e = k * 2 * dist + e0;
                        const double X = reg[e], Y = reg[e + dist];
                        reg[e] = redd(__dadd_rn(X, Y), q, qinv);
                        reg[e + dist] = mulred(redd(__dsub_rn(X, Y), q, qinv), W, q, qinv);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < G::R; e++)
                if (e < (1 << w)) sm[G::addr(g, base | (e << lo_bit))] = reg[e];
        }
        __syncthreads();
    }
}

}  // namespace hisa
