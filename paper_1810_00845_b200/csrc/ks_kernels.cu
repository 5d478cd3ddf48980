// ks_kernels.cu -- key-switch inner product fused with the forward-NTT row pass (K4, step a5).
//
// For output prime r (grid y = ri over q_0..q_l, p) and a tile of rows (grid x), loop over the
// digits j <= l: bring D_{j,r} for the tile on chip -- either the pass-1 output T1[j][ri] followed by
// the last log M2 CT stages in shared memory, or (r == q_j) the digit itself, which is already in
// the NTT domain -- then multiply with the key limbs (b and a) and accumulate in 128-bit
// registers (products < 2^122, at most 64 terms).  One Barrett reduction per output word.
// D never touches HBM in its NTT form; the key is streamed once per ciphertext.
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include "ntt_f64.cuh"
#include "launch.h"

namespace hisa {

// a key word of an FP64-engine limb: stored as the centred residue's exact double (internal key
// format, hisa.cu k_key_format), |K| <= q/2
__device__ __forceinline__ double kd(uint64_t raw) { return __longlong_as_double((long long)raw); }
// the same word as a uint64 representative in [0, q) for the integer MACs of k_ks_ip2
__device__ __forceinline__ uint64_t ku(uint64_t raw, double q) {
    const double d = kd(raw);
    return d2u(d < 0.0 ? __dadd_rn(d, q) : d);
}


// K4 for one row per CTA with two digits in flight (variant 30, FP64 output primes): the
// non-diagonal digits j != ri are processed in pairs -- both D tiles copied, both transformed by
// one interleaved engine call (fwd_engine_f64_rowtw2, twiddles staged once in shared memory),
// both multiplied into the same 128-bit accumulators -- then the diagonal digit (already in the
// NTT domain) is multiplied in.  Integer-engine primes (q >= 2^50) fall back to one digit at a time.
template <int LOG_M, int LOG_R, int MINB>
__global__ void __launch_bounds__((1 << LOG_M) / (1 << LOG_R), MINB) k_ks_ip2(KsJob job, Tables tb) {
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    uint64_t* sa = sm;
    uint64_t* sb = sm + G::STRIDE;
    double* tws = reinterpret_cast<double*>(sm + 2 * G::STRIDE);
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    // the special prime's CTAs (integer engine, slower) first, so they do not form the tail
    const int ri = job.ri_list[blockIdx.y];
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = blockIdx.x / nz;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const bool fp = (double)md.q < tb.f64_max_q;
    const double2 qd = fp ? tb.modd[mi] : make_double2(0, 0);
    const double tq52 = __dadd_rn(2.0 * qd.x, 4503599627370496.0);   // 2q + 2^52
    constexpr int NTHR = G::T;
    constexpr int EPT = G::R;
    U128 acc0[EPT], acc1[EPT];
#pragma unroll
    for (int k = 0; k < EPT; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    const int t = threadIdx.x;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)(ri < l1 ? ri : job.L) << log_n) + off0;
    if (fp) {
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - LOG_M;
        for (int idx = threadIdx.x + 1; idx < G::M; idx += NTHR) {
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            tws[idx] = twg[(1 << (s0 + u)) + (row0 << u) + m];
        }
    }
    auto copy_tile = [&](uint64_t* dst, int j) {
        const uint64_t* src = (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                                        : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            const unsigned s_ = (unsigned)__cvta_generic_to_shared(&dst[G::addr(0, i)]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_), "l"(src + i) : "memory");
        }
    };
    auto mac_tile = [&](const uint64_t* buf, int j, bool conv) {
        const uint64_t* kb = key_r + j * kstride_j;
        const uint64_t* ka = kb + kstride_p;
#pragma unroll
        for (int k = 0; k < EPT; k++) {
            const int i = threadIdx.x + k * NTHR;
            uint64_t D = buf[G::addr(0, i)];
            if (conv) D = d_rep4(__longlong_as_double((long long)D), tq52);   // in [0, 4q]
            const uint64_t Kb = __ldg(kb + i), Ka = __ldg(ka + i);
            mac128(acc0[k], D, fp ? ku(Kb, qd.x) : Kb);   // FP64 limbs: internal key format
            mac128(acc1[k], D, fp ? ku(Ka, qd.x) : Ka);
        }
    };
    // digits j != ri, in pairs
    int j = 0;
    auto next_nd = [&](int from) { return from == ri ? from + 1 : from; };
    j = next_nd(0);
    while (j < l1) {
        const int ja = j;
        int jb = next_nd(ja + 1);
        const bool two = fp && jb < l1;
        copy_tile(sa, ja);
        if (two) copy_tile(sb, jb);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (two) {
            fwd_engine_f64_rowtw2<LOG_M, LOG_R>(reinterpret_cast<double*>(sa), reinterpret_cast<double*>(sb), qd.x,
                                                qd.y, tws, t);
            mac_tile(sa, ja, true);
            mac_tile(sb, jb, true);
            j = next_nd(jb + 1);
        } else {
            if (fp)
                fwd_engine_f64_rowtw<LOG_M, LOG_R>(reinterpret_cast<double*>(sa), qd.x, qd.y, tws, t);
            else
                fwd_engine<LOG_M, LOG_R>(sa, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M,
                                         (uint32_t)row0, 0, t);
            mac_tile(sa, ja, fp);
            j = next_nd(ja + 1);
        }
        __syncthreads();
    }
    if (ri < l1) {   // the diagonal digit: D_{ri, q_ri} = d_ri, already in the NTT domain
        copy_tile(sa, ri);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        mac_tile(sa, ri, false);
    }
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
#pragma unroll
    for (int k = 0; k < EPT; k++) {
        const int i = threadIdx.x + k * NTHR;
        out0[i] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[i] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

// K4 for the integer-engine output primes at M = 256 (60-bit: the special prime, the 60-bit q_0 of
// configs 1, 3-5): one row per 64-thread CTA, the row's pass-1 words staged by cp.async, the last
// 8 CT stages with the integer (Shoup) engine, 128-bit lazy key MACs, one Barrett per output word.
// (The FP64 output primes run k_ks_ip6 below.)
#ifndef K5_MINB
#define K5_MINB 9     // k_ks_ip5 min CTAs / SM (64 threads)
#endif

template <int MINB>
__global__ void __launch_bounds__(64, MINB) k_ks_ip5(KsJob job, Tables tb) {
    constexpr int LOG_M = 8, LOG_R = 2;
    using G = Geo<LOG_M, LOG_R>;
    extern __shared__ uint64_t sm[];
    uint64_t* sa = sm;
    const int nz = job.nz;
    const int z = blockIdx.x % nz;
    const int ri = job.ri_list[blockIdx.y];
    const int l1 = job.l1;
    const int nri = l1 + 1;
    const int log_n = tb.log_n;
    const int row0 = blockIdx.x / nz;
    const long long off0 = (long long)row0 << LOG_M;
    const int mi = job.mod_map[ri];
    const Mod md = tb.mods[mi];
    const int t = threadIdx.x;
    const long long kstride_j = 2ll * (job.L + 1) << log_n;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const uint64_t* key_r = job.key + ((long long)(ri < l1 ? ri : job.L) << log_n) + off0;
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + off0;
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + off0;
    auto tile_src = [&](int j) -> const uint64_t* {
        return (j == ri) ? job.d[z] + ((long long)j << log_n) + off0
                         : job.t1[z] + (((long long)j * nri + ri) << log_n) + off0;
    };
    U128 acc0[4], acc1[4];
#pragma unroll
    for (int k = 0; k < 4; k++) { acc0[k] = U128{0, 0}; acc1[k] = U128{0, 0}; }
    for (int j = 0; j < l1 + 1; j++) {   // the non-diagonal digits, then the diagonal one (if ri < l1)
        if (j == l1 && ri >= l1) break;
        const int jj = j == l1 ? ri : j;
        if (j < l1 && j == ri) continue;
        const uint64_t* src = tile_src(jj);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = t + k * 64;
            const unsigned s_ = (unsigned)__cvta_generic_to_shared(&sa[G::addr(0, i)]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_), "l"(src + i) : "memory");
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        if (j < l1)
            fwd_engine<LOG_M, LOG_R>(sa, md.q, tb.fwd + ((long long)mi << log_n), log_n - LOG_M, (uint32_t)row0, 0, t);
        const uint64_t* kb = key_r + jj * kstride_j;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int i = t + k * 64;
            const uint64_t D = sa[G::addr(0, i)];
            mac128(acc0[k], D, __ldg(kb + i));
            mac128(acc1[k], D, __ldg(kb + kstride_p + i));
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        out0[t + k * 64] = barrett128(acc0[k].lo, acc0[k].hi, md);
        out1[t + k * 64] = barrett128(acc1[k].lo, acc1[k].hi, md);
    }
}

// ------------------------------------------------------------------------------------------
// K4 v6 (FP64 output primes, M = 256 rows: N = 2^15, 2^16).  ncu of k_ks_ip5 (profiles/
// r2_ncu_k4_v1.txt) showed the shared-memory data pipe, not the FP64 pipe, as the bound: 72 % LSU
// wavefronts against 35 % FP64, ~34 wavefronts per 32 element-digits (three radix-4 exchanges,
// row and key staging, 65 M bank-conflict wavefronts) and ~108 instructions per element-digit
// (the split 64-bit MACs alone ~30).  This kernel:
//  * runs each 256-point row as two radix-16 register phases with ONE exchange, 16 threads per
//    row (thread g holds elements 16a + g in phase 1, 16t + b in phase 2);
//  * accumulates the key inner product on the FP64 pipe: acc += mulred(D, K) with D the centred
//    phase-2 output (|D| <= 1.7 q, k4_full schedule) and K the key word, stored as its centred
//    residue's exact double (|K| <= q/2, internal key format): |mulred| <= q/2 + 1.5 2^-52 |D K|
//    <= 0.82 q, so eight products fit between re-centrings (|acc| < 7.1 q < 2^53): every step is
//    exact integer arithmetic, the result (one final canonical reduction) is the same residue as
//    the integer MAC's -- two doubles per output word instead of three 64-bit words, no 64-bit
//    multiplies;
//  * puts CG ciphertexts x RB rows (G = CG RB groups of 16 threads) in one CTA: the key rows are
//    staged once per row and shared by the CG ciphertexts;
//  * stages each step's rows and keys with cp.async one step ahead (double buffer); the key rows
//    are stored with the 16-byte chunks of every 128-byte line XOR-swizzled by the line index, so
//    the phase-2 pattern (thread t reads words 16t .. 16t+15 as 16-byte pairs) is conflict-free;
//    the exchange reuses the step's row buffer with the same swizzle; outputs leave through it
//    as coalesced 8-byte stores.
// Digit order: the l non-diagonal digits (pass-1 rows, two phases), then the diagonal digit d_ri
// (already in the NTT domain, canonical, staged swizzled, no NTT).
// ------------------------------------------------------------------------------------------
template <int CG, int RB>
struct Ip6 {
    static constexpr int G = CG * RB;            // 16-thread groups per CTA
    static constexpr int NT = 16 * G;
    static constexpr int STAGE_T1 = G * 256;     // words: one row per group
    static constexpr int STAGE_K = RB * 2 * 256; // b and a key rows per row
    static constexpr int STAGE = STAGE_T1 + STAGE_K;
    static constexpr size_t smem_bytes() { return (size_t)(256 * RB + 2 * STAGE) * 8; }
};

// K4 v6's row-pass schedule: X re-centred at stages 0, 4, 7 only (the round-1 engines: 0, 3, 6, 7).
// From a column-pass input |v| <= 2.41 q the magnitudes stay <= 4.23 q (< 2^52.1) and the output
// is <= 1.68 q, the MAC's operand bound (tests/test_f64_arith.py::test_k4_row_schedule).
__host__ __device__ constexpr bool k4_full(int u) { return u == 0 || u == 4 || u == 7; }

// word b of line t of a 256-word row in the pair-swizzled layout (lines of 16 words = 128 B)
__device__ __forceinline__ int swz(int t, int b) { return t * 16 + ((((b >> 1) ^ t) & 7) << 1) + (b & 1); }

template <int CG, int RB, int MINB>
__global__ void __launch_bounds__(16 * CG * RB, MINB) k_ks_ip6(KsJob job, Tables tb) {
    using P = Ip6<CG, RB>;
    extern __shared__ uint64_t sm[];
    double* tw_all = reinterpret_cast<double*>(sm);              // [RB][256] row twiddles (2^u + m)
    uint64_t* stage0 = sm + 256 * RB;
    const int l1 = job.l1, nri = l1 + 1, log_n = tb.log_n;
    const int ri = job.ri_list[blockIdx.y];
    const int nzb = job.nz / CG;                                 // ciphertext blocks
    const int zb = blockIdx.x % nzb;
    const int row_base = (blockIdx.x / nzb) * RB;
    const int tid = threadIdx.x;
    const int grp = tid >> 4, g = tid & 15;
    const int cz = grp % CG, rr = grp / CG;
    const int z = zb * CG + cz;
    const int row = row_base + rr;
    const int mi = job.mod_map[ri];
    const double2 qd = tb.modd[mi];
    const double q = qd.x, qinv = qd.y;
    const long long kstride_p = (long long)(job.L + 1) << log_n;
    const long long kstride_j = 2 * kstride_p;
    const uint64_t* key_ri = job.key + ((long long)(ri < l1 ? ri : job.L) << log_n);
    const int n_nd = l1 - 1;                                      // non-diagonal digits (ri < l1)
    const int nsteps = n_nd + 1;
    const double* tw = tw_all + rr * 256;

    // per-CTA source bases (hoisted out of the digit loop; the per-step offset is one add):
    // group k's pass-1 rows T1[zz][j][ri][row] and diagonal row d[zz][ri][row]
    const uint64_t* t1b[P::G];
    const uint64_t* db[P::G];
#pragma unroll
    for (int k = 0; k < P::G; k++) {
        const int zz = zb * CG + k % CG, rw = row_base + k / CG;
        t1b[k] = job.t1[zz] + ((long long)ri << log_n) + (rw << 8);
        db[k] = job.d[zz] + ((long long)ri << log_n) + (rw << 8);
    }
    const uint64_t* kb0 = key_ri + ((long long)row_base << 8);
    const long long t1_step = (long long)nri << log_n;
    // cp.async copies of step `st` into stage buffer `buf`
    auto issue = [&](int st, int buf) {
        uint64_t* base = stage0 + buf * P::STAGE;
        const bool diag = st == n_nd;
        const int j = diag ? ri : (st < ri ? st : st + 1);
        const long long joff = (long long)j * t1_step;
        // rows: group k's row (256 words = 128 chunks of 16 B); plain for pass-1 rows, swizzled for
        // the diagonal digit (read in the phase-2 pattern)
#pragma unroll
        for (int k = 0; k < P::G; k++) {
            for (int ch = tid; ch < 128; ch += P::NT) {
                const uint64_t* src = (diag ? db[k] : t1b[k] + joff) + ch * 2;
                const int line = ch >> 3, cc = ch & 7;
                const int dst = k * 256 + (diag ? line * 16 + ((cc ^ (line & 7)) << 1) : ch * 2);
                const unsigned sa = (unsigned)__cvta_generic_to_shared(base + dst);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
            }
        }
        // keys: per row, b and a (swizzled)
        uint64_t* kbase = base + P::STAGE_T1;
        const uint64_t* kj = kb0 + (long long)j * kstride_j;
        for (int c = tid; c < RB * 256; c += P::NT) {
            const int rk = c >> 8, h = (c >> 7) & 1, ch = c & 127;
            const uint64_t* src = kj + h * kstride_p + (rk << 8) + ch * 2;
            const int line = ch >> 3, cc = ch & 7;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(kbase + (rk * 2 + h) * 256 + line * 16 +
                                                                   ((cc ^ (line & 7)) << 1));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    issue(0, 0);
    {   // each row's twiddles: stage u (0..7 of the last 8 stages), group m -> tw[2^u + m]
        const double* twg = tb.fwd_d + ((long long)mi << log_n);
        const int s0 = log_n - 8;
        // phase 2 (u >= 4): thread g's k-th twiddle of stage u, m = g 2^(u-4) + k, is stored at
        // 2^u + 16 k + g, so the 16 threads of a row read 16 consecutive words (conflict-free)
        for (int i = tid; i < 256 * RB; i += P::NT) {
            const int rk = i >> 8, idx = i & 255;
            if (idx == 0) continue;
            const int u = 31 - __clz(idx), m = idx - (1 << u);
            const int pos = u < 4 ? idx : (1 << u) + ((m & ((1 << (u - 4)) - 1)) << 4) + (m >> (u - 4));
            tw_all[rk * 256 + pos] = twg[(1 << (s0 + u)) + ((row_base + rk) << u) + m];
        }
    }

    double accb[16], acca[16];
#pragma unroll
    for (int b = 0; b < 16; b++) { accb[b] = 0.0; acca[b] = 0.0; }

    for (int st = 0; st < nsteps; st++) {
        const int buf = st & 1;
        if (st + 1 < nsteps) {
            issue(st + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        uint64_t* base = stage0 + buf * P::STAGE;
        double* rowbuf = reinterpret_cast<double*>(base + grp * 256);
        const uint64_t* kb = base + P::STAGE_T1 + rr * 512;
        double r[16];
        if (st < n_nd) {
            // phase 1: elements 16a + g, stages u = 0..3 on a (twiddles uniform per row)
#pragma unroll
            for (int a = 0; a < 16; a++) r[a] = rowbuf[16 * a + g];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int dist = 8 >> u;
#pragma unroll
                for (int a = 0; a < 16; a++) {
                    if (a & dist) continue;
                    const double W = tw[(1 << u) + (a >> (4 - u))];
                    const double X = k4_full(u) ? redd(r[a], q, qinv) : r[a];
                    const double T = mulred(r[a + dist], W, q, qinv);
                    r[a] = __dadd_rn(X, T);
                    r[a + dist] = __dsub_rn(X, T);
                }
            }
            __syncwarp();
            // exchange in place (pair-swizzled): write (a, g), read line t = g
#pragma unroll
            for (int a = 0; a < 16; a++) rowbuf[swz(a, g)] = r[a];
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const double2 v = *reinterpret_cast<const double2*>(rowbuf + swz(g, 2 * c));
                r[2 * c] = v.x;
                r[2 * c + 1] = v.y;
            }
            // phase 2: elements 16t + b (t = g), stages u = 4..7 on b
#pragma unroll
            for (int u = 4; u < 8; u++) {
                const int dist = 8 >> (u - 4);
#pragma unroll
                for (int b = 0; b < 16; b++) {
                    if (b & dist) continue;
                    const double W = tw[(1 << u) + ((b >> (8 - u)) << 4) + g];
                    const double X = k4_full(u) ? redd(r[b], q, qinv) : r[b];
                    const double T = mulred(r[b + dist], W, q, qinv);
                    r[b] = __dadd_rn(X, T);
                    r[b + dist] = __dsub_rn(X, T);
                }
            }
        } else {
            // the diagonal digit d_ri: canonical NTT-domain words, staged swizzled
            const uint64_t* dv = reinterpret_cast<const uint64_t*>(rowbuf);
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(dv + swz(g, 2 * c));
                r[2 * c] = u2d(v.x);
                r[2 * c + 1] = u2d(v.y);
            }
        }
        // key inner product on the FP64 pipe (exact; see the header)
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const ulonglong2 vb = *reinterpret_cast<const ulonglong2*>(kb + swz(g, 2 * c));
            const ulonglong2 va = *reinterpret_cast<const ulonglong2*>(kb + 256 + swz(g, 2 * c));
            accb[2 * c] = __dadd_rn(accb[2 * c], mulred(r[2 * c], kd(vb.x), q, qinv));
            accb[2 * c + 1] = __dadd_rn(accb[2 * c + 1], mulred(r[2 * c + 1], kd(vb.y), q, qinv));
            acca[2 * c] = __dadd_rn(acca[2 * c], mulred(r[2 * c], kd(va.x), q, qinv));
            acca[2 * c + 1] = __dadd_rn(acca[2 * c + 1], mulred(r[2 * c + 1], kd(va.y), q, qinv));
        }
        if ((st & 7) == 7) {
#pragma unroll
            for (int b = 0; b < 16; b++) { accb[b] = redd(accb[b], q, qinv); acca[b] = redd(acca[b], q, qinv); }
        }
        __syncthreads();   // this buffer is refilled by the next step's issue
    }
    // outputs: canonical residues, transposed through the group's row buffer (free now) for
    // coalesced 8-byte stores
    uint64_t* obuf = stage0 + grp * 256;
    uint64_t* out0 = job.acc[z] + ((long long)ri << log_n) + (row << 8);
    uint64_t* out1 = job.acc[z] + ((long long)(nri + ri) << log_n) + (row << 8);
#pragma unroll
    for (int h = 0; h < 2; h++) {
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const double* acc = h ? acca : accb;
            *reinterpret_cast<ulonglong2*>(obuf + swz(g, 2 * c)) =
                make_ulonglong2(d_canon(acc[2 * c], q, qinv), d_canon(acc[2 * c + 1], q, qinv));
        }
        __syncwarp();
        uint64_t* o = h ? out1 : out0;
#pragma unroll
        for (int k = 0; k < 16; k++) o[16 * k + g] = obuf[swz(k, g)];
        __syncwarp();
    }
}

template <int CG, int RB, int MINB>
static cudaError_t ks_ip6_t(const KsJob& job, const Tables& tb, int nfp, cudaStream_t st) {
    using P = Ip6<CG, RB>;
    const int rows = 1 << (tb.log_n - 8);
    const size_t smem = P::smem_bytes();
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ks_ip6<CG, RB, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid((rows / RB) * (job.nz / CG), nfp, 1);
    k_ks_ip6<CG, RB, MINB><<<grid, P::NT, smem, st>>>(job, tb);
    return cudaGetLastError();
}

template <int MINB>
static cudaError_t ks_ip5_t(const KsJob& job, const Tables& tb, int nz, int nrows, cudaStream_t st) {
    const int rows = 1 << (tb.log_n - 8);
    const size_t smem = (size_t)Geo<8, 2>::STRIDE * sizeof(uint64_t);   // the row tile
    dim3 grid(rows * nz, nrows, 1);
    k_ks_ip5<MINB><<<grid, 64, smem, st>>>(job, tb);
    return cudaGetLastError();
}

template <int LOG_M, int LOG_R, int MINB>
static cudaError_t ks_ip2_t(const KsJob& job, const Tables& tb, int nz, cudaStream_t st) {
    using G = Geo<LOG_M, LOG_R>;
    const int rows = 1 << (tb.log_n - LOG_M);
    const size_t smem = (2 * (size_t)G::STRIDE + G::M) * sizeof(uint64_t);
    dim3 grid(rows * nz, job.l1 + 1, 1);
    k_ks_ip2<LOG_M, LOG_R, MINB><<<grid, G::T, smem, st>>>(job, tb);
    return cudaGetLastError();
}

#ifndef K6_MINB
#define K6_MINB 4      // 128 registers, no spills (5: spills)
#endif

// M = 256: the FP64 output primes run k_ks_ip6 (CG ciphertexts x RB rows per CTA: 8 x 1, 4 x 1,
// 2 x 2 or 1 x 4 by the largest of 8, 4, 2, 1 dividing nz), the integer-engine primes (60-bit: the special prime, q_0 of
// configs 1, 3-5) the integer path of k_ks_ip5, each as its own launch over its rows
static cudaError_t ks_ip_256(KsJob job, const Tables& tb, int nz, cudaStream_t st, const SideStream* side) {
    const int l2 = job.l1 + 1;
    int nfp = 0, nint = 0;
    uint8_t fp[MAXL], in[MAXL];
    for (int ri = 0; ri < l2; ri++) {
        if ((job.fp_rows >> ri) & 1) fp[nfp++] = (uint8_t)ri;
        else in[nint++] = (uint8_t)ri;
    }
    cudaError_t e;
    // the integer rows (one or two of ~25: a few percent of the work at 2.3x the cost per row)
    // run on the side stream beside the FP64 rows instead of as a serial tail
    const bool fork = side && nint && nfp;
    if (nint) {
        KsJob ji = job;
        memcpy(ji.ri_list, in, nint);
        cudaStream_t si = st;
        if (fork) {
            if ((e = cudaEventRecord(side->fork, st)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(side->s, side->fork, 0)) != cudaSuccess) return e;
            si = side->s;
        }
        if ((e = ks_ip5_t<K5_MINB>(ji, tb, nz, nint, si)) != cudaSuccess) return e;
        if (fork && (e = cudaEventRecord(side->join, side->s)) != cudaSuccess) return e;
    }
    if (nfp) {
        memcpy(job.ri_list, fp, nfp);
        // the batch in groups of 8 k / 4 / 2 / 1 ciphertexts, each group in the form that shares a
        // staged key row among all its ciphertexts (10 = 8 + 2, 5 = 4 + 1, 100 = 96 + 4)
        for (int z0 = 0; z0 < nz;) {
            const int rem = nz - z0;
            const int m = rem >= 8 ? rem - rem % 8 : rem >= 4 ? 4 : rem >= 2 ? 2 : 1;
            KsJob sub = job;
            for (int z = 0; z < m; z++) { sub.t1[z] = job.t1[z0 + z]; sub.d[z] = job.d[z0 + z]; sub.acc[z] = job.acc[z0 + z]; }
            sub.nz = m;
            if (m % 8 == 0) e = ks_ip6_t<8, 1, K6_MINB>(sub, tb, nfp, st);
            else if (m == 4) e = ks_ip6_t<4, 1, K6_MINB>(sub, tb, nfp, st);
            else if (m == 2) e = ks_ip6_t<2, 2, K6_MINB>(sub, tb, nfp, st);
            else e = ks_ip6_t<1, 4, K6_MINB>(sub, tb, nfp, st);
            if (e != cudaSuccess) return e;
            z0 += m;
        }
    }
    if (fork) return cudaStreamWaitEvent(st, side->join, 0);
    return cudaSuccess;
}

template <int LOG_M>
static cudaError_t ks_ip_m(KsJob job, const Tables& tb, int nz, cudaStream_t st, const SideStream* side) {
    // M = 256 rows -> ks_ip_256; other row lengths -> k_ks_ip2 (one row per 64-thread CTA,
    // radix-4 phases, two digits interleaved through the FP64 engine with the row's twiddles
    // staged in shared memory, >= 12 CTAs / SM; the special prime's CTAs first)
    if constexpr (LOG_M == 8) {
        return ks_ip_256(job, tb, nz, st, side);
    } else {
        job.ri_list[0] = (uint8_t)job.l1;
        for (int ri = 0; ri < job.l1; ri++) job.ri_list[ri + 1] = (uint8_t)ri;
        return ks_ip2_t<LOG_M, 2, 12>(job, tb, nz, st);
    }
}

cudaError_t launch_ks_ip(const KsJob& job, const Tables& tb, int nz, cudaStream_t st, const SideStream* side) {
    const int lm = tb.log_n - split_m1(tb.log_n);
    switch (lm) {
        case 4: return ks_ip_m<4>(job, tb, nz, st, side);
        case 5: return ks_ip_m<5>(job, tb, nz, st, side);
        case 6: return ks_ip_m<6>(job, tb, nz, st, side);
        case 7: return ks_ip_m<7>(job, tb, nz, st, side);
        case 8: return ks_ip_m<8>(job, tb, nz, st, side);
    }
    return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------------------
// K7: hoisted inner products, CG ciphertexts x R keys per thread-word (one word per thread).
// FP64 output primes (q < 2^50): the multiply-accumulates run on the FP64 pipe as in K4 v6 --
// acc += mulred(D, K), D (< q, the materialised ModUp output, exact u2d) and K (the internal key
// format's centred double, |K| <= q/2): |mulred| <= q/2 + 1.5 2^-52 q^2 / 2 < 0.69 q, so eight
// products fit between re-centrings (|acc| < 6.1 q < 2^53).  Two doubles per accumulator instead of a 128-bit pair: CG = 4, R = 4
// needs 64 accumulator registers (the 128-bit form needed 255 registers, one CTA per SM, and left
// the key stream latency-bound at ~0.4 of HBM), and the FP64 pipe's MAC rate is ~2x the integer
// pipe's (measured: hisa_microbench_mac vs _butterfly_f64).  Integer-engine output primes (60-bit)
// keep the 128-bit integer accumulation.
// ------------------------------------------------------------------------------------------
template <int CG, int R>
__global__ void __launch_bounds__(128) k_ks_ip_hoisted_f64(KsHoistMultiJob job, Tables tb) {
    // each thread's CG D words and 2R key words of digit j + 1 are copied into its own slots of a
    // double-buffered shared stage (cp.async) while digit j is multiplied: ncu of the direct-load
    // form (profiles/r2_ncu_k7_v2.txt) had 61 % of its stall samples on those loads
    constexpr int W = CG + 2 * R;
    extern __shared__ uint64_t k7sm[];                          // [2][W][128]
    const int ri = job.ri_list[blockIdx.y];
    const int l1 = job.l1, l2 = l1 + 1;
    const long long N = 1ll << tb.log_n;
    const long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (x >= N) return;
    const int mi = job.mod_map[ri];
    const double2 qd = tb.modd[mi];
    const double q = qd.x, qinv = qd.y;
    const int tid = threadIdx.x;
    auto issue = [&](int j, int buf) {
        uint64_t* st = k7sm + buf * W * 128 + tid;
#pragma unroll
        for (int c = 0; c < CG; c++) {
            const uint64_t* src = (j == ri) ? job.diag[c] + (long long)j * N + x
                                            : job.D[c] + ((long long)j * l2 + ri) * N + x;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(st + c * 128);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src) : "memory");
        }
#pragma unroll
        for (int k = 0; k < R; k++) {
            const int kL = job.kL[k];
            const long long kstride_p = (long long)(kL + 1) * N;
            const uint64_t* kb = job.key[k] + j * 2 * kstride_p + (long long)(ri < l1 ? ri : kL) * N + x;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(st + (CG + 2 * k) * 128);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(kb) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa + 1024u), "l"(kb + kstride_p)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double acc[CG][R][2];
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++) { acc[c][k][0] = 0.0; acc[c][k][1] = 0.0; }
    issue(0, 0);
    for (int j = 0; j < l1; j++) {
        if (j + 1 < l1) {
            issue(j + 1, (j + 1) & 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        const uint64_t* st = k7sm + (j & 1) * W * 128 + tid;
        double d[CG];
#pragma unroll
        for (int c = 0; c < CG; c++) d[c] = u2d(st[c * 128]);
#pragma unroll
        for (int k = 0; k < R; k++) {
            const double Kb = kd(st[(CG + 2 * k) * 128]), Ka = kd(st[(CG + 2 * k + 1) * 128]);   // internal format
#pragma unroll
            for (int c = 0; c < CG; c++) {
                acc[c][k][0] = __dadd_rn(acc[c][k][0], mulred(d[c], Kb, q, qinv));
                acc[c][k][1] = __dadd_rn(acc[c][k][1], mulred(d[c], Ka, q, qinv));
            }
        }
        if ((j & 7) == 7) {
#pragma unroll
            for (int c = 0; c < CG; c++)
#pragma unroll
                for (int k = 0; k < R; k++) {
                    acc[c][k][0] = redd(acc[c][k][0], q, qinv);
                    acc[c][k][1] = redd(acc[c][k][1], q, qinv);
                }
        }
    }
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                __stcs(&job.acc[c][k][((long long)h * l2 + ri) * N + x], d_canon(acc[c][k][h], q, qinv));
}

template <int CG, int R>
__global__ void __launch_bounds__(256) k_ks_ip_hoisted_multi(KsHoistMultiJob job, const Mod* __restrict__ mods,
                                                             int log_n) {
    const int ri = job.ri_list[blockIdx.y];
    const int l1 = job.l1, l2 = l1 + 1;
    const long long N = 1ll << log_n;
    const long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (x >= N) return;
    const int mi = job.mod_map[ri];
    const Mod md = mods[mi];
    U128 acc[CG][R][2];
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++) { acc[c][k][0] = U128{0, 0}; acc[c][k][1] = U128{0, 0}; }
    for (int j = 0; j < l1; j++) {
        uint64_t d[CG];
#pragma unroll
        for (int c = 0; c < CG; c++) {
            const uint64_t* src = (j == ri) ? job.diag[c] + (long long)j * N + x
                                            : job.D[c] + ((long long)j * l2 + ri) * N + x;
            d[c] = __ldcs(src);
        }
#pragma unroll
        for (int k = 0; k < R; k++) {
            const int kL = job.kL[k];
            const long long kstride_p = (long long)(kL + 1) * N;
            const uint64_t* kb = job.key[k] + j * 2 * kstride_p + (long long)(ri < l1 ? ri : kL) * N + x;
            const uint64_t b = __ldcs(kb), a = __ldcs(kb + kstride_p);
#pragma unroll
            for (int c = 0; c < CG; c++) {
                mac128(acc[c][k][0], d[c], b);
                mac128(acc[c][k][1], d[c], a);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < CG; c++)
#pragma unroll
        for (int k = 0; k < R; k++)
#pragma unroll
            for (int h = 0; h < 2; h++)
                job.acc[c][k][((long long)h * l2 + ri) * N + x] = barrett128(acc[c][k][h].lo, acc[c][k][h].hi, md);
}

cudaError_t launch_ks_ip_hoisted_multi(const KsHoistMultiJob& job_in, int R, const Tables& tb, cudaStream_t st) {
    const long long N = 1ll << tb.log_n;
    KsHoistMultiJob job = job_in;
    const int l2 = job.l1 + 1;
    uint8_t fp[MAXL], in[MAXL];
    int nfp = 0, nint = 0;
    for (int ri = 0; ri < l2; ri++) {
        if ((tb.fp_mods >> job.mod_map[ri]) & 1) fp[nfp++] = (uint8_t)ri;
        else in[nint++] = (uint8_t)ri;
    }
    if (nint) {
        memcpy(job.ri_list, in, nint);
        dim3 grid((unsigned)((N + 255) / 256), nint, 1);
#define C(CGV, RV) if (job.cg == CGV && R == RV) { k_ks_ip_hoisted_multi<CGV, RV><<<grid, 256, 0, st>>>(job, tb.mods, tb.log_n); } else
        C(4, 1) C(4, 2) C(4, 3) C(4, 4) C(2, 1) C(2, 2) C(2, 3) C(2, 4) C(3, 1) C(3, 2) C(3, 3) C(3, 4)
        C(1, 1) C(1, 2) C(1, 3) C(1, 4) return cudaErrorInvalidValue;
#undef C
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (nfp) {
        memcpy(job.ri_list, fp, nfp);
        dim3 grid((unsigned)((N + 127) / 128), nfp, 1);
#define C(CGV, RV) if (job.cg == CGV && R == RV) { \
            k_ks_ip_hoisted_f64<CGV, RV><<<grid, 128, (size_t)2 * (CGV + 2 * RV) * 128 * 8, st>>>(job, tb); } else
        C(4, 1) C(4, 2) C(4, 3) C(4, 4) C(2, 1) C(2, 2) C(2, 3) C(2, 4) C(3, 1) C(3, 2) C(3, 3) C(3, 4)
        C(1, 1) C(1, 2) C(1, 3) C(1, 4) return cudaErrorInvalidValue;
#undef C
    }
    return cudaGetLastError();
}

}  // namespace hisa
